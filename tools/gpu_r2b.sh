#!/bin/bash
mkdir -p gpurun_out
TAG=${1:-r2b}
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/build_$TAG.log 2>&1; echo "build+smoke rc=$?"; tail -2 gpurun_out/build_$TAG.log
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|FAILED|Error" gpurun_out/pytest_gpu_$TAG.log | head -20
grep -A60 "parity margins" gpurun_out/pytest_gpu_$TAG.log | head -70
cp gpurun_out/parity_margins.json gpurun_out/parity_margins_$TAG.json 2>/dev/null
for v in "" "--v-bf16" "" "--v-bf16"; do
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline $v > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench $v rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/bench_$TAG.json'))
print('value', round(d['value']), 'ms', round(d['ms_per_step'],3), 'frac', round(d['step_hbm']['frac'],3), 'roof', round(d['roofline']['frac'],3), 'exp_us', round(d['roofline']['launch_us'],1), 'shr_us', round(d['roofline']['shrink']['launch_us'],1))
print('e2e', d['e2e']['value'])"
done
