#!/bin/bash
# Round-2 first GPU batch: GPU parity (incl. the SGMV fixtures), sanitizers, quick bench.
mkdir -p gpurun_out
TAG=${1:-r2a}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"
tail -40 gpurun_out/pytest_gpu_$TAG.log
cp gpurun_out/parity_margins.json gpurun_out/parity_margins_$TAG.json 2>/dev/null
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck synccheck; do
  timeout 900 $CS --tool $tool --error-exitcode 9 python tools/sanitize_cases.py c1 splitk fwd_tc fwd_simt decode \
    > gpurun_out/sanitizer_${tool}_$TAG.txt 2>&1; echo "$tool rc=$?"; tail -4 gpurun_out/sanitizer_${tool}_$TAG.txt
done
timeout 900 $CS --tool racecheck --racecheck-report all --error-exitcode 9 python tools/sanitize_cases.py c1 fwd_tc fwd_simt decode \
  > gpurun_out/sanitizer_racecheck_$TAG.txt 2>&1; echo "racecheck rc=$?"; tail -4 gpurun_out/sanitizer_racecheck_$TAG.txt
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/bench_$TAG.json'))
print('value', round(d['value']), 'ms', round(d['ms_per_step'],3), 'frac', round(d['step_hbm']['frac'],3), 'roof', round(d['roofline']['frac'],3), 'exp_us', round(d['roofline']['launch_us'],1))
print('e2e', d['e2e']['value'])"
