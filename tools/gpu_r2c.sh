#!/bin/bash
mkdir -p gpurun_out
TAG=${1:-r2c}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
for v in "" "--v-bf16"; do
timeout 900 python bench.py --steps 10 --warmup 3 $v > gpurun_out/bench_${TAG}$v.json 2> gpurun_out/bench_${TAG}$v.err; echo "bench $v rc=$?"; tail -3 gpurun_out/bench_${TAG}$v.err
python -c "
import json; d=json.load(open('gpurun_out/bench_${TAG}$v.json'))
print('value', round(d['value']), 'ms', round(d['ms_per_step'],3), 'frac', round(d['step_hbm']['frac'],3), 'roof', round(d['roofline']['frac'],3), 'exp_us', round(d['roofline']['launch_us'],1), 'shr_us', round(d['roofline']['shrink']['launch_us'],1))
print('serial', d['serial_step']); print('e2e', d['e2e']['value']); print('dp1', d.get('dp_like_for_like')); print('c1', d.get('c1')); print('cpu', d.get('cpu_baseline'))"
done
timeout 900 python tools/tier_sweep.py time > gpurun_out/tier_sweep_time.json 2> gpurun_out/tier_sweep_time.err; echo "sweep rc=$?"; tail -2 gpurun_out/tier_sweep_time.err
if [ -s gpurun_out/tier_sweep_time.json ]; then
timeout 1500 ncu --metrics gpu__time_duration.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none -k regex:"tc_kernel|simt_" --csv --log-file gpurun_out/tier_ncu.csv python tools/tier_sweep.py ncu > gpurun_out/tier_ncu.log 2>&1; echo "ncu rc=$?"
python tools/tier_sweep.py report gpurun_out/tier_sweep_time.json gpurun_out/tier_ncu.csv > gpurun_out/tier_sweep.txt 2>&1; echo "report rc=$?"
fi
