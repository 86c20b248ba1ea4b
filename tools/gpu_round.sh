#!/bin/bash
# One GPU batch: parity suite (production and device-checked builds), bench (both arms), ncu launch
# list of one bench step, full ncu captures of the top kernels.  Every ncu command runs only after
# the same command exited 0 without ncu.
mkdir -p gpurun_out
TAG=${1:-r2}
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "build+smoke rc=$?"; tail -1 gpurun_out/smoke_$TAG.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed" gpurun_out/pytest_gpu_$TAG.log | tail -1
cp gpurun_out/parity_margins.json gpurun_out/parity_margins_$TAG.json 2>/dev/null
bash tools/gpu_checked.sh
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_$TAG.json 2>gpurun_out/bench_ref_$TAG.err; echo "ref rc=$?"
timeout 600 python bench.py --config decode --steps 10 --warmup 3 --no-cpu-baseline --no-extras > gpurun_out/bench_decode_$TAG.json 2>&1; echo "decode rc=$?"
if timeout 300 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-extras > gpurun_out/bench_small_$TAG.json 2>&1; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"tc_kernel|simt_|vimg" -c 700 --csv \
    --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-extras > gpurun_out/ncu_launch_$TAG.log 2>&1
  echo "ncu launches rc=$?"
fi
if timeout 300 python tools/prof_one.py 2 > gpurun_out/prof_one_$TAG.log 2>&1; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"tc_kernel|simt_" -s 4 -c 2 \
    -o gpurun_out/full_$TAG -f python tools/prof_one.py 2 > gpurun_out/ncu_full_$TAG.log 2>&1
  echo "ncu full rc=$?"
fi
if timeout 300 python tools/prof_group.py > gpurun_out/prof_group_$TAG.log 2>&1; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:group -s 3 -c 1 \
    -o gpurun_out/group_full_$TAG -f python tools/prof_group.py > gpurun_out/ncu_group_$TAG.log 2>&1
  echo "ncu layer kernel rc=$?"
  LSV_LAYER_KERNEL=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:group -s 12 -c 4 \
    -o gpurun_out/group4_full_$TAG -f python tools/prof_group.py > gpurun_out/ncu_group4_$TAG.log 2>&1
  echo "ncu group kernels rc=$?"
fi
timeout 300 python tools/timeline_step.py 4 > gpurun_out/timeline_$TAG.txt 2>&1; echo "timeline rc=$?"
if timeout 300 python tools/prof_fused.py 0 > gpurun_out/prof_fused_$TAG.log 2>&1; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fused" -s 2 -c 1 \
    -o gpurun_out/fused_full_$TAG -f python tools/prof_fused.py 0 > gpurun_out/ncu_fused_$TAG.log 2>&1
  echo "ncu fused rc=$?"
fi
lscpu | head -20 > gpurun_out/lscpu_$TAG.txt
python -c "
import json; d=json.load(open('gpurun_out/bench_$TAG.json'))
print('value', round(d['value']), 'ms', round(d['ms_per_step'],3), 'frac', round(d['step_hbm']['frac'],3), 'roof', round(d['roofline']['frac'],3), d['roofline']['kernel'])
print('serial', d['serial_step']['ms_per_step'], 'e2e', round(d['e2e']['value']), 'cpu', d['cpu_baseline']['value'])
print('dp1', round(d['dp_like_for_like']['value']), 'c1 us', round(d['c1']['us_per_call'],2), 'fused', d['fused_linear']['fused']['ms_per_layer'], d['fused_linear']['separate']['ms_per_layer'], d['fused_linear']['base']['ms_per_layer'])"
