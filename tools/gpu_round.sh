#!/bin/bash
# One GPU batch: parity suite, bench (both arms), ncu launch list of one bench step, one full
# ncu capture of the top kernels.  Every ncu command runs only after the same command exited 0.
set -x
mkdir -p gpurun_out
TAG=${1:-r1}
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu_$TAG.log
timeout 600 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_$TAG.json 2>gpurun_out/bench_ref_$TAG.err; echo "ref rc=$?"
if timeout 300 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/bench_small_$TAG.json 2>&1; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"tc_kernel|simt_|vimg" -c 700 --csv \
    --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch_$TAG.log 2>&1
  echo "ncu launches rc=$?"
fi
if timeout 300 python tools/prof_one.py 2 > gpurun_out/prof_one_$TAG.log 2>&1; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"tc_kernel|simt_" -s 4 -c 2 \
    -o gpurun_out/full_$TAG -f python tools/prof_one.py 2 > gpurun_out/ncu_full_$TAG.log 2>&1
  echo "ncu full rc=$?"
fi
lscpu | head -20 > gpurun_out/lscpu_$TAG.txt
