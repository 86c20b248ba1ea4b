#!/bin/bash
mkdir -p gpurun_out
TAG=${1:-r2d}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
timeout 600 python -m pytest tests/test_gpu_fused.py -q -x > gpurun_out/pytest_fused_$TAG.log 2>&1; echo "fused pytest rc=$?"
grep -E "passed|failed|Error|assert" gpurun_out/pytest_fused_$TAG.log | head -20
grep -A12 "parity margins" gpurun_out/pytest_fused_$TAG.log
timeout 600 python tools/fused_only.py > gpurun_out/fused_$TAG.json 2> gpurun_out/fused_$TAG.err; echo "fused bench rc=$?"; cat gpurun_out/fused_$TAG.json; tail -5 gpurun_out/fused_$TAG.err
if [ "$2" == "prof" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fused" -s 2 -c 1 \
    -o gpurun_out/fused_full_$TAG -f python tools/prof_fused.py 2 > gpurun_out/ncu_fused_$TAG.log 2>&1
  echo "ncu rc=$?"
fi
