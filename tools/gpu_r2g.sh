#!/bin/bash
mkdir -p gpurun_out
TAG=${1:-r2g}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
if timeout 300 python tools/prof_fused.py 2 > gpurun_out/prof_fused_$TAG.log 2>&1; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fused" -s 2 -c 1 \
    -o gpurun_out/fused_full_$TAG -f python tools/prof_fused.py 2 > gpurun_out/ncu_fused_$TAG.log 2>&1
  echo "ncu rc=$?"
fi
