#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_r2w.log 2>&1; echo "suite rc=$?"; grep -E "passed|failed|FAILED" gpurun_out/pytest_gpu_r2w.log | head
bash tools/gpu_checked.sh
