#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_fused.py -q -x 2>&1 | tail -2
timeout 300 python tools/fused_parts.py
