#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
echo "== with LoRA stages"; timeout 300 python tools/fused_parts.py
echo "== LSV_DEBUG_FUSED=1 (bare GEMM)"; LSV_DEBUG_FUSED=1 timeout 300 python tools/fused_parts.py
