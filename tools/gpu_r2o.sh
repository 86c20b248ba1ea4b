#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 300 python tools/trace_fused.py 0
echo "== dbg 1"; LSV_DEBUG_FUSED=1 timeout 300 python tools/trace_fused.py 0 | head -40
