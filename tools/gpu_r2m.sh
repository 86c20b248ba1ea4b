#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for d in 0 1 2 4 6 8; do echo "== LSV_DEBUG_FUSED=$d"; LSV_DEBUG_FUSED=$d timeout 300 python tools/fused_parts.py 2>&1 | cut -c1-130; done
