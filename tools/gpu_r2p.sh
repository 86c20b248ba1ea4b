#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 300 python tools/fused_parts.py
echo "== v bf16"; timeout 300 python tools/fused_only.py --v-bf16 | grep -E "ms_per_layer|speedup|overhead"
echo "== v split"; timeout 300 python tools/fused_only.py | grep -E "ms_per_layer|speedup|overhead"
