#!/bin/bash
# Runs one fixture case per process under each tier / kernel path (a failing kernel poisons its context).
mkdir -p gpurun_out
for lib in liblsv.so liblsv_checked.so; do for gk in 1 0; do for tier in 0 2; do
  echo -n "$lib group_kernel=$gk tier=$tier: "
  LSV_LIB_PATH=paper_2511_22880_b200/$lib LSV_GROUP_KERNEL=$gk timeout 120 python -c "
import sys; sys.path.insert(0, 'tests'); sys.path.insert(0, '.')
from _cases import fixture_case
c = fixture_case('${CASE:-rank_256}')
y, bp = c.run_gpu(tier_policy=$tier)
print('ok', float(y.float().abs().max()))
" 2>&1 | grep -E "^ok|check failed|Error" | head -3
done; done; done
