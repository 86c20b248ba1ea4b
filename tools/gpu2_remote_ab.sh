#!/bin/bash
# 2-GPU remote (C4) A/B: the headline bytes-only plan vs the NVLink-aware plan (remote flags: dynamic
# dispatch merges peer and local expand items), with the LPT remote weight 7 (default) and 1.
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
for w in 7 1; do for i in 1 2; do
  LSV_REMOTE_WEIGHT=$w timeout 900 $R --master-port $((29600 + w * 10 + i)) bench.py --gpus 2 --config remote --steps 10 --warmup 3 > gpurun_out/remote_w$w.log 2>&1
  grep "^{" gpurun_out/remote_w$w.log | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('weight $w: bytes-only', round(d['ms_per_step'],3), 'nvlink-aware', round(d['remote_nvlink_aware_plan']['ms_per_step'],3), 'local', round(d['all_local']['ms_per_step'],3))"
done; done
