#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests -m multigpu -q > gpurun_out/pytest_multi_tp.log 2>&1; echo "multigpu pytest rc=$?"; tail -3 gpurun_out/pytest_multi_tp.log
for pad in "" "--tp-padded"; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 2 --config tp --steps 3 --warmup 2 --tp-adapters 200 $pad > gpurun_out/tp2$pad.log 2>&1; echo "tp2 $pad rc=$?"
grep "^{" gpurun_out/tp2$pad.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('TP2', d['config']['shards'], round(d['value']), round(d['ms_per_step'],2), 'nccl', round(d['nccl_ms_per_step'],2), 'hbm frac', round(d['step_hbm']['frac'],3))"
done
