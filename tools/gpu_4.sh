#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
for pad in "" "--tp-padded"; do
timeout 900 $R --master-port 29613 bench.py --gpus 4 --config tp --steps 3 --warmup 2 $pad > gpurun_out/tp4$pad.log 2>&1; echo "tp4 $pad rc=$?"
grep "^{" gpurun_out/tp4$pad.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('TP4', d['config']['shards'], round(d['value']), round(d['ms_per_step'],2), 'nccl', round(d['nccl_ms_per_step'],2), 'hbm frac', round(d['step_hbm']['frac'],3))"
done
timeout 900 $R --master-port 29614 bench.py --gpus 4 --steps 10 --warmup 3 > gpurun_out/dp4.log 2>&1; echo "dp4 rc=$?"
grep "^{" gpurun_out/dp4.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('DP4', round(d['value']), round(d['ms_per_step'],3), [round(p['ms'],2) for p in d['config']['per_gpu']], 'frac', round(d['step_hbm']['frac'],3), 'e2e', round(d['e2e']['value']))"
timeout 900 $R --master-port 29615 bench.py --gpus 4 --config remote --steps 10 --warmup 3 > gpurun_out/remote4.log 2>&1; echo "remote4 rc=$?"
grep "^{" gpurun_out/remote4.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('REMOTE4', d['ms_per_step'], 'overhead', round(d['remote_overhead'],3), 'local', d['all_local']['ms_per_step'], 'split', d['remote_split']['by_remote_sms'], 'batch', d['batch_shape'])"
timeout 900 $R --master-port 29616 bench.py --gpus 4 --config c3 --steps 10 --warmup 3 > gpurun_out/c3x4.log 2>&1; echo "c3x4 rc=$?"
grep "^{" gpurun_out/c3x4.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C3x4', round(d['value']), round(d['ms_per_step'],3), [round(p['ms'],2) for p in d['config']['per_gpu']], 'frac', round(d['step_hbm']['frac'],3))"
timeout 600 python -m pytest tests -m multigpu -q > gpurun_out/pytest_multi4.log 2>&1; echo "multigpu pytest (4 GPUs) rc=$?"; tail -1 gpurun_out/pytest_multi4.log
