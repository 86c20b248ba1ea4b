#!/bin/bash
# 2-GPU box: multi-GPU tests, DP2 (and its reference arm), remote (C4), TP2 on the current kernels.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_2gpu.log 2>&1; echo "pytest (2 GPUs) rc=$?"; tail -1 gpurun_out/pytest_2gpu.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/dp2.log 2>&1; echo "dp2 rc=$?"
grep "^{" gpurun_out/dp2.log > gpurun_out/bench_dp2.json
python -c "import json; d=json.load(open('gpurun_out/bench_dp2.json')); print('DP2', round(d['value']), round(d['ms_per_step'],3), [round(p['ms'],2) for p in d['config']['per_gpu']], 'hbm', round(d['step_hbm']['frac'],3), 'e2e', round(d['e2e']['value']))"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --config remote --steps 10 --warmup 3 > gpurun_out/remote2.log 2>&1; echo "remote rc=$?"
grep "^{" gpurun_out/remote2.log > gpurun_out/bench_remote2.json
python -c "
import json; d=json.load(open('gpurun_out/bench_remote2.json'))
print('remote', round(d['value']), round(d['ms_per_step'],3), {k: v for k, v in d.items() if 'remote' in k or 'local' in k})" | cut -c 1-1200
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 2 --config tp --steps 3 --warmup 2 --tp-adapters 200 > gpurun_out/tp2.log 2>&1; echo "tp2 rc=$?"
grep "^{" gpurun_out/tp2.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('TP2', round(d['value']), round(d['ms_per_step'],2), 'nccl', round(d['nccl_ms_per_step'],2), 'hbm frac', round(d['step_hbm']['frac'],3))"
