#!/bin/bash
# 4-GPU box on the final kernels: the GPU suite (multi-GPU tests included), DP4, C3x4, remote x4, TP4.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_4gpu.log 2>&1; echo "pytest (4 GPUs) rc=$?"; tail -1 gpurun_out/pytest_4gpu.log
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 900 $R --master-port 29614 bench.py --gpus 4 --steps 10 --warmup 3 > gpurun_out/dp4.log 2>&1; echo "dp4 rc=$?"
grep "^{" gpurun_out/dp4.log > gpurun_out/bench_dp4.json
python -c "import json; d=json.load(open('gpurun_out/bench_dp4.json')); print('DP4', round(d['value']), round(d['ms_per_step'],3), [round(p['ms'],2) for p in d['config']['per_gpu']], 'frac', round(d['step_hbm']['frac'],3), 'e2e', round(d['e2e']['value']))"
timeout 900 $R --master-port 29616 bench.py --gpus 4 --config c3 --steps 10 --warmup 3 > gpurun_out/c3x4.log 2>&1; echo "c3x4 rc=$?"
grep "^{" gpurun_out/c3x4.log > gpurun_out/bench_c3x4.json
python -c "import json; d=json.load(open('gpurun_out/bench_c3x4.json')); print('C3x4', round(d['value']), round(d['ms_per_step'],3), [round(p['ms'],2) for p in d['config']['per_gpu']], 'frac', round(d['step_hbm']['frac'],3))"
timeout 900 $R --master-port 29615 bench.py --gpus 4 --config remote --steps 10 --warmup 3 > gpurun_out/remote4.log 2>&1; echo "remote4 rc=$?"
grep "^{" gpurun_out/remote4.log > gpurun_out/bench_remote4.json
python -c "import json; d=json.load(open('gpurun_out/bench_remote4.json')); print('REMOTE4', round(d['ms_per_step'],3), 'overhead', round(d['remote_overhead'],3), 'local', round(d['all_local']['ms_per_step'],3), 'nvlink_aware', round(d['remote_nvlink_aware_plan']['ms_per_step'],3))"
timeout 900 $R --master-port 29613 bench.py --gpus 4 --config tp --steps 3 --warmup 2 --tp-adapters 500 > gpurun_out/tp4.log 2>&1; echo "tp4 rc=$?"
grep "^{" gpurun_out/tp4.log > gpurun_out/bench_tp4.json
python -c "import json; d=json.load(open('gpurun_out/bench_tp4.json')); print('TP4', round(d['value']), round(d['ms_per_step'],2), 'nccl', round(d['nccl_ms_per_step'],2), 'hbm frac', round(d['step_hbm']['frac'],3))"
