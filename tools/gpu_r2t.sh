#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests -m multigpu -q > gpurun_out/pytest_multi2.log 2>&1; echo "multigpu pytest rc=$?"; tail -3 gpurun_out/pytest_multi2.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --config remote --steps 10 --warmup 3 > gpurun_out/remote2.log 2>&1; echo "remote rc=$?"
grep "^{" gpurun_out/remote2.log > gpurun_out/remote2.json; python -c "
import json; d=json.load(open('gpurun_out/remote2.json'))
print('direct', d['ms_per_step'], 'overhead', round(d['remote_overhead'],3), 'plain', d['remote_plain_plan'], 'prefetch', d['remote_prefetch']['ms_per_step'], 'local', d['all_local'], d['batch_shape'])
print({k: (v.get('sm_mhz'), v.get('reasons')) for k, v in d['clocks_per_arm'].items()})"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/dp2.log 2>&1; echo "dp2 rc=$?"; grep "^{" gpurun_out/dp2.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('DP2', round(d['value']), d['ms_per_step'], d['config']['per_gpu'], d['step_hbm']['frac'])"
