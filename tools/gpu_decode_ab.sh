#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_forward.py tests/test_gpu_parity.py -q -x -k "decode or simt or forward" 2>&1 | tail -1
for i in 1 2; do for v in 0 1; do
  echo -n "LSV_SIMT_WAIT=$v: "; LSV_SIMT_WAIT=$v timeout 600 python bench.py --config decode --steps 10 --warmup 3 --no-cpu-baseline --no-extras 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step'],3), 'serial', round(d['serial_step']['ms_per_step'],3), 'frac', round(d['step_hbm']['frac'],3))"
done; done
