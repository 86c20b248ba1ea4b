#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for t in auto simt; do
timeout 600 python bench.py --config decode --tier $t --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_decode_$t.json 2> gpurun_out/bench_decode_$t.err; echo "decode $t rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/bench_decode_$t.json'))
print('value', round(d['value']), 'ms', round(d['ms_per_step'],3), 'frac', round(d['step_hbm']['frac'],3), 'moved_frac', round(d['step_hbm']['moved_frac'],3), 'serial', round(d['serial_step']['ms_per_step'],3))"
done
timeout 1200 python tools/measure_cost_fit.py --out gpurun_out/b200_delta_cost.json > gpurun_out/cost_fit.log 2>&1; echo "cost fit rc=$?"; tail -2 gpurun_out/cost_fit.log
