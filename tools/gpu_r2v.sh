#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -k "decode or simt or SIMT or fixtures or forward or 1-" > gpurun_out/pytest_dec.log 2>&1; echo "pytest rc=$?"; grep -E "passed|failed|Error|assert" gpurun_out/pytest_dec.log | head -10
for f in 1 0; do
LSV_DECODE_FUSED=$f timeout 600 python bench.py --config decode --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_decode_f$f.json 2> gpurun_out/bench_decode_f$f.err; echo "decode fused=$f rc=$?"; tail -2 gpurun_out/bench_decode_f$f.err
python -c "
import json; d=json.load(open('gpurun_out/bench_decode_f$f.json'))
print('value', round(d['value']), 'ms', round(d['ms_per_step'],3), 'frac', round(d['step_hbm']['frac'],3), 'moved_frac', round(d['step_hbm']['moved_frac'],3), 'serial', round(d['serial_step']['ms_per_step'],3))"
done
