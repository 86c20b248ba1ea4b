#!/bin/bash
# A/B of library builds on the decode config, alternating: tools/gpu_decode_lib_ab.sh "liblsv.so liblsv_x.so"
LIBS=$1
timeout 600 python -m pytest tests/test_gpu_forward.py tests/test_gpu_parity.py -q -x -k "decode or simt or forward" 2>&1 | tail -1
for i in 1 2 3; do for lib in $LIBS; do
  echo -n "$lib: "; LSV_LIB_PATH=paper_2511_22880_b200/$lib timeout 600 python bench.py --config decode --steps 10 --warmup 3 --no-cpu-baseline --no-extras 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(round(d['value']), round(d['ms_per_step'],3), 'serial', round(d['serial_step']['ms_per_step'],3), 'frac', round(d['step_hbm']['frac'],3), 'exp', round(r['launch_us'],1), 'shr', round(r['shrink']['launch_us'],1))"
done; done
