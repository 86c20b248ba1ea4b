#!/bin/bash
# A/B of library builds on the same box, alternating: tools/gpu_ab_lib.sh "liblsv.so liblsv_prev.so" [bench args]
LIBS=$1; shift
for i in 1 2; do for lib in $LIBS; do
  echo -n "$lib: "; LSV_LIB_PATH=paper_2511_22880_b200/$lib timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-extras "$@" 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step'],3), 'serial', round(d['serial_step']['ms_per_step'],3), 'expand', round(d['roofline']['launch_us'],1), 'shrink', round(d['roofline']['shrink']['launch_us'],1))"
done; done
