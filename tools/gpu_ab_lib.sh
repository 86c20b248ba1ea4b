#!/bin/bash
# A/B of library builds on the same box, alternating: tools/gpu_ab_lib.sh "liblsv.so liblsv_prev.so" [bench args]
LIBS=$1; shift
for i in 1 2; do for lib in $LIBS; do
  echo -n "$lib: "; LSV_LIB_PATH=paper_2511_22880_b200/$lib timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-extras "$@" 2>/dev/null | python tools/ab_summary.py
done; done
