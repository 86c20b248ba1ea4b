#!/bin/bash
# A/B of an environment knob on the C2 bench, alternating: tools/gpu_ab_env.sh VAR "v1 v2" [extra bench args]
VAR=$1; VALS=$2; shift 2
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for i in 1 2; do for v in $VALS; do
  echo -n "$VAR=$v: "; env $VAR=$v timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-extras "$@" 2>/dev/null | python tools/ab_summary.py
done; done
