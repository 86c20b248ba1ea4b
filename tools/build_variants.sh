#!/bin/bash
# Builds A/B variants of liblsv.so: tools/build_variants.sh "o1:-DX=1 -DY=2" "o2:-DZ=3" ... -> liblsv_o1.so ...
# (then rebuilds the default library)
set -e
cd "$(dirname "$0")/.."
for spec in "$@"; do
  name=${spec%%:*}; defs=${spec#*:}
  LSV_NVCC_DEFINES="$defs" python -c "from paper_2511_22880_b200 import build; build.build(force=True)"
  cp paper_2511_22880_b200/liblsv.so paper_2511_22880_b200/liblsv_$name.so
  echo "built liblsv_$name.so ($defs)"
done
python -c "from paper_2511_22880_b200 import build; build.build(force=True)"
