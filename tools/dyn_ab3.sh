for i in 1 2 3; do
for cfg in "liblsv_t0.so 1" "liblsv.so 1" "liblsv.so 3" "liblsv_t0.so 3"; do
  set -- $cfg
  echo -n "$1 order $2: "; LSV_DYN_ORDER=$2 LSV_LIB_PATH=paper_2511_22880_b200/$1 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-extras 2>/dev/null | python tools/ab_summary.py
done; done
