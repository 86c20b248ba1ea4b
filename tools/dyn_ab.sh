for i in 1 2; do
for cfg in "LSV_DYN_EXPAND=0" "LSV_DYN_EXPAND=1 LSV_DYN_ORDER=0" "LSV_DYN_EXPAND=1 LSV_DYN_ORDER=1" "LSV_DYN_EXPAND=1 LSV_DYN_ORDER=2"; do
  echo -n "$cfg: "; env $cfg timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-extras 2>/dev/null | python tools/ab_summary.py
done; done
