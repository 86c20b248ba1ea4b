for i in 1 2; do
for lib in liblsv.so liblsv_d1.so liblsv_d2.so liblsv_d3.so liblsv_d4.so; do
  echo -n "$lib dyn: "; LSV_DYN_EXPAND=1 LSV_LIB_PATH=paper_2511_22880_b200/$lib timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-extras 2>/dev/null | python tools/ab_summary.py
done
echo -n "static: "; LSV_DYN_EXPAND=0 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-extras 2>/dev/null | python tools/ab_summary.py
done
