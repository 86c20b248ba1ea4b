# A/B: bench of library builds on the same box, alternating
for i in 1 2; do
for lib in ${AB_LIBS:-liblsv.so liblsv_ww.so}; do
  echo -n "$lib: "; LSV_LIB_PATH=paper_2511_22880_b200/$lib python bench.py --steps 10 --warmup 3 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step'],3), 'expand', round(d['roofline']['launch_us'],1), 'shrink', round(d['roofline']['shrink']['launch_us'],1))"
done; done
