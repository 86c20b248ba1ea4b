python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
python tools/trace_cta.py shrink:0 expand:4 expand:0 2>&1 | grep -E "==|loop GB|loop_done|reduce_done"
python bench.py --steps 10 --warmup 3 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['launch_us'], d['roofline']['shrink'])"
