python bench.py --steps 10 --warmup 3 --no-cpu-baseline | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('value', round(d['value']), 'ms', round(d['ms_per_step'],3), 'frac', round(d['step_hbm']['frac'],3), 'moved_frac', round(d['step_hbm'].get('moved_frac',0),3))
print('expand', round(d['roofline']['launch_us'],1), 'shrink', d['roofline']['shrink'])
print('e2e', d['e2e']['value'], 'launches', d['gpu_launches'])"
python tools/trace_cta.py shrink:0 shrink:4 shrink:3 shrink:6 2>&1 | grep -E "==|loop GB|loop_done|reduce_done"
