#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for d in 0 1; do
LSV_DEBUG_FUSED=$d timeout 600 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed,sm__pipe_tc_cycles_active.avg,sm__cycles_elapsed.avg,sm__inst_executed_pipe_uniform.sum,smsp__inst_executed_op_utcmma.sum,l1tex__data_pipe_tc_wavefronts_mem_shared.sum,lts__throughput.avg.pct_of_peak_sustained_elapsed \
  --clock-control none -k regex:"fused" -s 2 -c 1 python tools/prof_fused.py 0 2>&1 | grep -E "gpu__|sm__|smsp|l1tex|lts__" | sed "s/^/dbg$d /"
done
