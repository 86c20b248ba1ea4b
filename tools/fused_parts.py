"""Per-group timing of the fused linear's parts (development): cuBLAS GEMMs, the shrink of the
tile-aligned plan, the fused kernel without the shrink, and the same with LSV_DEBUG_FUSED=1 (no
LoRA stages: the bare GEMM).  python tools/fused_parts.py"""
import os
import sys
import zlib
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2511_22880_b200 import native, synth  # noqa: E402
from paper_2511_22880_b200.lora import LoraDeltaEngine  # noqa: E402
from paper_2511_22880_b200.shapes import ModelShape  # noqa: E402
from paper_2511_22880_b200.slab import AdapterSlab  # noqa: E402
import ctypes  # noqa: E402

wl = synth.c2_llama2_7b()
model = ModelShape("l7b-1l", 1, wl.model.projections)
dev = torch.device("cuda:0")
slab = AdapterSlab(model, AdapterSlab.capacity_for(model, wl.ranks), dev)
for aid, r in zip(wl.adapter_ids, wl.ranks):
    slab.fill_random(slab.allocate(aid, r), 1000 + zlib.crc32(aid.encode()) % 100000)
eng = LoraDeltaEngine(slab, v_bf16="--v-bf16" in sys.argv)
bp = eng.prepare(wl.segments, fused_linear=True)
N = wl.segments.num_tokens
S = wl.segments.num_segments


def timeit(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


for gi, (gname, members) in enumerate(eng.groups):
    pr0 = model.projections[members[0]]
    x = torch.randn(N, pr0.h_in, device=dev).to(torch.bfloat16)
    ws = [(torch.randn(model.projections[p].h_out, pr0.h_in, device=dev) / 64).to(torch.bfloat16) for p in members]
    ys = [torch.empty(N, model.projections[p].h_out, device=dev, dtype=torch.bfloat16) for p in members]
    gp = bp.group_plans[gi]
    P = len(model.projections)
    arr = lambda t, v: (t * len(v))(*v)   # noqa: E731
    wa, lw = arr(ctypes.c_void_p, [w.data_ptr() for w in ws]), arr(ctypes.c_int64, [w.stride(0) for w in ws])
    ya, ly = arr(ctypes.c_void_p, [y.data_ptr() for y in ys]), arr(ctypes.c_int64, [y.stride(0) for y in ys])
    ba = arr(ctypes.c_void_p, [bp.b_ptrs.data_ptr() + p * S * 8 for p in members])

    def fused_only():
        native.check(native.lib().lsv_lora_fused_linear(
            x.data_ptr(), x.stride(0), N, gp.h_in, None, ctypes.addressof(wa), ctypes.addressof(lw),
            ctypes.addressof(ya), ctypes.addressof(ly), ctypes.addressof(ba), gp.plan_dev.data_ptr(),
            gp.plan_host.ctypes.data, bp.workspace.data_ptr(), bp.workspace.numel(), torch.cuda.current_stream().cuda_stream))

    t_cublas = timeit(lambda: [torch.matmul(x, w.t(), out=y) for w, y in zip(ws, ys)])
    t_shrink = timeit(lambda: eng.shrink(bp, 0, members[0], x))
    t_fused = timeit(fused_only)
    t_all = timeit(lambda: eng.linear_group(bp, 0, gi, x, ws, ys))
    flops = sum(2 * N * pr0.h_in * model.projections[p].h_out for p in members)
    print(f"{gname:9s} cublas {t_cublas:8.1f} us ({flops / t_cublas / 1e6:6.0f} TF/s)  shrink {t_shrink:6.1f}  "
          f"fused-kernel {t_fused:8.1f} ({flops / t_fused / 1e6:6.0f} TF/s)  linear_group {t_all:8.1f}  "
          f"pieces {gp.summary[5]}", flush=True)
