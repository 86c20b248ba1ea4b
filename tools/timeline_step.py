"""Per-SM timeline of a multi-layer lsv_lora_forward (C2 shapes, L layers -> L layer kernels, or 4L
group kernels with LSV_LAYER_KERNEL=0):
when each launch's CTA enters, finishes its setup and exits on every SM, and how much SM time
the launch boundaries cost (exit of one CTA -> entry of the next on the same SM, plus setup).
    python tools/timeline_step.py [layers=4]"""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, '.')
from paper_2511_22880_b200 import native  # noqa: E402
from paper_2511_22880_b200.lora import LoraDeltaEngine  # noqa: E402
from paper_2511_22880_b200.segments import index_tokens  # noqa: E402
from paper_2511_22880_b200.shapes import LLAMA2_7B, ModelShape  # noqa: E402
from paper_2511_22880_b200.slab import AdapterSlab  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 4
model = ModelShape("l7b", L, LLAMA2_7B.projections)
dev = torch.device("cuda:0")
ranks = [8] * 44 + [16] * 22 + [32] * 14 + [64] * 11 + [128] * 9
slab = AdapterSlab(model, AdapterSlab.capacity_for(model, ranks), dev)
for i, r in enumerate(ranks):
    slab.fill_random(slab.allocate(f"a{i}", r), 1000 + i)
seg = index_tokens(np.random.default_rng(0).integers(0, 100, 4096), ranks)
eng = LoraDeltaEngine(slab)
bp = eng.prepare(seg)
xs = [{g: torch.randn(4096, model.projections[m[0]].h_in, device=dev).to(torch.bfloat16) for g, m in eng.groups}
      for _ in range(L)]
ys = [{p.name: torch.zeros(4096, p.h_out, device=dev, dtype=torch.bfloat16) for p in model.projections} for _ in range(L)]
for _ in range(3):
    eng.forward(bp, xs, ys)
torch.cuda.synchronize()
n = 4 * L
buf = torch.zeros(n * 148 * 16, dtype=torch.int64, device=dev)
lib = native.lib()
lib.lsv_debug_set_trace.argtypes = [ctypes.c_void_p, ctypes.c_int32]
lib.lsv_debug_set_trace(buf.data_ptr(), -n)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
import os
if os.environ.get("TL_GRAPH"):   # the step as bench.py runs it: one CUDA graph replay
    st = torch.cuda.Stream()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=st):
        eng.forward(bp, xs, ys, st)
    lib.lsv_debug_set_trace(None, 0)
    with torch.cuda.stream(st):
        graph.replay()          # warm
        torch.cuda.synchronize()
        buf.zero_()
        e0.record(st)
        graph.replay()
        e1.record(st)
    torch.cuda.synchronize()
else:
    e0.record()
    eng.forward(bp, xs, ys)
    e1.record()
    torch.cuda.synchronize()
lib.lsv_debug_set_trace(None, 0)
tl = buf.view(n, 148, 16).cpu().numpy().astype(np.int64)
n = int((tl[:, :, 0].max(axis=1) > 0).sum())   # launches recorded: 4L group kernels or L layer kernels
tl = tl[:n]
t0 = tl[:, :, 0][tl[:, :, 0] > 0].min()
kind = "group kernels" if n == 4 * L else "layer kernels"
print(f"{L} layers, {n} {kind}: {e0.elapsed_time(e1) * 1e3:.0f} us (events); per launch (us from first entry):")
names = [g for g, _ in eng.groups] * L if n == 4 * L else [f"layer {i}" for i in range(n)]
for i in range(n):
    ent, setup, ext = (tl[i, :, 0] - t0) / 1e3, (tl[i, :, 1] - tl[i, :, 0]) / 1e3, (tl[i, :, 2] - t0) / 1e3
    print(f"  {i:2d} {names[i]:9s} entry {ent.min():7.1f}..{ent.max():7.1f}  setup p50 {np.median(setup):4.2f}  "
          f"exit {ext.min():7.1f}..{ext.max():7.1f}")
# per SM: gaps between one launch's exit and the next launch's entry on the same SM
gaps, busy = [], 0.0
span = (tl[:, :, 2].max() - t0) / 1e3
for sm in range(148):
    iv = []
    for i in range(n):
        for c in range(148):
            if tl[i, c, 3] == sm and tl[i, c, 0] > 0:
                iv.append(((tl[i, c, 0] - t0) / 1e3, (tl[i, c, 1] - t0) / 1e3, (tl[i, c, 2] - t0) / 1e3))
    iv.sort()
    for a, b in zip(iv, iv[1:]):
        gaps.append(b[0] - a[2])
    busy += sum(x[2] - x[1] for x in iv)
gaps = np.array(gaps)
print(f"exit -> next entry on the same SM: mean {gaps.mean():.2f} us, p50 {np.median(gaps):.2f}, p90 {np.percentile(gaps, 90):.2f}; "
      f"SM time past setup / span: {busy / (148 * span) * 100:.1f}%")

if kind == "layer kernels":   # phase ends inside each layer kernel (epilogue warp 0 of every CTA)
    import os
    la = int(os.environ.get("LSV_PHASE_LOOKAHEAD", "3"))   # lsv_tc.cuh group_tc_kernel phase_of
    names4 = ["attn_in", "attn_out", "mlp_in", "mlp_mid"]
    npre, order = min(4, max(la, 1) + 1), []
    for i in range(8):
        if i < npre:
            order.append(f"S{i} {names4[i]}")
            continue
        j = i - npre
        if j < 2 * (4 - npre):
            g = j // 2 + (npre if j % 2 else 0)
            order.append(f"{'S' if j % 2 else 'E'}{g} {names4[g]}")
        else:
            g = (4 - npre) + j - 2 * (4 - npre)
            order.append(f"E{g} {names4[g]}")
    for i in range(min(n, 2)):
        ent = tl[i, :, 1]
        print(f"layer kernel {i}: phase end, us after the CTA's setup (p10 / p50 / max over CTAs)")
        prev = ent
        for ph in range(8):
            e = tl[i, :, 4 + ph]
            d = (e - ent) / 1e3
            dur = (e - prev) / 1e3
            print(f"  {order[ph]:12s} end {np.percentile(d, 10):7.1f} {np.median(d):7.1f} {d.max():7.1f}   "
                  f"phase length p50 {np.median(dur):6.1f}")
            prev = e
if len(sys.argv) > 2:   # raw [launch][cta][16] globaltimer stamps (+ each group's plan) for offline analysis
    np.save(sys.argv[2], tl)
    np.savez(sys.argv[2].replace(".npy", "_plans.npz"),
             **{g: np.asarray(gp.plan_host) for (g, _), gp in zip(eng.groups, bp.group_plans)})
