"""Per-stage timing of one shrink launch (C2 layer, one input group), LSV_DEBUG_SHRINK=16 stamps:
producer waits for a free slot, producer issues the stage's copies, MMA waits for the stage to land.
    LSV_DEBUG_SHRINK=16 python tools/trace_shrink_lat.py [group=0]"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, '.')
from paper_2511_22880_b200 import native  # noqa: E402
from paper_2511_22880_b200.lora import LoraDeltaEngine  # noqa: E402
from paper_2511_22880_b200.segments import index_tokens  # noqa: E402
from paper_2511_22880_b200.shapes import LLAMA2_7B, ModelShape  # noqa: E402
from paper_2511_22880_b200.slab import AdapterSlab  # noqa: E402

assert int(os.environ.get("LSV_DEBUG_SHRINK", "0")) & 16, "run with LSV_DEBUG_SHRINK=16"
gi = int(sys.argv[1]) if len(sys.argv) > 1 else 0
model = ModelShape("l7b-1l", 1, LLAMA2_7B.projections)
dev = torch.device("cuda:0")
ranks = [8] * 44 + [16] * 22 + [32] * 14 + [64] * 11 + [128] * 9
slab = AdapterSlab(model, AdapterSlab.capacity_for(model, ranks), dev)
for i, r in enumerate(ranks):
    slab.fill_random(slab.allocate(f"a{i}", r), 1000 + i)
seg = index_tokens(np.random.default_rng(0).integers(0, 100, 4096), ranks)
eng = LoraDeltaEngine(slab)
bp = eng.prepare(seg)
p0 = eng.groups[gi][1][0]
x = torch.randn(4096, model.projections[p0].h_in, device=dev).to(torch.bfloat16)
lib = native.lib()
lib.lsv_debug_set_trace.argtypes = [ctypes.c_void_p, ctypes.c_int32]
for _ in range(3):
    eng.shrink(bp, 0, p0, x)
torch.cuda.synchronize()
ITEMS = 256
buf = torch.zeros(148 * ITEMS * 16, dtype=torch.int64, device=dev)
lib.lsv_debug_set_trace(buf.data_ptr(), ITEMS)
eng.shrink(bp, 0, p0, x)
torch.cuda.synchronize()
lib.lsv_debug_set_trace(None, 0)
cyc = buf.view(148, ITEMS, 16).cpu().numpy().astype(np.int64)[:, :, 8:16]
st = {k: [] for k in ("prod_slot_wait", "prod_issue", "mma_full_wait", "stage_period")}
for c in range(148):
    n = int((cyc[c, :ITEMS - 1, 5] > 0).sum())
    for s in range(n):
        v = cyc[c, s]
        st["prod_slot_wait"].append(v[4] - v[3])
        st["prod_issue"].append(v[5] - v[4])
        if v[7] > 0:
            st["mma_full_wait"].append(v[7] - v[6])
        if s > 0:
            st["stage_period"].append(v[5] - cyc[c, s - 1, 5])
print(f"group {gi}: stages per CTA {np.mean([int((cyc[c, :ITEMS - 1, 5] > 0).sum()) for c in range(148)]):.1f}")
for k, v in st.items():
    v = np.array(v)
    print(f"{k:16s} n {len(v):5d}  mean {v.mean():7.0f}  p10 {np.percentile(v, 10):7.0f}  p50 {np.median(v):7.0f}  "
          f"p90 {np.percentile(v, 90):7.0f}")
ph = cyc[:, ITEMS - 1, :]   # phase stamps: 0 entry, 1 after TMEM alloc, 2 after PDL wait, 3 main loops done, 4 barrier passed, 5 reduction done
rel = lambda c, v: v - ph[c, 0]
for name, k in (("TMEM alloc", 1), ("start", 2), ("main loops done", 3), ("barrier passed", 4), ("reduction done", 5)):
    v = np.array([rel(c, ph[c, k]) for c in range(148)])
    print(f"{name:16s} p10 {np.percentile(v, 10):7.0f}  p50 {np.median(v):7.0f}  max {v.max():7.0f}")
first = np.array([rel(c, cyc[c, 0, 7]) for c in range(148)])
last = np.array([rel(c, cyc[c, int((cyc[c, :ITEMS - 1, 5] > 0).sum()) - 1, 7]) for c in range(148)])
print(f"first stage landed p50 {np.median(first):.0f}; last stage landed p50 {np.median(last):.0f} max {last.max():.0f}")
c = int(np.argmax(last))
n = int((cyc[c, :ITEMS - 1, 5] > 0).sum())
print(f"CTA {c} stages: slotwait_start issued mma_wait mma_got (rel. entry)")
for s in range(n):
    v = cyc[c, s]
    print(f"  {s:2d} {rel(c, v[3]):7d} {rel(c, v[5]):7d} {rel(c, v[6]):7d} {rel(c, v[7]):7d}")
