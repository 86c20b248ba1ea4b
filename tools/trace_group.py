"""Timeline of one group-kernel launch (C2 layer shapes, one input group as a 1-layer model):
per CTA, when its shrink records are stored, when its split-K shares are reduced, when its expand
items start / finish, and how long the expand producer waits for m-tiles to become ready.
Clock-only trace build: LSV_NVCC_DEFINES=-DLSV_TRACE_CLOCK_ONLY (liblsv_clk.so).
    python tools/trace_group.py [group=2]"""
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

gi = int(sys.argv[1]) if len(sys.argv) > 1 else 2
full = LLAMA2_7B.groups()[gi]
model = ModelShape("l7b-g", 1, tuple(LLAMA2_7B.projections[p] for p in full[1]))
dev = torch.device("cuda:0")
ranks = [8] * 44 + [16] * 22 + [32] * 14 + [64] * 11 + [128] * 9
slab = AdapterSlab(model, AdapterSlab.capacity_for(model, ranks), dev)
for i, r in enumerate(ranks):
    slab.fill_random(slab.allocate(f"a{i}", r), 1000 + i)
seg = index_tokens(np.random.default_rng(0).integers(0, 100, 4096), ranks)
eng = LoraDeltaEngine(slab)
bp = eng.prepare(seg)
gname = model.groups()[0][0]
xs = [{gname: torch.randn(4096, model.projections[0].h_in, device=dev).to(torch.bfloat16)}]
ys = [{p.name: torch.zeros(4096, p.h_out, device=dev, dtype=torch.bfloat16) for p in model.projections}]
for _ in range(3):
    eng.forward(bp, xs, ys)
torch.cuda.synchronize()
lib = native.lib()
lib.lsv_debug_set_trace.argtypes = [ctypes.c_void_p, ctypes.c_int32]
ITEMS = 128
buf = torch.zeros(2 * 148 * ITEMS * 16, dtype=torch.int64, device=dev)
lib.lsv_debug_set_trace(buf.data_ptr(), ITEMS)
eng.forward(bp, xs, ys)
torch.cuda.synchronize()
lib.lsv_debug_set_trace(None, 0)
tr = buf.view(2, 148, ITEMS, 16).cpu().numpy().astype(np.int64)
sc, ec = tr[0, :, :, 8:16], tr[1, :, :, 8:16]
eaux = tr[1, :, :, 0:8]
ph = sc[:, ITEMS - 1, :]
t0 = ph[:, 0]
rel = lambda v: v - t0   # noqa: E731
def pct(name, v):
    v = np.asarray(v)
    print(f"{name:34s} p10 {np.percentile(v, 10):8.0f}  p50 {np.median(v):8.0f}  max {v.max():8.0f}")
print(f"group {full[0]}: cycles after each CTA's setup (1.9 GHz: 1900 cycles = 1 us)")
pct("shrink records stored", rel(ph[:, 1]))
pct("shrink stages consumed (producer)", rel(ph[:, 2]))
pct("split-K shares reduced", rel(ph[:, 3]))
ne = (ec[:, :ITEMS - 1, 0] > 0).sum(1)
first = np.array([ec[c, 0, 0] for c in range(148)]) - t0
pct("first expand item: producer start", first)
pct("expand items stored", rel(ph[:, 4]))
waits = []
for c in range(148):
    for k in range(int(ne[c])):
        if eaux[c, k, 6] > 0:
            waits.append(eaux[c, k, 6] - eaux[c, k, 5])
waits = np.array(waits) if waits else np.zeros(1)
print(f"v-ready waits per item: mean {waits.mean():.0f}  p50 {np.median(waits):.0f}  p90 {np.percentile(waits, 90):.0f}  "
      f"sum per CTA {waits.sum() / 148:.0f}")
print(f"expand items per CTA {ne.mean():.1f}")
import os
if int(os.environ.get("LSV_DEBUG_SHRINK", "0")) & 16:   # per-stage shrink stamps (slots 3..7 of stage s)
    st = {k: [] for k in ("prod_slot_wait", "prod_issue", "mma_full_wait", "stage_period")}
    for c in range(148):
        n = int((sc[c, :ITEMS - 1, 5] > 0).sum())
        for s in range(n):
            v = sc[c, s]
            st["prod_slot_wait"].append(v[4] - v[3]); st["prod_issue"].append(v[5] - v[4])
            if v[7] > 0:
                st["mma_full_wait"].append(v[7] - v[6])
            if s > 0:
                st["stage_period"].append(v[5] - sc[c, s - 1, 5])
    for k, v in st.items():
        pct(k, v)
# expand items inside the group kernel: where an item's time goes (clock-only stamps)
es = {k: [] for k in ("ring_wait", "alloc->B_issued", "B->y_issued", "y->v_issued(vready wait)", "v_issued->next",
                      "load(alloc->landed)", "mma_full_wait", "mma_issue", "epi", "item_period")}
for c in range(148):
    n = int(ne[c])
    for i in range(n):
        v, a = ec[c, i], eaux[c, i]
        es["ring_wait"].append(v[1] - v[0])
        es["alloc->B_issued"].append(a[3] - v[1])
        if a[5] > 0:
            es["B->y_issued"].append(a[5] - a[3])
            es["y->v_issued(vready wait)"].append(a[4] - a[5])
        if i + 1 < n:
            es["v_issued->next"].append(ec[c, i + 1, 0] - a[4])
        es["load(alloc->landed)"].append(v[6] - v[1])
        es["mma_full_wait"].append(v[6] - v[5])
        es["mma_issue"].append(v[2] - v[6])
        es["epi"].append(v[4] - v[3])
        if i > 0:
            es["item_period"].append(v[4] - ec[c, i - 1, 4])
for k, v in es.items():
    if v:
        pct(k, v)
