"""Where an expand item's lifetime goes (C2 layer, gate/up group expand, one launch, all CTAs).

Per item (clock64 stamps, lsv_debug_set_trace): ring wait = producer start -> ring bytes
allocated; load = allocated -> MMA saw the full barrier (only items whose MMA was already waiting
on it, i.e. the landing time is observed); tempty wait = MMA ready -> accumulator free; epilogue =
epilogue got the accumulator -> done; occupancy = bytes in flight per CTA over the launch.
    python tools/trace_expand_lat.py [group=2]"""
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
model = ModelShape("l7b-1l", 1, LLAMA2_7B.projections)
dev = torch.device("cuda:0")
ranks = [8] * 44 + [16] * 22 + [32] * 14 + [64] * 11 + [128] * 9
slab = AdapterSlab(model, AdapterSlab.capacity_for(model, ranks), dev)
for i, r in enumerate(ranks):
    slab.fill_random(slab.allocate(f"a{i}", r), 1000 + i)
seg = index_tokens(np.random.default_rng(0).integers(0, 100, 4096), ranks)
eng = LoraDeltaEngine(slab)
bp = eng.prepare(seg)
members = eng.groups[gi][1]
p0 = members[0]
x = torch.randn(4096, model.projections[p0].h_in, device=dev).to(torch.bfloat16)
ys = [torch.zeros(4096, model.projections[p].h_out, device=dev, dtype=torch.bfloat16) for p in members]
lib = native.lib()
lib.lsv_debug_set_trace.argtypes = [ctypes.c_void_p, ctypes.c_int32]
eng.shrink(bp, 0, p0, x)
for _ in range(3):
    eng.expand_group(bp, 0, gi, ys)
torch.cuda.synchronize()
ITEMS = 96
buf = torch.zeros(148 * ITEMS * 16, dtype=torch.int64, device=dev)
lib.lsv_debug_set_trace(buf.data_ptr(), ITEMS)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
eng.expand_group(bp, 0, gi, ys)
e1.record()
torch.cuda.synchronize()
lib.lsv_debug_set_trace(None, 0)
print(f"group {gi} expand (traced): {e0.elapsed_time(e1) * 1e3:.1f} us")
tr = buf.view(148, ITEMS, 16).cpu().numpy().astype(np.int64)
cyc = tr[:, :, 8:16]
ns = tr[:, :, 0:8]
st = {k: [] for k in ("ring_wait", "load", "load_all", "tempty_wait", "mma_full_wait", "mma_issue", "mma_tail", "epi", "item_period")}
spans = []
for c in range(148):
    n = int((cyc[c, :ITEMS - 1, 0] > 0).sum())
    if n == 0:
        continue
    ph = tr[c, ITEMS - 1, 8:16]
    spans.append((cyc[c, 0, 0] - ph[0], cyc[c, n - 1, 4] - ph[0], n))
    for i in range(n):
        v = cyc[c, i]
        st["ring_wait"].append(v[1] - v[0])
        st["load_all"].append(v[6] - v[1])
        if v[6] - v[5] > 200:       # the MMA waited on the loads: landing time observed
            st["load"].append(v[6] - v[1])
            st["mma_full_wait"].append(v[6] - v[5])
        if i > 0:
            st["tempty_wait"].append(v[5] - cyc[c, i - 1, 2])
            st["item_period"].append(v[4] - cyc[c, i - 1, 4])
        st["epi"].append(v[4] - v[3])
        st["mma_issue"].append(v[2] - v[6])      # loads landed -> MMAs + commits issued
        st["mma_tail"].append(v[3] - v[2])       # commits issued -> epilogue sees the accumulator
print("cycles (1.9 GHz: 1900 cycles = 1 us)")
for k, v in st.items():
    v = np.array(v)
    if len(v) == 0:
        continue
    print(f"{k:14s} n {len(v):5d}  mean {v.mean():8.0f}  p10 {np.percentile(v, 10):8.0f}  p50 {np.median(v):8.0f}  "
          f"p90 {np.percentile(v, 90):8.0f}")
sp = np.array(spans)
print(f"CTA first item start (cycles after kernel entry): p50 {np.median(sp[:, 0]):.0f} max {sp[:, 0].max():.0f}")
print(f"CTA last epilogue done: min {sp[:, 1].min():.0f} p50 {np.median(sp[:, 1]):.0f} max {sp[:, 1].max():.0f}; items/CTA {sp[:, 2].mean():.1f}")
c = int(np.argmax(sp[:, 1]))
n = int(sp[c, 2])
print(f"slowest CTA {c}: {n} items")
print("   k  prod0  alloc | mma_te mma_fu commit | epi_in epi_out")
t0 = cyc[c, 0, 0]
for i in range(min(n, 24)):
    v = cyc[c, i] - t0
    print(f"  {i:2d} {v[0]:6d} {v[1]:6d} | {v[5]:6d} {v[6]:6d} {v[2]:6d} | {v[3]:6d} {v[4]:6d}")

# clock-only builds (-DLSV_TRACE_CLOCK_ONLY): the MMA warp's own chain from the aux stamps
aux = tr[:, :, 0:8]
if (aux[:, 1:, 1] > 0).any():
    ch = {k: [] for k in ("pop", "pre", "tempty", "full", "issue", "commit", "sync")}
    for c in range(148):
        n = int((cyc[c, :ITEMS - 1, 0] > 0).sum())
        for i in range(1, n):
            a, ap, v = aux[c, i], aux[c, i - 1], cyc[c, i]
            ch["pop"].append(a[1] - ap[0]); ch["pre"].append(a[2] - a[1]); ch["tempty"].append(v[5] - a[2])
            ch["full"].append(v[6] - v[5]); ch["issue"].append(v[7] - v[6]); ch["commit"].append(v[2] - v[7])
            ch["sync"].append(a[0] - v[2])
    print("MMA warp chain per item (cycles):")
    for k, v in ch.items():
        v = np.array(v)
        print(f"  {k:8s} mean {v.mean():7.0f}  p50 {np.median(v):7.0f}  p90 {np.percentile(v, 90):7.0f}")

# ring occupancy: items between allocation (stamp 1) and MMA completion (epilogue saw tfull, stamp 3),
# and items in the load phase (allocation -> landed, stamp 6), time-averaged per CTA
occ, ld = [], []
for c in range(148):
    n = int((cyc[c, :ITEMS - 1, 0] > 0).sum())
    if n < 4:
        continue
    a, l, e = cyc[c, :n, 1], cyc[c, :n, 6], cyc[c, :n, 3]
    T = e[-1] - a[0]
    occ.append(float((e - a).sum()) / T)
    ld.append(float((l - a).sum()) / T)
print(f"items resident in the ring (alloc -> MMA done), time average per CTA: mean {np.mean(occ):.2f}")
print(f"items in the load phase (alloc -> landed), time average per CTA: mean {np.mean(ld):.2f}")
ph = bp.group_plans[gi].plan_host
off_recs, off_cta = int(ph[57]), int(ph[58])
vs = int(ph[61])
inflight_b = []
for c in range(148):
    n = int((cyc[c, :ITEMS - 1, 0] > 0).sum())
    r0, r1 = int(ph[off_cta + c]), int(ph[off_cta + c + 1])
    recs = ph[off_recs + 8 * r0: off_recs + 8 * r1].reshape(-1, 8)
    if n < 4 or len(recs) < n:
        continue
    kp = ((recs[:n, 3] + 15) // 16) * 16
    np16 = ((recs[:n, 2] + 15) // 16) * 16
    size = 256 * kp * 2 + np16 * kp * 2 * (2 if vs else 1) + np16 * 256 * 2
    a, l = cyc[c, :n, 1], cyc[c, :n, 6]
    T = cyc[c, n - 1, 3] - a[0]
    inflight_b.append(float(((l - a) * size).sum()) / T)
print(f"bytes in the load phase, time average per CTA: mean {np.mean(inflight_b) / 1024:.1f} KB; "
      f"mean item {np.mean(size) / 1024:.1f} KB (last CTA)")
# ring bytes held by earlier items when the producer starts item k (prod0) and when it gets it (alloc)
at_start, at_alloc, waits_big = [], [], 0
for c in range(148):
    n = int((cyc[c, :ITEMS - 1, 0] > 0).sum())
    r0, r1 = int(ph[off_cta + c]), int(ph[off_cta + c + 1])
    recs = ph[off_recs + 8 * r0: off_recs + 8 * r1].reshape(-1, 8)
    if n < 4 or len(recs) < n:
        continue
    kp = ((recs[:n, 3] + 15) // 16) * 16
    np16 = ((recs[:n, 2] + 15) // 16) * 16
    size = 256 * kp * 2 + np16 * kp * 2 * (2 if vs else 1) + np16 * 256 * 2
    p0s, a, e = cyc[c, :n, 0], cyc[c, :n, 1], cyc[c, :n, 3]
    for k in range(1, n):
        held = lambda t: sum(int(size[j]) for j in range(k) if e[j] > t)
        at_start.append(held(p0s[k]) + size[k])
        at_alloc.append(held(a[k] - 1) + size[k])
at_start, at_alloc = np.array(at_start) / 1024, np.array(at_alloc) / 1024
print(f"ring KB needed at producer start (held + this item): p10 {np.percentile(at_start, 10):.0f} p50 {np.median(at_start):.0f} "
      f"p90 {np.percentile(at_start, 90):.0f}; >200 KB in {np.mean(at_start > 200) * 100:.0f}% of items")
c = 40
n = int((cyc[c, :ITEMS - 1, 0] > 0).sum())
r0, r1 = int(ph[off_cta + c]), int(ph[off_cta + c + 1])
recs = ph[off_recs + 8 * r0: off_recs + 8 * r1].reshape(-1, 8)
kp = ((recs[:n, 3] + 15) // 16) * 16
np16 = ((recs[:n, 2] + 15) // 16) * 16
size = 256 * kp * 2 + np16 * kp * 2 * (2 if vs else 1) + np16 * 256 * 2
p0s, a, l, e = cyc[c, :n, 0], cyc[c, :n, 1], cyc[c, :n, 6], cyc[c, :n, 3]
t0 = p0s[0]
print(f"CTA {c}: k rank ntok sizeKB held@start wait  | p0 alloc landed mma_done")
for k in range(min(n, 30)):
    held = sum(int(size[j]) for j in range(k) if e[j] > p0s[k]) / 1024
    print(f"  {k:2d} {recs[k, 3]:4d} {recs[k, 2]:4d} {size[k] / 1024:6.1f} {held:7.1f} {a[k] - p0s[k]:6d} | "
          f"{p0s[k] - t0:7d} {a[k] - t0:7d} {l[k] - t0:7d} {e[k] - t0:7d}")
if (aux[:, 1:, 3] > 0).any():
    pr = {k: [] for k in ("alloc->bulk_issued", "bulk->y_issued", "y_issued->next_p0")}
    for c in range(148):
        n = int((cyc[c, :ITEMS - 1, 0] > 0).sum())
        for i in range(n - 1):
            pr["alloc->bulk_issued"].append(aux[c, i, 3] - cyc[c, i, 1])
            pr["bulk->y_issued"].append(aux[c, i, 4] - aux[c, i, 3])
            pr["y_issued->next_p0"].append(cyc[c, i + 1, 0] - aux[c, i, 4])
    print("producer per item (cycles):")
    for k, v in pr.items():
        v = np.array(v)
        print(f"  {k:20s} mean {v.mean():7.0f}  p50 {np.median(v):7.0f}  p90 {np.percentile(v, 90):7.0f}")
