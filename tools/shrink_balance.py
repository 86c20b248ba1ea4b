"""Development tool: how well the shrink's static LPT cost model predicts each CTA's measured
main-loop time (q/k/v group of C2, layer 0).  Prints the correlation and a least-squares fit of the
per-CTA time to (bytes, records, stages) so the planner's fixed costs can be calibrated."""
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
gname, members = eng.groups[gi]
gp = bp.group_plans[gi]
blob = gp.plan_host
h = blob[:64]
n_shrink, shrink_grid, off_shrink, off_cta = int(h[8]), int(h[10]), int(h[17]), int(h[18])
recs = blob[off_shrink:off_shrink + 16 * n_shrink].reshape(-1, 16)
cta = blob[off_cta:off_cta + shrink_grid + 1]
feat = []
for c in range(shrink_grid):
    rr = recs[cta[c]:cta[c + 1]]
    byts = stages = 0
    for r in rr:
        np8 = -(-int(r[2]) // 8) * 8
        rows = int(r[14]) * int(r[3])
        nch = int(r[5]) - int(r[4])
        byts += (np8 + rows) * 128 * nch
        stages += -(-nch // int(r[6]))
    feat.append((byts, len(rr), stages))
feat = np.array(feat, dtype=np.float64)
x = torch.randn(4096, model.projections[members[0]].h_in, device=dev).to(torch.bfloat16)
for _ in range(3):
    eng.shrink(bp, 0, members[0], x)
torch.cuda.synchronize()
lib = native.lib()
lib.lsv_debug_set_trace.argtypes = [ctypes.c_void_p, ctypes.c_int32]
ITEMS = 64
times = []
for rep in range(5):
    buf = torch.zeros(148 * ITEMS * 16, dtype=torch.int64, device=dev)
    lib.lsv_debug_set_trace(buf.data_ptr(), ITEMS)
    eng.shrink(bp, 0, members[0], x)
    torch.cuda.synchronize()
    lib.lsv_debug_set_trace(None, 0)
    ph = buf.view(148, ITEMS, 16)[:, ITEMS - 1, :8].cpu().numpy().astype(np.float64)
    times.append((ph[:shrink_grid, 3] - ph[:shrink_grid, 2]) / 1e3)   # main loop, us
t = np.median(np.array(times), axis=0)
print(f"group {gname}: {shrink_grid} CTAs, main loop min {t.min():.2f} median {np.median(t):.2f} max {t.max():.2f} us")
print(f"corr(time, bytes) = {np.corrcoef(t, feat[:, 0])[0, 1]:.3f}")
a = np.column_stack([np.ones(len(t)), feat])
coef, *_ = np.linalg.lstsq(a, t, rcond=None)
pred = a @ coef
print("fit us = %.3f + %.3e*bytes + %.3f*records + %.3f*stages ; resid rms %.2f us" % (
    coef[0], coef[1], coef[2], coef[3], np.sqrt(np.mean((pred - t) ** 2))))
print("per-KB cost %.4f us -> record fixed = %.1f KB, stage fixed = %.1f KB equivalent" % (
    coef[1] * 1024, coef[2] / (coef[1] * 1024), coef[3] / (coef[1] * 1024)))
worst = np.argsort(t)[-5:]
for c in worst:
    print(f"  cta {c}: {t[c]:.2f} us, bytes {feat[c,0]/1e6:.2f} MB, records {int(feat[c,1])}, stages {int(feat[c,2])}")
