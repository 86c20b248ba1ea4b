"""Dump raw per-item stamps for a few CTAs (expand or shrink), in microseconds from kernel start."""
import sys, ctypes
import numpy as np, torch
sys.path.insert(0, '.')
from paper_2511_22880_b200 import native
from paper_2511_22880_b200.shapes import LLAMA2_7B, ModelShape
from paper_2511_22880_b200.slab import AdapterSlab
from paper_2511_22880_b200.lora import LoraDeltaEngine
from paper_2511_22880_b200.segments import index_tokens
proj = int(sys.argv[1]); kind = sys.argv[2]
model = ModelShape("l7b-1l", 1, LLAMA2_7B.projections); dev = torch.device("cuda:0")
ranks = [8]*44+[16]*22+[32]*14+[64]*11+[128]*9
slab = AdapterSlab(model, AdapterSlab.capacity_for(model, ranks), dev)
for i, r in enumerate(ranks):
    s = slab.allocate(f"a{i}", r); slab.fill_random(s, 1000+i)
seg = index_tokens(np.random.default_rng(0).integers(0, 100, 4096), ranks)
eng = LoraDeltaEngine(slab); bp = eng.prepare(seg); pr = model.projections[proj]
x = torch.randn(4096, pr.h_in, device=dev).to(torch.bfloat16); y = torch.zeros(4096, pr.h_out, device=dev, dtype=torch.bfloat16)
lib = native.lib(); lib.lsv_debug_set_trace.argtypes = [ctypes.c_void_p, ctypes.c_int32]
ITEMS = 64; buf = torch.zeros(148 * ITEMS * 16, dtype=torch.int64, device=dev)
for _ in range(3): eng.apply(bp, 0, proj, x, y)
torch.cuda.synchronize()
eng.shrink(bp, 0, proj, x); torch.cuda.synchronize()
lib.lsv_debug_set_trace(buf.data_ptr(), ITEMS)
if kind == "expand": eng.expand(bp, 0, proj, y)
else: eng.shrink(bp, 0, proj, x)
torch.cuda.synchronize(); lib.lsv_debug_set_trace(None, 0)
tt = buf.view(148, ITEMS, 16).cpu().numpy().astype(np.float64)
t = tt[:, :, :8]; cyc = tt[:, :, 8:]
t0 = t[t > 0].min()
for c in [int(a) for a in sys.argv[3:]] or [0, 77]:
    print(f"CTA {c} (us since first stamp; clock cycles since this CTA's first stamp)")
    c0 = cyc[c][cyc[c] > 0].min()
    for i in range(ITEMS):
        if t[c, i, 0] == 0 and t[c, i, 3] == 0: break
        print(f"  item {i:2d}: " + " ".join(f"{(t[c,i,k]-t0)/1e3:7.2f}" if t[c,i,k] > 0 else "      -" for k in range(6)) +
              "  | cyc " + " ".join(f"{int(cyc[c,i,k]-c0):7d}" if cyc[c,i,k] > 0 else "      -" for k in range(8)))
ends = np.nanmax(np.where(t > 0, t, np.nan), axis=(1, 2)) - t0
print("CTA end times (us): min %.1f median %.1f max %.1f" % (np.nanmin(ends)/1e3, np.nanmedian(ends)/1e3, np.nanmax(ends)/1e3))
