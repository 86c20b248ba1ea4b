"""Per-stage MMA-thread stamps of the shrink (LSV_DEBUG_SHRINK has bit 16): for a few CTAs, the
wait for each stage's full barrier and the issue time between stages (development aid)."""
import os, sys, ctypes
import numpy as np, torch
sys.path.insert(0, '.')
from paper_2511_22880_b200 import native
from paper_2511_22880_b200.shapes import LLAMA2_7B, ModelShape
from paper_2511_22880_b200.slab import AdapterSlab
from paper_2511_22880_b200.lora import LoraDeltaEngine
from paper_2511_22880_b200.segments import index_tokens
model = ModelShape("l7b-1l", 1, LLAMA2_7B.projections); dev = torch.device("cuda:0")
ranks = [8]*44+[16]*22+[32]*14+[64]*11+[128]*9
slab = AdapterSlab(model, AdapterSlab.capacity_for(model, ranks), dev)
for i, r in enumerate(ranks):
    s = slab.allocate(f"a{i}", r); slab.fill_random(s, 1000+i)
seg = index_tokens(np.random.default_rng(0).integers(0, 100, 4096), ranks)
eng = LoraDeltaEngine(slab); bp = eng.prepare(seg)
lib = native.lib(); lib.lsv_debug_set_trace.argtypes = [ctypes.c_void_p, ctypes.c_int32]
ITEMS = 128
proj = int(sys.argv[1]) if len(sys.argv) > 1 else 0
pr = model.projections[proj]
x = torch.randn(4096, pr.h_in, device=dev).to(torch.bfloat16); y = torch.zeros(4096, pr.h_out, device=dev, dtype=torch.bfloat16)
for _ in range(3): eng.apply(bp, 0, proj, x, y)
torch.cuda.synchronize()
buf = torch.zeros(148 * ITEMS * 16, dtype=torch.int64, device=dev)
lib.lsv_debug_set_trace(buf.data_ptr(), ITEMS)
eng.shrink(bp, 0, proj, x); torch.cuda.synchronize(); lib.lsv_debug_set_trace(None, 0)
tr = buf.view(148, ITEMS, 16).cpu().numpy().astype(np.float64)
for c in (0, 31, 91, 122):
    w0 = tr[c, :ITEMS - 1, 8 + 6]; w1 = tr[c, :ITEMS - 1, 8 + 7]
    n = int((w1 > 0).sum())
    waits = (w1[:n] - w0[:n])
    gaps = (w0[1:n] - w1[:n - 1])
    print(f"cta {c}: {n} stages; wait-for-full cycles: {np.round(waits).astype(int).tolist()}")
    print(f"         issue cycles between stages: {np.round(gaps).astype(int).tolist()}")
