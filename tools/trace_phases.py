"""CTA-level phase stamps of the tcgen05 kernels, relative to the earliest CTA entry, plus the
host-side event time of the same launch (development aid)."""
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
lib.lsv_debug_set_trace(buf.data_ptr(), ITEMS)
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record()
if kind == "expand": eng.expand(bp, 0, proj, y)
elif kind == "group":   # the one-launch expand of proj's whole input group (what forward runs)
    gi, _ = eng._member[proj]
    ysg = [torch.zeros(4096, model.projections[q].h_out, device=dev, dtype=torch.bfloat16) for q in eng.groups[gi][1]]
    eng.expand_group(bp, 0, gi, ysg); torch.cuda.synchronize()
    lib.lsv_debug_set_trace(buf.data_ptr(), ITEMS); e0.record()
    eng.expand_group(bp, 0, gi, ysg)
else: eng.shrink(bp, 0, proj, x)
e1.record(); torch.cuda.synchronize(); lib.lsv_debug_set_trace(None, 0)
ph = buf.view(148, ITEMS, 16)[:, ITEMS - 1, :8].cpu().numpy().astype(np.float64)
t0 = ph[:, 0][ph[:, 0] > 0].min()
names = ["entry", "prologue_done", "pdl_wait_done", "main_loop_done", "barrier_passed", "reduce_done"]
print(f"{kind} {pr.name}: event-timed {e0.elapsed_time(e1)*1e3:.1f} us")
for k, nm in enumerate(names):
    v = ph[:, k]; v = v[v > 0]
    if len(v): print(f"  {nm:>16s}: min {(v.min()-t0)/1e3:7.2f}  median {(np.median(v)-t0)/1e3:7.2f}  max {(v.max()-t0)/1e3:7.2f} us")
