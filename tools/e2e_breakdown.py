"""Where the e2e step's wall time goes (host indexing, planning + uploads, H2D, forward, D2H)."""
import sys, time
import numpy as np, torch
sys.path.insert(0, '.')
from paper_2511_22880_b200 import synth
from paper_2511_22880_b200.lora import LoraDeltaEngine
from paper_2511_22880_b200.segments import index_tokens
from paper_2511_22880_b200.slab import AdapterSlab
import zlib
wl = synth.WORKLOADS["c2"](); model = wl.model; dev = torch.device("cuda:0")
slab = AdapterSlab(model, AdapterSlab.capacity_for(model, wl.ranks), dev)
for aid, r in zip(wl.adapter_ids, wl.ranks):
    slab.fill_random(slab.allocate(aid, r), 1000 + zlib.crc32(aid.encode()) % 100000)
eng = LoraDeltaEngine(slab); seg = wl.segments; N = seg.num_tokens
xs = [{g: torch.randn(N, model.projections[m[0]].h_in, device=dev).to(torch.bfloat16) for g, m in model.groups()} for _ in range(model.layers)]
ys = [{p.name: torch.zeros(N, p.h_out, device=dev, dtype=torch.bfloat16) for p in model.projections} for _ in range(model.layers)]
tok = np.repeat(seg.seg_slot, seg.lengths())
x_host = torch.empty((N, 4096), dtype=torch.bfloat16, pin_memory=True); y_host = torch.empty((N, 4096), dtype=torch.bfloat16, pin_memory=True)
st = torch.cuda.Stream(dev)
for it in range(6):
    torch.cuda.synchronize(); t = [time.perf_counter()]
    s2 = index_tokens(tok, wl.ranks); t.append(time.perf_counter())
    bp = eng.prepare(s2); torch.cuda.synchronize(); t.append(time.perf_counter())
    with torch.cuda.stream(st):
        xs[0]["attn_in"].copy_(x_host, non_blocking=True); st.synchronize(); t.append(time.perf_counter())
        eng.forward(bp, xs, ys, st); t.append(time.perf_counter()); st.synchronize(); t.append(time.perf_counter())
        y_host.copy_(ys[-1]["down_proj"], non_blocking=True); st.synchronize(); t.append(time.perf_counter())
    d = np.diff(t) * 1e3
    print(f"index {d[0]:.2f} prepare {d[1]:.2f} h2d {d[2]:.2f} forward-issue {d[3]:.2f} forward-gpu {d[4]:.2f} d2h {d[5]:.2f} total {sum(d):.2f} ms")
