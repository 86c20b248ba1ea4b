"""Development tool: the bench's pipelined e2e loop (c2) instrumented per step — host time of
index / prepare / issue, and device time of H2D / forward / D2H from CUDA events — over several
windows, to see where the e2e variance between runs comes from."""
import sys, time, zlib, os
import numpy as np, torch
sys.path.insert(0, '.')
from paper_2511_22880_b200 import synth
from paper_2511_22880_b200.lora import LoraDeltaEngine
from paper_2511_22880_b200.segments import index_tokens
from paper_2511_22880_b200.slab import AdapterSlab
from paper_2511_22880_b200.shapes import input_group

wl = synth.WORKLOADS["c2"](); model = wl.model; dev = torch.device("cuda:0")
slab = AdapterSlab(model, AdapterSlab.capacity_for(model, wl.ranks), dev)
for aid, r in zip(wl.adapter_ids, wl.ranks):
    slab.fill_random(slab.allocate(aid, r), 1000 + zlib.crc32(aid.encode()) % 100000)
eng = LoraDeltaEngine(slab); seg = wl.segments; N = seg.num_tokens
xs = [{g: torch.randn(N, model.projections[m[0]].h_in, device=dev).to(torch.bfloat16) for g, m in model.groups()}
      for _ in range(model.layers)]
ys = [{p.name: torch.zeros(N, p.h_out, device=dev, dtype=torch.bfloat16) for p in model.projections}
      for _ in range(model.layers)]
tok = np.repeat(seg.seg_slot, seg.lengths())
x_host = torch.empty((N, 4096), dtype=torch.bfloat16, pin_memory=True)
y_host = torch.empty((N, 4096), dtype=torch.bfloat16, pin_memory=True)
x_dev0 = xs[0][input_group(model.projections[0].name)]
last = model.projections[-1]
stream = torch.cuda.Stream(dev)
import gc
_gct = {}
def _gccb(phase, info):
    if phase == "start": _gct["t"] = time.perf_counter()
    elif info["generation"] >= 1:
        dt = (time.perf_counter() - _gct["t"]) * 1e3
        if dt > 1: print(f"  gc gen{info['generation']} {dt:.1f} ms", flush=True)
gc.callbacks.append(_gccb)
print("affinity", sorted(os.sched_getaffinity(0))[:8], "... n =", len(os.sched_getaffinity(0)), flush=True)

def window(steps, detail):
    evs = []; host = []; keep = []
    stream.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        a = time.perf_counter()
        s2 = index_tokens(tok, wl.ranks); b = time.perf_counter()
        bp = eng.prepare(s2, stream=stream); c = time.perf_counter()
        e = [torch.cuda.Event(enable_timing=True) for _ in range(4)] if detail else None
        with torch.cuda.stream(stream):
            if e: e[0].record(stream)
            x_dev0.copy_(x_host, non_blocking=True)
            if e: e[1].record(stream)
            eng.forward(bp, xs, ys, stream)
            if e: e[2].record(stream)
            y_host.copy_(ys[-1][last.name], non_blocking=True)
            if e: e[3].record(stream)
        d = time.perf_counter()
        keep.append(bp); evs.append(e); host.append((b - a, c - b, d - c))
    stream.synchronize()
    wall = (time.perf_counter() - t0) / steps
    h = np.array(host) * 1e3
    out = f"wall/step {wall*1e3:6.2f} ms ({N/wall/1e3:6.1f}K tok/s)  host idx {h[:,0].mean():.2f} prep {h[:,1].mean():.2f} (max {h[:,1].max():.2f}) issue {h[:,2].mean():.2f} (max {h[:,2].max():.2f})"
    if detail:
        g = np.array([[e[0].elapsed_time(e[1]), e[1].elapsed_time(e[2]), e[2].elapsed_time(e[3])] for e in evs])
        gaps = [evs[i][0].elapsed_time(evs[i + 1][0]) for i in range(len(evs) - 1)]
        out += f" | gpu h2d {g[:,0].mean():.2f} fwd {g[:,1].mean():.2f} (max {g[:,1].max():.2f}) d2h {g[:,2].mean():.2f} step-gap mean {np.mean(gaps):.2f} max {np.max(gaps):.2f}"
    print(out, flush=True)

for _ in range(3):
    window(5, False)
for i in range(6):
    window(20, i % 2 == 1)
