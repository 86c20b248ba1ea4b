"""Decode-regime timing (development aid): B requests decoding one token each over the C2 roster
(Llama-2-7B shapes, 100 adapters), whole 32-layer step via LoraDeltaEngine.forward in a CUDA graph."""
import sys, zlib
import numpy as np, torch
sys.path.insert(0, '.')
from paper_2511_22880_b200 import synth, shapes
from paper_2511_22880_b200.lora import LoraDeltaEngine, algorithmic_bytes
from paper_2511_22880_b200.segments import index_tokens
from paper_2511_22880_b200.slab import AdapterSlab
wl = synth.WORKLOADS["c2"](); model = wl.model; dev = torch.device("cuda:0")
slab = AdapterSlab(model, AdapterSlab.capacity_for(model, wl.ranks), dev)
for aid, r in zip(wl.adapter_ids, wl.ranks):
    slab.fill_random(slab.allocate(aid, r), 1000 + zlib.crc32(aid.encode()) % 100000)
eng = LoraDeltaEngine(slab)
for B in (32, 128, 512):
    rng = np.random.default_rng(B)
    tok = rng.integers(0, len(wl.ranks), B)
    seg = index_tokens(tok, wl.ranks)
    bp = eng.prepare(seg)
    N = seg.num_tokens
    xs = [{g: torch.randn(N, model.projections[m[0]].h_in, device=dev).to(torch.bfloat16) for g, m in model.groups()} for _ in range(model.layers)]
    ys = [{p.name: torch.zeros(N, p.h_out, device=dev, dtype=torch.bfloat16) for p in model.projections} for _ in range(model.layers)]
    st = torch.cuda.Stream(dev)
    with torch.cuda.stream(st):
        eng.forward(bp, xs, ys, st)
    torch.cuda.synchronize()
    gph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gph, stream=st):
        eng.forward(bp, xs, ys, st)
    for _ in range(3): gph.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(10):
        with torch.cuda.stream(st): gph.replay()
    e1.record(st); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    byt = sum(algorithmic_bytes(seg, p.h_in, p.h_out) for p in model.projections) * model.layers
    print(f"decode B={B}: {seg.num_segments} segments, {ms:.3f} ms/step, {N/ms*1e3:.0f} tok/s, "
          f"{byt/ms/1e6:.0f} GB/s ({byt/ms/1e6/6541.1:.1%} of HBM), plan {bp.group_plans[0].summary}")
