"""Quick per-projection timing of one Llama-2-7B layer (C2 batch) — development aid."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, '.')
from paper_2511_22880_b200.shapes import LLAMA2_7B, ModelShape
from paper_2511_22880_b200.slab import AdapterSlab
from paper_2511_22880_b200.lora import LoraDeltaEngine, algorithmic_bytes, input_group
from paper_2511_22880_b200.segments import index_tokens

tier = int(sys.argv[1]) if len(sys.argv) > 1 else 0
layers = 2
model = ModelShape("l7b-2l", layers, LLAMA2_7B.projections)
dev = torch.device("cuda:0")
ranks = [8]*44+[16]*22+[32]*14+[64]*11+[128]*9
slab = AdapterSlab(model, AdapterSlab.capacity_for(model, ranks), dev)
t=time.time()
for i, r in enumerate(ranks):
    s = slab.allocate(f"a{i}", r); slab.fill_random(s, 1000+i)
torch.cuda.synchronize(); print("fill", time.time()-t)
rng = np.random.default_rng(0)
seg = index_tokens(rng.integers(0, 100, 4096), ranks)
eng = LoraDeltaEngine(slab, tier_policy=tier)
bp = eng.prepare(seg)
N = 4096
xs = [{g: torch.randn(N, h, device=dev).to(torch.bfloat16) for g, h in [("attn_in",4096),("attn_out",4096),("mlp_in",4096),("mlp_mid",11008)]} for _ in range(layers)]
ys = [{p.name: torch.zeros(N, p.h_out, device=dev, dtype=torch.bfloat16) for p in model.projections} for _ in range(layers)]
for _ in range(3): eng.forward(bp, xs, ys)
torch.cuda.synchronize()
tot_bytes = 0; tot_t = 0
for p, pr in enumerate(model.projections):
    evs = []
    for it in range(10):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        l = it % layers
        e0.record(); eng.apply(bp, l, p, xs[l][input_group(pr.name)], ys[l][pr.name]); e1.record()
        evs.append((e0, e1))
    torch.cuda.synchronize()
    ms = np.median([a.elapsed_time(b) for a, b in evs])
    byts = algorithmic_bytes(seg, pr.h_in, pr.h_out)
    tot_bytes += byts; tot_t += ms
    print(f"{pr.name:10s} {ms*1e3:8.1f} us  {byts/ms/1e6:8.1f} GB/s  ({byts/1e6:.1f} MB)")
print(f"layer: {tot_t*1e3:.1f} us, {tot_bytes/tot_t/1e6:.1f} GB/s, model(32L) tok/s = {4096/(tot_t*32/1e3):.0f}")
print(bp.shape_plans[(4096,4096)].summary)
# split timing: shrink vs expand
for p, pr in enumerate(model.projections[:1] + model.projections[4:5] + model.projections[6:7]):
    pi = [q.name for q in model.projections].index(pr.name)
    for kind in ("shrink", "expand"):
        evs = []
        for it in range(10):
            l = it % layers
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            if kind == "shrink": eng.shrink(bp, l, pi, xs[l][input_group(pr.name)])
            else: eng.expand(bp, l, pi, ys[l][pr.name])
            e1.record(); evs.append((e0, e1))
        torch.cuda.synchronize()
        ms = np.median([a.elapsed_time(b) for a, b in evs])
        n = seg.lengths().astype(np.int64); r = seg.seg_rank.astype(np.int64)
        byts = int(np.sum(2*n*pr.h_in + 2*r*pr.h_in)) if kind == "shrink" else int(np.sum(2*r*pr.h_out + 4*n*pr.h_out))
        print(f"  {pr.name:10s} {kind:6s} {ms*1e3:8.1f} us {byts/ms/1e6:8.1f} GB/s")
