"""One C2 layer (7 projections) through the public API, for ncu launch lists / captures."""
import sys
import numpy as np, torch
sys.path.insert(0, '.')
from paper_2511_22880_b200 import synth
from paper_2511_22880_b200.shapes import ModelShape
from paper_2511_22880_b200.slab import AdapterSlab
from paper_2511_22880_b200.lora import LoraDeltaEngine, input_group
wl = synth.c2_llama2_7b()
model = ModelShape("llama-2-7b-1layer", 1, wl.model.projections)
dev = torch.device("cuda:0")
slab = AdapterSlab(model, AdapterSlab.capacity_for(model, wl.ranks), dev)
for i, (aid, r) in enumerate(zip(wl.adapter_ids, wl.ranks)):
    slab.fill_random(slab.allocate(aid, r), 1000 + i)
eng = LoraDeltaEngine(slab)
bp = eng.prepare(wl.segments)
N = wl.segments.num_tokens
xs = [{g: torch.randn(N, h, device=dev).to(torch.bfloat16) for g, h in [("attn_in", 4096), ("attn_out", 4096), ("mlp_in", 4096), ("mlp_mid", 11008)]}]
ys = [{p.name: torch.randn(N, p.h_out, device=dev).to(torch.bfloat16) for p in model.projections}]
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
for _ in range(reps):
    eng.forward(bp, xs, ys)
torch.cuda.synchronize()
print("ok")
