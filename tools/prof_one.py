"""Minimal C2 one-layer workload for ncu captures: the step's mlp_in kernels (fused gate/up shrink
+ one-launch gate/up expand), three times; profile the last pair with -s 4 -c 2."""
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
from paper_2511_22880_b200.shapes import LLAMA2_7B, ModelShape
from paper_2511_22880_b200.slab import AdapterSlab
from paper_2511_22880_b200.lora import LoraDeltaEngine
from paper_2511_22880_b200.segments import index_tokens

model = ModelShape("l7b-1l", 1, LLAMA2_7B.projections)
dev = torch.device("cuda:0")
ranks = [8]*44+[16]*22+[32]*14+[64]*11+[128]*9
slab = AdapterSlab(model, AdapterSlab.capacity_for(model, ranks), dev)
for i, r in enumerate(ranks):
    s = slab.allocate(f"a{i}", r); slab.fill_random(s, 1000+i)
seg = index_tokens(np.random.default_rng(0).integers(0, 100, 4096), ranks)
eng = LoraDeltaEngine(slab)
bp = eng.prepare(seg)
gi = int(sys.argv[1]) if len(sys.argv) > 1 else 2          # 2 = mlp_in (gate/up)
gname, members = eng.groups[gi]
x = torch.randn(4096, model.projections[members[0]].h_in, device=dev).to(torch.bfloat16)
ys = [torch.zeros(4096, model.projections[p].h_out, device=dev, dtype=torch.bfloat16) for p in members]
for _ in range(3):
    eng.shrink(bp, 0, members[0], x)
    eng.expand_group(bp, 0, gi, ys)
torch.cuda.synchronize()
print("ok")
