"""One decode step (B=32) eager, for ncu launch lists (development aid)."""
import sys, zlib
import numpy as np, torch
sys.path.insert(0, '.')
from paper_2511_22880_b200 import synth
from paper_2511_22880_b200.lora import LoraDeltaEngine
from paper_2511_22880_b200.segments import index_tokens
from paper_2511_22880_b200.slab import AdapterSlab
from paper_2511_22880_b200.shapes import ModelShape, LLAMA2_7B
B = int(sys.argv[1]) if len(sys.argv) > 1 else 32
wl = synth.WORKLOADS["c2"](); model = ModelShape("l7b-2l", 2, LLAMA2_7B.projections); dev = torch.device("cuda:0")
slab = AdapterSlab(model, AdapterSlab.capacity_for(model, wl.ranks), dev)
for aid, r in zip(wl.adapter_ids, wl.ranks):
    slab.fill_random(slab.allocate(aid, r), 1000 + zlib.crc32(aid.encode()) % 100000)
eng = LoraDeltaEngine(slab)
seg = index_tokens(np.random.default_rng(B).integers(0, len(wl.ranks), B), wl.ranks)
bp = eng.prepare(seg); N = seg.num_tokens
xs = [{g: torch.randn(N, model.projections[m[0]].h_in, device=dev).to(torch.bfloat16) for g, m in model.groups()} for _ in range(model.layers)]
ys = [{p.name: torch.zeros(N, p.h_out, device=dev, dtype=torch.bfloat16) for p in model.projections} for _ in range(model.layers)]
for _ in range(2): eng.forward(bp, xs, ys)
torch.cuda.synchronize(); print("ok")
