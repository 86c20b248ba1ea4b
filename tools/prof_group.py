"""Minimal C2 one-layer workload for ncu captures: one lsv_lora_forward over a 1-layer Llama-2-7B,
four times.  Default: one layer-kernel launch per call (profile the last with -k regex:group -s 3
-c 1); with LSV_LAYER_KERNEL=0 four group-kernel launches per call (-s 12 -c 4)."""
import sys

import numpy as np
import torch

sys.path.insert(0, '.')
from paper_2511_22880_b200.lora import LoraDeltaEngine  # noqa: E402
from paper_2511_22880_b200.segments import index_tokens  # noqa: E402
from paper_2511_22880_b200.shapes import LLAMA2_7B, ModelShape  # noqa: E402
from paper_2511_22880_b200.slab import AdapterSlab  # noqa: E402

model = ModelShape("l7b-1l", 1, LLAMA2_7B.projections)
dev = torch.device("cuda:0")
ranks = [8] * 44 + [16] * 22 + [32] * 14 + [64] * 11 + [128] * 9
slab = AdapterSlab(model, AdapterSlab.capacity_for(model, ranks), dev)
for i, r in enumerate(ranks):
    slab.fill_random(slab.allocate(f"a{i}", r), 1000 + i)
seg = index_tokens(np.random.default_rng(0).integers(0, 100, 4096), ranks)
eng = LoraDeltaEngine(slab)
bp = eng.prepare(seg)
xs = [{g: torch.randn(4096, model.projections[m[0]].h_in, device=dev).to(torch.bfloat16) for g, m in eng.groups}]
ys = [{p.name: torch.zeros(4096, p.h_out, device=dev, dtype=torch.bfloat16) for p in model.projections}]
for _ in range(4):
    eng.forward(bp, xs, ys)
torch.cuda.synchronize()
print("ok")
