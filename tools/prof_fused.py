"""C2 one-layer fused linear (gate/up group: lsv_lora_fused_linear) for ncu captures; run 3 times,
profile the last with -k regex:fused -s 2 -c 1."""
import sys
import zlib
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2511_22880_b200 import synth  # noqa: E402
from paper_2511_22880_b200.lora import LoraDeltaEngine  # noqa: E402
from paper_2511_22880_b200.shapes import ModelShape  # noqa: E402
from paper_2511_22880_b200.slab import AdapterSlab  # noqa: E402

wl = synth.c2_llama2_7b()
model = ModelShape("l7b-1l", 1, wl.model.projections)
dev = torch.device("cuda:0")
slab = AdapterSlab(model, AdapterSlab.capacity_for(model, wl.ranks), dev)
for aid, r in zip(wl.adapter_ids, wl.ranks):
    slab.fill_random(slab.allocate(aid, r), 1000 + zlib.crc32(aid.encode()) % 100000)
eng = LoraDeltaEngine(slab, v_bf16="--v-bf16" in sys.argv)
bp = eng.prepare(wl.segments, fused_linear=True)
gi = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 2
gname, members = eng.groups[gi]
N = wl.segments.num_tokens
pr0 = model.projections[members[0]]
x = torch.randn(N, pr0.h_in, device=dev).to(torch.bfloat16)
ws = [(torch.randn(model.projections[p].h_out, pr0.h_in, device=dev) / 64).to(torch.bfloat16) for p in members]
ys = [torch.empty(N, model.projections[p].h_out, device=dev, dtype=torch.bfloat16) for p in members]
for _ in range(3):
    eng.linear_group(bp, 0, gi, x, ws, ys)
torch.cuda.synchronize()
print("ok")
