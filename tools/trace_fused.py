"""Per-item clock64 timeline of one fused_linear_kernel launch (C2 mlp_in group by default):
producer item start / base issued / LoRA issued, MMA got tempty / base issued / LoRA issued,
epilogue got tfull / done.  python tools/trace_fused.py [group]"""
import ctypes
import sys
import zlib
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2511_22880_b200 import native, synth  # noqa: E402
from paper_2511_22880_b200.lora import LoraDeltaEngine  # noqa: E402
from paper_2511_22880_b200.shapes import ModelShape  # noqa: E402
from paper_2511_22880_b200.slab import AdapterSlab  # noqa: E402

wl = synth.c2_llama2_7b()
model = ModelShape("l7b-1l", 1, wl.model.projections)
dev = torch.device("cuda:0")
slab = AdapterSlab(model, AdapterSlab.capacity_for(model, wl.ranks), dev)
for aid, r in zip(wl.adapter_ids, wl.ranks):
    slab.fill_random(slab.allocate(aid, r), 1000 + zlib.crc32(aid.encode()) % 100000)
eng = LoraDeltaEngine(slab)
bp = eng.prepare(wl.segments, fused_linear=True)
gi = int(sys.argv[1]) if len(sys.argv) > 1 else 0
gname, members = eng.groups[gi]
N = wl.segments.num_tokens
pr0 = model.projections[members[0]]
x = torch.randn(N, pr0.h_in, device=dev).to(torch.bfloat16)
ws = [(torch.randn(model.projections[p].h_out, pr0.h_in, device=dev) / 64).to(torch.bfloat16) for p in members]
ys = [torch.empty(N, model.projections[p].h_out, device=dev, dtype=torch.bfloat16) for p in members]
for _ in range(3):
    eng.linear_group(bp, 0, gi, x, ws, ys)
torch.cuda.synchronize()
ITEMS = 32
lib = native.lib()
buf = torch.zeros(148 * ITEMS * 16, dtype=torch.int64, device=dev)
lib.lsv_debug_set_trace(buf.data_ptr(), ITEMS)
eng.linear_group(bp, 0, gi, x, ws, ys)
torch.cuda.synchronize()
lib.lsv_debug_set_trace(None, 0)
tr = buf.view(148, ITEMS, 16).cpu().numpy().astype(np.int64)[:, :, 8:16]
for c in (0, 50, 100):
    n = int((tr[c, :, 3] > 0).sum())
    t0 = tr[c, 0, 0]
    print(f"cta {c}: {n} items (cycles rel. to item 0 producer start)")
    print("   k   p_start  p_base  p_lora |  m_tempty  m_base  m_lora |  e_tfull  e_done | m_item  m_lora_dt")
    for i in range(n):
        v = tr[c, i] - t0
        per = (tr[c, i + 1, 3] - tr[c, i, 3]) if i + 1 < n else 0
        print(f"  {i:2d} {v[0]:8d} {v[1]:7d} {v[2]:7d} | {v[3]:8d} {v[4]:7d} {v[5]:7d} | {v[6]:8d} {v[7]:7d} | {per:6d} {v[5] - v[4]:6d}")
