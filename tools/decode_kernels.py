"""Development tool: per-launch time and achieved bandwidth of the decode-regime (SIMT tier)
shrink and expand of every input group, on the bench's decode workload (128 requests x 1 token
over the C2 roster), one layer, CUDA events over repeated launches."""
import sys, zlib
import numpy as np, torch
sys.path.insert(0, '.')
from paper_2511_22880_b200 import synth
from paper_2511_22880_b200.lora import LoraDeltaEngine
from paper_2511_22880_b200.slab import AdapterSlab
from paper_2511_22880_b200.shapes import ModelShape, LLAMA2_7B

B = int(sys.argv[1]) if len(sys.argv) > 1 else 128
wl = synth.decode_llama2_7b(n_requests=B)
model = ModelShape("l7b-1l", 1, LLAMA2_7B.projections); dev = torch.device("cuda:0")
slab = AdapterSlab(model, AdapterSlab.capacity_for(model, wl.ranks), dev)
for aid, r in zip(wl.adapter_ids, wl.ranks):
    slab.fill_random(slab.allocate(aid, r), 1000 + zlib.crc32(aid.encode()) % 100000)
eng = LoraDeltaEngine(slab)
seg = wl.segments
bp = eng.prepare(seg); N = seg.num_tokens
rs = np.asarray(seg.seg_rank, dtype=np.int64)
print(f"B={B}: {seg.num_segments} segments, sum rank {rs.sum()}, tokens {N}")
REPS = 50
for gi, (gname, members) in enumerate(eng.groups):
    h_in = model.projections[members[0]].h_in
    x = torch.randn(N, h_in, device=dev).to(torch.bfloat16)
    ys = [torch.zeros(N, model.projections[p].h_out, device=dev, dtype=torch.bfloat16) for p in members]
    for _ in range(3):
        eng.shrink(bp, 0, members[0], x); eng.expand_group(bp, 0, gi, ys)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    ev[0].record()
    for _ in range(REPS): eng.shrink(bp, 0, members[0], x)
    ev[1].record()
    for _ in range(REPS): eng.expand_group(bp, 0, gi, ys)
    ev[2].record(); torch.cuda.synchronize()
    t_s = ev[0].elapsed_time(ev[1]) / REPS * 1e3
    t_e = ev[1].elapsed_time(ev[2]) / REPS * 1e3
    a_bytes = int(rs.sum()) * h_in * 2 * len(members) + N * h_in * 2
    h_outs = [model.projections[p].h_out for p in members]
    b_bytes = int(rs.sum()) * sum(h_outs) * 2 + 4 * N * sum(h_outs)
    print(f"{gname:9s} shrink {t_s:7.2f} us {a_bytes/1e6:7.1f} MB {a_bytes/t_s/1e3:7.0f} GB/s | "
          f"expand {t_e:7.2f} us {b_bytes/1e6:7.1f} MB {b_bytes/t_e/1e3:7.0f} GB/s")
