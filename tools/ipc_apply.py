"""Localise IPC-peer apply failures (torchrun --nproc-per-node 2, CUDA_LAUNCH_BLOCKING=1)."""
import os, sys, zlib
import numpy as np, torch, torch.distributed as dist
sys.path.insert(0, '.')
from paper_2511_22880_b200 import synth, native
from paper_2511_22880_b200.slab import AdapterSlab
from paper_2511_22880_b200.lora import LoraDeltaEngine, input_group
from paper_2511_22880_b200.shapes import ModelShape, LLAMA2_7B
rank = int(os.environ["RANK"]); world = int(os.environ["WORLD_SIZE"])
dev = torch.device("cuda", rank); torch.cuda.set_device(dev)
dist.init_process_group("nccl", device_id=dev)
tier = int(sys.argv[1]) if len(sys.argv) > 1 else 0
wl, owner = synth.remote_workload(world, rank)
model = ModelShape("l1", 1, LLAMA2_7B.projections[:1])
slab = AdapterSlab(model, AdapterSlab.capacity_for(model, wl.ranks), dev)
for aid, r in zip(wl.adapter_ids, wl.ranks):
    slab.fill_random(slab.allocate(aid, r), 1000 + zlib.crc32(aid.encode()) % 100000)
torch.cuda.synchronize()
hs = [None] * world
dist.all_gather_object(hs, slab.ipc_handle())
roster = list(zip(wl.adapter_ids, wl.ranks))
peers = {r: AdapterSlab.open_peer(model, hs[r], roster, dev) for r in range(world) if r != rank}
print(rank, "own base", hex(slab.base), "peer bases", {r: hex(p.base) for r, p in peers.items()}, "cap", slab.capacity, flush=True)
eng = LoraDeltaEngine(slab, tier_policy=tier)
seg = wl.segments
x = torch.randn(seg.num_tokens, 4096, device=dev).to(torch.bfloat16)
y1 = torch.zeros(seg.num_tokens, 4096, device=dev, dtype=torch.bfloat16); y2 = torch.zeros_like(y1)
bp = eng.prepare(seg)
eng.apply(bp, 0, 0, x, y1); torch.cuda.synchronize(); print(rank, "local ok", flush=True)
bpr = eng.prepare(seg, seg_owner=owner, peer_slabs=peers)
print(rank, "remote segs", int((owner != rank).sum()), "first remote a_ptr", hex(int(bpr.a_ptrs[0, int(np.argmax(owner != rank))])), flush=True)
eng.shrink(bpr, 0, 0, x); torch.cuda.synchronize(); print(rank, "remote shrink ok", flush=True)
eng.expand(bpr, 0, 0, y2); torch.cuda.synchronize(); print(rank, "remote expand ok", torch.equal(y1, y2), flush=True)
dist.barrier(); dist.destroy_process_group()
