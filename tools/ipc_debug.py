"""Debug CUDA IPC slab sharing between two ranks (torchrun --nproc-per-node 2)."""
import os, sys
import torch, torch.distributed as dist
sys.path.insert(0, '.')
from paper_2511_22880_b200 import native
rank = int(os.environ["RANK"]); world = int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
buf = torch.full((1 << 28,), rank + 1, dtype=torch.uint8, device=f"cuda:{rank}")
torch.cuda.synchronize()
h = buf.untyped_storage()._share_cuda_()
hs = [None] * world
dist.all_gather_object(hs, h)
if rank == 0:
    peer = hs[1]
    print("handle device", peer[0], "size", peer[2], "offset", peer[3], flush=True)
    st = torch.UntypedStorage._new_shared_cuda(*peer)
    print("storage device", st.device, "ptr", hex(st.data_ptr()), "own ptr", hex(buf.data_ptr()), flush=True)
    t = torch.empty(0, dtype=torch.uint8, device=st.device).set_(st)
    print("peer first bytes via torch", t[:4].cpu().tolist(), flush=True)
    rc = native.lib().lsv_enable_peer(0, int(peer[0]))
    print("enable peer rc", rc, native.lib().lsv_last_error(), flush=True)
    # device-0 copy kernel reading the peer pointer
    dst = torch.empty(16, dtype=torch.uint8, device="cuda:0")
    import ctypes
    cudart = ctypes.CDLL("libcudart.so.12")
    rc = cudart.cudaMemcpy(ctypes.c_void_p(dst.data_ptr()), ctypes.c_void_p(st.data_ptr()), ctypes.c_size_t(16), 3)
    torch.cuda.synchronize()
    print("cudaMemcpy D2D from peer rc", rc, dst.cpu().tolist(), flush=True)
    # tensor op on device 0 reading peer data through torch (peer copy)
    d0 = t[:16].to("cuda:0")
    print("torch peer copy", d0.cpu().tolist(), flush=True)
dist.barrier()
dist.destroy_process_group()
