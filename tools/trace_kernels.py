"""Device timeline of the tcgen05 kernels (debug): per-item globaltimer stamps per role."""
import ctypes, sys
import numpy as np
import torch
sys.path.insert(0, '.')
from paper_2511_22880_b200 import native
from paper_2511_22880_b200.shapes import LLAMA2_7B, ModelShape
from paper_2511_22880_b200.slab import AdapterSlab
from paper_2511_22880_b200.lora import LoraDeltaEngine
from paper_2511_22880_b200.segments import index_tokens

proj = int(sys.argv[1]) if len(sys.argv) > 1 else 0
kind = sys.argv[2] if len(sys.argv) > 2 else "expand"
model = ModelShape("l7b-1l", 1, LLAMA2_7B.projections)
dev = torch.device("cuda:0")
ranks = [8]*44+[16]*22+[32]*14+[64]*11+[128]*9
slab = AdapterSlab(model, AdapterSlab.capacity_for(model, ranks), dev)
for i, r in enumerate(ranks):
    s = slab.allocate(f"a{i}", r); slab.fill_random(s, 1000+i)
seg = index_tokens(np.random.default_rng(0).integers(0, 100, 4096), ranks)
eng = LoraDeltaEngine(slab)
bp = eng.prepare(seg)
pr = model.projections[proj]
x = torch.randn(4096, pr.h_in, device=dev).to(torch.bfloat16)
y = torch.zeros(4096, pr.h_out, device=dev, dtype=torch.bfloat16)
lib = native.lib()
lib.lsv_debug_set_trace.argtypes = [ctypes.c_void_p, ctypes.c_int32]
ITEMS = 64
buf = torch.zeros(148 * ITEMS * 16, dtype=torch.int64, device=dev)
for _ in range(2):
    eng.apply(bp, 0, proj, x, y)
torch.cuda.synchronize()
lib.lsv_debug_set_trace(buf.data_ptr(), ITEMS)
if kind == "expand":
    eng.shrink(bp, 0, proj, x); torch.cuda.synchronize(); buf.zero_()
    eng.expand(bp, 0, proj, y)
else:
    buf.zero_(); eng.shrink(bp, 0, proj, x)
torch.cuda.synchronize()
lib.lsv_debug_set_trace(None, 0)
tt = buf.view(148, ITEMS, 16).cpu().numpy().astype(np.float64)
t = tt[:, :, :8].copy(); cyc = tt[:, :, 8:]
valid = t[:, :, 0] > 0
t0 = t[valid][:, 0].min()
t = np.where(t > 0, t - t0, np.nan) / 1000.0  # us
print(f"{kind} proj {pr.name}: items/cta median {np.median(valid.sum(1))}, max {valid.sum(1).max()}")
names = (["claimed", "issued", "mma_commit", "epi_start", "epi_end", "unused"] if kind == "expand" else
         ["item_start", "all_issued", "mma_commit", "epi_start", "epi_written", "reduced"])
end = np.nanmax(t[:, :, :6])
print(f"kernel span (first issue -> last stamp) {end:.1f} us")
for k in range(1, 6 if kind != 'expand' else 5):
    d = t[:, :, k] - t[:, :, k - 1]
    print(f"  {names[k-1]:>16s} -> {names[k]:<12s} median {np.nanmedian(d):7.2f} us  p90 {np.nanpercentile(d, 90):7.2f}")
if kind == "expand":
    for a, b, nm in [(3, 5, "epi_start->chunk1"), (3, 6, "epi_start->loop_end"), (6, 7, "fence+syncwarp"), (7, 4, "arrives")]:
        d = t[:, :, b] - t[:, :, a]
        print(f"  {nm:>28s} median {np.nanmedian(d):7.2f} us  p90 {np.nanpercentile(d, 90):7.2f}")
a, b = (3, 6) if kind == "expand" else (0, 1)
dcyc = cyc[:, :, b] - cyc[:, :, a]; dns = tt[:, :, b] - tt[:, :, a]
ok = (tt[:, :, a] > 0) & (tt[:, :, b] > 0) & (dns > 2000)
print(f"  effective SM clock during the kernel: {np.median(dcyc[ok] / dns[ok]):.3f} GHz (n={ok.sum()})")
if kind == "expand":
    for a2, b2, nm in [(3, 5, "chunk0 cycles"), (5, 6, "chunk1 cycles"), (6, 7, "fence cycles"), (7, 4, "arrive cycles"), (4, 3, "to next start (neg=ok)")]:
        d = cyc[:, :, b2] - cyc[:, :, a2]
        m = (tt[:, :, a2] > 0) & (tt[:, :, b2] > 0)
        print(f"  {nm:>28s} median {np.median(d[m]):9.0f}  p10 {np.percentile(d[m],10):9.0f} p90 {np.percentile(d[m], 90):9.0f}")
ep = t[:, :, 3]
gaps = np.diff(ep, axis=1)
print(f"  epilogue start-to-start median {np.nanmedian(gaps):.2f} us")
for c in [0, 1, 74, 147]:
    row = t[c][valid[c]]
    print(f"cta {c}: " + " | ".join("/".join(f"{v:.1f}" for v in r[:6]) for r in row[:8]))
