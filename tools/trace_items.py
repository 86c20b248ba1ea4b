"""All per-item stamps of one expand launch for one CTA (clock64 cycles, relative): producer start /
issued, MMA got tempty / got full / MMAs issued / committed, epilogue got tfull / done."""
import sys, ctypes
import numpy as np, torch
sys.path.insert(0, '.')
from paper_2511_22880_b200 import native
from paper_2511_22880_b200.shapes import LLAMA2_7B, ModelShape
from paper_2511_22880_b200.slab import AdapterSlab
from paper_2511_22880_b200.lora import LoraDeltaEngine
from paper_2511_22880_b200.segments import index_tokens
model = ModelShape("l7b-1l", 1, LLAMA2_7B.projections); dev = torch.device("cuda:0")
ranks = [8]*44+[16]*22+[32]*14+[64]*11+[128]*9
slab = AdapterSlab(model, AdapterSlab.capacity_for(model, ranks), dev)
for i, r in enumerate(ranks):
    s = slab.allocate(f"a{i}", r); slab.fill_random(s, 1000+i)
seg = index_tokens(np.random.default_rng(0).integers(0, 100, 4096), ranks)
eng = LoraDeltaEngine(slab); bp = eng.prepare(seg)
lib = native.lib(); lib.lsv_debug_set_trace.argtypes = [ctypes.c_void_p, ctypes.c_int32]
ITEMS = 64
proj = int(sys.argv[1]); pr = model.projections[proj]
x = torch.randn(4096, pr.h_in, device=dev).to(torch.bfloat16); y = torch.zeros(4096, pr.h_out, device=dev, dtype=torch.bfloat16)
for _ in range(3): eng.apply(bp, 0, proj, x, y)
torch.cuda.synchronize()
buf = torch.zeros(148 * ITEMS * 16, dtype=torch.int64, device=dev)
lib.lsv_debug_set_trace(buf.data_ptr(), ITEMS)
eng.expand(bp, 0, proj, y); torch.cuda.synchronize(); lib.lsv_debug_set_trace(None, 0)
tr = buf.view(148, ITEMS, 16).cpu().numpy().astype(np.int64)
for c in (0, 77):
    cyc = tr[c, :ITEMS - 1, 8:16]
    n = int((cyc[:, 0] > 0).sum()); t0 = cyc[0, 0]
    print(f"cta {c}: {n} items (cycles rel. to item0 producer start)")
    print("   k  prod0  prod1 | mma_te mma_fu mma_is mma_cm | epi_in epi_out")
    for i in range(min(n, 14)):
        v = cyc[i] - t0
        print(f"  {i:2d} {v[0]:6d} {v[1]:6d} | {v[5]:6d} {v[6]:6d} {v[7]:6d} {v[2]:6d} | {v[3]:6d} {v[4]:6d}")

# aggregate over all CTAs (cycles): which stage paces the pipeline
st = {"aux_commit_sync": [], "aux_sync_pop": [], "aux_pop_pre": [], "aux_pre_tempty": [], "epi_busy": [], "mma_wait_tempty": [], "mma_wait_full": [], "mma_issue": [], "item_period": [], "prod_wait": []}
for c in range(148):
    cyc = tr[c, :ITEMS - 1, 8:16]
    n = int((cyc[:, 0] > 0).sum())
    for i in range(1, n):
        ax = tr[c, i, :8]; axp = tr[c, i - 1, :8]
        if ax[1] > 0:   # clock-only build: aux stamps (0 after the loop's syncwarp, 1 after pop, 2 before tempty wait)
            st["aux_commit_sync"].append(axp[0] - cyc[i - 1, 2])
            st["aux_sync_pop"].append(ax[1] - axp[0])
            st["aux_pop_pre"].append(ax[2] - ax[1])
            st["aux_pre_tempty"].append(cyc[i, 5] - ax[2])
        st["epi_busy"].append(cyc[i, 4] - cyc[i, 3])
        st["mma_wait_tempty"].append(cyc[i, 5] - cyc[i - 1, 2])
        st["mma_wait_full"].append(cyc[i, 6] - cyc[i, 5])
        st["mma_issue"].append(cyc[i, 2] - cyc[i, 6])
        st["item_period"].append(cyc[i, 4] - cyc[i - 1, 4])
        st["prod_wait"].append(cyc[i, 1] - cyc[i, 0])
for k, v in st.items():
    v = np.array(v)
    if len(v) == 0: continue
    print(f"{k:16s} mean {v.mean():8.1f}  p50 {np.median(v):8.1f}  p90 {np.percentile(v, 90):8.1f}")
