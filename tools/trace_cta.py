"""Per-CTA view of one tcgen05 launch: records, algorithmic bytes, main-loop time and bandwidth
per CTA, plus per-record producer timings (development aid; uses lsv_debug_set_trace)."""
import sys, ctypes
import numpy as np, torch
sys.path.insert(0, '.')
from paper_2511_22880_b200 import native
from paper_2511_22880_b200.shapes import LLAMA2_7B, ModelShape, kpad
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
ITEMS = 96
for arg in sys.argv[1:]:
    kind, proj = arg.split(":"); proj = int(proj); pr = model.projections[proj]
    x = torch.randn(4096, pr.h_in, device=dev).to(torch.bfloat16); y = torch.zeros(4096, pr.h_out, device=dev, dtype=torch.bfloat16)
    for _ in range(3): eng.apply(bp, 0, proj, x, y)
    torch.cuda.synchronize()
    buf = torch.zeros(148 * ITEMS * 16, dtype=torch.int64, device=dev)
    lib.lsv_debug_set_trace(buf.data_ptr(), ITEMS)
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    if kind == "expand": eng.expand(bp, 0, proj, y)
    else: eng.shrink(bp, 0, proj, x)
    e1.record(); torch.cuda.synchronize(); lib.lsv_debug_set_trace(None, 0)
    tr = buf.view(148, ITEMS, 16).cpu().numpy().astype(np.float64)
    plan = bp.shape_plans[(pr.h_in, pr.h_out)].plan_host.view(np.int32)
    off_recs, off_cta, grid = (plan[17], plan[18], plan[10]) if kind == "shrink" else (plan[19], plan[20], plan[11])
    rw = 16 if kind == "shrink" else 8
    recs = plan[off_recs:off_recs + rw * (plan[off_cta + grid])].reshape(-1, rw)
    ph = tr[:, ITEMS - 1, :8]
    t0 = ph[:, 0][ph[:, 0] > 0].min()
    print(f"== {kind} {pr.name}: event {e0.elapsed_time(e1)*1e3:.1f} us, grid {grid}, records {len(recs)}")
    names = ["entry", "prologue", "pdl_wait", "loop_done", "barrier", "reduce_done"]
    for k, nm in enumerate(names):
        v = ph[:, k]; v = v[v > 0]
        if len(v): print(f"  {nm:>12s}: min {(v.min()-t0)/1e3:7.2f} med {(np.median(v)-t0)/1e3:7.2f} max {(v.max()-t0)/1e3:7.2f}")
    rows = []
    for c in range(grid):
        rr = recs[plan[off_cta + c]:plan[off_cta + c + 1]]
        if kind == "shrink":
            b = sum((((r[2] + 7)//8*8) + r[3]) * 128 * (r[5] - r[4]) for r in rr)
        else:
            tw = 256 if pr.h_out % 256 == 0 else 128
            b = sum(tw * kpad(int(r[3])) * 2 + int(r[2]) * tw * 4 for r in rr)
        dt = (ph[c, 3] - ph[c, 2]) / 1e3
        rows.append((c, len(rr), b, dt, b / dt / 1e3 if dt > 0 else 0, (ph[c, 3] - t0) / 1e3))
    a = np.array(rows)
    print(f"  per-CTA bytes  min {a[:,2].min()/1e3:.0f}K med {np.median(a[:,2])/1e3:.0f}K max {a[:,2].max()/1e3:.0f}K; "
          f"records min {a[:,1].min():.0f} max {a[:,1].max():.0f}")
    print(f"  per-CTA loop GB/s min {a[:,4].min():.1f} med {np.median(a[:,4]):.1f} max {a[:,4].max():.1f} "
          f"(x148 = {np.median(a[:,4])*148:.0f})")
    for c in list(np.argsort(a[:, 5])[-3:]) + list(np.argsort(a[:, 5])[:2]):
        c = int(c); rr = recs[plan[off_cta + c]:plan[off_cta + c + 1]]
        print(f"  cta {c}: {len(rr)} recs, {a[c,2]/1e3:.0f} KB, loop {a[c,3]:.2f} us, ends {a[c,5]:.2f}")
        for i in range(min(len(rr), 8)):
            st = (tr[c, i, :6] - t0) / 1e3
            print("     rec", rr[i][:8].tolist(), " prod %.2f-%.2f mma %.2f epi %.2f-%.2f" % tuple(st[[0, 1, 2, 3, 4]]))
