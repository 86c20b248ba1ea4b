"""Small delta-path invocations for compute-sanitizer (memcheck / racecheck / synccheck).

    compute-sanitizer --tool memcheck python tools/sanitize_cases.py [case ...]

Cases (all through the C ABI, one GPU):
  c1       BASELINE config 1 (q_proj 4096x4096, ranks 8/16/64/128, 4 x 64 tokens), AUTO tier
  splitk   C2-like 100-adapter batch on one projection (split-K shrink: partials, grid barrier,
           grid-wide reduction), AUTO tier
  fwd_tc   2-layer Llama-2-7B-shaped forward (lsv_lora_forward: fused q/k/v + gate/up shrinks,
           group expands, PDL overlap), tensor-core tier, 24 adapters
  fwd_simt the same forward forced onto the SIMT tier (k-split shrink partials, expand sums)
  decode   decode-shaped batch (1-8 token segments, ranks 8..256) on AUTO (SIMT tier)
Each case checks its result against the CPU oracle, so a sanitizer run also shows the kernels
computed the right thing under instrumentation.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from oracle import oracle  # noqa: E402  (checker only)
from tests._cases import Case, bf16_bits  # noqa: E402


def run_case(case: Case, tier: int, label: str) -> None:
    y, bp = case.run_gpu(tier_policy=tier)
    n = case.seg.num_tokens
    err = oracle.max_rel_err(y.float().numpy()[:n], case.oracle_delta()[:n])
    print(f"{label}: max rel err {err:.3e} plan {bp.shape_plans}", flush=True)
    assert err <= 1e-2, err


def run_forward(tier: int, label: str) -> None:
    from paper_2511_22880_b200 import shapes
    from paper_2511_22880_b200.lora import LoraDeltaEngine
    from paper_2511_22880_b200.segments import index_tokens
    from paper_2511_22880_b200.shapes import ModelShape, input_group
    from paper_2511_22880_b200.slab import AdapterSlab
    model = ModelShape("llama-2-7b-2-layers", 2, shapes.LLAMA2_7B.projections)
    ranks = [8] * 10 + [16] * 5 + [32] * 4 + [64] * 3 + [128] * 2
    rng = np.random.default_rng(3)
    seg = index_tokens(rng.integers(0, len(ranks), 512), ranks)
    dev = torch.device("cuda:0")
    slab = AdapterSlab(model, AdapterSlab.capacity_for(model, ranks), dev)
    g = torch.Generator().manual_seed(5)
    w = {}
    for i, r in enumerate(ranks):
        slot = slab.allocate(f"a{i}", r)
        assert slot == i
        for layer in range(2):
            for p, pr in enumerate(model.projections):
                a = (torch.randn(r, pr.h_in, generator=g) / pr.h_in ** 0.5).to(torch.bfloat16)
                b = (torch.randn(pr.h_out, r, generator=g) / r ** 0.5).to(torch.bfloat16)
                slab.load(slot, layer, p, a.to(dev), b.to(dev))
                w[(i, layer, p)] = (a, b)
    eng = LoraDeltaEngine(slab, tier_policy=tier)
    bp = eng.prepare(seg)
    n = seg.num_tokens
    xs, ys = [], []
    for layer in range(2):
        xd = {}
        for pr in model.projections:
            grp = input_group(pr.name)
            if grp not in xd:
                xd[grp] = torch.randn(n, pr.h_in, generator=g).to(torch.bfloat16)
        xs.append(xd)
        ys.append({pr.name: torch.zeros(n, pr.h_out, dtype=torch.bfloat16) for pr in model.projections})
    xs_d = [{k: v.to(dev) for k, v in d.items()} for d in xs]
    ys_d = [{k: v.to(dev) for k, v in d.items()} for d in ys]
    eng.forward(bp, xs_d, ys_d)
    torch.cuda.synchronize()
    worst = 0.0
    for layer in range(2):
        for p, pr in enumerate(model.projections):
            x = xs[layer][input_group(pr.name)]
            ref = oracle.delta_c(bf16_bits(x), seg.seg_indptr, seg.seg_rank,
                                 [bf16_bits(w[(int(s), layer, p)][0]) for s in seg.seg_slot],
                                 [bf16_bits(w[(int(s), layer, p)][1]) for s in seg.seg_slot], pr.h_out)
            worst = max(worst, oracle.max_rel_err(ys_d[layer][pr.name].float().cpu().numpy(), ref))
    print(f"{label}: 2 layers x 7 projections, max rel err {worst:.3e}", flush=True)
    assert worst <= 1e-2, worst


def main(names) -> None:
    AUTO, SIMT, TC = 0, 1, 2
    rng = np.random.default_rng(6)
    todo = {
        "c1": lambda: run_case(Case(4096, 4096, [64] * 4, [8, 16, 64, 128], seed=1), AUTO, "c1"),
        "splitk": lambda: run_case(
            Case(4096, 4096, np.bincount(rng.integers(0, 100, 4096), minlength=100).tolist(),
                 [8] * 44 + [16] * 22 + [32] * 14 + [64] * 11 + [128] * 9, seed=6), AUTO, "splitk"),
        "fwd_tc": lambda: run_forward(TC, "fwd_tc"),
        "fwd_simt": lambda: run_forward(SIMT, "fwd_simt"),
        "decode": lambda: run_case(Case(4096, 4096, [1, 2, 3, 1, 5, 8, 1, 2, 7, 4],
                                        [8, 16, 32, 64, 128, 256, 8, 200, 24, 40], seed=12), AUTO, "decode"),
    }
    for name in names or list(todo):
        todo[name]()
    print("sanitize cases done", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:])
