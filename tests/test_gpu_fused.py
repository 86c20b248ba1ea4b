"""The base projection GEMM with the LoRA delta fused into its TMEM tile (
lsv_lora_fused_linear through LoraDeltaEngine.linear_group), against oracle(base) + oracle(delta):

    y_p = x · W_p^T + (x · A_s^T) · B_s^T            (segment s of each token)

The base GEMM's reference is a float64 numpy product of the same bf16 operands; the delta's is the
C oracle (pinned to the published SGMV algorithm, tests/test_sgmv_fixtures.py).  Contract as for
the delta: max|y_gpu − y_ref| / max|y_ref| ≤ 1e-2, y bf16 (written once)."""

import math

import numpy as np
import pytest
import torch

from oracle import oracle
from tests._cases import MARGINS, bf16_bits, bf16_ulp

pytestmark = pytest.mark.gpu

TOL = 1e-2


def _run(names_houts, h_in, lengths, ranks, seed, v_bf16=False, extra_tokens=0, tier=0):
    from paper_2511_22880_b200.lora import LoraDeltaEngine
    from paper_2511_22880_b200.segments import Segments
    from paper_2511_22880_b200.shapes import ModelShape, Projection
    from paper_2511_22880_b200.slab import AdapterSlab
    dev = torch.device("cuda:0")
    model = ModelShape("fused", 1, tuple(Projection(nm, h_in, h) for nm, h in names_houts))
    slab = AdapterSlab(model, AdapterSlab.capacity_for(model, ranks), dev)
    g = torch.Generator().manual_seed(seed)
    a, b = {}, {}
    for s, r in enumerate(ranks):
        slot = slab.allocate(f"a{s}", r)
        for p, pr in enumerate(model.projections):
            a[(s, p)] = (torch.randn(r, h_in, generator=g) / math.sqrt(h_in)).to(torch.bfloat16)
            b[(s, p)] = (torch.randn(pr.h_out, r, generator=g) / math.sqrt(r)).to(torch.bfloat16)
            slab.load(slot, 0, p, a[(s, p)].to(dev), b[(s, p)].to(dev))
    indptr = np.concatenate(([0], np.cumsum(lengths))).astype(np.int32)
    seg = Segments(np.arange(indptr[-1], dtype=np.int32), indptr, np.arange(len(ranks), dtype=np.int32),
                   np.asarray(ranks, dtype=np.int32), np.arange(len(ranks), dtype=np.int32))
    n = int(indptr[-1]) + extra_tokens
    x = torch.randn(n, h_in, generator=g).to(torch.bfloat16)
    ws = [(torch.randn(pr.h_out, h_in, generator=g) / math.sqrt(h_in)).to(torch.bfloat16) for pr in model.projections]
    eng = LoraDeltaEngine(slab, tier_policy=tier, v_bf16=v_bf16)
    bp = eng.prepare(seg, fused_linear=True)
    ys = [torch.full((n, pr.h_out), float("nan"), dtype=torch.bfloat16, device=dev) for pr in model.projections]
    eng.linear_group(bp, 0, 0, x.to(dev), [w.to(dev) for w in ws], ys)
    torch.cuda.synchronize()
    out = []
    xf = oracle.bf16_bits_to_f32(bf16_bits(x)).astype(np.float64)
    for p, pr in enumerate(model.projections):
        base = xf @ oracle.bf16_bits_to_f32(bf16_bits(ws[p])).astype(np.float64).T
        delta = oracle.delta_c(bf16_bits(x), seg.seg_indptr, seg.seg_rank, [bf16_bits(a[(s, p)]) for s in range(len(ranks))],
                               [bf16_bits(b[(s, p)]) for s in range(len(ranks))], pr.h_out).astype(np.float64)
        ref = base + delta
        got = ys[p].float().cpu().numpy().astype(np.float64)
        err = oracle.max_rel_err(got, ref)
        floor = float(np.max(np.abs(ref))) / 256
        ulps = float(np.max(np.abs(got - ref) / bf16_ulp(np.maximum(np.abs(ref), floor))))
        out.append({"key": f"fused/{pr.name}", "max_rel_err": err, "max_ulps": ulps,
                    "frac_rn_exact": float(np.mean(got == oracle.bf16_bits_to_f32(oracle.f32_to_bf16_bits(ref.astype(np.float32))))),
                    "delta_share": float(np.max(np.abs(delta)) / max(np.max(np.abs(ref)), 1e-30))})
    return out, bp


@pytest.mark.parametrize("v_bf16", [False, True])
def test_fused_qkv_group_ragged(request, v_bf16):
    """q/k/v in one launch; segments straddle 128-token tile boundaries, a 1-token segment, rank
    256 (4 K chunks of its v image), rank 24 (SWIZZLE_32B v image with a k pad), a partial last tile."""
    res, bp = _run([("q_proj", 512), ("k_proj", 256), ("v_proj", 256)], 1024,
                   [5, 100, 60, 1, 90, 44], [8, 64, 128, 16, 24, 256], seed=3, v_bf16=v_bf16)
    for m in res:
        MARGINS.append(dict(m, test=request.node.name, tier="fused"))
        assert m["max_rel_err"] <= TOL, m
    if not v_bf16:
        assert all(m["max_ulps"] <= 1.0 for m in res), res


def test_fused_config1_qproj(request):
    """BASELINE config 1 as a fused linear layer: q_proj 4096x4096, ranks 8/16/64/128, 4 x 64 tokens
    (two segments per 128-token tile)."""
    res, _ = _run([("q_proj", 4096)], 4096, [64, 64, 64, 64], [8, 16, 64, 128], seed=1)
    for m in res:
        MARGINS.append(dict(m, test=request.node.name, tier="fused"))
        assert m["max_rel_err"] <= TOL and m["max_ulps"] <= 1.0, m


def test_fused_mlp_in_many_segments(request):
    """gate/up (4096 -> 11008, 43 n-tiles each) over 40 segments and 1000 tokens."""
    rng = np.random.default_rng(9)
    ranks = ([8] * 18 + [16] * 9 + [32] * 6 + [64] * 4 + [128] * 3)
    lengths = np.bincount(rng.integers(0, len(ranks), 1000), minlength=len(ranks)).tolist()
    res, bp = _run([("gate_proj", 11008), ("up_proj", 11008)], 4096, lengths, ranks, seed=9)
    for m in res:
        MARGINS.append(dict(m, test=request.node.name, tier="fused"))
        assert m["max_rel_err"] <= TOL and m["max_ulps"] <= 1.0, m


def test_fused_rejects_a_plan_that_is_not_tile_aligned():
    from paper_2511_22880_b200.lora import LoraDeltaEngine
    from paper_2511_22880_b200.segments import index_requests
    from paper_2511_22880_b200.shapes import ModelShape, Projection
    from paper_2511_22880_b200.slab import AdapterSlab
    model = ModelShape("m", 1, (Projection("o_proj", 1024, 512),))
    slab = AdapterSlab(model, AdapterSlab.capacity_for(model, [8]), "cuda:0")
    slab.fill_random(slab.allocate("a", 8), 1)
    eng = LoraDeltaEngine(slab)
    seg = index_requests([0], [10], [8])
    x = torch.zeros(10, 1024, dtype=torch.bfloat16, device="cuda:0")
    w = torch.zeros(512, 1024, dtype=torch.bfloat16, device="cuda:0")
    y = torch.zeros(10, 512, dtype=torch.bfloat16, device="cuda:0")
    with pytest.raises(ValueError):
        eng.linear_group(eng.prepare(seg), 0, 0, x, [w], [y])
    bp = eng.prepare(seg, fused_linear=True)
    with pytest.raises(ValueError):          # the expand cannot consume tile-aligned images
        eng.apply(bp, 0, 0, x, y)
