"""GPU parity of the mixed-rank LoRA delta (liblsv via the C ABI) against the CPU oracle.

Tolerance (north star): max|Δ_gpu − Δ_cpu| / max|Δ_cpu| ≤ 1e-2 per projection,
with y_in = 0 so the bf16 output IS the delta.  Operands are bf16, accumulation fp32; the
tcgen05 tier carries v as a bf16 (hi, lo) pair (~16 bits; LSV_PLAN_V_BF16 rounds it to bf16).
"""

import numpy as np
import pytest
import torch

from oracle import oracle
from tests._cases import Case

pytestmark = pytest.mark.gpu

TOL = 1e-2
AUTO, SIMT, TC = 0, 1, 2


def _check(case, tier=AUTO, tol=TOL):
    y, bp = case.run_gpu(tier_policy=tier)
    ref = case.oracle_delta()
    n = case.seg.num_tokens
    got = y.float().numpy()
    err = oracle.max_rel_err(got[:n], ref[:n])
    assert err <= tol, f"max rel err {err:.3e} > {tol} (tier {tier}, summary {bp.shape_plans})"
    return err, bp


@pytest.mark.parametrize("tier", [AUTO, SIMT, TC])
def test_config1_qproj_4_adapters(tier):
    """BASELINE config 1: q_proj 4096x4096, ranks 8/16/64/128, 256-token batch (4 x 64)."""
    case = Case(4096, 4096, [64, 64, 64, 64], [8, 16, 64, 128], seed=1)
    err, bp = _check(case, tier)
    summ = bp.shape_plans[(4096, 4096)].summary
    if tier == SIMT:
        assert summ[5] == 0  # no tensor-core tiles
    else:
        assert summ[5] == 4  # four 64-token tiles on tcgen05


@pytest.mark.parametrize("h_in,h_out", [(4096, 11008), (11008, 4096), (5120, 13824), (8192, 1024), (4096, 1152)])
def test_llama_projection_shapes(h_in, h_out):
    case = Case(h_in, h_out, [41, 7, 130, 64, 1, 256], [128, 8, 32, 16, 64, 8], seed=2)
    _check(case)


def test_ragged_segments_both_tiers():
    lengths = [1, 3, 8, 9, 17, 127, 128, 129, 300, 0, 5]
    ranks = [8, 16, 32, 64, 128, 8, 16, 32, 64, 128, 24]
    case = Case(4096, 4096, lengths, ranks, seed=3)
    err, bp = _check(case)
    s = bp.shape_plans[(4096, 4096)].summary
    assert s[4] > 0 and s[5] > 0  # both tiers used


@pytest.mark.parametrize("tier", [AUTO, TC])
def test_every_rank_class_on_tensor_cores(tier):
    """Ranks that are not multiples of 16/32/64 exercise the K padding and each v-image swizzle."""
    ranks = [8, 16, 24, 32, 40, 48, 56, 64, 72, 96, 112, 128]
    lengths = [9, 17, 33, 64, 100, 128, 129, 20, 47, 5, 61, 90]
    case = Case(4096, 1024, lengths, ranks, seed=8)
    err, bp = _check(case, tier)
    assert bp.shape_plans[(4096, 1024)].summary[5] >= 10


def test_accumulates_into_y_and_leaves_other_rows():
    case = Case(4096, 4096, [50, 70], [16, 64], seed=4, y_scale=1.0, extra_tokens=9)
    y, _ = case.run_gpu()
    n = case.seg.num_tokens
    ref = case.y0.float().numpy()[:n] + case.oracle_delta()[:n]
    err = oracle.max_rel_err(y.float().numpy()[:n] - case.y0.float().numpy()[:n],
                             ref - case.y0.float().numpy()[:n])
    assert err <= 2e-2
    # tokens outside every segment are bit-identical
    assert torch.equal(y[n:], case.y0[n:])


def test_bit_deterministic():
    case = Case(4096, 11008, [41] * 20, [8, 16, 32, 64, 128] * 4, seed=5)
    outs, _ = case.run_gpu(repeat=3)
    assert torch.equal(outs[0], outs[1]) and torch.equal(outs[1], outs[2])


def test_many_segments_splitk():
    """C2-like: 100 adapters, 4096 tokens (exercises k-split reduction and LPT lists)."""
    rng = np.random.default_rng(6)
    ranks = [8] * 44 + [16] * 22 + [32] * 14 + [64] * 11 + [128] * 9
    lengths = np.bincount(rng.integers(0, 100, 4096), minlength=100).tolist()
    case = Case(4096, 4096, lengths, ranks, seed=6)
    err, bp = _check(case)
    assert bp.shape_plans[(4096, 4096)].summary[6] > bp.shape_plans[(4096, 4096)].summary[5]


def test_pack_roundtrip():
    from paper_2511_22880_b200.shapes import ModelShape, Projection
    from paper_2511_22880_b200.slab import AdapterSlab
    model = ModelShape("m", 2, (Projection("p", 4096, 11008), Projection("q", 11008, 4096),
                                Projection("o", 1024, 1152)))
    slab = AdapterSlab(model, 64 << 20, "cuda:0")
    g = torch.Generator(device="cuda:0").manual_seed(0)
    for r in (8, 24, 128):
        slot = slab.allocate(f"r{r}", r)
        for layer in range(2):
            for p, pr in enumerate(model.projections):
                a = torch.randn(r, pr.h_in, generator=g, device="cuda:0").to(torch.bfloat16)
                b = torch.randn(pr.h_out, r, generator=g, device="cuda:0").to(torch.bfloat16)
                slab.load(slot, layer, p, a, b)
                a2, b2 = slab.read(slot, layer, p)
                assert torch.equal(a, a2) and torch.equal(b, b2)


def test_shrink_expand_split_equals_apply():
    case = Case(4096, 4096, [64, 33, 200], [32, 8, 128], seed=7)
    y_ref, bp = case.run_gpu()
    from paper_2511_22880_b200.lora import LoraDeltaEngine
    from paper_2511_22880_b200.slab import AdapterSlab
    slab = AdapterSlab(case.model, 64 << 20, "cuda:0")
    for s, r in enumerate(case.ranks):
        slot = slab.allocate(f"a{s}", r)
        slab.load(slot, 0, 0, case.a[s].cuda(), case.b[s].cuda())
    eng = LoraDeltaEngine(slab)
    bp2 = eng.prepare(case.seg)
    y = case.y0.cuda()
    eng.shrink(bp2, 0, 0, case.x.cuda())
    eng.expand(bp2, 0, 0, y)
    torch.cuda.synchronize()
    assert torch.equal(y.cpu(), y_ref)


@pytest.mark.parametrize("h_in,h_out", [(11008, 4096), (4096, 11008), (1024, 2816)])
def test_decode_regime_simt(h_in, h_out):
    """Decode-shaped batches forced onto the SIMT tier: 1-8-token segments (the expand's 2-token
    passes, odd counts), ranks 8..256, and h_in up to 11008 (several shrink k-splits whose partials
    the expand sums in split order)."""
    lengths = [1, 2, 3, 1, 5, 8, 1, 2, 7, 4, 1, 6, 2, 1]
    ranks = [8, 16, 32, 64, 128, 256, 8, 200, 24, 40, 136, 16, 64, 8]
    case = Case(h_in, h_out, lengths, ranks, seed=12)
    err, bp = _check(case, SIMT)
    s = bp.shape_plans[(h_in, h_out)].summary
    assert s[5] == 0   # every segment on the SIMT tier
    outs, _ = case.run_gpu(tier_policy=SIMT, repeat=2)
    assert torch.equal(outs[0], outs[1])   # deterministic k-split sums


def test_full_token_budget_batch():
    """The reference's token budget (CostParams.token_budget = 8192, costmodel.py:54): a batch of
    8192 tokens over 60 power-law adapters on the gate projection shape."""
    rng = np.random.default_rng(40)
    ranks = [8] * 26 + [16] * 13 + [32] * 9 + [64] * 7 + [128] * 5
    lengths = np.bincount(rng.integers(0, len(ranks), 8192), minlength=len(ranks)).tolist()
    case = Case(4096, 11008, lengths, ranks, seed=40)
    err, bp = _check(case)
    assert bp.shape_plans[(4096, 11008)].summary[1] == 8192


def test_one_adapter_owns_the_whole_batch():
    """A single rank-128 adapter over 8192 tokens: 64 m-tiles of one segment (every tile the same
    B tiles; split-K over the same A for each), on the down projection shape."""
    case = Case(11008, 4096, [8192], [128], seed=41)
    err, bp = _check(case)
    assert bp.shape_plans[(11008, 4096)].summary[5] == 64
