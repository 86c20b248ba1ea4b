"""GPU parity against the published SGMV algorithm's outputs (tests/golden/sgmv_fixtures.npz, made
by vLLM's PyTorch Punica-SGMV restatement; see tests/golden/make_sgmv_fixtures.py).

Every case runs through the C ABI (LoraDeltaEngine -> liblsv), y_in = 0, so the bf16 output is
the delta.  Contract (north star): max|Δ_gpu − Δ_sgmv| / max|Δ_sgmv| ≤ 1e-2.  Each test
also records the error in bf16 ulps of the reference and the fraction of entries equal to the
reference rounded to bf16 (tests/conftest.py prints them at session end and saves
gpurun_out/parity_margins.json)."""

import numpy as np
import pytest

from tests._cases import FIXTURE_CASES, MARGINS, compare_to_fixture, fixture_case

pytestmark = pytest.mark.gpu

TOL = 1e-2
AUTO, SIMT, TC = 0, 1, 2


def _record(request, m, tier):
    m = dict(m, test=f"{request.node.name}", tier=tier)
    MARGINS.append(m)
    return m


@pytest.mark.parametrize("tier", [AUTO, SIMT, TC])
@pytest.mark.parametrize("name", [n for n in FIXTURE_CASES if n != "c2_layer"])
def test_case_matches_sgmv(request, name, tier):
    if tier == SIMT and name in ("token_budget_8192", "one_adapter_8192"):
        pytest.skip("8192-token segments on the decode tier: covered by AUTO/TC")
    case = fixture_case(name)
    y, bp = case.run_gpu(tier_policy=tier)
    n = case.seg.num_tokens
    m = _record(request, compare_to_fixture(y.float().numpy()[:n], name), tier)
    assert m["max_rel_err"] <= TOL, m


@pytest.mark.parametrize("tier", [AUTO, TC])
def test_c2_layer_matches_sgmv(request, tier):
    """One Llama-2-7B layer of config 2 (all 7 projections, 100 adapters, 4096 tokens) through the
    forward path (fused q/k/v and gate/up shrinks, group expands)."""
    case = fixture_case("c2_layer")
    ys, bp = case.run_gpu(tier_policy=tier)
    for pr in case.model.projections:
        m = _record(request, compare_to_fixture(ys[pr.name].float().numpy(), f"c2_layer/{pr.name}"), tier)
        assert m["max_rel_err"] <= TOL, m


@pytest.mark.parametrize("name", ["c1", "ragged", "rank_256", "one_adapter_8192"])
def test_split_v_is_within_one_ulp(request, name):
    """The tensor-core tier's default (hi, lo) v carries v to ~16 bits, so the bf16 output is the
    fp32 SGMV delta correctly rounded up to accumulation noise: at most one bf16 ulp of the
    reference anywhere (floored at max|ref| / 256, tests/_cases.compare_to_fixture)."""
    case = fixture_case(name)
    y, _ = case.run_gpu(tier_policy=TC)
    m = _record(request, compare_to_fixture(y.float().numpy()[:case.seg.num_tokens], name), TC)
    assert m["max_ulps"] <= 1.0 and m["frac_rn_exact"] >= 0.99, m


@pytest.mark.parametrize("name", ["c1", "token_budget_8192"])
def test_bf16_v_mode_within_contract(request, name):
    """LSV_PLAN_V_BF16 (v rounded to one bf16 image before the expand): still inside the contract."""
    case = fixture_case(name)
    y, _ = case.run_gpu(tier_policy=TC, v_bf16=True)
    m = _record(request, compare_to_fixture(y.float().numpy()[:case.seg.num_tokens], name), "tc/v_bf16")
    assert m["max_rel_err"] <= TOL, m
