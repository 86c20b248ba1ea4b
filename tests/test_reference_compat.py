"""The reference's own unit-test expectations (pkg/tests/test_costmodel.py, test_domain.py,
test_demand.py), restated against this package's mirror so the modelled drop-in keeps the
reference semantics, plus the SPEC acceptance properties for placement/routing."""

import itertools
import random

import pytest
from hypothesis import given, strategies as st

from paper_2511_22880_b200 import costmodel as cm
from paper_2511_22880_b200 import demand, domain, placement, routing

GIB = 1024 ** 3


# ---- cost model (reference test_costmodel.py:21-145) ---------------------------------------
def test_rank_ratio_anchor_2_7():
    p = cm.calibrate([cm.RatioAnchor(8, 128, 1, 2.7)], cm.CostParams(tp=1))
    assert cm.prefill_time([2000], [128], p) / cm.prefill_time([2000], [8], p) == pytest.approx(2.7, abs=0.05)


def test_rank_zero_is_base_model_and_mixed_pays_max():
    p = cm.CostParams(tp=1)
    assert cm.prefill_time([500], [0], p) == pytest.approx(p.prefill_base_s + 500 * p.prefill_token_s)
    assert cm.prefill_time([1000, 1000], [8, 128], p) == cm.prefill_time([1000, 1000], [128, 128], p)
    assert cm.prefill_time([100], [8], p, resident_max_rank=128) == pytest.approx(cm.prefill_time([100], [128], p))


def test_prefill_errors():
    with pytest.raises(ValueError):
        cm.prefill_time([101], [8], cm.CostParams(token_budget=100))
    with pytest.raises(ValueError):
        cm.prefill_time([], [], cm.CostParams())
    with pytest.raises(ValueError):
        cm.prefill_time([1, 2], [8], cm.CostParams())


@given(st.integers(1, 4000), st.integers(1, 4000), st.integers(0, 128), st.integers(0, 128),
       st.sampled_from([1, 2, 4, 8]))
def test_monotone_in_tokens_rank_and_tp(l1, l2, r1, r2, tp):
    p = cm.CostParams(tp=tp)
    if l1 <= l2 and r1 <= r2:
        assert cm.prefill_time([l1], [r1], p) <= cm.prefill_time([l2], [r2], p)
    assert cm.prefill_time([l1], [r1], cm.CostParams(tp=tp * 2)) <= cm.prefill_time([l1], [r1], p)


def test_decode_terms():
    p = cm.CostParams(tp=1)
    assert cm.decode_iter_time([0], [0], p) == pytest.approx(p.decode_base_s)
    p2 = cm.CostParams(tp=2)
    assert cm.decode_iter_time([100], [128], p2) - cm.decode_iter_time([100], [8], p2) == \
        pytest.approx(p2.decode_rank_s * 120 / 2)
    base = cm.decode_iter_time([400], [0], p) - p.decode_base_s
    assert cm.decode_iter_time([800], [0], p) - p.decode_base_s == pytest.approx(2 * base)


def test_fetch_latency():
    p = cm.CostParams(host_bw=20e9, rdma_bw=20e9, ssd_bw=2e9)
    host = cm.fetch_latency(2 * GIB, "host", p)
    assert cm.fetch_latency(2 * GIB, "remote_rdma", p) == pytest.approx(2 * host)
    assert host == pytest.approx(2 * GIB / 20e9)
    assert cm.fetch_latency(2 * GIB, "ssd", p) == pytest.approx(2 * GIB / 2e9)
    with pytest.raises(ValueError):
        cm.fetch_latency(0, "host", p)
    with pytest.raises(ValueError):
        cm.fetch_latency(1, "floppy", p)


@given(st.integers(1, 10 ** 12), st.integers(1, 5), st.sampled_from(["host", "remote_rdma", "ssd"]))
def test_fetch_linear_in_bytes(size, factor, source):
    p = cm.CostParams()
    assert cm.fetch_latency(size * factor, source, p) == pytest.approx(factor * cm.fetch_latency(size, source, p),
                                                                       rel=1e-9)


def test_calibration():
    p = cm.calibrate([cm.RatioAnchor(8, 128, 1, 2.7)])
    assert p.rank_coef == pytest.approx(1.7 / 106.4, rel=1e-12)
    c = p.rank_coef
    assert 1.15 <= (1 + 16 * c) / (1 + c) <= 1.30
    base = cm.CostParams(rank_coef=0.042)
    assert cm.calibrate([cm.RatioAnchor(64, 64, 1, 1.0)], base).rank_coef == base.rank_coef
    with pytest.raises(cm.CalibrationError):
        cm.calibrate([cm.RatioAnchor(8, 128, 1, 0.5)])
    with pytest.raises(cm.CalibrationError):
        cm.calibrate([cm.RatioAnchor(64, 64, 1, 2.0)])
    p70 = cm.calibrate([cm.RatioAnchor(8, 128, 1, 2.7)], model_preset="70B")
    c = p70.rank_coef
    assert (1 + 16 * c) / (1 + c) == pytest.approx(1.45, abs=1e-9)
    assert p70.prefill_token_s == pytest.approx(9 * cm.CostParams().prefill_token_s)
    target = (1 + 16 * 0.016) / (1 + 0.016)
    assert cm.solve_rank_coef(cm.RatioAnchor(8, 128, 8, target)) == pytest.approx(0.016, rel=1e-9)


# ---- domain (reference test_domain.py) -------------------------------------------------------
def test_domain_validation():
    with pytest.raises(ValueError):
        domain.Adapter("a", 0, 1)
    with pytest.raises(ValueError):
        domain.Request("r", "a", 0, 1, 0.0)
    with pytest.raises(ValueError):
        domain.RoutingTable.build({"a": [(0, 0.5), (1, 0.4)]})           # sum too far from 1
    with pytest.raises(ValueError):
        domain.RoutingTable.build({"a": [(0, 0.5), (0, 0.5)]})           # duplicate server
    t = domain.RoutingTable.build({"a": [(0, 0.5), (1, 0.5 + 5e-7)]})   # small drift renormalised
    assert abs(sum(e.phi for e in t.entries("a")) - 1.0) <= domain.PHI_SUM_TOL
    assert domain.validate_routing_table(t, ["a", "b"]) == ["no route entries for b"]
    with pytest.raises(ValueError):
        domain.OperatingPointTable({8: 100.0, 16: 200.0})               # must be non-increasing


@given(st.dictionaries(st.sampled_from([f"a{i}" for i in range(8)]),
                       st.lists(st.tuples(st.integers(0, 5), st.floats(0.01, 1.0)), min_size=1, max_size=4,
                                unique_by=lambda x: x[0]), min_size=1))
def test_assignment_route_roundtrip(raw):
    routes = {a: [(s, w / sum(x for _, x in e)) for s, w in e] for a, e in raw.items()}
    asg = domain.Assignment.from_routes(routes)
    back = asg.to_routes()
    assert {a: sorted(e) for a, e in back.items()} == {a: sorted(e) for a, e in routes.items()}


# ---- demand (reference test_demand.py) ---------------------------------------------------------
def test_demand_windows_and_extrapolation():
    h = demand.TpsHistory(10.0, ["a", "b"], floor_tps=1.0)
    h.record_request("a", 100, 1.0)
    h.record_request("a", 200, 12.0)        # closes window 0: a = 10 tps, b = 0
    assert h.closed_windows("a") == [10.0] and h.closed_windows("b") == [0.0]
    h.advance_to(20.0)                      # closes window 1: a = 20 tps
    assert h.extrapolate("a") == 30.0       # 20 + (20 - 10)
    assert h.extrapolate("b") == 1.0        # floor
    with pytest.raises(ValueError):
        h.record_request("a", 1, 5.0)       # time went backwards
    with pytest.raises(KeyError):
        h.record_request("zz", 1, 30.0)
    with pytest.raises(demand.ColdStartError):
        demand.TpsHistory(1.0, ["a"]).prev_timestep_tps("a")


# ---- SPEC acceptance properties ----------------------------------------------
@given(st.integers(1, 12), st.integers(1, 200), st.integers(0, 10 ** 6))
def test_acceptance2_coverage_and_budgets(k, n, seed):
    rng = random.Random(seed)
    ads = [domain.Adapter(f"a{i}", rng.choice((8, 16, 32, 64, 128)), 1) for i in range(n)]
    op = domain.OperatingPointTable({8: 4800.0, 16: 3800.0, 32: 3280.0, 64: 2600.0, 128: 1560.0})
    dem = demand.DemandEstimate({a.id: rng.expovariate(1 / 200) for a in ads})
    asg = placement.place_from_demand(list(range(k)), ads, dem, op)
    sums = asg.phi_sums()
    assert set(sums) == {a.id for a in ads}
    assert all(abs(v - 1.0) <= 1e-9 for v in sums.values())
    led = placement.compute_utilization(dem, ads, op, k)
    assert 0 <= placement.compute_rank_budgets(led, k).total() <= k


@pytest.mark.parametrize("seed", range(40))
def test_acceptance3_permutation_optimal(seed):
    rng = random.Random(seed)
    k = rng.randint(1, 6)
    ids = [f"a{i}" for i in range(rng.randint(1, 12))]
    dem = demand.DemandEstimate({a: rng.uniform(0, 100) for a in ids})
    def rand_asg():
        return domain.Assignment({s: [(a, rng.uniform(0.1, 1)) for a in rng.sample(ids, rng.randint(0, len(ids)))]
                                  for s in range(k)})
    fresh, prev = rand_asg(), rand_asg()
    out = placement.permute_assignment(fresh, prev, dem)
    m = placement.overlap_matrix(fresh, prev, dem, list(range(k)))
    best = max(sum(m[i][p[i]] for i in range(k)) for p in itertools.permutations(range(k)))
    if not any(prev.per_server.values()):
        return
    got = sum(m[i][j] for i in range(k) for j in range(k) if out.per_server[j] is fresh.per_server[i])
    assert got == pytest.approx(best, abs=1e-9)


def test_acceptance5_routing_converges():
    table = domain.RoutingTable.build({"A3": [(1, 0.7), (2, 0.3)]})
    rng = random.Random(0)
    hits = sum(routing.route(domain.Request("q", "A3", 1, 1, 0.0), table, rng) == 1 for _ in range(100000))
    assert abs(hits / 100000 - 0.7) <= 0.01
