"""Generate golden vectors for the host-side mirror of the reference API by running the reference
itself (/root/reference/pkg/src/lorasim, importable in the build container only).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes tests/golden/host_policy.json.  Floats are stored as float.hex() so the parity tests in
tests/test_host_parity.py compare bit-for-bit.  The GPU box never runs this script; the JSON is
committed and is all the tests need.
"""

from __future__ import annotations

import json
import random
import sys
from collections import deque
from pathlib import Path

REF = Path("/root/reference/pkg/src")
sys.path.insert(0, str(REF))

from lorasim import costmodel, demand, domain, placement, pool, routing, simengine, traces  # noqa: E402

OUT = Path(__file__).resolve().parent / "host_policy.json"
RANKS = (8, 16, 32, 64, 128)


def hx(v: float) -> str:
    return float(v).hex()


def enc_assignment(a: domain.Assignment):
    return {"generation": a.generation,
            "per_server": [[s, [[aid, hx(phi)] for aid, phi in a.per_server[s]]] for s in a.per_server]}


def rand_instance(rng: random.Random):
    k = rng.randint(1, 12)
    n = rng.randint(1, 120)
    ranks_used = rng.sample(RANKS, rng.randint(1, 5))
    adapters = []
    for i in range(n):
        r = rng.choice(ranks_used)
        adapters.append(domain.Adapter(id=f"a{i:03d}-r{r}", rank=r, size_bytes=r * 1024))
    rng.shuffle(adapters)
    tps = sorted((rng.uniform(200.0, 6000.0) for _ in RANKS), reverse=True)
    op = {r: t for r, t in zip(RANKS, tps)}
    dem = {}
    for a in adapters:
        u = rng.random()
        dem[a.id] = 0.0 if u < 0.05 else (1.0 if u < 0.15 else rng.expovariate(1.0 / 300.0))
    return list(range(k)), adapters, dem, op


def gen_placement(rng):
    cases = []
    # SPEC.md:161-181 hand trace (K=4, ranks {8,128}, demand {3000,1000}, op {2000,1000})
    ads = [domain.Adapter("A1", 8, 1), domain.Adapter("A2", 8, 1), domain.Adapter("A3", 8, 1),
           domain.Adapter("B1", 128, 1)]
    dem = {"A1": 1000.0, "A2": 800.0, "A3": 1200.0, "B1": 1000.0}
    op = {8: 2000.0, 128: 1000.0}
    specs = [([0, 1, 2, 3], ads, dem, op)]
    for _ in range(150):
        specs.append(rand_instance(rng))
    for servers, ads, dem, op in specs:
        opt = domain.OperatingPointTable(op)
        fresh = placement.place_from_demand(servers, ads, demand.DemandEstimate(dict(dem)), opt)
        dem2 = {a: v * rng.uniform(0.5, 1.5) for a, v in dem.items()}
        relabeled = placement.place_from_demand(servers, ads, demand.DemandEstimate(dem2), opt, previous=fresh)
        cases.append({
            "servers": servers, "adapters": [[a.id, a.rank, a.size_bytes] for a in ads],
            "demand": [[k, hx(v)] for k, v in dem.items()], "demand2": [[k, hx(v)] for k, v in dem2.items()],
            "op_points": [[r, hx(v)] for r, v in op.items()],
            "fresh": enc_assignment(fresh), "relabeled": enc_assignment(relabeled),
        })
    return cases


def gen_baselines(rng):
    out = []
    for i in range(20):
        servers, ads, _, _ = rand_instance(rng)
        out.append({"servers": servers, "adapters": [[a.id, a.rank, a.size_bytes] for a in ads], "seed": i,
                    "random": enc_assignment(placement.place_random(servers, ads, seed=i)),
                    "contiguous": enc_assignment(placement.place_contiguous(servers, ads))})
    return out


def gen_routing(rng, placements):
    out = []
    for case in placements[:12]:
        per = {s: [(aid, float.fromhex(p)) for aid, p in bundle] for s, bundle in case["relabeled"]["per_server"]}
        asg = domain.Assignment(per_server=per, generation=case["relabeled"]["generation"])
        table = routing.build_routing_table(asg)
        ids = [a[0] for a in case["adapters"]]
        r = random.Random(f"{len(out)}:route")
        reqs = [domain.Request(f"q{i}", rng.choice(ids), 10, 5, float(i)) for i in range(300)]
        out.append({"assignment": case["relabeled"], "adapters": [q.adapter for q in reqs],
                    "seed": f"{len(out)}:route",
                    "servers": [routing.route(q, table, r) for q in reqs]})
    top = []
    for i in range(100):
        p = costmodel.CostParams(tp=rng.choice([1, 2, 4, 8]))
        snaps = [routing.ServerSnapshot(s, rng.choice([0.0, rng.uniform(0, 3)]), rng.choice([0] + list(RANKS)))
                 for s in rng.sample(range(16), rng.randint(1, 8))]
        req = domain.Request("t", "x", rng.randint(1, 4000), 5, 0.0)
        rank = rng.choice(RANKS)
        top.append({"tp": p.tp, "snaps": [[s.server, hx(s.backlog_seconds), s.pending_max_rank] for s in snaps],
                    "prompt": req.prompt_length, "rank": rank,
                    "server": routing.route_toppings(req, snaps, rank, p)})
    return out, top


def gen_pool(rng):
    out = []
    for c in range(10):
        servers = list(range(rng.randint(1, 6)))
        ids = [f"ad{i}" for i in range(rng.randint(1, 12))]
        sizes = {a: rng.randint(1, 4) * (1 << 24) for a in ids}
        slots = rng.randint(1, 4)
        p = pool.AdapterPool(servers, sizes, gpu_slots=slots)
        ops, results = [], []
        for a in ids:
            holders = rng.sample(servers, rng.randint(1, len(servers)))
            p.register(a, holders)
            ops.append(["register", a, holders])
        params = costmodel.CostParams()
        for _ in range(80):
            a = rng.choice(ids)
            s = rng.choice(servers)
            kind = rng.random()
            if kind < 0.3:
                p.touch_gpu(s, a)
                ops.append(["touch", s, a])
                results.append(None)
            elif kind < 0.7:
                loads = {x: rng.choice([0.0, rng.uniform(0, 5)]) for x in servers}
                fp = p.plan_fetch(a, s, params, loads)
                ops.append(["plan", a, s, [[x, hx(v)] for x, v in loads.items()]])
                results.append([fp.kind, fp.size_bytes, hx(fp.latency_s), fp.source])
            else:
                routes = {}
                for x in ids:
                    hs = rng.sample(servers, rng.randint(1, len(servers)))
                    w = [rng.random() + 0.01 for _ in hs]
                    t = sum(w)
                    routes[x] = [(h, wi / t) for h, wi in zip(hs, w)]
                table = domain.RoutingTable.build(routes)
                ev = p.commit_migration(a, s, table)
                ops.append(["commit", a, s, [[x, [[h, hx(v)] for h, v in e]] for x, e in table.routes.items()]])
                results.append(sorted(ev))
        out.append({"servers": servers, "sizes": sizes, "slots": slots, "ops": ops, "results": results,
                    "final": {a: sorted(p.lookup(a)) for a in ids},
                    "max_resident": [[s, p.max_resident[s]] for s in servers],
                    "coverage": p.coverage_ok()})
    return out


def gen_costmodel(rng):
    out = []
    for _ in range(200):
        p = costmodel.CostParams(tp=rng.choice([1, 2, 4, 8]), token_budget=rng.choice([8192, 4096, 100000]))
        n = rng.randint(1, 6)
        lens = [rng.randint(1, 1500) for _ in range(n)]
        ranks = [rng.choice((0,) + RANKS) for _ in range(n)]
        res = rng.choice([0, 8, 128])
        try:
            pf = hx(costmodel.prefill_time(lens, ranks, p, resident_max_rank=res))
        except ValueError as e:
            pf = "ValueError"
        out.append({"tp": p.tp, "budget": p.token_budget, "lens": lens, "ranks": ranks, "res": res, "prefill": pf,
                    "decode": hx(costmodel.decode_iter_time(lens, ranks, p)),
                    "fetch": [hx(costmodel.fetch_latency(l * 4096, s, p)) for l, s in
                              zip(lens, ["host", "remote_rdma", "ssd"] * 3)]})
    cal = []
    for lo, hi, tp, ratio, preset in [(8, 128, 1, 2.7, "7B"), (8, 128, 1, 2.7, "70B"), (8, 128, 8, 1.2, "30B"),
                                      (16, 64, 2, 1.5, "7B"), (64, 64, 1, 1.0, "7B")]:
        p = costmodel.calibrate([costmodel.RatioAnchor(lo, hi, tp, ratio)], model_preset=preset)
        cal.append({"anchor": [lo, hi, tp, hx(ratio)], "preset": preset, "rank_coef": hx(p.rank_coef),
                    "prefill_token_s": hx(p.prefill_token_s), "prefill_base_s": hx(p.prefill_base_s)})
    return out, cal


def gen_traces(rng):
    counts = [[t, hx(a), {str(k): v for k, v in traces.assign_power_law_counts(t, RANKS, a).items()}]
              for t in (5, 6, 7, 10, 25, 50, 100, 333, 1000) for a in (0.5, 1.0, 1.5, 2.0)]
    gens = []
    for pop in traces.POPULARITIES:
        for arr in traces.ARRIVALS:
            cfg = traces.TraceConfig(duration_seconds=60.0, target_rps=5.0, arrival=arr, popularity=pop,
                                     adapters_per_rank=None, total_adapters=25, count_skew_alpha=1.0,
                                     lengths=traces.LengthModel(kind="lognormal"), seed=7)
            reqs = traces.generate_trace(cfg)[:200]
            gens.append({"popularity": pop, "arrival": arr,
                         "requests": [[r.request_id, r.adapter, r.prompt_length, r.output_length, hx(r.arrival_time)]
                                      for r in reqs]})
    return counts, gens


def gen_demand(rng):
    out = []
    for _ in range(20):
        ids = [f"d{i}" for i in range(rng.randint(1, 6))]
        w = rng.choice([1.0, 2.5, 10.0])
        h = demand.TpsHistory(w, ids, depth=rng.randint(2, 5), floor_tps=rng.choice([0.0, 1.0, 3.0]))
        ops = []
        t = 0.0
        for _ in range(rng.randint(1, 60)):
            t += rng.uniform(0, 2.0 * w)
            if rng.random() < 0.8:
                a = rng.choice(ids)
                tok = rng.randint(0, 900)
                h.record_request(a, tok, t)
                ops.append(["rec", a, tok, hx(t)])
            else:
                h.advance_to(t)
                ops.append(["adv", hx(t)])
        out.append({"window": hx(w), "ids": ids, "depth": h.depth, "floor": hx(h.floor_tps), "ops": ops,
                    "linear": [[a, hx(v)] for a, v in h.demand_estimate("linear").per_adapter.items()],
                    "ewma": [[a, hx(v)] for a, v in h.demand_estimate("ewma", 0.3).per_adapter.items()]})
    return out


def gen_schedule(rng):
    out = []
    for _ in range(60):
        p = costmodel.CostParams(token_budget=rng.choice([512, 2048, 8192]))
        srv = simengine.ServerSim(0)
        reqs = []
        for i in range(rng.randint(0, 25)):
            r = domain.Request(f"r{i}", f"ad{rng.randint(0, 5)}", rng.randint(1, min(p.token_budget, 1500)),
                               rng.randint(1, 50), rng.uniform(0, 10))
            rs = simengine.RequestState(r, rng.choice(RANKS))
            rs.ready = rng.random() < 0.8
            rs.solo_prefill_s = costmodel.prefill_time([r.prompt_length], [rs.rank], p)
            srv.wait_queue.append(rs)
            srv.committed_prefill_s += rs.solo_prefill_s
            reqs.append([r.request_id, r.adapter, rs.rank, r.prompt_length, hx(r.arrival_time), rs.ready])
        decodes = []
        for i in range(rng.randint(0, 4)):
            r = domain.Request(f"d{i}", "adx", 5, 5, 0.0)
            rs = simengine.RequestState(r, rng.choice(RANKS))
            rs.context = rng.randint(1, 900)
            srv.running_decodes.append(rs)
            decodes.append([r.request_id, rs.rank, rs.context])
        now = rng.uniform(5, 15)
        timeout = rng.choice([2.0, 5.0, 120.0])
        d = simengine.schedule_server(srv, now, p, timeout)
        out.append({"budget": p.token_budget, "requests": reqs, "decodes": decodes, "now": hx(now),
                    "timeout": hx(timeout), "kind": d.kind, "batch": [rs.req.request_id for rs in d.batch],
                    "duration": hx(d.duration), "ejected": [rs.req.request_id for rs in d.ejected],
                    "queue_after": [rs.req.request_id for rs in srv.wait_queue],
                    "committed_after": hx(srv.committed_prefill_s)})
    return out


def main():
    rng = random.Random(20261018)
    placements = gen_placement(rng)
    routes, toppings = gen_routing(rng, placements)
    cm, cal = gen_costmodel(rng)
    counts, gens = gen_traces(rng)
    doc = {"generator": "tests/golden/make_golden.py (reference: /root/reference/pkg/src/lorasim)",
           "placement": placements, "baselines": gen_baselines(rng), "routing": routes, "toppings": toppings,
           "pool": gen_pool(rng), "costmodel": cm, "calibrate": cal, "power_law_counts": counts,
           "traces": gens, "demand": gen_demand(rng), "schedule": gen_schedule(rng)}
    OUT.write_text(json.dumps(doc, separators=(",", ":")))
    print(f"wrote {OUT} ({OUT.stat().st_size / 1e6:.2f} MB)")


if __name__ == "__main__":
    main()
