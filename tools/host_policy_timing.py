"""the host-side policy on this path, timed on the host cores — this repo's
placement (Algorithm 1, place_from_demand) per rebalance and route() per request, beside the
reference's own code (imported from /root/reference when present, this container only).
    python tools/host_policy_timing.py
"""
import random
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def bench(place_mod, route_mod, dom, dem_mod, k=8, n=1000, reps=5):
    rng = random.Random(0)
    ads = [dom.Adapter(f"a{i}", rng.choice((8, 16, 32, 64, 128)), 1) for i in range(n)]
    op = dom.OperatingPointTable({8: 4800.0, 16: 3800.0, 32: 3280.0, 64: 2600.0, 128: 1560.0})
    dem = dem_mod.DemandEstimate({a.id: rng.expovariate(1 / 200) for a in ads})
    times = []
    asg = None
    for _ in range(reps):
        t0 = time.perf_counter()
        asg = place_mod.place_from_demand(list(range(k)), ads, dem, op)
        times.append(time.perf_counter() - t0)
    table = route_mod.build_routing_table(asg)
    reqs = [dom.Request(f"r{i}", ads[i % n].id, 128, 32, 0.0) for i in range(20000)]
    r = random.Random("0:route")
    t0 = time.perf_counter()
    for q in reqs:
        route_mod.route(q, table, r)
    t_route = (time.perf_counter() - t0) / len(reqs)
    return sorted(times)[len(times) // 2], t_route, asg


def main():
    from paper_2511_22880_b200 import demand, domain, placement, routing
    ours = bench(placement, routing, domain, demand)
    print(f"this repo : place_from_demand(1000 adapters, K=8) {ours[0] * 1e3:7.2f} ms   route {ours[1] * 1e6:6.2f} us/request")
    ref = Path("/root/reference/pkg/src")
    if ref.exists():
        sys.path.insert(0, str(ref))
        from lorasim import demand as rdem, domain as rdom, placement as rpl, routing as rrt
        theirs = bench(rpl, rrt, rdom, rdem)
        print(f"reference : place_from_demand(1000 adapters, K=8) {theirs[0] * 1e3:7.2f} ms   route {theirs[1] * 1e6:6.2f} us/request")
        same = {s: list(v) for s, v in ours[2].per_server.items()} == {s: list(v) for s, v in theirs[2].per_server.items()}
        print(f"placements identical: {same}")


if __name__ == "__main__":
    main()
