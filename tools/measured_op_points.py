"""Algorithm 1's operating points from the B200 cost instead of the max-rank model.

Runs the reference's own ``profile_operating_points`` (costmodel.py:215-281, which binary-searches
each rank's SLO-attaining load on its single-server simulator, simengine.run_single_server_probe)
twice: with the reference's modelled cost, and with the simulator's cost callbacks
(``lorasim.costmodel.prefill_time`` / ``decode_iter_time``, called by simengine.py:139/146)
replaced by ``FittedCost`` — the B200 measurements of tests/golden/b200_delta_cost.json
(tools/measure_cost_fit.py).  The simulator is the reference's (imported from /root/reference,
this container only); this repo does not rebuild it (SURVEY §8 scope).  Writes
tests/golden/op_points_b200.json, which tests/test_measured_op_points.py checks and which
placement.place_from_demand can consume like any OperatingPointTable.

    python tools/measured_op_points.py [--duration 60] [--slo 10]
"""
import argparse
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, "/root/reference/pkg/src")

RANKS = (8, 16, 32, 64, 128)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--duration", type=float, default=60.0)
    ap.add_argument("--slo", type=float, default=10.0)
    args = ap.parse_args()
    import lorasim.costmodel as rcm
    from paper_2511_22880_b200.costmodel import FittedCost

    params = rcm.CostParams()
    t0 = time.perf_counter()
    modelled = rcm.profile_operating_points(params, args.slo, RANKS, duration_seconds=args.duration, seed=0)
    t1 = time.perf_counter()
    fitted = FittedCost.from_json()
    saved = (rcm.prefill_time, rcm.decode_iter_time)
    try:
        rcm.prefill_time = fitted.prefill_time
        rcm.decode_iter_time = fitted.decode_iter_time
        measured = rcm.profile_operating_points(params, args.slo, RANKS, duration_seconds=args.duration, seed=0)
    finally:
        rcm.prefill_time, rcm.decode_iter_time = saved
    t2 = time.perf_counter()
    out = {
        "what": "per-rank single-server TPS capacity under the SLO (OperatingPointTable.max_tps), from the "
                "reference's profile_operating_points with its modelled cost and with the B200-fitted cost",
        "slo_seconds": args.slo, "duration_seconds": args.duration, "seed": 0, "ranks": list(RANKS),
        "cost_params": "lorasim.costmodel.CostParams() defaults",
        "modelled": {str(r): modelled[r] for r in modelled.ranks()},
        "b200_measured": {str(r): measured[r] for r in measured.ranks()},
        "seconds": {"modelled": round(t1 - t0, 2), "measured": round(t2 - t1, 2)},
    }
    path = ROOT / "tests" / "golden" / "op_points_b200.json"
    path.write_text(json.dumps(out, indent=1))
    for r in RANKS:
        print(f"rank {r:>3}: modelled {modelled[r]:10.1f} tok/s   B200 {measured[r]:10.1f} tok/s")


if __name__ == "__main__":
    main()
