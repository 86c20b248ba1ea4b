"""SIMT vs tcgen05 tier sweep over segment length n and rank r (the AUTO tier rule's evidence).

    python tools/tier_sweep.py time  > gpurun_out/tier_sweep_time.json
    ncu --metrics <see NCU_METRICS> -k regex:"tc_kernel|simt_" --csv --log-file gpurun_out/tier_ncu.csv \
        python tools/tier_sweep.py ncu
    python tools/tier_sweep.py report gpurun_out/tier_sweep_time.json gpurun_out/tier_ncu.csv > profiles/r2_tier_sweep.txt

Each point is one batch of S segments, all of n tokens and rank r (S = clamp(4096 // n, 16, 256)
distinct adapters), on the gate (4096 -> 11008) and down (11008 -> 4096) shapes, run through
lsv_lora_apply (shrink + expand) with the tier forced (LSV_TIER_SIMT / LSV_TIER_TC).
``time``: CUDA-graph replay of 10 applies, CUDA events, per-apply microseconds and algorithmic
GB/s (SURVEY §8d bytes).  ``ncu``: one apply per point, in the fixed order ``points()``, so the
CSV's launches map back to points (SIMT: shrink, expand; TC: shrink, expand).
"""

from __future__ import annotations

import csv
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

NS = (1, 2, 4, 8, 16, 32, 64, 128, 256)
RS = (8, 16, 32, 64, 128, 256)
SHAPES = {"gate": (4096, 11008), "down": (11008, 4096)}
TIERS = {"simt": 1, "tc": 2}
NCU_METRICS = ("gpu__time_duration.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,"
               "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum")


def points():
    for shape in SHAPES:
        for r in RS:
            for n in NS:
                for tier in TIERS:
                    yield shape, n, r, tier


def segments_for(n):
    return max(16, min(256, 4096 // n))


class Runner:
    """One slab per (shape, r): S adapters of rank r; batches of S segments of n tokens."""

    def __init__(self):
        import torch
        self.torch = torch
        self.dev = torch.device("cuda:0")
        self.cache = {}

    def engine(self, shape, r, tier):
        key = (shape, r, tier)
        if key not in self.cache:
            from paper_2511_22880_b200.lora import LoraDeltaEngine
            from paper_2511_22880_b200.shapes import ModelShape, Projection
            from paper_2511_22880_b200.slab import AdapterSlab
            h_in, h_out = SHAPES[shape]
            model = ModelShape(f"sweep-{shape}", 1, (Projection("p", h_in, h_out),))
            if (shape, r) not in self.cache:
                slab = AdapterSlab(model, AdapterSlab.capacity_for(model, [r] * 256), self.dev)
                for i in range(256):
                    slab.fill_random(slab.allocate(f"a{i}", r), 1000 + i)
                self.cache[(shape, r)] = slab
            self.cache[key] = LoraDeltaEngine(self.cache[(shape, r)], tier_policy=TIERS[tier])
        return self.cache[key]

    def batch(self, shape, n, r, tier):
        from paper_2511_22880_b200.segments import index_requests
        torch = self.torch
        S = segments_for(n)
        seg = index_requests(list(range(S)), [n] * S, [r] * S)
        eng = self.engine(shape, r, tier)
        bp = eng.prepare(seg)
        h_in, h_out = SHAPES[shape]
        N = seg.num_tokens
        x = torch.randn(N, h_in, device=self.dev).to(torch.bfloat16)
        y = torch.zeros(N, h_out, device=self.dev, dtype=torch.bfloat16)
        return eng, bp, x, y, seg

    def time_point(self, shape, n, r, tier, reps=10, replays=20):
        torch = self.torch
        from paper_2511_22880_b200.lora import algorithmic_bytes
        eng, bp, x, y, seg = self.batch(shape, n, r, tier)
        st = torch.cuda.Stream(self.dev)
        with torch.cuda.stream(st):
            eng.apply(bp, 0, 0, x, y, st)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            for _ in range(reps):
                eng.apply(bp, 0, 0, x, y, st)
        with torch.cuda.stream(st):
            g.replay()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            for _ in range(replays):
                g.replay()
            e1.record(st)
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / (reps * replays)
        h_in, h_out = SHAPES[shape]
        nb = algorithmic_bytes(seg, h_in, h_out)
        return {"shape": shape, "n": n, "r": r, "tier": tier, "segments": seg.num_segments, "us": us,
                "GBps": nb / (us * 1e-6) / 1e9, "bytes": nb}

    def ncu_point(self, shape, n, r, tier):
        eng, bp, x, y, seg = self.batch(shape, n, r, tier)
        self.torch.cuda.synchronize()
        eng.apply(bp, 0, 0, x, y)
        self.torch.cuda.synchronize()


def report(time_json, ncu_csv=None):
    rows = json.loads(Path(time_json).read_text())
    by = {(d["shape"], d["n"], d["r"], d["tier"]): d for d in rows}
    ncu = {}
    if ncu_csv and Path(ncu_csv).exists():
        # launches in points() order: two per point (shrink, expand)
        kern = []
        with open(ncu_csv) as f:
            lines = [ln for ln in f if ln.startswith('"')]
        rd = csv.DictReader(lines)
        cur = None
        for row in rd:
            key = (row["ID"], row["Kernel Name"])
            if key != cur:
                kern.append({"name": row["Kernel Name"]})
                cur = key
            try:
                kern[-1][row["Metric Name"]] = float(row["Metric Value"].replace(",", ""))
            except ValueError:
                pass
        it = iter(kern)
        for pt in points():
            ks = [next(it, None), next(it, None)]
            ncu[pt] = ks
    out = []
    out.append("# SIMT vs tcgen05 tier sweep (tools/tier_sweep.py): one batch of S segments of (n tokens, rank r),")
    out.append("# S = clamp(4096 // n, 16, 256); lsv_lora_apply with the tier forced; CUDA-graph replay, CUDA events.")
    out.append("# us = per apply (shrink + expand); GB/s = SURVEY 8d algorithmic bytes / time.")
    if ncu:
        out.append("# ncu (one apply per point, cold, serialised): dram% = gpu__dram_throughput of the longer kernel,")
        out.append("# tc% = sm__pipe_tc_cycles_active (pct of peak sustained active) of the tensor-core kernels.")
    for shape in SHAPES:
        out.append(f"\n== {shape} {SHAPES[shape][0]}->{SHAPES[shape][1]}")
        out.append(f"{'r':>4} {'n':>4} {'S':>4} | {'simt us':>9} {'GB/s':>6} | {'tc us':>9} {'GB/s':>6} | win  "
                   + ("| simt dram% | tc dram% tc-pipe%" if ncu else ""))
        for r in RS:
            for n in NS:
                a, b = by.get((shape, n, r, "simt")), by.get((shape, n, r, "tc"))
                if not a or not b:
                    continue
                win = "simt" if a["us"] < b["us"] else "tc"
                line = (f"{r:>4} {n:>4} {a['segments']:>4} | {a['us']:>9.1f} {a['GBps']:>6.0f} | {b['us']:>9.1f} "
                        f"{b['GBps']:>6.0f} | {win:4s} ")
                if ncu:
                    def dram(ks):
                        ks = [k for k in ks if k]
                        if not ks:
                            return float("nan")
                        k = max(ks, key=lambda k: k.get("gpu__time_duration.sum", 0))
                        return k.get("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", float("nan"))
                    sa, sb = ncu.get((shape, n, r, "simt"), []), ncu.get((shape, n, r, "tc"), [])
                    tcp = max((k.get("sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active", 0.0)
                               for k in sb if k), default=float("nan"))
                    line += f"| {dram(sa):9.1f} | {dram(sb):8.1f} {tcp:8.1f}"
                out.append(line)
        # crossover per rank: smallest n from which tc wins at every larger n
        out.append("crossover (smallest n with tc faster at it and every longer n):")
        for r in RS:
            wins = [(n, by[(shape, n, r, "tc")]["us"] < by[(shape, n, r, "simt")]["us"]) for n in NS
                    if (shape, n, r, "tc") in by and (shape, n, r, "simt") in by]
            xo = None
            for i, (n, w) in enumerate(wins):
                if all(ww for _, ww in wins[i:]):
                    xo = n
                    break
            out.append(f"  r={r:>3}: n >= {xo}")
    return "\n".join(out)


def main():
    mode = sys.argv[1] if len(sys.argv) > 1 else "time"
    if mode == "report":
        print(report(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else None))
        return
    run = Runner()
    if mode == "time":
        res = [run.time_point(*pt) for pt in points()]
        print(json.dumps(res))
    elif mode == "ncu":
        for pt in points():
            run.ncu_point(*pt)
        print("ncu points done", file=sys.stderr)


if __name__ == "__main__":
    main()
