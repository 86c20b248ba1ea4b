"""Adapter rosters and synthetic request traces (host-side mirror of the reference generator).

Reference: /root/reference/pkg/src/lorasim/traces.py.  The build needs the roster semantics to
size the benchmark configurations (BASELINE.json configs 2/3/5: rank counts apportioned by a
power law over rank index) and the trace generator for config 3's placement-driven batches.
Results are bit-identical to the reference for the same inputs (tests/test_host_parity.py
compares against golden vectors generated from the reference).
"""

from __future__ import annotations

import math
import random
from dataclasses import dataclass, field
from typing import Sequence

from .domain import Adapter, Request

DEFAULT_RANKS = (8, 16, 32, 64, 128)                     # traces.py:23
BYTES_PER_RANK_UNIT = 16 * 1024 * 1024                   # traces.py:25 (rank 128 -> 2 GiB)
ARRIVALS = ("uniform", "poisson")
POPULARITIES = ("uniform", "shifting_skew", "exponential", "power_law")


def assign_power_law_counts(total_adapters: int, ranks: Sequence[int], alpha: float) -> dict[int, int]:
    """Split ``total_adapters`` over ranks proportionally to k^-alpha (k = 1-based rank index).

    Largest-remainder rounding (ties to the lower index) hits the total exactly; a rank left at
    zero borrows one adapter from the currently largest count (ties to the lower index).
    Follows traces.py:94-122.
    """
    order = sorted(ranks)
    n = len(order)
    if total_adapters < n:
        raise ValueError(f"total {total_adapters} cannot give each of {n} ranks an adapter")
    share = [float(k) ** (-alpha) for k in range(1, n + 1)]
    norm = sum(share)
    exact = [total_adapters * w / norm for w in share]
    counts = [int(math.floor(e)) for e in exact]
    missing = total_adapters - sum(counts)
    by_remainder = sorted(range(n), key=lambda i: (counts[i] - exact[i], i))
    for i in by_remainder[:missing]:
        counts[i] += 1
    for i in range(n):
        while counts[i] < 1:
            donor = max(range(n), key=lambda j: (counts[j], -j))
            counts[donor] -= 1
            counts[i] += 1
    return dict(zip(order, counts))


@dataclass(frozen=True)
class LengthModel:
    """Prompt/output lengths: fixed, or lognormal pairs (traces.py:37-56)."""

    kind: str = "fixed"
    prompt: int = 512
    output: int = 128
    prompt_mu: float = 6.0
    prompt_sigma: float = 0.6
    output_mu: float = 4.5
    output_sigma: float = 0.6

    def sample(self, rng: random.Random) -> tuple[int, int]:
        if self.kind == "fixed":
            return self.prompt, self.output
        if self.kind == "lognormal":
            p = max(1, round(rng.lognormvariate(self.prompt_mu, self.prompt_sigma)))
            o = max(1, round(rng.lognormvariate(self.output_mu, self.output_sigma)))
            return p, o
        raise ValueError(f"unknown length model {self.kind!r}")


@dataclass(frozen=True)
class TraceConfig:
    """Synthetic trace parameters (same fields and validation as traces.py:59-91)."""

    duration_seconds: float = 600.0
    target_rps: float = 10.0
    arrival: str = "poisson"
    popularity: str = "uniform"
    popularity_alpha: float = 1.0
    ranks: tuple[int, ...] = DEFAULT_RANKS
    adapters_per_rank: int | None = 5
    total_adapters: int | None = None
    count_skew_alpha: float = 1.0
    lengths: LengthModel = field(default_factory=LengthModel)
    seed: int = 0

    def __post_init__(self):
        if self.target_rps <= 0:
            raise ValueError(f"target_rps must be > 0, got {self.target_rps}")
        if self.duration_seconds <= 0:
            raise ValueError("duration_seconds must be > 0")
        if self.arrival not in ARRIVALS:
            raise ValueError(f"arrival must be one of {ARRIVALS}, got {self.arrival!r}")
        if self.popularity not in POPULARITIES:
            raise ValueError(f"popularity must be one of {POPULARITIES}, got {self.popularity!r}")
        if self.popularity == "power_law" and self.popularity_alpha <= 0:
            raise ValueError("popularity_alpha must be > 0 for power_law popularity")
        if not self.ranks:
            raise ValueError("ranks must be non-empty")
        if self.adapters_per_rank is None and self.total_adapters is None:
            raise ValueError("one of adapters_per_rank / total_adapters is required")
        if self.total_adapters is not None and self.total_adapters < len(self.ranks):
            raise ValueError("total_adapters must cover at least one adapter per rank")


def adapter_counts(cfg: TraceConfig) -> dict[int, int]:
    if cfg.total_adapters is not None:
        return assign_power_law_counts(cfg.total_adapters, cfg.ranks, cfg.count_skew_alpha)
    return {r: cfg.adapters_per_rank for r in sorted(cfg.ranks)}


def trace_adapters(cfg: TraceConfig) -> list[Adapter]:
    """Roster ids ``adapter-r{rank}-{i:03d}``, ``size_bytes = rank * 16 MiB`` (traces.py:131-143)."""
    return [Adapter(id=f"adapter-r{rank}-{i:03d}", rank=rank, size_bytes=rank * BYTES_PER_RANK_UNIT)
            for rank, count in adapter_counts(cfg).items() for i in range(count)]


def roster(total_adapters: int, ranks: Sequence[int] = DEFAULT_RANKS, alpha: float = 1.0) -> list[Adapter]:
    """Power-law roster used by the benchmark configs (100 -> {8:44,16:22,32:14,64:11,128:9})."""
    return trace_adapters(TraceConfig(ranks=tuple(ranks), adapters_per_rank=None,
                                      total_adapters=total_adapters, count_skew_alpha=alpha))


def rank_shares(cfg: TraceConfig, normalized_time: float) -> dict[int, float]:
    """Per-rank request share at t/duration (traces.py:146-169)."""
    ranks = sorted(cfg.ranks)
    n = len(ranks)
    if n == 1:
        return {ranks[0]: 1.0}
    if cfg.popularity == "uniform":
        return {r: 1.0 / n for r in ranks}
    if cfg.popularity in ("exponential", "power_law"):
        if cfg.popularity == "exponential":
            w = [math.exp(-i) for i in range(n)]
        else:
            w = [(i + 1) ** (-cfg.popularity_alpha) for i in range(n)]
        tot = sum(w)
        return {r: wi / tot for r, wi in zip(ranks, w)}
    if cfg.popularity == "shifting_skew":
        tau = min(1.0, max(0.0, normalized_time))
        minor = 0.5 / (n - 1)
        shares = {r: minor for r in ranks}
        shares[ranks[-1]] = 0.5 + (minor - 0.5) * tau
        shares[ranks[0]] = minor + (0.5 - minor) * tau
        return shares
    raise ValueError(f"unknown popularity {cfg.popularity!r}")


def _arrivals(cfg: TraceConfig, rng: random.Random) -> list[float]:
    if cfg.arrival == "uniform":
        gap = 1.0 / cfg.target_rps
        return [i * gap for i in range(int(cfg.duration_seconds * cfg.target_rps))]
    out, t = [], 0.0
    while True:
        t += rng.expovariate(cfg.target_rps)
        if t > cfg.duration_seconds:
            return out
        out.append(t)


def generate_trace(cfg: TraceConfig) -> list[Request]:
    """Arrivals, then per request: rank draw, adapter within rank, lengths (traces.py:187-219)."""
    rng = random.Random(cfg.seed)
    ids_by_rank: dict[int, list[str]] = {}
    for a in trace_adapters(cfg):
        ids_by_rank.setdefault(a.rank, []).append(a.id)
    ranks = sorted(ids_by_rank)
    reqs = []
    for i, t in enumerate(_arrivals(cfg, rng)):
        shares = rank_shares(cfg, t / cfg.duration_seconds)
        u = rng.random()
        acc = 0.0
        pick = ranks[-1]
        for r in ranks:
            acc += shares[r]
            if u < acc:
                pick = r
                break
        pool = ids_by_rank[pick]
        adapter_id = pool[rng.randrange(len(pool))]
        p, o = cfg.lengths.sample(rng)
        reqs.append(Request(request_id=f"req-{i:06d}", adapter=adapter_id, prompt_length=p,
                            output_length=o, arrival_time=t))
    reqs.sort(key=lambda r: r.arrival_time)
    return reqs
