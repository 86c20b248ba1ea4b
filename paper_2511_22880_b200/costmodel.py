"""Cost callbacks of the delta path: the reference's boundary, modelled and measured.

The reference prices "apply this co-batched batch's LoRA deltas" with closed forms
(/root/reference/pkg/src/lorasim/costmodel.py):

    prefill_time(prompt_lengths, ranks, params, resident_max_rank=0)   costmodel.py:83-105
    decode_iter_time(context_lengths, ranks, params)                   costmodel.py:108-123
    fetch_latency(size_bytes, source, params)                          costmodel.py:129-143

This module keeps those signatures, errors and (in the default, *modelled* mode) the exact
numbers, so the reference's own cost-model tests pass against it (tests/test_costmodel_compat.py).
``MeasuredCost`` is the drop-in that prices the same call with the B200 path: it runs the batch
through LoraDeltaEngine and returns measured seconds, where each segment pays its own rank
instead of the whole batch paying ``max(ranks)`` (costmodel.py:104).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, replace
from typing import Iterable, NamedTuple, Sequence

from .domain import OperatingPointTable


class CalibrationError(ValueError):
    """The supplied anchors admit no non-negative rank coefficient."""


class ProfilingError(RuntimeError):
    """The SLO is unachievable for a rank even at minimal load."""


@dataclass(frozen=True)
class CostParams:
    """Latency-model coefficients (costmodel.py:29-70; same defaults)."""

    prefill_token_s: float = 0.25e-3
    prefill_base_s: float = 20e-3
    rank_coef: float = 1.7 / 106.4
    tp: int = 1
    decode_base_s: float = 25e-3
    decode_rank_s: float = 0.05e-3
    decode_ctx_s: float = 0.5e-6
    host_bw: float = 20e9
    rdma_bw: float = 20e9
    ssd_bw: float = 2e9
    token_budget: int = 8192

    def __post_init__(self):
        for name in ("prefill_token_s", "prefill_base_s", "rank_coef", "decode_base_s", "decode_rank_s",
                     "decode_ctx_s"):
            if getattr(self, name) < 0:
                raise ValueError(f"{name} must be >= 0")
        for name in ("host_bw", "rdma_bw", "ssd_bw"):
            if getattr(self, name) <= 0:
                raise ValueError(f"{name} must be > 0")
        if self.tp < 1:
            raise ValueError(f"tp must be >= 1, got {self.tp}")
        if self.token_budget < 1:
            raise ValueError(f"token_budget must be >= 1, got {self.token_budget}")

    def rank_factor(self, rank: int) -> float:
        return 1.0 + self.rank_coef * rank / self.tp


MODEL_PRESETS: dict[str, tuple[float, float | None]] = {"7B": (1.0, None), "30B": (4.0, 1.33), "70B": (9.0, 1.45)}


def _check_batch(lengths: Sequence[int], ranks: Sequence[int], what: str) -> None:
    if not lengths:
        raise ValueError(f"{what} batch must be non-empty")
    if len(lengths) != len(ranks):
        raise ValueError(f"{'prompt_lengths' if what == 'prefill' else 'context_lengths'} and ranks "
                         "must have equal length")


def prefill_time(prompt_lengths: Sequence[int], ranks: Sequence[int], params: CostParams,
                 resident_max_rank: int = 0) -> float:
    """Modelled seconds for one co-batched prefill: (base + per-token * total) * rank factor of
    the largest rank present (incl. co-scheduled decodes) — costmodel.py:83-105."""
    _check_batch(prompt_lengths, ranks, "prefill")
    tokens = sum(prompt_lengths)
    if tokens > params.token_budget:
        raise ValueError(f"prefill batch of {tokens} tokens exceeds token budget {params.token_budget}")
    worst = max(max(ranks), resident_max_rank)
    return (params.prefill_base_s + params.prefill_token_s * tokens) * params.rank_factor(worst)


def decode_iter_time(context_lengths: Sequence[int], ranks: Sequence[int], params: CostParams) -> float:
    """Modelled seconds for one decode iteration (costmodel.py:108-123)."""
    _check_batch(context_lengths, ranks, "decode")
    return params.decode_base_s + params.decode_rank_s * max(ranks) / params.tp + \
        params.decode_ctx_s * sum(context_lengths)


FETCH_SOURCES = ("host", "remote_rdma", "ssd")


def fetch_latency(size_bytes: int, source: str, params: CostParams) -> float:
    """Seconds to make an adapter GPU-resident from `source` (costmodel.py:129-143)."""
    if size_bytes <= 0:
        raise ValueError(f"size_bytes must be > 0, got {size_bytes}")
    if source == "host":
        return size_bytes / params.host_bw
    if source == "remote_rdma":
        return size_bytes / params.host_bw + size_bytes / params.rdma_bw
    if source == "ssd":
        return size_bytes / params.ssd_bw
    raise ValueError(f"unknown fetch source {source!r}; expected one of {FETCH_SOURCES}")


class RatioAnchor(NamedTuple):
    rank_lo: int
    rank_hi: int
    tp: int
    ratio: float


def solve_rank_coef(anchor: RatioAnchor) -> float | None:
    """c with (1 + c*hi/tp)/(1 + c*lo/tp) = ratio; None when the anchor does not constrain c
    (costmodel.py:155-175)."""
    lo, hi, tp, ratio = anchor
    if hi == lo:
        if math.isclose(ratio, 1.0):
            return None
        raise CalibrationError(f"equal ranks {lo} cannot produce ratio {ratio}")
    denom = hi - ratio * lo
    if denom <= 0:
        raise CalibrationError(f"anchor {anchor} admits no finite rank coefficient")
    coef = tp * (ratio - 1.0) / denom
    if coef < 0:
        raise CalibrationError(f"anchor {anchor} implies a negative rank coefficient")
    return coef


def calibrate(anchors: Iterable[RatioAnchor], base: CostParams | None = None, model_preset: str = "7B") -> CostParams:
    """Fit the rank coefficient to anchors and apply a model-size preset (costmodel.py:178-212)."""
    base = base or CostParams()
    if model_preset not in MODEL_PRESETS:
        raise CalibrationError(f"unknown model preset {model_preset!r}; expected one of {sorted(MODEL_PRESETS)}")
    solved = [solve_rank_coef(a) for a in anchors]
    coef = next((c for c in solved if c is not None), base.rank_coef)
    scale, tp8_ratio = MODEL_PRESETS[model_preset]
    if tp8_ratio is not None:
        coef = (tp8_ratio - 1.0) / (16.0 - tp8_ratio)
    return replace(base, rank_coef=coef, prefill_token_s=base.prefill_token_s * scale,
                   prefill_base_s=base.prefill_base_s * scale)


# ------------------------------------------------------------------------------------------
class MeasuredCost:
    """B200-measured drop-in for prefill_time / decode_iter_time.

    ``prefill_time(prompt_lengths, ranks)`` builds the batch the reference would price (one
    request per entry, distinct adapters of the given ranks), runs every layer/projection of the
    engine's model through the CUDA path and returns the measured seconds of the delta path
    (median of ``reps`` CUDA-graph-free launches).  Results are cached by the batch signature
    (sorted (length, rank) multiset), so a simulator can call it per batch.  The value is the
    LoRA-delta share of a prefill; the base model's own time is outside this path.
    """

    def __init__(self, engine, reps: int = 3):
        import torch
        self.engine = engine
        self.reps = reps
        self._cache: dict[tuple, float] = {}
        self._torch = torch

    def _measure(self, lengths: Sequence[int], ranks: Sequence[int]) -> float:
        torch = self._torch
        from .lora import input_group
        from .segments import index_requests
        eng = self.engine
        slab = eng.slab
        # one resident adapter per distinct rank in the slab is enough: the cost depends on rank
        by_rank = {}
        for info in slab.slots:
            by_rank.setdefault(info.rank, info.slot)
        missing = sorted(set(int(r) for r in ranks) - set(by_rank))
        if missing:
            raise ValueError(f"no resident adapter of rank(s) {missing} to measure with")
        slots = [by_rank[int(r)] * 0 + i for i, r in enumerate(ranks)]  # distinct segment per request
        seg = index_requests(slots, lengths, ranks)
        # map each request's segment to a resident slot of its rank
        seg = seg.__class__(seg.perm, seg.seg_indptr, seg.seg_slot.copy(), seg.seg_rank, seg.request_order)
        for s in range(seg.num_segments):
            seg.seg_slot[s] = by_rank[int(seg.seg_rank[s])]
        bp = eng.prepare(seg)
        n = seg.num_tokens
        dev = eng.device
        # the step the serving path runs: one fused shrink per input group and one group expand
        # (eng.forward), over a ring of RING distinct per-layer activation sets so the batch's x/y
        # are not served from L2 the way one buffer reused 32 times would be
        ring = 4
        bufs_x, bufs_y = [], []
        for _ in range(ring):
            xs = {}
            for pr in eng.model.projections:
                xs.setdefault(input_group(pr.name), torch.randn(n, pr.h_in, device=dev).to(torch.bfloat16))
            bufs_x.append(xs)
            bufs_y.append({pr.name: torch.zeros(n, pr.h_out, device=dev, dtype=torch.bfloat16)
                           for pr in eng.model.projections})
        L = eng.model.layers
        xs_l = [bufs_x[l % ring] for l in range(L)]
        ys_l = [bufs_y[l % ring] for l in range(L)]
        times = []
        for _ in range(self.reps + 1):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            eng.forward(bp, xs_l, ys_l)
            e1.record()
            torch.cuda.synchronize(dev)
            times.append(e0.elapsed_time(e1) / 1e3)
        times = sorted(times[1:])
        return times[len(times) // 2]

    def prefill_time(self, prompt_lengths: Sequence[int], ranks: Sequence[int], params: CostParams,
                     resident_max_rank: int = 0) -> float:
        """Same contract as the modelled prefill_time; ``resident_max_rank`` is accepted but has no
        effect: on the B200 path a co-scheduled decode's rank does not slow this batch down."""
        _check_batch(prompt_lengths, ranks, "prefill")
        if sum(prompt_lengths) > params.token_budget:
            raise ValueError(f"prefill batch of {sum(prompt_lengths)} tokens exceeds token budget "
                             f"{params.token_budget}")
        key = ("prefill",) + tuple(sorted(zip(map(int, prompt_lengths), map(int, ranks))))
        if key not in self._cache:
            self._cache[key] = self._measure(list(prompt_lengths), list(ranks))
        return self._cache[key]

    def decode_iter_time(self, context_lengths: Sequence[int], ranks: Sequence[int], params: CostParams) -> float:
        """One decode step = one token per request (the BGMV regime, SIMT tier)."""
        _check_batch(context_lengths, ranks, "decode")
        key = ("decode",) + tuple(sorted(map(int, ranks)))
        if key not in self._cache:
            self._cache[key] = self._measure([1] * len(ranks), list(ranks))
        return self._cache[key]


# ------------------------------------------------------------------------------------------
class FittedCost:
    """The B200 measurements as a closed form, usable where no GPU is (the reference simulator,
    ``profile_operating_points`` costmodel.py:215-281; tools/measured_op_points.py).

    tools/measure_cost_fit.py times the delta path (MeasuredCost, Llama-2-7B, every request its
    own segment) and fits, per regime,
        delta = t0 + k_tok * sum(lengths) + k_rank * sum(ranks)
    (the path is HBM-bound and moves X*sum(n) + W*sum(r) bytes).  The prefill /
    decode prices keep the reference's base-model terms and replace its max-rank multiplier
    (costmodel.py:104-105, :121) with that additive rank-aware delta, the rank term divided by
    ``tp`` like ``rank_factor`` (costmodel.py:69-70).  Same signatures and errors as the modelled
    functions."""

    def __init__(self, prefill_fit: dict, decode_fit: dict):
        self.prefill_fit = dict(prefill_fit)
        self.decode_fit = dict(decode_fit)

    @classmethod
    def from_json(cls, path=None) -> "FittedCost":
        import json
        from pathlib import Path
        p = Path(path) if path else Path(__file__).resolve().parent.parent / "tests" / "golden" / "b200_delta_cost.json"
        d = json.loads(p.read_text())
        return cls(d["prefill_fit"], d["decode_fit"])

    @staticmethod
    def _delta(fit: dict, lengths: Sequence[int], ranks: Sequence[int], tp: int) -> float:
        return max(0.0, fit["t0_s"] + fit["k_tok_s"] * sum(lengths) + fit["k_rank_s"] * sum(ranks) / tp)

    def prefill_time(self, prompt_lengths: Sequence[int], ranks: Sequence[int], params: CostParams,
                     resident_max_rank: int = 0) -> float:
        """Base-model prefill + the fitted B200 delta; ``resident_max_rank`` has no effect (a
        co-scheduled decode's rank does not slow this batch on the B200 path)."""
        _check_batch(prompt_lengths, ranks, "prefill")
        tokens = sum(prompt_lengths)
        if tokens > params.token_budget:
            raise ValueError(f"prefill batch of {tokens} tokens exceeds token budget {params.token_budget}")
        return params.prefill_base_s + params.prefill_token_s * tokens + \
            self._delta(self.prefill_fit, prompt_lengths, ranks, params.tp)

    def decode_iter_time(self, context_lengths: Sequence[int], ranks: Sequence[int], params: CostParams) -> float:
        _check_batch(context_lengths, ranks, "decode")
        return params.decode_base_s + params.decode_ctx_s * sum(context_lengths) + \
            self._delta(self.decode_fit, [1] * len(ranks), ranks, params.tp)
