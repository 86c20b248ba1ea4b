"""Seeded synthetic workloads for the BASELINE.json configurations.

Inputs are synthetic by necessity (no network for checkpoints or datasets): random-init
adapters (A ~ N(0, 1/h_in), B ~ N(0, 1/r), seed 1000 + adapter index) and N(0, 1)
activations; rosters follow the reference's power-law apportioning
(traces.assign_power_law_counts, traces.py:94-122); token -> adapter assignment is a uniform
draw per token from random.Random(seed).
"""

from __future__ import annotations

import random
from dataclasses import dataclass

import numpy as np

from . import shapes, traces
from .segments import Segments, index_requests, index_tokens


@dataclass
class Workload:
    name: str
    model: shapes.ModelShape
    ranks: list[int]          # rank of each adapter slot
    adapter_ids: list[str]
    segments: Segments
    description: str


def c1_qproj(seed: int = 0) -> Workload:
    """Config 1: Llama-7B q_proj (4096x4096), 4 adapters r=8/16/64/128, 256 tokens (4 x 64)."""
    ranks = [8, 16, 64, 128]
    seg = index_requests([0, 1, 2, 3], [64, 64, 64, 64], ranks)
    return Workload("c1_qproj", shapes.LLAMA7B_QPROJ, ranks, [f"adapter-r{r}-000" for r in ranks], seg,
                    "llama-7b q_proj 4096x4096, 4 adapters r=8/16/64/128, 4x64 tokens")


def c2_llama2_7b(n_tokens: int = 4096, n_adapters: int = 100, seed: int = 0) -> Workload:
    """Config 2: Llama-2-7B all projections, 100 power-law adapters r=8..128, 4096-token batch."""
    roster = traces.roster(n_adapters)
    ranks = [a.rank for a in roster]
    rng = random.Random(seed)
    tok = [rng.randrange(n_adapters) for _ in range(n_tokens)]
    seg = index_tokens(np.asarray(tok), ranks)
    counts = traces.assign_power_law_counts(n_adapters, traces.DEFAULT_RANKS, 1.0)
    return Workload("c2_llama2_7b", shapes.LLAMA2_7B, ranks, [a.id for a in roster], seg,
                    f"llama-2-7b 32 layers x 7 proj, {n_adapters} adapters {counts}, {n_tokens} tokens")


WORKLOADS = {"c1": c1_qproj, "c2": c2_llama2_7b}
