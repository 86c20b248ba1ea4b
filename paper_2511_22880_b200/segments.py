"""Segment indexer: a co-batched prefill batch -> adapter-contiguous segments.

The reference forms each server's prefill batch FIFO under the token budget
(simengine.py:96-152 ``schedule_server``) and prices it with
``costmodel.prefill_time([len...], [rank...])`` (costmodel.py:83-105) — one entry per request,
in batch (FIFO) order.  To apply the batch's LoRA deltas on the GPU the tokens of requests that
share an adapter must be contiguous.  The canonical order used everywhere in this package is a
STABLE sort of the batch by adapter slot (FIFO order preserved within an adapter), giving

    perm        [N] int32  sorted token position -> token index in the FIFO concatenation
    seg_indptr  [S+1] int32, seg_slot [S] int32, seg_rank [S] int32

with segments ordered by ascending slot.  Everything is integer work and bit-exact: the same
batch always yields the same arrays (tests/test_segments.py pins it).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Sequence

import numpy as np


@dataclass(frozen=True)
class Segments:
    perm: np.ndarray        # int32 [N]
    seg_indptr: np.ndarray  # int32 [S+1]
    seg_slot: np.ndarray    # int32 [S]
    seg_rank: np.ndarray    # int32 [S]
    request_order: np.ndarray  # int32 [R]: requests in segment order (stable by slot)

    @property
    def num_tokens(self) -> int:
        return int(self.seg_indptr[-1])

    @property
    def num_segments(self) -> int:
        return int(self.seg_slot.shape[0])

    def lengths(self) -> np.ndarray:
        return np.diff(self.seg_indptr)


def index_requests(slots: Sequence[int], lengths: Sequence[int], ranks: Sequence[int]) -> Segments:
    """Index a batch given per-request adapter slot, token count and rank (FIFO order).

    Mirrors the argument checks of costmodel.prefill_time (costmodel.py:95-98): the batch must
    be non-empty and the per-request sequences must have equal length.  A slot must always
    carry the same rank.
    """
    if len(lengths) == 0:
        raise ValueError("prefill batch must be non-empty")
    if not (len(slots) == len(lengths) == len(ranks)):
        raise ValueError("slots, lengths and ranks must have equal length")
    slots_a = np.asarray(slots, dtype=np.int64)
    lens_a = np.asarray(lengths, dtype=np.int64)
    ranks_a = np.asarray(ranks, dtype=np.int64)
    if np.any(lens_a < 1):
        raise ValueError("every request needs at least one token")
    if np.any(slots_a < 0):
        raise ValueError("adapter slots must be >= 0")
    order = np.argsort(slots_a, kind="stable")
    starts = np.concatenate(([0], np.cumsum(lens_a)[:-1]))
    sorted_slots = slots_a[order]
    boundaries = np.flatnonzero(np.diff(sorted_slots)) + 1
    group_first = np.concatenate(([0], boundaries))
    seg_slot = sorted_slots[group_first]
    seg_rank = ranks_a[order][group_first]
    # a slot must not appear with two different ranks
    rank_of_req = ranks_a[order]
    seg_id_of_req = np.repeat(np.arange(len(group_first)), np.diff(np.concatenate((group_first, [len(order)]))))
    if np.any(rank_of_req != seg_rank[seg_id_of_req]):
        raise ValueError("an adapter slot appears with two different ranks in one batch")
    seg_tokens = np.add.reduceat(lens_a[order], group_first)
    seg_indptr = np.concatenate(([0], np.cumsum(seg_tokens)))
    # tokens of request order[k] are starts[order[k]] + 0..len-1, laid out request after request
    lens_o = lens_a[order]
    excl = np.concatenate(([0], np.cumsum(lens_o)[:-1]))
    perm = np.arange(int(lens_o.sum()), dtype=np.int64) + np.repeat(starts[order] - excl, lens_o)
    return Segments(
        perm=perm.astype(np.int32),
        seg_indptr=seg_indptr.astype(np.int32),
        seg_slot=seg_slot.astype(np.int32),
        seg_rank=seg_rank.astype(np.int32),
        request_order=order.astype(np.int32),
    )


def index_tokens(token_slots: Sequence[int], slot_rank: Sequence[int]) -> Segments:
    """Index a batch given one adapter slot per token (each token its own 1-token request)."""
    slots = np.asarray(token_slots, dtype=np.int64)
    ranks = np.asarray(slot_rank, dtype=np.int64)[slots]
    return index_requests(slots, np.ones_like(slots), ranks)


def tile_counts(seg: Segments, tile_m: int = 128) -> np.ndarray:
    """Number of 128-token tensor-core tiles per segment (planning diagnostics)."""
    return (seg.lengths() + tile_m - 1) // tile_m
