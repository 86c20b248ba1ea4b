"""Segment indexer: stable adapter sort of a FIFO batch (bit-exact integer work)."""

import numpy as np
import pytest
from hypothesis import given, strategies as st

from paper_2511_22880_b200.segments import index_requests, index_tokens


def test_small_batch_golden():
    # FIFO batch as schedule_server would form it (simengine.py:116-137): slots, lengths, ranks
    seg = index_requests([3, 1, 3, 0, 1], [2, 1, 3, 1, 2], [64, 8, 64, 16, 8])
    assert seg.seg_slot.tolist() == [0, 1, 3]
    assert seg.seg_rank.tolist() == [16, 8, 64]
    assert seg.seg_indptr.tolist() == [0, 1, 4, 9]
    # request order stable within an adapter: slot0 req3; slot1 req1, req4; slot3 req0, req2
    assert seg.request_order.tolist() == [3, 1, 4, 0, 2]
    # token starts: req0 0-1, req1 2, req2 3-5, req3 6, req4 7-8
    assert seg.perm.tolist() == [6, 2, 7, 8, 0, 1, 3, 4, 5]
    assert all(a.dtype == np.int32 for a in (seg.perm, seg.seg_indptr, seg.seg_slot, seg.seg_rank))


def test_errors_mirror_prefill_time():
    with pytest.raises(ValueError):
        index_requests([], [], [])
    with pytest.raises(ValueError):
        index_requests([1, 2], [3], [8, 8])
    with pytest.raises(ValueError):
        index_requests([1, 1], [3, 4], [8, 16])  # one slot, two ranks
    with pytest.raises(ValueError):
        index_requests([0], [0], [8])


@given(st.lists(st.tuples(st.integers(0, 12), st.integers(1, 40)), min_size=1, max_size=60))
def test_indexer_invariants(reqs):
    slots = [s for s, _ in reqs]
    lens = [n for _, n in reqs]
    ranks = [8 * (1 + s % 16) for s in slots]
    seg = index_requests(slots, lens, ranks)
    assert seg.num_tokens == sum(lens)
    assert sorted(seg.perm.tolist()) == list(range(sum(lens)))      # a permutation
    assert np.all(np.diff(seg.seg_slot) > 0)                          # ascending, unique
    assert np.all(np.diff(seg.seg_indptr) > 0)
    # every token lands in the segment of its request's slot
    starts = np.concatenate(([0], np.cumsum(lens)))
    owner = np.repeat(np.arange(len(lens)), lens)
    for s in range(seg.num_segments):
        toks = seg.perm[seg.seg_indptr[s]:seg.seg_indptr[s + 1]]
        assert set(np.asarray(slots)[owner[toks]].tolist()) == {int(seg.seg_slot[s])}
        # FIFO within the segment
        assert np.all(np.diff(owner[toks]) >= 0)
    again = index_requests(slots, lens, ranks)
    assert all(np.array_equal(getattr(seg, f), getattr(again, f))
               for f in ("perm", "seg_indptr", "seg_slot", "seg_rank"))


def test_index_tokens_c2_roster():
    ranks = [8] * 44 + [16] * 22 + [32] * 14 + [64] * 11 + [128] * 9
    rng = np.random.default_rng(0)
    tok = rng.integers(0, 100, 4096)
    seg = index_tokens(tok, ranks)
    assert seg.num_tokens == 4096
    assert seg.num_segments == len(set(tok.tolist()))
    assert np.array_equal(np.diff(seg.seg_indptr), np.bincount(tok, minlength=100)[seg.seg_slot])
