"""liblsv C ABI on the CPU: the library loads, exports every symbol include/lsv.h declares, and
the host planner (no GPU needed) validates input and emits consistent work lists."""

import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

from paper_2511_22880_b200 import native

ROOT = Path(__file__).resolve().parent.parent


def test_library_exports_header_symbols():
    lib = native.load()
    header = (ROOT / "include" / "lsv.h").read_text()
    declared = set(re.findall(r"\b(lsv_[a-z0-9_]+)\s*\(", header))
    assert declared == set(native.EXPORTED_SYMBOLS)
    for name in declared:
        assert hasattr(lib, name), name
    assert lib.lsv_version() == native.ABI_VERSION


def _plan(indptr, ranks, h_in=4096, h_out=4096, policy=0):
    lib = native.load()
    indptr = np.asarray(indptr, dtype=np.int32)
    ranks = np.asarray(ranks, dtype=np.int32)
    pb, wb = ctypes.c_size_t(), ctypes.c_size_t()
    native.check(lib.lsv_plan_size(len(ranks), indptr.ctypes.data, ranks.ctypes.data, h_in, h_out, policy,
                                   ctypes.byref(pb), ctypes.byref(wb)))
    blob = np.zeros(pb.value // 4, dtype=np.int32)
    native.check(lib.lsv_plan_build(len(ranks), indptr.ctypes.data, ranks.ctypes.data, h_in, h_out, policy,
                                    blob.ctypes.data, pb.value))
    return blob, wb.value


def _decode(blob):
    h = blob[:64]
    names = ["magic", "version", "S", "N", "h_in", "h_out", "n_simt", "n_mtiles", "n_shrink", "n_expand",
             "shrink_grid", "expand_grid", "off_indptr", "off_rank", "off_tier", "off_simt", "off_mtiles",
             "off_shrink", "off_shrink_cta", "off_expand", "off_expand_cta", "total_ints"]
    d = {k: int(h[i]) for i, k in enumerate(names)}
    d["mtiles"] = blob[d["off_mtiles"]:d["off_mtiles"] + 8 * d["n_mtiles"]].reshape(-1, 8)
    d["shrink"] = blob[d["off_shrink"]:d["off_shrink"] + 16 * d["n_shrink"]].reshape(-1, 16)
    d["shrink_cta"] = blob[d["off_shrink_cta"]:d["off_shrink_cta"] + d["shrink_grid"] + 1]
    d["expand"] = blob[d["off_expand"]:d["off_expand"] + 8 * d["n_expand"]].reshape(-1, 8)
    d["expand_cta"] = blob[d["off_expand_cta"]:d["off_expand_cta"] + d["expand_grid"] + 1]
    d["simt"] = blob[d["off_simt"]:d["off_simt"] + 4 * d["n_simt"]].reshape(-1, 4)
    d["tier"] = blob[d["off_tier"]:d["off_tier"] + d["S"]]
    return d


@pytest.mark.parametrize("h_in,h_out", [(4096, 4096), (11008, 4096), (4096, 11008)])
def test_plan_covers_every_chunk_and_tile(h_in, h_out):
    rng = np.random.default_rng(0)
    ranks = [8] * 44 + [16] * 22 + [32] * 14 + [64] * 11 + [128] * 9
    lens = np.bincount(rng.integers(0, 100, 4096), minlength=100)
    lens[3] = 0
    lens[5] = 2    # SIMT-tier segment
    lens[7] = 300  # three tensor-core tiles
    indptr = np.concatenate(([0], np.cumsum(lens)))
    blob, ws = _plan(indptr, ranks, h_in, h_out)
    d = _decode(blob)
    assert d["magic"] == 0x5056534C and d["N"] == int(indptr[-1])
    chunks = h_in // 64
    # every mtile's k-range is covered exactly once by its splits (records: ShrinkRec, 16 int32)
    cover = {}
    for rec in d["shrink"]:
        cover.setdefault(int(rec[12]), []).append((int(rec[4]), int(rec[5]), int(rec[7])))
    for i, mt in enumerate(d["mtiles"]):
        parts = sorted(cover[i])
        assert parts[0][0] == 0 and parts[-1][1] == chunks
        assert all(parts[j][1] == parts[j + 1][0] for j in range(len(parts) - 1))
        assert sorted(p[2] for p in parts) == list(range(int(mt[4])))   # split ids 0..nsplit-1
    # every (mtile, h_out tile) appears exactly once in the expand records
    pairs = {(int(r[6]), int(r[4])) for r in d["expand"]}
    tw = 256 if h_out % 256 == 0 else 128
    assert len(pairs) == len(d["expand"]) == d["n_mtiles"] * (h_out // tw)
    # per-CTA record lists partition the record arrays
    for key in ("shrink_cta", "expand_cta"):
        off = d[key]
        assert off[0] == 0 and np.all(np.diff(off) >= 0)
    assert d["shrink_cta"][-1] == d["n_shrink"] and d["expand_cta"][-1] == d["n_expand"]
    assert d["shrink_grid"] <= 148 and d["expand_grid"] <= 148
    # tokens: mtiles + simt items tile every non-empty segment exactly
    covered = np.zeros(d["N"], dtype=int)
    for seg, tb, nt, *_ in d["mtiles"]:
        covered[tb:tb + nt] += 1
    for seg, tb, nt_rank, _ in d["simt"]:       # nt_rank = ntok | rank << 16
        nt = int(nt_rank) & 0xFFFF
        assert int(nt_rank) >> 16 == ranks[seg]
        covered[tb:tb + nt] += 1
    assert np.all(covered == 1)
    assert d["tier"][3] == 0 and d["tier"][5] == 1 and d["tier"][7] == 2
    # LPT balance: the most-loaded CTA carries at most ~2x the mean estimated bytes
    row = np.array([(int(-(-r[2] // 8) * 8) + int(r[3])) * 128 * (int(r[5]) - int(r[4])) for r in d["shrink"]])
    per_cta = np.add.reduceat(row, d["shrink_cta"][:-1]) if len(row) else row
    assert per_cta.max() <= 2.0 * per_cta.mean() + 1.5 * row.max()
    assert ws > 0


def test_plan_rejects_bad_input():
    with pytest.raises(ValueError, match="multiple of 128"):
        _plan([0, 4], [8], h_in=1000)
    with pytest.raises(ValueError, match="rank"):
        _plan([0, 4], [12])
    with pytest.raises(ValueError, match="non-decreasing"):
        _plan([0, 4, 2], [8, 8])
    with pytest.raises(ValueError, match="seg_indptr\\[0\\]"):
        _plan([1, 4], [8])


def test_forced_policies():
    d = _decode(_plan([0, 64, 128], [8, 128], policy=native.TIER_SIMT)[0])
    assert d["n_mtiles"] == 0 and d["n_simt"] == 16
    d = _decode(_plan([0, 2, 130], [8, 256], policy=native.TIER_TC)[0])
    # every segment on tcgen05; rank 256 on 64-token tiles with 128-wide expand items
    assert d["n_mtiles"] == 3 and list(d["tier"]) == [2, 2]
    assert [int(m[2]) for m in d["mtiles"]] == [2, 64, 64]
    items = {(int(r[6]), int(r[4])) for r in d["expand"]}
    assert len(items) == d["n_expand"] == 4096 // 256 + 2 * (4096 // 128)
    # AUTO: a long rank-256 segment is no longer sent to SIMT; a 1-token one is
    d = _decode(_plan([0, 1, 300], [256, 256])[0])
    assert list(d["tier"]) == [1, 2] and d["n_mtiles"] == 5   # 1-token rank 256: SIMT (sweep)


@pytest.mark.parametrize("n,r,tier", [(4, 8, 1), (5, 8, 2), (4, 16, 1), (8, 16, 2), (2, 32, 1), (3, 32, 2),
                                      (1, 64, 1), (2, 64, 2), (1, 128, 2), (1, 256, 1), (2, 256, 2)])
def test_auto_rule_follows_the_tier_sweep(n, r, tier):
    """The AUTO thresholds of profiles/r2_tier_sweep.txt (lsv_api.cu simt_max_tok), in a batch that
    launches the tensor-core tier anyway (a 64-token segment beside the probe)."""
    d = _decode(_plan([0, n, n + 64], [r, 8])[0])
    assert int(d["tier"][0]) == tier and int(d["tier"][1]) == 2


def test_decode_shaped_batches_stay_on_simt():
    """No segment longer than 8 tokens: the whole batch on the SIMT tier (no tcgen05 launches)."""
    d = _decode(_plan([0, 1, 3, 8, 9], [128, 64, 8, 256])[0])
    assert list(d["tier"]) == [1, 1, 1, 1] and d["n_mtiles"] == 0


def test_split_v_doubles_the_v_image_region():
    lib = native.load()
    indptr, ranks = [0, 40, 200, 201], [8, 64, 128]
    regions = []
    for flag in (0, native.PLAN_V_BF16):
        blob, _ = _plan(indptr, ranks, policy=native.TIER_AUTO | flag)
        off, nb = ctypes.c_size_t(), ctypes.c_size_t()
        native.check(lib.lsv_plan_vimg_region(blob.ctypes.data, ctypes.byref(off), ctypes.byref(nb)))
        assert int(blob[61]) == (0 if flag else 1)     # PlanHeader::vsplit
        regions.append(nb.value)
    assert regions[0] == 2 * regions[1]
    with pytest.raises(ValueError, match="flags"):
        _plan(indptr, ranks, policy=0x400)


def test_apply_rejects_missing_plan():
    lib = native.load()
    rc = lib.lsv_lora_apply(None, 0, None, 0, 0, 0, 4096, 4096, None, None, None, None, None, 0, None)
    with pytest.raises(ValueError):
        native.check(rc)
    rc = lib.lsv_lora_apply(None, 0, None, 0, 7, 0, 4096, 4096, None, None, None, None, None, 0, None)
    with pytest.raises(RuntimeError):
        native.check(rc)


def _plan_group(indptr, ranks, h_in, h_outs, policy=0):
    lib = native.load()
    indptr = np.asarray(indptr, dtype=np.int32)
    ranks = np.asarray(ranks, dtype=np.int32)
    hs = np.asarray(h_outs, dtype=np.int32)
    pb, wb = ctypes.c_size_t(), ctypes.c_size_t()
    native.check(lib.lsv_plan_size_group(len(ranks), indptr.ctypes.data, ranks.ctypes.data, h_in, len(hs),
                                         hs.ctypes.data, policy, ctypes.byref(pb), ctypes.byref(wb)))
    blob = np.zeros(pb.value // 4, dtype=np.int32)
    native.check(lib.lsv_plan_build_group(len(ranks), indptr.ctypes.data, ranks.ctypes.data, h_in, len(hs),
                                          hs.ctypes.data, policy, blob.ctypes.data, pb.value))
    return blob, wb.value


def test_group_plan_covers_every_projection():
    """A q/k/v group plan (Llama-3-70B-like widths: k/v narrower): every (m-tile, projection,
    chunk) is shrunk exactly once, records never exceed one N=256 MMA, rank 128 x 3 splits into
    {q,k} + {v}, and each projection has its own expand list over its own h_out tiles."""
    rng = np.random.default_rng(1)
    ranks = [8] * 20 + [16] * 10 + [64] * 5 + [128] * 5
    lens = rng.integers(9, 90, len(ranks))
    lens[2] = 3                                  # SIMT
    lens[-1] = 200                               # two m-tiles
    indptr = np.concatenate(([0], np.cumsum(lens)))
    h_outs = [4096, 1024, 1024]
    blob, ws = _plan_group(indptr, ranks, 4096, h_outs)
    h = blob[:64]
    P = int(h[33])
    assert P == 3 and list(h[37:40]) == h_outs
    d = _decode(blob)
    chunks = 4096 // 64
    seen = {}
    for rec in d["shrink"]:
        mt, p0, npj, r = int(rec[12]), int(rec[13]), int(rec[14]), int(rec[3])
        assert 1 <= npj and p0 + npj <= P and npj * r <= 256
        for pp in range(p0, p0 + npj):
            seen.setdefault((mt, pp), []).append((int(rec[4]), int(rec[5])))
    for i, mt in enumerate(d["mtiles"]):
        r = int(mt[3])
        for pp in range(P):
            parts = sorted(seen[(i, pp)])
            assert parts[0][0] == 0 and parts[-1][1] == chunks
            assert all(parts[j][1] == parts[j + 1][0] for j in range(len(parts) - 1))
        subsets = {(int(rec[13]), int(rec[14])) for rec in d["shrink"] if int(rec[12]) == i}
        assert subsets == ({(0, 2), (2, 1)} if r == 128 else {(0, 3)})
    off_recs, off_cta, grids, nitems = h[41:45], h[45:49], h[49:53], h[53:57]
    for pp in range(P):
        tw = 256 if h_outs[pp] % 256 == 0 else 128
        recs = blob[off_recs[pp]:off_recs[pp] + 8 * nitems[pp]].reshape(-1, 8)
        assert {(int(r[6]), int(r[4])) for r in recs} == {(i, j) for i in range(d["n_mtiles"]) for j in range(h_outs[pp] // tw)}
        cta = blob[off_cta[pp]:off_cta[pp] + grids[pp] + 1]
        assert cta[0] == 0 and cta[-1] == nitems[pp]
    # workspace: P v-image regions of vimg_stride bytes each
    assert int(h[34]) % 1024 == 0 and ws >= int(h[34]) * P


def test_group_plan_of_one_is_the_single_plan():
    ranks = [8, 16, 64, 128]
    indptr = [0, 40, 90, 130, 300]
    a, wa = _plan(indptr, ranks, 4096, 11008)
    b, wb = _plan_group(indptr, ranks, 4096, [11008])
    assert wa == wb and np.array_equal(a, b)


def test_group_pack_rejects_bad_member():
    lib = native.load()
    with pytest.raises(ValueError):
        native.check(lib.lsv_pack_adapter_group(None, 3, 3, 8, 4096, None, None))
    with pytest.raises(ValueError):
        native.check(lib.lsv_pack_adapter_group(None, 5, 0, 8, 4096, None, None))
    assert lib.lsv_adapter_a_group_bytes(3, 16, 4096) == 3 * 16 * 4096 * 2


@pytest.mark.parametrize("P", [1, 3])
def test_simt_tail_row_block_map(P):
    """The SIMT tier's plan tail (lsv_plan.h): items carry ntok | rank << 16; the row-block prefix
    counts each item's 16-row blocks of its group A (P * rank rows); the map gives every shrink
    block its (item, row block) in item order."""
    ranks = [8, 24, 128, 256, 40, 16]
    lens = [1, 3, 8, 2, 5, 1]
    indptr = np.concatenate(([0], np.cumsum(lens)))
    blob, _ = (_plan_group(indptr, ranks, 4096, [1024] * P, policy=native.TIER_SIMT) if P > 1
               else _plan(indptr, ranks, 4096, 1024, policy=native.TIER_SIMT))
    d = _decode(blob)
    n = d["n_simt"]
    assert n == len(ranks) and d["n_mtiles"] == 0
    items = d["simt"]
    assert [int(it[2]) & 0xFFFF for it in items] == lens
    assert [int(it[2]) >> 16 for it in items] == ranks
    pre = blob[d["off_simt"] + 4 * n:d["off_simt"] + 5 * n + 1]
    nrb = [-(-P * r // 16) for r in ranks]
    assert list(np.diff(pre)) == nrb and pre[0] == 0
    rbmap = blob[d["off_simt"] + 5 * n + 1:d["off_simt"] + 5 * n + 1 + int(pre[-1])]
    want = [i << 8 | rb for i in range(n) for rb in range(nrb[i])]
    assert list(rbmap) == want


def test_tile_aligned_plan_pieces():
    """LSV_PLAN_TILE_ALIGNED: segments are cut at the batch's 128-token tile boundaries, every piece
    is a tensor-core m-tile with a 128-row v image, and the tail [tiles + 1] indexes each tile's
    first piece."""
    lens = [5, 100, 60, 1, 90, 44]
    ranks = [8, 64, 128, 16, 24, 256]
    indptr = np.concatenate(([0], np.cumsum(lens)))
    blob, _ = _plan(indptr, ranks, 1024, 512, policy=native.TIER_AUTO | native.PLAN_TILE_ALIGNED)
    d = _decode(blob)
    assert int(blob[62]) == 1 and d["n_simt"] == 0          # PlanHeader::tile_aligned; no SIMT items
    mts = d["mtiles"]
    for seg, tb, nt, r, *_ in mts:
        assert tb // 128 == (tb + nt - 1) // 128            # never crosses a tile boundary
    covered = np.zeros(int(indptr[-1]), dtype=int)
    for seg, tb, nt, *_ in mts:
        covered[tb:tb + nt] += 1
    assert np.all(covered == 1)
    ntiles = -(-int(indptr[-1]) // 128)
    tail = blob[d["total_ints"] - ntiles - 1:d["total_ints"]]
    assert tail[0] == 0 and tail[-1] == len(mts)
    for t in range(ntiles):
        for j in range(tail[t], tail[t + 1]):
            assert int(mts[j][1]) // 128 == t
    # v images: 128 rows x kpad(rank), hi + lo
    offs = [int(m[6]) for m in mts]
    kp = [max(16, -(-int(m[3]) // 16) * 16) for m in mts]
    sizes = [(-(-128 * k * 2 // 1024) * 1024) * 2 for k in kp]
    assert offs == list(np.concatenate(([0], np.cumsum(sizes)[:-1])))
    with pytest.raises(ValueError, match="tile-aligned"):
        _plan(indptr, ranks, 1024, 512, policy=native.TIER_SIMT | native.PLAN_TILE_ALIGNED)


def _plan_group_flags(indptr, ranks, flags, h_in=4096, h_outs=(4096,)):
    lib = native.load()
    indptr = np.asarray(indptr, dtype=np.int32)
    ranks = np.asarray(ranks, dtype=np.int32)
    fl = None if flags is None else np.asarray(flags, dtype=np.int32)
    hs = np.asarray(h_outs, dtype=np.int32)
    pb, wb = ctypes.c_size_t(), ctypes.c_size_t()
    fp = None if fl is None else fl.ctypes.data
    native.check(lib.lsv_plan_size_group_ex(len(ranks), indptr.ctypes.data, ranks.ctypes.data, fp, h_in, len(hs),
                                            hs.ctypes.data, 0, ctypes.byref(pb), ctypes.byref(wb)))
    blob = np.zeros(pb.value // 4, dtype=np.int32)
    native.check(lib.lsv_plan_build_group_ex(len(ranks), indptr.ctypes.data, ranks.ctypes.data, fp, h_in, len(hs),
                                             hs.ctypes.data, 0, blob.ctypes.data, pb.value))
    return blob


def test_remote_segments_spread_and_interleave():
    """LSV_SEG_REMOTE: the same work items (coverage unchanged), remote expand items spread over the
    CTAs (no CTA carries far more than its share) and alternating with local ones in each list."""
    rng = np.random.default_rng(5)
    ranks = [8] * 44 + [16] * 22 + [32] * 14 + [64] * 11 + [128] * 9
    lens = np.bincount(rng.integers(0, 100, 4096), minlength=100)
    indptr = np.concatenate(([0], np.cumsum(lens)))
    flags = (np.arange(100) % 3 == 0).astype(np.int32)      # a third of the adapters on a peer
    d0 = _decode(_plan_group_flags(indptr, ranks, None))
    d1 = _decode(_plan_group_flags(indptr, ranks, flags))
    key = lambda d: sorted(map(tuple, d["expand"].tolist()))   # noqa: E731
    assert key(d0) == key(d1) and sorted(map(tuple, d0["shrink"].tolist())) == sorted(map(tuple, d1["shrink"].tolist()))
    off = d1["expand_cta"]
    rem_bytes = []
    for c in range(d1["expand_grid"]):
        recs = d1["expand"][off[c]:off[c + 1]]
        isrem = [bool(flags[int(r[0])]) for r in recs]
        rem_bytes.append(sum(int(r[3]) for r, f in zip(recs, isrem) if f))
        # alternation: no two remote records in a row while local ones remain later in the list
        for i in range(len(isrem) - 1):
            if isrem[i] and isrem[i + 1]:
                assert not any(not f for f in isrem[i + 1:])
    rem_bytes = np.array(rem_bytes, dtype=float)
    assert rem_bytes.max() <= 2.5 * rem_bytes.mean() + 256


def test_skip_flags_and_sm_budget():
    """LSV_SEG_SKIP segments get no work; LSV_PLAN_SMS(n) caps every grid at n CTAs."""
    ranks = [8, 64, 128, 16]
    lens = [100, 300, 50, 200]
    indptr = np.concatenate(([0], np.cumsum(lens)))
    skip = np.array([0, 2, 0, 2], dtype=np.int32)
    d = _decode(_plan_group_flags(indptr, ranks, skip))
    assert {int(m[0]) for m in d["mtiles"]} == {0, 2}
    assert {int(r[0]) for r in d["expand"]} == {0, 2}
    lib = native.load()
    blob, _ = _plan(indptr, ranks, policy=native.PLAN_SMS(20))
    d = _decode(blob)
    assert d["shrink_grid"] <= 20 and d["expand_grid"] <= 20 and d["n_mtiles"] == 1 + 3 + 1 + 2


def test_dynamic_dispatch_order_is_a_permutation_of_the_group_list():
    """PlanHeader::off_dyn (the layer kernel's dynamic expand dispatch order) lists every item of
    the group kernel's expand list (all members when num_proj > 1, else member 0's) exactly once."""
    rng = np.random.default_rng(5)
    ranks = [8] * 30 + [16] * 10 + [32] * 8 + [64] * 6 + [128] * 6
    lens = rng.integers(9, 120, len(ranks))
    indptr = np.concatenate(([0], np.cumsum(lens)))
    for h_in, h_outs in ((4096, [11008, 11008]), (4096, [4096, 1024, 1024]), (11008, [4096])):
        blob, _ = _plan_group(indptr, ranks, h_in, h_outs)
        h = blob[:64]
        P, off_dyn = int(h[33]), int(h[63])
        n = int(h[60]) if P > 1 else int(h[53])
        assert off_dyn > 0 and off_dyn + n <= int(h[21])
        order = blob[off_dyn:off_dyn + n]
        assert np.array_equal(np.sort(order), np.arange(n))
