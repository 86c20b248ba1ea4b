"""Input-group shrink through the C ABI: the A matrices of three projections that share x (q/k/v,
Llama-3-70B-like output widths 4096/1024/1024) packed into one group tile
(lsv_pack_adapter_group), one fused shrink (lsv_plan_build_group + lsv_lora_shrink) and one
expand per member (lsv_lora_expand_proj) reproduce the CPU oracle for every member within the
bf16 tolerance — across both tiers, split-K m-tiles and rank 128 (whose 3x128-row group is
shrunk as {q,k} + {v} record subsets)."""

import ctypes

import numpy as np
import pytest
import torch

from oracle import oracle
from tests._cases import Case

pytestmark = pytest.mark.gpu
TOL = 1e-2


def _run_group(cases, tier, dev="cuda:0", one_launch=False):
    from paper_2511_22880_b200 import native
    lib = native.load()
    P = len(cases)
    c0 = cases[0]
    ranks = c0.ranks
    S = len(ranks)
    h_in = c0.h_in
    h_outs = np.array([c.h_out for c in cases], dtype=np.int32)
    st = torch.cuda.current_stream().cuda_stream
    # group A tiles per segment, B tiles per (segment, projection)
    a_bufs, b_bufs = [], []
    for s, r in enumerate(ranks):
        ag = torch.zeros(lib.lsv_adapter_a_group_bytes(P, r, h_in), dtype=torch.uint8, device=dev)
        for p, c in enumerate(cases):
            a = c.a[s].to(dev)
            native.check(lib.lsv_pack_adapter_group(a.data_ptr(), P, p, r, h_in, ag.data_ptr(), st))
            # the group tile round-trips member by member
            back = torch.empty_like(a)
            native.check(lib.lsv_unpack_adapter_group(ag.data_ptr(), P, p, r, h_in, back.data_ptr(), st))
            assert torch.equal(back, a)
        a_bufs.append(ag)
        row = []
        for c in cases:
            bt = torch.zeros(lib.lsv_adapter_b_bytes(r, c.h_out), dtype=torch.uint8, device=dev)
            native.check(lib.lsv_pack_adapter(None, c.b[s].to(dev).data_ptr(), r, h_in, c.h_out, None,
                                              bt.data_ptr(), st))
            row.append(bt)
        b_bufs.append(row)
    indptr = np.ascontiguousarray(c0.seg.seg_indptr, dtype=np.int32)
    rk = np.ascontiguousarray(ranks, dtype=np.int32)
    pb, wb = ctypes.c_size_t(), ctypes.c_size_t()
    native.check(lib.lsv_plan_size_group(S, indptr.ctypes.data, rk.ctypes.data, h_in, P, h_outs.ctypes.data, tier,
                                         ctypes.byref(pb), ctypes.byref(wb)))
    plan = np.zeros(pb.value // 4, dtype=np.int32)
    native.check(lib.lsv_plan_build_group(S, indptr.ctypes.data, rk.ctypes.data, h_in, P, h_outs.ctypes.data, tier,
                                          plan.ctypes.data, pb.value))
    plan_dev = torch.from_numpy(plan).to(dev)
    ws = torch.zeros(max(wb.value, 256), dtype=torch.uint8, device=dev)
    a_ptrs = torch.tensor([t.data_ptr() for t in a_bufs], dtype=torch.int64, device=dev)
    x = c0.x.to(dev)
    native.check(lib.lsv_lora_shrink(x.data_ptr(), x.stride(0), x.shape[0], h_in, a_ptrs.data_ptr(),
                                     plan_dev.data_ptr(), plan.ctypes.data, ws.data_ptr(), ws.numel(), st))
    outs, tables = [], []
    for p, c in enumerate(cases):
        b_ptrs = torch.tensor([b_bufs[s][p].data_ptr() for s in range(S)], dtype=torch.int64, device=dev)
        tables.append(b_ptrs)
        y = torch.zeros(c.n_tok, c.h_out, dtype=torch.bfloat16, device=dev)
        if not one_launch:
            native.check(lib.lsv_lora_expand_proj(y.data_ptr(), y.stride(0), y.shape[0], c.h_out, p,
                                                  b_ptrs.data_ptr(), plan_dev.data_ptr(), plan.ctypes.data,
                                                  ws.data_ptr(), ws.numel(), st))
        outs.append(y)
    if one_launch:   # lsv_lora_expand_group: every member in one launch
        ya = (ctypes.c_void_p * P)(*[y.data_ptr() for y in outs])
        la = (ctypes.c_int64 * P)(*[y.stride(0) for y in outs])
        ba = (ctypes.c_void_p * P)(*[t.data_ptr() for t in tables])
        native.check(lib.lsv_lora_expand_group(ctypes.addressof(ya), ctypes.addressof(la), outs[0].shape[0],
                                               ctypes.addressof(ba), plan_dev.data_ptr(), plan.ctypes.data,
                                               ws.data_ptr(), ws.numel(), st))
    torch.cuda.synchronize()
    return [o.float().cpu().numpy() for o in outs], plan


def _cases(lengths, ranks, seed, h_outs=(4096, 1024, 1024), h_in=4096):
    # same x (seed) for every member, different adapters per member
    cases = [Case(h_in, h_out, lengths, ranks, seed=seed) for h_out in h_outs]
    for p, c in enumerate(cases[1:], 1):
        g = torch.Generator().manual_seed(seed * 131 + p)
        c.a = [(torch.randn(r, h_in, generator=g) / h_in ** 0.5).to(torch.bfloat16) for r in ranks]
        c.b = [(torch.randn(c.h_out, r, generator=g) / r ** 0.5).to(torch.bfloat16) for r in ranks]
        c.x = cases[0].x
    return cases


@pytest.mark.parametrize("tier,one_launch", [(0, False), (1, False), (2, False), (0, True), (2, True)])
def test_qkv_group_matches_oracle(tier, one_launch):
    lengths = [41, 3, 130, 64, 17, 9, 200, 0, 45]
    ranks = [8, 16, 128, 64, 24, 32, 128, 8, 40]
    cases = _cases(lengths, ranks, seed=11)
    outs, plan = _run_group(cases, tier, one_launch=one_launch)
    n = cases[0].seg.num_tokens
    for p, c in enumerate(cases):
        err = oracle.max_rel_err(outs[p][:n], c.oracle_delta()[:n])
        assert err <= TOL, f"member {p}: max rel err {err:.3e}"


def test_gate_up_group_split_k():
    """Two 11008-wide members (gate/up) on few long segments: every m-tile is k-split, so the
    grid-wide reduction writes both members' v images."""
    lengths = [128, 128, 96, 64]
    ranks = [128, 64, 16, 8]
    cases = _cases(lengths, ranks, seed=12, h_outs=(11008, 11008))
    outs, plan = _run_group(cases, 0, one_launch=True)
    n = cases[0].seg.num_tokens
    assert int(plan[30]) > 0   # n_red: split tiles present
    for p, c in enumerate(cases):
        err = oracle.max_rel_err(outs[p][:n], c.oracle_delta()[:n])
        assert err <= TOL, f"member {p}: max rel err {err:.3e}"
