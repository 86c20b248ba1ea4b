"""Out-of-bounds write checks (the compute-sanitizer memcheck substitute; the tool is closed on the
GPU pool).  Every output and the workspace sit inside sentinel-filled guard bands; after the delta
path runs, every guard byte must be unchanged.  Run under the production library and, by
tools/gpu_checked.sh, under liblsv_checked.so (LSV_DEVICE_CHECKS=1: kernels assert their plan
records, ring allocations and workspace offsets and trap on a violation)."""

import ctypes

import numpy as np
import pytest
import torch

from tests._cases import Case

pytestmark = pytest.mark.gpu

SENTINEL = -12345.0   # exactly representable in bf16


def _guarded(n, h, dev, pad_rows=5, pad_cols=40):
    """A [n, h] bf16 view (row stride h + pad_cols) inside a sentinel-filled buffer."""
    buf = torch.full((n + 2 * pad_rows, h + pad_cols), SENTINEL, dtype=torch.bfloat16, device=dev)
    return buf, buf[pad_rows:pad_rows + n, 8:8 + h]


def _guard_intact(buf, view):
    mask = torch.ones_like(buf, dtype=torch.bool)
    r0 = view.data_ptr() - buf.data_ptr()
    rows, cols = view.shape
    ld = buf.shape[1]
    r, c = divmod(r0 // 2, ld)
    mask[r:r + rows, c:c + cols] = False
    return bool(torch.all(buf[mask] == SENTINEL))


@pytest.mark.parametrize("tier", [0, 1, 2])
def test_apply_writes_only_its_rows_and_columns(tier):
    from paper_2511_22880_b200.lora import LoraDeltaEngine
    from paper_2511_22880_b200.slab import AdapterSlab
    case = Case(1024, 1280, [1, 3, 8, 9, 17, 127, 128, 129, 40], [8, 16, 32, 64, 128, 256, 24, 40, 136], seed=33)
    dev = torch.device("cuda:0")
    slab = AdapterSlab(case.model, AdapterSlab.capacity_for(case.model, case.ranks), dev)
    for s, r in enumerate(case.ranks):
        slab.load(slab.allocate(f"a{s}", r), 0, 0, case.a[s].to(dev), case.b[s].to(dev))
    eng = LoraDeltaEngine(slab, tier_policy=tier)
    bp = eng.prepare(case.seg)
    # workspace tail past what the plan needs: sentinel bytes that must survive
    lib = __import__("paper_2511_22880_b200.native", fromlist=["lib"]).lib()
    ph = (ctypes.c_void_p * 1)(bp.group_plans[0].plan_host.ctypes.data)
    need = lib.lsv_lora_forward_workspace(1, 1, ctypes.addressof(ph))
    ws = bp.workspace
    tail = ws[need:]
    tail.fill_(0xA5)
    n = case.seg.num_tokens
    xbuf, x = _guarded(n, 1024, dev)
    x.copy_(case.x[:n].to(dev))
    ybuf, y = _guarded(n, 1280, dev)
    y.zero_()
    eng.apply(bp, 0, 0, x, y)
    eng.apply(bp, 0, 0, x, y)
    torch.cuda.synchronize()
    assert _guard_intact(ybuf, y)
    assert _guard_intact(xbuf, x)
    assert bool(torch.all(tail == 0xA5))
    assert bool(torch.all(ws[:64 * 1024] == 0))          # barrier header back to zero at rest


def test_forward_writes_only_its_outputs():
    from paper_2511_22880_b200.lora import LoraDeltaEngine
    from paper_2511_22880_b200.segments import index_tokens
    from paper_2511_22880_b200.shapes import LLAMA2_7B, ModelShape
    from paper_2511_22880_b200.slab import AdapterSlab
    dev = torch.device("cuda:0")
    model = ModelShape("l7b-2l", 2, LLAMA2_7B.projections)
    ranks = [8, 16, 32, 64, 128, 8, 24]
    slab = AdapterSlab(model, AdapterSlab.capacity_for(model, ranks), dev)
    for i, r in enumerate(ranks):
        slab.fill_random(slab.allocate(f"a{i}", r), 77 + i)
    tok = np.random.default_rng(8).integers(0, len(ranks), 600)
    seg = index_tokens(tok, ranks)
    eng = LoraDeltaEngine(slab)
    bp = eng.prepare(seg)
    N = seg.num_tokens
    g = torch.Generator(device=dev).manual_seed(3)
    xs = [{gname: torch.randn(N, model.projections[m[0]].h_in, device=dev, generator=g).to(torch.bfloat16)
           for gname, m in model.groups()} for _ in range(2)]
    bufs, ys = [], []
    for _ in range(2):
        d = {}
        for pr in model.projections:
            b, v = _guarded(N, pr.h_out, dev, pad_cols=64)
            v.zero_()
            bufs.append((b, v))
            d[pr.name] = v
        ys.append(d)
    eng.forward(bp, xs, ys)
    eng.forward(bp, xs, ys, serial=True)
    torch.cuda.synchronize()
    assert all(_guard_intact(b, v) for b, v in bufs)
    assert bool(torch.all(bp.workspace[:64 * 1024] == 0))


def test_checked_library_when_requested():
    """tools/gpu_checked.sh sets LSV_EXPECT_CHECKED=1: the loaded library must be the checked build."""
    import os
    from paper_2511_22880_b200 import native
    info = native.lib().lsv_build_info()
    if os.environ.get("LSV_EXPECT_CHECKED") == "1":
        assert info & 1, "expected liblsv_checked.so (LSV_DEVICE_CHECKS)"
    else:
        assert info in (0, 1)
