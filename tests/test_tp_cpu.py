"""Tensor-parallel sharding logic on CPU (gloo, world size 2): the shards shard_adapter cuts,
combined with the same collectives the GPU path issues (all-gather of v for column-parallel
projections, all-reduce of v for row-parallel ones), reproduce the unsharded delta
x·A^T·B^T — the host half of tests/test_gpu_tp.py without a GPU."""

import os
import socket

import pytest
import torch
import torch.multiprocessing as mp

from paper_2511_22880_b200.shapes import LLAMA3_70B, ModelShape, Projection
from paper_2511_22880_b200.tp import padded_rank, shard_specs


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_padded_rank_whole_kgroups():
    for tp in (1, 2, 4, 8):
        for r in (8, 16, 24, 32, 64, 128, 256):
            rp = padded_rank(r, tp)
            assert rp >= r and rp % (8 * tp) == 0 and rp - r < 8 * tp


def test_shard_specs_llama3_70b():
    for tp in (2, 4, 8):
        specs = shard_specs(LLAMA3_70B, tp)
        for sp, pr in zip(specs, LLAMA3_70B.projections):
            assert sp.h_out * tp == pr.h_out
            assert sp.h_in * (1 if sp.column else tp) == pr.h_in
        assert [s.column for s in specs] == [p.name not in ("o_proj", "down_proj") for p in LLAMA3_70B.projections]


def test_shard_specs_reject_unsplittable():
    with pytest.raises(ValueError):
        shard_specs(ModelShape("x", 1, (Projection("q_proj", 256, 384),)), 2)


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2511_22880_b200.tp import shard_adapter
        model = ModelShape("t", 1, (Projection("q_proj", 512, 768), Projection("o_proj", 768, 512)))
        specs = shard_specs(model, world)
        out = []
        for r in (8, 24, 64):
            g = torch.Generator().manual_seed(r)
            for sp, pr in zip(specs, model.projections):
                a = torch.randn(r, pr.h_in, generator=g, dtype=torch.float64)
                b = torch.randn(pr.h_out, r, generator=g, dtype=torch.float64)
                x = torch.randn(37, pr.h_in, generator=g, dtype=torch.float64)
                a_t, b_t = shard_adapter(a, b, sp, world, rank)
                assert a_t.shape == (sp.a_rank(r, world), sp.h_in) and b_t.shape == (sp.h_out, sp.b_rank(r, world))
                if sp.column:
                    v_t = x @ a_t.T
                    parts = [torch.zeros_like(v_t) for _ in range(world)]
                    dist.all_gather(parts, v_t)
                    v = torch.cat(parts, 1)
                else:
                    v = x[:, rank * sp.h_in:(rank + 1) * sp.h_in] @ a_t.T
                    dist.all_reduce(v)
                y_t = v @ b_t.T
                ys = [torch.zeros_like(y_t) for _ in range(world)]
                dist.all_gather(ys, y_t)
                err = (torch.cat(ys, 1) - x @ a.T @ b.T).abs().max().item()
                out.append((r, sp.name, err))
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(180)
def test_tp2_shard_math_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=150) for _ in range(2)]
    for p in procs:
        p.join(timeout=30)
        assert p.exitcode == 0
    for _, rows in res:
        assert len(rows) == 6
        for r, name, err in rows:
            assert err < 1e-9, (r, name, err)


def test_balanced_shards_cover_every_row_once_and_reassemble():
    """Balanced (round-robin 8-row group) shards: every row of A on exactly one rank, no padding, and
    the kernels' column map (full column 8*(t + tp*(k//8)) + k%8 of rank t's local column k) rebuilds
    v = x·A^T exactly from the per-rank shrinks."""
    from paper_2511_22880_b200.tp import ShardSpec, balanced_rows, shard_adapter
    g = torch.Generator().manual_seed(3)
    for tp in (2, 4, 8):
        for r in (8, 16, 24, 40, 64, 128):
            rows = [balanced_rows(r, tp, t) for t in range(tp)]
            allr = sorted(int(i) for rr in rows for i in rr)
            assert allr == list(range(r))
            sp = ShardSpec("q_proj", True, 256, 128 // tp * tp // tp)
            a = torch.randn(r, 256, generator=g)
            b = torch.randn(sp.h_out * tp, r, generator=g)
            x = torch.randn(5, 256, generator=g)
            v = torch.zeros(5, r)
            for t in range(tp):
                a_t, b_t = shard_adapter(a, b, sp, tp, t, balanced=True)
                assert a_t.shape[0] == len(rows[t]) and b_t.shape[1] == r      # B keeps the true rank
                assert sp.a_rank(r, tp, t, balanced=True) == a_t.shape[0]
                v_t = x @ a_t.T
                for k in range(0, a_t.shape[0], 8):
                    col = 8 * (t + tp * (k // 8))
                    v[:, col:col + 8] = v_t[:, k:k + 8]
            assert torch.allclose(v, x @ a.T, atol=1e-5)
