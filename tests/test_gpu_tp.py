"""Tensor-parallel delta path on 2 B200s (config 5's data path): column-parallel (rank-sharded A,
NCCL all-gather of v, assembled full-rank images) and row-parallel (h_in-sharded A, NCCL
all-reduce of v) shards reproduce the CPU oracle's unsharded delta within the bf16 tolerance."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]

TOL = 1e-2


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    try:
        from tests._cases import Case
        from paper_2511_22880_b200.shapes import ModelShape, Projection
        from paper_2511_22880_b200.tp import TPLoraDeltaEngine, TPSlab
        lengths = [64, 41, 130, 17, 9]
        ranks = [8, 16, 128, 64, 24]
        cq = Case(4096, 4096, lengths, ranks, seed=31)   # q_proj (column-parallel)
        co = Case(4096, 4096, lengths, ranks, seed=32)   # o_proj (row-parallel)
        model = ModelShape("tp-test", 1, (Projection("q_proj", 4096, 4096), Projection("o_proj", 4096, 4096)))
        slab = TPSlab(model, world, rank, ranks, dev)
        for s in range(len(ranks)):
            slab.load_full(s, 0, 0, cq.a[s].to(dev), cq.b[s].to(dev))
            slab.load_full(s, 0, 1, co.a[s].to(dev), co.b[s].to(dev))
        eng = TPLoraDeltaEngine(slab)
        st = eng.prepare(cq.seg)
        n = cq.seg.num_tokens
        sl = slice(rank * 2048, (rank + 1) * 2048)
        yq = torch.zeros(n, 2048, dtype=torch.bfloat16, device=dev)
        yo = torch.zeros(n, 2048, dtype=torch.bfloat16, device=dev)
        eng.apply(st, 0, 0, cq.x[:n].to(dev), yq)
        eng.apply(st, 0, 1, co.x[:n, sl].contiguous().to(dev), yo)
        torch.cuda.synchronize()
        gq = [torch.zeros_like(yq) for _ in range(world)]
        go = [torch.zeros_like(yo) for _ in range(world)]
        dist.all_gather(gq, yq)
        dist.all_gather(go, yo)
        if rank == 0:
            q.put((torch.cat(gq, 1).float().cpu().numpy(), torch.cat(go, 1).float().cpu().numpy(),
                   cq.oracle_delta()[:n], co.oracle_delta()[:n]))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(600)
def test_tp2_column_and_row_parallel():
    from oracle import oracle
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    import queue as _queue
    res = None
    for _ in range(600):
        try:
            res = q.get(timeout=1)
            break
        except _queue.Empty:
            if any(p.exitcode not in (None, 0) for p in procs):
                break
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res is not None
    yq, yo, refq, refo = res
    assert oracle.max_rel_err(yq, refq) <= TOL
    assert oracle.max_rel_err(yo, refo) <= TOL
