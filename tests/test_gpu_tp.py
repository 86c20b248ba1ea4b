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


def _worker_groups(rank, world, port, q, balanced=False):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    try:
        from oracle import oracle
        from tests._cases import bf16_bits
        from paper_2511_22880_b200.segments import index_tokens
        from paper_2511_22880_b200.shapes import ModelShape, Projection
        from paper_2511_22880_b200.tp import TPLoraDeltaEngine, TPSlab
        h, kv, inter = 1024, 256, 2816
        model = ModelShape("tp-mini", 2, (Projection("q_proj", h, h), Projection("k_proj", h, kv),
                                          Projection("v_proj", h, kv), Projection("o_proj", h, h),
                                          Projection("gate_proj", h, inter), Projection("up_proj", h, inter),
                                          Projection("down_proj", inter, h)))
        ranks = [8, 24, 128, 64, 16]
        tok = np.concatenate([np.full(n, s) for s, n in enumerate([41, 130, 17, 64, 9])])
        seg = index_tokens(tok, ranks)
        N = seg.num_tokens
        g = torch.Generator().manual_seed(17)
        full = {}
        for s_, r in enumerate(ranks):           # the same full adapters on every rank
            for l in range(model.layers):
                for p, pr in enumerate(model.projections):
                    full[(s_, l, p)] = ((torch.randn(r, pr.h_in, generator=g) / pr.h_in ** 0.5).to(torch.bfloat16),
                                        (torch.randn(pr.h_out, r, generator=g) / r ** 0.5).to(torch.bfloat16))
        slab = TPSlab(model, world, rank, ranks, dev, balanced=balanced)
        for (s_, l, p), (a, b) in full.items():
            slab.load_full(s_, l, p, a, b)
        eng = TPLoraDeltaEngine(slab)
        st = eng.prepare(seg)
        xs_full = [{n: torch.randn(N, model.projections[m[0]].h_in, generator=g).to(torch.bfloat16)
                    for n, m in model.groups()} for _ in range(model.layers)]
        xs, ys = [], []
        for l in range(model.layers):
            xd, yd = {}, {}
            for n, m in model.groups():
                sp0 = slab.specs[m[0]]
                xf = xs_full[l][n]
                xd[n] = (xf if sp0.column else xf[:, rank * sp0.h_in:(rank + 1) * sp0.h_in]).contiguous().to(dev)
                for p in m:
                    yd[model.projections[p].name] = torch.zeros(N, slab.specs[p].h_out, dtype=torch.bfloat16, device=dev)
            xs.append(xd)
            ys.append(yd)
        eng.forward(st, xs, ys)                      # fused column-group exchange (NVLink stores)
        ys2 = [{k: torch.zeros_like(v) for k, v in yd.items()} for yd in ys]
        if not balanced:
            eng.forward(st, xs, ys2, fused=False)    # every group through NCCL (equal padded shards only)
        ys3 = [{k: torch.zeros_like(v) for k, v in yd.items()} for yd in ys]
        eng.forward(st, xs, ys3, row_fused=True)     # row groups' all-reduce in the kernels too
        torch.cuda.synchronize()
        assert st.get("fused") is not None
        # column groups: the fused exchange moves the same bf16 units NCCL's all-gather moves (identical
        # bits); row groups: fp32 partials summed once vs NCCL's bf16 all-reduce (both within tolerance)
        col = {model.projections[p].name for n, m in model.groups() for p in m if slab.specs[p].column}
        same = balanced or all(torch.equal(ys[l][k], ys2[l][k]) for l in range(model.layers) for k in ys[l] if k in col)
        errs = [("fused == nccl", same)]
        for l in range(model.layers):
            for p, pr in enumerate(model.projections):
                parts = [torch.zeros_like(ys[l][pr.name]) for _ in range(world)]
                dist.all_gather(parts, ys[l][pr.name])
                if rank == 0:
                    got = torch.cat(parts, 1).float().cpu().numpy()
                    grp = [n for n, m in model.groups() if p in m][0]
                    ref = oracle.delta_c(bf16_bits(xs_full[l][grp]), seg.seg_indptr, seg.seg_rank,
                                         [bf16_bits(full[(int(sl), l, p)][0]) for sl in seg.seg_slot],
                                         [bf16_bits(full[(int(sl), l, p)][1]) for sl in seg.seg_slot], pr.h_out)
                    errs.append((l, pr.name, oracle.max_rel_err(got[:N], ref[:N])))
                parts3 = [torch.zeros_like(ys3[l][pr.name]) for _ in range(world)]
                dist.all_gather(parts3, ys3[l][pr.name])
                if rank == 0:
                    got3 = torch.cat(parts3, 1).float().cpu().numpy()
                    errs.append((l, pr.name + "/row_fused", oracle.max_rel_err(got3[:N], ref[:N])))
        if rank == 0:
            q.put(errs)
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(600)
@pytest.mark.parametrize("balanced", [False, True])
def test_tp2_forward_input_groups(balanced):
    """TP2 forward over every input group of a 2-layer mini Llama with every exchange inside the
    kernels over NVLink: fused q/k/v and gate/up shrinks store each rank-shard of v into every rank's
    full-rank image (bit-identical to the NCCL all-gather path); o/down shrinks store fp32 partial v
    into every rank's slot and the expands sum them — every projection within the bf16 tolerance of
    the unsharded oracle.  ``balanced``: round-robin 8-row-group shards (LSV_TP_ROUND_ROBIN, ranks
    with no rows of an adapter skip it via LSV_SEG_NOSHRINK) instead of ranks padded to 16."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker_groups, args=(r, 2, port, q, balanced)) for r in range(2)]
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
    assert res is not None and len(res) == 29
    assert res[0] == ("fused == nccl", True)      # the in-kernel NVLink exchange gives NCCL's bits
    for layer, name, err in res[1:]:
        assert err <= TOL, (layer, name, err)
