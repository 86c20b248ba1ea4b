"""World-size-2 gloo tests of the data-parallel host logic (no GPU): every rank derives the same
LoRAServe placement and routing independently, the per-rank batches partition the routed
requests, and the bench's max-over-ranks reduction picks the slowest rank."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2511_22880_b200 import synth
        wls = synth.dp_workloads(world)
        mine = wls[rank]
        # placement fingerprint must agree across ranks
        import zlib
        fp = zlib.crc32(repr(sorted(mine.placement.per_server.items())).encode())  # process-independent
        t = torch.tensor([fp & 0x7FFFFFFF, mine.segments.num_tokens, len(mine.resident)], dtype=torch.int64)
        got = [torch.zeros_like(t) for _ in range(world)]
        dist.all_gather(got, t)
        # bench-style max-over-ranks of a per-rank time
        ms = torch.tensor([1.0 + rank], dtype=torch.float64)
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        q.put((rank, [g.tolist() for g in got], float(ms.item()), sorted(mine.resident)))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(180)
def test_dp_placement_consistent_across_ranks():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=150) for _ in range(world)]
    for p in procs:
        p.join(timeout=30)
        assert p.exitcode == 0
    res.sort()
    fps = {tuple(row[0] for row in r[1]) for r in res}
    assert len(fps) == 1 and len(set(next(iter(fps)))) == 1          # same placement everywhere
    assert all(r[2] == 2.0 for r in res)                              # max over ranks
    # every adapter is resident somewhere (coverage), ranks hold only their placed adapters
    from paper_2511_22880_b200 import synth
    wls = synth.dp_workloads(world)
    assert set(res[0][3]) | set(res[1][3]) == {a for w in wls for a in w.resident}
    assert all(w.segments.num_tokens <= 4096 for w in wls)


@pytest.mark.parametrize("world", [4, 8])
def test_dp_workloads_at_scale(world):
    """The driver's scaling run goes to 8 GPUs (gpurun reaches 4): every rank's batch is non-empty
    and within the token budget, every segment's adapter is resident on that rank, and weak
    scaling keeps tokens per GPU fixed."""
    from paper_2511_22880_b200 import shapes, synth
    for model in (shapes.LLAMA2_7B, shapes.LLAMA2_13B):
        wls = synth.dp_workloads(world, model=model)
        assert len(wls) == world
        toks = {w.segments.num_tokens for w in wls}
        assert len(toks) == 1 and 0 < toks.pop() <= 4096
        for w in wls:
            assert w.segments.num_segments > 0
            used = {w.adapter_ids[int(s)] for s in w.segments.seg_slot}
            assert used <= set(w.resident)
