"""Multi-GPU (>= 2 B200) tests: in-kernel NVLink peer loads of adapters resident in another GPU's
slab give bit-identical deltas to the all-local run (config 4's data path)."""

import numpy as np
import pytest
import torch

from tests._cases import Case

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]


def test_peer_adapter_loads_bit_identical():
    from paper_2511_22880_b200 import native
    from paper_2511_22880_b200.lora import LoraDeltaEngine
    from paper_2511_22880_b200.slab import AdapterSlab
    native.check(native.lib().lsv_enable_peer(0, 1))
    case = Case(4096, 4096, [64, 41, 200, 5, 130], [128, 8, 32, 16, 64], seed=21)
    slabs = []
    for dev in ("cuda:0", "cuda:1"):
        slab = AdapterSlab(case.model, AdapterSlab.capacity_for(case.model, case.ranks), dev)
        for s, r in enumerate(case.ranks):
            slab.load(slab.allocate(f"a{s}", r), 0, 0, case.a[s].to(dev), case.b[s].to(dev))
        slabs.append(slab)
    torch.cuda.synchronize("cuda:1")
    eng = LoraDeltaEngine(slabs[0])
    owner = np.array([1, 0, 1, 1, 0], dtype=np.int32)     # three segments read GPU 1's HBM
    bp_local = eng.prepare(case.seg)
    bp_peer = eng.prepare(case.seg, seg_owner=owner, peer_slabs={1: slabs[1]})
    x = case.x.to("cuda:0")
    y1 = torch.zeros(case.n_tok, 4096, dtype=torch.bfloat16, device="cuda:0")
    y2 = torch.zeros_like(y1)
    eng.apply(bp_local, 0, 0, x, y1)
    eng.apply(bp_peer, 0, 0, x, y2)
    torch.cuda.synchronize("cuda:0")
    assert torch.equal(y1, y2)
    assert int(bp_peer.a_ptrs[0, 0]) != int(bp_local.a_ptrs[0, 0])   # really a different address


def test_remote_prefetch_forward_bit_identical():
    """The copy-engine fetch path (RemotePrefetch + forward_prefetch: the next layer's peer-owned
    tiles staged in local HBM while the current layer computes) gives the all-local step's bits on
    a 3-layer model with every input group."""
    from paper_2511_22880_b200 import native
    from paper_2511_22880_b200.lora import LoraDeltaEngine, RemotePrefetch
    from paper_2511_22880_b200.segments import index_tokens
    from paper_2511_22880_b200.shapes import ModelShape, Projection
    from paper_2511_22880_b200.slab import AdapterSlab
    native.check(native.lib().lsv_enable_peer(0, 1))
    h, inter = 1024, 2816
    model = ModelShape("mini3", 3, (Projection("q_proj", h, h), Projection("k_proj", h, 256), Projection("v_proj", h, 256),
                                     Projection("o_proj", h, h), Projection("gate_proj", h, inter),
                                     Projection("up_proj", h, inter), Projection("down_proj", inter, h)))
    ranks = [8, 16, 128, 64, 24, 32]
    slabs = []
    for dev in ("cuda:0", "cuda:1"):
        slab = AdapterSlab(model, AdapterSlab.capacity_for(model, ranks), dev)
        for i, r in enumerate(ranks):
            slab.fill_random(slab.allocate(f"a{i}", r), 700 + i)
        slabs.append(slab)
    torch.cuda.synchronize("cuda:1")
    tok = np.concatenate([np.full(n, s) for s, n in enumerate([41, 3, 150, 64, 17, 90])])
    seg = index_tokens(tok, ranks)
    owner = np.array([1, 0, 1, 1, 0, 1], dtype=np.int32)
    eng = LoraDeltaEngine(slabs[0])
    bp_local = eng.prepare(seg)
    pf = RemotePrefetch(eng, seg, owner, {1: slabs[1]})
    bp_pf = pf.plan()
    N = seg.num_tokens
    g = torch.Generator().manual_seed(3)
    xs = [{n: torch.randn(N, model.projections[m[0]].h_in, generator=g).to(torch.bfloat16).to("cuda:0")
           for n, m in model.groups()} for _ in range(model.layers)]
    ya = [{p.name: torch.zeros(N, p.h_out, dtype=torch.bfloat16, device="cuda:0") for p in model.projections}
          for _ in range(model.layers)]
    yb = [{p.name: torch.zeros(N, p.h_out, dtype=torch.bfloat16, device="cuda:0") for p in model.projections}
          for _ in range(model.layers)]
    eng.forward(bp_local, xs, ya)
    eng.forward_prefetch(bp_pf, pf, xs, yb)
    torch.cuda.synchronize("cuda:0")
    for layer in range(model.layers):
        for p in model.projections:
            assert torch.equal(ya[layer][p.name], yb[layer][p.name]), (layer, p.name)
    assert pf.bytes_per_layer > 0


def test_migrate_from_peer_bit_identical():
    """Copy-on-first-use (the reference's commit_migration, pool.py:134-162): a peer-owned adapter
    copied into a local slot verbatim (one copy-engine transfer over NVLink) unpacks to the same
    weights and gives the oracle's delta, whatever local slot order the copies land in."""
    from paper_2511_22880_b200 import native
    from paper_2511_22880_b200.lora import LoraDeltaEngine
    from paper_2511_22880_b200.slab import AdapterSlab
    native.check(native.lib().lsv_enable_peer(0, 1))
    case = Case(4096, 4096, [64, 41, 200, 5, 130], [128, 8, 32, 16, 64], seed=23)
    peer = AdapterSlab(case.model, AdapterSlab.capacity_for(case.model, case.ranks), "cuda:1")
    for s, r in enumerate(case.ranks):
        peer.load(peer.allocate(f"a{s}", r), 0, 0, case.a[s].to("cuda:1"), case.b[s].to("cuda:1"))
    torch.cuda.synchronize("cuda:1")
    local = AdapterSlab(case.model, AdapterSlab.capacity_for(case.model, case.ranks), "cuda:0")
    # migrate in a different order than the peer's slots: offsets differ, bytes move verbatim
    for s in reversed(range(len(case.ranks))):
        local.migrate_from_peer(f"a{s}", peer)
    torch.cuda.synchronize("cuda:0")
    for s in range(len(case.ranks)):
        a0, b0 = local.read(local.by_id[f"a{s}"], 0, 0)
        assert torch.equal(a0.cpu(), case.a[s]) and torch.equal(b0.cpu(), case.b[s])
    seg = case.seg
    seg.seg_slot[:] = [local.by_id[f"a{s}"] for s in range(len(case.ranks))]
    eng = LoraDeltaEngine(local)
    y = torch.zeros(case.n_tok, 4096, dtype=torch.bfloat16, device="cuda:0")
    eng.apply(eng.prepare(seg), 0, 0, case.x.to("cuda:0"), y)
    torch.cuda.synchronize("cuda:0")
    from oracle import oracle
    err = oracle.max_rel_err(y.float().cpu().numpy()[:seg.num_tokens], case.oracle_delta()[:seg.num_tokens])
    assert err <= 1e-2


def test_split_step_matches_all_local():
    """SplitStep (peer-owned segments on a few CTAs and their own stream, local ones on the rest)
    gives the all-local deltas within the contract (k-split choices differ with the SM budget, so
    fp32 summation order may differ: not bit-identical)."""
    from oracle import oracle
    from paper_2511_22880_b200 import native
    from paper_2511_22880_b200.lora import LoraDeltaEngine, SplitStep
    from paper_2511_22880_b200.segments import index_tokens
    from paper_2511_22880_b200.shapes import LLAMA2_7B, ModelShape
    from paper_2511_22880_b200.slab import AdapterSlab
    native.check(native.lib().lsv_enable_peer(0, 1))
    model = ModelShape("l7b-2l", 2, LLAMA2_7B.projections)
    ranks = [8, 16, 32, 64, 128, 8, 16, 64]
    slabs = []
    for dev in ("cuda:0", "cuda:1"):
        slab = AdapterSlab(model, AdapterSlab.capacity_for(model, ranks), dev)
        for i, r in enumerate(ranks):
            slab.fill_random(slab.allocate(f"a{i}", r), 500 + i)
        slabs.append(slab)
    torch.cuda.synchronize("cuda:1")
    seg = index_tokens(np.random.default_rng(4).integers(0, len(ranks), 700), ranks)
    owner = (np.arange(seg.num_segments) % 2).astype(np.int32)
    N = seg.num_tokens
    g = torch.Generator(device="cuda:0").manual_seed(2)
    xs = [{gname: torch.randn(N, model.projections[m[0]].h_in, device="cuda:0", generator=g).to(torch.bfloat16)
           for gname, m in model.groups()} for _ in range(2)]
    ys_a = [{p.name: torch.zeros(N, p.h_out, dtype=torch.bfloat16, device="cuda:0") for p in model.projections}
            for _ in range(2)]
    ys_b = [{k: v.clone() for k, v in d.items()} for d in ys_a]
    eng = LoraDeltaEngine(slabs[0])
    eng.forward(eng.prepare(seg), xs, ys_a)
    sp = SplitStep(slabs[0], seg, owner, {1: slabs[1]}, remote_sms=16)
    sp.forward(xs, ys_b)
    torch.cuda.synchronize("cuda:0")
    for l in range(2):
        for k in ys_a[l]:
            a, b = ys_a[l][k].float().cpu().numpy(), ys_b[l][k].float().cpu().numpy()
            assert oracle.max_rel_err(b, a) <= 1e-2, (l, k)
            assert np.mean(a == b) > 0.97
