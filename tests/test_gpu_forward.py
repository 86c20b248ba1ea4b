"""Whole-step path (lsv_lora_forward: every layer's input groups, fused shrinks + one-launch group
expands, per-(layer, group) workspace slices, shrinks overlapping the previous expand's tail)
against the CPU oracle, on a 2-layer Llama-shaped model with all four input groups, and
bit-identical to issuing the same work group by group."""

import numpy as np
import pytest
import torch

from oracle import oracle
from tests._cases import bf16_bits

pytestmark = pytest.mark.gpu
TOL = 1e-2


def _setup(dev, tier=0):
    from paper_2511_22880_b200.lora import LoraDeltaEngine
    from paper_2511_22880_b200.segments import index_tokens
    from paper_2511_22880_b200.shapes import ModelShape, Projection
    from paper_2511_22880_b200.slab import AdapterSlab
    h, inter, kv = 1024, 2816, 256
    model = ModelShape("mini", 2, (Projection("q_proj", h, h), Projection("k_proj", h, kv), Projection("v_proj", h, kv),
                                    Projection("o_proj", h, h), Projection("gate_proj", h, inter),
                                    Projection("up_proj", h, inter), Projection("down_proj", inter, h)))
    ranks = [8, 16, 128, 64, 24, 32, 8, 128]
    slab = AdapterSlab(model, AdapterSlab.capacity_for(model, ranks), dev)
    for i, r in enumerate(ranks):
        slab.fill_random(slab.allocate(f"a{i}", r), 500 + i)
    rng = np.random.default_rng(5)
    tok = np.concatenate([np.full(n, s) for s, n in enumerate([41, 3, 150, 64, 17, 0, 90, 33])])
    rng.shuffle(tok)
    seg = index_tokens(tok, ranks)
    eng = LoraDeltaEngine(slab, tier_policy=tier)
    bp = eng.prepare(seg)
    N = seg.num_tokens
    g = torch.Generator().manual_seed(9)
    xs = [{name: torch.randn(N, model.projections[m[0]].h_in, generator=g).to(torch.bfloat16).to(dev)
           for name, m in model.groups()} for _ in range(model.layers)]
    return model, slab, seg, eng, bp, xs


@pytest.mark.parametrize("tier", [0, 2])
def test_forward_matches_oracle_and_per_group_calls(tier):
    dev = torch.device("cuda:0")
    model, slab, seg, eng, bp, xs = _setup(dev, tier)
    N = seg.num_tokens
    ys = [{p.name: torch.zeros(N, p.h_out, dtype=torch.bfloat16, device=dev) for p in model.projections}
          for _ in range(model.layers)]
    eng.forward(bp, xs, ys)
    torch.cuda.synchronize()
    # the same work issued group by group (shrink + expand_group per group)
    ys2 = [{p.name: torch.zeros(N, p.h_out, dtype=torch.bfloat16, device=dev) for p in model.projections}
           for _ in range(model.layers)]
    for layer in range(model.layers):
        for gi, (name, members) in enumerate(model.groups()):
            eng.shrink(bp, layer, members[0], xs[layer][name])
            eng.expand_group(bp, layer, gi, [ys2[layer][model.projections[p].name] for p in members])
    torch.cuda.synchronize()
    for layer in range(model.layers):
        for p, pr in enumerate(model.projections):
            got = ys[layer][pr.name]
            assert torch.equal(got, ys2[layer][pr.name]), (layer, pr.name)
            a_list, b_list = [], []
            for slot in seg.seg_slot:
                a, b = slab.read(int(slot), layer, p)
                a_list.append(bf16_bits(a.cpu()))
                b_list.append(bf16_bits(b.cpu()))
            x = xs[layer][[n for n, m in model.groups() if p in m][0]]
            ref = oracle.delta_c(bf16_bits(x.cpu()), seg.seg_indptr, seg.seg_rank, a_list, b_list, pr.h_out)
            err = oracle.max_rel_err(got.float().cpu().numpy()[:N], ref[:N])
            assert err <= TOL, (layer, pr.name, err)


def test_forward_repeats_bit_identical():
    """Two back-to-back steps on the same inputs (the second reuses the workspace slices, whose
    split counters the kernels re-arm) give bit-identical outputs."""
    dev = torch.device("cuda:0")
    model, slab, seg, eng, bp, xs = _setup(dev)
    N = seg.num_tokens
    outs = []
    for _ in range(2):
        ys = [{p.name: torch.zeros(N, p.h_out, dtype=torch.bfloat16, device=dev) for p in model.projections}
              for _ in range(model.layers)]
        eng.forward(bp, xs, ys)
        torch.cuda.synchronize()
        outs.append(ys)
    for layer in range(model.layers):
        for pr in model.projections:
            assert torch.equal(outs[0][layer][pr.name], outs[1][layer][pr.name])


def test_stream_prepared_plans_ring_and_staleness():
    """prepare(stream=...) uploads through the engine's reused pinned+device arenas: results are
    bit-identical to a synchronously uploaded plan, and a plan whose arena slot a later prepare
    reused fails loudly instead of reading another batch's plan."""
    dev = torch.device("cuda:0")
    model, slab, seg, eng, bp, xs = _setup(dev)
    N = seg.num_tokens
    st = torch.cuda.Stream(dev)

    def run(plan, stream=None):
        ys = [{p.name: torch.zeros(N, p.h_out, dtype=torch.bfloat16, device=dev) for p in model.projections}
              for _ in range(model.layers)]
        eng.forward(plan, xs, ys, stream)
        torch.cuda.synchronize()
        return ys

    ref = run(bp)
    plans = []
    for _ in range(6):     # more than the ring depth; each plan consumed on its stream right away
        plans.append(eng.prepare(seg, stream=st))
        with torch.cuda.stream(st):
            got = run(plans[-1], st)
        for layer in range(model.layers):
            for p in model.projections:
                assert torch.equal(got[layer][p.name], ref[layer][p.name])
    with pytest.raises(RuntimeError, match="stale"):
        run(plans[0])
    run(plans[-1])   # the newest one is still live


def test_decode_groups_simt_ksplit_against_oracle():
    """Decode-shaped batch (1-5 tokens per adapter) through lsv_lora_forward on a full-width
    layer (h = 4096, inter = 11008): the SIMT tier's group shrinks (q/k/v: N = 3r rows in 16-row
    blocks that straddle members) with k-splits (48-chunk ranges: 1 for h_in 4096, 3 for 11008),
    the one-launch multi-member expands, and the four groups on concurrent streams (an overlap-free
    forward without layer kernels), against the oracle for every projection."""
    from paper_2511_22880_b200.lora import LoraDeltaEngine
    from paper_2511_22880_b200.segments import index_tokens
    from paper_2511_22880_b200.shapes import LLAMA2_7B, ModelShape
    from paper_2511_22880_b200.slab import AdapterSlab
    dev = torch.device("cuda:0")
    model = ModelShape("l7b-1l", 1, LLAMA2_7B.projections)
    ranks = [8, 24, 128, 64, 16, 40, 256, 8]
    slab = AdapterSlab(model, AdapterSlab.capacity_for(model, ranks), dev)
    for i, r in enumerate(ranks):
        slab.fill_random(slab.allocate(f"d{i}", r), 900 + i)
    tok = np.concatenate([np.full(n, s) for s, n in enumerate([1, 2, 5, 1, 3, 1, 2, 4])])
    np.random.default_rng(3).shuffle(tok)
    seg = index_tokens(tok, ranks)
    eng = LoraDeltaEngine(slab, tier_policy=1)       # forced SIMT (AUTO sends rank >= 128 / n > 4 to tcgen05)
    bp = eng.prepare(seg)
    assert all(gp.summary[5] == 0 for gp in bp.group_plans)   # every segment on the SIMT tier
    N = seg.num_tokens
    g = torch.Generator().manual_seed(31)
    xs = [{name: torch.randn(N, model.projections[m[0]].h_in, generator=g).to(torch.bfloat16).to(dev)
           for name, m in model.groups()}]
    ys = [{p.name: torch.zeros(N, p.h_out, dtype=torch.bfloat16, device=dev) for p in model.projections}]
    eng.forward(bp, xs, ys)
    torch.cuda.synchronize()
    for p, pr in enumerate(model.projections):
        a_list, b_list = [], []
        for slot in seg.seg_slot:
            a, b = slab.read(int(slot), 0, p)
            a_list.append(bf16_bits(a.cpu()))
            b_list.append(bf16_bits(b.cpu()))
        x = xs[0][[n for n, m in model.groups() if p in m][0]]
        ref = oracle.delta_c(bf16_bits(x.cpu()), seg.seg_indptr, seg.seg_rank, a_list, b_list, pr.h_out)
        err = oracle.max_rel_err(ys[0][pr.name].float().cpu().numpy()[:N], ref[:N])
        assert err <= TOL, (pr.name, err)


def test_group_kernel_full_layer_bit_identical_to_split_launches():
    """One full Llama-2-7B layer at C2 scale (100 adapters, 4096 tokens, every group kernel path:
    split tiles, member subsets of rank 128, down_proj's long split-K) through lsv_lora_forward
    (one group kernel per input group) and through the separate shrink / expand launches: the
    outputs are bit-identical (same split-K summation order, same v images)."""
    from paper_2511_22880_b200.lora import LoraDeltaEngine
    from paper_2511_22880_b200.segments import index_tokens
    from paper_2511_22880_b200.shapes import LLAMA2_7B, ModelShape
    from paper_2511_22880_b200.slab import AdapterSlab
    dev = torch.device("cuda:0")
    model = ModelShape("l7b-1l", 1, LLAMA2_7B.projections)
    ranks = [8] * 44 + [16] * 22 + [32] * 14 + [64] * 11 + [128] * 9
    slab = AdapterSlab(model, AdapterSlab.capacity_for(model, ranks), dev)
    for i, r in enumerate(ranks):
        slab.fill_random(slab.allocate(f"a{i}", r), 700 + i)
    seg = index_tokens(np.random.default_rng(3).integers(0, 100, 4096), ranks)
    eng = LoraDeltaEngine(slab)
    bp = eng.prepare(seg)
    g = torch.Generator().manual_seed(4)
    xs = [{name: (torch.randn(4096, model.projections[m[0]].h_in, generator=g) * 2).to(torch.bfloat16).to(dev)
           for name, m in model.groups()}]
    ys = [{p.name: torch.randn(4096, p.h_out, generator=g).to(torch.bfloat16).to(dev) for p in model.projections}]
    ys2 = [{k: v.clone() for k, v in ys[0].items()}]
    eng.forward(bp, xs, ys)
    for gi, (name, members) in enumerate(model.groups()):
        eng.shrink(bp, 0, members[0], xs[0][name])
        eng.expand_group(bp, 0, gi, [ys2[0][model.projections[p].name] for p in members])
    torch.cuda.synchronize()
    for pr in model.projections:
        assert torch.equal(ys[0][pr.name], ys2[0][pr.name]), pr.name


def test_layer_kernel_dynamic_dispatch_c2_three_layers_bit_identical():
    """Three Llama-2-7B layers of the C2 batch through lsv_lora_forward — one layer kernel per
    layer: all four input groups' shrink stages and expand items through one shared-memory byte
    ring, every shrink before any expand, expand items taken from per-(layer, group) global cursors
    (dynamic dispatch, multi-layer calls) — against the separate shrink / expand launches of the
    same work: bit-identical (which CTA computes an item does not change its bits)."""
    from paper_2511_22880_b200.lora import LoraDeltaEngine
    from paper_2511_22880_b200.segments import index_tokens
    from paper_2511_22880_b200.shapes import LLAMA2_7B, ModelShape
    from paper_2511_22880_b200.slab import AdapterSlab
    dev = torch.device("cuda:0")
    model = ModelShape("l7b-3l", 3, LLAMA2_7B.projections)
    ranks = [8] * 44 + [16] * 22 + [32] * 14 + [64] * 11 + [128] * 9
    slab = AdapterSlab(model, AdapterSlab.capacity_for(model, ranks), dev)
    for i, r in enumerate(ranks):
        slab.fill_random(slab.allocate(f"a{i}", r), 900 + i)
    seg = index_tokens(np.random.default_rng(11).integers(0, 100, 4096), ranks)
    eng = LoraDeltaEngine(slab)
    bp = eng.prepare(seg)
    assert eng.launches_per_step(bp) == model.layers     # one layer kernel per layer
    g = torch.Generator().manual_seed(12)
    xs = [{name: torch.randn(4096, model.projections[m[0]].h_in, generator=g).to(torch.bfloat16).to(dev)
           for name, m in model.groups()} for _ in range(model.layers)]
    ys = [{p.name: torch.randn(4096, p.h_out, generator=g).to(torch.bfloat16).to(dev) for p in model.projections}
          for _ in range(model.layers)]
    ys2 = [{k: v.clone() for k, v in d.items()} for d in ys]
    eng.forward(bp, xs, ys)
    eng.forward(bp, xs, ys)                                  # twice: the cursors are re-armed per call
    for _ in range(2):
        for layer in range(model.layers):
            for gi, (name, members) in enumerate(model.groups()):
                eng.shrink(bp, layer, members[0], xs[layer][name])
                eng.expand_group(bp, layer, gi, [ys2[layer][model.projections[p].name] for p in members])
    torch.cuda.synchronize()
    for layer in range(model.layers):
        for pr in model.projections:
            assert torch.equal(ys[layer][pr.name], ys2[layer][pr.name]), (layer, pr.name)


@pytest.mark.parametrize("names", [("q_proj", "k_proj", "v_proj", "o_proj"),            # 2 groups: layer kernel
                                   ("q_proj", "o_proj", "gate_proj", "up_proj", "down_proj", "k_proj")])   # 5 groups
def test_forward_group_counts_bit_identical(names):
    """lsv_lora_forward with 2 input groups (one layer kernel per layer, two groups back to back) and
    with 5 groups (more than a layer kernel holds: one group kernel per group), 3 layers, against
    the same work issued group by group."""
    from paper_2511_22880_b200.lora import LoraDeltaEngine
    from paper_2511_22880_b200.segments import index_tokens
    from paper_2511_22880_b200.shapes import ModelShape, Projection
    from paper_2511_22880_b200.slab import AdapterSlab
    dev = torch.device("cuda:0")
    h, inter, kv = 1024, 2816, 256
    shapes = {"q_proj": (h, h), "k_proj": (h, kv), "v_proj": (h, kv), "o_proj": (h, h), "gate_proj": (h, inter),
              "up_proj": (h, inter), "down_proj": (inter, h)}
    model = ModelShape("mini", 3, tuple(Projection(n, *shapes[n]) for n in names))
    ranks = [8, 16, 128, 64, 24, 32]
    slab = AdapterSlab(model, AdapterSlab.capacity_for(model, ranks), dev)
    for i, r in enumerate(ranks):
        slab.fill_random(slab.allocate(f"a{i}", r), 300 + i)
    tok = np.concatenate([np.full(n, s) for s, n in enumerate([70, 33, 150, 64, 17, 90])])
    np.random.default_rng(2).shuffle(tok)
    seg = index_tokens(tok, ranks)
    eng = LoraDeltaEngine(slab, tier_policy=2)
    bp = eng.prepare(seg)
    N = seg.num_tokens
    g = torch.Generator().manual_seed(6)
    xs = [{name: torch.randn(N, model.projections[m[0]].h_in, generator=g).to(torch.bfloat16).to(dev)
           for name, m in model.groups()} for _ in range(model.layers)]
    ys = [{p.name: torch.randn(N, p.h_out, generator=g).to(torch.bfloat16).to(dev) for p in model.projections}
          for _ in range(model.layers)]
    ys2 = [{k: v.clone() for k, v in d.items()} for d in ys]
    eng.forward(bp, xs, ys)
    for layer in range(model.layers):
        for gi, (name, members) in enumerate(model.groups()):
            eng.shrink(bp, layer, members[0], xs[layer][name])
            eng.expand_group(bp, layer, gi, [ys2[layer][model.projections[p].name] for p in members])
    torch.cuda.synchronize()
    assert len(model.groups()) == (2 if len(names) == 4 else 5)
    for layer in range(model.layers):
        for pr in model.projections:
            assert torch.equal(ys[layer][pr.name], ys2[layer][pr.name]), (layer, pr.name)
