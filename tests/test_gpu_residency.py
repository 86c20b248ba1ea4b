"""Adapter residency on the GPU (pool.py:88-132 data path): host -> HBM slab loading through pinned
memory, eviction to a per-rank free list and slot reuse, all bit-exact through pack/unpack."""

import pytest
import torch

pytestmark = pytest.mark.gpu


def test_load_from_host_evict_and_reuse():
    from paper_2511_22880_b200.shapes import LLAMA2_7B, ModelShape
    from paper_2511_22880_b200.slab import AdapterSlab
    model = ModelShape("l7b-2l", 2, LLAMA2_7B.projections)
    slab = AdapterSlab(model, AdapterSlab.capacity_for(model, [16, 64, 16]), "cuda:0")
    s0 = slab.allocate("a", 16)
    s1 = slab.allocate("b", 64)
    g = torch.Generator().manual_seed(4)
    weights = {}
    for l in range(model.layers):
        for p, pr in enumerate(model.projections):
            weights[(l, p)] = (torch.randn(64, pr.h_in, generator=g).to(torch.bfloat16).pin_memory(),
                               torch.randn(pr.h_out, 64, generator=g).to(torch.bfloat16).pin_memory())
    slab.load_from_host(s1, weights)
    torch.cuda.synchronize()
    for (l, p), (a, b) in weights.items():
        ra, rb = slab.read(s1, l, p)
        assert torch.equal(ra.cpu(), a) and torch.equal(rb.cpu(), b)
    # evict "a", a new rank-16 adapter takes its slot (same offsets); other ranks get new space
    off = slab.a_group_offset(s0, 1, 4)
    assert slab.free("a") == s0
    assert "a" not in slab.by_id
    s2 = slab.allocate("c", 16)
    assert s2 == s0 and slab.a_group_offset(s2, 1, 4) == off
    s3 = slab.allocate("d", 16)
    assert s3 not in (s0, s1)
    with pytest.raises(KeyError):
        slab.free("a")
