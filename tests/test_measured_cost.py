"""MeasuredCost: the B200-measured drop-in for the reference's prefill_time / decode_iter_time
(costmodel.py:83-123).  Same signatures and argument errors (CPU), and on the GPU: positive
timings, per-segment rank cost — a mixed-rank batch costs less than the same batch at the max rank,
which the reference's model charges (costmodel.py:104) — cached by batch signature."""

import pytest

from paper_2511_22880_b200 import costmodel


def test_measured_cost_argument_errors_match_reference():
    mc = costmodel.MeasuredCost(engine=None)
    params = costmodel.CostParams()
    with pytest.raises(ValueError):
        mc.prefill_time([], [], params)
    with pytest.raises(ValueError):
        mc.prefill_time([10, 20], [8], params)
    with pytest.raises(ValueError):
        mc.prefill_time([params.token_budget + 1], [8], params)
    with pytest.raises(ValueError):
        mc.decode_iter_time([], [], params)


@pytest.mark.gpu
def test_measured_prefill_is_rank_aware():
    import torch
    from paper_2511_22880_b200.lora import LoraDeltaEngine
    from paper_2511_22880_b200.shapes import LLAMA2_7B, ModelShape
    from paper_2511_22880_b200.slab import AdapterSlab
    model = ModelShape("l7b-4l", 4, LLAMA2_7B.projections)
    ranks = [8, 16, 32, 64, 128]
    slab = AdapterSlab(model, AdapterSlab.capacity_for(model, ranks), "cuda:0")
    for r in ranks:
        slab.fill_random(slab.allocate(f"r{r}", r), r)
    mc = costmodel.MeasuredCost(LoraDeltaEngine(slab), reps=3)
    params = costmodel.CostParams()
    lengths = [512, 512, 512, 512]
    mixed = mc.prefill_time(lengths, [8, 8, 8, 128], params)
    all_max = mc.prefill_time(lengths, [128, 128, 128, 128], params)
    all_min = mc.prefill_time(lengths, [8, 8, 8, 8], params)
    assert 0 < all_min < mixed < all_max
    # the reference's model charges the mixed batch exactly the max-rank batch (costmodel.py:104)
    assert costmodel.prefill_time(lengths, [8, 8, 8, 128], params) == costmodel.prefill_time(lengths, [128] * 4, params)
    assert mc.prefill_time(lengths, [128, 8, 8, 8], params) == mixed            # cached by signature
    dec = mc.decode_iter_time([100] * 16, [8] * 8 + [64] * 8, params)
    assert dec > 0
    torch.cuda.synchronize()
