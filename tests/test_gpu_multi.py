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
