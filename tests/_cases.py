"""Seeded LoRA-delta cases shared by the parity tests (inputs generated on the CPU so the GPU
path and the CPU oracle see identical bf16 bits)."""

from __future__ import annotations

import math

import numpy as np
import torch

from oracle import oracle
from paper_2511_22880_b200.segments import Segments, index_requests
from paper_2511_22880_b200.shapes import ModelShape, Projection


def bf16_bits(t: torch.Tensor) -> np.ndarray:
    return t.contiguous().view(torch.int16).numpy().view(np.uint16)


class Case:
    """One projection, a batch of segments (lengths, ranks), seeded inputs."""

    def __init__(self, h_in, h_out, lengths, ranks, seed=0, y_scale=0.0, extra_tokens=0):
        self.h_in, self.h_out = h_in, h_out
        self.model = ModelShape("case", 1, (Projection("proj", h_in, h_out),))
        # one request per segment, slot = index; zero-length segments handled separately
        self.lengths = list(lengths)
        self.ranks = list(ranks)
        indptr = np.concatenate(([0], np.cumsum(self.lengths))).astype(np.int32)
        self.seg = Segments(perm=np.arange(indptr[-1], dtype=np.int32), seg_indptr=indptr,
                            seg_slot=np.arange(len(ranks), dtype=np.int32),
                            seg_rank=np.asarray(ranks, dtype=np.int32),
                            request_order=np.arange(len(ranks), dtype=np.int32))
        self.n_tok = int(indptr[-1]) + extra_tokens
        g = torch.Generator().manual_seed(seed)
        self.x = torch.randn(self.n_tok, h_in, generator=g).to(torch.bfloat16)
        self.y0 = (torch.randn(self.n_tok, h_out, generator=g) * y_scale).to(torch.bfloat16)
        self.a, self.b = [], []
        for s, r in enumerate(ranks):
            ga = torch.Generator().manual_seed(1000 + seed * 7919 + s)
            self.a.append((torch.randn(r, h_in, generator=ga) / math.sqrt(h_in)).to(torch.bfloat16))
            self.b.append((torch.randn(h_out, r, generator=ga) / math.sqrt(r)).to(torch.bfloat16))

    def oracle_delta(self) -> np.ndarray:
        return oracle.delta_c(bf16_bits(self.x), self.seg.seg_indptr, self.seg.seg_rank,
                              [bf16_bits(a) for a in self.a], [bf16_bits(b) for b in self.b], self.h_out)

    def oracle_delta_f64(self) -> np.ndarray:
        return oracle.delta_f64(bf16_bits(self.x), self.seg.seg_indptr, self.seg.seg_rank,
                                [bf16_bits(a) for a in self.a], [bf16_bits(b) for b in self.b], self.h_out)

    def run_gpu(self, tier_policy=0, device="cuda:0", repeat=1):
        from paper_2511_22880_b200.lora import LoraDeltaEngine
        from paper_2511_22880_b200.slab import AdapterSlab
        slab_bytes = AdapterSlab.capacity_for(self.model, self.ranks)
        slab = AdapterSlab(self.model, slab_bytes, device)
        for s, r in enumerate(self.ranks):
            slot = slab.allocate(f"a{s}", r)
            slab.load(slot, 0, 0, self.a[s].to(device), self.b[s].to(device))
        eng = LoraDeltaEngine(slab, tier_policy=tier_policy)
        bp = eng.prepare(self.seg)
        x = self.x.to(device)
        outs = []
        for _ in range(repeat):
            y = self.y0.to(device)
            eng.apply(bp, 0, 0, x, y)
            torch.cuda.synchronize(device)
            outs.append(y.cpu())
        return outs if repeat > 1 else outs[0], bp
