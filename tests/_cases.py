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

    def run_gpu(self, tier_policy=0, device="cuda:0", repeat=1, v_bf16=False):
        from paper_2511_22880_b200.lora import LoraDeltaEngine
        from paper_2511_22880_b200.slab import AdapterSlab
        slab_bytes = AdapterSlab.capacity_for(self.model, self.ranks)
        slab = AdapterSlab(self.model, slab_bytes, device)
        for s, r in enumerate(self.ranks):
            slot = slab.allocate(f"a{s}", r)
            slab.load(slot, 0, 0, self.a[s].to(device), self.b[s].to(device))
        eng = LoraDeltaEngine(slab, tier_policy=tier_policy, v_bf16=v_bf16)
        bp = eng.prepare(self.seg)
        x = self.x.to(device)
        outs = []
        for _ in range(repeat):
            y = self.y0.to(device)
            eng.apply(bp, 0, 0, x, y)
            torch.cuda.synchronize(device)
            outs.append(y.cpu())
        return outs if repeat > 1 else outs[0], bp


class LayerCase:
    """One Llama-2-7B layer of config 2 (all 7 projections): the C2 batch (4096 tokens over the
    100-adapter power-law roster, synth.c2_llama2_7b), one x per input group (q/k/v share one,
    gate/up another), A/B per (adapter, projection).  Seeded on the CPU like ``Case``."""

    def __init__(self, seed=20):
        from paper_2511_22880_b200 import shapes, synth
        wl = synth.c2_llama2_7b()
        self.wl = wl
        self.model = ModelShape("llama-2-7b-1-layer", 1, shapes.LLAMA2_7B.projections)
        self.seg = wl.segments
        n = self.seg.num_tokens
        g = torch.Generator().manual_seed(seed)
        self.x = {}
        for pr in self.model.projections:
            grp = shapes.input_group(pr.name)
            if grp not in self.x:
                self.x[grp] = torch.randn(n, pr.h_in, generator=g).to(torch.bfloat16)
        self.a, self.b = {}, {}      # (slot, proj) -> bf16 tensors
        for slot in sorted(set(int(s) for s in self.seg.seg_slot)):
            r = wl.ranks[slot]
            ga = torch.Generator().manual_seed(1000 + seed * 7919 + slot)
            for p, pr in enumerate(self.model.projections):
                self.a[(slot, p)] = (torch.randn(r, pr.h_in, generator=ga) / math.sqrt(pr.h_in)).to(torch.bfloat16)
                self.b[(slot, p)] = (torch.randn(pr.h_out, r, generator=ga) / math.sqrt(r)).to(torch.bfloat16)

    def proj_inputs(self, p):
        """(x bf16, [A_s], [B_s]) of projection p in segment order."""
        from paper_2511_22880_b200.shapes import input_group
        pr = self.model.projections[p]
        slots = [int(s) for s in self.seg.seg_slot]
        return self.x[input_group(pr.name)], [self.a[(s, p)] for s in slots], [self.b[(s, p)] for s in slots]

    def oracle_delta(self, p) -> np.ndarray:
        x, a, b = self.proj_inputs(p)
        return oracle.delta_c(bf16_bits(x), self.seg.seg_indptr, self.seg.seg_rank,
                              [bf16_bits(t) for t in a], [bf16_bits(t) for t in b], self.model.projections[p].h_out)

    def run_gpu(self, tier_policy=0, device="cuda:0", v_bf16=False):
        """The product path: every projection of the layer through one LoraDeltaEngine.forward
        (fused input-group shrinks + group expands), y_in = 0.  Returns {proj name: y (CPU bf16)}."""
        from paper_2511_22880_b200.lora import LoraDeltaEngine
        from paper_2511_22880_b200.shapes import input_group
        from paper_2511_22880_b200.slab import AdapterSlab
        wl = self.wl
        slots = sorted(set(int(s) for s in self.seg.seg_slot))
        slab = AdapterSlab(self.model, AdapterSlab.capacity_for(self.model, [wl.ranks[s] for s in slots]), device)
        slot_of = {}
        for s in slots:
            slot_of[s] = slab.allocate(wl.adapter_ids[s], wl.ranks[s])
            for p in range(len(self.model.projections)):
                slab.load(slot_of[s], 0, p, self.a[(s, p)].to(device), self.b[(s, p)].to(device))
        seg = Segments(self.seg.perm, self.seg.seg_indptr, np.asarray([slot_of[int(s)] for s in self.seg.seg_slot],
                                                                      dtype=np.int32),
                       self.seg.seg_rank, self.seg.request_order)
        eng = LoraDeltaEngine(slab, tier_policy=tier_policy, v_bf16=v_bf16)
        bp = eng.prepare(seg)
        n = self.seg.num_tokens
        xs = [{g: t.to(device) for g, t in self.x.items()}]
        ys = [{pr.name: torch.zeros(n, pr.h_out, dtype=torch.bfloat16, device=device) for pr in self.model.projections}]
        eng.forward(bp, xs, ys)
        torch.cuda.synchronize(device)
        return {k: v.cpu() for k, v in ys[0].items()}, bp


# ---- fixtures of the published SGMV algorithm (tests/golden/make_sgmv_fixtures.py) --------------
# name -> Case arguments; "c2_layer" is the LayerCase.  `cols`: None = every column, else
# (first, stride): columns [0, first) plus every stride-th column after it.
FIXTURE_CASES = {
    "c1": dict(h_in=4096, h_out=4096, lengths=[64, 64, 64, 64], ranks=[8, 16, 64, 128], seed=1, cols=None),
    "ragged": dict(h_in=4096, h_out=4096, lengths=[1, 3, 8, 9, 17, 127, 128, 129, 300, 0, 5],
                   ranks=[8, 16, 32, 64, 128, 8, 16, 32, 64, 128, 24], seed=3, cols=None),
    "rank_classes": dict(h_in=4096, h_out=1024, lengths=[9, 17, 33, 64, 100, 128, 129, 20, 47, 5, 61, 90],
                         ranks=[8, 16, 24, 32, 40, 48, 56, 64, 72, 96, 112, 128], seed=8, cols=None),
    "rank_256": dict(h_in=4096, h_out=4096, lengths=[1, 2, 3, 7, 40, 130, 9, 64],
                     ranks=[256, 200, 136, 256, 256, 256, 144, 24], seed=13, cols=None),
    "token_budget_8192": dict(h_in=4096, h_out=11008, lengths=None, ranks=None, seed=40, cols=(256, 37)),
    "one_adapter_8192": dict(h_in=11008, h_out=4096, lengths=[8192], ranks=[128], seed=41, cols=None),
    "c2_layer": dict(seed=20, cols=(256, 37)),
}


def budget_case_roster():
    """test_full_token_budget_batch's batch: 8192 tokens over 60 power-law adapters."""
    rng = np.random.default_rng(40)
    ranks = [8] * 26 + [16] * 13 + [32] * 9 + [64] * 7 + [128] * 5
    lengths = np.bincount(rng.integers(0, len(ranks), 8192), minlength=len(ranks)).tolist()
    return lengths, ranks


def fixture_case(name):
    spec = dict(FIXTURE_CASES[name])
    spec.pop("cols")
    if name == "c2_layer":
        return LayerCase(**spec)
    if spec["lengths"] is None:
        spec["lengths"], spec["ranks"] = budget_case_roster()
    return Case(**spec)


def fixture_rows(seg, max_random=8, seed=0):
    """Sampled tokens of a case: the first and last token of every non-empty segment plus a few
    seeded random ones (sorted, unique)."""
    rows = set()
    for s in range(seg.num_segments):
        t0, t1 = int(seg.seg_indptr[s]), int(seg.seg_indptr[s + 1])
        if t1 > t0:
            rows.update((t0, t1 - 1))
    rng = np.random.default_rng(seed)
    n = seg.num_tokens
    rows.update(int(t) for t in rng.integers(0, n, min(max_random, n)))
    return np.asarray(sorted(rows), dtype=np.int64)


def fixture_cols(h_out, cols):
    if cols is None:
        return np.arange(h_out, dtype=np.int64)
    first, stride = cols
    return np.concatenate([np.arange(min(first, h_out)), np.arange(first, h_out, stride)]).astype(np.int64)


_FIXTURES = None
# parity margins recorded by the GPU tests (printed and saved by tests/conftest.py at session end)
MARGINS: list[dict] = []


def load_fixtures():
    global _FIXTURES
    if _FIXTURES is None:
        from pathlib import Path
        _FIXTURES = dict(np.load(Path(__file__).resolve().parent / "golden" / "sgmv_fixtures.npz"))
    return _FIXTURES


def fixture_keys(name):
    """Fixture keys of a case: [name] or [name/proj, ...] for the layer case."""
    fx = load_fixtures()
    if f"{name}/rows" in fx:
        return [name]
    return sorted({k.rsplit("/", 1)[0] for k in fx if k.startswith(name + "/") and k.count("/") == 2})


def bf16_ulp(v: np.ndarray) -> np.ndarray:
    """Spacing of bf16 numbers at |v| (2^(e-7) for |v| in [2^e, 2^(e+1))); the smallest normal's
    spacing below it."""
    a = np.maximum(np.abs(np.asarray(v, dtype=np.float64)), 2.0 ** -126)
    return 2.0 ** (np.floor(np.log2(a)) - 7)


def compare_to_fixture(y: np.ndarray, key: str) -> dict:
    """Compare a full [tokens, h_out] delta against the fixture `key`: the north-star metric
    max|y - ref| / max|ref| on the sampled entries, the worst error in bf16 ulps of the reference
    (what a bf16 output can at best reach is 0.5), and the per-token checksums."""
    fx = load_fixtures()
    rows, cols, ref, chk = fx[f"{key}/rows"], fx[f"{key}/cols"], fx[f"{key}/y"], fx[f"{key}/chk"]
    got = np.asarray(y, dtype=np.float64)[np.ix_(rows, cols)]
    ref64 = ref.astype(np.float64)
    err = oracle.max_rel_err(got, ref64)
    # ulps of the reference value, floored at the ulp of max|ref| / 256: below that an fp32
    # accumulation's absolute error (~1e-7 of the largest terms) is not measurable in bf16 ulps
    floor = float(np.max(np.abs(ref64))) / 256 if ref.size else 0.0
    ulps = float(np.max(np.abs(got - ref64) / bf16_ulp(np.maximum(np.abs(ref64), floor)))) if ref.size else 0.0
    rn = oracle.bf16_bits_to_f32(oracle.f32_to_bf16_bits(ref)).astype(np.float64)
    exact = float(np.mean(got == rn)) if ref.size else 1.0
    yd = np.asarray(y, dtype=np.float64)[: chk.shape[0]]
    w = np.cos(np.arange(yd.shape[1], dtype=np.float64))
    mine = np.stack([yd.sum(1), yd @ w], axis=1)
    scale = np.maximum(chk[:, 2:3], 1e-30)
    chk_err = float(np.max(np.abs(mine - chk[:, :2]) / scale)) if chk.size else 0.0
    return {"key": key, "max_rel_err": err, "max_ulps": ulps, "frac_rn_exact": exact, "chk_rel_err": chk_err,
            "entries": int(ref.size)}
