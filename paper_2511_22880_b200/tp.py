"""Tensor-parallel delta path for large models (BASELINE config 5), one process per GPU.

S-LoRA-style sharding of each layer over a TP group of size T (PAPER.md:179 — "TP shards the
adapter"; the reference models it only as the divisor in CostParams.rank_factor,
costmodel.py:69-70):

* column-parallel projections (q, k, v, gate, up; the base weight is split along h_out):
  every rank holds the full x, the rank-shard A_t = lora_A[t*rs:(t+1)*rs, :] (rs = r'/T,
  r' = r rounded up to a multiple of 8T, zero-padded, so a shard is whole 8-row k-groups) and B_t = lora_B[h_out slice, :].
  shrink -> v_t [N x rs]; **NCCL all-gather of the v images** over NVLink; liblsv assembles the
  full-rank images (lsv_vimg_assemble); expand writes this rank's h_out slice of y.
* row-parallel projections (o, down; split along h_in): rank t holds x[:, h_in slice],
  A_t = lora_A[:, h_in slice], B_t = lora_B[h_out slice, :].  shrink -> partial v [N x r];
  **NCCL all-reduce (sum) of the v images**; expand writes this rank's h_out slice of y.

Every collective is one NCCL call on the compute stream (torch.distributed, backend "nccl").
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

from . import native
from .lora import build_shape_plan, input_group
from .segments import Segments
from .shapes import ModelShape, Projection, kpad

COLUMN_PARALLEL = {"q_proj", "k_proj", "v_proj", "gate_proj", "up_proj"}


def padded_rank(rank: int, tp: int) -> int:
    """Column-parallel rank rounded up to a multiple of 8*tp so each shard is whole 8-row k-groups."""
    q = 8 * tp
    return max(q, (rank + q - 1) // q * q)


@dataclass(frozen=True)
class ShardSpec:
    name: str
    column: bool
    h_in: int        # this rank's input width
    h_out: int       # this rank's output width

    def a_rank(self, rank: int, tp: int) -> int:
        return padded_rank(rank, tp) // tp if self.column else rank

    def b_rank(self, rank: int, tp: int) -> int:
        return padded_rank(rank, tp) if self.column else rank


def shard_specs(model: ModelShape, tp: int) -> list[ShardSpec]:
    out = []
    for p in model.projections:
        col = p.name in COLUMN_PARALLEL
        if p.h_out % (128 * tp) or (not col and p.h_in % (128 * tp)):
            raise ValueError(f"{p.name} {p.h_in}->{p.h_out} does not split into {tp} shards of 128")
        out.append(ShardSpec(p.name, col, p.h_in if col else p.h_in // tp, p.h_out // tp))
    return out


def shard_adapter(lora_a: torch.Tensor, lora_b: torch.Tensor, sp: ShardSpec, tp: int, t: int):
    """Rank t's (A_t, B_t) of a full PEFT-layout adapter (lora_A [r, h_in], lora_B [h_out, r]).

    Column-parallel: the rank is zero-padded to padded_rank(r, tp); A_t is rank rows
    [t*rs, (t+1)*rs) of the padded A, B_t the h_out slice of the padded B (all rp columns, since
    the all-gathered v is full rank).  Row-parallel: A_t is the h_in column slice, B_t the h_out
    row slice, both at the full rank (v is a partial sum, all-reduced)."""
    r = lora_a.shape[0]
    if sp.column:
        rp = padded_rank(r, tp)
        a_pad = lora_a.new_zeros((rp, lora_a.shape[1]))
        a_pad[:r] = lora_a
        b_pad = lora_b.new_zeros((lora_b.shape[0], rp))
        b_pad[:, :r] = lora_b
        rs = rp // tp
        return (a_pad[t * rs:(t + 1) * rs].contiguous(),
                b_pad[t * sp.h_out:(t + 1) * sp.h_out].contiguous())
    return (lora_a[:, t * sp.h_in:(t + 1) * sp.h_in].contiguous(),
            lora_b[t * sp.h_out:(t + 1) * sp.h_out].contiguous())


class TPSlab:
    """One rank's shard of every adapter: A and B tiles at their own (shard) ranks."""

    ALIGN = 1024

    def __init__(self, model: ModelShape, tp: int, rank: int, ranks: list[int], device):
        self.model, self.tp, self.rank = model, tp, rank
        self.specs = shard_specs(model, tp)
        self.device = torch.device(device)
        self.ranks = list(ranks)
        L, P = model.layers, len(self.specs)
        self.a_off = np.zeros((len(ranks), L, P), dtype=np.int64)
        self.b_off = np.zeros((len(ranks), L, P), dtype=np.int64)
        cur = 0
        for s, r in enumerate(ranks):
            cur = (cur + self.ALIGN - 1) // self.ALIGN * self.ALIGN
            for l in range(L):
                for p, sp in enumerate(self.specs):
                    ra, rb = sp.a_rank(r, tp), sp.b_rank(r, tp)
                    self.a_off[s, l, p] = cur
                    cur += 2 * ra * sp.h_in
                    self.b_off[s, l, p] = cur
                    cur += 2 * kpad(rb) * sp.h_out
        self.capacity = cur + self.ALIGN
        ptr = ctypes.c_void_p()
        native.check(native.lib().lsv_slab_alloc(self.capacity, self.device.index or 0, ctypes.byref(ptr)))
        self.base = int(ptr.value)

    def __del__(self):
        try:
            native.lib().lsv_slab_free(self.base)
        except Exception:
            pass

    def load_full(self, slot: int, layer: int, proj: int, lora_a: torch.Tensor, lora_b: torch.Tensor,
                  stream=None) -> None:
        """Pack this rank's shard of a full PEFT-layout adapter (lora_A [r, h_in], lora_B [h_out, r])."""
        sp, tp, t = self.specs[proj], self.tp, self.rank
        r = self.ranks[slot]
        st = (stream or torch.cuda.current_stream(self.device)).cuda_stream
        a_sh, b_sh = shard_adapter(lora_a.to(self.device), lora_b.to(self.device), sp, tp, t)
        ra, rb = sp.a_rank(r, tp), sp.b_rank(r, tp)
        lib = native.lib()
        native.check(lib.lsv_pack_adapter(a_sh.data_ptr(), None, ra, sp.h_in, sp.h_out,
                                          self.base + int(self.a_off[slot, layer, proj]), None, st))
        native.check(lib.lsv_pack_adapter(None, b_sh.data_ptr(), rb, sp.h_in, sp.h_out, None,
                                          self.base + int(self.b_off[slot, layer, proj]), st))

    def fill_random_full(self, slot: int, seed: int, full: ModelShape) -> None:
        """Seeded full adapter (same on every rank), this rank's shard packed."""
        r = self.ranks[slot]
        g = torch.Generator(device=self.device)
        g.manual_seed(seed)
        for l in range(self.model.layers):
            for p, pr in enumerate(full.projections):
                a = (torch.randn((r, pr.h_in), generator=g, device=self.device) / math.sqrt(pr.h_in)).to(torch.bfloat16)
                b = (torch.randn((pr.h_out, r), generator=g, device=self.device) / math.sqrt(r)).to(torch.bfloat16)
                self.load_full(slot, l, p, a, b)

    def fill_random_shards(self, slot: int, seed: int) -> None:
        """Benchmark fill: random shard tensors generated directly at shard shape (no full adapter)."""
        r = self.ranks[slot]
        g = torch.Generator(device=self.device)
        g.manual_seed(seed)
        lib = native.lib()
        st = torch.cuda.current_stream(self.device).cuda_stream
        for l in range(self.model.layers):
            for p, sp in enumerate(self.specs):
                ra, rb = sp.a_rank(r, self.tp), sp.b_rank(r, self.tp)
                a = (torch.randn((ra, sp.h_in), generator=g, device=self.device) * 0.02).to(torch.bfloat16)
                b = (torch.randn((sp.h_out, rb), generator=g, device=self.device) * 0.1).to(torch.bfloat16)
                native.check(lib.lsv_pack_adapter(a.data_ptr(), None, ra, sp.h_in, sp.h_out,
                                                  self.base + int(self.a_off[slot, l, p]), None, st))
                native.check(lib.lsv_pack_adapter(None, b.data_ptr(), rb, sp.h_in, sp.h_out, None,
                                                  self.base + int(self.b_off[slot, l, p]), st))

    def pointer_tables(self, seg_slots) -> tuple[torch.Tensor, torch.Tensor]:
        L, P = self.model.layers, len(self.specs)
        slots = np.asarray(seg_slots, dtype=np.int64)
        a = (self.base + self.a_off[slots]).reshape(len(slots), L * P).T.copy()
        b = (self.base + self.b_off[slots]).reshape(len(slots), L * P).T.copy()
        return torch.from_numpy(a).to(self.device), torch.from_numpy(b).to(self.device)


class TPLoraDeltaEngine:
    """Delta path of one TP rank: shrink -> NCCL exchange of v -> (assemble) -> expand."""

    def __init__(self, slab: TPSlab, group=None):
        native.load()
        self.slab, self.group = slab, group
        self.tp, self.rank, self.device = slab.tp, slab.rank, slab.device
        self.specs = slab.specs

    def prepare(self, seg: Segments) -> dict:
        """Per projection: shrink plan (A ranks) and expand plan (B ranks); all tensor-core tier so
        every rank's plans tile the batch identically."""
        tp = self.tp
        plans = {}
        ws_need = 0
        for p, sp in enumerate(self.specs):
            ra = np.array([sp.a_rank(int(r), tp) for r in seg.seg_rank], dtype=np.int32)
            rb = np.array([sp.b_rank(int(r), tp) for r in seg.seg_rank], dtype=np.int32)
            key_a = (sp.h_in, sp.h_out, tuple(ra))
            key_b = (sp.h_in, sp.h_out, tuple(rb))
            for key, rr in ((key_a, ra), (key_b, rb)):
                if key not in plans:
                    s2 = Segments(seg.perm, seg.seg_indptr, seg.seg_slot, rr, seg.request_order)
                    plans[key] = build_shape_plan(s2, sp.h_in, sp.h_out, native.TIER_TC, self.device)
                    ws_need = max(ws_need, plans[key].workspace_bytes)
            plans[p] = (plans[key_a], plans[key_b])
        ws = [torch.zeros(max(ws_need, 256), dtype=torch.uint8, device=self.device) for _ in range(2)]
        a_ptrs, b_ptrs = self.slab.pointer_tables(seg.seg_slot)
        region = max(self._region(plans[p][0])[1] for p in range(len(self.specs)))
        gathered = torch.empty(self.tp * max(region, 16), dtype=torch.uint8, device=self.device)
        return {"seg": seg, "plans": plans, "ws": ws, "a_ptrs": a_ptrs, "b_ptrs": b_ptrs, "gathered": gathered}

    @staticmethod
    def _region(sp) -> tuple[int, int]:
        off, nb = ctypes.c_size_t(), ctypes.c_size_t()
        native.check(native.lib().lsv_plan_vimg_region(sp.plan_host.ctypes.data, ctypes.byref(off), ctypes.byref(nb)))
        return off.value, nb.value

    def apply(self, st: dict, layer: int, proj: int, x: torch.Tensor, y: torch.Tensor, stream=None) -> None:
        """x: this rank's input (full h_in for column-parallel, its h_in slice for row-parallel);
        y: this rank's h_out slice."""
        lib = native.lib()
        sp = self.specs[proj]
        plan_a, plan_b = st["plans"][proj]
        seg = st["seg"]
        S = seg.num_segments
        row = layer * len(self.specs) + proj
        strm = stream or torch.cuda.current_stream(self.device)
        ws_a, ws_b = st["ws"]
        native.check(lib.lsv_lora_shrink(x.data_ptr(), x.stride(0), x.shape[0], sp.h_in,
                                         st["a_ptrs"].data_ptr() + row * S * 8, plan_a.plan_dev.data_ptr(),
                                         plan_a.plan_host.ctypes.data, ws_a.data_ptr(), ws_a.numel(), strm.cuda_stream))
        off, nb = self._region(plan_a)
        with torch.cuda.stream(strm):
            if sp.column:
                src = ws_a[off:off + nb]
                dst = st["gathered"][:self.tp * nb]
                dist.all_gather_into_tensor(dst, src, group=self.group)
                native.check(lib.lsv_vimg_assemble(dst.data_ptr(), nb, self.tp, plan_a.plan_dev.data_ptr(),
                                                   plan_a.plan_host.ctypes.data, plan_b.plan_dev.data_ptr(),
                                                   plan_b.plan_host.ctypes.data, ws_b.data_ptr(), strm.cuda_stream))
                ws_e = ws_b
            else:
                v = ws_a[off:off + nb].view(torch.bfloat16)
                dist.all_reduce(v, group=self.group)     # sum of the per-rank partial v images
                ws_e = ws_a
        native.check(lib.lsv_lora_expand(y.data_ptr(), y.stride(0), y.shape[0], sp.h_out,
                                         st["b_ptrs"].data_ptr() + row * S * 8, plan_b.plan_dev.data_ptr(),
                                         plan_b.plan_host.ctypes.data, ws_e.data_ptr(), ws_e.numel(), strm.cuda_stream))

    def forward(self, st: dict, xs, ys, stream=None) -> None:
        for layer in range(self.slab.model.layers):
            for p, sp in enumerate(self.specs):
                self.apply(st, layer, p, xs[layer][input_group(sp.name)], ys[layer][sp.name], stream)
