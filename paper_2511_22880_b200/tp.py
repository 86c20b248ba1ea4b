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
from .lora import build_group_plan, input_group  # noqa: F401
from .segments import Segments
from .shapes import ModelShape, Projection, kpad

COLUMN_PARALLEL = {"q_proj", "k_proj", "v_proj", "gate_proj", "up_proj"}


def padded_rank(rank: int, tp: int) -> int:
    """Column-parallel rank rounded up to a multiple of 8*tp so each shard is whole 8-row k-groups."""
    q = 8 * tp
    return max(q, (rank + q - 1) // q * q)


def balanced_rows(rank: int, tp: int, t: int) -> np.ndarray:
    """Balanced shard (LSV_TP_ROUND_ROBIN): rank t's rows of a column-parallel adapter, the 8-row
    groups g with g % tp == t, in order.  Rank 8 at TP4 puts its one group on rank 0 and none on
    the others, instead of padding every adapter to 8*tp rows (+47% of the column groups' adapter
    bytes at TP4 for the 500-adapter roster)."""
    groups = np.arange(t, rank // 8, tp)
    return (groups[:, None] * 8 + np.arange(8)[None, :]).reshape(-1)


@dataclass(frozen=True)
class ShardSpec:
    name: str
    column: bool
    h_in: int        # this rank's input width
    h_out: int       # this rank's output width

    def a_rank(self, rank: int, tp: int, t: int = 0, balanced: bool = False) -> int:
        if not self.column:
            return rank
        return len(balanced_rows(rank, tp, t)) if balanced else padded_rank(rank, tp) // tp

    def b_rank(self, rank: int, tp: int, balanced: bool = False) -> int:
        return (rank if balanced else padded_rank(rank, tp)) if self.column else rank


def shard_specs(model: ModelShape, tp: int) -> list[ShardSpec]:
    out = []
    for p in model.projections:
        col = p.name in COLUMN_PARALLEL
        if p.h_out % (128 * tp) or (not col and p.h_in % (128 * tp)):
            raise ValueError(f"{p.name} {p.h_in}->{p.h_out} does not split into {tp} shards of 128")
        out.append(ShardSpec(p.name, col, p.h_in if col else p.h_in // tp, p.h_out // tp))
    return out


def shard_adapter(lora_a: torch.Tensor, lora_b: torch.Tensor, sp: ShardSpec, tp: int, t: int,
                  balanced: bool = False):
    """Rank t's (A_t, B_t) of a full PEFT-layout adapter (lora_A [r, h_in], lora_B [h_out, r]).

    Column-parallel: the rank is zero-padded to padded_rank(r, tp); A_t is rank rows
    [t*rs, (t+1)*rs) of the padded A, B_t the h_out slice of the padded B (all rp columns, since
    the all-gathered v is full rank).  Row-parallel: A_t is the h_in column slice, B_t the h_out
    row slice, both at the full rank (v is a partial sum, all-reduced)."""
    r = lora_a.shape[0]
    if sp.column and balanced:   # rank t's 8-row groups of A; B at the true rank
        rows = torch.as_tensor(balanced_rows(r, tp, t), dtype=torch.long, device=lora_a.device)
        return (lora_a.index_select(0, rows).contiguous(),
                lora_b[t * sp.h_out:(t + 1) * sp.h_out].contiguous())
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
    """One rank's shard of every adapter.  Per layer and input group (model.groups(): column groups
    q/k/v and gate/up, row groups o and down) one group A tile of the members' A shards at their
    shard rank (lsv_pack_adapter_group), and per projection its B shard at the B rank."""

    ALIGN = 1024

    def __init__(self, model: ModelShape, tp: int, rank: int, ranks: list[int], device, balanced: bool = False):
        """``balanced``: column-parallel A shards are round-robin 8-row groups (no padding; only the
        in-kernel NVLink exchange path consumes them, tp.TPLoraDeltaEngine.forward(fused=True))."""
        self.model, self.tp, self.rank = model, tp, rank
        self.balanced = balanced
        self.specs = shard_specs(model, tp)
        self.groups = model.groups()
        self._member = {p: (gi, i, len(m)) for gi, (_, m) in enumerate(self.groups) for i, p in enumerate(m)}
        self.device = torch.device(device)
        self.ranks = list(ranks)
        big = sorted({int(r) for r in ranks if (int(r) if balanced else padded_rank(int(r), tp)) > 128})
        if big:
            # rank > 128 runs on 64-token tensor-core tiles (lsv_common.cuh mtile_rows), which a
            # rank shard of at most 128 does not get: the shard and full-rank plans would tile the
            # batch differently.  The paper's rosters stop at 128 (traces.py:23).
            raise ValueError(f"tensor parallelism supports padded ranks up to 128, got {big}")
        L, P, G = model.layers, len(self.specs), len(self.groups)
        self.g_off = np.zeros((len(ranks), L, G), dtype=np.int64)
        self.b_off = np.zeros((len(ranks), L, P), dtype=np.int64)
        cur = 0
        for s, r in enumerate(ranks):
            cur = (cur + self.ALIGN - 1) // self.ALIGN * self.ALIGN
            for l in range(L):
                for gi, (_, members) in enumerate(self.groups):
                    sp0 = self.specs[members[0]]
                    self.g_off[s, l, gi] = cur
                    cur += 2 * len(members) * sp0.a_rank(r, tp, rank, balanced) * sp0.h_in
                    for p in members:
                        sp = self.specs[p]
                        self.b_off[s, l, p] = cur
                        cur += 2 * kpad(sp.b_rank(r, tp, balanced)) * sp.h_out
        self.capacity = cur + self.ALIGN
        ptr = ctypes.c_void_p()
        native.check(native.lib().lsv_slab_alloc(self.capacity, self.device.index or 0, ctypes.byref(ptr)))
        self.base = int(ptr.value)

    def __del__(self):
        try:
            native.lib().lsv_slab_free(self.base)
        except Exception:
            pass

    def _pack(self, slot: int, layer: int, proj: int, a_sh: torch.Tensor, b_sh: torch.Tensor, st) -> None:
        sp = self.specs[proj]
        r = self.ranks[slot]
        gi, idx, nproj = self._member[proj]
        ra, rb = sp.a_rank(r, self.tp, self.rank, self.balanced), sp.b_rank(r, self.tp, self.balanced)
        lib = native.lib()
        if ra > 0:   # a balanced shard may hold no rows of this adapter
            native.check(lib.lsv_pack_adapter_group(a_sh.data_ptr(), nproj, idx, ra, sp.h_in,
                                                    self.base + int(self.g_off[slot, layer, gi]), st))
        native.check(lib.lsv_pack_adapter(None, b_sh.data_ptr(), rb, sp.h_in, sp.h_out, None,
                                          self.base + int(self.b_off[slot, layer, proj]), st))

    def load_full(self, slot: int, layer: int, proj: int, lora_a: torch.Tensor, lora_b: torch.Tensor,
                  stream=None) -> None:
        """Pack this rank's shard of a full PEFT-layout adapter (lora_A [r, h_in], lora_B [h_out, r])."""
        sp = self.specs[proj]
        st = (stream or torch.cuda.current_stream(self.device)).cuda_stream
        a_sh, b_sh = shard_adapter(lora_a.to(self.device), lora_b.to(self.device), sp, self.tp, self.rank,
                                   self.balanced)
        self._pack(slot, layer, proj, a_sh.contiguous(), b_sh.contiguous(), st)

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
        st = torch.cuda.current_stream(self.device).cuda_stream
        for l in range(self.model.layers):
            for p, sp in enumerate(self.specs):
                ra, rb = sp.a_rank(r, self.tp, self.rank, self.balanced), sp.b_rank(r, self.tp, self.balanced)
                a = (torch.randn((max(ra, 8), sp.h_in), generator=g, device=self.device) * 0.02).to(torch.bfloat16)
                b = (torch.randn((sp.h_out, rb), generator=g, device=self.device) * 0.1).to(torch.bfloat16)
                self._pack(slot, l, p, a, b, st)

    def pointer_tables(self, seg_slots) -> tuple[torch.Tensor, torch.Tensor]:
        """Device tables: group A tiles [layers*groups, S], B tiles [layers*projections, S]."""
        L, P, G = self.model.layers, len(self.specs), len(self.groups)
        slots = np.asarray(seg_slots, dtype=np.int64)
        a = (self.base + self.g_off[slots]).reshape(len(slots), L * G).T.copy()
        b = (self.base + self.b_off[slots]).reshape(len(slots), L * P).T.copy()
        return torch.from_numpy(a).to(self.device), torch.from_numpy(b).to(self.device)


class TPLoraDeltaEngine:
    """Delta path of one TP rank, per layer and input group: fused shrink of the group's A shards
    -> one NCCL exchange of every member's v images (all-gather for a column group, all-reduce for
    a row group) -> (column: lsv_vimg_assemble to full rank) -> one-launch group expand."""

    def __init__(self, slab: TPSlab, group=None):
        native.load()
        self.slab, self.group = slab, group
        self.tp, self.rank, self.device = slab.tp, slab.rank, slab.device
        self.specs = slab.specs
        self.groups = slab.groups
        self._member = {p: (gi, i) for gi, (_, m) in enumerate(self.groups) for i, p in enumerate(m)}

    def prepare(self, seg: Segments) -> dict:
        """Per input group: shrink plan (A shard ranks) and expand plan (B ranks; the same plan for
        a row group); all tensor-core tier so every rank's plans tile the batch identically."""
        tp = self.tp
        plans = {}
        ws_a_need = ws_b_need = 0
        bal = self.slab.balanced
        for gi, (_, members) in enumerate(self.groups):
            sp0 = self.specs[members[0]]
            ra = np.array([sp0.a_rank(int(r), tp, self.rank, bal) for r in seg.seg_rank], dtype=np.int32)
            rb = np.array([sp0.b_rank(int(r), tp, bal) for r in seg.seg_rank], dtype=np.int32)
            # a balanced shard with no rows of an adapter: keep its m-tiles (same tiles as the full-rank
            # plan), no shrink work (LSV_SEG_NOSHRINK; the rank passed is a placeholder)
            flags = np.where(ra == 0, native.SEG_NOSHRINK, 0).astype(np.int32) if (ra == 0).any() else None
            ra = np.maximum(ra, 8)
            h_outs = [self.specs[p].h_out for p in members]
            mk = lambda rr, fl=None: build_group_plan(  # noqa: E731
                Segments(seg.perm, seg.seg_indptr, seg.seg_slot, rr, seg.request_order),
                sp0.h_in, h_outs, native.TIER_TC, self.device, members, seg_flags=fl)
            plan_a = mk(ra, flags)
            plan_b = mk(rb) if sp0.column else plan_a
            plans[gi] = (plan_a, plan_b)
            ws_a_need = max(ws_a_need, plan_a.workspace_bytes)
            ws_b_need = max(ws_b_need, plan_b.workspace_bytes)
        ws = [torch.zeros(max(ws_a_need, 256), dtype=torch.uint8, device=self.device),
              torch.zeros(max(ws_b_need, 256), dtype=torch.uint8, device=self.device)]
        a_ptrs, b_ptrs = self.slab.pointer_tables(seg.seg_slot)
        region = max(self._region(plans[gi][0])[1] for gi in range(len(self.groups)))
        gathered = torch.empty(self.tp * max(region, 16), dtype=torch.uint8, device=self.device)
        # pipelined forward: every group has its own shrink/exchange/expand buffers, so group g's
        # collective runs on the side stream while group g-1's assembly and expand compute
        per_group = []
        for gi in range(len(self.groups)):
            pa, pb = plans[gi]
            per_group.append({
                "ws_a": torch.zeros(max(pa.workspace_bytes, 256), dtype=torch.uint8, device=self.device),
                "ws_b": (torch.zeros(max(pb.workspace_bytes, 256), dtype=torch.uint8, device=self.device)
                         if pb is not pa else None),
                "gathered": torch.empty(self.tp * max(self._region(pa)[1], 16), dtype=torch.uint8, device=self.device),
            })
        st = {"seg": seg, "plans": plans, "ws": ws, "a_ptrs": a_ptrs, "b_ptrs": b_ptrs, "gathered": gathered,
              "per_group": per_group, "comm": torch.cuda.Stream(self.device)}
        self._prepare_fused(st)
        # the workspaces' zero fills (their split counters and grid barriers start at zero) ran on
        # the current stream; forward may run on any stream, so they must be complete first
        torch.cuda.current_stream(self.device).synchronize()
        return st

    def _prepare_fused(self, st: dict) -> None:
        """Fused column-group exchange: one CUDA-IPC-exportable buffer per rank holding the full-rank v
        images of every (layer, column group) and a flag pair per (layer, group); every rank maps
        every other rank's buffer, so a shrink can store its shard straight into all of them."""
        if self.tp > 8 or not dist.is_available() or not dist.is_initialized():
            st["fused"] = None
            return
        L, G = self.slab.model.layers, len(self.groups)
        col_off, per_layer = {}, 0
        for gi, (_, members) in enumerate(self.groups):
            _, nb = self._region(st["plans"][gi][1])
            col_off[gi] = per_layer
            if self.specs[members[0]].column:     # full-rank bf16 v images
                per_layer += (nb + 1023) // 1024 * 1024
            else:                                 # tp slots of fp32 partial v (2x the bf16 images)
                per_layer += self.tp * 2 * ((nb + 1023) // 1024 * 1024)
        flags_off = per_layer * L
        nbytes = flags_off + L * G * 8 + 1024
        lib = native.lib()
        ptr = ctypes.c_void_p()
        native.check(lib.lsv_slab_alloc(nbytes, self.device.index or 0, ctypes.byref(ptr)))
        base = int(ptr.value)
        torch.cuda.synchronize(self.device)
        flags = torch.zeros(L * G * 2, dtype=torch.int32, device=self.device)    # zero the flag area
        native.check(lib.lsv_copy_blocks(1, (ctypes.c_void_p * 1)(flags.data_ptr()),
                                         (ctypes.c_void_p * 1)(base + flags_off),
                                         (ctypes.c_size_t * 1)(flags.numel() * 4),
                                         torch.cuda.current_stream(self.device).cuda_stream))
        torch.cuda.synchronize(self.device)
        handle = (ctypes.c_char * 64)()
        native.check(lib.lsv_ipc_get_handle(base, ctypes.addressof(handle)))
        handles = [None] * self.tp
        dist.all_gather_object(handles, bytes(handle), group=self.group)
        bases = []
        for d, h in enumerate(handles):
            if d == self.rank:
                bases.append(base)
                continue
            hb = (ctypes.c_char * 64).from_buffer_copy(h)
            peer = ctypes.c_void_p()
            native.check(lib.lsv_ipc_open_handle(ctypes.addressof(hb), self.device.index or 0, ctypes.byref(peer)))
            bases.append(int(peer.value))
        st["fused"] = {"base": base, "bases": bases, "col_off": col_off, "per_layer": per_layer,
                       "flags_off": flags_off, "G": G}

    def _fused_addrs(self, st: dict, layer: int, gi: int):
        f = st["fused"]
        off = layer * f["per_layer"] + f["col_off"][gi]
        foff = f["flags_off"] + (layer * f["G"] + gi) * 8
        vdst = (ctypes.c_void_p * self.tp)(*[b + off for b in f["bases"]])
        flags = (ctypes.c_void_p * self.tp)(*[b + foff for b in f["bases"]])
        return vdst, flags, f["base"] + off, f["base"] + foff

    @staticmethod
    def _region(sp) -> tuple[int, int]:
        off, nb = ctypes.c_size_t(), ctypes.c_size_t()
        native.check(native.lib().lsv_plan_vimg_region(sp.plan_host.ctypes.data, ctypes.byref(off), ctypes.byref(nb)))
        return off.value, nb.value

    def _shrink_exchange(self, st: dict, layer: int, gi: int, x: torch.Tensor, strm) -> torch.Tensor:
        """Fused shrink of group gi + its NCCL exchange; returns the workspace the expand reads."""
        lib = native.lib()
        members = self.groups[gi][1]
        sp0 = self.specs[members[0]]
        if sp0.column and self.slab.balanced:
            raise ValueError("the NCCL all-gather path needs equal (padded) shards: TPSlab(balanced=False)")
        plan_a, plan_b = st["plans"][gi]
        S = st["seg"].num_segments
        row = layer * len(self.groups) + gi
        ws_a, ws_b = st["ws"]
        native.check(lib.lsv_lora_shrink(x.data_ptr(), x.stride(0), x.shape[0], sp0.h_in,
                                         st["a_ptrs"].data_ptr() + row * S * 8, plan_a.plan_dev.data_ptr(),
                                         plan_a.plan_host.ctypes.data, ws_a.data_ptr(), ws_a.numel(), strm.cuda_stream))
        off, nb = self._region(plan_a)
        with torch.cuda.stream(strm):
            if sp0.column:
                dst = st["gathered"][:self.tp * nb]
                dist.all_gather_into_tensor(dst, ws_a[off:off + nb], group=self.group)
                native.check(lib.lsv_vimg_assemble(dst.data_ptr(), nb, self.tp, plan_a.plan_dev.data_ptr(),
                                                   plan_a.plan_host.ctypes.data, plan_b.plan_dev.data_ptr(),
                                                   plan_b.plan_host.ctypes.data, ws_b.data_ptr(), strm.cuda_stream))
                return ws_b
            dist.all_reduce(ws_a[off:off + nb].view(torch.bfloat16), group=self.group)   # partial v sums
            return ws_a

    def apply_group(self, st: dict, layer: int, gi: int, x: torch.Tensor, ys: list[torch.Tensor], stream=None) -> None:
        """Every member of input group gi: x is this rank's input (full h_in for a column group, its
        h_in slice for a row group); ys[i] member i's h_out slice."""
        strm = stream or torch.cuda.current_stream(self.device)
        ws_e = self._shrink_exchange(st, layer, gi, x, strm)
        members = self.groups[gi][1]
        plan_b = st["plans"][gi][1]
        S = st["seg"].num_segments
        P = len(self.specs)
        n = len(members)
        y_arr = (ctypes.c_void_p * n)(*[y.data_ptr() for y in ys])
        ld_arr = (ctypes.c_int64 * n)(*[y.stride(0) for y in ys])
        b_arr = (ctypes.c_void_p * n)(*[st["b_ptrs"].data_ptr() + (layer * P + p) * S * 8 for p in members])
        native.check(native.lib().lsv_lora_expand_group(
            ctypes.addressof(y_arr), ctypes.addressof(ld_arr), ys[0].shape[0], ctypes.addressof(b_arr),
            plan_b.plan_dev.data_ptr(), plan_b.plan_host.ctypes.data, ws_e.data_ptr(), ws_e.numel(), strm.cuda_stream))

    def apply(self, st: dict, layer: int, proj: int, x: torch.Tensor, y: torch.Tensor, stream=None) -> None:
        """One projection (its group's shrink and exchange, then its own expand)."""
        strm = stream or torch.cuda.current_stream(self.device)
        gi, idx = self._member[proj]
        ws_e = self._shrink_exchange(st, layer, gi, x, strm)
        plan_b = st["plans"][gi][1]
        S = st["seg"].num_segments
        row = layer * len(self.specs) + proj
        sp = self.specs[proj]
        native.check(native.lib().lsv_lora_expand_proj(
            y.data_ptr(), y.stride(0), y.shape[0], sp.h_out, idx, st["b_ptrs"].data_ptr() + row * S * 8,
            plan_b.plan_dev.data_ptr(), plan_b.plan_host.ctypes.data, ws_e.data_ptr(), ws_e.numel(), strm.cuda_stream))

    def forward(self, st: dict, xs, ys, stream=None, fused: bool = True, row_fused: bool = False) -> None:
        """Every layer and group.  fused (default when prepared with peers mapped): every exchange
        happens inside the kernels over NVLink, no NCCL — a column group's shrink stores its shard
        of v into every rank's full-rank image, a row group's shrink stores its fp32 partial v into
        its slot on every rank and the expand sums the slots (rank order: identical bits on every
        rank); each expand waits for every rank's signal.  Row groups take the in-kernel path only
        with row_fused=True (measured slower at TP2: the expand's sum phase and grid barrier delay its
        pipeline more than the NCCL all-reduce costs); by default they all-reduce with NCCL.
        fused=False: every group through NCCL, software-pipelined (group g's collective on a side
        stream under group g-1's expand)."""
        if fused and st.get("fused"):
            return self._forward_fused(st, xs, ys, stream, row_fused)
        return self._forward_nccl(st, xs, ys, stream)

    def _forward_fused(self, st: dict, xs, ys, stream=None, row_fused: bool = False) -> None:
        lib = native.lib()
        strm = stream or torch.cuda.current_stream(self.device)
        S = st["seg"].num_segments
        P, G = len(self.specs), len(self.groups)
        for layer in range(self.slab.model.layers):
            for gi, (gname, members) in enumerate(self.groups):
                sp0 = self.specs[members[0]]
                ys_m = [ys[layer][self.specs[p].name] for p in members]
                plan_a, plan_b = st["plans"][gi]
                ws_a = st["per_group"][gi]["ws_a"]
                x = xs[layer][gname]
                vdst, flags, vimg, flag = self._fused_addrs(st, layer, gi)
                n = len(members)
                y_arr = (ctypes.c_void_p * n)(*[y.data_ptr() for y in ys_m])
                ld_arr = (ctypes.c_int64 * n)(*[y.stride(0) for y in ys_m])
                b_arr = (ctypes.c_void_p * n)(*[st["b_ptrs"].data_ptr() + (layer * P + p) * S * 8 for p in members])
                if not sp0.column and not row_fused:
                    self.apply_group(st, layer, gi, x, ys_m, strm)
                    continue
                if not sp0.column:   # row group: fp32 partials to every rank's slot, summed in the expand
                    native.check(lib.lsv_lora_shrink_tp_partials(
                        x.data_ptr(), x.stride(0), x.shape[0], sp0.h_in,
                        st["a_ptrs"].data_ptr() + (layer * G + gi) * S * 8, plan_a.plan_dev.data_ptr(),
                        plan_a.plan_host.ctypes.data, ws_a.data_ptr(), ws_a.numel(), self.tp, self.rank,
                        ctypes.addressof(vdst), ctypes.addressof(flags), strm.cuda_stream))
                    native.check(lib.lsv_lora_expand_group_tp_sum(
                        ctypes.addressof(y_arr), ctypes.addressof(ld_arr), ys_m[0].shape[0], ctypes.addressof(b_arr),
                        plan_a.plan_dev.data_ptr(), plan_a.plan_host.ctypes.data, ws_a.data_ptr(), ws_a.numel(),
                        vimg, self.tp, flag, strm.cuda_stream))
                    continue
                native.check(lib.lsv_lora_shrink_tp_scatter(
                    x.data_ptr(), x.stride(0), x.shape[0], sp0.h_in,
                    st["a_ptrs"].data_ptr() + (layer * G + gi) * S * 8, plan_a.plan_dev.data_ptr(),
                    plan_a.plan_host.ctypes.data, ws_a.data_ptr(), ws_a.numel(),
                    self.tp | (native.TP_ROUND_ROBIN if self.slab.balanced else 0), self.rank,
                    ctypes.addressof(vdst), plan_b.plan_dev.data_ptr(), plan_b.plan_host.ctypes.data,
                    ctypes.addressof(flags), strm.cuda_stream))
                native.check(lib.lsv_lora_expand_group_tp(
                    ctypes.addressof(y_arr), ctypes.addressof(ld_arr), ys_m[0].shape[0], ctypes.addressof(b_arr),
                    plan_b.plan_dev.data_ptr(), plan_b.plan_host.ctypes.data, vimg, flag, self.tp, strm.cuda_stream))

    def _forward_nccl(self, st: dict, xs, ys, stream=None) -> None:
        """Every layer and group, software-pipelined: the shrink of group g and its NCCL collective
        (side stream) overlap the assembly + expand of group g-1 on the compute stream."""
        if self.slab.balanced:
            raise ValueError("the NCCL all-gather path needs equal (padded) shards: TPSlab(balanced=False)")
        lib = native.lib()
        comp = stream or torch.cuda.current_stream(self.device)
        comm = st["comm"]
        S = st["seg"].num_segments
        P, G = len(self.specs), len(self.groups)
        pending = None

        def finish(item):
            layer, gi, ev = item
            members = self.groups[gi][1]
            sp0 = self.specs[members[0]]
            plan_a, plan_b = st["plans"][gi]
            buf = st["per_group"][gi]
            comp.wait_event(ev)
            if sp0.column:
                off, nb = self._region(plan_a)
                native.check(lib.lsv_vimg_assemble(buf["gathered"].data_ptr(), nb, self.tp, plan_a.plan_dev.data_ptr(),
                                                   plan_a.plan_host.ctypes.data, plan_b.plan_dev.data_ptr(),
                                                   plan_b.plan_host.ctypes.data, buf["ws_b"].data_ptr(), comp.cuda_stream))
                ws_e = buf["ws_b"]
            else:
                ws_e = buf["ws_a"]
            ys_m = [ys[layer][self.specs[p].name] for p in members]
            n = len(members)
            y_arr = (ctypes.c_void_p * n)(*[y.data_ptr() for y in ys_m])
            ld_arr = (ctypes.c_int64 * n)(*[y.stride(0) for y in ys_m])
            b_arr = (ctypes.c_void_p * n)(*[st["b_ptrs"].data_ptr() + (layer * P + p) * S * 8 for p in members])
            native.check(lib.lsv_lora_expand_group(
                ctypes.addressof(y_arr), ctypes.addressof(ld_arr), ys_m[0].shape[0], ctypes.addressof(b_arr),
                plan_b.plan_dev.data_ptr(), plan_b.plan_host.ctypes.data, ws_e.data_ptr(), ws_e.numel(),
                comp.cuda_stream))

        for layer in range(self.slab.model.layers):
            for gi, (gname, members) in enumerate(self.groups):
                sp0 = self.specs[members[0]]
                plan_a = st["plans"][gi][0]
                buf = st["per_group"][gi]
                x = xs[layer][gname]
                ws_a = buf["ws_a"]
                native.check(lib.lsv_lora_shrink(x.data_ptr(), x.stride(0), x.shape[0], sp0.h_in,
                                                 st["a_ptrs"].data_ptr() + (layer * G + gi) * S * 8,
                                                 plan_a.plan_dev.data_ptr(), plan_a.plan_host.ctypes.data,
                                                 ws_a.data_ptr(), ws_a.numel(), comp.cuda_stream))
                shrunk = torch.cuda.Event()
                shrunk.record(comp)
                off, nb = self._region(plan_a)
                with torch.cuda.stream(comm):
                    comm.wait_event(shrunk)
                    if sp0.column:
                        dist.all_gather_into_tensor(buf["gathered"][:self.tp * nb], ws_a[off:off + nb], group=self.group)
                    else:
                        dist.all_reduce(ws_a[off:off + nb].view(torch.bfloat16), group=self.group)
                    exchanged = torch.cuda.Event()
                    exchanged.record(comm)
                if pending is not None:
                    finish(pending)
                pending = (layer, gi, exchanged)
        if pending is not None:
            finish(pending)
        comp.wait_stream(comm)
