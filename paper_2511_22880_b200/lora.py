"""LoraDeltaEngine: apply a co-batched, mixed-rank batch's LoRA deltas on one B200.

This is the operator the reference only prices: ``schedule_server`` forms a prefill batch
(simengine.py:96-152) and calls ``costmodel.prefill_time(lengths, ranks, params)``
(costmodel.py:83-105), which charges the whole batch the maximum rank.  Here the batch is
indexed into adapter segments (segments.py) and planned once per input group by liblsv's host
planner (per-segment tier + LPT work lists).  Per layer, each input group (q/k/v, o, gate/up,
down) is one fused ``lsv_lora_shrink`` (x read once, v = x·A_s^T for every member) followed by
one ``lsv_lora_expand_proj`` per member (y += v·B_s^T): y[t] += (x[t]·A_s^T)·B_s^T with each
segment paying its own rank.
"""

from __future__ import annotations

import concurrent.futures
import ctypes
import os
from dataclasses import dataclass, field

import numpy as np
import torch

from . import native
from .segments import Segments
from .shapes import INPUT_GROUPS, ModelShape, input_group  # noqa: F401  (re-exported)
from .slab import AdapterSlab


@dataclass
class ShapePlan:
    """One liblsv plan: an input group's fused shrink + each member's expand (h_outs[i]); a single
    projection is the one-member case (h_out = h_outs[0])."""
    h_in: int
    h_out: int
    plan_host: np.ndarray       # int32 blob (liblsv plan)
    plan_dev: torch.Tensor      # same blob in HBM
    workspace_bytes: int
    summary: tuple[int, ...]    # (S, N, h_in, h_out, simt_segs, mtiles, shrink_items, expand_items)
    h_outs: tuple[int, ...] = ()
    members: tuple[int, ...] = ()


@dataclass
class BatchPlan:
    segments: Segments
    group_plans: list[ShapePlan]   # one per model.groups() entry
    a_ptrs: torch.Tensor        # int64 [layers*groups, S]: group A tiles
    b_ptrs: torch.Tensor        # int64 [layers*projections, S]
    workspace: torch.Tensor     # uint8, zero-filled once
    tier_policy: int = native.TIER_AUTO
    extra: dict = field(default_factory=dict)

    @property
    def num_tokens(self) -> int:
        return self.segments.num_tokens

    @property
    def shape_plans(self) -> dict[tuple[int, int], ShapePlan]:
        """(h_in, h_out) -> the plan of the first group with a member of that shape."""
        out: dict[tuple[int, int], ShapePlan] = {}
        for gp in self.group_plans:
            for h in gp.h_outs:
                out.setdefault((gp.h_in, h), gp)
        return out


class _UploadRing:
    """Pinned host arena + device arena pairs for asynchronous plan uploads, reused round robin.

    A slot's host arena is refilled only after the event behind its last H2D copy has completed
    (normally long ago); its device arena is overwritten by a copy issued on the caller's stream,
    so it is stream-ordered behind every kernel that read the previous plan in that slot.  Steady
    state therefore allocates nothing (a cudaMalloc / cudaHostAlloc can serialise the device and
    drain a serving loop's pipeline) and waits for nothing.  Each reuse bumps the slot's
    generation; a plan whose slot has been reused is rejected (``check``)."""

    def __init__(self, slots: int = 4):
        self.host: list[torch.Tensor | None] = [None] * slots
        self.dev: list[torch.Tensor | None] = [None] * slots
        self.ev: list[torch.cuda.Event | None] = [None] * slots
        self.gen = [0] * slots
        self.last_stream: list = [None] * slots
        self.i = 0

    def upload(self, arrays: list[np.ndarray], device: torch.device, stream) -> tuple[list[torch.Tensor], tuple]:
        offs, total = [], 0
        for a in arrays:
            offs.append(total)
            total += (a.nbytes + 255) // 256 * 256
        k = self.i
        self.i = (self.i + 1) % len(self.host)
        if self.ev[k] is not None:
            self.ev[k].synchronize()
        if self.host[k] is None or self.host[k].numel() < total:
            cap = max(total, 1 << 20) * 3 // 2
            # size every never-used slot too, so growth happens once and not inside a later window
            for j in range(len(self.host)):
                if j == k or (self.ev[j] is None and (self.host[j] is None or self.host[j].numel() < cap)):
                    if self.dev[j] is not None and self.last_stream[j] is not None:
                        self.dev[j].record_stream(self.last_stream[j])   # in-flight readers keep it alive
                    self.host[j] = torch.empty(cap, dtype=torch.uint8, pin_memory=True)
                    self.dev[j] = torch.empty(cap, dtype=torch.uint8, device=device)
        self.gen[k] += 1
        self.last_stream[k] = stream
        host = self.host[k].numpy()
        for a, o in zip(arrays, offs):
            host[o:o + a.nbytes] = np.ascontiguousarray(a).reshape(-1).view(np.uint8)
        with torch.cuda.stream(stream):
            self.dev[k][:total].copy_(self.host[k][:total], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(stream)
        self.ev[k] = ev
        outs = [self.dev[k][o:o + a.nbytes].view(torch.from_numpy(a[:0]).dtype).view(a.shape)
                for a, o in zip(arrays, offs)]
        return outs, (k, self.gen[k])

    def check(self, tag: tuple) -> None:
        k, g = tag
        if self.gen[k] != g:
            raise RuntimeError(f"batch plan is stale: its upload slot was reused by a later prepare(stream=...) "
                               f"(at most {len(self.host)} stream-prepared plans are live at once)")


def build_group_plan(seg: Segments, h_in: int, h_outs, tier_policy: int, device: torch.device,
                     members: tuple[int, ...] = (), upload: bool = True,
                     seg_flags: np.ndarray | None = None) -> ShapePlan:
    """``seg_flags`` [S] int32 (LSV_SEG_REMOTE for peer-owned adapters) or None."""
    lib = native.lib()
    S = seg.num_segments
    indptr = np.ascontiguousarray(seg.seg_indptr, dtype=np.int32)
    ranks = np.ascontiguousarray(seg.seg_rank, dtype=np.int32)
    hs = np.ascontiguousarray(h_outs, dtype=np.int32)
    fl = None if seg_flags is None else np.ascontiguousarray(seg_flags, dtype=np.int32)
    fptr = None if fl is None else fl.ctypes.data
    pb = ctypes.c_size_t()
    wb = ctypes.c_size_t()
    native.check(lib.lsv_plan_size_group_ex(S, indptr.ctypes.data, ranks.ctypes.data, fptr, h_in, len(hs),
                                            hs.ctypes.data, tier_policy, ctypes.byref(pb), ctypes.byref(wb)))
    blob = np.zeros(pb.value // 4, dtype=np.int32)
    native.check(lib.lsv_plan_build_group_ex(S, indptr.ctypes.data, ranks.ctypes.data, fptr, h_in, len(hs),
                                             hs.ctypes.data, tier_policy, blob.ctypes.data, pb.value))
    summ = np.zeros(8, dtype=np.int32)
    native.check(lib.lsv_plan_summary(blob.ctypes.data, summ.ctypes.data))
    dev = torch.from_numpy(blob).to(device) if upload else None
    return ShapePlan(h_in, int(hs[0]), blob, dev, int(wb.value), tuple(int(v) for v in summ),
                     tuple(int(h) for h in hs), tuple(members))


def build_shape_plan(seg: Segments, h_in: int, h_out: int, tier_policy: int,
                     device: torch.device) -> ShapePlan:
    return build_group_plan(seg, h_in, [h_out], tier_policy, device)


class LoraDeltaEngine:
    """Mixed-rank LoRA delta over all layers/projections of one model on one GPU.

    Per layer and input group (model.groups(): q/k/v, o, gate/up, down) one fused shrink reads
    the group's x once and writes every member's v images; each member's expand follows."""

    def __init__(self, slab: AdapterSlab, tier_policy: int = native.TIER_AUTO, v_bf16: bool = False):
        """``v_bf16``: keep the tensor-core tier's intermediate v as one bf16 image
        (LSV_PLAN_V_BF16) instead of the default bf16 (hi, lo) pair (include/lsv.h)."""
        native.load()
        self.slab = slab
        self.model: ModelShape = slab.model
        self.device = slab.device
        self.tier_policy = tier_policy | (native.PLAN_V_BF16 if v_bf16 else 0)
        self.groups = self.model.groups()
        self._member = {p: (gi, i) for gi, (_, m) in enumerate(self.groups) for i, p in enumerate(m)}
        self._workspace: torch.Tensor | None = None
        self._ring = _UploadRing()
        self._pool = concurrent.futures.ThreadPoolExecutor(max_workers=max(1, len(self.groups)))

    # -- planning ----------------------------------------------------------------------
    def prepare(self, seg: Segments, seg_owner: np.ndarray | None = None,
                peer_slabs: dict[int, AdapterSlab] | None = None, stream=None,
                fused_linear: bool = False, remote_aware: bool = False, skip: np.ndarray | None = None,
                max_sms: int = 0) -> BatchPlan:
        """Plan a batch: one liblsv plan per input group + pointer tables.  With ``stream`` the
        uploads are asynchronous on that stream (pinned staging), so a serving loop can plan batch
        k+1 on the host while batch k still runs there.  ``fused_linear``: tile-aligned plans for
        ``linear_group`` (base GEMM with the delta fused, LSV_PLAN_TILE_ALIGNED; tensor-core tier).
        ``skip`` [S] bool: segments that keep their tokens but get no work (LSV_SEG_SKIP); ``max_sms``:
        grids of at most that many CTAs (LSV_PLAN_SMS) — together they split a batch into two plans
        that run side by side on disjoint SMs (``SplitStep``).  ``remote_aware``: mark peer-owned
        segments LSV_SEG_REMOTE (NVLink-weighted LPT cost, remote/local interleaving); off by default
        (the bytes-only plan measured faster with the layer kernel: 12.53 vs 12.95 ms on 2 GPUs)."""
        ws_need = 0
        projs = self.model.projections
        # the group plans are independent host work; ctypes drops the GIL inside the C++ planner,
        # so they build in parallel
        policy = self.tier_policy | (native.PLAN_TILE_ALIGNED if fused_linear else 0) | native.PLAN_SMS(max_sms)
        flags = None
        if seg_owner is not None and peer_slabs and remote_aware:
            me = self.device.index or 0
            own = np.asarray(seg_owner)
            remote = (own != me) & np.isin(own, list(peer_slabs))
            if remote.any():   # NVLink-aware LPT cost + remote/local interleaving (lsv_plan_build_group_ex)
                flags = np.where(remote, native.SEG_REMOTE, 0).astype(np.int32)
        if skip is not None and np.any(skip):
            flags = (np.zeros(seg.num_segments, dtype=np.int32) if flags is None else flags) | \
                np.where(np.asarray(skip, dtype=bool), native.SEG_SKIP, 0).astype(np.int32)
        futs = [self._pool.submit(build_group_plan, seg, projs[members[0]].h_in, [projs[p].h_out for p in members],
                                  policy, self.device, members, stream is None, flags)
                for _, members in self.groups]
        plans = [f.result() for f in futs]
        # forward: one workspace slice per (layer, group) (lsv_lora_forward_workspace)
        ph = (ctypes.c_void_p * len(plans))(*[gp.plan_host.ctypes.data for gp in plans])
        ws_need = native.lib().lsv_lora_forward_workspace(self.model.layers, len(plans), ctypes.addressof(ph))
        if self._workspace is None or self._workspace.numel() < ws_need:
            self._grow_workspace(ws_need, stream)
        a_tab, b_tab = self.slab.pointer_tables(seg.seg_slot, peer_slabs=peer_slabs, seg_owner=seg_owner,
                                                as_numpy=True)
        if stream is None:
            a_dev, b_dev = torch.from_numpy(a_tab).to(self.device), torch.from_numpy(b_tab).to(self.device)
        else:    # everything through one pinned arena, asynchronously on the stream
            up, tag = self._ring.upload([gp.plan_host for gp in plans] + [a_tab, b_tab], self.device, stream)
            for gp, t in zip(plans, up):
                gp.plan_dev = t
            a_dev, b_dev = up[-2], up[-1]
        bp = BatchPlan(seg, plans, a_dev, b_dev, self._workspace, policy)
        if stream is not None:
            bp.extra["ring_tag"] = tag
        return bp

    def _grow_workspace(self, need: int, stream) -> None:
        """Replace the shared workspace by a larger zero-filled one (growth only, rare).

        The split-K / TP grid barriers need zeroed counters, so the memset must be ordered before
        every kernel that uses the new buffer: it is issued on the stream the batch will run on
        (``stream``, or the current stream for eager callers, which is then synchronised).  The old
        buffer may still be read by kernels in flight on any stream, so the device is drained before
        it goes back to the caching allocator."""
        if self._workspace is not None:
            torch.cuda.synchronize(self.device)
            self._workspace = None
        st = stream if stream is not None else torch.cuda.current_stream(self.device)
        with torch.cuda.stream(st):
            # zero-filled once: the kernels leave their split counters at zero on exit
            ws = torch.zeros(max(need, 256), dtype=torch.uint8, device=self.device)
        ws.record_stream(st)
        if stream is None:
            st.synchronize()
        self._workspace = ws

    def _live(self, bp: BatchPlan) -> None:
        tag = bp.extra.get("ring_tag")
        if tag is not None:
            self._ring.check(tag)

    # -- execution ---------------------------------------------------------------------
    def apply(self, bp: BatchPlan, layer: int, proj: int, x: torch.Tensor, y: torch.Tensor,
              stream: torch.cuda.Stream | None = None) -> None:
        """y[:N] += delta for one (layer, projection); x [N, h_in], y [N, h_out] bf16.  (Runs the
        projection's whole group shrink; ``forward`` shares it across the group.)"""
        pr = self.model.projections[proj]
        self._check_io(x, y, pr.h_in, pr.h_out, bp.num_tokens)
        self.shrink(bp, layer, proj, x, stream)
        self.expand(bp, layer, proj, y, stream)

    def shrink(self, bp: BatchPlan, layer: int, proj: int, x: torch.Tensor, stream=None) -> None:
        """Fused shrink of proj's input group (v images of every member)."""
        self._live(bp)
        gi, _ = self._member[proj]
        gp = bp.group_plans[gi]
        S = bp.segments.num_segments
        row = layer * len(self.groups) + gi
        st = stream or torch.cuda.current_stream(self.device)
        native.check(native.lib().lsv_lora_shrink(
            x.data_ptr(), x.stride(0), x.shape[0], gp.h_in, bp.a_ptrs.data_ptr() + row * S * 8,
            gp.plan_dev.data_ptr(), gp.plan_host.ctypes.data, bp.workspace.data_ptr(),
            bp.workspace.numel(), st.cuda_stream))

    def expand(self, bp: BatchPlan, layer: int, proj: int, y: torch.Tensor, stream=None) -> None:
        self._live(bp)
        pr = self.model.projections[proj]
        gi, idx = self._member[proj]
        gp = bp.group_plans[gi]
        S = bp.segments.num_segments
        row = layer * len(self.model.projections) + proj
        st = stream or torch.cuda.current_stream(self.device)
        native.check(native.lib().lsv_lora_expand_proj(
            y.data_ptr(), y.stride(0), y.shape[0], pr.h_out, idx, bp.b_ptrs.data_ptr() + row * S * 8,
            gp.plan_dev.data_ptr(), gp.plan_host.ctypes.data, bp.workspace.data_ptr(),
            bp.workspace.numel(), st.cuda_stream))

    def expand_group(self, bp: BatchPlan, layer: int, gi: int, ys: list[torch.Tensor], stream=None) -> None:
        """Every member of input group gi in one launch (one LPT list over all members' items)."""
        self._live(bp)
        gp = bp.group_plans[gi]
        members = self.groups[gi][1]
        S = bp.segments.num_segments
        P = len(self.model.projections)
        st = stream or torch.cuda.current_stream(self.device)
        n = len(members)
        y_arr = (ctypes.c_void_p * n)(*[y.data_ptr() for y in ys])
        ld_arr = (ctypes.c_int64 * n)(*[y.stride(0) for y in ys])
        b_arr = (ctypes.c_void_p * n)(*[bp.b_ptrs.data_ptr() + (layer * P + p) * S * 8 for p in members])
        native.check(native.lib().lsv_lora_expand_group(
            ctypes.addressof(y_arr), ctypes.addressof(ld_arr), ys[0].shape[0], ctypes.addressof(b_arr),
            gp.plan_dev.data_ptr(), gp.plan_host.ctypes.data, bp.workspace.data_ptr(), bp.workspace.numel(),
            st.cuda_stream))

    def forward(self, bp: BatchPlan, xs: list[dict[str, torch.Tensor]], ys: list[dict[str, torch.Tensor]],
                stream=None, serial: bool = False) -> None:
        """Every layer and projection: xs[l][input_group], ys[l][proj_name] — one native call
        (lsv_lora_forward_ex) that issues each layer's group shrinks and group expands in order.
        ``serial``: every launch waits for the previous one (no shrink starting under the previous
        group's expand), as in a model where each group's input depends on the previous output."""
        self._live(bp)
        projs = self.model.projections
        L, G = self.model.layers, len(self.groups)
        order = [p for _, m in self.groups for p in m]
        if order != list(range(len(projs))):
            raise ValueError("projections must be numbered group by group")
        xl, ldx, yl, ldy = [], [], [], []
        for layer in range(L):
            for gname, members in self.groups:
                x = xs[layer][gname]
                xl.append(x.data_ptr()); ldx.append(x.stride(0))
                for p in members:
                    y = ys[layer][projs[p].name]
                    self._check_io(x, y, projs[p].h_in, projs[p].h_out, bp.num_tokens)
                    yl.append(y.data_ptr()); ldy.append(y.stride(0))
        arr = lambda t, v: (t * len(v))(*v)   # noqa: E731
        pd = arr(ctypes.c_void_p, [gp.plan_dev.data_ptr() for gp in bp.group_plans])
        ph = arr(ctypes.c_void_p, [gp.plan_host.ctypes.data for gp in bp.group_plans])
        xa, la, ya, lya = (arr(ctypes.c_void_p, xl), arr(ctypes.c_int64, ldx), arr(ctypes.c_void_p, yl),
                           arr(ctypes.c_int64, ldy))
        st = stream or torch.cuda.current_stream(self.device)
        native.check(native.lib().lsv_lora_forward_ex(
            L, G, ctypes.addressof(pd), ctypes.addressof(ph), ctypes.addressof(xa), ctypes.addressof(la),
            ctypes.addressof(ya), ctypes.addressof(lya), bp.a_ptrs.data_ptr(), bp.b_ptrs.data_ptr(),
            xs[0][self.groups[0][0]].shape[0], bp.workspace.data_ptr(), bp.workspace.numel(),
            native.FWD_SERIAL if serial else 0, st.cuda_stream))

    def linear_group(self, bp: BatchPlan, layer: int, gi: int, x: torch.Tensor, weights: list[torch.Tensor],
                     ys: list[torch.Tensor], stream=None) -> None:
        """One LoRA linear layer for input group gi: ys[i] = x · weights[i]^T + delta_i for every member
        (weights[i]: the base projection's nn.Linear weight [h_out, h_in] bf16), with the delta
        accumulated into the base GEMM's TMEM tile (lsv_lora_fused_linear: the group's shrink, then
        one fused GEMM launch for every member).  ``bp`` from ``prepare(seg, fused_linear=True)``."""
        self._live(bp)
        if not (bp.tier_policy & native.PLAN_TILE_ALIGNED):
            raise ValueError("linear_group needs a plan from prepare(seg, fused_linear=True)")
        gp = bp.group_plans[gi]
        members = self.groups[gi][1]
        n = len(members)
        if len(weights) != n or len(ys) != n:
            raise ValueError(f"input group {self.groups[gi][0]} has {n} members")
        projs = self.model.projections
        for w, y, p in zip(weights, ys, members):
            self._check_io(x, y, projs[p].h_in, projs[p].h_out, bp.num_tokens)
            if w.dtype != torch.bfloat16 or tuple(w.shape) != (projs[p].h_out, projs[p].h_in) or w.stride(1) != 1:
                raise ValueError(f"weight of {projs[p].name} must be bf16 [{projs[p].h_out}, {projs[p].h_in}]")
        S = bp.segments.num_segments
        P = len(projs)
        st = stream or torch.cuda.current_stream(self.device)
        arr = lambda t, v: (t * len(v))(*v)   # noqa: E731
        wa, lw = arr(ctypes.c_void_p, [w.data_ptr() for w in weights]), arr(ctypes.c_int64, [w.stride(0) for w in weights])
        ya, ly = arr(ctypes.c_void_p, [y.data_ptr() for y in ys]), arr(ctypes.c_int64, [y.stride(0) for y in ys])
        ba = arr(ctypes.c_void_p, [bp.b_ptrs.data_ptr() + (layer * P + p) * S * 8 for p in members])
        native.check(native.lib().lsv_lora_fused_linear(
            x.data_ptr(), x.stride(0), x.shape[0], gp.h_in, bp.a_ptrs.data_ptr() + (layer * len(self.groups) + gi) * S * 8,
            ctypes.addressof(wa), ctypes.addressof(lw), ctypes.addressof(ya), ctypes.addressof(ly), ctypes.addressof(ba),
            gp.plan_dev.data_ptr(), gp.plan_host.ctypes.data, bp.workspace.data_ptr(), bp.workspace.numel(),
            st.cuda_stream))

    def forward_prefetch(self, bp: BatchPlan, pf: "RemotePrefetch", xs, ys, stream=None) -> None:
        """``forward`` with peer-owned adapters fetched one layer ahead into local staging buffers by
        the copy engines (lsv_copy_blocks) while the current layer computes, so the kernels only
        read local HBM.  ``bp`` must come from ``pf.plan``."""
        self._live(bp)
        st = stream or torch.cuda.current_stream(self.device)
        cs = pf.copy_stream
        L = self.model.layers
        cs.wait_stream(st)                                # fork: the copy stream joins st's work
        pf.fetch(0, cs)
        for layer in range(L):
            if layer + 1 < L:
                if layer >= 1:                            # buffer (layer+1)%2 was read by layer-1
                    cs.wait_event(pf.done[(layer - 1) % 2])
                pf.fetch(layer + 1, cs)
            st.wait_event(pf.ready[layer % 2])
            self._forward_layers(bp, xs, ys, st, layer, 1)
            pf.done[layer % 2].record(st)
        st.wait_stream(cs)                                # join

    def _forward_layers(self, bp, xs, ys, st, l0: int, nl: int) -> None:
        projs = self.model.projections
        G, P = len(self.groups), len(projs)
        S = bp.segments.num_segments
        xl, ldx, yl, ldy = [], [], [], []
        for layer in range(l0, l0 + nl):
            for gname, members in self.groups:
                x = xs[layer][gname]
                xl.append(x.data_ptr()); ldx.append(x.stride(0))
                for p in members:
                    y = ys[layer][projs[p].name]
                    yl.append(y.data_ptr()); ldy.append(y.stride(0))
        arr = lambda t, v: (t * len(v))(*v)   # noqa: E731
        pd = arr(ctypes.c_void_p, [gp.plan_dev.data_ptr() for gp in bp.group_plans])
        ph = arr(ctypes.c_void_p, [gp.plan_host.ctypes.data for gp in bp.group_plans])
        xa, la, ya, lya = (arr(ctypes.c_void_p, xl), arr(ctypes.c_int64, ldx), arr(ctypes.c_void_p, yl),
                           arr(ctypes.c_int64, ldy))
        # the whole workspace: this call's layers reuse the slices (and barrier pairs) of layers
        # [0, nl); its first launch is a plain one, ordered after the previous call's kernels
        native.check(native.lib().lsv_lora_forward(
            nl, G, ctypes.addressof(pd), ctypes.addressof(ph), ctypes.addressof(xa), ctypes.addressof(la),
            ctypes.addressof(ya), ctypes.addressof(lya), bp.a_ptrs.data_ptr() + l0 * G * S * 8,
            bp.b_ptrs.data_ptr() + l0 * P * S * 8, xs[l0][self.groups[0][0]].shape[0],
            bp.workspace.data_ptr(), bp.workspace.numel(), st.cuda_stream))

    @staticmethod
    def group_kernel_eligible(gp) -> bool:
        """Whether ``forward`` runs this group plan as one group kernel (lsv_api.cu
        group_kernel_eligible: tcgen05 tier only, not tile-aligned, LSV_GROUP_KERNEL not 0)."""
        h = gp.plan_host[:64]
        n_exp = int(h[60]) if int(h[33]) > 1 else int(h[53])
        return (os.environ.get("LSV_GROUP_KERNEL", "1") != "0" and int(h[6]) == 0 and int(h[62]) == 0
                and int(h[8]) > 0 and n_exp > 0)

    def launches_per_step(self, bp: BatchPlan, serial: bool = False) -> int:
        """Kernels one ``forward`` launches: one layer kernel per layer when every group runs as a
        group kernel (overlap-free calls, at most 4 groups); else one group kernel per tcgen05-only
        group, otherwise SIMT + tcgen05 shrink per group and SIMT (per member) + tcgen05 expand."""
        if (not serial and os.environ.get("LSV_LAYER_KERNEL", "1") != "0" and len(bp.group_plans) <= 4
                and all(self.group_kernel_eligible(gp) for gp in bp.group_plans)):
            return self.model.layers
        n = 0
        for gp in bp.group_plans:
            if self.group_kernel_eligible(gp):
                n += 1
                continue
            simt = 1 if gp.summary[4] else 0
            h = gp.plan_host[:64]
            n += simt + (1 if gp.summary[6] else 0)                     # shrink
            n += simt * len(gp.h_outs) + (1 if int(h[60]) else 0)       # expand: SIMT per member + one tcgen05
        return n * self.model.layers

    def forward_layer(self, bp: BatchPlan, layer: int, xs_l: dict[str, torch.Tensor], ys_l: dict[str, torch.Tensor],
                      stream=None) -> None:
        """Every input group of one layer through lsv_lora_forward_ex (one layer): the layer kernel when
        every group plan is eligible (bench.py times the dominant kernel with it)."""
        self._live(bp)
        projs = self.model.projections
        G, P, S = len(self.groups), len(projs), bp.segments.num_segments
        arr = lambda t, v: (t * len(v))(*v)   # noqa: E731
        xl = [xs_l[g] for g, _ in self.groups]
        yl = [ys_l[projs[p].name] for _, m in self.groups for p in m]
        pd = arr(ctypes.c_void_p, [gp.plan_dev.data_ptr() for gp in bp.group_plans])
        ph = arr(ctypes.c_void_p, [gp.plan_host.ctypes.data for gp in bp.group_plans])
        xa, la = arr(ctypes.c_void_p, [x.data_ptr() for x in xl]), arr(ctypes.c_int64, [x.stride(0) for x in xl])
        ya, lya = arr(ctypes.c_void_p, [y.data_ptr() for y in yl]), arr(ctypes.c_int64, [y.stride(0) for y in yl])
        st = stream or torch.cuda.current_stream(self.device)
        native.check(native.lib().lsv_lora_forward_ex(
            1, G, ctypes.addressof(pd), ctypes.addressof(ph), ctypes.addressof(xa), ctypes.addressof(la),
            ctypes.addressof(ya), ctypes.addressof(lya), bp.a_ptrs.data_ptr() + layer * G * S * 8,
            bp.b_ptrs.data_ptr() + layer * P * S * 8, xl[0].shape[0], bp.workspace.data_ptr(),
            bp.workspace.numel(), 0, st.cuda_stream))

    def forward_group(self, bp: BatchPlan, layer: int, gi: int, x: torch.Tensor, ys: list[torch.Tensor],
                      stream=None) -> None:
        """Input group gi of one layer through lsv_lora_forward_ex (one layer, one group): the group
        kernel when the plan is eligible (bench.py times the dominant kernel with it)."""
        self._live(bp)
        gp = bp.group_plans[gi]
        members = self.groups[gi][1]
        S = bp.segments.num_segments
        P = len(self.model.projections)
        G = len(self.groups)
        arr = lambda t, v: (t * len(v))(*v)   # noqa: E731
        pd, ph = arr(ctypes.c_void_p, [gp.plan_dev.data_ptr()]), arr(ctypes.c_void_p, [gp.plan_host.ctypes.data])
        xa, la = arr(ctypes.c_void_p, [x.data_ptr()]), arr(ctypes.c_int64, [x.stride(0)])
        ya, lya = arr(ctypes.c_void_p, [y.data_ptr() for y in ys]), arr(ctypes.c_int64, [y.stride(0) for y in ys])
        # a_ptrs rows are (layer, group), b_ptrs rows (layer, projection): this group's rows only
        a_tab = bp.a_ptrs.data_ptr() + (layer * G + gi) * S * 8
        b_tab = bp.b_ptrs.data_ptr() + (layer * P + members[0]) * S * 8
        st = stream or torch.cuda.current_stream(self.device)
        native.check(native.lib().lsv_lora_forward_ex(
            1, 1, ctypes.addressof(pd), ctypes.addressof(ph), ctypes.addressof(xa), ctypes.addressof(la),
            ctypes.addressof(ya), ctypes.addressof(lya), a_tab, b_tab, x.shape[0], bp.workspace.data_ptr(),
            bp.workspace.numel(), 0, st.cuda_stream))

    @staticmethod
    def _check_io(x: torch.Tensor, y: torch.Tensor, h_in: int, h_out: int, n: int) -> None:
        if x.dtype != torch.bfloat16 or y.dtype != torch.bfloat16:
            raise ValueError("x and y must be bfloat16")
        if x.dim() != 2 or y.dim() != 2 or x.shape[1] != h_in or y.shape[1] != h_out:
            raise ValueError(f"expected x [N, {h_in}] and y [N, {h_out}], got {tuple(x.shape)}, {tuple(y.shape)}")
        if x.shape[0] < n or y.shape[0] < n:
            raise ValueError(f"x/y have fewer rows than the batch's {n} tokens")
        if x.stride(1) != 1 or y.stride(1) != 1:
            raise ValueError("x and y rows must be contiguous")


def moved_bytes(seg: Segments, model: ModelShape) -> int:
    """Bytes one layer moves with input-group fusion: x read once per group, A/B once per segment,
    y read+write per projection (v and metadata excluded)."""
    n = seg.lengths().astype(np.int64)
    r = seg.seg_rank.astype(np.int64)
    total = 0
    for _, members in model.groups():
        total += int(np.sum(2 * n * model.projections[members[0]].h_in))
        for p in members:
            pr = model.projections[p]
            total += int(np.sum(2 * r * pr.h_in + 2 * r * pr.h_out + 4 * n * pr.h_out))
    return total


def algorithmic_bytes(seg: Segments, h_in: int, h_out: int) -> int:
    """Bytes one projection must move: x read, A and B read once per segment,
    y read+write, bf16.  v and metadata excluded."""
    n = seg.lengths().astype(np.int64)
    r = seg.seg_rank.astype(np.int64)
    return int(np.sum(2 * n * h_in + 2 * r * h_in + 2 * r * h_out + 4 * n * h_out))


def algorithmic_flops(seg: Segments, h_in: int, h_out: int) -> int:
    n = seg.lengths().astype(np.int64)
    r = seg.seg_rank.astype(np.int64)
    return int(np.sum(2 * n * r * (h_in + h_out)))


class SplitStep:
    """Config 4 with the SMs partitioned: the batch's peer-owned segments run on ``remote_sms`` CTAs
    (their plan skips every local segment) while the local segments run on the rest (their plan skips
    the remote ones), each as its own forward on its own stream.  NVLink reads then stream at the
    link's rate on a few SMs without holding up the local HBM pipeline in the same CTAs (in-order
    rings make a slow peer tile stall every local item queued behind it).  y rows of the two plans
    are disjoint segments, so the two forwards never touch the same output."""

    def __init__(self, slab: AdapterSlab, seg: Segments, seg_owner: np.ndarray,
                 peer_slabs: dict[int, AdapterSlab], remote_sms: int = 24, v_bf16: bool = False):
        me = slab.device.index or 0
        remote = np.asarray(seg_owner) != me
        self.local_eng = LoraDeltaEngine(slab, v_bf16=v_bf16)
        self.remote_eng = LoraDeltaEngine(slab, v_bf16=v_bf16)   # its own workspace
        nsm = native.lib().lsv_num_sms()
        self.bp_local = self.local_eng.prepare(seg, skip=remote, max_sms=max(1, nsm - remote_sms))
        self.bp_remote = self.remote_eng.prepare(seg, seg_owner=seg_owner, peer_slabs=peer_slabs, skip=~remote,
                                                 max_sms=remote_sms, remote_aware=False)
        self.side = torch.cuda.Stream(slab.device)

    def forward(self, xs, ys, stream=None) -> None:
        st = stream or torch.cuda.current_stream(self.local_eng.device)
        self.side.wait_stream(st)
        self.remote_eng.forward(self.bp_remote, xs, ys, self.side)
        self.local_eng.forward(self.bp_local, xs, ys, st)
        st.wait_stream(self.side)


class RemotePrefetch:
    """Peer-owned adapters fetched a layer ahead (the reference's fetch_remote, pool.py:101-132,
    as copy-engine copies over NVLink instead of in-kernel peer loads).

    Segment s with ``seg_owner[s] != this GPU`` has its layer-l block (all group A tiles and B tiles
    of the layer, contiguous in the owner's slab, ``AdapterSlab.layer_block``) copied into staging
    buffer l % 2; ``plan`` builds a BatchPlan whose pointer tables send those segments' layer-l
    pointers to the staging copy."""

    ALIGN = 1024

    def __init__(self, eng: LoraDeltaEngine, seg: Segments, seg_owner: np.ndarray,
                 peer_slabs: dict[int, AdapterSlab]):
        self.eng, self.seg = eng, seg
        self.device = eng.device
        me = eng.device.index or 0
        model = eng.model
        self.remote = [s for s in range(seg.num_segments)
                       if int(seg_owner[s]) != me and int(seg_owner[s]) in peer_slabs]
        self.owner = seg_owner
        self.peers = peer_slabs
        self.stage_off = {}
        cur = 0
        for s in self.remote:
            self.stage_off[s] = cur
            cur += (model.adapter_bytes(int(seg.seg_rank[s])) // model.layers + self.ALIGN - 1) // self.ALIGN * self.ALIGN
        self.stage_bytes = max(cur, self.ALIGN)
        self.stage = [torch.empty(self.stage_bytes, dtype=torch.uint8, device=self.device) for _ in range(2)]
        # per layer: source addresses, destinations (buffer l % 2), sizes
        self._src = np.zeros((model.layers, len(self.remote)), dtype=np.uint64)
        self._dst = np.zeros((model.layers, len(self.remote)), dtype=np.uint64)
        self._len = np.zeros(len(self.remote), dtype=np.uint64)
        for i, s in enumerate(self.remote):
            peer = peer_slabs[int(seg_owner[s])]
            slot = int(seg.seg_slot[s])
            for l in range(model.layers):
                off, nb = peer.layer_block(slot, l)
                self._src[l, i] = peer.base + off
                self._dst[l, i] = self.stage[l % 2].data_ptr() + self.stage_off[s]
                self._len[i] = nb
        self.copy_stream = torch.cuda.Stream(self.device)
        self.ready = [torch.cuda.Event() for _ in range(2)]
        self.done = [torch.cuda.Event() for _ in range(2)]

    @property
    def bytes_per_layer(self) -> int:
        return int(self._len.sum())

    def fetch(self, layer: int, stream) -> None:
        """Copy layer ``layer`` of every remote segment into staging buffer layer % 2 on ``stream``
        and record ``ready[layer % 2]`` there."""
        n = len(self.remote)
        if n:
            native.check(native.lib().lsv_copy_blocks(
                n, self._src[layer].ctypes.data, self._dst[layer].ctypes.data, self._len.ctypes.data,
                stream.cuda_stream))
        self.ready[layer % 2].record(stream)

    def plan(self) -> BatchPlan:
        """BatchPlan whose remote segments point into the staging buffers (layer parity)."""
        eng, seg, model = self.eng, self.seg, self.eng.model
        bp = eng.prepare(seg)                       # local pointers everywhere
        L, G, P = model.layers, len(eng.groups), len(model.projections)
        S = seg.num_segments
        a = bp.a_ptrs.cpu().numpy().reshape(L, G, S).copy()
        b = bp.b_ptrs.cpu().numpy().reshape(L, P, S).copy()
        for s in self.remote:
            peer = self.peers[int(self.owner[s])]
            slot = int(seg.seg_slot[s])
            for l in range(L):
                base, _ = peer.layer_block(slot, l)
                dst = self.stage[l % 2].data_ptr() + self.stage_off[s]
                for gi in range(G):
                    a[l, gi, s] = dst + int(peer._g_off_rows[slot][l, gi]) - base
                for p in range(P):
                    b[l, p, s] = dst + int(peer._b_off_rows[slot][l, p]) - base
        bp.a_ptrs = torch.from_numpy(a.reshape(L * G, S)).to(self.device)
        bp.b_ptrs = torch.from_numpy(b.reshape(L * P, S)).to(self.device)
        return bp
