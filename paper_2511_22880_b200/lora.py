"""LoraDeltaEngine: apply a co-batched, mixed-rank batch's LoRA deltas on one B200.

This is the operator the reference only prices: ``schedule_server`` forms a prefill batch
(simengine.py:96-152) and calls ``costmodel.prefill_time(lengths, ranks, params)``
(costmodel.py:83-105), which charges the whole batch the maximum rank.  Here the batch is
indexed into adapter segments (segments.py), planned once per projection shape by liblsv's
host planner (per-segment tier + LPT work lists), and every layer/projection is one
``lsv_lora_apply`` call: y[t] += (x[t]·A_s^T)·B_s^T with each segment paying its own rank.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np
import torch

from . import native
from .segments import Segments
from .shapes import ModelShape
from .slab import AdapterSlab


@dataclass
class ShapePlan:
    h_in: int
    h_out: int
    plan_host: np.ndarray       # int32 blob (liblsv plan)
    plan_dev: torch.Tensor      # same blob in HBM
    workspace_bytes: int
    summary: tuple[int, ...]    # (S, N, h_in, h_out, simt_segs, mtiles, shrink_items, expand_items)


@dataclass
class BatchPlan:
    segments: Segments
    shape_plans: dict[tuple[int, int], ShapePlan]
    a_ptrs: torch.Tensor        # int64 [layers*projections, S]
    b_ptrs: torch.Tensor
    workspace: torch.Tensor     # uint8, zero-filled once
    tier_policy: int = native.TIER_AUTO
    extra: dict = field(default_factory=dict)

    @property
    def num_tokens(self) -> int:
        return self.segments.num_tokens


def build_shape_plan(seg: Segments, h_in: int, h_out: int, tier_policy: int,
                     device: torch.device) -> ShapePlan:
    lib = native.lib()
    S = seg.num_segments
    indptr = np.ascontiguousarray(seg.seg_indptr, dtype=np.int32)
    ranks = np.ascontiguousarray(seg.seg_rank, dtype=np.int32)
    pb = ctypes.c_size_t()
    wb = ctypes.c_size_t()
    native.check(lib.lsv_plan_size(S, indptr.ctypes.data, ranks.ctypes.data, h_in, h_out, tier_policy,
                                   ctypes.byref(pb), ctypes.byref(wb)))
    blob = np.zeros(pb.value // 4, dtype=np.int32)
    native.check(lib.lsv_plan_build(S, indptr.ctypes.data, ranks.ctypes.data, h_in, h_out, tier_policy,
                                    blob.ctypes.data, pb.value))
    summ = np.zeros(8, dtype=np.int32)
    native.check(lib.lsv_plan_summary(blob.ctypes.data, summ.ctypes.data))
    dev = torch.from_numpy(blob).to(device)
    return ShapePlan(h_in, h_out, blob, dev, int(wb.value), tuple(int(v) for v in summ))


class LoraDeltaEngine:
    """Mixed-rank LoRA delta over all layers/projections of one model on one GPU."""

    def __init__(self, slab: AdapterSlab, tier_policy: int = native.TIER_AUTO):
        native.load()
        self.slab = slab
        self.model: ModelShape = slab.model
        self.device = slab.device
        self.tier_policy = tier_policy
        self._workspace: torch.Tensor | None = None

    # -- planning ----------------------------------------------------------------------
    def prepare(self, seg: Segments, seg_owner: np.ndarray | None = None,
                peer_slabs: dict[int, AdapterSlab] | None = None) -> BatchPlan:
        """Plan a batch: one liblsv plan per distinct projection shape + pointer tables."""
        plans = {}
        ws_need = 0
        for (h_in, h_out) in self.model.shapes():
            sp = build_shape_plan(seg, h_in, h_out, self.tier_policy, self.device)
            plans[(h_in, h_out)] = sp
            ws_need = max(ws_need, sp.workspace_bytes)
        if self._workspace is None or self._workspace.numel() < ws_need:
            # zero-filled once: the kernels leave their split counters at zero on exit
            self._workspace = torch.zeros(max(ws_need, 256), dtype=torch.uint8, device=self.device)
        a_ptrs, b_ptrs = self.slab.pointer_tables(seg.seg_slot, peer_slabs=peer_slabs, seg_owner=seg_owner)
        return BatchPlan(seg, plans, a_ptrs, b_ptrs, self._workspace, self.tier_policy)

    # -- execution ---------------------------------------------------------------------
    def apply(self, bp: BatchPlan, layer: int, proj: int, x: torch.Tensor, y: torch.Tensor,
              stream: torch.cuda.Stream | None = None) -> None:
        """y[:N] += delta for one (layer, projection); x [N, h_in], y [N, h_out] bf16."""
        pr = self.model.projections[proj]
        sp = bp.shape_plans[(pr.h_in, pr.h_out)]
        self._check_io(x, y, pr.h_in, pr.h_out, bp.num_tokens)
        S = bp.segments.num_segments
        row = layer * len(self.model.projections) + proj
        st = stream or torch.cuda.current_stream(self.device)
        native.check(native.lib().lsv_lora_apply(
            x.data_ptr(), x.stride(0), y.data_ptr(), y.stride(0), native.LSV_DTYPE_BF16, x.shape[0],
            pr.h_in, pr.h_out, bp.a_ptrs.data_ptr() + row * S * 8, bp.b_ptrs.data_ptr() + row * S * 8,
            sp.plan_dev.data_ptr(), sp.plan_host.ctypes.data, bp.workspace.data_ptr(),
            bp.workspace.numel(), st.cuda_stream))

    def shrink(self, bp: BatchPlan, layer: int, proj: int, x: torch.Tensor, stream=None) -> None:
        pr = self.model.projections[proj]
        sp = bp.shape_plans[(pr.h_in, pr.h_out)]
        S = bp.segments.num_segments
        row = layer * len(self.model.projections) + proj
        st = stream or torch.cuda.current_stream(self.device)
        native.check(native.lib().lsv_lora_shrink(
            x.data_ptr(), x.stride(0), x.shape[0], pr.h_in, bp.a_ptrs.data_ptr() + row * S * 8,
            sp.plan_dev.data_ptr(), sp.plan_host.ctypes.data, bp.workspace.data_ptr(),
            bp.workspace.numel(), st.cuda_stream))

    def expand(self, bp: BatchPlan, layer: int, proj: int, y: torch.Tensor, stream=None) -> None:
        pr = self.model.projections[proj]
        sp = bp.shape_plans[(pr.h_in, pr.h_out)]
        S = bp.segments.num_segments
        row = layer * len(self.model.projections) + proj
        st = stream or torch.cuda.current_stream(self.device)
        native.check(native.lib().lsv_lora_expand(
            y.data_ptr(), y.stride(0), y.shape[0], pr.h_out, bp.b_ptrs.data_ptr() + row * S * 8,
            sp.plan_dev.data_ptr(), sp.plan_host.ctypes.data, bp.workspace.data_ptr(),
            bp.workspace.numel(), st.cuda_stream))

    def forward(self, bp: BatchPlan, xs: list[dict[str, torch.Tensor]], ys: list[dict[str, torch.Tensor]],
                stream=None) -> None:
        """Every layer and projection: xs[l][input_group], ys[l][proj_name]."""
        for layer in range(self.model.layers):
            for p, pr in enumerate(self.model.projections):
                self.apply(bp, layer, p, xs[layer][input_group(pr.name)], ys[layer][pr.name], stream)

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


INPUT_GROUPS = {"q_proj": "attn_in", "k_proj": "attn_in", "v_proj": "attn_in", "o_proj": "attn_out",
                "gate_proj": "mlp_in", "up_proj": "mlp_in", "down_proj": "mlp_mid"}


def input_group(proj_name: str) -> str:
    """Which activation a projection reads (q/k/v share the attention input, gate/up the MLP input)."""
    return INPUT_GROUPS.get(proj_name, proj_name)


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
