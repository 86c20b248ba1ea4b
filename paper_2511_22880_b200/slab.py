"""HBM adapter slab: the B200 form of the reference's per-server GPU adapter slots.

Reference: ``AdapterPool`` keeps, per server, an LRU set of GPU-resident adapters
(pool.py:88-99 ``touch_gpu``/``is_gpu_resident``, capacity ``gpu_slots`` config.py:29,
pool.py:20) and prices making one resident (``plan_fetch`` pool.py:101-132,
``fetch_latency`` costmodel.py:129-143).  Here a resident adapter is real memory: for every
layer and projection of the model, its lora_A/lora_B packed once into the tiled layouts the
kernels move with single bulk copies (include/lsv.h ``lsv_pack_adapter``).  The A matrices of the
projections that read the same activation (q/k/v, gate/up: ``ModelShape.groups``) share one group
tile per layer (``lsv_pack_adapter_group``), so one shrink reads x once for all of them.  Slots are
allocated from one large device buffer sized for B200's 180 GB of HBM; a segment's A/B
pointers are ``base + offset`` — or an NVLink peer address when the adapter lives in another
GPU's slab (the reference's ``fetch_remote``).
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import native
from .shapes import ModelShape, kpad


@dataclass
class SlotInfo:
    slot: int
    adapter_id: str
    rank: int
    offset: int        # byte offset of the slot inside the slab buffer
    nbytes: int


class AdapterSlab:
    """Adapters of one model resident in one GPU's HBM."""

    ALIGN = 1024

    def __init__(self, model: ModelShape, capacity_bytes: int, device: torch.device | str,
                 _peer_base: int | None = None):
        self.model = model
        self.device = torch.device(device)
        self.capacity = int(capacity_bytes)
        self._owned = _peer_base is None
        if self._owned:   # one cudaMalloc owned by liblsv: its base is exactly what IPC exports
            ptr = ctypes.c_void_p()
            native.check(native.lib().lsv_slab_alloc(self.capacity, self.device.index or 0, ctypes.byref(ptr)))
            self.base = int(ptr.value)
        else:             # a view of another process's slab, mapped over NVLink (open_peer)
            self.base = int(_peer_base)
        self.slots: list[SlotInfo] = []
        self.by_id: dict[str, int] = {}
        self._cursor = 0
        self._a_off_rows: list[np.ndarray] = []   # per slot: [layers, projections] byte offsets
        self._g_off_rows: list[np.ndarray] = []   # per slot: [layers, input groups] group A tiles
        self._member = {p: (gi, i, len(m)) for gi, (_, m) in enumerate(model.groups()) for i, p in enumerate(m)}
        self._b_off_rows: list[np.ndarray] = []
        self._slot_offsets_dev: tuple[torch.Tensor, torch.Tensor] | None = None
        self._free: dict[int, list[int]] = {}      # rank -> freed slots (reused by allocate)

    # -- allocation --------------------------------------------------------------------
    def slot_bytes(self, rank: int) -> int:
        return self.model.adapter_bytes(rank)

    @staticmethod
    def capacity_for(model: ModelShape, ranks) -> int:
        """Slab bytes for a roster of adapter ranks (with slot alignment)."""
        return sum(model.adapter_bytes(int(r)) + AdapterSlab.ALIGN for r in ranks) + AdapterSlab.ALIGN

    def free_bytes(self) -> int:
        return self.capacity - self._cursor

    def allocate(self, adapter_id: str, rank: int) -> int:
        """A slot for the adapter: a freed slot of the same rank (same size, same offsets) if there is
        one (pool.py:91-99: an evicted GPU slot is reused), else new space after the last slot."""
        if adapter_id in self.by_id:
            raise ValueError(f"adapter {adapter_id!r} already resident")
        if rank < 8 or rank % 8 or rank > 256:
            raise ValueError(f"adapter {adapter_id!r}: rank must be a multiple of 8 in [8, 256], got {rank}")
        free = self._free.get(rank)
        if free:
            slot = free.pop()
            self.slots[slot].adapter_id = adapter_id
            self.by_id[adapter_id] = slot
            return slot
        nbytes = self.slot_bytes(rank)
        start = (self._cursor + self.ALIGN - 1) // self.ALIGN * self.ALIGN
        if start + nbytes > self.capacity:
            raise MemoryError(f"slab full: adapter {adapter_id!r} needs {nbytes} bytes, "
                              f"{self.capacity - start} free")
        slot = len(self.slots)
        self.slots.append(SlotInfo(slot, adapter_id, rank, start, nbytes))
        self.by_id[adapter_id] = slot
        L, P = self.model.layers, len(self.model.projections)
        groups = self.model.groups()
        a_off = np.empty((L, P), dtype=np.int64)
        g_off = np.empty((L, len(groups)), dtype=np.int64)
        b_off = np.empty((L, P), dtype=np.int64)
        cur = start
        kp = kpad(rank)
        for l in range(L):
            for gi, (_, members) in enumerate(groups):
                # one group A tile [h_in/64][len(members)*rank][64]: member i's rows start at i*rank
                g_off[l, gi] = cur
                for i, p in enumerate(members):
                    a_off[l, p] = cur + i * rank * 128
                cur += 2 * len(members) * rank * self.model.projections[members[0]].h_in
                for p in members:
                    b_off[l, p] = cur
                    cur += 2 * kp * self.model.projections[p].h_out
        assert cur - start == nbytes
        self._a_off_rows.append(a_off)
        self._g_off_rows.append(g_off)
        self._b_off_rows.append(b_off)
        self._cursor = start + nbytes
        self._slot_offsets_dev = None
        return slot

    def free(self, adapter_id: str) -> int:
        """Evict an adapter (the reference's LRU eviction of a GPU slot, pool.py:91-99): its slot
        joins the free list of its rank.  Returns the slot."""
        if adapter_id not in self.by_id:
            raise KeyError(f"adapter {adapter_id!r} is not resident")
        slot = self.by_id.pop(adapter_id)
        info = self.slots[slot]
        info.adapter_id = ""
        self._free.setdefault(info.rank, []).append(slot)
        return slot

    def load_from_host(self, slot: int, weights, stream: torch.cuda.Stream | None = None) -> None:
        """Make an adapter resident from host memory (the reference's load_from_host fetch,
        pool.py:119-124): weights[(layer, proj)] = (lora_A [r, h_in], lora_B [h_out, r]) bf16 CPU
        tensors (pinned for asynchronous copies); each pair is copied to the device and packed."""
        st = stream or torch.cuda.current_stream(self.device)
        with torch.cuda.stream(st):
            for (layer, proj), (a, b) in weights.items():
                self.load(slot, layer, proj, a.to(self.device, non_blocking=True),
                          b.to(self.device, non_blocking=True), st)

    def migrate_from_peer(self, adapter_id: str, peer: "AdapterSlab", stream: torch.cuda.Stream | None = None) -> int:
        """Copy-on-first-use of a peer-owned adapter (the reference's commit_migration,
        pool.py:134-162: the target becomes a holder): a local slot of the same rank, filled by one
        copy-engine transfer of the peer slot's bytes over NVLink (slots of one model share their
        internal layout, so the bytes move verbatim).  Returns the local slot."""
        ps = peer.slots[peer.by_id[adapter_id]]
        slot = self.allocate(adapter_id, ps.rank)
        dst = self.slots[slot]
        st = stream or torch.cuda.current_stream(self.device)
        native.check(native.lib().lsv_copy_blocks(
            1, (ctypes.c_void_p * 1)(peer.base + ps.offset), (ctypes.c_void_p * 1)(self.base + dst.offset),
            (ctypes.c_size_t * 1)(ps.nbytes), st.cuda_stream))
        return slot

    def a_offset(self, slot: int, layer: int, proj: int) -> int:
        """Offset of proj's first A row inside its group tile (rows repeat every group*rank rows)."""
        return int(self._a_off_rows[slot][layer, proj])

    def layer_block(self, slot: int, layer: int) -> tuple[int, int]:
        """(offset, bytes) of one layer of a slot: every group A tile and B tile of that layer,
        contiguous (what a remote fetch moves for the layer)."""
        info = self.slots[slot]
        per_layer = self.model.adapter_bytes(info.rank) // self.model.layers
        return int(self._g_off_rows[slot][layer, 0]), per_layer

    def a_group_offset(self, slot: int, layer: int, proj: int) -> int:
        return int(self._g_off_rows[slot][layer, self._member[proj][0]])

    def b_offset(self, slot: int, layer: int, proj: int) -> int:
        return int(self._b_off_rows[slot][layer, proj])

    # -- weights -----------------------------------------------------------------------
    def load(self, slot: int, layer: int, proj: int, lora_a: torch.Tensor, lora_b: torch.Tensor,
             stream: torch.cuda.Stream | None = None) -> None:
        """Pack PEFT-layout lora_A [r, h_in] / lora_B [h_out, r] (bf16, on this device)."""
        info = self.slots[slot]
        pr = self.model.projections[proj]
        r = info.rank
        if tuple(lora_a.shape) != (r, pr.h_in) or tuple(lora_b.shape) != (pr.h_out, r):
            raise ValueError(f"expected lora_A {(r, pr.h_in)} and lora_B {(pr.h_out, r)}, got "
                             f"{tuple(lora_a.shape)} and {tuple(lora_b.shape)}")
        if lora_a.dtype != torch.bfloat16 or lora_b.dtype != torch.bfloat16:
            raise ValueError("lora weights must be bfloat16")
        lora_a = lora_a.contiguous()
        lora_b = lora_b.contiguous()
        st = stream or torch.cuda.current_stream(self.device)
        _, idx, nproj = self._member[proj]
        lib = native.lib()
        native.check(lib.lsv_pack_adapter_group(lora_a.data_ptr(), nproj, idx, r, pr.h_in,
                                                self.base + self.a_group_offset(slot, layer, proj), st.cuda_stream))
        native.check(lib.lsv_pack_adapter(None, lora_b.data_ptr(), r, pr.h_in, pr.h_out, None,
                                          self.base + self.b_offset(slot, layer, proj), st.cuda_stream))

    def read(self, slot: int, layer: int, proj: int) -> tuple[torch.Tensor, torch.Tensor]:
        """Unpack a resident adapter back to PEFT layout (tests, migration checks)."""
        info = self.slots[slot]
        pr = self.model.projections[proj]
        a = torch.empty((info.rank, pr.h_in), dtype=torch.bfloat16, device=self.device)
        b = torch.empty((pr.h_out, info.rank), dtype=torch.bfloat16, device=self.device)
        st = torch.cuda.current_stream(self.device).cuda_stream
        _, idx, nproj = self._member[proj]
        lib = native.lib()
        native.check(lib.lsv_unpack_adapter_group(self.base + self.a_group_offset(slot, layer, proj), nproj, idx,
                                                  info.rank, pr.h_in, a.data_ptr(), st))
        native.check(lib.lsv_unpack_adapter(None, self.base + self.b_offset(slot, layer, proj), info.rank, pr.h_in,
                                            pr.h_out, None, b.data_ptr(), st))
        return a, b

    def fill_random(self, slot: int, seed: int, layers: range | None = None) -> None:
        """Random-init adapter weights on the device: A ~ N(0, 1/h_in), B ~ N(0, 1/r)
        (B non-zero so the delta is not trivially 0).  Deterministic per seed."""
        info = self.slots[slot]
        gen = torch.Generator(device=self.device)
        gen.manual_seed(seed)
        for layer in (layers if layers is not None else range(self.model.layers)):
            for p, pr in enumerate(self.model.projections):
                a = (torch.randn((info.rank, pr.h_in), generator=gen, device=self.device)
                     * (1.0 / math.sqrt(pr.h_in))).to(torch.bfloat16)
                b = (torch.randn((pr.h_out, info.rank), generator=gen, device=self.device)
                     * (1.0 / math.sqrt(info.rank))).to(torch.bfloat16)
                self.load(slot, layer, p, a, b)

    # -- NVLink peers (the reference's remote holder, pool.py:101-132) -------------------
    def ipc_handle(self) -> bytes:
        """64-byte CUDA IPC handle of the slab allocation, for peers to map it with ``open_peer``."""
        buf = (ctypes.c_char * 64)()
        native.check(native.lib().lsv_ipc_get_handle(self.base, ctypes.addressof(buf)))
        return bytes(buf)

    def __del__(self):
        try:
            if getattr(self, "_owned", False) and self.base:
                native.lib().lsv_slab_free(self.base)
                self.base = 0
            else:
                self.close_peer()
        except Exception:
            pass

    @classmethod
    def open_peer(cls, model: ModelShape, handle, roster: list[tuple[str, int]], device) -> "AdapterSlab":
        """Map a peer process's slab into this GPU's address space (CUDA IPC opened in this device's
        context, peer access enabled) so kernels here read it over NVLink.  ``roster`` is the (id,
        rank) allocation order the owner used, replayed to rebuild the slot offsets; no data moves."""
        device = torch.device(device)
        buf = (ctypes.c_char * 64).from_buffer_copy(handle)
        ptr = ctypes.c_void_p()
        native.check(native.lib().lsv_ipc_open_handle(ctypes.addressof(buf), device.index, ctypes.byref(ptr)))
        size = sum(model.adapter_bytes(r) + cls.ALIGN for _, r in roster) + cls.ALIGN
        view = cls(model, size, device, _peer_base=ptr.value)
        view._ipc_base = ptr.value
        for aid, rank in roster:
            view.allocate(aid, rank)
        return view

    def close_peer(self) -> None:
        if getattr(self, "_ipc_base", None):
            native.check(native.lib().lsv_ipc_close_handle(self._ipc_base))
            self._ipc_base = None

    # -- pointer tables ----------------------------------------------------------------
    def _offset_tables(self) -> tuple[np.ndarray, np.ndarray]:
        """Per-slot offset rows stacked into [slots, L, groups] / [slots, L, projections] (cached)."""
        n = len(self.slots)
        if getattr(self, "_tables_n", -1) != n:
            L = self.model.layers
            self._g_tab = (np.stack(self._g_off_rows) if n else
                           np.zeros((0, L, len(self.model.groups())), dtype=np.int64))
            self._b_tab = (np.stack(self._b_off_rows) if n else
                           np.zeros((0, L, len(self.model.projections)), dtype=np.int64))
            self._tables_n = n
        return self._g_tab, self._b_tab

    def pointer_tables(self, seg_slots: np.ndarray, peer_slabs: dict[int, "AdapterSlab"] | None = None,
                       seg_owner: np.ndarray | None = None, as_numpy: bool = False):
        """Device int64 tables for the segments: group A tiles [layers*groups, S] (model.groups())
        and B tiles [layers*projections, S].

        ``seg_owner[s]`` (optional) names the GPU whose slab holds segment s; entries other than
        this slab's device resolve through ``peer_slabs`` to NVLink peer addresses."""
        L, P, G = self.model.layers, len(self.model.projections), len(self.model.groups())
        slots = np.asarray(seg_slots, dtype=np.int64)
        S = len(slots)
        g_all, b_all = self._offset_tables()
        a = g_all[slots].reshape(S, L * G).T + self.base        # [L*G, S]
        b = b_all[slots].reshape(S, L * P).T + self.base
        if seg_owner is not None and peer_slabs is not None:
            for s in range(S):     # segments whose adapter lives in a peer GPU's slab (its own slots)
                owner = int(seg_owner[s])
                if owner in peer_slabs and peer_slabs[owner] is not self:
                    peer = peer_slabs[owner]
                    pg, pb_ = peer._offset_tables()
                    a[:, s] = pg[slots[s]].reshape(-1) + peer.base
                    b[:, s] = pb_[slots[s]].reshape(-1) + peer.base
        a = np.ascontiguousarray(a)
        b = np.ascontiguousarray(b)
        if as_numpy:
            return a, b
        return (torch.from_numpy(a).to(self.device, non_blocking=False),
                torch.from_numpy(b).to(self.device, non_blocking=False))
