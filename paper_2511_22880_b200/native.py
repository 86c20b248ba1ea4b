"""ctypes binding of liblsv (include/lsv.h).

Nonzero returns become the exception types the reference raises at the boundary this path
replaces: ValueError for bad shapes / metadata / workspace (costmodel.py:95-103 raises
ValueError for an empty batch, length mismatch or budget overflow) and RuntimeError for CUDA
failures.  There is no fallback: if liblsv.so is missing the import of this module's
functions raises, so a GPU run can never silently take a CPU or PyTorch path.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

LIB_NAME = "liblsv.so"
# LSV_LIB_PATH: development override (A/B timing of two builds of the same library on one box)
LIB_PATH = Path(os.environ.get("LSV_LIB_PATH") or Path(__file__).resolve().parent / LIB_NAME)

LSV_OK, LSV_EINVAL, LSV_ECUDA, LSV_EUNSUPPORTED, LSV_EWORKSPACE = 0, 1, 2, 3, 4
LSV_DTYPE_BF16 = 0
ABI_VERSION = 3
TIER_AUTO, TIER_SIMT, TIER_TC = 0, 1, 2
FWD_SERIAL = 1
SEG_NOSHRINK = 4    # per-segment plan flag: m-tiles kept, no shrink work (balanced TP shard with no rows)
TP_ROUND_ROBIN = 0x100   # lsv_lora_shrink_tp_scatter: balanced round-robin 8-row-group shards
SEG_SKIP = 2        # per-segment plan flag: token range kept, no work in this plan
SEG_REMOTE = 1      # per-segment plan flag: adapter resident in an NVLink peer's slab
def PLAN_SMS(n: int) -> int:   # noqa: N802  plan flag: at most n CTAs per kernel
    return (n & 0xff) << 16


PLAN_TILE_ALIGNED = 0x200   # plan flag: tile-aligned v images for lsv_lora_fused_linear
PLAN_V_BF16 = 0x100   # plan flag: single bf16 v image on the tensor-core tier (default: hi/lo pair)

# every symbol include/lsv.h declares (tests/test_native_abi.py checks the library exports them)
EXPORTED_SYMBOLS = (
    "lsv_version", "lsv_last_error", "lsv_adapter_a_bytes", "lsv_adapter_b_bytes",
    "lsv_pack_adapter", "lsv_unpack_adapter", "lsv_plan_size", "lsv_plan_build",
    "lsv_plan_summary", "lsv_lora_apply", "lsv_lora_shrink", "lsv_lora_expand",
    "lsv_enable_peer", "lsv_num_sms", "lsv_ipc_get_handle", "lsv_ipc_open_handle", "lsv_ipc_close_handle",
    "lsv_slab_alloc", "lsv_slab_free", "lsv_vimg_assemble", "lsv_plan_vimg_region",
    "lsv_adapter_a_group_bytes", "lsv_pack_adapter_group", "lsv_unpack_adapter_group",
    "lsv_plan_size_group", "lsv_plan_build_group", "lsv_lora_expand_proj", "lsv_lora_expand_group",
    "lsv_lora_forward", "lsv_lora_forward_ex", "lsv_lora_forward_workspace", "lsv_copy_blocks",
    "lsv_lora_shrink_tp_scatter", "lsv_lora_expand_group_tp",
    "lsv_lora_shrink_tp_partials", "lsv_lora_expand_group_tp_sum", "lsv_debug_set_trace",
    "lsv_lora_fused_linear", "lsv_plan_size_group_ex", "lsv_plan_build_group_ex", "lsv_build_info",
)

_lib = None

_vp, _i32, _i64, _sz = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t
_SIGNATURES = {
    "lsv_version": (ctypes.c_int, []),
    "lsv_last_error": (ctypes.c_char_p, []),
    "lsv_num_sms": (ctypes.c_int, []),
    "lsv_build_info": (ctypes.c_int, []),
    "lsv_debug_set_trace": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32]),
    "lsv_adapter_a_bytes": (_sz, [_i32, _i32]),
    "lsv_adapter_b_bytes": (_sz, [_i32, _i32]),
    "lsv_pack_adapter": (ctypes.c_int, [_vp, _vp, _i32, _i32, _i32, _vp, _vp, _vp]),
    "lsv_unpack_adapter": (ctypes.c_int, [_vp, _vp, _i32, _i32, _i32, _vp, _vp, _vp]),
    "lsv_plan_size": (ctypes.c_int, [_i32, _vp, _vp, _i32, _i32, _i32, ctypes.POINTER(_sz),
                                     ctypes.POINTER(_sz)]),
    "lsv_plan_build": (ctypes.c_int, [_i32, _vp, _vp, _i32, _i32, _i32, _vp, _sz]),
    "lsv_plan_summary": (ctypes.c_int, [_vp, _vp]),
    "lsv_lora_apply": (ctypes.c_int, [_vp, _i64, _vp, _i64, _i32, _i32, _i32, _i32, _vp, _vp, _vp,
                                      _vp, _vp, _sz, _vp]),
    "lsv_lora_shrink": (ctypes.c_int, [_vp, _i64, _i32, _i32, _vp, _vp, _vp, _vp, _sz, _vp]),
    "lsv_lora_expand": (ctypes.c_int, [_vp, _i64, _i32, _i32, _vp, _vp, _vp, _vp, _sz, _vp]),
    "lsv_enable_peer": (ctypes.c_int, [_i32, _i32]),
    "lsv_ipc_get_handle": (ctypes.c_int, [_vp, _vp]),
    "lsv_slab_alloc": (ctypes.c_int, [_sz, _i32, ctypes.POINTER(_vp)]),
    "lsv_slab_free": (ctypes.c_int, [_vp]),
    "lsv_vimg_assemble": (ctypes.c_int, [_vp, _sz, _i32, _vp, _vp, _vp, _vp, _vp, _vp]),
    "lsv_plan_vimg_region": (ctypes.c_int, [_vp, ctypes.POINTER(_sz), ctypes.POINTER(_sz)]),
    "lsv_ipc_open_handle": (ctypes.c_int, [_vp, _i32, ctypes.POINTER(_vp)]),
    "lsv_ipc_close_handle": (ctypes.c_int, [_vp]),
    "lsv_adapter_a_group_bytes": (_sz, [_i32, _i32, _i32]),
    "lsv_pack_adapter_group": (ctypes.c_int, [_vp, _i32, _i32, _i32, _i32, _vp, _vp]),
    "lsv_unpack_adapter_group": (ctypes.c_int, [_vp, _i32, _i32, _i32, _i32, _vp, _vp]),
    "lsv_plan_size_group": (ctypes.c_int, [_i32, _vp, _vp, _i32, _i32, _vp, _i32, ctypes.POINTER(_sz),
                                           ctypes.POINTER(_sz)]),
    "lsv_plan_build_group": (ctypes.c_int, [_i32, _vp, _vp, _i32, _i32, _vp, _i32, _vp, _sz]),
    "lsv_lora_expand_proj": (ctypes.c_int, [_vp, _i64, _i32, _i32, _i32, _vp, _vp, _vp, _vp, _sz, _vp]),
    "lsv_lora_expand_group": (ctypes.c_int, [_vp, _vp, _i32, _vp, _vp, _vp, _vp, _sz, _vp]),
    "lsv_lora_forward": (ctypes.c_int, [_i32, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i32, _vp, _sz, _vp]),
    "lsv_lora_forward_ex": (ctypes.c_int, [_i32, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i32, _vp, _sz, _i32,
                                           _vp]),
    "lsv_lora_forward_workspace": (_sz, [_i32, _i32, _vp]),
    "lsv_copy_blocks": (ctypes.c_int, [_i32, _vp, _vp, _vp, _vp]),
    "lsv_lora_shrink_tp_scatter": (ctypes.c_int, [_vp, _i64, _i32, _i32, _vp, _vp, _vp, _vp, _sz, _i32, _i32,
                                                  _vp, _vp, _vp, _vp, _vp]),
    "lsv_lora_expand_group_tp": (ctypes.c_int, [_vp, _vp, _i32, _vp, _vp, _vp, _vp, _vp, _i32, _vp]),
    "lsv_lora_shrink_tp_partials": (ctypes.c_int, [_vp, _i64, _i32, _i32, _vp, _vp, _vp, _vp, _sz, _i32, _i32,
                                                   _vp, _vp, _vp]),
    "lsv_lora_expand_group_tp_sum": (ctypes.c_int, [_vp, _vp, _i32, _vp, _vp, _vp, _vp, _sz, _vp, _i32, _vp, _vp]),
    "lsv_plan_size_group_ex": (ctypes.c_int, [_i32, _vp, _vp, _vp, _i32, _i32, _vp, _i32, ctypes.POINTER(_sz),
                                              ctypes.POINTER(_sz)]),
    "lsv_plan_build_group_ex": (ctypes.c_int, [_i32, _vp, _vp, _vp, _i32, _i32, _vp, _i32, _vp, _sz]),
    "lsv_lora_fused_linear": (ctypes.c_int, [_vp, _i64, _i32, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _sz,
                                             _vp]),
}


class LsvError(RuntimeError):
    """CUDA-side failure inside liblsv."""


def load():
    """Load liblsv.so (built in-tree by paper_2511_22880_b200.build); raise if absent."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                "(there is no CPU fallback for the LoRA delta path)")
        lib = ctypes.CDLL(str(LIB_PATH))
        for name, (res, args) in _SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.lsv_version() != ABI_VERSION:
            raise RuntimeError(f"liblsv ABI version {lib.lsv_version()} != {ABI_VERSION}")
        _lib = lib
    return _lib


def check(rc: int) -> None:
    if rc == LSV_OK:
        return
    msg = load().lsv_last_error().decode(errors="replace")
    if rc in (LSV_EINVAL, LSV_EWORKSPACE):
        raise ValueError(msg)
    raise LsvError(msg)


def lib():
    return load()
