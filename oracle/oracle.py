"""CPU oracle for the mixed-rank LoRA delta — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and ``--impl reference``)
may import this module, and only as the checker / the timed CPU baseline.  The product path
(paper_2511_22880_b200) never imports it and fails loudly without its CUDA library.

PARITY UNPINNED BY THE REFERENCE for the delta arithmetic: the reference LoRAServe simulator
(/root/reference/pkg/src/lorasim) has no tensor code (the path exists only as the
cost callback costmodel.prefill_time, costmodel.py:83-105).  ``delta_c`` runs the C restatement
(oracle/lsv_oracle.c, built by oracle/Makefile into oracle/build/); ``delta_f64`` is an
independent float64 numpy restatement used to pin the C oracle (tests/test_oracle.py).

Math (PEFT layouts): for each segment s covering tokens
[seg_indptr[s], seg_indptr[s+1]) with lora_A_s [r, h_in] and lora_B_s [h_out, r]:
    delta[t] = (x[t] @ lora_A_s.T) @ lora_B_s.T
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_LIB_PATH = _HERE / "build" / "liblsv_oracle.so"
_lib = None


def build() -> Path:
    """Compile the C oracle (idempotent)."""
    src = _HERE / "lsv_oracle.c"
    if not _LIB_PATH.exists() or _LIB_PATH.stat().st_mtime < src.stat().st_mtime:
        subprocess.run(["make", "-s", "-C", str(_HERE)], check=True)
    return _LIB_PATH


def _load():
    global _lib
    if _lib is None:
        if not _LIB_PATH.exists():
            build()
        lib = ctypes.CDLL(str(_LIB_PATH))
        lib.lsv_oracle_delta.restype = ctypes.c_int
        lib.lsv_oracle_delta.argtypes = [
            ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
            ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
            ctypes.c_int32,
        ]
        lib.lsv_oracle_threads.restype = ctypes.c_int
        _lib = lib
    return _lib


def cpu_threads() -> int:
    return int(_load().lsv_oracle_threads())


def bf16_bits_to_f32(bits: np.ndarray) -> np.ndarray:
    """Exact widening of bf16 bit patterns (uint16) to float32."""
    return (bits.astype(np.uint32) << 16).view(np.float32)


def f32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even float32 -> bf16 bit patterns (uint16)."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    rounded = (u + 0x7FFF + ((u >> 16) & 1)) >> 16
    return rounded.astype(np.uint16)


def delta_c(x_bits: np.ndarray, seg_indptr, seg_rank, lora_a_bits, lora_b_bits, h_out: int,
            threads: int = 0) -> np.ndarray:
    """fp32 delta [num_tokens, h_out] from the C oracle (rows outside segments are 0)."""
    lib = _load()
    x_bits = np.ascontiguousarray(x_bits, dtype=np.uint16)
    n_tok, h_in = x_bits.shape
    indptr = np.ascontiguousarray(seg_indptr, dtype=np.int32)
    ranks = np.ascontiguousarray(seg_rank, dtype=np.int32)
    S = len(ranks)
    a_arrs = [np.ascontiguousarray(a, dtype=np.uint16) for a in lora_a_bits]
    b_arrs = [np.ascontiguousarray(b, dtype=np.uint16) for b in lora_b_bits]
    for s in range(S):
        assert a_arrs[s].shape == (ranks[s], h_in), (s, a_arrs[s].shape)
        assert b_arrs[s].shape == (h_out, ranks[s]), (s, b_arrs[s].shape)
    a_ptrs = (ctypes.c_void_p * max(S, 1))(*[a.ctypes.data for a in a_arrs])
    b_ptrs = (ctypes.c_void_p * max(S, 1))(*[b.ctypes.data for b in b_arrs])
    delta = np.zeros((n_tok, h_out), dtype=np.float32)
    rc = lib.lsv_oracle_delta(x_bits.ctypes.data, h_in, h_in, h_out, S, indptr.ctypes.data,
                              ranks.ctypes.data, ctypes.cast(a_ptrs, ctypes.c_void_p),
                              ctypes.cast(b_ptrs, ctypes.c_void_p), delta.ctypes.data, threads)
    if rc != 0:
        raise RuntimeError(f"lsv_oracle_delta failed with {rc}")
    return delta


def delta_f64(x_bits, seg_indptr, seg_rank, lora_a_bits, lora_b_bits, h_out: int) -> np.ndarray:
    """Independent float64 numpy restatement (pins the C oracle)."""
    x = bf16_bits_to_f32(np.asarray(x_bits, dtype=np.uint16)).astype(np.float64)
    out = np.zeros((x.shape[0], h_out), dtype=np.float64)
    for s in range(len(seg_rank)):
        t0, t1 = int(seg_indptr[s]), int(seg_indptr[s + 1])
        if t1 <= t0:
            continue
        a = bf16_bits_to_f32(np.asarray(lora_a_bits[s])).astype(np.float64)
        b = bf16_bits_to_f32(np.asarray(lora_b_bits[s])).astype(np.float64)
        out[t0:t1] = (x[t0:t1] @ a.T) @ b.T
    return out


def max_rel_err(got: np.ndarray, ref: np.ndarray) -> float:
    """The north-star error metric: max|got - ref| / max|ref| (norm-relative)."""
    ref = np.asarray(ref, dtype=np.float64)
    denom = float(np.max(np.abs(ref))) if ref.size else 0.0
    if denom == 0.0:
        return float(np.max(np.abs(np.asarray(got, dtype=np.float64)))) if ref.size else 0.0
    return float(np.max(np.abs(np.asarray(got, dtype=np.float64) - ref)) / denom)
