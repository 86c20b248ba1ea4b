"""Generate tests/golden/sgmv_fixtures.npz: golden LoRA deltas from the published SGMV algorithm.

TEST INFRASTRUCTURE.  The reference (LoRAServe) has no tensor code: its delta path is a cost
callback (costmodel.prefill_time, /root/reference/pkg/src/lorasim/costmodel.py:83-105) standing
for the Punica SGMV / S-LoRA kernels the paper runs on,
which are not under /root/reference (no go.mod / Cargo.lock / package.json / submodule).  The
published algorithm is in this image as vLLM 0.22's pure-PyTorch restatement of Punica's SGMV,
``vllm.lora.ops.torch_ops`` (sgmv_shrink: v = scaling * x @ A_i^T per segment; sgmv_expand:
y += v @ B_i^T per segment, ``add_inputs=True``).  vLLM does not travel to the GPU box, so its
outputs are committed here as fixtures.

Each case (tests/_cases.FIXTURE_CASES) regenerates the seeded bf16 inputs exactly as the parity
tests do (tests/_cases.Case / LayerCase), widens them to fp32 (exact), and runs vLLM's
sgmv_shrink -> sgmv_expand in fp32 on the CPU with the real segment metadata
(b_seq_start_loc / seq_len / lora_indices).  The adapters of one call are stacked into vLLM's
[num_loras, max_rank, h_in] / [num_loras, h_out, max_rank] layout, zero-padded past each rank
(exact: the padding adds only zero products); tokens go through in 64-token chunks to bound the
[tokens, rank, h] weight gather of bgmv.  Stored per case (and per projection for the C2 layer):
  rows   sampled tokens (first and last of every segment + 8 seeded random)
  cols   sampled output columns (all, or a prefix plus a stride)
  y      fp32 delta at [rows][cols]
  chk    fp64 [tokens, 3]: per token sum_j y, sum_j y * w_j (w_j = cos(j)), sum_j |y|

Run (in this container): python tests/golden/make_sgmv_fixtures.py
"""

from __future__ import annotations

import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from tests._cases import FIXTURE_CASES, LayerCase, fixture_case, fixture_cols, fixture_rows  # noqa: E402

OUT = Path(__file__).resolve().parent / "sgmv_fixtures.npz"
CHUNK = 64


def checksum_weights(h_out: int) -> np.ndarray:
    return np.cos(np.arange(h_out, dtype=np.float64))


def sgmv_delta(x: torch.Tensor, seg_indptr, seg_rank, a_list, b_list, h_out: int) -> torch.Tensor:
    """fp32 [N, h_out] delta via vLLM's published SGMV restatement (torch_ops), y_in = 0."""
    from vllm.lora.ops.torch_ops import sgmv_expand, sgmv_shrink
    S = len(seg_rank)
    n = int(seg_indptr[-1])
    h_in = x.shape[1]
    max_r = max([int(r) for r in seg_rank] + [1])
    lora_a = torch.zeros(max(S, 1), max_r, h_in, dtype=torch.float32)
    lora_b = torch.zeros(max(S, 1), h_out, max_r, dtype=torch.float32)
    for s in range(S):
        r = int(seg_rank[s])
        lora_a[s, :r] = a_list[s].float()
        lora_b[s, :, :r] = b_list[s].float()
    xf = x[:n].float()
    y = torch.zeros(n, h_out, dtype=torch.float32)
    for c0 in range(0, n, CHUNK):
        c1 = min(n, c0 + CHUNK)
        starts, lens, idx = [], [], []
        for s in range(S):     # the segments' pieces inside this chunk, in token order
            t0, t1 = max(c0, int(seg_indptr[s])), min(c1, int(seg_indptr[s + 1]))
            if t1 > t0:
                starts.append(t0 - c0)
                lens.append(t1 - t0)
                idx.append(s)
        b_seq_start_loc = torch.tensor(starts, dtype=torch.int64)
        seq_len = torch.tensor(lens, dtype=torch.int64)
        lora_idx = torch.tensor(idx, dtype=torch.int64)
        v = torch.zeros(c1 - c0, max_r, dtype=torch.float32)
        sgmv_shrink(xf[c0:c1], lora_a, v, b_seq_start_loc, seq_len, lora_idx, len(idx), max(lens), c1 - c0, 1.0)
        out = y[c0:c1]
        sgmv_expand(v, lora_b, out, b_seq_start_loc, seq_len, lora_idx, len(idx), max(lens), c1 - c0,
                    add_inputs=True)
    return y


def record(store: dict, key: str, y: torch.Tensor, seg, cols_spec) -> None:
    yd = y.double().numpy()
    rows = fixture_rows(seg)
    cols = fixture_cols(y.shape[1], cols_spec)
    w = checksum_weights(y.shape[1])
    store[f"{key}/rows"] = rows
    store[f"{key}/cols"] = cols
    store[f"{key}/y"] = y.numpy()[np.ix_(rows, cols)].astype(np.float32)
    store[f"{key}/chk"] = np.stack([yd.sum(1), yd @ w, np.abs(yd).sum(1)], axis=1)


def main() -> None:
    torch.set_num_threads(max(1, torch.get_num_threads()))
    store: dict[str, np.ndarray] = {}
    meta = {"generator": "vllm.lora.ops.torch_ops sgmv_shrink/sgmv_expand (fp32, CPU)", "cases": {}}
    try:
        import vllm
        meta["vllm_version"] = vllm.__version__
    except Exception:   # pragma: no cover
        meta["vllm_version"] = "unknown"
    for name, spec in FIXTURE_CASES.items():
        t0 = time.time()
        case = fixture_case(name)
        if isinstance(case, LayerCase):
            for p, pr in enumerate(case.model.projections):
                x, a, b = case.proj_inputs(p)
                y = sgmv_delta(x, case.seg.seg_indptr, case.seg.seg_rank, a, b, pr.h_out)
                record(store, f"{name}/{pr.name}", y, case.seg, spec["cols"])
            meta["cases"][name] = {"projections": [pr.name for pr in case.model.projections],
                                   "tokens": case.seg.num_tokens, "segments": case.seg.num_segments}
        else:
            y = sgmv_delta(case.x, case.seg.seg_indptr, case.seg.seg_rank, case.a, case.b, case.h_out)
            record(store, name, y, case.seg, spec["cols"])
            meta["cases"][name] = {"h_in": case.h_in, "h_out": case.h_out, "tokens": case.seg.num_tokens,
                                   "segments": case.seg.num_segments}
        print(f"{name}: {time.time() - t0:.1f} s", flush=True)
    store["meta"] = np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8)
    np.savez_compressed(OUT, **store)
    print(f"wrote {OUT} ({OUT.stat().st_size / 1e6:.2f} MB)")


if __name__ == "__main__":
    main()
