"""Measure the B200 LoRA-delta cost of co-batched prefill and decode batches (Llama-2-7B, 32
layers x 7 projections, every request its own segment, as the reference prices them) and fit
    t = t0 + k_tok * sum(lengths) + k_rank * sum(ranks)
per regime by least squares: the path is HBM-bound and its bytes are X*sum(n) + W*sum(r)
(SURVEY 8d).  Writes tests/golden/b200_delta_cost.json (samples + fits), which
costmodel.FittedCost and tools/measured_op_points.py read.  Run on a GPU box:
    python tools/measure_cost_fit.py [--out gpurun_out/b200_delta_cost.json]
"""
import argparse
import json
import random
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2511_22880_b200 import costmodel, shapes  # noqa: E402
from paper_2511_22880_b200.lora import LoraDeltaEngine  # noqa: E402
from paper_2511_22880_b200.slab import AdapterSlab  # noqa: E402

RANKS = (8, 16, 32, 64, 128)


def fit(rows, with_tok=True):
    """Least squares on relative residuals (rows weighted by 1/t: the fit is judged per sample as
    |pred - t| / t); decode (one token per request) fits without the token term, which is
    collinear with sum(ranks) there and carries no bytes of its own worth resolving."""
    a = np.array([[1.0, r["sum_len"] if with_tok else 0.0, r["sum_rank"]] for r in rows])
    t = np.array([r["seconds"] for r in rows])
    cols = [0, 1, 2] if with_tok else [0, 2]
    w = 1.0 / t
    coef_sub, *_ = np.linalg.lstsq(a[:, cols] * w[:, None], t * w, rcond=None)
    coef = np.zeros(3)
    coef[cols] = coef_sub
    pred = a @ coef
    return {"t0_s": float(coef[0]), "k_tok_s": float(coef[1]), "k_rank_s": float(coef[2]),
            "max_rel_resid": float(np.max(np.abs(pred - t) / t))}


def refit(path):
    """Recompute the fits of an existing sample file (no GPU)."""
    d = json.loads(Path(path).read_text())
    d["prefill_fit"] = fit(d["prefill_samples"])
    d["decode_fit"] = fit(d["decode_samples"], with_tok=False)
    return d


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=str(ROOT / "tests" / "golden" / "b200_delta_cost.json"))
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    model = shapes.LLAMA2_7B
    slab = AdapterSlab(model, AdapterSlab.capacity_for(model, RANKS), dev)
    for r in RANKS:
        slab.fill_random(slab.allocate(f"r{r}", r), seed=r)
    measured = costmodel.MeasuredCost(LoraDeltaEngine(slab), reps=3)
    rng = random.Random(0)
    prefill, decode = [], []
    for _ in range(36):                     # prefill: 1-16 requests of 16-1024 tokens (<= 8192)
        n = rng.randint(1, 16)
        lens = [rng.choice((16, 64, 128, 256, 512, 1024)) for _ in range(n)]
        while sum(lens) > 8192:
            lens.pop()
        ranks = [rng.choice(RANKS) for _ in lens]
        prefill.append({"lengths": lens, "ranks": ranks, "sum_len": sum(lens), "sum_rank": sum(ranks),
                        "seconds": measured._measure(lens, ranks)})
    for _ in range(24):                     # decode: 1-128 requests, one token each
        n = rng.choice((1, 2, 4, 8, 16, 32, 64, 128))
        ranks = [rng.choice(RANKS) for _ in range(n)]
        decode.append({"lengths": [1] * n, "ranks": ranks, "sum_len": n, "sum_rank": sum(ranks),
                       "seconds": measured._measure([1] * n, ranks)})
    out = {"model": model.name, "device": torch.cuda.get_device_name(dev),
           "form": "t = t0 + k_tok * sum(lengths) + k_rank * sum(ranks)  (LoRA delta only, every request its own segment)",
           "prefill_fit": fit(prefill), "decode_fit": fit(decode, with_tok=False), "prefill_samples": prefill,
           "decode_samples": decode}
    path = Path(args.out)
    path.parent.mkdir(parents=True, exist_ok=True)
    path.write_text(json.dumps(out, indent=1))
    print(json.dumps({k: out[k] for k in ("prefill_fit", "decode_fit")}))


if __name__ == "__main__":
    main()
