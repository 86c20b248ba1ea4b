"""Model projection shapes for the benchmark configurations (BASELINE.json ``configs``).

Each projection a LoRA adapter attaches to is (name, h_in, h_out).  Llama-2 7B/13B use MHA
(k/v out = hidden); Llama-3 70B uses GQA with 8 KV heads of 128 (k/v out = 1024).
"""

from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class Projection:
    name: str
    h_in: int
    h_out: int


# Which activation each projection reads: q/k/v share the attention input, gate/up the MLP input.
INPUT_GROUPS = {"q_proj": "attn_in", "k_proj": "attn_in", "v_proj": "attn_in", "o_proj": "attn_out",
                "gate_proj": "mlp_in", "up_proj": "mlp_in", "down_proj": "mlp_mid"}


def input_group(proj_name: str) -> str:
    return INPUT_GROUPS.get(proj_name, proj_name)


@dataclass(frozen=True)
class ModelShape:
    name: str
    layers: int
    projections: tuple[Projection, ...]

    def groups(self) -> list[tuple[str, tuple[int, ...]]]:
        """Input groups: runs of consecutive projections that read the same activation (same h_in).
        Their A matrices share one slab tile and one shrink (include/lsv.h, lsv_plan_build_group)."""
        out: list[tuple[str, list[int]]] = []
        for i, p in enumerate(self.projections):
            g = input_group(p.name)
            if out and out[-1][0] == g and self.projections[out[-1][1][0]].h_in == p.h_in and len(out[-1][1]) < 4:
                out[-1][1].append(i)
            else:
                out.append((g, [i]))
        return [(g, tuple(m)) for g, m in out]

    def shapes(self) -> list[tuple[int, int]]:
        """Distinct (h_in, h_out) pairs, in first-use order (one plan each)."""
        seen: list[tuple[int, int]] = []
        for p in self.projections:
            if (p.h_in, p.h_out) not in seen:
                seen.append((p.h_in, p.h_out))
        return seen

    def rank_units_bytes(self) -> int:
        """bf16 bytes of one rank unit of an adapter across every layer/projection."""
        return self.layers * sum(2 * (p.h_in + p.h_out) for p in self.projections)

    def adapter_bytes(self, rank: int) -> int:
        """HBM bytes of one resident adapter in the slab format (B rows padded to 16, include/lsv.h)."""
        kp = kpad(rank)
        return self.layers * sum(2 * (rank * p.h_in + kp * p.h_out) for p in self.projections)


def kpad(rank: int) -> int:
    """Rank padded to the 16-wide tensor-core K step (lsv_common.cuh kpad)."""
    return max(16, (rank + 15) // 16 * 16)


def _llama(name: str, hidden: int, inter: int, layers: int, kv_out: int | None = None) -> ModelShape:
    kv = hidden if kv_out is None else kv_out
    return ModelShape(name, layers, (
        Projection("q_proj", hidden, hidden),
        Projection("k_proj", hidden, kv),
        Projection("v_proj", hidden, kv),
        Projection("o_proj", hidden, hidden),
        Projection("gate_proj", hidden, inter),
        Projection("up_proj", hidden, inter),
        Projection("down_proj", inter, hidden),
    ))


LLAMA2_7B = _llama("llama-2-7b", 4096, 11008, 32)
LLAMA2_13B = _llama("llama-2-13b", 5120, 13824, 40)
LLAMA3_70B = _llama("llama-3-70b", 8192, 28672, 80, kv_out=1024)
LLAMA7B_QPROJ = ModelShape("llama-7b-q_proj", 1, (Projection("q_proj", 4096, 4096),))

MODELS = {m.name: m for m in (LLAMA2_7B, LLAMA2_13B, LLAMA3_70B, LLAMA7B_QPROJ)}


def tp_shard(model: ModelShape, tp: int) -> ModelShape:
    """Per-GPU projection shapes under S-LoRA-style tensor parallelism (column-parallel
    q/k/v/gate/up shard h_out, row-parallel o/down shard h_in)."""
    col = {"q_proj", "k_proj", "v_proj", "gate_proj", "up_proj"}
    projs = []
    for p in model.projections:
        if p.name in col:
            if p.h_out % (tp * 128):
                raise ValueError(f"{p.name}: h_out {p.h_out} not divisible into {tp} shards of 128")
            projs.append(Projection(p.name, p.h_in, p.h_out // tp))
        else:
            if p.h_in % (tp * 128):
                raise ValueError(f"{p.name}: h_in {p.h_in} not divisible into {tp} shards of 128")
            projs.append(Projection(p.name, p.h_in // tp, p.h_out))
    return ModelShape(f"{model.name}-tp{tp}", model.layers, tuple(projs))
