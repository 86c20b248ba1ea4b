"""Seeded synthetic workloads for the BASELINE.json configurations.

Inputs are synthetic by necessity (no network for checkpoints or datasets): random-init
adapters (A ~ N(0, 1/h_in), B ~ N(0, 1/r), seed 1000 + adapter index) and N(0, 1)
activations; rosters follow the reference's power-law apportioning
(traces.assign_power_law_counts, traces.py:94-122); token -> adapter assignment is a uniform
draw per token from random.Random(seed).
"""

from __future__ import annotations

import random
from dataclasses import dataclass

import numpy as np

from . import shapes, traces
from .segments import Segments, index_requests, index_tokens


@dataclass
class Workload:
    name: str
    model: shapes.ModelShape
    ranks: list[int]          # rank of each adapter slot
    adapter_ids: list[str]
    segments: Segments
    description: str


def c1_qproj(seed: int = 0) -> Workload:
    """Config 1: Llama-7B q_proj (4096x4096), 4 adapters r=8/16/64/128, 256 tokens (4 x 64)."""
    ranks = [8, 16, 64, 128]
    seg = index_requests([0, 1, 2, 3], [64, 64, 64, 64], ranks)
    return Workload("c1_qproj", shapes.LLAMA7B_QPROJ, ranks, [f"adapter-r{r}-000" for r in ranks], seg,
                    "llama-7b q_proj 4096x4096, 4 adapters r=8/16/64/128, 4x64 tokens")


def c2_llama2_7b(n_tokens: int = 4096, n_adapters: int = 100, seed: int = 0) -> Workload:
    """Config 2: Llama-2-7B all projections, 100 power-law adapters r=8..128, 4096-token batch."""
    roster = traces.roster(n_adapters)
    ranks = [a.rank for a in roster]
    rng = random.Random(seed)
    tok = [rng.randrange(n_adapters) for _ in range(n_tokens)]
    seg = index_tokens(np.asarray(tok), ranks)
    counts = traces.assign_power_law_counts(n_adapters, traces.DEFAULT_RANKS, 1.0)
    return Workload("c2_llama2_7b", shapes.LLAMA2_7B, ranks, [a.id for a in roster], seg,
                    f"llama-2-7b 32 layers x 7 proj, {n_adapters} adapters {counts}, {n_tokens} tokens")


def decode_llama2_7b(n_requests: int = 128, n_adapters: int = 100, seed: int = 0) -> Workload:
    """Decode step (the reference's decode_iter_time regime, costmodel.py:108-123): C2's roster and
    shapes, ``n_requests`` requests each decoding one token (one token per request, so segments of
    a few tokens: the SIMT tier)."""
    roster = traces.roster(n_adapters)
    ranks = [a.rank for a in roster]
    rng = random.Random(seed)
    tok = [rng.randrange(n_adapters) for _ in range(n_requests)]
    seg = index_tokens(np.asarray(tok), ranks)
    return Workload("decode_llama2_7b", shapes.LLAMA2_7B, ranks, [a.id for a in roster], seg,
                    f"llama-2-7b 32 layers x 7 proj decode step: {n_requests} requests x 1 token over "
                    f"{n_adapters} adapters ({seg.num_segments} active)")


WORKLOADS = {"c1": c1_qproj, "c2": c2_llama2_7b, "decode": decode_llama2_7b}


# ---- data-parallel serving across GPUs (configs 3/4): placement + routing decide each GPU's batch
# Operating points of one server per rank under the SLO (the reference's profile at SLO 10 s,
# TP1 — SURVEY §6; `lorasim profile --slo 10`).
DEFAULT_OP_POINTS = {8: 4800.0, 16: 3800.0, 32: 3280.0, 64: 2600.0, 128: 1560.0}


@dataclass
class ServerWorkload(Workload):
    server: int = 0
    resident: list[str] | None = None      # adapter ids with phi > 0 on this GPU (its slab)
    placement: object = None               # the Assignment all GPUs computed
    routed_tokens: int = 0                 # tokens routed to this GPU in the trace window


def dp_workloads(num_servers: int, model: shapes.ModelShape = shapes.LLAMA2_7B, n_adapters: int = 100,
                 tokens_per_gpu: int = 4096, prompt_len: int = 41, popularity: str = "power_law",
                 seed: int = 0) -> list[ServerWorkload]:
    """Each GPU is one reference server.  A rank-skewed trace (traces.generate_trace) feeds the
    demand history of its first window; LoRAServe placement (placement.place_from_demand) decides
    every GPU's resident adapters; phi-weighted routing (routing.route, seeded "seed:route" as in
    simengine.py:294) sends each request to a GPU, which forms its batch FIFO up to
    ``tokens_per_gpu`` tokens.  Deterministic: every rank computes the same thing."""
    from . import demand, domain, placement, routing
    cfg = traces.TraceConfig(duration_seconds=120.0, target_rps=max(1.0, 6.0 * num_servers * tokens_per_gpu / prompt_len / 60.0),
                             arrival="poisson", popularity=popularity, adapters_per_rank=None,
                             total_adapters=n_adapters, count_skew_alpha=1.0,
                             lengths=traces.LengthModel(kind="fixed", prompt=prompt_len, output=1), seed=seed)
    roster = traces.trace_adapters(cfg)
    reqs = traces.generate_trace(cfg)
    hist = demand.TpsHistory(60.0, [a.id for a in roster])
    for r in reqs:
        if r.arrival_time >= 60.0:
            break
        hist.record_request(r.adapter, r.total_tokens, r.arrival_time)
    hist.advance_to(60.0)
    asg = placement.place_from_demand(list(range(num_servers)), roster, hist.demand_estimate(),
                                      domain.OperatingPointTable(DEFAULT_OP_POINTS))
    table = routing.build_routing_table(asg)
    rng = random.Random(f"{seed}:route")
    per_gpu: list[list] = [[] for _ in range(num_servers)]
    fill = [0] * num_servers
    routed = [0] * num_servers
    for r in reqs:
        if r.arrival_time < 60.0:
            continue
        srv = routing.route(r, table, rng)
        routed[srv] += r.prompt_length
        if fill[srv] + r.prompt_length <= tokens_per_gpu:
            per_gpu[srv].append(r)
            fill[srv] += r.prompt_length
        if all(f + prompt_len > tokens_per_gpu for f in fill):
            break
    rank_of = {a.id: a.rank for a in roster}
    out = []
    for srv in range(num_servers):
        resident = [a.id for a in roster if asg.per_server and any(aid == a.id and phi > 0 for aid, phi in asg.per_server[srv])]
        slot_of = {aid: i for i, aid in enumerate(resident)}
        batch = per_gpu[srv]
        if not batch:
            raise RuntimeError(f"GPU {srv} received no requests; lengthen the trace")
        seg = index_requests([slot_of[r.adapter] for r in batch], [r.prompt_length for r in batch],
                             [rank_of[r.adapter] for r in batch])
        out.append(ServerWorkload(
            name=f"dp{num_servers}_gpu{srv}", model=model, ranks=[rank_of[a] for a in resident],
            adapter_ids=resident, segments=seg,
            description=(f"{model.name} {model.layers} layers x {len(model.projections)} proj; LoRAServe placement + "
                         f"phi routing over {num_servers} GPUs; {n_adapters} adapters, {popularity} rank popularity; "
                         f"{tokens_per_gpu} tokens/GPU from {prompt_len}-token requests"),
            server=srv, resident=resident, placement=asg, routed_tokens=routed[srv]))
    return out


def remote_workload(num_gpus: int, rank: int, remote_frac: float = 0.3, n_tokens: int = 4096,
                    n_adapters: int = 100, seed: int = 0):
    """Config 4: the C2 roster/model on every GPU; adapter i is owned by GPU i % num_gpus.  The GPU's
    4096-token batch draws ``remote_frac`` of its tokens from adapters owned by other GPUs (read
    in-kernel over NVLink) and the rest from its own.  Returns (workload, seg_owner)."""
    roster = traces.roster(n_adapters)
    ranks = [a.rank for a in roster]
    own = [i for i in range(n_adapters) if i % num_gpus == rank]
    other = [i for i in range(n_adapters) if i % num_gpus != rank] or own
    rng = random.Random(f"{seed}:remote:{rank}")
    tok = [(rng.choice(other) if rng.random() < remote_frac else rng.choice(own)) for _ in range(n_tokens)]
    seg = index_tokens(np.asarray(tok), ranks)
    owner = np.asarray([int(s) % num_gpus for s in seg.seg_slot], dtype=np.int32)
    remote_tokens = int(np.sum(seg.lengths()[owner != rank]))
    wl = Workload(f"remote{num_gpus}_gpu{rank}", shapes.LLAMA2_7B, ranks, [a.id for a in roster], seg,
                  f"llama-2-7b 32 layers x 7 proj, {n_adapters} adapters owned round-robin by {num_gpus} GPUs; "
                  f"{n_tokens} tokens/GPU, {remote_tokens / n_tokens:.0%} on peer-owned adapters (NVLink loads)")
    return wl, owner
