"""Per-GPU co-batch formation: the caller of the delta path (mirror of simengine.schedule_server).

The reference forms a server's next prefill batch FIFO under the token budget, passing over
requests still waiting on an adapter fetch (their place is kept), ejecting requests whose TTFT
has overshot the timeout, stopping at the budget, and otherwise running one decode iteration
over every in-flight decode (/root/reference/pkg/src/lorasim/simengine.py:96-152).  The batch it
returns is what ``costmodel.prefill_time`` prices; here it is what the GPU executes:
``to_segments`` indexes it (segments.index_requests) into the adapter-contiguous segments the
liblsv plan consumes.
"""

from __future__ import annotations

from collections import deque
from dataclasses import dataclass, field
from typing import Callable, Mapping

from .costmodel import CostParams, decode_iter_time, prefill_time
from .segments import Segments, index_requests


@dataclass
class QueuedRequest:
    """The fields of the reference's RequestState (simengine.py:38-57) the batch former reads."""

    request_id: str
    adapter: str
    rank: int
    prompt_length: int
    arrival_time: float
    ready: bool = True
    solo_prefill_s: float = 0.0
    context: int = 0


@dataclass
class BatchDecision:
    kind: str                      # "prefill" | "decode" | "idle"
    batch: list[QueuedRequest]
    duration: float
    ejected: list[QueuedRequest] = field(default_factory=list)


@dataclass
class ServerQueue:
    """Mutable per-GPU queues (the parts of simengine.ServerSim the former touches)."""

    wait_queue: deque = field(default_factory=deque)
    running_decodes: list = field(default_factory=list)
    committed_prefill_s: float = 0.0


def schedule_server(server: ServerQueue, now: float, params: CostParams, timeout_seconds: float,
                    prefill_cost: Callable = prefill_time, decode_cost: Callable = decode_iter_time) -> BatchDecision:
    """Next batch for an idle GPU.  Same policy and bookkeeping as simengine.py:96-152;
    ``prefill_cost``/``decode_cost`` default to the modelled callbacks and can be the measured
    B200 ones (costmodel.MeasuredCost)."""
    ejected: list[QueuedRequest] = []
    batch: list[QueuedRequest] = []
    deferred: list[QueuedRequest] = []
    used = 0
    full = False
    while server.wait_queue:
        rq = server.wait_queue.popleft()
        if now - rq.arrival_time > timeout_seconds:
            server.committed_prefill_s -= rq.solo_prefill_s
            ejected.append(rq)
            continue
        if full or not rq.ready:
            deferred.append(rq)
            continue
        if rq.prompt_length > params.token_budget:
            raise RuntimeError(f"request {rq.request_id!r} prompt of {rq.prompt_length} tokens exceeds the "
                               f"{params.token_budget}-token batch budget")
        if used + rq.prompt_length > params.token_budget:
            deferred.append(rq)
            full = True
            continue
        server.committed_prefill_s -= rq.solo_prefill_s
        batch.append(rq)
        used += rq.prompt_length
    server.wait_queue.extend(deferred)
    if batch:
        return BatchDecision("prefill", batch, prefill_cost([r.prompt_length for r in batch],
                                                            [r.rank for r in batch], params), ejected)
    if server.running_decodes:
        decodes = list(server.running_decodes)
        return BatchDecision("decode", decodes, decode_cost([r.context for r in decodes],
                                                            [r.rank for r in decodes], params), ejected)
    return BatchDecision("idle", [], 0.0, ejected)


def to_segments(batch: list[QueuedRequest], slot_of: Mapping[str, int], decode: bool = False) -> Segments:
    """Index a formed batch (FIFO order) into adapter segments: one token per request for a decode
    step, ``prompt_length`` tokens per request for a prefill."""
    return index_requests([slot_of[r.adapter] for r in batch],
                          [1 if decode else r.prompt_length for r in batch], [r.rank for r in batch])
