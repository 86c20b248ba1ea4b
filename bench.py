#!/usr/bin/env python
"""Benchmark of the B200 mixed-rank LoRA delta path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c2|c1]

One step = the delta path over one co-batched batch through every layer and projection of
the model (config c2: Llama-2-7B, 32 layers x 7 projections, 100 power-law adapters
r=8..128, 4096 tokens; synthetic inputs, random-init adapters).  ``value`` is whole-job
tokens/s with inputs resident in HBM (CUDA-graph replay, CUDA events, max over ranks);
``e2e`` is the same metric through the public API (host segment indexing + planning, plan
upload, H2D of the batch's input activations from pinned memory, eager kernel launches for
all layers, D2H of the final projection's output).  ``--impl reference`` times the CPU
restatement (oracle/, test infrastructure) on this box's host cores: the reference itself has
no tensor code, so its CPU "implementation" of this path is that restatement.
Under torchrun every rank runs its own full batch (weak scaling; the path has no exchange
step in data-parallel serving — SURVEY §8e).
"""

from __future__ import annotations

import argparse
import gc
import json
import os
import statistics
import subprocess
import sys
import threading
import time
import zlib
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "mixed-rank LoRA tokens/s at 1/2/4/8 B200; % HBM roofline; remote-fetch overhead"
HBM_FALLBACK_GBS = 6650.0


def parse_args(argv=None):
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--config", choices=("c2", "c1", "dp", "c3", "remote", "tp", "decode"), default="c2",
                    help="c2: the metric's 1-GPU config; dp: LoRAServe placement + routing across the ranks "
                         "(default when launched with more than one rank)")
    ap.add_argument("--tier", choices=("auto", "simt", "tc"), default="auto")
    ap.add_argument("--v-bf16", action="store_true",
                    help="tensor-core tier keeps v as one bf16 image (LSV_PLAN_V_BF16) instead of the hi/lo pair")
    ap.add_argument("--act-sets", type=int, default=0,
                    help="activation buffer sets reused round robin over the layers (0: one per layer)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip the N=1 dp-workload and config-1 lines")
    ap.add_argument("--tp-adapters", type=int, default=0,
                    help="config tp: roster size (default 1000 at TP8, scaled by TP/8 below that to fit HBM)")
    ap.add_argument("--cpu-budget-s", type=float, default=20.0)
    ap.add_argument("--tp-padded", action="store_true",
                    help="config tp: column-group ranks padded to 8*TP (equal shards) instead of balanced shards")
    return ap.parse_args(argv)


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            d = json.loads(p.read_text())
            return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
        except Exception:
            pass
    return HBM_FALLBACK_GBS, "fallback (B200_PROFILING.md)"


# ---------------------------------------------------------------------------------------
# clocks sampled during the timed region
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.dev = device_index
        self.rows: list[list[str]] = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms", "100",
                 "-i", str(self.dev)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        def reader():
            for line in self.proc.stdout:
                self.rows.append([c.strip() for c in line.split(",")])
        self.thread = threading.Thread(target=reader, daemon=True)
        self.thread.start()

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=1)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[1]))
                smax.append(float(r[2]))
                for name, flag in zip(names, r[5:9]):
                    if flag.strip().lower() in ("active", "1"):
                        reasons.add(name)
            except (ValueError, IndexError):
                continue
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------------------
def cpu_layer_sample(wl, x_layer0: dict, adapters_l0: dict, budget_s: float):
    """Time the CPU oracle on one full layer (all projections) of the workload; returns
    (seconds per layer (median over reps), reps, threads)."""
    from oracle import oracle
    from paper_2511_22880_b200.lora import input_group
    seg = wl.segments
    threads = oracle.cpu_threads()
    times = []
    t_start = time.perf_counter()
    while True:
        t0 = time.perf_counter()
        for p, pr in enumerate(wl.model.projections):
            a_list = [adapters_l0[(int(slot), p)][0] for slot in seg.seg_slot]
            b_list = [adapters_l0[(int(slot), p)][1] for slot in seg.seg_slot]
            oracle.delta_c(x_layer0[input_group(pr.name)], seg.seg_indptr, seg.seg_rank, a_list, b_list,
                           pr.h_out, threads=threads)
        times.append(time.perf_counter() - t0)
        if time.perf_counter() - t_start > budget_s * 0.5 or len(times) >= 10:
            break
    return statistics.median(times), len(times), threads


def host_layer_inputs(wl, seed=0):
    """CPU-generated layer-0 inputs for the reference arm (x and adapters, bf16 bit patterns)."""
    import torch
    from paper_2511_22880_b200.lora import input_group
    g = torch.Generator().manual_seed(seed)
    n = wl.segments.num_tokens
    xs = {}
    for pr in wl.model.projections:
        grp = input_group(pr.name)
        if grp not in xs:
            xs[grp] = torch.randn(n, pr.h_in, generator=g).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    ads = {}
    for slot, r in enumerate(wl.ranks):
        ga = torch.Generator().manual_seed(1000 + slot)
        for p, pr in enumerate(wl.model.projections):
            a = (torch.randn(r, pr.h_in, generator=ga) / pr.h_in ** 0.5).to(torch.bfloat16)
            b = (torch.randn(pr.h_out, r, generator=ga) / r ** 0.5).to(torch.bfloat16)
            ads[(slot, p)] = (a.view(torch.int16).numpy().view(np.uint16), b.view(torch.int16).numpy().view(np.uint16))
    return xs, ads


def run_reference(args, rank):
    """--impl reference: the CPU restatement on the host cores, bounded sample per step.  Same
    workload as our arm: under torchrun (N > 1) that is the data-parallel job (one LoRAServe-routed
    batch per GPU), which rank 0 runs on its host cores batch after batch."""
    from paper_2511_22880_b200 import shapes as _shapes, synth
    if rank != 0:
        return None
    world = int(os.environ.get("WORLD_SIZE", "1"))
    config = args.config if not (world > 1 and args.config == "c2") else "dp"
    if config in ("dp", "c3"):
        wls = synth.dp_workloads(world, model=_shapes.LLAMA2_13B if config == "c3" else _shapes.LLAMA2_7B)
    else:
        wls = [synth.WORKLOADS[config]()]
    wl = wls[0]
    inputs = [host_layer_inputs(w) for w in wls]
    layers = wl.model.layers
    tokens = sum(w.segments.num_tokens for w in wls)
    per_step = []
    for i in range(args.warmup + args.steps):
        t_layer = 0.0
        for w, (xs, ads) in zip(wls, inputs):       # one layer of every batch per step
            t, _, threads = cpu_layer_sample(w, xs, ads, budget_s=0.0)
            t_layer += t
        if i >= args.warmup:
            per_step.append(t_layer)
    t_layer = statistics.median(per_step)
    value = tokens / (t_layer * layers)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_layer * layers * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16 in, fp32 accumulate",
        "data": "synthetic",
        "config": {"workload": wl.description if len(wls) == 1 else
                   f"{config}: {len(wls)} per-GPU batches ({wl.model.name}, LoRAServe placement + routing)",
                   "config": config, "sample": "1 layer per step of every batch, x layers"},
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": threads, "kind": "port",
                         "sample": f"1 of {layers} layers (all {len(wl.model.projections)} projections) of "
                                   f"{len(wls)} batch(es) per step, extrapolated x{layers}"},
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    return line


# ---------------------------------------------------------------------------------------
def run_ours(args, rank, world, local_rank):
    import torch
    from paper_2511_22880_b200 import native, synth
    from paper_2511_22880_b200.lora import (LoraDeltaEngine, algorithmic_bytes, algorithmic_flops,
                                            input_group, moved_bytes)
    from paper_2511_22880_b200.segments import index_tokens
    from paper_2511_22880_b200.slab import AdapterSlab

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    tier = {"auto": native.TIER_AUTO, "simt": native.TIER_SIMT, "tc": native.TIER_TC}[args.tier]
    config = args.config if not (world > 1 and args.config == "c2") else "dp"
    if config == "dp":
        wl = synth.dp_workloads(world)[rank]
    elif config == "c3":      # BASELINE config 3: Llama-2-13B shapes, LoRAServe placement + routing
        from paper_2511_22880_b200 import shapes as _shapes
        wl = synth.dp_workloads(world, model=_shapes.LLAMA2_13B)[rank]
    else:
        wl = synth.WORKLOADS[config]()
    model = wl.model
    seg = wl.segments
    N = seg.num_tokens

    # adapters resident in this GPU's HBM slab (random-init, seeded per adapter id)
    slab_bytes = AdapterSlab.capacity_for(model, wl.ranks)
    slab = AdapterSlab(model, slab_bytes, dev)
    for aid, r in zip(wl.adapter_ids, wl.ranks):
        slab.fill_random(slab.allocate(aid, r), 1000 + zlib.crc32(aid.encode()) % 100000)
    eng = LoraDeltaEngine(slab, tier_policy=tier, v_bf16=args.v_bf16)
    bp = eng.prepare(seg)

    # per-layer activations (distinct buffers; every step moves far more than the 126 MB L2)
    g = torch.Generator(device=dev).manual_seed(1 + rank)
    groups = {}
    for pr in model.projections:
        groups.setdefault(input_group(pr.name), pr.h_in)
    n_sets = model.layers if args.act_sets <= 0 else min(args.act_sets, model.layers)
    xs = [{grp: torch.randn(N, h, device=dev, generator=g).to(torch.bfloat16) for grp, h in groups.items()}
          for _ in range(n_sets)]
    ys = [{pr.name: torch.randn(N, pr.h_out, device=dev, generator=g).to(torch.bfloat16) for pr in model.projections}
          for _ in range(n_sets)]
    xs = [xs[l % n_sets] for l in range(model.layers)]
    ys = [ys[l % n_sets] for l in range(model.layers)]
    stream = torch.cuda.Stream(dev)
    torch.cuda.synchronize(dev)

    # ---- device-resident throughput: CUDA-graph replay of the whole step ----
    with torch.cuda.stream(stream):
        eng.forward(bp, xs, ys, stream)   # warm the tensor-map cache before capture
    torch.cuda.synchronize(dev)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=stream):
        eng.forward(bp, xs, ys, stream)
    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            graph.replay()
    torch.cuda.synchronize(dev)
    sampler = ClockSampler(dev.index)
    sampler.start()
    time.sleep(0.3)
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        e0.record(stream)
        for _ in range(args.steps):
            graph.replay()
        e1.record(stream)
    torch.cuda.synchronize(dev)
    clocks = sampler.stop()
    ms_local = e0.elapsed_time(e1) / args.steps
    ms = ms_local
    # the same step with every launch waiting for its predecessor (no group shrink starting under the
    # previous group's expand): what a model whose next input depends on the previous output gets
    ms_serial = time_graph(torch, eng, bp, xs, ys, stream, args.steps, args.warmup, dev,
                           step_fn=lambda: eng.forward(bp, xs, ys, stream, serial=True))
    tokens_all = N * world
    per_rank = [[ms_local, N]]
    if world > 1:
        t = torch.tensor([ms_local, float(N)], device=dev)
        gathered = [torch.zeros_like(t) for _ in range(world)]
        torch.distributed.all_gather(gathered, t)
        per_rank = [g.tolist() for g in gathered]
        ms = max(p[0] for p in per_rank)
        tokens_all = int(sum(p[1] for p in per_rank))
    value = tokens_all / (ms / 1e3)

    # launches per step (our kernels only)
    launches = eng.launches_per_step(bp)

    # ---- algorithmic bytes / flops of the step ----
    # algorithmic: SURVEY §8d per projection (x counted once per projection); moved: what the
    # input-group path actually has to move (x once per group: q/k/v and gate/up share it)
    step_bytes = sum(algorithmic_bytes(seg, pr.h_in, pr.h_out) for pr in model.projections) * model.layers
    step_moved = moved_bytes(seg, model) * model.layers
    step_flops = sum(algorithmic_flops(seg, pr.h_in, pr.h_out) for pr in model.projections) * model.layers
    if world > 1:   # whole-job bytes/flops: every rank's own batch
        t = torch.tensor([float(step_bytes), float(step_flops), float(step_moved)], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(t)
        step_bytes, step_flops, step_moved = int(t[0].item()), int(t[1].item()), int(t[2].item())
    hbm_peak, peak_src = peaks()

    # ---- dominant kernel roofline: the one-launch expand of the input group with the most expand
    # bytes (gate/up on Llama), timed with CUDA events on its stream; its group's fused shrink beside it
    n_l = seg.lengths().astype(np.int64)
    r_l = seg.seg_rank.astype(np.int64)
    groups = model.groups()

    def grp_expand_bytes(members):
        return sum(int(np.sum(2 * r_l * model.projections[p].h_out + 4 * n_l * model.projections[p].h_out))
                   for p in members)
    gi = max(range(len(groups)), key=lambda i: grp_expand_bytes(groups[i][1]))
    gname, members = groups[gi]
    exp_bytes = grp_expand_bytes(members)
    h_in = model.projections[members[0]].h_in
    shr_bytes = int(np.sum(2 * n_l * h_in + 2 * len(members) * r_l * h_in))
    names = "/".join(model.projections[p].name for p in members)
    ylist = [ys[0][model.projections[p].name] for p in members]
    reps = 20
    with torch.cuda.stream(stream):
        eng.shrink(bp, 0, members[0], xs[0][gname], stream)
        k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        k0.record(stream)
        for _ in range(reps):
            eng.expand_group(bp, 0, gi, ylist, stream)
        k1.record(stream)
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        for _ in range(reps):
            eng.shrink(bp, 0, members[0], xs[0][gname], stream)
        s1.record(stream)
    torch.cuda.synchronize(dev)
    exp_us = k0.elapsed_time(k1) / reps * 1e3
    shr_us = s0.elapsed_time(s1) / reps * 1e3
    # the production path: one layer kernel per layer (every group's shrink and expand in one
    # launch, lsv_lora_forward); each call is one counter memset (~4 KB) + the kernel, so the time is
    # an upper bound.  The group kernel of the largest group alone beside it.
    grp_kernel = all(eng.group_kernel_eligible(gp) for gp in bp.group_plans)
    grp_us = lay_us = None
    if grp_kernel:
        with torch.cuda.stream(stream):
            eng.forward_layer(bp, 0, xs[0], ys[0], stream)
            l0e, l1e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            l0e.record(stream)
            for _ in range(reps):
                eng.forward_layer(bp, 0, xs[0], ys[0], stream)
            l1e.record(stream)
            eng.forward_group(bp, 0, gi, xs[0][gname], ylist, stream)
            g0e, g1e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            g0e.record(stream)
            for _ in range(reps):
                eng.forward_group(bp, 0, gi, xs[0][gname], ylist, stream)
            g1e.record(stream)
        torch.cuda.synchronize(dev)
        lay_us = l0e.elapsed_time(l1e) / reps * 1e3
        grp_us = g0e.elapsed_time(g1e) / reps * 1e3
    achieved = exp_bytes / (exp_us * 1e-6) / 1e9
    # which tier the group's work runs on (plan summary: [.., simt segments, m-tiles, ..])
    gsum = bp.group_plans[gi].summary
    simt_only = gsum[4] > 0 and gsum[5] == 0
    if simt_only:     # decode-regime batches: every segment on the SIMT tier
        exp_label = f"simt_expand_kernel ({names}, one launch per member)"
    else:
        exp_label = f"expand_tc_kernel ({names}, one launch)"
    traffic = measured_traffic(config, exp_label)
    grp_label = f"group_tc_kernel ({gname}: fused {names} shrink + expand, one launch)"
    grp_bytes = shr_bytes + exp_bytes      # x once per group, A, B, y read + write
    lay_label = "group_tc_kernel<4> (layer kernel: " + ", ".join(g for g, _ in groups) + ", one launch per layer)"
    lay_bytes = moved_bytes(seg, model)    # one layer: x once per group, A, B, y read + write

    # ---- e2e through the public API with host buffers ----
    from paper_2511_22880_b200.segments import index_tokens as _ix
    # E2E_BATCHES distinct batches of the same workload family (seeds 0..3 of the token -> adapter
    # draw), each in arrival order (tokens unsorted: the indexer computes a real permutation), fed
    # round robin so every step pays indexing and planning of a batch it has not just planned
    tok_batches = e2e_token_batches(config, wl, world, rank)
    x_host = torch.empty((N, model.projections[0].h_in), dtype=torch.bfloat16, pin_memory=True)
    x_host.copy_(xs[0][input_group(model.projections[0].name)].cpu())
    last = model.projections[-1]
    y_host = torch.empty((N, last.h_out), dtype=torch.bfloat16, pin_memory=True)
    g0 = input_group(model.projections[0].name)
    h2d_bytes = x_host.numel() * 2
    d2h_bytes = y_host.numel() * 2
    # double-buffered layer-0 input and last-layer output, so the H2D of step k+1 and the D2H of
    # step k run on the copy engines (own streams) while step k's kernels run
    xs_buf = [xs, [dict(d) for d in xs]]
    ys_buf = [ys, [dict(d) for d in ys]]
    xs_buf[1][0][g0] = torch.empty_like(xs[0][g0])
    ys_buf[1][-1][last.name] = torch.zeros_like(ys[-1][last.name])
    h2d_st, d2h_st = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    ev_h2d = [torch.cuda.Event(), torch.cuda.Event()]
    ev_fwd = [torch.cuda.Event(), torch.cuda.Event()]
    ev_d2h = [torch.cuda.Event(), torch.cuda.Event()]
    for e in ev_fwd + ev_d2h:
        e.record(stream)
    step_no = [0]

    def e2e_step():
        """One step through the public API: index the host batch, plan it (uploads asynchronous on
        the compute stream), H2D of x, the whole-model delta, D2H of y.  Nothing waits for the GPU,
        so the host work of step k+1 overlaps the GPU work of step k (a serving loop), and the
        copies of neighbouring steps overlap step k's kernels."""
        b = step_no[0] & 1
        seg_i = _ix(tok_batches[step_no[0] % len(tok_batches)], wl.ranks)   # host segment indexing
        step_no[0] += 1
        bp_i = eng.prepare(seg_i, stream=stream)                   # host planning + async plan/pointer upload
        h2d_st.wait_event(ev_fwd[b])                               # step k-2 done reading this x buffer
        with torch.cuda.stream(h2d_st):
            xs_buf[b][0][g0].copy_(x_host, non_blocking=True)      # H2D of the batch's input
            ev_h2d[b].record(h2d_st)
        stream.wait_event(ev_h2d[b])
        stream.wait_event(ev_d2h[b])                               # step k-2's result read out
        eng.forward(bp_i, xs_buf[b], ys_buf[b], stream)
        ev_fwd[b].record(stream)
        d2h_st.wait_event(ev_fwd[b])
        with torch.cuda.stream(d2h_st):
            y_host.copy_(ys_buf[b][-1][last.name], non_blocking=True)   # D2H of the result
            ev_d2h[b].record(d2h_st)
        return bp_i

    keep = []
    for _ in range(max(args.warmup, 8)):      # cycles every slot of the engine's upload ring
        keep.append(e2e_step())
    torch.cuda.synchronize(dev)
    gc.collect()
    if world > 1:
        torch.distributed.barrier()
    keep.clear()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        keep.append(e2e_step())                                    # plans stay alive until the sync
    torch.cuda.synchronize(dev)
    e2e_s = (time.perf_counter() - t0) / args.steps
    bp_last = keep[-1]
    plan_bytes = sum(sp.plan_host.nbytes for sp in bp_last.group_plans) + \
        (bp_last.a_ptrs.numel() + bp_last.b_ptrs.numel()) * 8
    keep.clear()
    if world > 1:
        t = torch.tensor([e2e_s], device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e_value = tokens_all / e2e_s

    # ---- CPU baseline (rank 0, N=1 only): the oracle on one full layer, extrapolated ----
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        x_l0 = {grp: t.view(torch.int16).cpu().numpy().view(np.uint16) for grp, t in xs[0].items()}
        ads = {}
        for slot in seg.seg_slot:
            for p in range(len(model.projections)):
                a, b = slab.read(int(slot), 0, p)
                ads[(int(slot), p)] = (a.view(torch.int16).cpu().numpy().view(np.uint16),
                                       b.view(torch.int16).cpu().numpy().view(np.uint16))
        t_layer, reps_cpu, threads = cpu_layer_sample(wl, x_l0, ads, args.cpu_budget_s)
        cpu = {"value": N / (t_layer * model.layers), "unit": "tokens/s", "cores": threads, "kind": "port",
               "sample": f"layer 0 of {model.layers} (all {len(model.projections)} projections, {N} tokens), "
                         f"median of {reps_cpu} reps, extrapolated x{model.layers}"}

    # N = 1 extras: the data-parallel workload of one server (like for like with the N > 1 lines)
    # and config 1 (launch-bound per-call time by CUDA-graph replay, the full CPU oracle beside it)
    extra = {}
    if world == 1 and config == "c2" and not args.no_extras:
        del graph
        torch.cuda.synchronize(dev)
        extra["dp_like_for_like"] = dp_one_server(args, torch, dev)
        extra["c1"] = c1_line(args, torch, dev)
        extra["fused_linear"] = fused_linear_line(args, torch, dev, wl)

    if rank != 0:
        return None
    line = {
        "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic (random-init adapters, N(0,1) activations)",
        "config": {"workload": wl.description, "config": config, "tier_policy": args.tier,
                   "v_precision": "bf16" if args.v_bf16 else "bf16 hi/lo pair (~16 bits)",
                   "per_gpu": [{"ms": p[0], "tokens": int(p[1])} for p in per_rank] if world > 1 else None,
                   "l2": ("inputs larger than L2 (per-layer activation buffers; %.1f GB moved per step)" % (step_bytes / 1e9)
                          if n_sets == model.layers else
                          "inputs larger than L2 (%d activation buffer sets reused round robin over the layers, as a "
                          "model reuses its activation memory; each layer's x + y are %.0f MB, %.1f GB moved per "
                          "step)" % (n_sets, sum(x.numel() * 2 for x in xs[0].values()) / 1e6 +
                                     sum(y.numel() * 2 for y in ys[0].values()) / 1e6, step_bytes / 1e9)),
                   "timing": "CUDA-graph replay of the whole step, CUDA events, max over ranks"},
        "step_hbm": {"algorithmic_bytes": step_bytes, "achieved_GBs": step_bytes / (ms * 1e-3) / 1e9,
                     "frac": step_bytes / (ms * 1e-3) / 1e9 / (hbm_peak * world), "flops": step_flops,
                     "moved_bytes": step_moved, "moved_frac": step_moved / (ms * 1e-3) / 1e9 / (hbm_peak * world),
                     "note": "whole-job algorithmic bytes (SURVEY 8d, x per projection) / step time / (peak x GPUs); "
                             "moved: x once per input group (q/k/v, gate/up share one fused shrink)"},
        "roofline": ({"bound": "hbm", "kernel": lay_label,
                      "achieved": lay_bytes / (lay_us * 1e-6) / 1e9, "peak": hbm_peak, "peak_source": peak_src,
                      "unit": "GB/s", "frac": lay_bytes / (lay_us * 1e-6) / 1e9 / hbm_peak,
                      "traffic": measured_traffic(config, lay_label), "launch_us": lay_us,
                      "algorithmic_bytes_per_launch": lay_bytes,
                      "bytes_note": "one layer: x once per input group + A of every member (shrinks) + B and y read + "
                                    "write of every projection (expands); v images, split-K partials and metadata "
                                    "excluded",
                      "timing": f"CUDA events around {reps} one-layer lsv_lora_forward_ex calls on the launching "
                                "stream (each call: a ~4 KB counter memset + the kernel)",
                      "traffic_source": "profiles/traffic.json: dram__bytes_read.sum + dram__bytes_write.sum of the "
                                        "same launch from one ncu --set full capture (tools/prof_group.py)",
                      # inside the step the layer kernels run back to back (PDL, dynamic expand dispatch):
                      # the step time over its launches is their average duration there
                      "in_step": ({"launch_us": ms * 1e3 / launches,
                                   "frac": lay_bytes / (ms * 1e-3 / launches) / 1e9 / hbm_peak,
                                   "note": "step time / layer-kernel launches per step (the step is only these "
                                           "launches and one counter memset)"}
                                  if launches == wl.model.layers and world == 1 else None),
                      "group_kernel": {"kernel": grp_label, "launch_us": grp_us, "algorithmic_bytes_per_launch": grp_bytes,
                                       "achieved": grp_bytes / (grp_us * 1e-6) / 1e9,
                                       "frac": grp_bytes / (grp_us * 1e-6) / 1e9 / hbm_peak},
                      "split_launches": {"expand": {"kernel": exp_label, "launch_us": exp_us,
                                                    "algorithmic_bytes_per_launch": exp_bytes, "achieved": achieved},
                                         "shrink": {"kernel": f"shrink_tc_kernel (fused {len(members)}-projection group {names})",
                                                    "launch_us": shr_us, "algorithmic_bytes_per_launch": shr_bytes,
                                                    "achieved": shr_bytes / (shr_us * 1e-6) / 1e9}}}
                     if grp_kernel else
                     {"bound": "hbm", "kernel": exp_label,
                      "achieved": achieved, "peak": hbm_peak, "peak_source": peak_src, "unit": "GB/s",
                      "frac": achieved / hbm_peak, "traffic": traffic, "launch_us": exp_us,
                      "algorithmic_bytes_per_launch": exp_bytes,
                      "traffic_source": "profiles/traffic.json: dram__bytes_read.sum + dram__bytes_write.sum of the "
                                        "same launch from one ncu --set full capture (tools/prof_one.py)",
                      "shrink": {"kernel": (f"simt_shrink_kernel ({names}, one launch)" if simt_only else
                                            f"shrink_tc_kernel (fused {len(members)}-projection group {names})"),
                                 "launch_us": shr_us, "algorithmic_bytes_per_launch": shr_bytes,
                                 "achieved": shr_bytes / (shr_us * 1e-6) / 1e9}}),
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_value, "unit": "tokens/s", "h2d_bytes_per_step": h2d_bytes + plan_bytes,
                "d2h_bytes_per_step": d2h_bytes,
                "path": "per step: index_tokens -> LoraDeltaEngine.prepare (async uploads) -> H2D x -> forward "
                        "(one lsv_lora_forward call) -> D2H y; steps issued back to back (host planning of step k+1 "
                        "overlaps the GPU work of step k; H2D/D2H on their own streams with double-buffered "
                        "x/y overlap neighbouring steps' kernels), wall clock over all steps after one final sync",
                "batches": f"{len(tok_batches)} distinct seeded batches round robin, tokens in arrival order "
                           "(the indexer's stable sort by adapter slot is a real permutation); the host batch "
                           "former lays x out in segment order before the H2D"},
        "gpu_launches": launches * args.steps,
        "serial_step": {"ms_per_step": ms_serial, "value": tokens_all / (ms_serial / 1e3) if world == 1 else None,
                        "note": "the same step with every launch waiting for its predecessor (lsv_lora_forward_ex "
                                "LSV_FWD_SERIAL): no group shrink under the previous group's expand"},
        "clocks": clocks,
    }
    if extra:
        line.update(extra)
    return line


def e2e_token_batches(config, wl, world, rank, n=4):
    """Per-token adapter slots of ``n`` distinct batches of the workload, in arrival order (shuffled).
    c2: seeds 0..n-1 of its token -> adapter draw (same roster); other configs: batches resampled
    from this GPU's batch (same resident adapters, same per-adapter token distribution)."""
    from paper_2511_22880_b200 import synth
    base = np.repeat(wl.segments.seg_slot, wl.segments.lengths())
    out = []
    for k in range(n):
        rng = np.random.default_rng(100 + k)
        if config == "c2":
            w = synth.c2_llama2_7b(seed=k)
            slots = np.repeat(w.segments.seg_slot, w.segments.lengths())
        else:
            slots = rng.choice(base, size=len(base), replace=True) if k > 0 else base
        out.append(rng.permutation(slots))
    return out


def dp_one_server(args, torch, dev):
    """The data-parallel workload (LoRAServe placement + routing) with one server: what the N > 1
    lines run per GPU, so the 1 -> N curve is like for like."""
    import zlib
    from paper_2511_22880_b200 import synth
    from paper_2511_22880_b200.lora import LoraDeltaEngine, input_group
    from paper_2511_22880_b200.slab import AdapterSlab
    wl = synth.dp_workloads(1)[0]
    model, seg = wl.model, wl.segments
    N = seg.num_tokens
    slab = AdapterSlab(model, AdapterSlab.capacity_for(model, wl.ranks), dev)
    for aid, r in zip(wl.adapter_ids, wl.ranks):
        slab.fill_random(slab.allocate(aid, r), 1000 + zlib.crc32(aid.encode()) % 100000)
    eng = LoraDeltaEngine(slab, v_bf16=args.v_bf16)
    bp = eng.prepare(seg)
    g = torch.Generator(device=dev).manual_seed(11)
    groups = {}
    for pr in model.projections:
        groups.setdefault(input_group(pr.name), pr.h_in)
    xs = [{k: torch.randn(N, h, device=dev, generator=g).to(torch.bfloat16) for k, h in groups.items()}
          for _ in range(model.layers)]
    ys = [{pr.name: torch.randn(N, pr.h_out, device=dev, generator=g).to(torch.bfloat16) for pr in model.projections}
          for _ in range(model.layers)]
    stream = torch.cuda.Stream(dev)
    ms = time_graph(torch, eng, bp, xs, ys, stream, args.steps, args.warmup, dev)
    out = {"workload": wl.description, "value": N / (ms / 1e3), "ms_per_step": ms, "tokens": N,
           "note": "synth.dp_workloads(1): the per-GPU workload family of the N > 1 lines with one server"}
    del eng, bp, slab, xs, ys
    torch.cuda.synchronize(dev)
    return out


def c1_line(args, torch, dev, replays=1000):
    """BASELINE config 1 (q_proj 4096x4096, 4 adapters r=8/16/64/128, 4 x 64 tokens): per-call time
    of one lsv_lora_apply by CUDA-graph replay (launch-bound), and the full (not extrapolated) CPU
    oracle on the same inputs."""
    from oracle import oracle
    from paper_2511_22880_b200 import synth
    from paper_2511_22880_b200.lora import LoraDeltaEngine
    from paper_2511_22880_b200.slab import AdapterSlab
    wl = synth.c1_qproj()
    pr = wl.model.projections[0]
    seg = wl.segments
    g = torch.Generator().manual_seed(0)
    x = torch.randn(seg.num_tokens, pr.h_in, generator=g).to(torch.bfloat16)
    slab = AdapterSlab(wl.model, AdapterSlab.capacity_for(wl.model, wl.ranks), dev)
    a_bits, b_bits = [], []
    for i, r in enumerate(wl.ranks):
        ga = torch.Generator().manual_seed(1000 + i)
        a = (torch.randn(r, pr.h_in, generator=ga) / pr.h_in ** 0.5).to(torch.bfloat16)
        b = (torch.randn(pr.h_out, r, generator=ga) / r ** 0.5).to(torch.bfloat16)
        slab.load(slab.allocate(wl.adapter_ids[i], r), 0, 0, a.to(dev), b.to(dev))
        a_bits.append(a.view(torch.int16).numpy().view(np.uint16))
        b_bits.append(b.view(torch.int16).numpy().view(np.uint16))
    eng = LoraDeltaEngine(slab, v_bf16=args.v_bf16)
    bp = eng.prepare(seg)
    xd = x.to(dev)
    y = torch.zeros(seg.num_tokens, pr.h_out, dtype=torch.bfloat16, device=dev)
    stream = torch.cuda.Stream(dev)
    with torch.cuda.stream(stream):
        eng.apply(bp, 0, 0, xd, y, stream)
    torch.cuda.synchronize(dev)
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr, stream=stream):
        for _ in range(10):
            eng.apply(bp, 0, 0, xd, y, stream)
    with torch.cuda.stream(stream):
        for _ in range(3):
            gr.replay()
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(replays // 10):
            gr.replay()
        e1.record(stream)
    torch.cuda.synchronize(dev)
    us = e0.elapsed_time(e1) * 1e3 / replays
    from paper_2511_22880_b200.lora import algorithmic_bytes
    nbytes = algorithmic_bytes(seg, pr.h_in, pr.h_out)
    # the CPU oracle on all of config 1 (no extrapolation), all host threads
    xb = x.view(torch.int16).numpy().view(np.uint16)
    a_l = [a_bits[s] for s in seg.seg_slot]
    b_l = [b_bits[s] for s in seg.seg_slot]
    oracle.delta_c(xb, seg.seg_indptr, seg.seg_rank, a_l, b_l, pr.h_out)
    reps, t0 = 0, time.perf_counter()
    while reps < 200 and time.perf_counter() - t0 < 5.0:
        oracle.delta_c(xb, seg.seg_indptr, seg.seg_rank, a_l, b_l, pr.h_out)
        reps += 1
    cpu_us = (time.perf_counter() - t0) / reps * 1e6
    return {"workload": wl.description, "us_per_call": us, "tokens_per_s": seg.num_tokens / (us * 1e-6),
            "hbm_frac": nbytes / (us * 1e-6) / 1e9 / peaks()[0], "algorithmic_bytes": nbytes,
            "timing": f"CUDA graph of 10 lsv_lora_apply calls replayed {replays // 10}x (shrink + expand launches "
                      "back to back), CUDA events",
            "cpu": {"us_per_call": cpu_us, "tokens_per_s": seg.num_tokens / (cpu_us * 1e-6),
                    "cores": oracle.cpu_threads(), "kind": "port",
                    "sample": f"all of config 1, {reps} calls, no extrapolation"}}


def fused_linear_line(args, torch, dev, wl, layers=4):
    """a LoRA linear layer = base projection GEMM + the adapter delta, on C2's
    batch and shapes (Llama-2-7B, 4096 tokens, 100 adapters), ``layers`` distinct layers per step
    (weights and activations beyond L2).  Three ways on the same box, CUDA-graph replay:
      base      cuBLAS (torch.matmul) base GEMMs only, the floor the delta adds to
      separate  cuBLAS base GEMMs + the delta path (fused group shrink + group expand: y += delta)
      fused     lsv_lora_fused_linear: group shrink + one GEMM whose TMEM tile also accumulates v·B
    Tensor roofline: (base + LoRA) FLOPs / time against MEASURED_PEAKS.json bf16_tflops_sustained."""
    import zlib
    from paper_2511_22880_b200.lora import LoraDeltaEngine, algorithmic_flops, input_group
    from paper_2511_22880_b200.shapes import ModelShape
    from paper_2511_22880_b200.slab import AdapterSlab
    model = ModelShape("llama-2-7b-%d-layers" % layers, layers, wl.model.projections)
    seg = wl.segments
    N = seg.num_tokens
    slab = AdapterSlab(model, AdapterSlab.capacity_for(model, wl.ranks), dev)
    for aid, r in zip(wl.adapter_ids, wl.ranks):
        slab.fill_random(slab.allocate(aid, r), 1000 + zlib.crc32(aid.encode()) % 100000)
    eng = LoraDeltaEngine(slab, v_bf16=args.v_bf16)
    bp_sep = eng.prepare(seg)
    bp_fus = eng.prepare(seg, fused_linear=True)
    g = torch.Generator(device=dev).manual_seed(5)
    projs = model.projections
    W = [[(torch.randn(pr.h_out, pr.h_in, device=dev, generator=g) / pr.h_in ** 0.5).to(torch.bfloat16)
          for pr in projs] for _ in range(layers)]
    xs = [{input_group(pr.name): torch.randn(N, pr.h_in, device=dev, generator=g).to(torch.bfloat16)
           for pr in projs} for _ in range(layers)]
    ys = [[torch.empty(N, pr.h_out, device=dev, dtype=torch.bfloat16) for pr in projs] for _ in range(layers)]
    stream = torch.cuda.Stream(dev)

    def base():
        for l in range(layers):
            for p, pr in enumerate(projs):
                torch.matmul(xs[l][input_group(pr.name)], W[l][p].t(), out=ys[l][p])

    def separate():
        base()
        for l in range(layers):
            for gi, (gname, members) in enumerate(eng.groups):
                eng.shrink(bp_sep, l, members[0], xs[l][gname], stream)
                eng.expand_group(bp_sep, l, gi, [ys[l][p] for p in members], stream)

    def fused():
        for l in range(layers):
            for gi, (gname, members) in enumerate(eng.groups):
                eng.linear_group(bp_fus, l, gi, xs[l][gname], [W[l][p] for p in members], [ys[l][p] for p in members],
                                 stream)

    res = {}
    for name, fn in (("base", base), ("separate", separate), ("fused", fused)):
        res[name] = time_graph(torch, eng, None, None, None, stream, max(args.steps, 10), args.warmup, dev,
                               step_fn=fn) / layers
    # parity of the fused layer against the separate path on one projection (both bf16 outputs)
    y_ref = torch.matmul(xs[0]["attn_in"], W[0][0].t())
    y_sep = y_ref.clone()
    eng.shrink(bp_sep, 0, 0, xs[0]["attn_in"])
    eng.expand(bp_sep, 0, 0, y_sep)
    fused()
    torch.cuda.synchronize(dev)
    agree = float((ys[0][0].float() - y_sep.float()).abs().max() / y_sep.float().abs().max())
    base_flops = sum(2 * N * pr.h_in * pr.h_out for pr in projs)
    lora_flops = sum(algorithmic_flops(seg, pr.h_in, pr.h_out) for pr in projs)
    peak = tflops_peak()
    out = {"workload": f"{wl.description.split(',')[0].replace('32 layers', '%d layers' % layers)}; base GEMMs "
                       f"{N}x{{4096,11008}}, per layer", "layers_timed": layers,
           "tokens": N, "peak_tflops": peak[0], "peak_source": peak[1],
           "agreement_vs_separate": agree,
           "timing": "CUDA-graph replay of the whole multi-layer step, CUDA events, per layer"}
    for name, ms in res.items():
        fl = base_flops + (lora_flops if name != "base" else 0)
        out[name] = {"ms_per_layer": ms, "tokens_per_s": N / (ms * 1e-3), "tflops": fl / (ms * 1e-3) / 1e12,
                     "tensor_frac": fl / (ms * 1e-3) / 1e12 / peak[0]}
    out["fused_vs_separate_speedup"] = res["separate"] / res["fused"]
    out["delta_overhead_separate"] = res["separate"] / res["base"] - 1
    out["delta_overhead_fused"] = res["fused"] / res["base"] - 1
    del eng, bp_sep, bp_fus, slab, W, xs, ys
    torch.cuda.synchronize(dev)
    return out


def tflops_peak():
    p = ROOT / "MEASURED_PEAKS.json"
    try:
        d = json.loads(p.read_text())
        return float(d["bf16_tflops_sustained"]), "measured sustained (MEASURED_PEAKS.json)"
    except Exception:
        return 2250.0 * 0.6, "fallback"


def measured_traffic(config, label):
    """DRAM bytes per launch of the roofline kernel, from the committed ncu capture (or None)."""
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "traffic.json")
    try:
        with open(path) as f:
            return json.load(f).get(config, {}).get(label)
    except (OSError, ValueError):
        return None


def time_graph(torch, eng, bp, xs, ys, stream, steps, warmup, dev, step_fn=None):
    """CUDA-graph the whole step once, replay warmup + steps, return ms per step (CUDA events)."""
    step_fn = step_fn or (lambda: eng.forward(bp, xs, ys, stream))
    with torch.cuda.stream(stream):
        step_fn()
    torch.cuda.synchronize(dev)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        step_fn()
    with torch.cuda.stream(stream):
        for _ in range(warmup):
            g.replay()
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            g.replay()
        e1.record(stream)
    torch.cuda.synchronize(dev)
    return e0.elapsed_time(e1) / steps


def run_remote(args, rank, world, local_rank):
    """Config 4: 30% of each GPU's tokens hit adapters owned by a peer GPU (CUDA-IPC-mapped peer
    slabs, no NCCL).  Two ways to use them: fetched a layer ahead into local staging buffers by the
    copy engines over NVLink while the current layer computes (``prefetch``, the headline), or read
    in-kernel over NVLink (``direct``).  Reports tokens/s and the overhead against the same batch
    with every adapter local."""
    import torch
    from paper_2511_22880_b200 import synth
    from paper_2511_22880_b200.lora import LoraDeltaEngine, RemotePrefetch, algorithmic_bytes, input_group
    from paper_2511_22880_b200.slab import AdapterSlab
    if world < 2:
        raise SystemExit("--config remote needs >= 2 ranks (torchrun)")
    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    wl, owner = synth.remote_workload(world, rank)
    model, seg = wl.model, wl.segments
    N = seg.num_tokens
    slab = AdapterSlab(model, AdapterSlab.capacity_for(model, wl.ranks), dev)
    for aid, r in zip(wl.adapter_ids, wl.ranks):
        slab.fill_random(slab.allocate(aid, r), 1000 + zlib.crc32(aid.encode()) % 100000)
    torch.cuda.synchronize(dev)
    handles = [None] * world
    torch.distributed.all_gather_object(handles, slab.ipc_handle())
    roster = list(zip(wl.adapter_ids, wl.ranks))
    peers = {r: AdapterSlab.open_peer(model, handles[r], roster, dev) for r in range(world) if r != rank}
    eng = LoraDeltaEngine(slab)
    bp_local = eng.prepare(seg)
    bp_remote = eng.prepare(seg, seg_owner=owner, peer_slabs=peers)              # bytes-only LPT plan (default)
    bp_remote_aware = eng.prepare(seg, seg_owner=owner, peer_slabs=peers, remote_aware=True)   # NVLink-aware LPT
    pf = RemotePrefetch(eng, seg, owner, peers)
    bp_pf = pf.plan()
    g = torch.Generator(device=dev).manual_seed(1 + rank)
    groups = {}
    for pr in model.projections:
        groups.setdefault(input_group(pr.name), pr.h_in)
    xs = [{k: torch.randn(N, h, device=dev, generator=g).to(torch.bfloat16) for k, h in groups.items()}
          for _ in range(model.layers)]
    ys = [{pr.name: torch.randn(N, pr.h_out, device=dev, generator=g).to(torch.bfloat16) for pr in model.projections}
          for _ in range(model.layers)]
    # remote reads produce bit-identical deltas (same weights, same math)
    y_l = torch.zeros(N, model.projections[0].h_out, device=dev, dtype=torch.bfloat16)
    y_r = torch.zeros_like(y_l)
    eng.apply(bp_local, 0, 0, xs[0][input_group(model.projections[0].name)], y_l)
    eng.apply(bp_remote, 0, 0, xs[0][input_group(model.projections[0].name)], y_r)
    torch.cuda.synchronize(dev)
    identical = bool(torch.equal(y_l, y_r))
    # the prefetched step must give the all-local step's bits on every layer and projection
    ys_a = [{pr.name: torch.zeros(N, pr.h_out, device=dev, dtype=torch.bfloat16) for pr in model.projections}
            for _ in range(model.layers)]
    ys_b = [{pr.name: torch.zeros(N, pr.h_out, device=dev, dtype=torch.bfloat16) for pr in model.projections}
            for _ in range(model.layers)]
    eng.forward(bp_local, xs, ys_a)
    eng.forward_prefetch(bp_pf, pf, xs, ys_b)
    torch.cuda.synchronize(dev)
    identical_pf = all(torch.equal(ys_a[l][k], ys_b[l][k]) for l in range(model.layers) for k in ys_a[l])
    del ys_a, ys_b
    stream = torch.cuda.Stream(dev)
    arm_clocks = {}

    def timed(name, bp_, fn=None):
        torch.distributed.barrier()
        smp = ClockSampler(dev.index)
        smp.start()
        ms_ = time_graph(torch, eng, bp_, xs, ys, stream, args.steps, args.warmup, dev, step_fn=fn)
        arm_clocks[name] = smp.stop()
        return ms_
    ms_local = timed("all_local", bp_local)
    ms_pf = timed("prefetch", bp_pf, lambda: eng.forward_prefetch(bp_pf, pf, xs, ys, stream))
    ms_plain = timed("direct_nvlink_aware_plan", bp_remote_aware)
    ms_direct = timed("direct", bp_remote)
    # SM-partitioned: peer-owned segments on a few CTAs (own stream), local ones on the rest
    from paper_2511_22880_b200.lora import SplitStep
    split = {}
    for rs in (16, 32):
        sp = SplitStep(slab, seg, owner, peers, remote_sms=rs)
        split[rs] = timed(f"split{rs}", None, lambda sp=sp: sp.forward(xs, ys, stream))
        del sp
    rs_best = min(split, key=split.get)
    ms_split = split[rs_best]
    clocks = arm_clocks["direct"]
    # copy-on-first-use (the reference's commit_migration): every peer-owned adapter this GPU's
    # batch uses, copied once into a local slab by the copy engines; afterwards the batch runs
    # all-local (ms_local).  Break-even: how many steps of direct peer loads the copy costs.
    peer_aids = sorted({(wl.adapter_ids[int(sl)], int(o)) for sl, o in zip(seg.seg_slot, owner) if int(o) != rank})
    mig = AdapterSlab(model, AdapterSlab.capacity_for(model, [wl.ranks[wl.adapter_ids.index(a)] for a, _ in peer_aids]), dev)
    torch.cuda.synchronize(dev)
    torch.distributed.barrier()
    m0, m1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    m0.record(stream)
    for aid, o in peer_aids:
        mig.migrate_from_peer(aid, peers[o], stream)
    m1.record(stream)
    torch.cuda.synchronize(dev)
    ms_mig = m0.elapsed_time(m1)
    mig_bytes = sum(mig.slots[sl].nbytes for sl in mig.by_id.values())
    L_, P_ = model.layers - 1, len(model.projections) - 1   # the slot's last bytes: A and B of the last layer

    def _same(aid):
        (a1, b1), (a2, b2) = mig.read(mig.by_id[aid], L_, P_), slab.read(slab.by_id[aid], L_, P_)
        return torch.equal(a1, a2) and torch.equal(b1, b2)
    mig_identical = all(_same(a) for a, _ in peer_aids[:4])
    del mig
    t = torch.tensor([ms_local, ms_direct, float(identical and identical_pf and mig_identical), ms_pf, ms_mig,
                      float(mig_bytes), ms_plain] + [split[k] for k in sorted(split)], device=dev, dtype=torch.float64)
    per = [torch.zeros_like(t) for _ in range(world)]
    torch.distributed.all_gather(per, t)
    per = [p.tolist() for p in per]
    ms_l = max(p[0] for p in per)
    ms_r = max(p[1] for p in per)      # headline: in-kernel NVLink peer loads
    ms_p = max(p[3] for p in per)
    ms_pl = max(p[6] for p in per)
    ms_sp = {k: max(p[7 + i] for p in per) for i, k in enumerate(sorted(split))}
    lens = seg.lengths()
    remote_frac = float(np.sum(seg.lengths()[owner != rank])) / N
    step_bytes = sum(algorithmic_bytes(seg, pr.h_in, pr.h_out) for pr in model.projections) * model.layers
    hbm_peak, peak_src = peaks()
    if rank != 0:
        return None
    return {
        "metric": METRIC, "value": N * world / (ms_r / 1e3), "unit": "tokens/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_r, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic (random-init adapters)",
        "config": {"workload": wl.description, "config": "remote", "remote_token_fraction": remote_frac,
                   "remote_mode": "in-kernel NVLink peer loads from CUDA-IPC-mapped peer slabs",
                   "per_gpu": [{"ms_local": p[0], "ms_remote_direct": p[1], "ms_remote_prefetch": p[3],
                                "bit_identical": bool(p[2])} for p in per],
                   "timing": "CUDA-graph replay, CUDA events, max over ranks"},
        "remote_overhead": ms_r / ms_l - 1.0,
        "remote_split": {"ms_per_step": min(ms_sp.values()), "overhead": min(ms_sp.values()) / ms_l - 1.0,
                         "by_remote_sms": ms_sp,
                         "mode": "SplitStep: peer-owned segments on R CTAs (their own plan and stream), local ones on "
                                 "the other 148 - R (LSV_SEG_SKIP + LSV_PLAN_SMS)"},
        "remote_nvlink_aware_plan": {"ms_per_step": ms_pl, "overhead": ms_pl / ms_l - 1.0,
                                     "note": "the same peer reads with the plan built with LSV_SEG_REMOTE (peer bytes "
                                             "weighted 7x in the LPT cost, remote and local records interleaved); the "
                                             "headline uses the bytes-only plan, measured faster with the layer kernel"},
        "batch_shape": {"segments": int(seg.num_segments), "mean_tokens_per_segment": float(np.mean(lens)),
                        "segments_under_32_tokens": int(np.sum(lens < 32)),
                        "note": "70% of the GPU's tokens on its 100/N own adapters, 30% spread over the others' "
                                "(synth.remote_workload): smaller segments than C2's (41 tokens each) as N grows"},
        "remote_prefetch": {"ms_per_step": ms_p, "value": N * world / (ms_p / 1e3), "overhead": ms_p / ms_l - 1.0,
                            "mode": "copy-engine fetch (lsv_copy_blocks) of the next layer's peer-owned tiles into "
                                    f"local staging while the current layer computes; {pf.bytes_per_layer / 1e6:.1f} "
                                    f"MB/layer over NVLink on GPU {rank}"},
        "all_local": {"ms_per_step": ms_l, "value": N * world / (ms_l / 1e3),
                      "hbm_frac": step_bytes / (ms_l * 1e-3) / 1e9 / hbm_peak},
        "remote_migration": {"mode": "copy-on-first-use: every peer-owned adapter of the batch copied once into a "
                                     "local slot (AdapterSlab.migrate_from_peer, lsv_copy_blocks over NVLink)",
                             "ms": max(p[4] for p in per), "bytes_per_gpu": [int(p[5]) for p in per],
                             "GBps": min(p[5] / (p[4] * 1e-3) / 1e9 for p in per),
                             "break_even_steps": max(p[4] for p in per) / max(ms_r - ms_l, 1e-9)},
        "step_hbm": {"frac_local_bytes": step_bytes / (ms_r * 1e-3) / 1e9 / hbm_peak},
        "clocks": clocks, "clocks_per_arm": arm_clocks,
    }


def run_tp(args, rank, world, local_rank):
    """Config 5: Llama-3-70B shapes tensor-parallel over the ranks (TP = world size); column-parallel
    projections all-gather the rank-sharded shrink output with NCCL, row-parallel ones all-reduce
    it.  value = tokens/s of the TP group (one batch over all ranks); the NCCL share is reported."""
    import torch
    from paper_2511_22880_b200 import shapes, traces
    from paper_2511_22880_b200.segments import index_tokens
    from paper_2511_22880_b200.tp import TPLoraDeltaEngine, TPSlab
    from paper_2511_22880_b200.lora import input_group
    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    model = shapes.LLAMA3_70B
    n_ad = args.tp_adapters or max(50, 1000 * world // 8)
    roster = traces.roster(n_ad)
    ranks = [a.rank for a in roster]
    rng = np.random.default_rng(0)
    tok = rng.integers(0, n_ad, 4096)
    seg = index_tokens(tok, ranks)
    slab = TPSlab(model, world, rank, ranks, dev, balanced=not args.tp_padded)
    for s_, r in enumerate(ranks):
        slab.fill_random_shards(s_, 1000 + s_)
    eng = TPLoraDeltaEngine(slab)
    st = eng.prepare(seg)
    N = seg.num_tokens
    g = torch.Generator(device=dev).manual_seed(7)
    xs, ys = [], []
    for _ in range(model.layers):
        xd, yd = {}, {}
        for sp in eng.specs:
            grp = input_group(sp.name)
            if grp not in xd:
                xd[grp] = torch.randn(N, sp.h_in, device=dev, generator=g).to(torch.bfloat16)
            yd[sp.name] = torch.zeros(N, sp.h_out, device=dev, dtype=torch.bfloat16)
        xs.append(xd)
        ys.append(yd)
    stream = torch.cuda.Stream(dev)
    torch.cuda.synchronize(dev)
    with torch.cuda.stream(stream):
        eng.forward(st, xs, ys, stream)          # warm tensor maps / NCCL before capture
    torch.cuda.synchronize(dev)
    torch.distributed.barrier()
    # the whole step (kernels and NCCL collectives) as one CUDA graph, replayed
    graph = torch.cuda.CUDAGraph()
    try:
        with torch.cuda.graph(graph, stream=stream):
            eng.forward(st, xs, ys, stream)
        timing = "CUDA-graph replay of the whole step incl. NCCL collectives, CUDA events, max over ranks"
        step = graph.replay
    except Exception as exc:   # capture unsupported here: time the eager step
        print(f"[bench] TP graph capture failed ({exc}); timing eager launches", file=sys.stderr)
        torch.cuda.synchronize(dev)
        timing = "eager launches incl. NCCL collectives, CUDA events, max over ranks"
        step = lambda: eng.forward(st, xs, ys, stream)   # noqa: E731
    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            step()
    torch.cuda.synchronize(dev)
    torch.distributed.barrier()
    sampler = ClockSampler(dev.index)
    sampler.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
    torch.cuda.synchronize(dev)
    clocks = sampler.stop()
    ms = e0.elapsed_time(e1) / args.steps
    # NCCL share: the same number of collectives on the same v regions, alone
    import torch.distributed as dist
    coll = []       # the NCCL collectives the step still issues: all-reduce of each row group's partial v
    fused = st.get("fused") is not None   # column groups exchange inside the kernels (NVLink stores)
    for gi, (_, members) in enumerate(eng.groups):
        plan_a = st["plans"][gi][0]
        off, nb = eng._region(plan_a)
        if not (fused and eng.specs[members[0]].column):   # row groups keep NCCL (forward's default)
            coll.append((eng.specs[members[0]].column, off, nb))
    torch.cuda.synchronize(dev)
    dist.barrier()                 # every rank enters the timed collectives together (no host skew inside)
    torch.cuda.synchronize(dev)
    c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ws_a = st["ws"][0]
    with torch.cuda.stream(stream):
        c0.record(stream)
        for _ in range(model.layers):
            for col, off, nb in coll:
                if col:
                    dist.all_gather_into_tensor(st["gathered"][:world * nb], ws_a[off:off + nb])
                else:
                    dist.all_reduce(ws_a[off:off + nb].view(torch.bfloat16))
        c1.record(stream)
    torch.cuda.synchronize(dev)
    coll_ms = c0.elapsed_time(c1)
    t = torch.tensor([ms, coll_ms], device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms, coll_ms = t.tolist()
    # algorithmic HBM bytes per GPU per step of ideal S-LoRA sharding (unpadded ranks; SURVEY 8d
    # per shard: x once per projection, the rank- or h_in-shard of A, the h_out shard of B and y)
    from paper_2511_22880_b200.tp import COLUMN_PARALLEL
    n_s = seg.lengths().astype(np.float64)
    r_s = seg.seg_rank.astype(np.float64)
    per_layer = 0.0
    for pr in model.projections:
        ho = pr.h_out / world
        if pr.name in COLUMN_PARALLEL:     # x full, A rank-shard
            per_layer += np.sum(2 * n_s * pr.h_in + 2 * (r_s / world) * pr.h_in + 2 * r_s * ho + 4 * n_s * ho)
        else:                              # x and A h_in-shards
            hi = pr.h_in / world
            per_layer += np.sum(2 * n_s * hi + 2 * r_s * hi + 2 * r_s * ho + 4 * n_s * ho)
    gpu_bytes = per_layer * model.layers
    hbm_peak, peak_src = peaks()
    if rank != 0:
        return None
    return {
        "metric": METRIC, "value": N / (ms / 1e3), "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic (random-init adapter shards)",
        "config": {"workload": f"llama-3-70b 80 layers x 7 proj, TP{world} (S-LoRA sharding), {n_ad} adapters "
                               f"{traces.assign_power_law_counts(n_ad, traces.DEFAULT_RANKS, 1.0)}, {N} tokens, "
                               f"{seg.num_segments} active", "config": "tp",
                   "shards": "padded to 8*TP" if args.tp_padded else "balanced (round-robin 8-row groups)",
                   "timing": timing},
        "nccl_ms_per_step": coll_ms, "nccl_share": coll_ms / ms,
        "step_hbm": {"algorithmic_bytes_per_gpu": gpu_bytes, "achieved_GBs_per_gpu": gpu_bytes / (ms * 1e-3) / 1e9,
                     "peak": hbm_peak, "peak_source": peak_src,
                     "frac": gpu_bytes / (ms * 1e-3) / 1e9 / hbm_peak,
                     "note": "ideal S-LoRA sharding with unpadded ranks" + (
                         "; this run pads column-group ranks to a multiple of 8*TP (--tp-padded)" if args.tp_padded else
                         "; column groups use balanced shards (round-robin 8-row groups, LSV_TP_ROUND_ROBIN): "
                         "the kernels move the unpadded bytes")},
        "exchange": ("column groups (q/k/v, gate/up): shrink epilogue stores each shard into every rank's full-rank "
                     "v image over NVLink + flag (no NCCL); row groups (o, down): NCCL all-reduce") if fused
                    else "NCCL all-gather (column groups) / all-reduce (row groups)",
        "clocks": clocks,
    }


def main(argv=None):
    args = parse_args(argv)
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        line = run_reference(args, rank)
        if line is not None:
            print(json.dumps(line), flush=True)
        return 0
    if world > 1 or args.config == "tp":
        import torch
        torch.cuda.set_device(local_rank)
        if world == 1:
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29533")
            torch.distributed.init_process_group("nccl", rank=0, world_size=1,
                                                 device_id=torch.device("cuda", local_rank))
        else:
            torch.distributed.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    if args.config == "remote":
        line = run_remote(args, rank, world, local_rank)
    elif args.config == "tp":
        line = run_tp(args, rank, world, local_rank)
    else:
        line = run_ours(args, rank, world, local_rank)
    if line is not None:
        print(json.dumps(line), flush=True)
    import torch
    if torch.distributed.is_available() and torch.distributed.is_initialized():
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
