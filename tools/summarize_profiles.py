"""Regenerate the committed ncu summaries under profiles/ from a gpu_round.sh capture.

    python tools/summarize_profiles.py TAG      # reads gpurun_out/launches_TAG.csv, full_TAG.ncu-rep

writes profiles/<TAG>_launch_summary.txt, profiles/<TAG>_launches_c2_step.csv (the launch list),
profiles/<TAG>_ncu_full_mlp_in.txt and updates profiles/traffic.json (dram bytes per launch of the
roofline kernel, read by bench.py)."""
import csv
import io
import json
import subprocess
import sys
from collections import OrderedDict

TAG = sys.argv[1] if len(sys.argv) > 1 else "r1e"
OUT = sys.argv[2] if len(sys.argv) > 2 else TAG
DECODE = len(sys.argv) > 3 and sys.argv[3] == "decode"
WL = ("decode (C2 roster, 128 requests x 1 token, 73 active adapters; SIMT tier)" if DECODE else
      "config 2 (Llama-2-7B shapes, 100 adapters, 4096 tokens)")
CMD = "python bench.py --config decode --steps 1 --warmup 3 --no-cpu-baseline --no-extras" if DECODE else \
      "python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-extras"
GROUPS = ["attn_in (q/k/v fused)", "attn_out (o)", "mlp_in (gate/up fused)", "mlp_mid (down)"]
METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__cycles_active.avg", "gpc__cycles_elapsed.max",
           "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
           "launch__shared_mem_per_block_dynamic", "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active",
           "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smsp__cycles_active.avg"]


def launches():
    text = open(f"gpurun_out/launches_{TAG}.csv").read()
    body = text[text.index('"ID"'):]
    rows = [r for r in csv.DictReader(io.StringIO(body)) if r["Metric Name"] == "gpu__time_duration.sum"]
    scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "msecond": 1e3}
    out = [(r["Kernel Name"].split("(")[0], float(r["Metric Value"].replace(",", "")) * scale[r["Metric Unit"]])
           for r in rows]
    with open(f"profiles/{OUT}_launches{'' if DECODE else '_c2'}_step.csv", "w") as f:
        f.write("launch,kernel,us\n")
        for i, (k, us) in enumerate(out):
            f.write(f"{i},{k},{us:.3f}\n")
    agg = OrderedDict()
    for k, us in out:
        n, t = agg.get(k, (0, 0.0))
        agg[k] = (n + 1, t + us)
    total = sum(t for _, t in agg.values())
    lines = [f"# ncu launch list, {WL}, warm-up + one bench.py step",
             "# command: ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'tc_kernel|simt_|vimg' "
             "--csv \\",
             f"#          {CMD}   (after the same command exited 0 without ncu)",
             "# ncu serialises launches and replays with cold caches: absolute times run above the CUDA-graph step;",
             "# the per-kernel SHARE of the step is what to compare.  Full list: "
             f"profiles/{OUT}_launches{'' if DECODE else '_c2'}_step.csv",
             "# (the capture also holds bench.py's serialised-step replay and its roofline calls after the step)", "",
             f"{'kernel':20s} {'launches':>8s} {'total_us':>10s} {'mean_us':>9s} {'share':>7s}"]
    for k, (n, t) in agg.items():
        lines.append(f"{k:20s} {n:8d} {t:10.1f} {t / n:9.2f} {t / total:7.3f}")
    lines += ["", "per layer (first 3 layers of the capture, us):"]
    first = out[0][0] if out else ""
    layered = "group_tc_kernel<4>" in first
    grouped = not layered and "group_tc_kernel" in first
    per = 1 if layered else 4 if grouped else 8
    for layer in range(3):
        seg = out[layer * per:(layer + 1) * per]
        parts = []
        for g in range(1 if layered else 4):
            if layered:
                parts.append(f"layer kernel (all four groups) {seg[0][1]:.1f}")
            elif grouped:
                parts.append(f"group kernel {GROUPS[g]} {seg[g][1]:.1f}")
            else:
                parts.append(f"shrink {GROUPS[g]} {seg[2 * g][1]:.1f}")
                parts.append(f"expand {GROUPS[g].split(' ')[0]} (one launch) {seg[2 * g + 1][1]:.1f}")
        lines.append("  " + ", ".join(parts))
    step = out[:per * 32]
    lines += ["", f"one step = 32 layers x {per} launches = {len(step)} launches, sum {sum(u for _, u in step):.1f} us "
              "(serialised, cold caches)"]
    open(f"profiles/{OUT}_launch_summary.txt", "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


def full():
    raw = subprocess.run(["ncu", "-i", f"gpurun_out/full_{TAG}.ncu-rep", "--page", "raw", "--csv"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw[raw.index('"ID"'):])))
    hdr, units, data = rows[0], rows[1], rows[2:]
    col = {h: i for i, h in enumerate(hdr)}
    if DECODE:
        lines = ["# ncu --set full --clock-control none --import-source on -k regex:'simt_' -s 16 -c 2 "
                 "python tools/decode_one.py 128",
                 "# decode batch (128 requests x 1 token), 2-layer Llama-2-7B: the 17th-18th SIMT launches",
                 "# run only after `python tools/decode_one.py 128` exited 0 without ncu.  Cold-cache, serialised.", ""]
    else:
        lines = ["# ncu --set full --clock-control none --import-source on -k regex:'tc_kernel|simt_' -s 4 -c 2 "
                 "python tools/prof_one.py 2",
                 "# config 2, layer-0 mlp_in group: fused gate/up shrink + one-launch gate/up expand (the step's "
                 "largest pair);",
                 "# run only after `python tools/prof_one.py 2` exited 0 without ncu.  Cold-cache, serialised replay.", ""]
    traffic = {}
    for r in data:
        name = r[col["Kernel Name"]].split("(")[0]
        lines.append(f"== {name}")
        for m in METRICS:
            if m in col:
                lines.append(f"  {m:60s} {r[col[m]]:>20s} {units[col[m]]}")
        rd = float(r[col["dram__bytes_read.sum"]].replace(",", ""))
        wr = float(r[col["dram__bytes_write.sum"]].replace(",", ""))
        mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        b = rd * mult[units[col["dram__bytes_read.sum"]]] + wr * mult[units[col["dram__bytes_write.sum"]]]
        lines.append(f"  dram read+write bytes per launch: {b / 1e6:.1f} MB")
        lines.append("")
        traffic[name] = b
    open(f"profiles/{OUT}_ncu_full{'' if DECODE else '_mlp_in'}.txt", "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))
    if DECODE:
        return
    tj = json.load(open("profiles/traffic.json"))
    for k in tj["c2"]:
        kern = k.split(" ")[0]
        if kern in traffic:
            tj["c2"][k] = traffic[kern]
    tj["note"] = (f"dram__bytes_read.sum + dram__bytes_write.sum per launch: split launches from "
                  f"profiles/{OUT}_ncu_full_mlp_in.txt, the group kernel from profiles/{OUT}_ncu_group.txt. "
                  "Writes land in L2 and are partly evicted after the launch, so write bytes undercount.")
    json.dump(tj, open("profiles/traffic.json", "w"), indent=1)


def group():
    """The four group kernels of one layer (tools/prof_group.py capture) -> profiles/<OUT>_ncu_group.txt,
    and the mlp_in launch's DRAM bytes into traffic.json (bench.py's group-kernel roofline)."""
    import os
    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    lines, traffic = [], []
    for rep, hdr_lines, names in (
            (f"gpurun_out/group_full_{TAG}.ncu-rep",
             ["# ncu --set full --clock-control none --import-source on -k regex:group -s 3 -c 1 python tools/prof_group.py",
              "# config 2, one Llama-2-7B layer through lsv_lora_forward: the layer kernel (all four groups, one launch)"],
             ["layer kernel (attn_in, attn_out, mlp_in, mlp_mid)"]),
            (f"gpurun_out/group4_full_{TAG}.ncu-rep",
             ["# LSV_LAYER_KERNEL=0 ncu ... -k regex:group -s 12 -c 4 python tools/prof_group.py: the same layer as four",
              "# group kernels in order"], GROUPS)):
        if not os.path.exists(rep):
            continue
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
        rows = list(csv.reader(io.StringIO(raw[raw.index('"ID"'):])))
        hdr, units, data = rows[0], rows[1], rows[2:]
        col = {h: i for i, h in enumerate(hdr)}
        lines += hdr_lines + ["# run only after `python tools/prof_group.py` exited 0 without ncu.  Cold-cache, serialised.", ""]
        for g, r in enumerate(data):
            lines.append(f"== group_tc_kernel {names[g] if g < len(names) else g}")
            for m in METRICS:
                if m in col:
                    lines.append(f"  {m:60s} {r[col[m]]:>20s} {units[col[m]]}")
            b = float(r[col["dram__bytes_read.sum"]].replace(",", "")) * mult[units[col["dram__bytes_read.sum"]]] + \
                float(r[col["dram__bytes_write.sum"]].replace(",", "")) * mult[units[col["dram__bytes_write.sum"]]]
            lines.append(f"  dram read+write bytes per launch: {b / 1e6:.1f} MB")
            lines.append("")
            traffic.append((names[g] if g < len(names) else str(g), b))
    if not lines:
        return
    open(f"profiles/{OUT}_ncu_group.txt", "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))
    tj = json.load(open("profiles/traffic.json"))
    for name, b in traffic:
        for k in tj["c2"]:
            if name.startswith("layer kernel") and k.startswith("group_tc_kernel<4> (layer kernel"):
                tj["c2"][k] = b
            if name.startswith("mlp_in") and k.startswith("group_tc_kernel (mlp_in"):
                tj["c2"][k] = b
    json.dump(tj, open("profiles/traffic.json", "w"), indent=1)


if __name__ == "__main__":
    launches()
    full()
    group()
