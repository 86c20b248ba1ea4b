"""One-line summary of a bench.py JSON line on stdin (A/B scripts)."""
import json
import sys

d = json.loads(sys.stdin.read())
r = d["roofline"]
parts = [str(round(d["value"])), str(round(d["ms_per_step"], 3)), "serial", str(round(d["serial_step"]["ms_per_step"], 3))]
if "split_launches" in r:
    if "group_kernel" in r:
        parts += ["layer", str(round(r["launch_us"], 1)), f"({r['frac']:.3f})", "group", str(round(r["group_kernel"]["launch_us"], 1))]
    else:
        parts += ["group", str(round(r["launch_us"], 1))]
    parts += ["expand", str(round(r["split_launches"]["expand"]["launch_us"], 1)),
              "shrink", str(round(r["split_launches"]["shrink"]["launch_us"], 1))]
else:
    parts += ["expand", str(round(r["launch_us"], 1)), "shrink", str(round(r["shrink"]["launch_us"], 1))]
if "e2e" in d:
    parts += ["e2e", str(round(d["e2e"]["value"]))]
print(" ".join(parts))
