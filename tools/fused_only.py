"""Run bench.py's fused-linear comparison alone (development): python tools/fused_only.py [--v-bf16]"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402

args = bench.parse_args(sys.argv[1:])
import torch  # noqa: E402
from paper_2511_22880_b200 import synth  # noqa: E402
dev = torch.device("cuda:0")
print(json.dumps(bench.fused_linear_line(args, torch, dev, synth.c2_llama2_7b()), indent=1))
