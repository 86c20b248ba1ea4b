"""Build liblsv.so in-tree for sm_100a (explicit nvcc; the .so travels to the GPU box with gpurun)."""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
REPO = PKG.parent
CSRC = PKG / "csrc"
OUT = PKG / "liblsv.so"
SOURCES = [CSRC / "lsv_api.cu"]
DEPS = sorted(CSRC.glob("*.cu*")) + sorted(CSRC.glob("*.h")) + [REPO / "include" / "lsv.h"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared", "-cudart", "static",
    "-Xptxas", "-v",
]


def nvcc() -> str:
    cand = os.environ.get("NVCC") or "/usr/local/cuda/bin/nvcc"
    return cand if Path(cand).exists() else "nvcc"


def needs_build() -> bool:
    if not OUT.exists():
        return True
    t = OUT.stat().st_mtime
    return any(p.stat().st_mtime > t for p in DEPS)


CHECKED = PKG / "liblsv_checked.so"   # LSV_DEVICE_CHECKS=1: device-side bounds checks (tools/gpu_checked.sh)


def build(force: bool = False, verbose: bool = False, checked: bool = False) -> Path:
    out = CHECKED if checked else OUT
    if not force and out.exists() and not any(p.stat().st_mtime > out.stat().st_mtime for p in DEPS):
        return out
    tmp = out.with_suffix(".so.tmp")
    extra = ["-DLSV_DEVICE_CHECKS=1"] if checked else []
    extra += os.environ.get("LSV_NVCC_DEFINES", "").split()   # development variants (A/B builds)
    cmd = [nvcc(), *NVCC_FLAGS, *extra, "-o", str(tmp), *map(str, SOURCES), "-ldl", "-lpthread", "-lrt"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    log = PKG / ("build_checked.log" if checked else "build.log")
    log.write_text(" ".join(cmd) + "\n" + res.stdout + res.stderr)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError(f"nvcc failed (see {log})")
    if verbose:
        sys.stdout.write(res.stderr)
    os.replace(tmp, out)
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
