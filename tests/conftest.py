import os
import random
import sys
from pathlib import Path

import pytest
from hypothesis import HealthCheck, settings

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

# Same hypothesis profile as the reference suite (pkg/tests/conftest.py:6-13).
settings.register_profile(
    "default", derandomize=True, max_examples=50,
    suppress_health_check=[HealthCheck.too_slow], deadline=None,
)
settings.load_profile("default")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run via gpurun)")
    config.addinivalue_line("markers", "multigpu: needs >= 2 GPUs")


@pytest.fixture
def rng():
    return random.Random(12345)


def pytest_collection_modifyitems(config, items):
    try:
        import torch
        have_gpu = torch.cuda.is_available()
        ngpu = torch.cuda.device_count() if have_gpu else 0
    except Exception:  # pragma: no cover
        have_gpu, ngpu = False, 0
    skip_gpu = pytest.mark.skip(reason="no CUDA device")
    skip_multi = pytest.mark.skip(reason="needs >= 2 GPUs")
    for item in items:
        if "gpu" in item.keywords and not have_gpu:
            item.add_marker(skip_gpu)
        if "multigpu" in item.keywords and ngpu < 2:
            item.add_marker(skip_multi)


def pytest_terminal_summary(terminalreporter, exitstatus, config):
    """Print every parity margin the GPU tests recorded (tests._cases.MARGINS) and save them to
    gpurun_out/parity_margins.json (the worst error of each test against the 1e-2 contract)."""
    try:
        from tests._cases import MARGINS
    except Exception:  # pragma: no cover
        return
    if not MARGINS:
        return
    import json
    tr = terminalreporter
    tr.write_sep("=", "parity margins (max|gpu-ref|/max|ref| vs the 1e-2 contract; ulps of ref)")
    for m in MARGINS:
        tr.write_line(f"{m.get('test', '?')[:60]:60s} {m.get('key', '')[:26]:26s} err {m['max_rel_err']:.3e} "
                      f"(x{1e-2 / max(m['max_rel_err'], 1e-12):.1f} headroom)  ulps {m.get('max_ulps', float('nan')):.2f}  "
                      f"rn-exact {m.get('frac_rn_exact', float('nan')):.4f}")
    out = ROOT / "gpurun_out"
    out.mkdir(exist_ok=True)
    (out / "parity_margins.json").write_text(json.dumps(MARGINS, indent=1))
