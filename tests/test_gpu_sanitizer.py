"""Sanitizer tier (SURVEY 4 tier 5, 5): compute-sanitizer memcheck, racecheck, synccheck and initcheck
over a small workload that exercises every kernel family -- the TMA/mbarrier relaxation rings, the
persistent lexicographic wavefront (mode 2), the speculative walkers, the band, the tracker, the
per-cell band and a row-slab group (tools/sanitize_run.py).  Each tool must report 0 errors."""
import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SAN = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck", "initcheck"])
def test_compute_sanitizer(tool):
    if not os.path.exists(SAN):
        pytest.skip("compute-sanitizer not installed")
    env = dict(os.environ, TWG_SANITIZE="1")
    cmd = [SAN, "--tool", tool, "--error-exitcode", "9", "--print-limit", "20", "--target-processes", "all"]
    if tool == "initcheck":
        cmd += ["--track-unused-memory", "no"]
    cmd += [sys.executable, os.path.join(ROOT, "tools", "sanitize_run.py")]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=3000, env=env, cwd=ROOT)
    log = out.stdout + out.stderr
    if "compute-sanitizer is closed" in log:
        pytest.skip("compute-sanitizer is closed on this GPU pool (the pool's wrapper refuses to run it)")
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", f"sanitizer_{tool}.log"), "w") as f:
        f.write(log)
    assert "sanitize workload ok" in log, log[-3000:]
    assert out.returncode == 0 and "ERROR SUMMARY: 0 errors" in log, log[-3000:]
