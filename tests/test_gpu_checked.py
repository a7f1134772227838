"""Checked build (the sanitizer tier's substitute where the GPU pool closes compute-sanitizer): libtwg
compiled with -DTWG_CHECKED turns the device-side bounds checks (TWG_CHECK: stored rows / columns of
the relaxation tiles, band shared-memory runs and path cells, walk cells, stamp boxes) into traps, and
tools/sanitize_run.py -- every kernel family: TMA/mbarrier relaxation rings (packed, goal and scalar
paths), the lexicographic wavefront, Jacobi, speculative walkers, band, tracker, per-cell band, a row-
slab group -- must finish with no failed check and bit-exact results in the smoke part."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_checked_build_runs_clean():
    sys.path.insert(0, ROOT)
    from paper_1903_07441_b200 import build as B
    out = os.path.join(ROOT, "paper_1903_07441_b200", "libtwg_checked.so")
    B.build(out=out, defines=["TWG_CHECKED"])
    env = dict(os.environ, TWG_LIB_PATH=out)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize_run.py")], capture_output=True,
                       text=True, timeout=1200, env=env, cwd=ROOT)
    log = r.stdout + r.stderr
    assert "TWG_CHECK failed" not in log, log[-3000:]
    assert r.returncode == 0 and "sanitize workload ok" in log, log[-3000:]
