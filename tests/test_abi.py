"""The C-ABI library builds for sm_100a, loads without a GPU and exports every
symbol include/twg.h declares (no compute calls here)."""
import ctypes
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "twg.h")).read()
    return sorted(set(re.findall(r"TWG_API[^;(]*?\b(twg_\w+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = _declared()
    for n in ("twg_create", "twg_set_obstacles", "twg_relax", "twg_extract_path", "twg_plan_step"):
        assert n in names


def test_library_exports_every_declared_symbol():
    from paper_1903_07441_b200 import build, twg
    build.build()
    L = ctypes.CDLL(twg.LIB_PATH)
    for n in _declared():
        assert hasattr(L, n), n
    assert sorted(n for n, _, _ in twg.SIGNATURES) == _declared()


def test_library_is_sm100a_and_uses_tma():
    from paper_1903_07441_b200 import build, twg
    build.build()
    out = subprocess.run(["cuobjdump", "-lelf", twg.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", twg.LIB_PATH], capture_output=True, text=True).stdout
    assert "UTMALDG" in sass            # TMA tile loads in k_rb_tblock
    assert "HMMA" not in sass           # no legacy tensor-core path (the stencil is not a contraction)


def test_create_without_gpu_fails_cleanly():
    from paper_1903_07441_b200 import twg
    import pytest
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except ImportError:
        pass
    with pytest.raises(twg.TwgError):
        twg.Planner(8, 8)


def test_create_validates_arguments_before_touching_a_device():
    import pytest
    from paper_1903_07441_b200 import twg
    for kw in (dict(width=0, height=8), dict(width=8, height=8, batch=0), dict(width=8, height=8, batch=70000),
               dict(width=8, height=8, cell_size=0.0), dict(width=8, height=8, ghost_rows=4)):
        w, h = kw.pop("width"), kw.pop("height")
        with pytest.raises(twg.TwgError) as e:
            twg.Planner(w, h, **kw)
        assert e.value.status == twg.E_INVALID_ARG
