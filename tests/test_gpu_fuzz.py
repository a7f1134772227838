"""Randomised GPU <-> oracle parity over small scenes (rows a1-a9): random sizes (1..150 per side,
ragged), wall densities, track counts, temporal depths, sweep budgets, band iterations, batch
sizes, warm ticks.  Every field, cell list and smoothed path must be bit-identical."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import oracle  # noqa: E402
from paper_1903_07441_b200 import Planner, band_cfg, relax_cfg, warp_cfg  # noqa: E402
from scenes.gen import Scene  # noqa: E402
from scenes import default_warp_cfg  # noqa: E402


def _random_scene(rng, W, H):
    static = (rng.random((H, W)) < rng.uniform(0.0, 0.25)).astype(np.uint8)
    free = np.argwhere(static == 0)
    if len(free) == 0:
        static[0, 0] = 0
        free = np.argwhere(static == 0)
    gy, gx = free[rng.integers(len(free))]
    ry, rx = free[rng.integers(len(free))]
    n = int(rng.integers(0, 6))
    tracks = np.zeros((n, 20))
    for i in range(n):
        tracks[i, :2] = rng.uniform(0, [W * 0.1, H * 0.1])
        tracks[i, 2:4] = rng.normal(0, 0.3, 2)
        s = rng.choice([0.0025, 0.25])
        tracks[i, 4:] = np.diag([s, s, 4 * s, 4 * s]).reshape(16)
    robot = ((rx + rng.uniform(0.05, 0.95)) * 0.1, (ry + rng.uniform(0.05, 0.95)) * 0.1,
             rng.uniform(-np.pi, np.pi), rng.uniform(0.1, 1.0))
    return Scene("fz", W, H, 0.1, (0.0, 0.0), static, robot, (int(gx), int(gy)), tracks, default_warp_cfg(), 0)


@pytest.mark.parametrize("seed", range(60))
def test_random_plan_steps_bit_exact(seed):
    rng = np.random.default_rng(1000 + seed)
    W, H = int(rng.integers(1, 151)), int(rng.integers(1, 151))
    B = int(rng.integers(1, 4))
    scs = [_random_scene(rng, W, H) for _ in range(B)]
    T = int(rng.integers(1, 9))
    S = int(rng.integers(0, 300))
    iters = int(rng.integers(0, 30))
    pl = Planner(W, H, B, 0.1, (0.0, 0.0), device=0, stream=torch.cuda.current_stream().cuda_stream)
    for b, sc in enumerate(scs):
        pl.set_static(sc.static, b=b)
    max_len = 4 * (W + H) + 8
    rc = relax_cfg(max_sweeps=S, temporal_depth=T, warm_start=1)
    bc = band_cfg(iters, max_len, 8 * max_len)
    prev = [None] * B
    for tick in range(2):  # a cold tick, then a warm one with moved tracks
        if tick:
            for sc in scs:
                if len(sc.tracks):
                    sc.tracks[:, :2] += sc.tracks[:, 2:4] * 0.1
        st, res, cells, sm = pl.plan_step(-1, [s.robot for s in scs], [s.goal for s in scs],
                                          np.concatenate([s.tracks for s in scs]) if B else None,
                                          [s.n_tracks for s in scs], warp_cfg(), rc, bc)
        for b, sc in enumerate(scs):
            ref = oracle.plan_step(sc, max_sweeps=S, iters=iters, max_len=max_len, prev=prev[b])
            assert res[b].sweeps == ref["sweeps"]
            assert np.array_equal(pl.get_field(b, 1), ref["u"]), (seed, tick, b)
            assert res[b].walk_status == ref["walk_status"]
            if ref["walk_status"] == 0:
                assert np.array_equal(cells[b, :res[b].n_cells], ref["cells"])
                n = min(res[b].n_smooth, bc.max_smooth)
                assert np.array_equal(sm[b, :n], ref["smooth"][:n])
            prev[b] = ref
