"""Long parity cases: a >= 5000-waypoint path through band (Eqs. 4-6,
PAPER.md:290-316, C10-C14), resampling (C15) and the next waypoint (Alg. 1) at the bench's
max_len / max_smooth, and SURVEY 8(d)'s C2 loop -- 512^2, tick 0 relaxed to the exact fp32 fixed
point, then 200 warm ticks of S = 100 (Alg. 1, C7) -- every tick bit-identical to the oracle
replaying the same poses."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import oracle  # noqa: E402
from paper_1903_07441_b200 import Planner, band_cfg, relax_cfg, warp_cfg  # noqa: E402
from paper_1903_07441_b200 import twg as T  # noqa: E402
from scenes import advance_scene, scene_c2  # noqa: E402

THREADS = oracle.host_cores()


def _stream():
    return torch.cuda.current_stream().cuda_stream


def _long_field(N=2600):
    """A smooth field u = 1 - d / (1.01 d_max) (d = distance to the goal cell centre) on an N x N grid
    with disks of obstacle cells beside the diagonal (four of them touch the walk: Chebyshev distance
    1): the descent walk from (5, 5) is a staircase of ~2N cells that reaches the goal, and the band
    turns it into a diagonal, with the candidates that fall on the disks skipped (C14)."""
    gx, gy = N - 6, N - 6
    yy, xx = np.mgrid[0:N, 0:N].astype(np.float64)
    d = np.hypot(xx - gx, yy - gy)
    u = (1.0 - d / (1.01 * d.max())).astype(np.float32)
    static = np.zeros((N, N), np.uint8)
    for cx, cy, r in ((1000, 1004, 2), (1200, 1205, 3), (700, 703, 1), (1600, 1603, 2), (1500, 1480, 9), (1900, 1920, 12)):
        static[(xx - cx) ** 2 + (yy - cy) ** 2 <= r * r] = 1
    u[static == 1] = 0.0
    u[gy, gx] = 1.0
    cls = static.copy()
    cls[gy, gx] = oracle.GOAL
    raw = np.where(cls == oracle.OBSTACLE, np.float32(0.0), -u).astype(np.float32)
    raw[gy, gx] = 1.0
    return u, cls, static, raw, (gx, gy)


# I = 50 (the bench): k_band_pre with the field box staged in shared memory; I = 64: staged, but the
# boxes of the diagonal runs exceed the tile and read the field from global memory inside the same
# kernel; I = 100: the unstaged instance (I step > 16)
@pytest.mark.parametrize("iters", [50, 64, 100])
def test_long_path_band_resample_next_bit_exact(iters):
    N = 2600
    u, cls, static, raw, goal = _long_field(N)
    max_len, max_smooth = 4 * (N + N), 8 * (N + N)  # the bench's capacities
    pl = Planner(N, N, 1, 0.1, (0.0, 0.0), device=0, stream=_stream())
    pl.set_static(static)
    robot = (5.5 * 0.1, 5.5 * 0.1, 0.0, 0.4)
    pl.set_obstacles(0, robot, goal, np.zeros((0, 20)), warp_cfg(), warm=0)
    pl.set_field(raw)
    st, cells, smooth, ns, nxt = pl.extract_path(0, band_cfg(iters, max_len, max_smooth))
    wst, ref_cells = oracle.walk(cls, u, (5, 5), max_len)
    assert wst == oracle.OK and st == T.OK
    assert len(ref_cells) >= 5000
    assert np.array_equal(cells, ref_cells)
    w = oracle.band(cls, u, oracle.cells_to_waypoints(ref_cells), iters, threads=THREADS)
    sm, cnt = oracle.resample(w)
    k, nx, ny = oracle.next_waypoint(sm)
    assert ns == cnt and smooth.shape == sm.shape
    assert np.abs(smooth - sm).max() <= 1e-4            # the a8/a9 gate
    assert np.array_equal(smooth.view(np.uint32), sm.view(np.uint32))  # bit-exact target (C10)
    assert nxt == (nx, ny)
    # the band moved the staircase (not a fixed point) and never onto an obstacle cell
    assert np.abs(w - oracle.cells_to_waypoints(ref_cells)).max() > 0.2
    wc = np.floor(w).astype(np.int64)
    assert not static[wc[:, 1], wc[:, 0]].any()
    pl.close()


def test_c2_loop_200_ticks_from_the_fixed_point():
    sc0 = scene_c2(0)
    pl = Planner(sc0.W, sc0.H, 1, sc0.cell_size, sc0.origin, device=0, stream=_stream())
    pl.set_static(sc0.static)
    wc, bc = warp_cfg(), band_cfg(50, 4 * 1024, 8 * 1024)
    prev = None
    ok = 0
    for tick in range(201):
        sc = advance_scene(sc0, tick)
        if tick == 0:  # cold, relaxed until the fp32 field stops changing (residual exactly 0)
            rc = relax_cfg(max_sweeps=400000, check_every=1000, tol=1e-38, warm_start=0, sync_every=8)
        else:
            rc = relax_cfg(max_sweeps=100, warm_start=1)
        st, res, cells, sm = pl.plan_step(0, [sc.robot], [sc.goal], sc.tracks, [sc.n_tracks], wc, rc, bc)
        ref = oracle.plan_step(sc, max_sweeps=rc.max_sweeps, check_every=rc.check_every or None, tol=rc.tol,
                               iters=50, max_len=bc.max_len, prev=prev, threads=THREADS)
        prev = ref
        r = res[0]
        if tick == 0:
            assert ref["residual"] == 0.0 and ref["sweeps"] < 400000
        assert r.sweeps == ref["sweeps"] and np.float32(r.residual) == np.float32(ref["residual"]), tick
        assert np.array_equal(pl.get_field(0, 1).view(np.uint32), ref["u"].view(np.uint32)), tick
        assert r.walk_status == ref["walk_status"], tick
        if r.walk_status == T.OK:
            ok += 1
            assert np.array_equal(cells[0, : r.n_cells], ref["cells"]), tick
            got = sm[0, : r.n_smooth]
            assert got.shape == ref["smooth"].shape, tick
            assert np.array_equal(got.view(np.uint32), ref["smooth"].view(np.uint32)), tick
            assert (r.next_x, r.next_y) == ref["next"], tick
    assert ok >= 190  # the warm loop keeps finding its path
    pl.close()


def test_batch_band_more_than_8_scenarios_bit_exact():
    """Batches of more than 8 scenarios take the batch band k_band (1024-waypoint chunks, updates of
    settled waypoints skipped -- DESIGN.md §6): 12 scenarios with imported smooth fields (the
    _long_field construction at 192^2, goal and disks varied per scenario), one warm plan step
    (warm encode, no sweeps -- the imported field is the path's field --, walk, 50 band iterations,
    resampling, next waypoint) against the oracle's walk + band + resample on the same inputs
    (C10-C15)."""
    B, N = 12, 192
    pl = Planner(N, N, B, 0.1, (0.0, 0.0), device=0, stream=_stream())
    yy, xx = np.mgrid[0:N, 0:N].astype(np.float64)
    refs, robots, goals = [], [], []
    for b in range(B):
        gx, gy = N - 6 - 7 * b, N - 20 - 5 * (b % 4)
        d = np.hypot(xx - gx, yy - gy)
        u = (1.0 - d / (1.01 * d.max())).astype(np.float32)
        static = np.zeros((N, N), np.uint8)
        for cx, cy, r in ((60 + 3 * b, 63, 2), (100, 104 + b, 4), (40 + b, 120, 3)):
            static[(xx - cx) ** 2 + (yy - cy) ** 2 <= r * r] = 1
        u[static == 1] = 0.0
        u[gy, gx] = 1.0
        cls = static.copy()
        cls[gy, gx] = oracle.GOAL
        raw = np.where(cls == oracle.OBSTACLE, np.float32(0.0), -u).astype(np.float32)
        raw[gy, gx] = 1.0
        rx, ry = 5 + b, 5 + 2 * b
        robot = ((rx + 0.5) * 0.1, (ry + 0.5) * 0.1, 0.0, 0.4)
        pl.set_static(static, b)
        pl.set_obstacles(b, robot, (gx, gy), np.zeros((0, 20)), warp_cfg(), warm=0)
        pl.set_field(raw, b)
        refs.append((cls, u, (rx, ry)))
        robots.append(robot)
        goals.append((gx, gy))
    bc = band_cfg(50, 4096, 8192)
    st, res, cells, sm = pl.plan_step(-1, robots, goals, np.zeros((0, 20)), [0] * B, warp_cfg(),
                                      relax_cfg(max_sweeps=0, warm_start=1), bc)
    for b, (cls, u, start) in enumerate(refs):
        u1 = u
        assert res[b].sweeps == 0
        wst, ref_cells = oracle.walk(cls, u1, start, 4096)
        assert wst == oracle.OK and res[b].walk_status == 0
        assert np.array_equal(cells[b, : res[b].n_cells], ref_cells)
        w = oracle.band(cls, u1, oracle.cells_to_waypoints(ref_cells), 50, threads=THREADS)
        ref_sm, cnt = oracle.resample(w)
        assert res[b].n_smooth == cnt
        got = sm[b, :cnt]
        assert np.array_equal(got.view(np.uint32), ref_sm.view(np.uint32))
        _k, nx, ny = oracle.next_waypoint(ref_sm)
        assert (res[b].next_x, res[b].next_y) == (nx, ny)
        # the band moved the staircase
        assert np.abs(w - oracle.cells_to_waypoints(ref_cells)).max() > 0.2
    pl.close()
