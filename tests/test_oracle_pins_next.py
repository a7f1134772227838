"""Pins of the oracle functions behind the SURVEY.md 8(f) rows (no GPU).

P15  f4 ring-time horizon (north_star "the time the robot needs to reach that grid ring").
P16  f3 Jacobi relaxation, Eq. 1, in fp32.
P17  f3 full-grid index matrix M_idx (Eq. 3; Alg. 1).
P18  f3 per-cell warp map (kernel 1; the numbered ellipses of P:438-456).
P19  f4 posterior-covariance footprint ("uncertainty given by Kalman filter at each
     step (Equation 12)").
Expected values come from arithmetic done by hand, closed forms, dense solves, textbook spectral
radii and brute-force definitions, never from re-calling the function under test.
"""
import math

import numpy as np
import pytest

from scenes import random_small_map, default_warp_cfg, Scene


# --------------------------------------------------------------------- P15 (f4)
def test_p15_ring_horizon_arithmetic(orc):
    # ring t at t*w metres, robot at speed s: t*w/s seconds = t*w/(s*dt) Kalman steps
    assert orc.horizon_ring(1, 1.0, 10.0, 0.1) == 1        # 1 m at 10 m/s = 0.1 s = 1 step
    assert orc.horizon_ring(2, 0.5, 2.0, 0.1) == 5         # 1 m at 2 m/s = 0.5 s = 5 steps
    assert orc.horizon_ring(3, 1.0, 0.4, 0.1) == 20        # 75 steps -> clamped to horizon_max
    assert orc.horizon_ring(3, 1.0, 0.4, 0.1, 100) == 75
    assert orc.horizon_ring(1, 1.25, 1.0, 0.5) == 3        # 2.5 -> 3 (half away from zero, C25)
    assert orc.horizon_ring(1, 0.375, 1.0, 0.25) == 2      # 1.5 -> 2
    assert orc.horizon_ring(1, 0.3, 1.0, 0.25) == 1        # 1.2 -> 1
    assert orc.horizon_ring(4, 1.0, 0.0, 0.1) == 20        # robot at rest: never reaches the ring
    assert orc.horizon_ring(4, 1.0, -1.0, 0.1, 7) == 7


def test_p15_ring_horizon_monotone_in_t(orc):
    for s in (0.3, 1.0, 2.7):
        js = [orc.horizon_ring(t, 1.0, s, 0.1, 10_000) for t in range(1, 40)]
        assert all(b >= a for a, b in zip(js, js[1:]))
        assert all(abs(j - t / (s * 0.1)) <= 0.5 + 1e-9 for t, j in zip(range(1, 40), js))


# --------------------------------------------------------------------- P16 (f3)
def test_p16_jacobi_three_by_three_fixed_point(orc):
    # exact: edges u = 1/3, corners 1/6 (e = (1 + 2c)/4, c = e/2)
    cls = np.zeros((3, 3), np.uint8); cls[1, 1] = orc.GOAL
    u = orc.init_u32(cls)
    s, r = orc.relax_jacobi_f32(cls, u, 1000, 1, 1e-30)
    assert r == 0.0 and s < 1000
    assert all(abs(u[y, x] - 1 / 3) <= 6e-8 for x, y in ((1, 0), (0, 1), (2, 1), (1, 2)))
    assert all(abs(u[y, x] - 1 / 6) <= 3e-8 for x, y in ((0, 0), (2, 0), (0, 2), (2, 2)))
    assert u[1, 1] == 1.0


def test_p16_jacobi_first_sweeps_by_hand(orc):
    # 1 x 3 strip: goal at x=0, free x=1,2 (cold start u = 1/2, C5); outside = 0.  Jacobi:
    # sweep 1: ((1 + 1/2)/4, (1/2)/4) = (3/8, 1/8),          residual 3/8
    # sweep 2: ((1 + 1/8)/4, (3/8)/4) = (9/32, 3/32),        residual 3/32
    # sweep 3: ((1 + 3/32)/4, (9/32)/4) = (35/128, 9/128),   residual 3/128
    cls = np.array([[orc.GOAL, 0, 0]], np.uint8)
    u = orc.init_u32(cls)
    assert u.tolist() == [[1.0, 0.5, 0.5]]
    assert orc.relax_jacobi_f32(cls, u, 1) == (1, 0.375) and u.tolist() == [[1.0, 0.375, 0.125]]
    assert orc.relax_jacobi_f32(cls, u, 1) == (1, 3 / 32) and u.tolist() == [[1.0, 9 / 32, 3 / 32]]
    assert orc.relax_jacobi_f32(cls, u, 1) == (1, 3 / 128) and u.tolist() == [[1.0, 35 / 128, 9 / 128]]
    # red-black differs: colour 0 (x=2) first, then x=1 sees its new value:
    # sweep 1 = ((1 + 1/8)/4, (1/2)/4) = (9/32, 1/8)
    v = orc.init_u32(cls)
    orc.relax_f32(cls, v, 1)
    assert v.tolist() == [[1.0, 9 / 32, 1 / 8]]


@pytest.mark.parametrize("seed", range(4))
def test_p16_jacobi_converges_to_dense_solve(orc, seed):
    from test_oracle_pins import _direct_solve
    static, g, _ = random_small_map(300 + seed, 14 + 3 * seed, n_disks=(1, 3), n_walls=(0, 1))
    cls = static.copy(); cls[g[1], g[0]] = orc.GOAL
    u = orc.init_u32(cls)
    orc.relax_jacobi_f32(cls, u, 200_000, 1, 1e-9)
    ref = _direct_solve(cls, orc.init_u64(cls))
    assert np.max(np.abs(u - ref)) < 2e-5


def test_p16_jacobi_spectral_radius_fp32(orc):
    # all-Dirichlet N x N square: Jacobi contraction cos(pi / (N + 1)) per sweep
    N = 16
    cls = np.zeros((N, N), np.uint8)
    u = np.full((N, N), 0.5, np.float32)
    res = [orc.relax_jacobi_f32(cls, u, 1)[1] for _ in range(400)]
    assert abs(res[-1] / res[-2] - math.cos(math.pi / (N + 1))) < 2e-3


@pytest.mark.parametrize("poly", ["affine", "x2-y2", "xy"])
def test_p16_jacobi_discrete_harmonic(orc, poly):
    N = 16
    yy, xx = np.mgrid[0:N, 0:N].astype(np.float64)
    f = {"affine": 0.2 + 0.01 * xx + 0.02 * yy,
         "x2-y2": 0.5 + 0.001 * (xx ** 2 - yy ** 2),
         "xy": 0.1 + 0.002 * xx * yy}[poly]
    cls = np.zeros((N, N), np.uint8)
    cls[0, :] = cls[-1, :] = cls[:, 0] = cls[:, -1] = orc.OBSTACLE
    u = np.where(cls > 0, f, 0.5).astype(np.float32)
    orc.relax_jacobi_f32(cls, u, 100_000, 1, 1e-9)
    assert np.max(np.abs(u - f)) < 2e-6


# --------------------------------------------------------------------- P17 (f3)
def test_p17_index_matrix_three_by_three(orc):
    cls = np.zeros((3, 3), np.uint8); cls[1, 1] = orc.GOAL
    u = np.array([[1 / 6, 1 / 3, 1 / 6], [1 / 3, 1, 1 / 3], [1 / 6, 1 / 3, 1 / 6]], np.float32)
    m = orc.index_matrix(cls, u)
    # edges point at the goal; corners at their larger (equal) neighbours, first in +x,-x,+y,-y
    assert m.tolist() == [[0, 2, 1],
                          [0, 4, 1],
                          [0, 3, 1]]
    cls[0, 0] = orc.OBSTACLE
    assert orc.index_matrix(cls, u)[0, 0] == 5
    one = orc.index_matrix(np.zeros((1, 1), np.uint8), np.zeros((1, 1), np.float32))
    assert one.tolist() == [[6]]


@pytest.mark.parametrize("seed", range(4))
def test_p17_index_matrix_brute_force_and_walk(orc, seed):
    static, g, _ = random_small_map(500 + seed, 24, n_disks=(1, 4), n_walls=(0, 2))
    cls = static.copy(); cls[g[1], g[0]] = orc.GOAL
    u = orc.init_u32(cls)
    orc.relax_f32(cls, u, 20_000, 1, 0.0)
    m = orc.index_matrix(cls, u)
    H, W = cls.shape
    steps = ((1, 0), (-1, 0), (0, 1), (0, -1))
    for y in range(H):
        for x in range(W):
            if cls[y, x] == orc.GOAL:
                assert m[y, x] == 4
                continue
            if cls[y, x] == orc.OBSTACLE:
                assert m[y, x] == 5
                continue
            cand = [(u[y + dy, x + dx], d) for d, (dx, dy) in enumerate(steps)
                    if 0 <= x + dx < W and 0 <= y + dy < H]
            best = max(v for v, _ in cand)
            assert m[y, x] == min(d for v, d in cand if v == best)   # first maximum
    # the descent walk (pinned against BFS reachability, P11) follows M_idx step by step
    free = np.argwhere(cls == 0)
    for (y, x) in free[:: max(1, len(free) // 20)]:
        st, cells = orc.walk(cls, u, (int(x), int(y)), 4 * H * W)
        if st != 0:
            continue
        for (ax, ay), (bx, by) in zip(cells[:-1], cells[1:]):
            dx, dy = steps[m[ay, ax]]
            assert (ax + dx, ay + dy) == (bx, by)


# --------------------------------------------------------------------- P18 (f3)
def _scene(W, H, robot, w=1.0, cs=0.1, origin=(0.0, 0.0)):
    wc = default_warp_cfg()
    wc.warp_spacing = w
    return Scene(name="wm", W=W, H=H, cell_size=cs, origin=origin, static=np.zeros((H, W), np.uint8),
                 robot=robot, goal=(0, 0), tracks=np.zeros((0, 20)), warp=wc, seed=0, truth=None)


def test_p18_warp_map_axis_values(orc):
    # robot at a cell centre heading +x; cell centres on the axis at distance d:
    # ahead r = d / 1.9, behind r = 10 d, t = max(1, ceil(r / w))
    sc = _scene(200, 9, (100.5 * 0.1, 4.5 * 0.1, 0.0, 1.0), w=0.5)
    m = orc.warp_map(sc)
    for k in range(-99, 100):
        d = abs(k) * 0.1
        r = d / 1.9 if k >= 0 else 10.0 * d
        exp = max(1, math.ceil(r / 0.5 - 1e-12))
        got = m[4, 100 + k]
        if abs(r / 0.5 - round(r / 0.5)) > 1e-9:     # skip exact ring boundaries
            assert got == exp, (k, got, exp)


def test_p18_warp_map_rings_nested_and_rotation(orc):
    # rings are nested: along any ray from the robot t never decreases (rays along the 16
    # lattice directions, whose cell centres lie exactly on the ray; robot at a cell centre)
    N = 81
    c0 = N // 2
    c = (c0 + 0.5) * 0.1
    dirs = [(dx, dy) for dx in range(-2, 3) for dy in range(-2, 3)
            if (dx, dy) != (0, 0) and math.gcd(abs(dx), abs(dy)) == 1]
    for th in (0.0, 0.7, math.pi / 2, -2.2):
        m = orc.warp_map(_scene(N, N, (c, c, th, 1.0), w=0.3))
        assert m[c0, c0] == 1
        for dx, dy in dirs:
            ts = [m[c0 + k * dy, c0 + k * dx] for k in range(0, c0 // 2)]
            assert all(b >= a for a, b in zip(ts, ts[1:])), (th, dx, dy, ts)
    # heading +y on a square grid centred on the robot = transpose of heading +x
    a = orc.warp_map(_scene(N, N, (c, c, 0.0, 1.0), w=0.3))
    b = orc.warp_map(_scene(N, N, (c, c, math.pi / 2, 1.0), w=0.3))
    assert np.array_equal(a.T, b)


# --------------------------------------------------------------------- P19 (f4)
def test_p19_posterior_footprint_ignores_horizon(orc):
    # footprint_mode 1: R^2 = max(2 ln 2 sigma^2, rs^2) of the track's own P, whatever j is
    wc = default_warp_cfg()
    sc = _scene(60, 60, (0.55, 0.55, 0.0, 0.4))
    sc.goal = (50, 50)
    s2 = 0.5
    tr = np.zeros((3, 20))
    for i, (x, v) in enumerate(((3.0, 0.4), (4.0, 0.0), (5.0, 0.8))):
        tr[i, :4] = (x, 3.0, v, 0.0)
        tr[i, 4:] = np.diag([s2, s2, 0.01, 0.01]).ravel()
    sc.tracks = tr
    st0, _, _, j0, p0 = orc.classify(sc, 0, 0)
    st1, _, _, j1, p1 = orc.classify(sc, 0, 1)
    assert np.array_equal(j0, j1) and np.array_equal(p0[:, :2], p1[:, :2])
    exp = max(2 * math.log(2) * s2, wc.safety_radius ** 2)
    assert np.allclose(p1[:, 2], exp, rtol=0, atol=1e-12)
    assert np.all(p0[:, 2] >= p1[:, 2] - 1e-12)         # prediction only inflates P (Q >= 0)
    assert np.any(p0[:, 2] > p1[:, 2] + 1e-6)


def test_p19_ring_horizon_in_classify(orc):
    sc = _scene(60, 60, (0.55, 0.55, 0.0, 0.4))
    sc.goal = (50, 50)
    tr = np.zeros((1, 20)); tr[0, :4] = (3.0, 0.55, -0.2, 0.0); tr[0, 4:] = np.eye(4).ravel() * 0.01
    sc.tracks = tr
    _, _, t, j, p = orc.classify(sc, 1, 0)
    # ahead along the heading at d = 2.45 m: r = d / 1.9, t = ceil(r), j = round(t w / (s dt))
    d = 3.0 - 0.55
    tt = math.ceil(d / 1.9)
    assert t[0] == tt
    assert j[0] == min(20, round(tt * sc.warp.warp_spacing / (0.4 * sc.warp.dt)))
    assert abs(p[0, 0] - (3.0 - 0.2 * j[0] * sc.warp.dt)) < 1e-12


# --------------------------------------------------------------------- P24 (f3 lexicographic)
def test_p24_lex_first_sweeps_by_hand(orc):
    # 1 x 3 strip, goal at x=0, cold 1/2: x=1 sees the goal (W) and the old 1/2 (E): 3/8; x=2 sees
    # the new 3/8 (W): 3/32.  Sweep 2: x=1: (1 + 3/32)/4 = 35/128; x=2: (35/128)/4 = 35/512.
    cls = np.array([[orc.GOAL, 0, 0]], np.uint8)
    u = orc.init_u32(cls)
    assert orc.relax_lex_f32(cls, u, 1) == (1, 0.40625) and u.tolist() == [[1.0, 0.375, 0.09375]]
    s, r = orc.relax_lex_f32(cls, u, 1)
    assert u.tolist() == [[1.0, 35 / 128, 35 / 512]] and r == pytest.approx(0.375 - 35 / 128, abs=0)
    # a 2 x 2 block: (0,0) goal; (1,0) from W=1 (new), S old 1/2; (0,1) from N=1 (new), E old 1/2;
    # (1,1) from W, N new: ((0 + 3/8) + (3/8 + 0)) / 4 = 3/16
    cls = np.zeros((2, 2), np.uint8); cls[0, 0] = orc.GOAL
    u = orc.init_u32(cls)
    orc.relax_lex_f32(cls, u, 1)
    assert u.tolist() == [[1.0, 0.375], [0.375, 0.1875]]


@pytest.mark.parametrize("seed", range(3))
def test_p24_lex_converges_to_dense_solve(orc, seed):
    from test_oracle_pins import _direct_solve
    static, g, _ = random_small_map(700 + seed, 16 + 4 * seed, n_disks=(1, 3), n_walls=(0, 1))
    cls = static.copy(); cls[g[1], g[0]] = orc.GOAL
    u = orc.init_u32(cls)
    orc.relax_lex_f32(cls, u, 100_000, 1, 1e-9)
    ref = _direct_solve(cls, orc.init_u64(cls))
    assert np.max(np.abs(u - ref)) < 2e-5


def test_p24_lex_spectral_radius(orc):
    # lexicographic Gauss-Seidel contracts by cos^2(pi / (N + 1)) per sweep (model problem)
    N = 16
    cls = np.zeros((N, N), np.uint8)
    u = np.full((N, N), 0.5, np.float32)
    res = [orc.relax_lex_f32(cls, u, 1)[1] for _ in range(200)]
    assert abs(res[-1] / res[-2] - math.cos(math.pi / (N + 1)) ** 2) < 2e-3


# --------------------------------------------------------------------- P25 (O8 resample / next waypoint)
def test_p25_resample_and_next_waypoint_by_hand(orc):
    # C15: a segment of length l becomes ceil(max(l, 1)) equal sub-steps, the last waypoint appended
    w = np.array([[0.5, 0.5], [3.0, 0.5], [3.0, 1.0]], np.float32)
    pts, cnt = orc.resample(w)
    # segment 1: l = 2.5 -> 3 sub-steps of 5/6; segment 2: l = 0.5 -> 1 sub-step; + last
    exp = [[0.5, 0.5], [0.5 + 2.5 / 3, 0.5], [0.5 + 5.0 / 3, 0.5], [3.0, 0.5], [3.0, 1.0]]
    assert cnt == 5 and np.allclose(pts, exp, atol=1e-6)
    # a9: the first resampled point >= 1 cell from the first one: (0.5 + 5/3, 0.5) at distance 1.67
    k, nx, ny = orc.next_waypoint(pts)
    assert k == 2 and abs(nx - (0.5 + 5.0 / 3)) < 1e-6 and ny == 0.5
    # all within 1 cell: the last point (the goal)
    k, nx, ny = orc.next_waypoint(np.array([[0.5, 0.5], [1.0, 0.5], [1.2, 0.9]], np.float32))
    assert (nx, ny) == (np.float32(1.2), np.float32(0.9))
    # exactly 1 cell away counts (>= 1)
    k, nx, ny = orc.next_waypoint(np.array([[0.5, 0.5], [1.0, 0.5], [1.5, 0.5], [9.5, 0.5]], np.float32))
    assert k == 2 and (nx, ny) == (1.5, 0.5)


# --------------------------------------------------------------------- P26 (C7 warm start)
def test_p26_warm_init_by_hand(orc):
    # C7: free cells keep the previous value, including a cell that was an obstacle last tick
    # (u = 0); a released goal restarts at u = 0 like a released obstacle (it must not stay a free
    # cell at the maximum u = 1: that is a spurious maximum, the descent-walk trap C7 avoids);
    # fixed cells take their class value (goal 1, obstacle 0)
    prev = np.array([[0.375, 0.0, 1.0], [0.75, 0.25, 0.125]], np.float32)
    cls_prev = np.array([[0, 1, 2], [0, 0, 0]], np.uint8)
    cls = np.array([[0, 0, 0], [1, 2, 0]], np.uint8)   # the old obstacle (0,1) and goal (0,2) are free now
    u = orc.init_u32(cls, prev, cls_prev)
    assert u.tolist() == [[0.375, 0.0, 0.0], [0.0, 1.0, 0.125]]
    # without the previous class grid nothing is known to be released: every free cell keeps its value
    assert orc.init_u32(cls, prev).tolist() == [[0.375, 0.0, 1.0], [0.0, 1.0, 0.125]]
    # a goal that stays put is re-fixed at 1
    assert orc.init_u32(cls_prev, prev, cls_prev).tolist() == [[0.375, 0.0, 1.0], [0.75, 0.25, 0.125]]
    # cold: free 0.5
    assert orc.init_u32(cls).tolist() == [[0.5, 0.5, 0.5], [0.0, 1.0, 0.5]]


# --------------------------------------------------------------------- P27 (f3 per-cell band, C37)
def test_p27_cellband_2x2_by_hand(orc):
    # goal (1,1); u(1,0) = 0.5, u(0,1) = 0.4, u(0,0) = 0.25.  Eq. 3: M(0,0) = +x (0.5 > 0.4).
    # Per-cell band (Alg. 1, reading C37), k_t = 1, cell (0,0):
    #   n = (1,0): F = 1/0.5 - 1/0.25 = -2, M(n) = goal -> R = (-F - 1, 1) = (1, 1), |R|^2 = 2
    #   n = (0,1): F = 1/0.4 - 1/0.25 = -1.5, M(n) = goal -> R = (1, -F - 1) = (1, 0.5), |R|^2 = 1.25
    # so (0,0) switches to +y (code 2); (1,0) and (0,1) point at the goal with R = 0 and keep it.
    cls = np.array([[0, 0], [0, orc.GOAL]], np.uint8)
    u = np.array([[0.25, 0.5], [0.4, 1.0]], np.float32)
    m = orc.index_matrix(cls, u)
    assert m.tolist() == [[0, 2], [0, 4]]
    b = orc.cellband(cls, u, m, iters=1)
    assert b.tolist() == [[2, 2], [0, 4]]
    st, cells = orc.walk_dir(b, (0, 0), 10)
    assert st == orc.OK and cells.tolist() == [[0, 0], [0, 1], [1, 1]]
    # more iterations change nothing (a fixed point), I = 0 is the identity
    assert np.array_equal(orc.cellband(cls, u, m, iters=5), b)
    assert np.array_equal(orc.cellband(cls, u, m, iters=0), m)


def test_p27_cellband_3x3_centre_goal_is_a_fixed_point(orc):
    # the exact fixed point of P5 (edges u = 1/3, corners 1/6): an edge keeps the goal (|R|^2 = (3 - 2)^2
    # = 1 against (6 - 3 + 2)^2 = 25 for a corner), a corner's two candidates tie (both |R|^2 =
    # (F + 1)^2 + 1) and the current successor is kept
    cls = np.zeros((3, 3), np.uint8)
    cls[1, 1] = orc.GOAL
    u = orc.init_u32(cls)
    orc.relax_f32(cls, u, 1000, 1, 0.0)
    m = orc.index_matrix(cls, u)
    assert np.array_equal(orc.cellband(cls, u, m, iters=10), m)


def test_p27_cellband_straight_corridor_unchanged(orc):
    # a 1-wide corridor: every cell's only alternatives are walls or the cell behind it, whose
    # tensions point forward (2 k_t) -- the matrix stays the steepest-ascent one
    W = 12
    cls = np.ones((3, W), np.uint8)
    cls[1, :] = 0
    cls[1, W - 1] = orc.GOAL
    u = orc.init_u32(cls)
    orc.relax_f32(cls, u, 10000, 1, 0.0)
    m = orc.index_matrix(cls, u)
    assert (m[1, :W - 1] == 0).all()
    assert np.array_equal(orc.cellband(cls, u, m, iters=50), m)


def test_p27_cellband_properties_random_maps(orc):
    # on random converged maps: goal / obstacle / successor-less codes never change, every code the band
    # changed points at an in-grid non-obstacle neighbour (Eq. 3's own choice may be an obstacle in a
    # goal-less region, u = 0, which the band skips); the walk along Eq. 3's matrix is the implicit walk
    rng = np.random.default_rng(27)
    for trial in range(20):
        H, W = int(rng.integers(5, 30)), int(rng.integers(5, 30))
        cls = (rng.random((H, W)) < 0.15).astype(np.uint8)
        gy, gx = int(rng.integers(0, H)), int(rng.integers(0, W))
        cls[gy, gx] = orc.GOAL
        u = orc.init_u32(cls)
        orc.relax_f32(cls, u, 3000, 1, 0.0)
        m = orc.index_matrix(cls, u)
        b = orc.cellband(cls, u, m, iters=int(rng.integers(1, 20)), kt=float(rng.choice([0.5, 1.0, 2.0])))
        assert np.array_equal(b[m > 3], m[m > 3])
        ys, xs = np.nonzero((b <= 3) & (b != m))
        dx = np.array([1, -1, 0, 0])[b[ys, xs]]
        dy = np.array([0, 0, 1, -1])[b[ys, xs]]
        nx, ny = xs + dx, ys + dy
        assert ((nx >= 0) & (nx < W) & (ny >= 0) & (ny < H)).all()
        assert (cls[ny, nx] != orc.OBSTACLE).all()
        free = np.argwhere(cls == 0)
        sy, sx = free[int(rng.integers(0, len(free)))]
        st1, c1 = orc.walk(cls, u, (int(sx), int(sy)), 4 * W * H)
        st2, c2 = orc.walk_dir(m, (int(sx), int(sy)), 4 * W * H)
        assert st1 == st2 and np.array_equal(c1, c2)
