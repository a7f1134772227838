"""Pins of the CPU oracle against what the paper and mathematics fix (no GPU).

Each test names the pin of DESIGN.md "Oracle pins" (= SURVEY.md 8(c) P1-P14)
and the passage it follows.  None of these re-calls an oracle formula to
produce its expected value: expectations come from closed forms, the paper's
implicit equations, library linear solvers, brute force, textbook spectral
radii, or an independent implementation (golden fixture).
"""
import hashlib
import json
import math
import os
from collections import deque

import numpy as np
import pytest

from scenes import scene_c1, random_small_map, annulus_fixed, default_warp_cfg

GOLD = os.path.join(os.path.dirname(__file__), "golden")


# --------------------------------------------------------------------- P1 (O1)
def _eq14(xr, yr, th, xo, yo, rx):
    """PAPER.md:458-465 Eq. 14 with x_c = x_r + 0.9 r_x cos(theta), r_y = r_x / 4."""
    c, s = math.cos(th), math.sin(th)
    xc, yc = xr + 0.9 * rx * c, yr + 0.9 * rx * s
    ry = rx / 4.0
    A = c * (xo - xc) + s * (yo - yc)
    B = s * (xo - xc) - c * (yo - yc)
    return A * A / (rx * rx) + B * B / (ry * ry)


def test_p1_closed_form_satisfies_eq14(orc):
    rng = np.random.default_rng(1)
    worst = 0.0
    for _ in range(20000):
        xr, yr, xo, yo = rng.uniform(-50, 50, 4)
        th = rng.uniform(-math.pi, math.pi)
        r = orc.warp_radius(xr, yr, th, xo, yo)
        assert r >= 0.0
        worst = max(worst, abs(_eq14(xr, yr, th, xo, yo, r) - 1.0))
    assert worst < 1e-12


def test_p1_spec_examples(orc):
    # r = 0 at the robot; r = d / 1.9 straight ahead; r = 1 at (0.9, 0.25)
    assert orc.warp_radius(0, 0, 0.0, 0, 0) == 0.0
    assert abs(orc.warp_radius(0, 0, 0.0, 1.9, 0.0) - 1.0) < 1e-12
    assert abs(orc.warp_radius(0, 0, 0.0, 0.9, 0.25) - 1.0) < 1e-12
    for d in (0.5, 1.0, 3.7):
        assert abs(orc.warp_radius(0, 0, 0.0, d, 0.0) - d / 1.9) < 1e-12     # ahead: r = d - 0.9 r
        assert abs(orc.warp_radius(0, 0, 0.0, -d, 0.0) - 10.0 * d) < 1e-12  # behind: r = d + 0.9 r


def test_p1_monotone_ahead_label_decreases_frame_invariant(orc):
    prev = -1.0
    for d in np.linspace(0.01, 30, 300):
        r = orc.warp_radius(0, 0, 0.0, d, 0.0)
        assert r > prev
        prev = r
    # PAPER.md:436 "if an obstacle moves towards the robot, its label decreases"
    labels = [orc.warp_number(orc.warp_radius(0, 0, 0.0, d, 0.0), 1.0) for d in np.linspace(20, 0, 200)]
    assert all(a >= b for a, b in zip(labels, labels[1:]))
    rng = np.random.default_rng(3)
    for _ in range(500):
        xr, yr, xo, yo, tx, ty = rng.uniform(-20, 20, 6)
        th, rot = rng.uniform(-math.pi, math.pi, 2)
        c, s = math.cos(rot), math.sin(rot)
        R = lambda x, y: (c * x - s * y + tx, s * x + c * y + ty)
        a = orc.warp_radius(xr, yr, th, xo, yo)
        b = orc.warp_radius(*R(xr, yr), th + rot, *R(xo, yo))
        assert abs(a - b) <= 1e-9 * max(1.0, a)


# --------------------------------------------------------------------- P2 (O1-O2)
def test_p2_warp_number_and_horizon(orc):
    # SPEC.md:350-352
    assert orc.warp_number(0.0, 1.0) == 1
    assert orc.warp_number(1.0, 1.0) == 1
    assert orc.warp_number(2.3, 1.0) == 3
    # SPEC.md:359-361 (Eq. 16 "v is the ratio of the velocity of the robot to the moving obstacle")
    assert orc.horizon(3, 0.4, 0.4, 0.0) == 3
    assert orc.horizon(4, 0.4, 0.0, 0.8) == 2
    # near-stationary: v = 0.4 / 0.05 = 8, t = 3 -> 24 -> clamped to horizon_max = 20
    assert orc.horizon(3, 0.4, 0.001, 0.0, 0.05, 20) == 20
    assert orc.horizon(1, 0.4, 0.0, 0.0, 0.05, 20) == 8
    # half away from zero (C25): v t = 2.5 -> 3
    assert orc.horizon(5, 0.25, 0.5, 0.0) == 3


# --------------------------------------------------------------------- P3 (O2)
def _A(dt):
    A = np.eye(4)
    A[0, 2] = A[1, 3] = dt
    return A


def test_p3_predict_constant_velocity(orc):
    x, P = orc.predict([0, 0, 1, 0], np.eye(4), np.zeros(16), 0.1, 5)
    assert np.allclose(x, [0.5, 0, 1, 0], atol=1e-15)
    _, P1 = orc.predict([0, 0, 0, 0], np.eye(4), np.zeros(16), 0.1, 1)
    A = np.array([[1, 0, .1, 0], [0, 1, 0, .1], [0, 0, 1, 0], [0, 0, 0, 1]])
    assert np.allclose(P1, A @ A.T, atol=1e-15)


def test_p3_predict_closed_form_and_composition(orc):
    rng = np.random.default_rng(7)
    for _ in range(50):
        dt = rng.uniform(0.01, 0.5)
        j = int(rng.integers(0, 25))
        x = rng.normal(size=4)
        M = rng.normal(size=(4, 4)); P = M @ M.T
        N = rng.normal(size=(4, 4)); Q = 1e-2 * (N @ N.T)
        xo, Po = orc.predict(x, P, Q, dt, j)
        # closed form P_j = A^j P A^jT + sum_{m<j} A^m Q A^mT, A^m = [[I, m dt I], [0, I]]
        Am = lambda m: _A(m * dt)
        ref = Am(j) @ P @ Am(j).T + sum((Am(m) @ Q @ Am(m).T for m in range(j)), np.zeros((4, 4)))
        assert np.allclose(xo, Am(j) @ x, rtol=1e-12, atol=1e-12)
        assert np.allclose(Po, ref, rtol=1e-11, atol=1e-12)
        a = int(rng.integers(0, 10)); b = int(rng.integers(0, 10))
        xa, Pa = orc.predict(x, P, Q, dt, a)
        xab, Pab = orc.predict(xa, Pa, Q, dt, b)
        xs, Ps = orc.predict(x, P, Q, dt, a + b)
        assert np.allclose(xab, xs, rtol=1e-12, atol=1e-12)
        assert np.allclose(Pab, Ps, rtol=1e-11, atol=1e-12)


def test_p3_footprint_gaussian_threshold(orc):
    # marked iff Gaussian >= 1/2 or within the safety distance.
    rng = np.random.default_rng(11)
    for _ in range(200):
        s2 = rng.uniform(0.001, 4.0)
        P = np.diag([s2 * rng.uniform(0.5, 1.5), 0, 0, 0.0])
        P[1, 1] = 2 * s2 - P[0, 0]
        rs = rng.uniform(0.0, 1.0)
        R2 = orc.footprint_r2(P, rs)
        sig2 = s2
        for d in rng.uniform(0, 4, 50):
            if abs(d * d - R2) < 1e-9:
                continue
            marked = math.exp(-d * d / (2 * sig2)) >= 0.5 or d <= rs
            assert marked == (d * d <= R2)


# --------------------------------------------------------------------- P4 (O3)
def test_p4_nine_cell_disk_and_box_equals_bruteforce(orc):
    # sigma -> 0, r_s = 0.15 m, 0.1 m cells, centre on a cell centre -> exactly 9 cells
    R2 = orc.footprint_r2(np.zeros(16), 0.15)
    m = orc.stamp_disk(32, 32, 0.1, 0.0, 0.0, 1.05, 1.05, R2)
    assert m.sum() == 9
    ys, xs = np.nonzero(m)
    assert set(zip(xs.tolist(), ys.tolist())) == {(x, y) for x in (9, 10, 11) for y in (9, 10, 11)}
    rng = np.random.default_rng(5)
    for _ in range(300):
        W, H = int(rng.integers(1, 60)), int(rng.integers(1, 60))
        cs = rng.uniform(0.05, 0.3)
        ox, oy = rng.uniform(-2, 2, 2)
        xp, yp = rng.uniform(-3, 3 + W * cs), rng.uniform(-3, 3 + H * cs)
        R2 = rng.uniform(0, 3) ** 2
        a = orc.stamp_disk(W, H, cs, ox, oy, xp, yp, R2, brute=True)
        b = orc.stamp_disk(W, H, cs, ox, oy, xp, yp, R2, brute=False)
        assert np.array_equal(a, b)


def _scene_with_tracks(tracks, goal=(30, 30), robot=(0.55, 0.55, 0.0, 0.4), N=40):
    from scenes.gen import Scene
    return Scene("t", N, N, 0.1, (0.0, 0.0), np.zeros((N, N), np.uint8), robot, goal,
                 np.asarray(tracks, np.float64).reshape(-1, 20), default_warp_cfg(), 0)


def test_p4_union_idempotent_goal_survives_robot_exempt(orc):
    P = np.diag([0.0025, 0.0025, 0.01, 0.01]).reshape(16)
    trk = np.concatenate([[2.0, 2.0, 0.0, 0.0], P])
    st1, c1, *_ = orc.classify(_scene_with_tracks([trk]))
    st2, c2, *_ = orc.classify(_scene_with_tracks([trk, trk]))
    assert st1 == st2 == 0 and np.array_equal(c1, c2) and (c1 == 1).sum() > 0
    # footprint centred on the goal: goal survives, warning returned
    on_goal = np.concatenate([[3.05, 3.05, 0.0, 0.0], P])
    st, c, *_ = orc.classify(_scene_with_tracks([on_goal]))
    assert st == orc.W_GOAL_SWALLOWED and c[30, 30] == orc.GOAL and c[30, 31] == orc.OBSTACLE
    # footprint over the robot: robot cell stays free (C22)
    on_robot = np.concatenate([[0.55, 0.55, 0.0, 0.0], P])
    st, c, *_ = orc.classify(_scene_with_tracks([on_robot]))
    assert c[5, 5] == orc.FREE and c[5, 6] == orc.OBSTACLE


def test_p4_validation_errors(orc):
    sc = _scene_with_tracks(np.zeros((0, 20)), goal=(40, 3))
    assert orc.classify(sc)[0] == orc.E_OUT_OF_BOUNDS
    sc = _scene_with_tracks(np.zeros((0, 20)))
    sc.static[30, 30] = 1
    assert orc.classify(sc)[0] == orc.E_OVERLAPPING
    sc = _scene_with_tracks(np.zeros((0, 20)))
    sc.static[5, 5] = 1
    assert orc.classify(sc)[0] == orc.E_INVALID_START


# --------------------------------------------------------------------- P5 (O4-O5, O6)
def test_p5_three_by_three_exact_fixed_point(orc):
    cls = np.zeros((3, 3), np.uint8); cls[1, 1] = orc.GOAL
    # exact phi: edges 2/3, corners 5/6 (e = (2c + 1)/4, c = (e + 1)/2) -> u = 1/3, 1/6
    u = orc.init_u32(cls)
    s, r = orc.relax_f32(cls, u, 1000, 1, 1e-30)
    assert s == 14 and r == 0.0
    assert all(u[y, x] == np.float32(1 / 3) for x, y in ((1, 0), (0, 1), (2, 1), (1, 2)))
    assert all(u[y, x] == np.float32(1 / 6) for x, y in ((0, 0), (2, 0), (0, 2), (2, 2)))
    u64 = orc.init_u64(cls)
    s, r = orc.relax_f64(cls, u64, 1000, 1, 1e-300)
    assert s == 28 and r == 0.0
    assert abs(u64[0, 1] - 1 / 3) < 1e-15 and abs(u64[0, 0] - 1 / 6) < 1e-15
    st, cells = orc.walk(cls, u, (0, 0), 10)
    assert st == 0 and cells.tolist() == [[0, 0], [1, 0], [1, 1]]  # SPEC.md:152, tie -> +x


def test_p5_zero_sweeps_and_all_fixed(orc):
    cls = np.ones((5, 5), np.uint8); cls[2, 2] = orc.GOAL
    u = orc.init_u32(cls)
    assert orc.relax_f32(cls, u, 10) == (10, 0.0)            # nothing to relax
    cls = np.zeros((5, 5), np.uint8); cls[0, 0] = orc.GOAL
    u = orc.init_u32(cls); u0 = u.copy()
    assert orc.relax_f32(cls, u, 0) == (0, 0.0) and np.array_equal(u, u0)


# --------------------------------------------------------------------- P6 (O4)
def _direct_solve(cls, fixed_u):
    """Dense direct solve of the 5-point Laplace system (outside the grid u = 0)."""
    H, W = cls.shape
    idx = -np.ones((H, W), int)
    free = np.argwhere(cls == 0)
    for k, (y, x) in enumerate(free):
        idx[y, x] = k
    n = len(free)
    A = np.zeros((n, n)); b = np.zeros(n)
    for k, (y, x) in enumerate(free):
        A[k, k] = 4.0
        for yy, xx in ((y, x + 1), (y, x - 1), (y + 1, x), (y - 1, x)):
            if 0 <= yy < H and 0 <= xx < W:
                if idx[yy, xx] >= 0:
                    A[k, idx[yy, xx]] -= 1.0
                else:
                    b[k] += fixed_u[yy, xx]
    sol = np.linalg.solve(A, b)
    out = fixed_u.astype(np.float64).copy()
    out[cls == 0] = sol
    return out


@pytest.mark.parametrize("seed", range(6))
def test_p6_converged_equals_dense_solve(orc, seed):
    rng = np.random.default_rng(seed)
    N = int(rng.integers(8, 25))
    static, g, _ = random_small_map(100 + seed, N, n_disks=(1, 3), n_walls=(0, 1))
    cls = static.copy(); cls[g[1], g[0]] = orc.GOAL
    u = orc.init_u64(cls)
    orc.relax_f64(cls, u, 2_000_000, 1, 1e-14)
    ref = _direct_solve(cls, orc.init_u64(cls))
    assert np.max(np.abs(u - ref)) < 1e-9


def test_p6_spec_16x16_corner_goal(orc):
    # 16 x 16, one goal corner cell, tol 1e-12 -> dense solve within 1e-9
    cls = np.zeros((16, 16), np.uint8); cls[0, 0] = orc.GOAL
    u = orc.init_u64(cls)
    orc.relax_f64(cls, u, 100000, 1, 1e-12)
    ref = _direct_solve(cls, orc.init_u64(cls))
    assert np.max(np.abs(u - ref)) < 1e-9


# --------------------------------------------------------------------- P7 (O4-O5)
def test_p7_spectral_radius_red_black_and_jacobi(orc):
    N = 16
    cls = np.zeros((N, N), np.uint8)         # all free, outside = 0 (all-Dirichlet)
    u = np.full((N, N), 0.5)
    res = []
    for _ in range(600):
        res.append(orc.relax_f64(cls, u, 1)[1])
    rb = res[-1] / res[-2]
    assert abs(rb - math.cos(math.pi / (N + 1)) ** 2) < 1e-8
    u = np.full((N, N), 0.5)
    res = []
    for _ in range(1500):
        res.append(orc.jacobi_f64(cls, u, 1)[1])
    jr = res[-1] / res[-2]
    assert abs(jr - math.cos(math.pi / (N + 1))) < 1e-8


# --------------------------------------------------------------------- P8 (O4)
@pytest.mark.parametrize("poly", ["affine", "x2-y2", "xy", "cubic"])
def test_p8_discrete_harmonic_polynomials(orc, poly):
    N = 20
    yy, xx = np.mgrid[0:N, 0:N].astype(np.float64)
    f = {"affine": 0.2 + 0.01 * xx + 0.02 * yy,
         "x2-y2": 0.5 + 0.001 * (xx ** 2 - yy ** 2),
         "xy": 0.1 + 0.002 * xx * yy,
         "cubic": 0.5 + 1e-4 * (xx ** 3 - 3 * xx * yy ** 2)}[poly]
    cls = np.zeros((N, N), np.uint8)
    cls[0, :] = cls[-1, :] = cls[:, 0] = cls[:, -1] = orc.OBSTACLE   # fixed ring carries the data
    u = np.where(cls > 0, f, 0.5).astype(np.float64)
    orc.relax_f64(cls, u, 200000, 1, 1e-15)
    assert np.max(np.abs(u - f)) < 1e-12


# --------------------------------------------------------------------- P9 (O4)
def _annulus_stats(orc, N):
    goal, obst, r = annulus_fixed(N)
    cls = np.zeros((N, N), np.uint8)
    cls[obst] = orc.OBSTACLE
    cls[goal] = orc.GOAL
    u = orc.init_u64(cls)
    orc.relax_f64(cls, u, 5_000_000, 16, 1e-13)
    r1, r2 = 0.1 * N, 0.45 * N
    exact = np.log(r2 / r) / np.log(r2 / r1)         # u = ln(r2/r)/ln(r2/r1)
    free = cls == 0
    A = np.vstack([np.log(r[free]), np.ones(free.sum())]).T
    (slope, icpt), *_ = np.linalg.lstsq(A, u[free], rcond=None)
    inner = free & (r >= r1 + 0.1 * N) & (r <= r2 - 0.1 * N)
    return (abs(slope + 1 / np.log(4.5)), np.max(np.abs(u - exact)[inner]),
            np.max(np.abs(A @ [slope, icpt] - u[free])))


@pytest.mark.slow
def test_p9_annulus_log_solution(orc):
    s64 = _annulus_stats(orc, 64)
    s128 = _annulus_stats(orc, 128)
    # SURVEY.md App. A chk9 (exact discrete solve): N=64: 0.0395, 2.3e-2, 2.2e-2; N=128: 0.0114, 4.9e-3, 9.1e-3
    assert s128[0] < 1.5e-2 and s128[1] < 6e-3 and s128[2] < 1e-2
    assert all(b < a for a, b in zip(s64, s128))


# --------------------------------------------------------------------- P10 (O4, O6)
def _goal_component(cls, g):
    H, W = cls.shape
    seen = np.zeros_like(cls, bool)
    q = deque([g]); seen[g[1], g[0]] = True
    while q:
        x, y = q.popleft()
        for xx, yy in ((x + 1, y), (x - 1, y), (x, y + 1), (x, y - 1)):
            if 0 <= xx < W and 0 <= yy < H and not seen[yy, xx] and cls[yy, xx] != 1:
                seen[yy, xx] = True
                q.append((xx, yy))
    return seen


def test_p10_maximum_principle(orc):
    for seed in range(50):
        static, g, _ = random_small_map(seed, 32)
        cls = static.copy(); cls[g[1], g[0]] = orc.GOAL
        u = orc.init_u64(cls)
        orc.relax_f64(cls, u, 2_000_000, 8, 1e-13)
        comp = _goal_component(cls, g)
        H, W = cls.shape
        for y, x in np.argwhere((cls == 0) & comp):
            nb = [u[yy, xx] if 0 <= xx < W and 0 <= yy < H else 0.0
                  for xx, yy in ((x + 1, y), (x - 1, y), (x, y + 1), (x, y - 1))]
            assert max(nb) > u[y, x] > min(nb)            # no interior extremum
        far = (cls == 0) & ~comp
        assert np.all(u[far] < 1e-9)                      # goal-less components -> 0


def test_p10_range_after_every_sweep_fp32(orc):
    static, g, _ = random_small_map(77, 40)
    cls = static.copy(); cls[g[1], g[0]] = orc.GOAL
    u = orc.init_u32(cls)
    for _ in range(300):
        orc.relax_f32(cls, u, 1)
        assert u.min() >= 0.0 and u.max() <= 1.0


# --------------------------------------------------------------------- P11 (O6)
def test_p11_walk_equals_bfs_reachability(orc):
    found = 0
    for seed in range(60):
        static, g, s = random_small_map(1000 + seed, 48)
        cls = static.copy(); cls[g[1], g[0]] = orc.GOAL
        u64 = orc.init_u64(cls)
        orc.relax_f64(cls, u64, 3_000_000, 16, 1e-14)
        u = u64.astype(np.float32)
        st, cells = orc.walk(cls, u, s, 48 * 48)
        reach = _goal_component(cls, g)[s[1], s[0]]
        assert (st == 0) == bool(reach)
        if st == 0:
            found += 1
            vals = [u[y, x] for x, y in cells]
            assert all(b > a for a, b in zip(vals, vals[1:]))   # strictly ascending u
            assert tuple(cells[-1]) == g
            steps = np.abs(np.diff(cells, axis=0)).sum(axis=1)
            assert np.all(steps == 1)
    assert found >= 40


def test_p11_degenerate_walks(orc):
    cls = np.zeros((5, 5), np.uint8); cls[2, 2] = orc.GOAL
    u = orc.init_u32(cls); orc.relax_f32(cls, u, 100)
    assert orc.walk(cls, u, (2, 2), 1)[1].tolist() == [[2, 2]]       # start = goal
    assert orc.walk(cls, u, (0, 0), 2)[0] == orc.E_NO_PATH          # longer than max_len
    cls = np.zeros((9, 9), np.uint8); cls[8, 8] = orc.GOAL
    cls[0:3, 2] = 1; cls[2, 0:3] = 1                                 # enclosed start
    u = orc.init_u32(cls); orc.relax_f32(cls, u, 500)
    st, cells = orc.walk(cls, u, (0, 0), 81)
    assert st == orc.E_NO_PATH and len(cells) == 0


# --------------------------------------------------------------------- P12 (O4)
def test_p12_jacobi_and_red_black_share_fixed_point(orc):
    static, g, _ = random_small_map(9, 20, n_disks=(1, 3))
    cls = static.copy(); cls[g[1], g[0]] = orc.GOAL
    a = orc.init_u64(cls); orc.relax_f64(cls, a, 1_000_000, 1, 1e-14)
    b = orc.init_u64(cls); orc.jacobi_f64(cls, b, 4_000_000, 1e-14)
    assert np.max(np.abs(a - b)) < 1e-9


# --------------------------------------------------------------------- P13 (O7)
def _plen(w):
    return float(np.sum(np.hypot(*np.diff(np.asarray(w, np.float64), axis=0).T)))


def test_p13_eq6_on_linear_field(orc):
    # u = a + b (x - 0.5) along x is reproduced exactly by bilinear interpolation, so one band
    # step can be predicted by hand from Eqs. 4-6 and the tension law (C11).
    N = 16
    a, b = 0.02, 0.05
    u = np.tile((a + b * np.arange(N)).astype(np.float32), (N, 1))
    cls = np.zeros((N, N), np.uint8)
    for x in (3.3, 7.6, 10.1):
        assert abs(orc.bilerp(u, x, 8.2) - (a + b * (x - 0.5))) < 1e-6
    # chain (1,8) - (2.5,9) - (4,8): the tensions alone pick (2.5, 8.75); with the potential
    # force of Eq. 6 the minimum resultant moves to (2.25, 8.75).
    w = np.array([[1.0, 8.0], [2.5, 9.0], [4.0, 8.0]], np.float32)
    out = orc.band(cls, u, w, iters=1, step=0.25)

    def hand(useF):
        best, bestv = None, None
        uw = a + b * (2.5 - 0.5)
        for dx, dy in [(0, 0), (1, 0), (-1, 0), (0, 1), (0, -1), (1, 1), (1, -1), (-1, 1), (-1, -1)]:
            cx, cy = 2.5 + 0.25 * dx, 9.0 + 0.25 * dy
            F = np.zeros(2)
            if (dx, dy) != (0, 0) and useF:
                Fs = 1 / (a + b * (cx - 0.5)) - 1 / uw          # Eq. 6 with 1 - phi = u
                F = -Fs * np.array([dx, dy]) / math.hypot(dx, dy)
            R = F + (w[0] - [cx, cy]) + (w[2] - [cx, cy])      # Eq. 4 resultant, k_t = 1
            v = R @ R
            if bestv is None or v < bestv - 1e-9:
                best, bestv = (cx, cy), v
        return best

    assert hand(True) == (2.25, 8.75) and hand(False) == (2.5, 8.75)
    assert tuple(out[1].tolist()) == hand(True)
    assert np.array_equal(out[[0, 2]], w[[0, 2]])
    # Eq. 6 arithmetic: u 0.5 -> 0.25 is phi 0.5 -> 0.75, F = 1/0.25 - 1/0.5 = 2
    assert (1 / np.float32(0.25) - 1 / np.float32(0.5)) == 2.0


def test_p13_band_properties(orc):
    N = 64
    cls = np.zeros((N, N), np.uint8); cls[32, 60] = orc.GOAL
    u = orc.init_u32(cls); orc.relax_f32(cls, u, 3000)
    straight = np.array([[x + 0.5, 32.5] for x in range(35, 61)], np.float32)
    assert np.array_equal(orc.band(cls, u, straight, 50), straight)        # equilibrium chain
    assert np.array_equal(orc.band(cls, u, straight, 0), straight)          # I = 0 identity
    stair = np.array([[x + 0.5, y + 0.5] for x, y in
                      [(40 + k // 2 + k % 2, 20 + k // 2) for k in range(24)]], np.float32)
    out = orc.band(cls, u, stair, 50)
    assert _plen(out) < _plen(stair)                                         # a staircase shortens
    assert np.array_equal(out[[0, -1]], stair[[0, -1]])                      # endpoints bit-identical


def test_p13_c1_golden_band(orc):
    gold = json.load(open(os.path.join(GOLD, "c1_64.json")))
    sc = scene_c1()
    st, cls, *_ = orc.classify(sc)
    u = orc.init_u32(cls)
    orc.relax_f32(cls, u, 10 ** 6, 1, 1e-6)
    st, cells = orc.walk(cls, u, orc.robot_cell(sc), 10000)
    w0 = orc.cells_to_waypoints(cells)
    for it, L in gold["band_length"].items():
        out = orc.band(cls, u, w0, int(it))
        assert abs(_plen(out) - L) < 1e-3
        xs = np.floor(out).astype(int)
        assert np.all(cls[xs[:, 1], xs[:, 0]] != orc.OBSTACLE)               # never inside an obstacle
    sm, n = orc.resample(orc.band(cls, u, w0, 50))
    seg = np.hypot(*np.diff(sm, axis=0).T)
    assert np.all(seg <= 1.0 + 1e-6) and n == len(sm)
    assert np.array_equal(sm[0], w0[0]) and np.array_equal(sm[-1], w0[-1])


# --------------------------------------------------------------------- golden C1 (O3-O6)
def test_c1_golden_independent_mirror(orc):
    gold = json.load(open(os.path.join(GOLD, "c1_64.json")))
    sc = scene_c1()
    assert int(sc.static.sum()) == gold["disk_cells"]
    assert list(orc.robot_cell(sc)) == gold["robot_cell"]
    st, cls, *_ = orc.classify(sc)
    u = orc.init_u32(cls)
    s, r = orc.relax_f32(cls, u, 10 ** 6, 1, gold["tol"])
    assert s == gold["sweeps_check1"] and np.float32(r) == np.float32(gold["residual_check1"])
    assert hashlib.sha256(np.abs(u).tobytes()).hexdigest()[:16] == gold["u_abs_sha256_prefix"]
    u8 = orc.init_u32(cls)
    assert orc.relax_f32(cls, u8, 10 ** 6, 8, gold["tol"])[0] == gold["sweeps_check8"]
    st, cells = orc.walk(cls, u, orc.robot_cell(sc), 10000)
    assert st == 0 and len(cells) == gold["walk_len"]
    assert cells[:2].tolist() == gold["walk_first"] and cells[-3:].tolist() == gold["walk_last"]
    assert [cells[:, 1].min(), cells[:, 1].max()] == gold["walk_rows"]


# --------------------------------------------------------------------- P14
def test_p14_determinism(orc):
    from scenes import scene_c2
    sc = scene_c2(3)
    a = orc.plan_step(sc, max_sweeps=60, iters=5)
    b = orc.plan_step(sc, max_sweeps=60, iters=5)
    assert np.array_equal(a["u"], b["u"]) and np.array_equal(a["cls"], b["cls"])
    assert a["sweeps"] == b["sweeps"] == 60


def test_p14_openmp_variants_bit_identical(orc):
    # the OpenMP timing variants (colour passes / band parity phases split over
    # threads) are bit-identical to the single-thread oracle -- same field, sweeps, residual, band
    from scenes import scene_random
    sc = scene_random("p14", 128, 3, 6, 8)  # a seed whose walk reaches the goal at tol 1e-7
    threads = max(2, min(8, orc.host_cores()))
    st, cls, *_ = orc.classify(sc)
    u1 = orc.init_u32(cls)
    u2 = u1.copy()
    for S, ce, tol in ((37, 37, 0.0), (40000, 10, 1e-7)):
        s1, r1 = orc.relax_f32(cls, u1, S, ce, tol)
        s2, r2 = orc.relax_f32(cls, u2, S, ce, tol, threads=threads)
        assert (s1, np.float32(r1)) == (s2, np.float32(r2))
        assert np.array_equal(u1.view(np.uint32), u2.view(np.uint32))
    wst, cells = orc.walk(cls, u1, orc.robot_cell(sc), 10000)
    assert wst == 0
    w0 = orc.cells_to_waypoints(cells)
    b1 = orc.band(cls, u1, w0, 30)
    b2 = orc.band(cls, u1, w0, 30, threads=threads)
    assert np.array_equal(b1.view(np.uint32), b2.view(np.uint32))
    p1 = orc.plan_step(sc, max_sweeps=50, iters=10)
    p2 = orc.plan_step(sc, max_sweeps=50, iters=10, threads=threads)
    assert np.array_equal(p1["u"], p2["u"]) and np.array_equal(p1["smooth"], p2["smooth"])
