"""Seeded synthetic scenes shaped like the paper's Pioneer P3-DX indoor runs.

Recipe (SURVEY.md 8(d) "Synthetic scenes"):
  * 0.1 m cells ("divided into 10 cm by 10 cm cells").
  * Robot radius 0.25 m, speed 0.4 m/s, heading toward the goal; robot at
    (5 %, 5 %) of the extent, goal at (95 %, 95 %), both cleared of walls.
  * Moving obstacles are robot-sized ("moving obstacles are
    simulated by the MobileSim software"), speed U(0.2, 0.5) m/s, heading
    U(-pi, pi), constant velocity ("mostly constant velocity").
  * Tracks = truth + N(0, 0.05^2) on position and velocity.  90 % "converged"
    covariance diag(0.0025, 0.0025, 0.01, 0.01), 10 % "fresh"
    diag(0.25, 0.25, 1, 1) (SPEC.md:293 spawn covariance).
  * Q = 1e-3 diag(dt^4/4, dt^4/4, dt^2, dt^2), dt = 0.1 s (
    PAPER.md:567-569 "process noise ... assumed to be very small").
  * Walls: 1-cell axis-aligned segments of U(3, 15) m (open plan, no rooms).

Everything is drawn from numpy PCG64 ``default_rng(seed)``.  No function in
this file evaluates any equation of the method.
"""
from __future__ import annotations

from dataclasses import dataclass, field, replace
import math

import numpy as np


@dataclass
class WarpCfg:
    """Inputs of rows a1-a2 (time-warp and Kalman predict configuration)."""

    dt: float = 0.1
    Q: np.ndarray = field(default_factory=lambda: np.zeros(16))
    warp_spacing: float = 1.0
    eps_v: float = 0.05
    safety_radius: float = 0.5
    horizon_max: int = 20


def default_warp_cfg(dt: float = 0.1, q: float = 1e-3) -> WarpCfg:
    Q = np.zeros((4, 4))
    Q[0, 0] = Q[1, 1] = q * dt ** 4 / 4.0
    Q[2, 2] = Q[3, 3] = q * dt ** 2
    return WarpCfg(dt=dt, Q=Q.reshape(16).copy())


@dataclass
class Scene:
    name: str
    W: int
    H: int
    cell_size: float
    origin: tuple
    static: np.ndarray          # uint8 [H, W], 1 = wall
    robot: tuple                # (x [m], y [m], theta [rad], speed [m/s])
    goal: tuple                 # (gx, gy) cell
    tracks: np.ndarray          # float64 [n, 20] = x[4] then P[16] row-major
    warp: WarpCfg
    seed: int
    truth: np.ndarray = None    # float64 [n, 4] true obstacle states (x, y, vx, vy)

    @property
    def n_tracks(self) -> int:
        return int(self.tracks.shape[0])


def _paint_segment(static: np.ndarray, x0: int, y0: int, x1: int, y1: int) -> None:
    """Axis-aligned 1-cell wall (its supercover is the cell run itself)."""
    H, W = static.shape
    if y0 == y1:
        a, b = sorted((x0, x1))
        static[y0, max(a, 0):min(b, W - 1) + 1] = 1
    else:
        a, b = sorted((y0, y1))
        static[max(a, 0):min(b, H - 1) + 1, x0] = 1


def _clear_disk(static: np.ndarray, cx: float, cy: float, r_cells: float) -> None:
    H, W = static.shape
    y0, y1 = max(int(cy - r_cells) - 1, 0), min(int(cy + r_cells) + 2, H)
    x0, x1 = max(int(cx - r_cells) - 1, 0), min(int(cx + r_cells) + 2, W)
    yy, xx = np.mgrid[y0:y1, x0:x1]
    m = (xx + 0.5 - cx) ** 2 + (yy + 0.5 - cy) ** 2 <= r_cells ** 2
    static[y0:y1, x0:x1][m] = 0


def _walls(rng: np.random.Generator, W: int, H: int, cs: float, n_seg: int,
           lmin: float = 3.0, lmax: float = 15.0) -> np.ndarray:
    static = np.zeros((H, W), np.uint8)
    for _ in range(n_seg):
        L = int(round(rng.uniform(lmin, lmax) / cs))
        if rng.random() < 0.5:
            y = int(rng.integers(0, H))
            x = int(rng.integers(0, max(W - L, 1)))
            _paint_segment(static, x, y, min(x + L, W - 1), y)
        else:
            x = int(rng.integers(0, W))
            y = int(rng.integers(0, max(H - L, 1)))
            _paint_segment(static, x, y, x, min(y + L, H - 1))
    return static


def _tracks(rng: np.random.Generator, n: int, W: int, H: int, cs: float, static: np.ndarray,
            robot_xy, goal_xy, fresh_frac: float = 0.1):
    """Obstacle truths in free space plus noisy Kalman tracks (x[4], P[16])."""
    truth = np.zeros((n, 4))
    tracks = np.zeros((n, 20))
    ext_x, ext_y = W * cs, H * cs
    k = 0
    while k < n:
        x = rng.uniform(0.5, ext_x - 0.5)
        y = rng.uniform(0.5, ext_y - 0.5)
        cx, cy = int(x / cs), int(y / cs)
        if static[cy, cx]:
            continue
        if math.hypot(x - robot_xy[0], y - robot_xy[1]) < 2.0:
            continue
        if math.hypot(x - goal_xy[0], y - goal_xy[1]) < 1.0:
            continue
        sp = rng.uniform(0.2, 0.5)
        hd = rng.uniform(-math.pi, math.pi)
        truth[k] = (x, y, sp * math.cos(hd), sp * math.sin(hd))
        k += 1
    fresh = rng.random(n) < fresh_frac
    for i in range(n):
        xh = truth[i] + rng.normal(0.0, 0.05, 4)
        P = np.diag([0.25, 0.25, 1.0, 1.0]) if fresh[i] else np.diag([0.0025, 0.0025, 0.01, 0.01])
        tracks[i, :4] = xh
        tracks[i, 4:] = P.reshape(16)
    return truth, tracks


def scene_random(name: str, N: int, n_seg: int, n_obs: int, seed: int, cs: float = 0.1,
                 speed: float = 0.4) -> Scene:
    """Open-plan N x N scene: n_seg wall segments, n_obs moving obstacles."""
    rng = np.random.default_rng(seed)
    W = H = N
    static = _walls(rng, W, H, cs, n_seg)
    rx, ry = 0.05 * W * cs, 0.05 * H * cs
    gx, gy = int(0.95 * W), int(0.95 * H)
    _clear_disk(static, rx / cs, ry / cs, 1.5 / cs)
    _clear_disk(static, gx + 0.5, gy + 0.5, 1.5 / cs)
    theta = math.atan2((gy + 0.5) * cs - ry, (gx + 0.5) * cs - rx)
    truth, tracks = _tracks(rng, n_obs, W, H, cs, static, (rx, ry), ((gx + 0.5) * cs, (gy + 0.5) * cs))
    return Scene(name, W, H, cs, (0.0, 0.0), static, (rx, ry, theta, speed), (gx, gy),
                 tracks, default_warp_cfg(), seed, truth)


def scene_c1() -> Scene:
    """BASELINE.json configs[0]: 64 x 64, one static circular obstacle, no tracks.

    Disk: cells whose centre lies within 0.8 m of (3.2 m, 3.2 m) (208 cells);
    robot cell (8, 32); goal cell (56, 32).
    """
    N, cs = 64, 0.1
    static = np.zeros((N, N), np.uint8)
    for j in range(N):
        for i in range(N):
            dx = (i + 0.5) * cs - 3.2
            dy = (j + 0.5) * cs - 3.2
            if dx * dx + dy * dy <= 0.8 * 0.8:
                static[j, i] = 1
    robot = (8.5 * cs, 32.5 * cs, 0.0, 0.4)
    return Scene("c1_64", N, N, cs, (0.0, 0.0), static, robot, (56, 32),
                 np.zeros((0, 20)), default_warp_cfg(), 0, np.zeros((0, 4)))


def scene_c2(seed: int = 0) -> Scene:
    """BASELINE.json configs[1]: 512 x 512, 8 wall segments, 20 moving obstacles."""
    return scene_random(f"c2_512_s{seed}", 512, 8, 20, seed)


def scene_c3(seed: int = 0) -> Scene:
    """BASELINE.json configs[2]: 4096 x 4096, 512 segments, 200 moving obstacles."""
    return scene_random(f"c3_4096_s{seed}", 4096, 512, 200, seed)


def scene_c4(seed: int = 0) -> Scene:
    """BASELINE.json configs[3]: 16384 x 16384, 8192 segments, 3200 obstacles."""
    return scene_random(f"c4_16384_s{seed}", 16384, 8192, 3200, seed)


def scene_c5(n: int = 1024, first_seed: int = 0):
    """BASELINE.json configs[4]: a batch of independent 512 x 512 dynamic scenarios."""
    return [scene_random(f"c5_512_s{s}", 512, 8, 20, s) for s in range(first_seed, first_seed + n)]


def advance_scene(scene: Scene, tick: int, robot_step: float = 0.04) -> Scene:
    """Scene at tick `tick` of a scripted plan loop (warm-start replay).

    Obstacle truths move at constant velocity with specular reflection at the
    grid border; the robot advances `robot_step` m per tick straight toward
    the goal (scripted, so the oracle can replay the same poses); tracks are
    re-drawn around the truth with a per-tick seed.  Input plumbing only.
    """
    rng = np.random.default_rng([scene.seed, tick])
    dt = scene.warp.dt
    ext_x, ext_y = scene.W * scene.cell_size, scene.H * scene.cell_size
    truth = scene.truth.copy()
    for _ in range(tick):
        truth[:, 0] += truth[:, 2] * dt
        truth[:, 1] += truth[:, 3] * dt
        for ax, ext in ((0, ext_x), (1, ext_y)):
            lo = truth[:, ax] < 0.3
            hi = truth[:, ax] > ext - 0.3
            truth[lo | hi, 2 + ax] *= -1.0
            truth[lo, ax] = 0.3
            truth[hi, ax] = ext - 0.3
    tracks = scene.tracks.copy()
    if len(truth):
        tracks[:, :4] = truth + rng.normal(0.0, 0.05, truth.shape)
    rx, ry, th, sp = scene.robot
    gxm = (scene.goal[0] + 0.5) * scene.cell_size
    gym = (scene.goal[1] + 0.5) * scene.cell_size
    d = math.hypot(gxm - rx, gym - ry)
    adv = min(robot_step * tick, max(d - 0.5, 0.0))
    rx2 = rx + adv * math.cos(th)
    ry2 = ry + adv * math.sin(th)
    return replace(scene, name=f"{scene.name}_t{tick}", robot=(rx2, ry2, th, sp), tracks=tracks, truth=truth)


def detections(scene: Scene, tick: int, sigma_z: float = 0.05, p_miss: float = 0.05, n_clutter: int = 0,
               shuffle: bool = True) -> np.ndarray:
    """Noisy position detections [m, 2] of the obstacle truths at tick `tick` (advance_scene motion):
    each truth is seen with probability 1 - p_miss, with N(0, sigma_z^2) noise per axis,
    plus `n_clutter` uniform false detections, in random order.  Input plumbing only."""
    rng = np.random.default_rng([scene.seed, tick, 7])
    truth = advance_scene(scene, tick).truth if tick else scene.truth
    seen = rng.random(len(truth)) >= p_miss
    z = truth[seen, :2] + rng.normal(0.0, sigma_z, (int(seen.sum()), 2))
    if n_clutter:
        ext = np.array([scene.W * scene.cell_size, scene.H * scene.cell_size])
        z = np.concatenate([z, rng.uniform(0.0, 1.0, (n_clutter, 2)) * ext])
    if shuffle:
        z = z[rng.permutation(len(z))]
    return np.ascontiguousarray(z)


@dataclass
class SimCfg:
    """Closed-loop simulator configuration (row f2; C31-C35).  Plain inputs."""
    dt: float = 0.1
    robot_radius: float = 0.25
    obstacle_radius: float = 0.25
    goal_radius: float = 0.3
    turn_distance: float = 0.5
    heading_sigma: float = 0.02
    det_sigma: float = 0.05
    turn_max: float = 0.15707963267948966  # 9 degrees per tick = 90 deg/s
    seed: int = 1
    max_ticks: int = 1000
    init_tol: float = 1e-6       # Alg. 1 "Initialize ... harmonic potential values": relax the
    init_max_sweeps: int = 1_000_000  # tick-0 static field to this residual (checked every 100 sweeps)


def scene_sim(seed: int, n_obs: int, N: int = 256, n_seg: int = 6, cs: float = 0.1) -> Scene:
    """A 25.6 m x 25.6 m map with `n_seg` wall segments, the robot near one corner heading
    to a goal near the opposite one, and `n_obs` robot-sized obstacles wandering at 0.2-0.5 m/s
    (Table 1 uses 1, 2, 4, 8, 12, 16).  truth = obstacle states (x, y, vx, vy); no tracks (the
    tracker spawns them from detections)."""
    rng = np.random.default_rng([seed, 1903])
    W = H = N
    static = _walls(rng, W, H, cs, n_seg, lmin=2.0, lmax=8.0)
    rx, ry = 1.55, 1.55
    gx, gy = N - 16, N - 16
    _clear_disk(static, rx / cs, ry / cs, 1.5 / cs)
    _clear_disk(static, gx + 0.5, gy + 0.5, 1.5 / cs)
    theta = math.atan2((gy + 0.5) * cs - ry, (gx + 0.5) * cs - rx)
    truth, _ = _tracks(rng, n_obs, W, H, cs, static, (rx, ry), ((gx + 0.5) * cs, (gy + 0.5) * cs))
    return Scene(f"sim_s{seed}_n{n_obs}", W, H, cs, (0.0, 0.0), static, (rx, ry, theta, 0.4), (gx, gy),
                 np.zeros((0, 20)), default_warp_cfg(), seed, truth)


def random_small_map(seed: int, N: int = 48, n_disks=(3, 11), n_walls=(0, 4)):
    """Random N x N static map with disks and walls plus a goal cell and a start cell.

    Used by the maximum-principle / BFS pins.
    Returns (static uint8 [N, N], goal (x, y), start (x, y)).
    """
    rng = np.random.default_rng(seed)
    static = np.zeros((N, N), np.uint8)
    for _ in range(int(rng.integers(n_disks[0], n_disks[1] + 1))):
        cx, cy = rng.uniform(0, N, 2)
        r = rng.uniform(1.5, N / 8)
        yy, xx = np.mgrid[0:N, 0:N]
        static[(xx + 0.5 - cx) ** 2 + (yy + 0.5 - cy) ** 2 <= r * r] = 1
    for _ in range(int(rng.integers(n_walls[0], n_walls[1] + 1))):
        L = int(rng.integers(N // 4, N // 2))
        if rng.random() < 0.5:
            y, x = int(rng.integers(0, N)), int(rng.integers(0, N - L))
            _paint_segment(static, x, y, x + L, y)
        else:
            x, y = int(rng.integers(0, N)), int(rng.integers(0, N - L))
            _paint_segment(static, x, y, x, y + L)
    while True:
        g = (int(rng.integers(0, N)), int(rng.integers(0, N)))
        if not static[g[1], g[0]]:
            break
    while True:
        s = (int(rng.integers(0, N)), int(rng.integers(0, N)))
        if not static[s[1], s[0]] and s != g:
            break
    return static, g, s


def annulus_fixed(N: int):
    """Annulus geometry for pin P9: centre (N/2, N/2), goal disk r <= 0.1 N,
    obstacle ring r >= 0.45 N.  Returns (goal mask, obstacle mask, r) over cell centres."""
    yy, xx = np.mgrid[0:N, 0:N]
    r = np.hypot(xx + 0.5 - N / 2, yy + 0.5 - N / 2)
    return r <= 0.1 * N, r >= 0.45 * N, r


CONFIGS = {
    "c1": "64x64, one static disk, relax to residual 1e-6",
    "c2": "512x512, 20 moving obstacles, plan loop",
    "c3": "4096x4096, 200 moving obstacles, relaxation + path",
    "c4": "16384x16384 row-slab sharded",
    "c5": "batch of 1024 x 512x512 scenarios",
}
