"""CPU oracle for the Time-Warped Grid hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
/ ``--impl reference`` legs may import this package.  The product path
(``paper_1903_07441_b200``) never imports it, and the two share no code: the
only common dependency is the input generator ``scenes/``.

The arithmetic lives in ``twg_oracle.c`` (plain C, built with
``-O2 -ffp-contract=off -fno-fast-math``); this module only builds it and
marshals numpy arrays through ctypes.  ``plan_step`` composes the steps O1-O8
in the order of Algorithm 1.

Parity unpinned (stated here and in DESIGN.md): the exact smoothed path on
general scenes (only properties of ``band`` are pinned), the warm-start
trajectory over many ticks, and the next-waypoint choice.
"""
from __future__ import annotations

import ctypes as C
import math
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "twg_oracle.c")
_LIB = os.path.join(_HERE, "libtwg_oracle.so")
_lib = None

FREE, OBSTACLE, GOAL = 0, 1, 2
OK, W_GOAL_SWALLOWED, E_INVALID_ARG, E_OUT_OF_BOUNDS, E_OVERLAPPING, E_INVALID_START, E_NO_PATH = 0, 1, -1, -2, -3, -4, -5


def build(force: bool = False) -> str:
    """Compile the oracle (no FMA contraction, no fast-math, no FTZ/DAZ)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-fPIC", "-shared",
               "-Wall", "-o", _LIB, _SRC, "-lm"]
        subprocess.check_call(cmd)
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_LIB)
        d, i32, i64, f32 = C.c_double, C.c_int32, C.c_int64, C.c_float
        P = C.c_void_p
        L.orc_warp_radius.restype = d
        L.orc_warp_radius.argtypes = [d] * 6
        L.orc_warp_number.restype = i32
        L.orc_warp_number.argtypes = [d, d]
        L.orc_horizon.restype = i32
        L.orc_horizon.argtypes = [i32, d, d, d, d, i32]
        L.orc_predict.restype = None
        L.orc_predict.argtypes = [P, P, P, d, i32, P, P]
        L.orc_footprint_r2.restype = d
        L.orc_footprint_r2.argtypes = [P, d]
        L.orc_stamp_bruteforce.restype = None
        L.orc_stamp_bruteforce.argtypes = [i32, i32, d, d, d, d, d, d, P]
        L.orc_stamp_box.restype = None
        L.orc_stamp_box.argtypes = [i32, i32, d, d, d, d, d, d, P]
        L.orc_classify.restype = i32
        L.orc_classify.argtypes = [i32, i32, d, d, d, P, i32, i32, d, d, d, d, i32, P,
                                   d, P, d, d, d, i32, i32, i32, P, P, P, P]
        L.orc_horizon_ring.restype = i32
        L.orc_horizon_ring.argtypes = [i32, d, d, d, i32]
        L.orc_relax_jacobi_f32.restype = i32
        L.orc_relax_jacobi_f32.argtypes = [i32, i32, P, P, i32, i32, f32, P]
        L.orc_relax_lex_f32.restype = i32
        L.orc_relax_lex_f32.argtypes = [i32, i32, P, P, i32, i32, f32, P]
        L.orc_index_matrix.restype = None
        L.orc_index_matrix.argtypes = [i32, i32, P, P, P]
        L.orc_kalman_update.restype = i32
        L.orc_kalman_update.argtypes = [P, P, P, P]
        L.orc_associate.restype = None
        L.orc_associate.argtypes = [i32, P, i32, P, d, P, P]
        L.orc_track_step.restype = i32
        L.orc_track_step.argtypes = [i32, P, P, i32, i32, P, d, P, d, d, d, d, i32, i32, P]
        u64 = C.c_uint64
        L.orc_rng_u01.restype = d
        L.orc_rng_u01.argtypes = [u64, u64, u64, u64, u64]
        L.orc_rng_normal.restype = d
        L.orc_rng_normal.argtypes = [u64, u64, u64, u64, u64]
        L.orc_sim_sense.restype = None
        L.orc_sim_sense.argtypes = [i32, P, d, u64, u64, u64, P]
        L.orc_sim_move.restype = None
        L.orc_sim_move.argtypes = [i32, i32, d, d, d, P, P, P, P, d, d, i32, d, d, i32, P, P, P, i32, u64, u64,
                                   P, P]
        L.orc_cellband.restype = None
        L.orc_cellband.argtypes = [i32, i32, P, P, P, i32, f32]
        L.orc_walk_dir.restype = i32
        L.orc_walk_dir.argtypes = [i32, i32, P, i32, i32, i32, P, P]
        L.orc_warp_map.restype = None
        L.orc_warp_map.argtypes = [i32, i32, d, d, d, d, d, d, d, P]
        L.orc_init_u32.restype = None
        L.orc_init_u32.argtypes = [i64, P, P, P, P]
        L.orc_init_u64.restype = None
        L.orc_init_u64.argtypes = [i64, P, P]
        L.orc_relax_f32.restype = i32
        L.orc_relax_f32.argtypes = [i32, i32, P, P, i32, i32, f32, P]
        L.orc_relax_f32_omp.restype = i32
        L.orc_relax_f32_omp.argtypes = [i32, i32, P, P, i32, i32, f32, i32, P]
        L.orc_band_omp.restype = None
        L.orc_band_omp.argtypes = [i32, i32, P, P, i32, P, i32, f32, f32, i32]
        L.orc_relax_f32_ex.restype = i32
        L.orc_relax_f32_ex.argtypes = [i32, i32, P, P, i32, i32, f32, i32, i32, i32, P]
        L.orc_relax_f64.restype = i32
        L.orc_relax_f64.argtypes = [i32, i32, P, P, i32, i32, d, P]
        L.orc_jacobi_f64.restype = i32
        L.orc_jacobi_f64.argtypes = [i32, i32, P, P, i32, d, P]
        L.orc_walk.restype = i32
        L.orc_walk.argtypes = [i32, i32, P, P, i32, i32, i32, P, P]
        L.orc_bilerp.restype = f32
        L.orc_bilerp.argtypes = [i32, i32, P, f32, f32]
        L.orc_band.restype = None
        L.orc_band.argtypes = [i32, i32, P, P, i32, P, i32, f32, f32]
        L.orc_resample.restype = i32
        L.orc_resample.argtypes = [i32, P, i32, P]
        L.orc_next_waypoint.restype = i32
        L.orc_next_waypoint.argtypes = [i32, P, P, P]
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


# ---------------------------------------------------------------- O1, O2
def warp_radius(xr, yr, theta, xo, yo):
    return lib().orc_warp_radius(xr, yr, math.cos(theta), math.sin(theta), xo, yo)


def warp_number(rx, w=1.0):
    return lib().orc_warp_number(rx, w)


def horizon(t, speed_r, vx, vy, eps_v=0.05, hmax=20):
    return lib().orc_horizon(t, speed_r, vx, vy, eps_v, hmax)


def horizon_ring(t, w, speed_r, dt, hmax=20):
    return lib().orc_horizon_ring(t, w, speed_r, dt, hmax)


def predict(x, P, Q, dt, j):
    x = np.ascontiguousarray(x, np.float64).reshape(4)
    P = np.ascontiguousarray(P, np.float64).reshape(16)
    Q = np.ascontiguousarray(Q, np.float64).reshape(16)
    xo = np.zeros(4)
    Po = np.zeros(16)
    lib().orc_predict(_p(x), _p(P), _p(Q), dt, int(j), _p(xo), _p(Po))
    return xo, Po.reshape(4, 4)


def footprint_r2(P, rs):
    P = np.ascontiguousarray(P, np.float64).reshape(16)
    return lib().orc_footprint_r2(_p(P), rs)


def stamp_disk(W, H, cs, ox, oy, xp, yp, R2, brute=True):
    m = np.zeros((H, W), np.uint8)
    f = lib().orc_stamp_bruteforce if brute else lib().orc_stamp_box
    f(W, H, cs, ox, oy, xp, yp, R2, _p(m))
    return m


# ---------------------------------------------------------------- O3
def classify(scene, horizon_mode=0, footprint_mode=0):
    """Class grid (uint8 H x W: 0 free, 1 obstacle, 2 goal) plus per-track t, j, (xp, yp, R2)."""
    W, H = scene.W, scene.H
    static = np.ascontiguousarray(scene.static, np.uint8)
    tracks = np.ascontiguousarray(scene.tracks, np.float64).reshape(-1, 20)
    n = tracks.shape[0]
    cls = np.zeros((H, W), np.uint8)
    t = np.zeros(max(n, 1), np.int32)
    j = np.zeros(max(n, 1), np.int32)
    pred = np.zeros((max(n, 1), 3))
    wc = scene.warp
    Q = np.ascontiguousarray(wc.Q, np.float64).reshape(16)
    xr, yr, th, sp = scene.robot
    st = lib().orc_classify(W, H, scene.cell_size, scene.origin[0], scene.origin[1], _p(static),
                            int(scene.goal[0]), int(scene.goal[1]), xr, yr, th, sp,
                            n, _p(tracks), wc.dt, _p(Q), wc.warp_spacing, wc.eps_v,
                            wc.safety_radius, int(wc.horizon_max), int(horizon_mode), int(footprint_mode),
                            _p(cls), _p(t), _p(j), _p(pred))
    return st, cls, t[:n], j[:n], pred[:n]


def robot_cell(scene):
    xr, yr = scene.robot[0], scene.robot[1]
    return (int(math.floor((xr - scene.origin[0]) / scene.cell_size)),
            int(math.floor((yr - scene.origin[1]) / scene.cell_size)))


def init_u32(cls, u_prev=None, cls_prev=None):
    """cold (u_prev None): goal 1, obstacle 0, free 0.5; warm: free cells keep u_prev, a released
    goal (cls_prev GOAL, free now) restarts at 0 (C7)."""
    cls = np.ascontiguousarray(cls, np.uint8)
    u = np.zeros(cls.shape, np.float32)
    if u_prev is None:
        lib().orc_init_u32(cls.size, _p(cls), None, None, _p(u))
    else:
        up = np.ascontiguousarray(u_prev, np.float32)
        cp = None if cls_prev is None else np.ascontiguousarray(cls_prev, np.uint8)
        lib().orc_init_u32(cls.size, _p(cls), _p(up), None if cp is None else _p(cp), _p(u))
    return u


def init_u64(cls):
    cls = np.ascontiguousarray(cls, np.uint8)
    u = np.zeros(cls.shape, np.float64)
    lib().orc_init_u64(cls.size, _p(cls), _p(u))
    return u


# ---------------------------------------------------------------- O4, O5
def host_cores():
    """Host cores this process may use (the OpenMP timing variants' default thread count)."""
    return len(os.sched_getaffinity(0))


def relax_f32(cls, u, max_sweeps, check_every=1, tol=0.0, threads=1):
    """In-place red-black relaxation of float32 u.  Returns (sweeps, residual).  threads > 1: the
    OpenMP variant (bit-identical, P14)."""
    assert u.dtype == np.float32 and u.flags.c_contiguous
    cls = np.ascontiguousarray(cls, np.uint8)
    H, W = u.shape
    r = np.zeros(1, np.float32)
    if threads > 1:
        s = lib().orc_relax_f32_omp(W, H, _p(cls), _p(u), int(max_sweeps), int(check_every), float(tol),
                                    int(threads), _p(r))
    else:
        s = lib().orc_relax_f32(W, H, _p(cls), _p(u), int(max_sweeps), int(check_every), float(tol), _p(r))
    return int(s), float(r[0])


def relax_f32_ex(cls, u, max_sweeps, check_every=1, tol=0.0, row_parity=0, res_rows=None):
    """relax_f32 with colour parity (x + row_parity + y) and the residual over rows res_rows only."""
    assert u.dtype == np.float32 and u.flags.c_contiguous
    cls = np.ascontiguousarray(cls, np.uint8)
    H, W = u.shape
    r0, r1 = res_rows if res_rows is not None else (0, H)
    r = np.zeros(1, np.float32)
    s = lib().orc_relax_f32_ex(W, H, _p(cls), _p(u), int(max_sweeps), int(check_every), float(tol),
                               int(row_parity) & 1, int(r0), int(r1), _p(r))
    return int(s), float(r[0])


def relax_f64(cls, u, max_sweeps, check_every=1, tol=0.0):
    assert u.dtype == np.float64 and u.flags.c_contiguous
    cls = np.ascontiguousarray(cls, np.uint8)
    H, W = u.shape
    r = np.zeros(1, np.float64)
    s = lib().orc_relax_f64(W, H, _p(cls), _p(u), int(max_sweeps), int(check_every), float(tol), _p(r))
    return int(s), float(r[0])


def relax_jacobi_f32(cls, u, max_sweeps, check_every=1, tol=0.0):
    assert u.dtype == np.float32 and u.flags.c_contiguous
    cls = np.ascontiguousarray(cls, np.uint8)
    H, W = u.shape
    r = np.zeros(1, np.float32)
    s = lib().orc_relax_jacobi_f32(W, H, _p(cls), _p(u), int(max_sweeps), int(check_every), float(tol), _p(r))
    return int(s), float(r[0])


def relax_lex_f32(cls, u, max_sweeps, check_every=1, tol=0.0):
    assert u.dtype == np.float32 and u.flags.c_contiguous
    cls = np.ascontiguousarray(cls, np.uint8)
    H, W = u.shape
    r = np.zeros(1, np.float32)
    s = lib().orc_relax_lex_f32(W, H, _p(cls), _p(u), int(max_sweeps), int(check_every), float(tol), _p(r))
    return int(s), float(r[0])


def index_matrix(cls, u):
    cls = np.ascontiguousarray(cls, np.uint8)
    u = np.ascontiguousarray(u, np.float32)
    out = np.zeros(u.shape, np.uint8)
    H, W = u.shape
    lib().orc_index_matrix(W, H, _p(cls), _p(u), _p(out))
    return out


def cellband(cls, u, dir_in, iters=50, kt=1.0):
    """Per-cell rubber band on the index matrix (orc_cellband, Alg. 1, C37): returns the
    optimised matrix (dir_in is not modified)."""
    cls = np.ascontiguousarray(cls, np.uint8)
    u = np.ascontiguousarray(u, np.float32)
    d = np.ascontiguousarray(dir_in, np.uint8).copy()
    H, W = u.shape
    lib().orc_cellband(W, H, _p(cls), _p(u), _p(d), int(iters), np.float32(kt))
    return d


def walk_dir(dir_m, start, max_len):
    """Walk along an index matrix from start (orc_walk_dir): (status, cells [n, 2])."""
    d = np.ascontiguousarray(dir_m, np.uint8)
    H, W = d.shape
    cells = np.zeros((max(max_len, 1), 2), np.int32)
    n = np.zeros(1, np.int32)
    st = lib().orc_walk_dir(W, H, _p(d), int(start[0]), int(start[1]), int(max_len), _p(cells), _p(n))
    return st, cells[: int(n[0])].copy()


def warp_map(scene):
    out = np.zeros((scene.H, scene.W), np.int32)
    xr, yr, th, _ = scene.robot
    lib().orc_warp_map(scene.W, scene.H, scene.cell_size, scene.origin[0], scene.origin[1], xr, yr, th,
                       scene.warp.warp_spacing, _p(out))
    return out


W_TRUNCATED, W_SINGULAR = 2, 3


def kalman_update(x, P, z, R):
    """Eqs. 11-13 (returns status, x', P'); inputs are not modified."""
    x = np.array(x, np.float64).reshape(4).copy()
    P = np.array(P, np.float64).reshape(16).copy()
    z = np.ascontiguousarray(z, np.float64).reshape(2)
    R = np.ascontiguousarray(R, np.float64).reshape(4)
    st = lib().orc_kalman_update(_p(x), _p(P), _p(z), _p(R))
    return st, x, P.reshape(4, 4)


def associate(pxy, z, gate):
    pxy = np.ascontiguousarray(pxy, np.float64).reshape(-1, 2)
    z = np.ascontiguousarray(z, np.float64).reshape(-1, 2)
    n, m = len(pxy), len(z)
    mt = np.zeros(max(n, 1), np.int32)
    du = np.zeros(max(m, 1), np.uint8)
    lib().orc_associate(n, _p(pxy), m, _p(z), float(gate), _p(mt), _p(du))
    return mt[:n], du[:m].astype(bool)


def track_step(tracks, missed, z, dt=0.1, Q=None, sigma_z=0.05, gate=0.5, var_pos=0.25, var_vel=1.0,
               prune_after=10, max_tracks=0):
    """One tracker tick (orc_track_step).  tracks [n, 20], missed [n], z [m, 2] -> (status, tracks, missed)."""
    tracks = np.asarray(tracks, np.float64).reshape(-1, 20)
    z = np.ascontiguousarray(z, np.float64).reshape(-1, 2)
    n, m = len(tracks), len(z)
    cap = n + m + 1
    trk = np.zeros((cap, 20))
    trk[:n] = tracks
    mis = np.zeros(cap, np.int32)
    mis[:n] = np.asarray(missed, np.int32).reshape(n)
    if Q is None:
        Q = np.zeros(16)
        Q[0] = Q[5] = 1e-3 * dt ** 4 / 4.0
        Q[10] = Q[15] = 1e-3 * dt ** 2
    Q = np.ascontiguousarray(Q, np.float64).reshape(16)
    n_out = np.zeros(1, np.int32)
    st = lib().orc_track_step(n, _p(trk), _p(mis), cap, m, _p(z), float(dt), _p(Q), float(sigma_z), float(gate),
                              float(var_pos), float(var_vel), int(prune_after), int(max_tracks), _p(n_out))
    k = int(n_out[0])
    return st, trk[:k].copy(), mis[:k].copy()


def jacobi_f64(cls, u, max_sweeps, tol=0.0):
    assert u.dtype == np.float64 and u.flags.c_contiguous
    cls = np.ascontiguousarray(cls, np.uint8)
    H, W = u.shape
    r = np.zeros(1, np.float64)
    s = lib().orc_jacobi_f64(W, H, _p(cls), _p(u), int(max_sweeps), float(tol), _p(r))
    return int(s), float(r[0])


# ---------------------------------------------------------------- O6-O8
def walk(cls, u, start, max_len):
    cls = np.ascontiguousarray(cls, np.uint8)
    u = np.ascontiguousarray(u, np.float32)
    H, W = u.shape
    cells = np.zeros((max(max_len, 1), 2), np.int32)
    n = np.zeros(1, np.int32)
    st = lib().orc_walk(W, H, _p(cls), _p(u), int(start[0]), int(start[1]), int(max_len), _p(cells), _p(n))
    return st, cells[: int(n[0])].copy()


def bilerp(u, px, py):
    u = np.ascontiguousarray(u, np.float32)
    H, W = u.shape
    return lib().orc_bilerp(W, H, _p(u), float(px), float(py))


def band(cls, u, waypoints, iters=50, step=0.25, kt=1.0, threads=1):
    cls = np.ascontiguousarray(cls, np.uint8)
    u = np.ascontiguousarray(u, np.float32)
    H, W = u.shape
    w = np.ascontiguousarray(waypoints, np.float32).reshape(-1, 2).copy()
    if threads > 1:
        lib().orc_band_omp(W, H, _p(cls), _p(u), w.shape[0], _p(w), int(iters), np.float32(step), np.float32(kt),
                           int(threads))
    else:
        lib().orc_band(W, H, _p(cls), _p(u), w.shape[0], _p(w), int(iters), np.float32(step), np.float32(kt))
    return w


def cells_to_waypoints(cells):
    return (np.asarray(cells, np.float32).reshape(-1, 2) + np.float32(0.5)).astype(np.float32)


def resample(w, max_out=None):
    w = np.ascontiguousarray(w, np.float32).reshape(-1, 2)
    cnt = lib().orc_resample(w.shape[0], _p(w), 0, None) if max_out is None else None
    m = cnt if max_out is None else max_out
    out = np.zeros((max(m, 1), 2), np.float32)
    cnt = lib().orc_resample(w.shape[0], _p(w), m, _p(out))
    return out[: min(cnt, m)].copy(), int(cnt)


def next_waypoint(pts):
    pts = np.ascontiguousarray(pts, np.float32).reshape(-1, 2)
    nx = np.zeros(1, np.float32)
    ny = np.zeros(1, np.float32)
    k = lib().orc_next_waypoint(pts.shape[0], _p(pts), _p(nx), _p(ny))
    return k, float(nx[0]), float(ny[0])


def plan_step(scene, max_sweeps=100, check_every=None, tol=0.0, iters=50, step=0.25, kt=1.0,
              max_len=None, prev=None, jacobi=False, horizon_mode=0, footprint_mode=0, lex=False, threads=1):
    """One planning tick, Algorithm 1 on the CPU.

    prev: None (cold start) or the dict returned by the previous call (warm
    start, C7).  Returns a dict with class grid, field (float32 u), sweeps,
    residual, walk status/cells, smoothed path and next waypoint.
    """
    st, cls, t, j, pred = classify(scene, horizon_mode, footprint_mode)
    if st < 0:
        return {"status": st}
    if prev is None:
        u = init_u32(cls)
    else:
        u = init_u32(cls, prev["u"], prev.get("cls"))
    if jacobi or lex:
        relax = relax_jacobi_f32 if jacobi else relax_lex_f32
        sweeps, res = relax(cls, u, max_sweeps, check_every or max(max_sweeps, 1), tol)
    else:
        sweeps, res = relax_f32(cls, u, max_sweeps, check_every or max(max_sweeps, 1), tol, threads=threads)
    if max_len is None:
        max_len = 4 * (scene.W + scene.H)
    wst, cells = walk(cls, u, robot_cell(scene), max_len)
    out = {"status": st, "cls": cls, "u": u, "t": t, "j": j, "pred": pred, "sweeps": sweeps,
           "residual": res, "walk_status": wst, "cells": cells}
    if wst == OK:
        w = band(cls, u, cells_to_waypoints(cells), iters, step, kt, threads=threads)
        sm, _ = resample(w)
        k, nx, ny = next_waypoint(sm)
        out.update(band=w, smooth=sm, next=(nx, ny))
    else:
        out.update(band=np.zeros((0, 2), np.float32), smooth=np.zeros((0, 2), np.float32), next=None)
    return out


# ----------------------------------------------------------------------------- f2 simulator
SIM_RUNNING, SIM_SUCCESS, SIM_COLLISION, SIM_TIMEOUT = 0, 1, 2, 3


def rng_u01(seed, trial, tick, entity, k):
    return lib().orc_rng_u01(seed, trial, tick, entity, k)


def rng_normal(seed, trial, tick, entity, stream):
    return lib().orc_rng_normal(seed, trial, tick, entity, stream)


def sim_sense(obs, sigma_z, seed, trial, tick):
    obs = np.ascontiguousarray(obs, np.float64).reshape(-1, 4)
    z = np.zeros((max(len(obs), 1), 2))
    lib().orc_sim_sense(len(obs), _p(obs), float(sigma_z), seed, trial, tick, _p(z))
    return z[: len(obs)].copy()


def sim_cos_bins():
    """cos(5 k degrees), k = 0..36: the turning-angle histogram thresholds (C35)."""
    return np.array([math.cos(k * 5.0 * math.pi / 180.0) for k in range(37)], np.float64)


class SimState:
    """One trial: robot [x, y, hx, hy, speed, length], ticks, status, obstacles [n, 4], speeds, histogram."""

    def __init__(self, scene, cfg):
        xr, yr, th, sp = scene.robot
        self.rob = np.array([xr, yr, math.cos(th), math.sin(th), sp, 0.0])
        self.ticks = np.zeros(1, np.int32)
        self.status = np.zeros(1, np.int32)
        self.obs = np.ascontiguousarray(scene.truth, np.float64).reshape(-1, 4).copy()
        self.speed = np.sqrt(self.obs[:, 2] * self.obs[:, 2] + self.obs[:, 3] * self.obs[:, 3])
        self.hist = np.zeros(36, np.int32)
        self.goal = (scene.origin[0] + (scene.goal[0] + 0.5) * scene.cell_size,
                     scene.origin[1] + (scene.goal[1] + 0.5) * scene.cell_size)


def sim_move(scene, state, wp, cfg, trial):
    """One simulator tick (orc_sim_move); wp = (x, y) cell units or None (blocked)."""
    c = np.array([cfg.dt, cfg.robot_radius, cfg.obstacle_radius, cfg.goal_radius, cfg.turn_distance,
                  cfg.heading_sigma, math.cos(cfg.turn_max), math.sin(cfg.turn_max)])
    mask = np.ascontiguousarray(scene.static, np.uint8)
    bins = sim_cos_bins()
    has = 0 if wp is None else 1
    wx, wy = (0.0, 0.0) if wp is None else (float(wp[0]), float(wp[1]))
    lib().orc_sim_move(scene.W, scene.H, scene.cell_size, scene.origin[0], scene.origin[1], _p(mask),
                       _p(state.rob), _p(state.ticks), _p(state.status), state.goal[0], state.goal[1], has, wx, wy,
                       len(state.obs), _p(state.obs), _p(state.speed), _p(c), int(cfg.max_ticks), cfg.seed, trial,
                       _p(bins), _p(state.hist))


def sim_run(scene, cfg, trial=0, max_ticks=None, sweeps=100, iters=50, max_len=4096, tracker=None, warp_scene=None):
    """Closed loop of Algorithm 1 on the CPU (sense -> track -> plan -> move), until the trial ends or
    max_ticks ticks ran.  Returns the final SimState and the per-tick records."""
    from dataclasses import replace
    tk = tracker or {}
    st = SimState(scene, cfg)
    z = sim_sense(st.obs, cfg.det_sigma, cfg.seed, trial, 0)
    tracks, missed = np.zeros((0, 20)), np.zeros(0, np.int32)
    # Alg. 1 "Initialize the 2D map and harmonic potential values" (C36): the static map and
    # goal, no tracks, relaxed cold to init_tol (checked every 100 sweeps)
    _, cls0, *_ = classify(replace(scene, tracks=np.zeros((0, 20))))
    u0 = init_u32(cls0)
    init_sweeps, _ = relax_f32(cls0, u0, cfg.init_max_sweeps, 100, cfg.init_tol)
    prev = {"u": u0, "init_sweeps": init_sweeps}
    recs = []
    Q = np.ascontiguousarray(scene.warp.Q, np.float64).reshape(16)
    lim = cfg.max_ticks if max_ticks is None else max_ticks
    while st.status[0] == SIM_RUNNING and st.ticks[0] < lim:
        _, tracks, missed = track_step(tracks, missed, z, dt=scene.warp.dt, Q=Q, **tk)
        th = math.atan2(st.rob[3], st.rob[2])
        sc = replace(scene, robot=(float(st.rob[0]), float(st.rob[1]), th, float(st.rob[4])), tracks=tracks)
        ref = plan_step(sc, max_sweeps=sweeps, iters=iters, max_len=max_len, prev=prev)
        wp = ref["next"] if ref.get("walk_status", -1) == OK else None
        sim_move(scene, st, wp, cfg, trial)
        recs.append({"rob": st.rob.copy(), "obs": st.obs.copy(), "n_tracks": len(tracks), "wp": wp,
                     "status": int(st.status[0]), "u": ref.get("u")})
        z = sim_sense(st.obs, cfg.det_sigma, cfg.seed, trial, int(st.ticks[0]))
        prev = ref
    st.tracks, st.missed = tracks, missed
    return st, recs
