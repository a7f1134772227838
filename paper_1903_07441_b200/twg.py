"""Thin ctypes binding of include/twg.h (argument marshalling only).

Every function below forwards to the C ABI of ``libtwg.so`` with the same name;
every step of the hot path runs in the library's sm_100a kernels.  Arrays may
be numpy arrays (host) or torch CUDA tensors (device); PyTorch is used only
for device memory and streams.  There is no CPU fallback: if the library is
missing or fails to load, :func:`lib` raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libtwg.so")
# TWG_LIB_PATH: an alternative build of the same library (kernel-variant timing experiments, tools/)
LIB_PATH = os.environ.get("TWG_LIB_PATH") or LIB_PATH

OK, W_GOAL_SWALLOWED, W_TRUNCATED = 0, 1, 2
E_INVALID_ARG, E_OUT_OF_BOUNDS, E_OVERLAPPING_CLASSES, E_INVALID_START = -1, -2, -3, -4
E_NO_PATH, E_CUDA, E_NCCL, E_NO_MEMORY = -5, -6, -7, -8
W_SINGULAR_INNOVATION = 3
RESIDENT_TRACKS = -1


class GridDesc(C.Structure):
    _fields_ = [("width", C.c_int32), ("height", C.c_int32), ("batch", C.c_int32), ("row_offset", C.c_int32),
                ("ghost_rows", C.c_int32), ("exchange_every", C.c_int32),
                ("cell_size", C.c_double), ("origin_x", C.c_double), ("origin_y", C.c_double)]


class Robot(C.Structure):
    _fields_ = [("x", C.c_double), ("y", C.c_double), ("theta", C.c_double), ("speed", C.c_double)]


class Track(C.Structure):
    _fields_ = [("x", C.c_double * 4), ("P", C.c_double * 16)]


class WarpCfg(C.Structure):
    _fields_ = [("dt", C.c_double), ("Q", C.c_double * 16), ("warp_spacing", C.c_double), ("eps_v", C.c_double),
                ("safety_radius", C.c_double), ("horizon_max", C.c_int32), ("horizon_mode", C.c_int32),
                ("footprint_mode", C.c_int32), ("reserved", C.c_int32)]


class RelaxCfg(C.Structure):
    _fields_ = [("max_sweeps", C.c_int32), ("check_every", C.c_int32), ("warm_start", C.c_int32),
                ("temporal_depth", C.c_int32), ("tol", C.c_float), ("rows_per_warp", C.c_int32),
                ("sync_every", C.c_int32), ("mode", C.c_int32)]


class BandCfg(C.Structure):
    _fields_ = [("iterations", C.c_int32), ("max_len", C.c_int32), ("max_smooth", C.c_int32),
                ("reserved", C.c_int32), ("step", C.c_float), ("k_t", C.c_float)]


class TrackerCfg(C.Structure):
    _fields_ = [("sigma_z", C.c_double), ("gate", C.c_double), ("spawn_var_pos", C.c_double),
                ("spawn_var_vel", C.c_double), ("prune_after", C.c_int32), ("max_tracks", C.c_int32)]


class SimCfg(C.Structure):
    _fields_ = [("dt", C.c_double), ("robot_radius", C.c_double), ("obstacle_radius", C.c_double),
                ("goal_radius", C.c_double), ("turn_distance", C.c_double), ("heading_sigma", C.c_double),
                ("det_sigma", C.c_double), ("turn_max", C.c_double), ("seed", C.c_uint64),
                ("max_ticks", C.c_int32), ("init_max_sweeps", C.c_int32), ("init_tol", C.c_float),
                ("reserved", C.c_int32)]


class SimTrial(C.Structure):
    _fields_ = [("x", C.c_double), ("y", C.c_double), ("hx", C.c_double), ("hy", C.c_double),
                ("speed", C.c_double), ("length", C.c_double), ("ticks", C.c_int32), ("status", C.c_int32)]


class PlanResult(C.Structure):
    _fields_ = [("status", C.c_int32), ("sweeps", C.c_int32), ("n_cells", C.c_int32), ("n_smooth", C.c_int32),
                ("residual", C.c_float), ("next_x", C.c_float), ("next_y", C.c_float), ("walk_status", C.c_int32)]


# (name, restype, argtypes) for every symbol of include/twg.h
_P = C.c_void_p
SIGNATURES = [
    ("twg_create", C.c_int32, [C.POINTER(GridDesc), C.c_int32, _P, _P, C.POINTER(_P)]),
    ("twg_create_group", C.c_int32, [C.POINTER(GridDesc), C.c_int32, C.c_int32, _P, _P]),
    ("twg_slab_info", C.c_int32, [_P, _P]),
    ("twg_nccl_unique_id", C.c_int32, [_P, C.c_int32]),
    ("twg_nccl_comm_init", C.c_int32, [C.c_int32, _P, C.c_int32, C.c_int32, C.POINTER(_P)]),
    ("twg_nccl_comm_destroy", C.c_int32, [_P]),
    ("twg_destroy", C.c_int32, [_P]),
    ("twg_set_static", C.c_int32, [_P, C.c_int32, _P]),
    ("twg_set_obstacles", C.c_int32, [_P, C.c_int32, C.POINTER(Robot), C.c_int32, C.c_int32, _P, C.c_int32,
                                      C.POINTER(WarpCfg), C.c_int32]),
    ("twg_relax", C.c_int32, [_P, C.POINTER(RelaxCfg), _P, _P]),
    ("twg_extract_path", C.c_int32, [_P, C.c_int32, C.POINTER(BandCfg), _P, _P, _P, _P, _P]),
    ("twg_plan_step", C.c_int32, [_P, C.c_int32, _P, _P, _P, _P, C.POINTER(WarpCfg), C.POINTER(RelaxCfg),
                                  C.POINTER(BandCfg), _P, _P, _P]),
    ("twg_get_field", C.c_int32, [_P, C.c_int32, _P, C.c_int32]),
    ("twg_set_field", C.c_int32, [_P, C.c_int32, _P]),
    ("twg_get_warp", C.c_int32, [_P, C.c_int32, C.c_int32, _P, _P, _P]),
    ("twg_track_update", C.c_int32, [_P, C.c_int32, _P, _P, C.POINTER(WarpCfg), C.POINTER(TrackerCfg), _P]),
    ("twg_get_tracks", C.c_int32, [_P, C.c_int32, _P, _P, C.c_int32, C.POINTER(C.c_int32)]),
    ("twg_sim_reset", C.c_int32, [_P, C.c_int32, C.POINTER(Robot), C.c_int32, C.c_int32, _P, C.c_int32,
                                  C.POINTER(SimCfg)]),
    ("twg_sim_tick", C.c_int32, [_P, C.POINTER(SimCfg), C.POINTER(WarpCfg), C.POINTER(RelaxCfg), C.POINTER(BandCfg),
                                 C.POINTER(TrackerCfg), _P, C.POINTER(C.c_int32)]),
    ("twg_sim_histogram", C.c_int32, [_P, C.c_int32, _P]),
    ("twg_walk_from", C.c_int32, [_P, C.c_int32, C.c_int32, C.c_int32, C.c_int32, _P, C.POINTER(C.c_int32),
                                  C.POINTER(C.c_int32), _P]),
    ("twg_index_matrix", C.c_int32, [_P, C.c_int32, _P]),
    ("twg_band_index", C.c_int32, [_P, C.c_int32, C.POINTER(BandCfg), _P, _P, C.POINTER(C.c_int32)]),
    ("twg_warp_map", C.c_int32, [_P, C.POINTER(Robot), C.c_double, _P]),
    ("twg_field_ptr", C.c_int32, [_P, C.c_int32, C.POINTER(_P), C.POINTER(C.c_int64)]),
    ("twg_debug_walk", C.c_int32, [_P, C.c_int32, _P]),
    ("twg_kernel_launches", C.c_int64, [_P]),
    ("twg_profile", C.c_int32, [_P, C.c_int32]),
    ("twg_profile_read", C.c_int32, [_P, C.POINTER(C.c_double), C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    ("twg_last_error", C.c_char_p, [_P]),
]

_lib = None


def lib():
    """Load libtwg.so (raises if it is missing: there is no fallback path)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is not built; run __graft_entry__.build()")
        L = C.CDLL(LIB_PATH)
        for name, res, args in SIGNATURES:
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


class TwgError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"twg status {status}: {msg}")
        self.status = status


def _ptr(a):
    """Raw address of a numpy array or torch tensor (None -> NULL)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        assert a.flags.c_contiguous
        return a.ctypes.data
    if hasattr(a, "data_ptr"):
        assert a.is_contiguous()
        return a.data_ptr()
    raise TypeError(type(a))


def _check(ctx, st, ok=(OK, W_GOAL_SWALLOWED, W_TRUNCATED)):
    if st not in ok:
        raise TwgError(st, lib().twg_last_error(ctx).decode())
    return st


def warp_cfg(dt=0.1, Q=None, warp_spacing=1.0, eps_v=0.05, safety_radius=0.5, horizon_max=20, horizon_mode=0,
             footprint_mode=0):
    c = WarpCfg()
    c.dt = dt
    q = np.zeros(16) if Q is None else np.asarray(Q, np.float64).reshape(16)
    if Q is None:
        q[0] = q[5] = 1e-3 * dt ** 4 / 4.0
        q[10] = q[15] = 1e-3 * dt ** 2
    for k in range(16):
        c.Q[k] = float(q[k])
    c.warp_spacing, c.eps_v, c.safety_radius, c.horizon_max = warp_spacing, eps_v, safety_radius, horizon_max
    c.horizon_mode, c.footprint_mode = horizon_mode, footprint_mode
    return c


def relax_cfg(max_sweeps=100, check_every=0, warm_start=1, temporal_depth=0, tol=0.0, rows_per_warp=0,
              sync_every=0, mode=0):
    """mode 0: red-black Gauss-Seidel (Eq. 2); 1: Jacobi (Eq. 1); 2: lexicographic Gauss-Seidel."""
    return RelaxCfg(max_sweeps, check_every, warm_start, temporal_depth, tol, rows_per_warp, sync_every, mode)


def tracker_cfg(sigma_z=0.05, gate=0.5, spawn_var_pos=0.25, spawn_var_vel=1.0, prune_after=10, max_tracks=0):
    return TrackerCfg(sigma_z, gate, spawn_var_pos, spawn_var_vel, prune_after, max_tracks)


def sim_cfg(dt=0.1, robot_radius=0.25, obstacle_radius=0.25, goal_radius=0.3, turn_distance=0.5, heading_sigma=0.02,
            det_sigma=0.05, turn_max=0.15707963267948966, seed=1, max_ticks=1000, init_max_sweeps=1_000_000,
            init_tol=1e-6):
    return SimCfg(dt, robot_radius, obstacle_radius, goal_radius, turn_distance, heading_sigma, det_sigma, turn_max,
                  seed, max_ticks, init_max_sweeps, init_tol, 0)


def band_cfg(iterations=50, max_len=4096, max_smooth=8192, step=0.25, k_t=1.0):
    return BandCfg(iterations, max_len, max_smooth, 0, step, k_t)


def tracks_array(tracks):
    """float64 [n, 20] (x[4], P[16]) -> contiguous array with the twg_track layout."""
    t = np.ascontiguousarray(np.asarray(tracks, np.float64).reshape(-1, 20))
    return t


def nccl_unique_id() -> bytes:
    """twg_nccl_unique_id: 128 opaque bytes to broadcast to every rank."""
    buf = (C.c_uint8 * 128)()
    st = lib().twg_nccl_unique_id(buf, 128)
    if st != OK:
        raise TwgError(st, lib().twg_last_error(None).decode())
    return bytes(buf)


def nccl_comm_init(nranks: int, uid: bytes, rank: int, device: int) -> int:
    """twg_nccl_comm_init: an ncclComm_t (as an integer handle) for `rank` of `nranks`."""
    buf = (C.c_uint8 * 128).from_buffer_copy(uid)
    h = C.c_void_p()
    st = lib().twg_nccl_comm_init(int(nranks), buf, int(rank), int(device), C.byref(h))
    if st != OK:
        raise TwgError(st, lib().twg_last_error(None).decode())
    return h.value


def nccl_comm_destroy(comm: int):
    st = lib().twg_nccl_comm_destroy(C.c_void_p(comm))
    if st != OK:
        raise TwgError(st, lib().twg_last_error(None).decode())


class Planner:
    """Owns one twg_ctx.  Method names mirror the C ABI (twg_<name>).

    nccl_comm (an ncclComm_t handle, e.g. from :func:`nccl_comm_init`) with exchange_every = k makes
    this context the caller's row slab of the global width x height grid (twg_create)."""

    def __init__(self, width, height, batch=1, cell_size=0.1, origin=(0.0, 0.0), device=0, stream=None,
                 row_offset=0, ghost_rows=0, nccl_comm=None, exchange_every=0, _ctx=None):
        self.W, self.B = int(width), int(batch)
        if _ctx is not None:  # a member of twg_create_group
            self.ctx = _ctx
        else:
            d = GridDesc(self.W, int(height), self.B, int(row_offset), int(ghost_rows), int(exchange_every),
                         float(cell_size), float(origin[0]), float(origin[1]))
            h = C.c_void_p()
            st = lib().twg_create(C.byref(d), int(device), stream, None if nccl_comm is None else C.c_void_p(nccl_comm),
                                  C.byref(h))
            if st != OK:
                raise TwgError(st, lib().twg_last_error(None).decode())
            self.ctx = h
        info = self.slab_info()
        self.rank, self.nranks, self.r0, self.r1 = info[0], info[1], info[2], info[3]
        self.row_offset, self.ghost_rows, self.exchange_every, self.H = info[4], info[5], info[6], info[7]

    @staticmethod
    def create_group(width, height, nslabs, exchange_every, cell_size=0.1, origin=(0.0, 0.0), device=0, stream=None):
        """twg_create_group: nslabs row-slab Planners of one global grid on one device (local group)."""
        d = GridDesc(int(width), int(height), 1, 0, 0, int(exchange_every), float(cell_size), float(origin[0]),
                     float(origin[1]))
        hs = (C.c_void_p * int(nslabs))()
        st = lib().twg_create_group(C.byref(d), int(nslabs), int(device), stream, hs)
        if st != OK:
            raise TwgError(st, lib().twg_last_error(None).decode())
        return [Planner(width, 0, 1, _ctx=C.c_void_p(hs[r])) for r in range(int(nslabs))]

    def slab_info(self):
        out = np.zeros(8, np.int32)
        _check(self.ctx, lib().twg_slab_info(self.ctx, _ptr(out)))
        return [int(v) for v in out]

    def close(self):
        if self.ctx:
            lib().twg_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- a1-a3
    def set_static(self, occ, b=-1):
        return _check(self.ctx, lib().twg_set_static(self.ctx, b, _ptr(occ)))

    def set_obstacles(self, b, robot, goal, tracks, cfg, warm=0):
        """tracks=None: use the resident tracker table (twg_track_update)."""
        r = Robot(*[float(v) for v in robot])
        if tracks is None:
            return _check(self.ctx, lib().twg_set_obstacles(self.ctx, b, C.byref(r), int(goal[0]), int(goal[1]),
                                                            None, RESIDENT_TRACKS, C.byref(cfg), int(warm)))
        t = tracks if hasattr(tracks, "data_ptr") else tracks_array(tracks)
        n = int(t.shape[0])
        return _check(self.ctx, lib().twg_set_obstacles(self.ctx, b, C.byref(r), int(goal[0]), int(goal[1]),
                                                        _ptr(t) if n else None, n, C.byref(cfg), int(warm)))

    # -- a4-a6
    def relax(self, cfg, want_result=True):
        if not want_result:
            _check(self.ctx, lib().twg_relax(self.ctx, C.byref(cfg), None, None))
            return None, None
        sw = np.zeros(self.B, np.int32)
        res = np.zeros(self.B, np.float32)
        _check(self.ctx, lib().twg_relax(self.ctx, C.byref(cfg), _ptr(sw), _ptr(res)))
        return sw, res

    # -- a7-a9
    def extract_path(self, b, cfg):
        cells = np.zeros((cfg.max_len, 2), np.int32)
        sm = np.zeros((cfg.max_smooth, 2), np.float32)
        nc = C.c_int32()
        ns = C.c_int32()
        nxt = np.zeros(2, np.float32)
        st = lib().twg_extract_path(self.ctx, b, C.byref(cfg), _ptr(cells), C.byref(nc), _ptr(sm), C.byref(ns),
                                    _ptr(nxt))
        _check(self.ctx, st, ok=(OK, W_TRUNCATED, E_NO_PATH))
        return st, cells[: nc.value].copy(), sm[: min(ns.value, cfg.max_smooth)].copy(), ns.value, (float(nxt[0]), float(nxt[1]))

    def plan_step(self, b, robots, goals, tracks, n_tracks, wcfg, rcfg, bcfg, want_paths=True):
        """b >= 0: one scenario; b = -1: all.  tracks: concatenated [sum n, 20] (numpy or CUDA tensor)."""
        nb = 1 if b >= 0 else self.B
        rob = np.ascontiguousarray(np.asarray(robots, np.float64).reshape(nb, 4))  # twg_robot = 4 doubles
        g = np.ascontiguousarray(np.asarray(goals, np.int32).reshape(nb, 2))
        resident = tracks is None and n_tracks is None
        nt = None if resident else np.ascontiguousarray(np.asarray(n_tracks, np.int32).reshape(nb))
        t = None if resident else (tracks if hasattr(tracks, "data_ptr") else tracks_array(tracks))
        out = (PlanResult * nb)()
        cells = np.zeros((nb, bcfg.max_len, 2), np.int32) if want_paths else None
        sm = np.zeros((nb, bcfg.max_smooth, 2), np.float32) if want_paths else None
        st = lib().twg_plan_step(self.ctx, b, _ptr(rob), _ptr(g), _ptr(t) if (nt is not None and int(nt.sum())) else None,
                                 _ptr(nt),
                                 C.byref(wcfg), C.byref(rcfg), C.byref(bcfg), out, _ptr(cells), _ptr(sm))
        _check(self.ctx, st, ok=(OK, W_GOAL_SWALLOWED, W_TRUNCATED, E_NO_PATH))
        return st, list(out), cells, sm

    # -- field access
    def get_field(self, b=0, mode=1, out=None):
        if out is None:
            out = np.zeros((self.H, self.W), np.float32)
        _check(self.ctx, lib().twg_get_field(self.ctx, b, _ptr(out), int(mode)))
        return out

    def set_field(self, raw, b=0):
        return _check(self.ctx, lib().twg_set_field(self.ctx, b, _ptr(raw)))

    def get_warp(self, b, n):
        t = np.zeros(max(n, 1), np.int32)
        j = np.zeros(max(n, 1), np.int32)
        pred = np.zeros((max(n, 1), 3))
        _check(self.ctx, lib().twg_get_warp(self.ctx, b, n, _ptr(t), _ptr(j), _ptr(pred)))
        return t[:n], j[:n], pred[:n]

    # -- f1 tracker
    def track_update(self, b, det, n_det, wcfg, tcfg):
        """twg_track_update: det [sum n_det, 2] float64 (numpy or CUDA tensor); returns (status, n_tracks)."""
        nb = 1 if b >= 0 else self.B
        nd = np.ascontiguousarray(np.asarray(n_det, np.int32).reshape(nb))
        d = det if hasattr(det, "data_ptr") else np.ascontiguousarray(np.asarray(det, np.float64).reshape(-1, 2))
        nt = np.zeros(nb, np.int32)
        st = lib().twg_track_update(self.ctx, b, _ptr(d) if int(nd.sum()) else None, _ptr(nd), C.byref(wcfg),
                                    C.byref(tcfg), _ptr(nt))
        _check(self.ctx, st, ok=(OK, W_TRUNCATED, W_SINGULAR_INNOVATION))
        return st, nt

    def get_tracks(self, b=0):
        """twg_get_tracks: (tracks [n, 20] float64, missed [n] int32) of the resident table."""
        n = C.c_int32()
        _check(self.ctx, lib().twg_get_tracks(self.ctx, b, None, None, 0, C.byref(n)))
        out = np.zeros((max(n.value, 1), 20))
        mis = np.zeros(max(n.value, 1), np.int32)
        _check(self.ctx, lib().twg_get_tracks(self.ctx, b, _ptr(out), _ptr(mis), n.value, C.byref(n)))
        return out[: n.value], mis[: n.value]

    # -- f2 closed-loop simulator
    def sim_reset(self, b, robot, goal, obstacles, cfg):
        """twg_sim_reset: obstacles [n, 4] (x, y, vx, vy) true states."""
        o = np.ascontiguousarray(np.asarray(obstacles, np.float64).reshape(-1, 4))
        r = Robot(*[float(v) for v in robot])
        return _check(self.ctx, lib().twg_sim_reset(self.ctx, b, C.byref(r), int(goal[0]), int(goal[1]),
                                                    _ptr(o) if len(o) else None, len(o), C.byref(cfg)))

    def sim_tick(self, cfg, wcfg, rcfg, bcfg, tcfg):
        """twg_sim_tick: returns (status, [SimTrial] * batch, running)."""
        out = (SimTrial * self.B)()
        run = C.c_int32()
        st = lib().twg_sim_tick(self.ctx, C.byref(cfg), C.byref(wcfg), C.byref(rcfg), C.byref(bcfg), C.byref(tcfg),
                                out, C.byref(run))
        _check(self.ctx, st, ok=(OK, W_GOAL_SWALLOWED, W_TRUNCATED, W_SINGULAR_INNOVATION))
        return st, list(out), run.value

    def sim_histogram(self, b=0):
        h = np.zeros(36, np.int32)
        _check(self.ctx, lib().twg_sim_histogram(self.ctx, b, _ptr(h)))
        return h

    def walk_from(self, b, x, y, max_cells):
        """twg_walk_from: (code, cells [n, 2] local, next (x, y) local or None); code 0 goal, 1 / 2 handed
        to the slab above / below, E_NO_PATH."""
        cells = np.zeros((max(max_cells, 1), 2), np.int32)
        n, code = C.c_int32(), C.c_int32()
        nxt = np.zeros(2, np.int32)
        _check(self.ctx, lib().twg_walk_from(self.ctx, b, int(x), int(y), int(max_cells), _ptr(cells), C.byref(n),
                                             C.byref(code), _ptr(nxt)))
        c = code.value
        return c, cells[: n.value].copy(), (int(nxt[0]), int(nxt[1])) if c in (1, 2) else None

    def index_matrix(self, b=0, out=None):
        """twg_index_matrix: uint8 [H, W] M_idx of scenario b (0..3 move, 4 goal, 5 obstacle, 6 none)."""
        out = np.zeros((self.H, self.W), np.uint8) if out is None else out
        _check(self.ctx, lib().twg_index_matrix(self.ctx, b, _ptr(out)))
        return out

    def band_index(self, b, cfg, out=None):
        """twg_band_index (f3 per-cell band): (status, optimised uint8 [H, W] matrix, walk cells [n, 2])."""
        out = np.zeros((self.H, self.W), np.uint8) if out is None else out
        cells = np.zeros((cfg.max_len, 2), np.int32)
        n = C.c_int32()
        st = lib().twg_band_index(self.ctx, b, C.byref(cfg), _ptr(out), _ptr(cells), C.byref(n))
        _check(self.ctx, st, ok=(OK, E_NO_PATH))
        return st, out, cells[: n.value].copy()

    def warp_map(self, robot, warp_spacing=1.0, out=None):
        """twg_warp_map: int32 [H, W] warp number of every cell centre for the robot pose."""
        out = np.zeros((self.H, self.W), np.int32) if out is None else out
        r = Robot(*[float(v) for v in robot])
        _check(self.ctx, lib().twg_warp_map(self.ctx, C.byref(r), float(warp_spacing), _ptr(out)))
        return out

    def field_ptr(self, b=0):
        p = C.c_void_p()
        pitch = C.c_int64()
        _check(self.ctx, lib().twg_field_ptr(self.ctx, b, C.byref(p), C.byref(pitch)))
        return p.value, pitch.value

    def debug_walk(self, b=0):
        out = np.zeros(4, np.int32)
        _check(self.ctx, lib().twg_debug_walk(self.ctx, b, _ptr(out)))
        return {"stage_kcyc": int(out[0]), "chase_kcyc": int(out[1]), "flush_kcyc": int(out[2]), "windows": int(out[3])}

    def kernel_launches(self):
        return int(lib().twg_kernel_launches(self.ctx))

    def profile(self, enable):
        return _check(self.ctx, lib().twg_profile(self.ctx, int(enable)))

    def profile_read(self):
        ms = C.c_double()
        nl = C.c_int64()
        cells = C.c_int64()
        _check(self.ctx, lib().twg_profile_read(self.ctx, C.byref(ms), C.byref(nl), C.byref(cells)))
        return ms.value, nl.value, cells.value
