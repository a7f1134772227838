"""GPU <-> oracle parity of the SURVEY.md 8(f) rows through the C ABI (libtwg.so).

f3: Jacobi relaxation (twg_relax_cfg.mode = 1; Eq. 1), the full-grid index matrix
    (twg_index_matrix; Eq. 3) and the per-cell warp map (twg_warp_map).
f4: the ring-time horizon and posterior-covariance footprint readings (twg_warp_cfg
    horizon_mode / footprint_mode; C26, C27).
Bars as for rows a1-a9: integer outputs and the fp32 field bit-exact (the 1e-5 gate asserted too).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import oracle  # noqa: E402
from paper_1903_07441_b200 import Planner, band_cfg, relax_cfg, warp_cfg  # noqa: E402
from paper_1903_07441_b200 import twg as T  # noqa: E402
from scenes import scene_c1, scene_c2, scene_random, advance_scene, default_warp_cfg  # noqa: E402
from scenes.gen import Scene  # noqa: E402


def _stream():
    return torch.cuda.current_stream().cuda_stream


def _planner(sc, batch=1):
    pl = Planner(sc.W, sc.H, batch, sc.cell_size, sc.origin, device=0, stream=_stream())
    pl.set_static(sc.static)
    return pl


def _assert_field(u_gpu, u_ref):
    assert np.max(np.abs(u_gpu - u_ref)) <= 1e-5
    assert np.array_equal(u_gpu, u_ref)


def _rand_scene(W, H, seed, p_wall=0.08):
    rng = np.random.default_rng(seed)
    static = (rng.random((H, W)) < p_wall).astype(np.uint8)
    g = (int(rng.integers(0, W)), int(rng.integers(0, H)))
    r = (int(rng.integers(0, W)), int(rng.integers(0, H)))
    static[g[1], g[0]] = 0
    static[r[1], r[0]] = 0
    return Scene("t", W, H, 0.1, (0.0, 0.0), static, ((r[0] + 0.5) * 0.1, (r[1] + 0.5) * 0.1, 0.3, 0.4), g,
                 np.zeros((0, 20)), default_warp_cfg(), seed)


# ------------------------------------------------------------------ f3 Jacobi
@pytest.mark.parametrize("W,H", [(64, 64), (300, 211), (129, 1000), (1000, 37), (1, 1), (5, 3), (2048, 70)])
def test_jacobi_fixed_budget(W, H):
    sc = _rand_scene(W, H, W * 3 + H)
    pl = _planner(sc)
    pl.set_obstacles(0, sc.robot, sc.goal, sc.tracks, warp_cfg(), warm=0)
    S = 41
    sw, res = pl.relax(relax_cfg(max_sweeps=S, mode=1))
    _, cls, *_ = oracle.classify(sc)
    u = oracle.init_u32(cls)
    s_ref, r_ref = oracle.relax_jacobi_f32(cls, u, S, S, 0.0)
    assert int(sw[0]) == s_ref == S and np.float32(res[0]) == np.float32(r_ref)
    _assert_field(pl.get_field(0, 1), u)


@pytest.mark.parametrize("check_every", [1, 7])
def test_jacobi_c1_tolerance_stop(check_every):
    sc = scene_c1()
    pl = _planner(sc)
    pl.set_obstacles(0, sc.robot, sc.goal, sc.tracks, warp_cfg(), warm=0)
    sw, res = pl.relax(relax_cfg(max_sweeps=100_000, check_every=check_every, tol=1e-5, sync_every=4, mode=1))
    ref = oracle.plan_step(sc, max_sweeps=100_000, check_every=check_every, tol=1e-5, iters=0, jacobi=True)
    assert int(sw[0]) == ref["sweeps"] < 100_000 and int(sw[0]) % check_every == 0
    assert np.float32(res[0]) == np.float32(ref["residual"])
    _assert_field(pl.get_field(0, 1), ref["u"])
    # Jacobi needs about twice the red-black sweeps for the same tolerance (spectral radius squared)
    pl2 = _planner(sc)
    pl2.set_obstacles(0, sc.robot, sc.goal, sc.tracks, warp_cfg(), warm=0)
    sw_rb, _ = pl2.relax(relax_cfg(max_sweeps=100_000, check_every=check_every, tol=1e-5))
    assert 1.6 * sw_rb[0] < sw[0] < 2.4 * sw_rb[0]


def test_jacobi_batch_mixed_and_end_to_end():
    scs = [scene_random(f"b{k}", 160, 5, 6, 40 + k) for k in range(3)]
    pl = Planner(160, 160, 3, 0.1, (0.0, 0.0), device=0, stream=_stream())
    for k, sc in enumerate(scs):
        pl.set_static(sc.static, b=k)
    robots = [sc.robot for sc in scs]
    goals = [sc.goal for sc in scs]
    tracks = np.concatenate([sc.tracks for sc in scs])
    nt = [sc.n_tracks for sc in scs]
    rc = relax_cfg(max_sweeps=3000, check_every=10, tol=2e-5, warm_start=0, mode=1)
    st, res, cells, sm = pl.plan_step(-1, robots, goals, tracks, nt, warp_cfg(), rc, band_cfg(30, 2000, 4000))
    for k, sc in enumerate(scs):
        ref = oracle.plan_step(sc, max_sweeps=3000, check_every=10, tol=2e-5, iters=30, max_len=2000, jacobi=True)
        assert res[k].sweeps == ref["sweeps"]
        _assert_field(pl.get_field(k, 1), ref["u"])
        if ref["walk_status"] == 0:
            n = res[k].n_cells
            assert np.array_equal(cells[k, :n], ref["cells"])
            assert np.array_equal(sm[k, :res[k].n_smooth], ref["smooth"])


def test_jacobi_invalid_mode():
    sc = scene_c1()
    pl = _planner(sc)
    pl.set_obstacles(0, sc.robot, sc.goal, sc.tracks, warp_cfg(), warm=0)
    with pytest.raises(T.TwgError):
        pl.relax(relax_cfg(max_sweeps=3, mode=3))


# ------------------------------------------------------------------ f3 index matrix
@pytest.mark.parametrize("W,H,S", [(64, 64, 3000), (300, 211, 500), (1, 1, 1), (2, 1, 3), (1000, 37, 200)])
def test_index_matrix_bit_exact(W, H, S):
    sc = _rand_scene(W, H, W + 5 * H, p_wall=0.1)
    pl = _planner(sc)
    pl.set_obstacles(0, sc.robot, sc.goal, sc.tracks, warp_cfg(), warm=0)
    pl.relax(relax_cfg(max_sweeps=S))
    _, cls, *_ = oracle.classify(sc)
    u = oracle.init_u32(cls)
    oracle.relax_f32(cls, u, S, S, 0.0)
    _assert_field(pl.get_field(0, 1), u)
    m = pl.index_matrix(0)
    assert np.array_equal(m, oracle.index_matrix(cls, u))
    # device output
    d = torch.zeros((H, W), dtype=torch.uint8, device="cuda")
    pl.index_matrix(0, out=d)
    assert np.array_equal(d.cpu().numpy(), m)


def test_index_matrix_batch_scenario_select():
    scs = [scene_random(f"m{k}", 128, 4, 5, 70 + k) for k in range(2)]
    pl = Planner(128, 128, 2, 0.1, (0.0, 0.0), device=0, stream=_stream())
    for k, sc in enumerate(scs):
        pl.set_static(sc.static, b=k)
        pl.set_obstacles(k, sc.robot, sc.goal, sc.tracks, warp_cfg(), warm=0)
    pl.relax(relax_cfg(max_sweeps=77, temporal_depth=5))
    for k, sc in enumerate(scs):
        _, cls, *_ = oracle.classify(sc)
        u = oracle.init_u32(cls)
        oracle.relax_f32(cls, u, 77, 77, 0.0)
        assert np.array_equal(pl.index_matrix(k), oracle.index_matrix(cls, u))


# ------------------------------------------------------------------ f3 warp map
@pytest.mark.parametrize("W,H", [(64, 64), (333, 97), (1, 1), (1024, 8)])
@pytest.mark.parametrize("theta,w", [(0.0, 1.0), (0.7, 0.35), (-2.9, 2.0)])
def test_warp_map_bit_exact(W, H, theta, w):
    rng = np.random.default_rng(W + H)
    origin = (-1.3, 2.2)
    robot = (origin[0] + rng.uniform(0, W * 0.1), origin[1] + rng.uniform(0, H * 0.1), theta, 0.4)
    pl = Planner(W, H, 1, 0.1, origin, device=0, stream=_stream())
    sc = Scene("wm", W, H, 0.1, origin, np.zeros((H, W), np.uint8), robot, (0, 0), np.zeros((0, 20)),
               default_warp_cfg(), 0)
    sc.warp.warp_spacing = w
    got = pl.warp_map(robot, w)
    assert np.array_equal(got, oracle.warp_map(sc))
    d = torch.zeros((H, W), dtype=torch.int32, device="cuda")
    pl.warp_map(robot, w, out=d)
    assert np.array_equal(d.cpu().numpy(), got)
    with pytest.raises(T.TwgError):
        pl.warp_map(robot, 0.0)


@pytest.mark.parametrize("w", [0.05, 0.35, 3.0])
@pytest.mark.parametrize("centred", [False, True])
def test_warp_map_bit_exact_large(w, centred):
    # 2048^2 (4.2 M cells, hundreds of thousands on or next to ring boundaries at small w): the fp32
    # screen of k_warp_map must hand every undecided cell to the fp64 sequence.  A robot at a cell
    # centre gives a cell with d = 0 and rings through cell centres along the axes.
    W = H = 2048
    origin = (1000.3, -2000.7)
    xr = origin[0] + (1000 + 0.5) * 0.1 if centred else origin[0] + 100.0123
    yr = origin[1] + (700 + 0.5) * 0.1 if centred else origin[1] + 71.9
    robot = (xr, yr, 0.0 if centred else 2.2, 0.4)
    pl = Planner(W, H, 1, 0.1, origin, device=0, stream=_stream())
    sc = Scene("wm", W, H, 0.1, origin, np.zeros((H, W), np.uint8), robot, (0, 0), np.zeros((0, 20)),
               default_warp_cfg(), 0)
    sc.warp.warp_spacing = w
    assert np.array_equal(pl.warp_map(robot, w), oracle.warp_map(sc))


def test_warp_map_agrees_with_track_labels():
    # a track sitting exactly at a cell centre gets that cell's warp number (rows a1 vs f3)
    sc = scene_random("wl", 256, 6, 30, 5)
    pl = _planner(sc)
    pl.set_obstacles(0, sc.robot, sc.goal, sc.tracks, warp_cfg(), warm=0)
    tr = sc.tracks.copy()
    cx = np.floor(tr[:, 0] / 0.1).astype(int).clip(0, 255)
    cy = np.floor(tr[:, 1] / 0.1).astype(int).clip(0, 255)
    tr[:, 0] = (cx + 0.5) * 0.1
    tr[:, 1] = (cy + 0.5) * 0.1
    pl.set_obstacles(0, sc.robot, sc.goal, tr, warp_cfg(), warm=0)
    t, _, _ = pl.get_warp(0, len(tr))
    m = pl.warp_map(sc.robot, sc.warp.warp_spacing)
    assert np.array_equal(t, m[cy, cx])


# ------------------------------------------------------------------ f4 horizon / footprint readings
@pytest.mark.parametrize("hm,fm", [(1, 0), (0, 1), (1, 1)])
@pytest.mark.parametrize("seed", [0, 4])
def test_horizon_footprint_modes_bit_exact(hm, fm, seed):
    sc = scene_random("hf", 500, 12, 50, seed)
    pl = _planner(sc)
    st = pl.set_obstacles(0, sc.robot, sc.goal, sc.tracks, warp_cfg(horizon_mode=hm, footprint_mode=fm), warm=0)
    ost, cls, t, j, pred = oracle.classify(sc, hm, fm)
    assert st == ost
    tg, jg, pg = pl.get_warp(0, sc.n_tracks)
    assert np.array_equal(tg, t) and np.array_equal(jg, j) and np.array_equal(pg, pred)
    raw = pl.get_field(0, 0)
    bits = raw.view(np.uint32)
    gcls = np.zeros(raw.shape, np.uint8)
    gcls[bits == 0] = oracle.OBSTACLE
    gcls[bits == 0x3F800000] = oracle.GOAL
    assert np.array_equal(gcls, cls)
    # the readings differ from the default ones on this scene
    _, cls0, _, j0, _ = oracle.classify(sc)
    assert not np.array_equal(cls0, cls) or not np.array_equal(j0, j)


def test_modes_warm_plan_loop():
    sc = scene_c2(3)
    pl = _planner(sc)
    wc = warp_cfg(horizon_mode=1, footprint_mode=1)
    rc = relax_cfg(max_sweeps=60, warm_start=1)
    bc = band_cfg(20, 3000, 6000)
    prev = None
    for tick in range(3):
        s = advance_scene(sc, tick)
        st, res, cells, sm = pl.plan_step(0, [s.robot], [s.goal], s.tracks, [s.n_tracks], wc, rc, bc)
        ref = oracle.plan_step(s, max_sweeps=60, iters=20, max_len=3000, prev=prev, horizon_mode=1,
                               footprint_mode=1)
        _assert_field(pl.get_field(0, 1), ref["u"])
        if ref["walk_status"] == 0:
            assert np.array_equal(cells[0, :res[0].n_cells], ref["cells"])
        prev = ref


def test_invalid_modes_rejected():
    sc = scene_c1()
    pl = _planner(sc)
    with pytest.raises(T.TwgError):
        pl.set_obstacles(0, sc.robot, sc.goal, sc.tracks, warp_cfg(horizon_mode=2), warm=0)
    with pytest.raises(T.TwgError):
        pl.set_obstacles(0, sc.robot, sc.goal, sc.tracks, warp_cfg(footprint_mode=-1), warm=0)


# ------------------------------------------------------------------ f3 lexicographic Gauss-Seidel
@pytest.mark.parametrize("W,H", [(64, 64), (300, 211), (33, 97), (1, 1), (5, 3), (1000, 40)])
def test_lex_fixed_budget(W, H):
    sc = _rand_scene(W, H, W * 5 + H)
    pl = _planner(sc)
    pl.set_obstacles(0, sc.robot, sc.goal, sc.tracks, warp_cfg(), warm=0)
    S = 23
    sw, res = pl.relax(relax_cfg(max_sweeps=S, mode=2))
    _, cls, *_ = oracle.classify(sc)
    u = oracle.init_u32(cls)
    s_ref, r_ref = oracle.relax_lex_f32(cls, u, S, S, 0.0)
    assert int(sw[0]) == s_ref == S and np.float32(res[0]) == np.float32(r_ref)
    _assert_field(pl.get_field(0, 1), u)


def test_lex_tolerance_batch_and_plan():
    scs = [scene_random(f"lx{k}", 128, 3, 4, 90 + k) for k in range(3)]
    pl = Planner(128, 128, 3, 0.1, (0.0, 0.0), device=0, stream=_stream())
    for k, sc in enumerate(scs):
        pl.set_static(sc.static, b=k)
    rc = relax_cfg(max_sweeps=4000, check_every=25, tol=1e-5, warm_start=0, mode=2, sync_every=2)
    st, res, cells, sm = pl.plan_step(-1, [s.robot for s in scs], [s.goal for s in scs],
                                      np.concatenate([s.tracks for s in scs]), [s.n_tracks for s in scs],
                                      warp_cfg(), rc, band_cfg(10, 2000, 4000))
    for k, sc in enumerate(scs):
        ref = oracle.plan_step(sc, max_sweeps=4000, check_every=25, tol=1e-5, iters=10, max_len=2000, lex=True)
        assert res[k].sweeps == ref["sweeps"] and res[k].sweeps % 25 == 0
        _assert_field(pl.get_field(k, 1), ref["u"])
        if ref["walk_status"] == 0:
            assert np.array_equal(cells[k, :res[k].n_cells], ref["cells"])


def test_lex_large_grid_sampled():
    # 2048^2, 6 sweeps: parity on row bands (the oracle relaxes the full grid)
    sc = scene_random("lxL", 2048, 64, 100, 3)
    pl = _planner(sc)
    pl.set_obstacles(0, sc.robot, sc.goal, sc.tracks, warp_cfg(), warm=0)
    sw, res = pl.relax(relax_cfg(max_sweeps=6, mode=2))
    _, cls, *_ = oracle.classify(sc)
    u = oracle.init_u32(cls)
    s_ref, r_ref = oracle.relax_lex_f32(cls, u, 6, 6, 0.0)
    assert np.float32(res[0]) == np.float32(r_ref)
    _assert_field(pl.get_field(0, 1), u)
