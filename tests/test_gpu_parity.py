"""GPU <-> oracle parity through the C ABI (libtwg.so), rows a1-a9.

Bars: stamped class grid, walk cells and per-track t/j
bit-exact; the fp32 field bit-exact (the BASELINE.json gate of 1e-5 of the
potential range is the backstop and is asserted too); the smoothed path
bit-exact target with a 1e-4 cell gate; sweeps and residual equal.
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
from scenes import scene_c1, scene_c2, scene_random, advance_scene, random_small_map  # noqa: E402


def _stream():
    return torch.cuda.current_stream().cuda_stream


def _planner(sc, batch=1):
    pl = Planner(sc.W, sc.H, batch, sc.cell_size, sc.origin, device=0, stream=_stream())
    pl.set_static(sc.static)
    return pl


def _classes_from_raw(raw):
    bits = raw.view(np.uint32)
    cls = np.zeros(raw.shape, np.uint8)
    cls[bits == 0] = oracle.OBSTACLE
    cls[bits == 0x3F800000] = oracle.GOAL
    return cls


def _assert_field(u_gpu, u_ref):
    assert np.max(np.abs(u_gpu - u_ref)) <= 1e-5  # BASELINE.json north_star gate (range of u is 1)
    assert np.array_equal(u_gpu, u_ref)


# ------------------------------------------------------------------ C1 end to end
@pytest.mark.parametrize("check_every", [1, 8])
def test_c1_end_to_end(check_every):
    sc = scene_c1()
    pl = _planner(sc)
    pl.set_obstacles(0, sc.robot, sc.goal, sc.tracks, warp_cfg(), warm=0)
    sw, res = pl.relax(relax_cfg(max_sweeps=10 ** 6, check_every=check_every, tol=1e-6))
    ref = oracle.plan_step(sc, max_sweeps=10 ** 6, check_every=check_every, tol=1e-6, iters=50, max_len=2000)
    assert int(sw[0]) == ref["sweeps"] == (1347 if check_every == 1 else 1352)
    assert np.float32(res[0]) == np.float32(ref["residual"])
    _assert_field(pl.get_field(0, 1), ref["u"])
    st, cells, smooth, ns, nxt = pl.extract_path(0, band_cfg(50, 2000, 8000))
    assert st == T.OK and np.array_equal(cells, ref["cells"])
    assert smooth.shape == ref["smooth"].shape and np.abs(smooth - ref["smooth"]).max() <= 1e-4
    assert np.array_equal(smooth, ref["smooth"])
    assert np.allclose(nxt, ref["next"], atol=1e-4)


# ------------------------------------------------------------------ a4-a6 tiling / T / ragged tails
@pytest.mark.parametrize("W,H", [(300, 211), (1000, 37), (129, 1000), (1, 1), (5, 3), (2048, 64)])
@pytest.mark.parametrize("T_", [1, 2, 3, 4, 5, 8])
def test_relax_fixed_budget_all_T(W, H, T_):
    rng = np.random.default_rng(W * 7 + H + T_)
    static = (rng.random((H, W)) < 0.08).astype(np.uint8)
    g = (int(rng.integers(0, W)), int(rng.integers(0, H)))
    static[g[1], g[0]] = 0
    from scenes.gen import Scene
    from scenes import default_warp_cfg
    sc = Scene("t", W, H, 0.1, (0.0, 0.0), static, ((g[0] + 0.5) * 0.1, (g[1] + 0.5) * 0.1, 0.0, 0.4), g,
               np.zeros((0, 20)), default_warp_cfg(), 0)
    pl = _planner(sc)
    pl.set_obstacles(0, sc.robot, sc.goal, sc.tracks, warp_cfg(), warm=0)
    S = 37
    sw, res = pl.relax(relax_cfg(max_sweeps=S, temporal_depth=T_))
    st, cls, *_ = oracle.classify(sc)
    u = oracle.init_u32(cls)
    s_ref, r_ref = oracle.relax_f32(cls, u, S, S, 0.0)
    assert int(sw[0]) == s_ref == S and np.float32(res[0]) == np.float32(r_ref)
    _assert_field(pl.get_field(0, 1), u)


@pytest.mark.parametrize("rows", [2, 6, 64, 1000])
def test_relax_rows_per_warp_invariance(rows):
    sc = scene_c2(1)
    pl = _planner(sc)
    pl.set_obstacles(0, sc.robot, sc.goal, sc.tracks, warp_cfg(), warm=0)
    pl.relax(relax_cfg(max_sweeps=64, temporal_depth=4, rows_per_warp=rows), want_result=False)
    ref = oracle.plan_step(sc, max_sweeps=64, iters=0)
    _assert_field(pl.get_field(0, 1), ref["u"])


def test_relax_tolerance_stop_and_check_every():
    sc = scene_random("t", 200, 6, 5, 11)
    pl = _planner(sc)
    pl.set_obstacles(0, sc.robot, sc.goal, sc.tracks, warp_cfg(), warm=0)
    sw, res = pl.relax(relax_cfg(max_sweeps=5000, check_every=12, tol=3e-4, temporal_depth=4, sync_every=3))
    ref = oracle.plan_step(sc, max_sweeps=5000, check_every=12, tol=3e-4, iters=0)
    assert int(sw[0]) == ref["sweeps"] and int(sw[0]) % 12 == 0 and int(sw[0]) < 5000
    assert np.float32(res[0]) == np.float32(ref["residual"])
    _assert_field(pl.get_field(0, 1), ref["u"])


def test_zero_sweeps_is_identity():
    sc = scene_c1()
    pl = _planner(sc)
    pl.set_obstacles(0, sc.robot, sc.goal, sc.tracks, warp_cfg(), warm=0)
    u0 = pl.get_field(0, 0)
    sw, res = pl.relax(relax_cfg(max_sweeps=0))
    assert sw[0] == 0 and res[0] == 0.0 and np.array_equal(pl.get_field(0, 0).view(np.uint32), u0.view(np.uint32))


# ------------------------------------------------------------------ a1-a3 stamping
@pytest.mark.parametrize("seed", [0, 3])
def test_stamping_bit_exact(seed):
    sc = scene_random("st", 700, 20, 60, seed)
    pl = _planner(sc)
    st = pl.set_obstacles(0, sc.robot, sc.goal, sc.tracks, warp_cfg(), warm=0)
    ost, cls, t, j, pred = oracle.classify(sc)
    assert st == ost
    tg, jg, pg = pl.get_warp(0, sc.n_tracks)
    assert np.array_equal(tg, t) and np.array_equal(jg, j) and np.array_equal(pg, pred)
    raw = pl.get_field(0, 0)
    assert np.array_equal(_classes_from_raw(raw), cls)
    assert np.all(raw[cls == oracle.FREE] == np.float32(-0.5))


def test_goal_swallowed_warning_and_robot_exemption():
    sc = scene_c2(2)
    P = np.diag([0.0025, 0.0025, 0.01, 0.01]).reshape(16)
    gx, gy = sc.goal
    rx, ry = sc.robot[0], sc.robot[1]
    extra = np.array([np.concatenate([[(gx + 0.5) * 0.1, (gy + 0.5) * 0.1, 0, 0], P]),
                      np.concatenate([[rx, ry, 0, 0], P])])
    sc2 = sc.__class__(**{**sc.__dict__, "tracks": np.vstack([sc.tracks, extra])})
    pl = _planner(sc2)
    st = pl.set_obstacles(0, sc2.robot, sc2.goal, sc2.tracks, warp_cfg(), warm=0)
    ost, cls, *_ = oracle.classify(sc2)
    assert st == ost == T.W_GOAL_SWALLOWED
    assert np.array_equal(_classes_from_raw(pl.get_field(0, 0)), cls)


def test_validation_errors():
    sc = scene_c1()
    pl = _planner(sc)
    with pytest.raises(T.TwgError) as e:
        pl.set_obstacles(0, sc.robot, (64, 3), sc.tracks, warp_cfg())
    assert e.value.status == T.E_OUT_OF_BOUNDS
    with pytest.raises(T.TwgError) as e:
        pl.set_obstacles(0, sc.robot, (32, 32), sc.tracks, warp_cfg())  # inside the static disk
    assert e.value.status == T.E_OVERLAPPING_CLASSES
    with pytest.raises(T.TwgError) as e:
        pl.set_obstacles(0, (3.2, 3.2, 0.0, 0.4), sc.goal, sc.tracks, warp_cfg())
    assert e.value.status == T.E_INVALID_START


# ------------------------------------------------------------------ a7-a9 + warm plan loop
def test_plan_loop_warm_parity_c2():
    sc0 = scene_c2(0)
    pl = _planner(sc0)
    wc, bc = warp_cfg(), band_cfg(50, 4000, 8000)
    prev = None
    for tick in range(4):
        sc = advance_scene(sc0, tick * 5)
        rc = relax_cfg(max_sweeps=3000 if tick == 0 else 100, warm_start=1)
        st, res, cells, sm = pl.plan_step(0, [sc.robot], [sc.goal], sc.tracks, [sc.n_tracks], wc, rc, bc)
        ref = oracle.plan_step(sc, max_sweeps=rc.max_sweeps, iters=50, max_len=4000, prev=prev)
        prev = ref
        r = res[0]
        assert r.sweeps == ref["sweeps"] and np.float32(r.residual) == np.float32(ref["residual"])
        _assert_field(pl.get_field(0, 1), ref["u"])
        assert np.array_equal(_classes_from_raw(pl.get_field(0, 0)), ref["cls"])
        assert r.walk_status == ref["walk_status"]
        if r.walk_status == T.OK:
            assert np.array_equal(cells[0, : r.n_cells], ref["cells"])
            got = sm[0, : r.n_smooth]
            assert got.shape == ref["smooth"].shape and np.abs(got - ref["smooth"]).max() <= 1e-4
            assert np.allclose((r.next_x, r.next_y), ref["next"], atol=1e-4)


def test_no_path_enclosed_start():
    static, g, _ = random_small_map(5, 48)
    static[:] = 0
    static[0:6, 5] = 1
    static[5, 0:6] = 1
    from scenes.gen import Scene
    from scenes import default_warp_cfg
    sc = Scene("np", 48, 48, 0.1, (0.0, 0.0), static, (0.15, 0.15, 0.0, 0.4), (40, 40), np.zeros((0, 20)),
               default_warp_cfg(), 0)
    pl = _planner(sc)
    pl.set_obstacles(0, sc.robot, sc.goal, sc.tracks, warp_cfg(), warm=0)
    pl.relax(relax_cfg(max_sweeps=500))
    st, cells, smooth, ns, nxt = pl.extract_path(0, band_cfg(10, 2304, 4000))
    ref = oracle.plan_step(sc, max_sweeps=500, iters=10, max_len=2304)
    assert st == T.E_NO_PATH == ref["walk_status"] and len(cells) == 0 and ns == 0


def test_max_len_exceeded_is_no_path():
    sc = scene_c1()
    pl = _planner(sc)
    pl.set_obstacles(0, sc.robot, sc.goal, sc.tracks, warp_cfg(), warm=0)
    pl.relax(relax_cfg(max_sweeps=3000))
    st, cells, *_ = pl.extract_path(0, band_cfg(5, 50, 400))
    assert st == T.E_NO_PATH and len(cells) == 0


# ------------------------------------------------------------------ batch
def test_batch_equals_single_scenarios():
    scs = [scene_c2(s) for s in range(3)]
    B = len(scs)
    pl = Planner(512, 512, B, 0.1, (0.0, 0.0), device=0, stream=_stream())
    for b, sc in enumerate(scs):
        pl.set_static(sc.static, b)
    wc, bc = warp_cfg(), band_cfg(20, 3000, 6000)
    rc = relax_cfg(max_sweeps=200, warm_start=0)
    tracks = np.vstack([sc.tracks for sc in scs])
    st, res, cells, sm = pl.plan_step(-1, [sc.robot for sc in scs], [sc.goal for sc in scs], tracks,
                                      [sc.n_tracks for sc in scs], wc, rc, bc)
    for b, sc in enumerate(scs):
        ref = oracle.plan_step(sc, max_sweeps=200, iters=20, max_len=3000)
        _assert_field(pl.get_field(b, 1), ref["u"])
        assert res[b].walk_status == ref["walk_status"]
        if ref["walk_status"] == 0:
            assert np.array_equal(cells[b, : res[b].n_cells], ref["cells"])
            assert np.abs(sm[b, : res[b].n_smooth] - ref["smooth"]).max() <= 1e-4
    # one scenario of the batch alone: the others are untouched
    before = pl.get_field(1, 0).copy()
    pl.plan_step(0, [scs[0].robot], [scs[0].goal], scs[0].tracks, [scs[0].n_tracks], wc,
                 relax_cfg(max_sweeps=7, warm_start=1), bc)
    assert np.array_equal(pl.get_field(1, 0).view(np.uint32), before.view(np.uint32))


def test_device_tracks_equal_host_tracks():
    sc = scene_c2(4)
    a, b = _planner(sc), _planner(sc)
    a.set_obstacles(0, sc.robot, sc.goal, sc.tracks, warp_cfg(), warm=0)
    dt = torch.from_numpy(np.ascontiguousarray(sc.tracks)).cuda()
    b.set_obstacles(0, sc.robot, sc.goal, dt, warp_cfg(), warm=0)
    assert np.array_equal(a.get_field(0, 0).view(np.uint32), b.get_field(0, 0).view(np.uint32))


# ------------------------------------------------------------------ field import / export, P8 on device
def test_set_field_dirichlet_polynomial():
    N = 40
    yy, xx = np.mgrid[0:N, 0:N].astype(np.float64)
    f = (0.5 + 0.0003 * (xx ** 2 - yy ** 2)).astype(np.float32)  # in [0.04, 0.97]: fixed cells are >= 0
    ring = np.zeros((N, N), bool)
    ring[0, :] = ring[-1, :] = ring[:, 0] = ring[:, -1] = True
    raw = np.where(ring, f, -np.float32(0.5)).astype(np.float32)
    pl = Planner(N, N, 1, 0.1, (0, 0), device=0, stream=_stream())
    pl.set_field(raw)
    pl.relax(relax_cfg(max_sweeps=4000, temporal_depth=4))
    u = pl.get_field(0, 1)
    cls = ring.astype(np.uint8)
    uo = np.where(ring, f, np.float32(0.5)).astype(np.float32)
    oracle.relax_f32(cls, uo, 4000, 4000, 0.0)
    assert np.array_equal(u, uo)
    assert np.max(np.abs(u - f)) < 2e-5  # discrete-harmonic data are reproduced (pin P8, fp32)
    phi = pl.get_field(0, 2)
    assert np.array_equal(phi, (np.float32(1) - u))


# ------------------------------------------------------------------ full size (bench configuration)
@pytest.mark.slow
def test_c3_full_size_fixed_budget():
    from scenes import scene_c3
    sc = scene_c3(0)
    pl = _planner(sc)
    pl.set_obstacles(0, sc.robot, sc.goal, sc.tracks, warp_cfg(), warm=0)
    S = 40
    sw, res = pl.relax(relax_cfg(max_sweeps=S))  # auto T and tiling, as bench.py times it
    ref = oracle.plan_step(sc, max_sweeps=S, iters=0, max_len=20000)
    assert np.array_equal(_classes_from_raw(pl.get_field(0, 0)), ref["cls"])
    assert int(sw[0]) == S and np.float32(res[0]) == np.float32(ref["residual"])
    _assert_field(pl.get_field(0, 1), ref["u"])
    st, cells, *_ = pl.extract_path(0, band_cfg(0, 20000, 40000))
    assert st == ref["walk_status"]
    if st == T.OK:
        assert np.array_equal(cells, ref["cells"])


def test_single_scenario_relax_leaves_others_bitwise_untouched():
    """twg_plan_step(b) relaxes scenario b only; with an odd number of launches and an early stop
    the other scenarios' fields must not move (regression: stale per-scenario buffer indices)."""
    scs = [scene_c2(s) for s in range(3)]
    pl = Planner(512, 512, 3, 0.1, (0.0, 0.0), device=0, stream=_stream())
    for b, sc in enumerate(scs):
        pl.set_static(sc.static, b)
        pl.set_obstacles(b, sc.robot, sc.goal, sc.tracks, warp_cfg(), warm=0)
    pl.relax(relax_cfg(max_sweeps=7, temporal_depth=3))
    before = [pl.get_field(b, 0).copy() for b in range(3)]
    for sweeps, T_, tol in ((5, 2, 0.0), (9, 3, 0.0), (40, 4, 1e-2)):
        pl.plan_step(1, [scs[1].robot], [scs[1].goal], scs[1].tracks, [scs[1].n_tracks], warp_cfg(),
                     relax_cfg(max_sweeps=sweeps, check_every=4, tol=tol, temporal_depth=T_), band_cfg(5, 3000, 6000))
        for b in (0, 2):
            assert np.array_equal(pl.get_field(b, 0).view(np.uint32), before[b].view(np.uint32))


# ------------------------------------------------------------------ degenerate cases
def test_start_equals_goal_and_zero_band_iterations():
    from scenes.gen import Scene
    from scenes import default_warp_cfg
    N = 40
    static = np.zeros((N, N), np.uint8)
    sc = Scene("sg", N, N, 0.1, (0.0, 0.0), static, (2.05, 2.05, 0.0, 0.4), (20, 20), np.zeros((0, 20)),
               default_warp_cfg(), 0)
    pl = _planner(sc)
    pl.set_obstacles(0, sc.robot, sc.goal, sc.tracks, warp_cfg(), warm=0)
    pl.relax(relax_cfg(max_sweeps=50))
    st, cells, smooth, ns, nxt = pl.extract_path(0, band_cfg(50, 100, 200))
    assert st == T.OK and cells.tolist() == [[20, 20]] and ns == 1 and np.allclose(smooth, [[20.5, 20.5]])
    assert nxt == (20.5, 20.5)
    sc2 = Scene("sg2", N, N, 0.1, (0.0, 0.0), static, (0.55, 0.55, 0.0, 0.4), (30, 33), np.zeros((0, 20)),
                default_warp_cfg(), 0)
    pl2 = _planner(sc2)
    pl2.set_obstacles(0, sc2.robot, sc2.goal, sc2.tracks, warp_cfg(), warm=0)
    pl2.relax(relax_cfg(max_sweeps=4000))
    st, cells, smooth, ns, nxt = pl2.extract_path(0, band_cfg(0, 400, 800))
    ref = oracle.plan_step(sc2, max_sweeps=4000, iters=0, max_len=400)
    assert np.array_equal(cells, ref["cells"]) and np.array_equal(smooth, ref["smooth"])


def test_goal_less_field_relaxes_to_zero_and_walk_fails():
    """No goal reachable (the goal is walled in): free cells decay towards u = 0, the walk reports NoPath."""
    from scenes.gen import Scene
    from scenes import default_warp_cfg
    N = 48
    static = np.zeros((N, N), np.uint8)
    static[20:29, 20] = 1; static[20:29, 28] = 1; static[20, 20:29] = 1; static[28, 20:29] = 1
    sc = Scene("gl", N, N, 0.1, (0.0, 0.0), static, (0.55, 0.55, 0.0, 0.4), (24, 24), np.zeros((0, 20)),
               default_warp_cfg(), 0)
    pl = _planner(sc)
    pl.set_obstacles(0, sc.robot, sc.goal, sc.tracks, warp_cfg(), warm=0)
    sw, res = pl.relax(relax_cfg(max_sweeps=3000, temporal_depth=5))
    ref = oracle.plan_step(sc, max_sweeps=3000, iters=5, max_len=3000)
    _assert_field(pl.get_field(0, 1), ref["u"])
    st, cells, *_ = pl.extract_path(0, band_cfg(5, 3000, 6000))
    assert st == T.E_NO_PATH == ref["walk_status"]


# ------------------------------------------------------------------ full sizes of BASELINE configs 4 and 5
@pytest.mark.slow
def test_c4_full_size_sampled_rows():
    """16384^2 (BASELINE configs[3]) on one GPU: 8 sweeps in the default launch configuration; the
    oracle relaxes row bands independently (a band of R rows plus 2 * 8 rows of context is exact
    for 8 sweeps) and the sampled rows must match bit for bit."""
    from scenes import scene_c4
    sc = scene_c4(0)
    pl = _planner(sc)
    pl.set_obstacles(0, sc.robot, sc.goal, sc.tracks, warp_cfg(), warm=0)
    S = 8
    pl.relax(relax_cfg(max_sweeps=S))
    raw = pl.get_field(0, 0)
    st, cls, *_ = oracle.classify(sc)
    assert np.array_equal(_classes_from_raw(raw), cls)
    for r0 in (0, 5000, 16384 - 40):
        lo, hi = max(r0 - 2 * S, 0), min(r0 + 40 + 2 * S, sc.H)
        sub_cls = np.ascontiguousarray(cls[lo:hi])
        # rows outside the band act as walls only where the band ends inside the grid: their
        # influence reaches at most 2S rows in, which the context absorbs
        u = oracle.init_u32(sub_cls)
        oracle.relax_f32_ex(sub_cls, u, S, S, 0.0, row_parity=lo)
        assert np.array_equal(np.abs(raw[r0:r0 + 40]), u[r0 - lo:r0 - lo + 40])


@pytest.mark.slow
def test_c5_full_batch_sampled_scenarios():
    """1024 x 512^2 (BASELINE configs[4]) in one batched context: a cold plan step with S = 100
    for all scenarios; 6 sampled scenarios are replayed by the oracle."""
    from scenes import scene_c5
    scs = scene_c5(1024)
    pl = Planner(512, 512, 1024, 0.1, (0.0, 0.0), device=0, stream=_stream())
    for b, sc in enumerate(scs):
        pl.set_static(sc.static, b)
    tracks = np.vstack([sc.tracks for sc in scs])
    bc = band_cfg(50, 2048, 4096)
    st, res, cells, sm = pl.plan_step(-1, [sc.robot for sc in scs], [sc.goal for sc in scs], tracks,
                                      [sc.n_tracks for sc in scs], warp_cfg(), relax_cfg(max_sweeps=100, warm_start=0),
                                      bc)
    for b in (0, 1, 313, 512, 777, 1023):
        ref = oracle.plan_step(scs[b], max_sweeps=100, iters=50, max_len=2048)
        _assert_field(pl.get_field(b, 1), ref["u"])
        assert res[b].walk_status == ref["walk_status"] and res[b].sweeps == 100
        if ref["walk_status"] == 0:
            assert np.array_equal(cells[b, : res[b].n_cells], ref["cells"])
            assert np.abs(sm[b, : res[b].n_smooth] - ref["smooth"]).max() <= 1e-4


@pytest.mark.parametrize("T_", [3, 6])
def test_batch_tolerance_stop_scenarios_finish_at_different_sweeps(T_):
    # red-black batch with a tolerance: each scenario stops at its own check sweep; the fields of
    # those that stopped early are moved back into place (k_fixup) -- all equal to the oracle
    scs = [scene_random(f"bt{k}", 96, 2 + k, 2 * k, 60 + k) for k in range(4)]
    pl = Planner(96, 96, 4, 0.1, (0.0, 0.0), device=0, stream=_stream())
    for k, sc in enumerate(scs):
        pl.set_static(sc.static, b=k)
        pl.set_obstacles(k, sc.robot, sc.goal, sc.tracks, warp_cfg(), warm=0)
    sw, res = pl.relax(relax_cfg(max_sweeps=20000, check_every=7, tol=1e-5, temporal_depth=T_, sync_every=2))
    got = set()
    for k, sc in enumerate(scs):
        ref = oracle.plan_step(sc, max_sweeps=20000, check_every=7, tol=1e-5, iters=0)
        assert int(sw[k]) == ref["sweeps"] and np.float32(res[k]) == np.float32(ref["residual"])
        _assert_field(pl.get_field(k, 1), ref["u"])
        got.add(int(sw[k]))
    assert len(got) > 1  # they really stopped at different sweeps


@pytest.mark.slow
def test_plan_loop_warm_parity_c2_long():
    # SURVEY C2-style long warm plan loop (tick 0 cold to the exact fp32 fixed point, then S = 100
    # per tick): every tick's field, cells and smoothed path bit-identical to the oracle replaying
    # the same poses (192^2 so that the oracle's cold solve stays a few seconds)
    sc0 = scene_random("long", 192, 4, 8, 3)
    pl = _planner(sc0)
    wc, bc = warp_cfg(), band_cfg(50, 4000, 8000)
    prev = None
    walks = 0
    for tick in range(40):
        sc = advance_scene(sc0, tick)
        if tick == 0:
            rc = relax_cfg(max_sweeps=400_000, check_every=500, tol=1e-38, warm_start=1)
        else:
            rc = relax_cfg(max_sweeps=100, warm_start=1)
        st, res, cells, sm = pl.plan_step(0, [sc.robot], [sc.goal], sc.tracks, [sc.n_tracks], wc, rc, bc)
        ref = oracle.plan_step(sc, max_sweeps=rc.max_sweeps, check_every=rc.check_every or None, tol=rc.tol,
                               iters=50, max_len=4000, prev=prev)
        prev = ref
        r = res[0]
        assert r.sweeps == ref["sweeps"], tick
        assert np.array_equal(pl.get_field(0, 1), ref["u"]), tick
        assert r.walk_status == ref["walk_status"], tick
        if r.walk_status == T.OK:
            walks += 1
            assert np.array_equal(cells[0, : r.n_cells], ref["cells"]), tick
            assert np.array_equal(sm[0, : r.n_smooth], ref["smooth"]), tick
    assert walks >= 30
