"""GPU <-> oracle parity of row f1 (tracker tick: Kalman update Eqs. 11-13, association, spawn/prune)
through the C ABI (twg_track_update, twg_get_tracks, resident tracks in twg_set_obstacles /
twg_plan_step).  Bar: track states (fp64), missed counters, counts and statuses bit-exact."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import oracle  # noqa: E402
from paper_1903_07441_b200 import Planner, band_cfg, relax_cfg, warp_cfg, tracker_cfg  # noqa: E402
from paper_1903_07441_b200 import twg as T  # noqa: E402
from scenes import scene_c2, scene_c3, scene_random, detections, advance_scene  # noqa: E402
from dataclasses import replace  # noqa: E402


def _stream():
    return torch.cuda.current_stream().cuda_stream


def _planner(sc, batch=1):
    pl = Planner(sc.W, sc.H, batch, sc.cell_size, sc.origin, device=0, stream=_stream())
    pl.set_static(sc.static)
    return pl


def _run_ticks(sc, ticks, tc_kw, p_miss=0.05, n_clutter=0, wkw=None):
    pl = _planner(sc)
    wc = warp_cfg(**(wkw or {}))
    pl.set_obstacles(0, sc.robot, sc.goal, sc.tracks, wc, warm=0)  # seeds the resident table
    trk, mis = sc.tracks.copy(), np.zeros(sc.n_tracks, np.int32)
    Q = np.array(wc.Q[:], np.float64)
    for tick in range(1, ticks + 1):
        z = detections(sc, tick, p_miss=p_miss, n_clutter=n_clutter)
        st, nt = pl.track_update(0, z, [len(z)], wc, tracker_cfg(**tc_kw))
        ost, trk, mis = oracle.track_step(trk, mis, z, dt=wc.dt, Q=Q, **tc_kw)
        assert st == ost and int(nt[0]) == len(trk)
        g, gm = pl.get_tracks(0)
        assert np.array_equal(g, trk) and np.array_equal(gm, mis)
    return pl, trk, mis


def test_tracker_ticks_c2():
    _run_ticks(scene_c2(1), 6, {})


def test_tracker_misses_clutter_prune():
    pl, trk, mis = _run_ticks(scene_c2(2), 14, dict(prune_after=2, gate=0.3), p_miss=0.35, n_clutter=4)
    assert mis.max() <= 2


def test_tracker_capacity_truncation():
    sc = scene_c2(3)
    pl, trk, mis = _run_ticks(sc, 3, dict(max_tracks=12), n_clutter=6)
    assert len(trk) == 12


def test_tracker_dense_cluster_pair_overflow():
    # 300 tracks and 300 detections inside a 0.3 m square: 90 000 gated pairs > the initial list,
    # exercising the grow-and-retry path and the global-memory sort
    rng = np.random.default_rng(9)
    sc = scene_c2(4)
    tr = np.zeros((300, 20))
    tr[:, :2] = 10.0 + rng.uniform(0, 0.3, (300, 2))
    tr[:, 2:4] = rng.normal(0, 0.1, (300, 2))
    tr[:, 4:] = (np.eye(4) * 0.01).reshape(16)
    sc = replace(sc, tracks=tr)
    pl = _planner(sc)
    wc = warp_cfg()
    pl.set_obstacles(0, sc.robot, sc.goal, tr, wc, warm=0)
    z = 10.0 + rng.uniform(0, 0.3, (300, 2))
    st, nt = pl.track_update(0, z, [300], wc, tracker_cfg(gate=1.0))
    ost, trk, mis = oracle.track_step(tr, np.zeros(300, np.int32), z, Q=np.array(wc.Q[:]), gate=1.0)
    g, gm = pl.get_tracks(0)
    assert st == ost and np.array_equal(g, trk) and np.array_equal(gm, mis)


def test_tracker_batch_mixed_counts():
    scs = [scene_random(f"tb{k}", 200, 4, n, 30 + k) for k, n in enumerate((0, 5, 40, 17))]
    pl = Planner(200, 200, 4, 0.1, (0.0, 0.0), device=0, stream=_stream())
    wc = warp_cfg()
    ref = []
    for k, sc in enumerate(scs):
        pl.set_static(sc.static, b=k)
        pl.set_obstacles(k, sc.robot, sc.goal, sc.tracks, wc, warm=0)
        ref.append((sc.tracks.copy(), np.zeros(sc.n_tracks, np.int32)))
    Q = np.array(wc.Q[:])
    for tick in range(1, 4):
        zs = [detections(sc, tick, p_miss=0.2, n_clutter=k) if sc.n_tracks else np.zeros((k, 2)) + 3.0
              for k, sc in enumerate(scs)]
        st, nt = pl.track_update(-1, np.concatenate(zs), [len(z) for z in zs], wc, tracker_cfg())
        for k in range(4):
            _, trk, mis = oracle.track_step(ref[k][0], ref[k][1], zs[k], Q=Q)
            ref[k] = (trk, mis)
            g, gm = pl.get_tracks(k)
            assert int(nt[k]) == len(trk) and np.array_equal(g, trk) and np.array_equal(gm, mis)


def test_tracker_device_detections_and_single_scenario_of_batch():
    scs = [scene_random(f"td{k}", 128, 3, 8, 50 + k) for k in range(2)]
    pl = Planner(128, 128, 2, 0.1, (0.0, 0.0), device=0, stream=_stream())
    wc = warp_cfg()
    for k, sc in enumerate(scs):
        pl.set_static(sc.static, b=k)
        pl.set_obstacles(k, sc.robot, sc.goal, sc.tracks, wc, warm=0)
    z = detections(scs[1], 1)
    zd = torch.as_tensor(z, device="cuda")
    st, nt = pl.track_update(1, zd, [len(z)], wc, tracker_cfg())
    _, trk, mis = oracle.track_step(scs[1].tracks, np.zeros(8, np.int32), z, Q=np.array(wc.Q[:]))
    g, gm = pl.get_tracks(1)
    assert np.array_equal(g, trk) and np.array_equal(gm, mis)
    g0, gm0 = pl.get_tracks(0)                      # scenario 0 untouched
    assert np.array_equal(g0, scs[0].tracks) and not gm0.any()


def test_tracker_singular_innovation():
    sc = scene_c2(5)
    tr = sc.tracks[:3].copy()
    tr[:, 4:] = np.diag([0.0, 0.0, 0.0, 0.0]).reshape(16)
    pl = _planner(sc)
    wc = warp_cfg(Q=np.zeros(16))
    pl.set_obstacles(0, sc.robot, sc.goal, tr, wc, warm=0)
    z = tr[:, :2] + 0.01
    st, nt = pl.track_update(0, z, [3], wc, tracker_cfg(sigma_z=0.0))
    ost, trk, mis = oracle.track_step(tr, np.zeros(3, np.int32), z, Q=np.zeros(16), sigma_z=0.0)
    assert st == ost == T.W_SINGULAR_INNOVATION
    g, gm = pl.get_tracks(0)
    assert np.array_equal(g, trk) and np.array_equal(gm, mis) and gm.tolist() == [1, 1, 1]


def test_tracker_empty_and_validation():
    sc = scene_c2(6)
    pl = _planner(sc)
    wc = warp_cfg()
    pl.set_obstacles(0, sc.robot, sc.goal, np.zeros((0, 20)), wc, warm=0)
    st, nt = pl.track_update(0, np.zeros((0, 2)), [0], wc, tracker_cfg())
    assert st == T.OK and nt.tolist() == [0]
    st, nt = pl.track_update(0, [[1.0, 1.0]], [1], wc, tracker_cfg())
    g, gm = pl.get_tracks(0)
    assert nt.tolist() == [1] and g[0, :4].tolist() == [1.0, 1.0, 0.0, 0.0]
    for bad in (dict(sigma_z=-1.0), dict(gate=-0.1), dict(prune_after=-1), dict(max_tracks=-2)):
        with pytest.raises(T.TwgError):
            pl.track_update(0, np.zeros((0, 2)), [0], wc, tracker_cfg(**bad))


def test_resident_tracks_closed_loop_plan():
    # Map Update on the device end to end: tracker tick -> stamping from the resident table -> plan
    sc = scene_c2(7)
    pl = _planner(sc)
    wc = warp_cfg()
    rc = relax_cfg(max_sweeps=80, warm_start=1)
    bc = band_cfg(20, 3000, 6000)
    pl.set_obstacles(0, sc.robot, sc.goal, sc.tracks, wc, warm=0)
    trk, mis = sc.tracks.copy(), np.zeros(sc.n_tracks, np.int32)
    prev = None
    for tick in range(1, 4):
        s = advance_scene(sc, tick)
        z = detections(sc, tick)
        pl.track_update(0, z, [len(z)], wc, tracker_cfg())
        _, trk, mis = oracle.track_step(trk, mis, z, Q=np.array(wc.Q[:]))
        rct = rc if tick > 1 else relax_cfg(max_sweeps=80, warm_start=0)
        st, res, cells, sm = pl.plan_step(0, [s.robot], [s.goal], None, None, wc, rct, bc)
        ref = oracle.plan_step(replace(s, tracks=trk), max_sweeps=80, iters=20, max_len=3000, prev=prev)
        assert st == ref["status"] or (ref["walk_status"] != 0)
        u = pl.get_field(0, 1)
        assert np.array_equal(u, ref["u"])
        if ref["walk_status"] == 0:
            assert np.array_equal(cells[0, :res[0].n_cells], ref["cells"])
        prev = ref
    # set_obstacles with the resident table too
    t, j, pred = pl.get_warp(0, len(trk))
    st2 = pl.set_obstacles(0, s.robot, s.goal, None, wc, warm=0)
    ost, cls, ot, oj, opred = oracle.classify(replace(s, tracks=trk))
    assert st2 == ost
    tg, jg, pg = pl.get_warp(0, len(trk))
    assert np.array_equal(tg, ot) and np.array_equal(jg, oj) and np.array_equal(pg, opred)


def test_tracker_c3_full_size():
    _run_ticks(scene_c3(0), 3, {}, n_clutter=10)


def test_tracker_1000_tracks():
    sc = scene_random("t1k", 2048, 40, 1000, 11)
    _run_ticks(sc, 2, {})
