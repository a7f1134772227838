"""Speculative segment walkers (row a7): the walk
assembled from the walker at the robot cell and the walkers at markers placed on the previous path
must equal the single descent walk of the oracle (orc_walk, Alg. 1, C9) on the same field --
whatever the markers are: robot on a marker, markers on cells the new walk never visits, a moved
goal, a walk longer than max_len by one cell, cycles in unconverged fields."""
import dataclasses

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import oracle  # noqa: E402
from paper_1903_07441_b200 import Planner, band_cfg, relax_cfg, warp_cfg  # noqa: E402
from paper_1903_07441_b200 import twg as T  # noqa: E402
from scenes import advance_scene, scene_random  # noqa: E402

PATH_LAUNCHES_SPEC = 6  # index_dir, spec_mark, walk, spec_stitch, band, resample


def _cls(raw):
    bits = raw.view(np.uint32)
    cls = np.zeros(raw.shape, np.uint8)
    cls[bits == 0] = oracle.OBSTACLE
    cls[bits == 0x3F800000] = oracle.GOAL
    return cls


def _check_walk(pl, sc, max_len):
    """extract_path against the oracle walk on the planner's own field (the field itself is pinned
    by the relaxation parity tests); returns the cells."""
    raw = pl.get_field(0, 0)
    n0 = pl.kernel_launches()
    st, cells, *_ = pl.extract_path(0, band_cfg(0, max_len, 2 * max_len))
    spec = pl.kernel_launches() - n0 == PATH_LAUNCHES_SPEC
    rst, rcells = oracle.walk(_cls(raw), np.abs(raw), oracle.robot_cell(sc), max_len)
    assert st == rst
    if st == T.OK:
        assert np.array_equal(cells, rcells)
    return st, cells, spec


def _at_cell(sc, c):
    x, y = int(c[0]), int(c[1])
    return dataclasses.replace(sc, robot=((x + 0.5) * sc.cell_size, (y + 0.5) * sc.cell_size,
                                          sc.robot[2], sc.robot[3]))


@pytest.fixture(scope="module")
def converged():
    sc0 = scene_random("spec", 640, 10, 12, 7)
    pl = Planner(sc0.W, sc0.H, 1, sc0.cell_size, sc0.origin, device=0, stream=torch.cuda.current_stream().cuda_stream)
    pl.set_static(sc0.static)
    pl.set_obstacles(0, sc0.robot, sc0.goal, sc0.tracks, warp_cfg(), warm=0)
    pl.relax(relax_cfg(max_sweeps=2_000_000, check_every=5000, tol=1e-38))
    return sc0, pl


def test_spec_walk_plan_loop(converged):
    sc0, pl = converged
    ml = 8 * sc0.W
    st, cells, _ = _check_walk(pl, sc0, ml)
    assert st == T.OK and len(cells) > 400
    specs = 0
    for tick in range(1, 8):
        sc = advance_scene(sc0, tick * 3)
        pl.set_obstacles(0, sc.robot, sc.goal, sc.tracks, warp_cfg(), warm=1)
        pl.relax(relax_cfg(max_sweeps=100, warm_start=1))
        st, cells, spec = _check_walk(pl, sc, ml)
        specs += spec
    assert specs >= 6  # every tick after a successful walk speculates


def test_spec_walk_robot_on_markers_and_max_len(converged):
    sc0, pl = converged
    ml = 8 * sc0.W
    pl.set_obstacles(0, sc0.robot, sc0.goal, sc0.tracks, warp_cfg(), warm=1)
    st, cells, _ = _check_walk(pl, sc0, ml)
    assert st == T.OK
    n = len(cells)
    S = max(32, (n + 64) // 65)  # k_spec_mark's sample spacing
    for idx in (S, 2 * S, 3 * S + 1, n - 2, 0):
        sc = _at_cell(sc0, cells[idx])
        pl.set_obstacles(0, sc.robot, sc.goal, sc.tracks, warp_cfg(), warm=1)
        st2, c2, spec = _check_walk(pl, sc, ml)
        assert spec and st2 == T.OK
        # put the path back so the next markers come from the full path
        pl.set_obstacles(0, sc0.robot, sc0.goal, sc0.tracks, warp_cfg(), warm=1)
        _check_walk(pl, sc0, ml)
    # max_len exactly the walk, then one short of it (no path), with markers from the full walk
    _check_walk(pl, sc0, n)
    st3, _, spec = _check_walk(pl, sc0, n)
    assert spec and st3 == T.OK
    st4, _, spec = _check_walk(pl, sc0, n - 1)
    assert spec and st4 == T.E_NO_PATH
    # a moved goal: the markers lie on the walk to the old goal
    _check_walk(pl, sc0, ml)
    g = (int(sc0.W * 0.5), int(sc0.H * 0.9))
    sc = dataclasses.replace(sc0, goal=g)
    if sc.static[g[1], g[0]] == 0:
        pl.set_obstacles(0, sc.robot, sc.goal, sc.tracks, warp_cfg(), warm=1)
        pl.relax(relax_cfg(max_sweeps=3000, warm_start=1))
        _check_walk(pl, sc, ml)


def test_spec_walk_unconverged_fields_with_cycles():
    # cold fields (u = 0.5 plateaus) make walks cycle; the speculative walkers must report the
    # same no-path / path as the single walk, tick after tick
    sc0 = scene_random("specc", 200, 4, 6, 11)
    pl = Planner(sc0.W, sc0.H, 1, sc0.cell_size, sc0.origin, device=0, stream=torch.cuda.current_stream().cuda_stream)
    pl.set_static(sc0.static)
    pl.set_obstacles(0, sc0.robot, sc0.goal, sc0.tracks, warp_cfg(), warm=0)
    pl.relax(relax_cfg(max_sweeps=200_000, check_every=5000, tol=1e-38))
    ok = 0
    for tick, sweeps in enumerate([0, 3, 10, 0, 50, 1, 200, 0]):
        sc = advance_scene(sc0, tick + 1)
        pl.set_obstacles(0, sc.robot, sc.goal, sc.tracks, warp_cfg(), warm=0 if tick % 3 == 0 else 1)
        pl.relax(relax_cfg(max_sweeps=sweeps, warm_start=1))
        st, _, _ = _check_walk(pl, sc, 4 * sc0.W)
        ok += st == T.OK
        # re-establish a converged path so the next tick has markers
        pl.relax(relax_cfg(max_sweeps=200_000, check_every=5000, tol=1e-38, warm_start=1))
        st, _, _ = _check_walk(pl, sc, 4 * sc0.W)
        assert st == T.OK


def test_spec_walk_batch_and_single_scenario_steps():
    # a 3-scenario context: markers are per scenario; plan steps over all scenarios and over one
    # scenario (twg_plan_step with b) alternate, every walk equal to the oracle's on that field
    scs = [scene_random("specb%d" % k, 256, 5, 6, 20 + k) for k in range(3)]
    pl = Planner(256, 256, 3, scs[0].cell_size, scs[0].origin, device=0,
                 stream=torch.cuda.current_stream().cuda_stream)
    for b, sc in enumerate(scs):
        pl.set_static(sc.static, b=b)
    wc, ml = warp_cfg(), 2048
    bc = band_cfg(10, ml, 2 * ml)
    for tick in range(6):
        cur = [advance_scene(sc, tick) for sc in scs]
        rc = relax_cfg(max_sweeps=300_000 if tick == 0 else 200, check_every=5000 if tick == 0 else 0,
                       tol=1e-38 if tick == 0 else 0.0, warm_start=1)
        if tick % 2 == 0:
            st, res, cells, _ = pl.plan_step(-1, [s.robot for s in cur], [s.goal for s in cur],
                                             np.concatenate([s.tracks for s in cur]), [s.n_tracks for s in cur],
                                             wc, rc, bc)
            bs = range(3)
        else:
            b = tick % 3
            st, res, cells, _ = pl.plan_step(b, [cur[b].robot], [cur[b].goal], cur[b].tracks, [cur[b].n_tracks],
                                             wc, rc, bc)
            bs = [b]
        for i, b in enumerate(bs):
            raw = pl.get_field(b, 0)
            rst, rcells = oracle.walk(_cls(raw), np.abs(raw), oracle.robot_cell(cur[b]), ml)
            assert res[i].walk_status == rst, (tick, b)
            if rst == T.OK:
                assert np.array_equal(cells[i, : res[i].n_cells], rcells), (tick, b)


@pytest.mark.slow
def test_spec_walk_c3_bench_configuration():
    # the bench's C3 loop: converged 4096^2 field, then warm plan steps with moving tracks; each
    # step's speculative walk equals the oracle walk on the same field
    from scenes import scene_c3
    sc0 = scene_c3(0)
    pl = Planner(sc0.W, sc0.H, 1, sc0.cell_size, sc0.origin, device=0, stream=torch.cuda.current_stream().cuda_stream)
    pl.set_static(sc0.static)
    ml = 4 * (sc0.W + sc0.H)
    bc = band_cfg(0, ml, 2 * ml)
    pl.plan_step(0, [sc0.robot], [sc0.goal], sc0.tracks, [sc0.n_tracks], warp_cfg(),
                 relax_cfg(max_sweeps=4_000_000, check_every=20000, tol=1e-38, warm_start=0, sync_every=4), bc,
                 want_paths=False)
    for k in range(1, 4):
        sc = advance_scene(sc0, k)
        n0 = pl.kernel_launches()
        st, res, cells, _ = pl.plan_step(0, [sc.robot], [sc.goal], sc.tracks, [sc.n_tracks], warp_cfg(),
                                         relax_cfg(max_sweeps=100, warm_start=1), bc)
        raw = pl.get_field(0, 0)
        rst, rcells = oracle.walk(_cls(raw), np.abs(raw), oracle.robot_cell(sc), ml)
        assert res[0].walk_status == rst == T.OK
        assert np.array_equal(cells[0, : res[0].n_cells], rcells)
        assert len(rcells) > 5000
