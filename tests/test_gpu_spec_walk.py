"""Speculative segment walkers (row a7): the walk
assembled from the walker at the robot cell and the walkers at markers placed on the previous path
must equal the single descent walk of the oracle (orc_walk, Alg. 1, C9) -- whatever the
markers are: robot on a marker, markers on cells the new walk never visits, a moved goal, a walk
longer than max_len by one cell, cycles in unconverged fields, several scenarios per context.

Expected values come from oracle.plan_step replaying the same scenes (its own field, warm-started
from its own previous tick); the GPU field is compared too.  At the C3 bench size, where the
oracle cannot converge the field, the walk is checked by properties that hold at any size."""
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

COLD = dict(max_sweeps=400_000, check_every=1000, tol=1e-38)  # to the exact fp32 fixed point


def _planner(sc, B=1):
    return Planner(sc.W, sc.H, B, sc.cell_size, sc.origin, device=0, stream=torch.cuda.current_stream().cuda_stream)


class Loop:
    """GPU plan steps and oracle plan steps of the same scenes, tick after tick."""

    def __init__(self, sc0):
        self.pl = _planner(sc0)
        self.pl.set_static(sc0.static)
        self.prev = None

    def step(self, sc, max_sweeps, max_len, check_every=0, tol=0.0, warm=1):
        rc = relax_cfg(max_sweeps=max_sweeps, check_every=check_every, tol=tol, warm_start=warm)
        st, res, cells, _ = self.pl.plan_step(0, [sc.robot], [sc.goal], sc.tracks, [sc.n_tracks], warp_cfg(), rc,
                                              band_cfg(0, max_len, 2 * max_len))
        ref = oracle.plan_step(sc, max_sweeps=max_sweeps, check_every=check_every or None, tol=tol, iters=0,
                               max_len=max_len, prev=self.prev if warm else None)
        assert res[0].sweeps == ref["sweeps"]
        assert np.array_equal(self.pl.get_field(0, 1), ref["u"])
        assert res[0].walk_status == ref["walk_status"]
        if ref["walk_status"] == T.OK:
            assert np.array_equal(cells[0, : res[0].n_cells], ref["cells"])
        self.prev = ref
        return ref


def _at_cell(sc, c):
    x, y = int(c[0]), int(c[1])
    return dataclasses.replace(sc, robot=((x + 0.5) * sc.cell_size, (y + 0.5) * sc.cell_size,
                                          sc.robot[2], sc.robot[3]))


@pytest.fixture(scope="module")
def scene():
    return scene_random("spec", 160, 6, 8, 7)


def test_spec_walk_plan_loop(scene):
    lp = Loop(scene)
    ml = 8 * scene.W
    ref = lp.step(scene, warm=0, max_len=ml, **COLD)
    assert ref["walk_status"] == T.OK and len(ref["cells"]) > 150
    ok = 0
    for tick in range(1, 9):
        ref = lp.step(advance_scene(scene, tick * 2), 100, ml)
        ok += ref["walk_status"] == T.OK
    assert ok >= 6


def test_spec_walk_robot_on_markers_max_len_and_moved_goal(scene):
    lp = Loop(scene)
    ml = 8 * scene.W
    ref0 = lp.step(scene, warm=0, max_len=ml, **COLD)
    cells = ref0["cells"]
    n = len(cells)
    assert ref0["walk_status"] == T.OK and n > 100
    S = max(32, (n + 64) // 65)  # k_spec_mark's sample spacing
    for idx in (S, 2 * S, 3 * S + 1, n - 2, 0):
        ref = lp.step(_at_cell(scene, cells[idx]), 20, ml)  # the robot stands on a (former) marker
        assert ref["walk_status"] == T.OK
        lp.step(scene, 20, ml)  # back to the full path: the next markers come from it
    # max_len exactly the walk, then one cell short of it (no path), markers from the full walk
    ref = lp.step(scene, 0, ml)
    n = len(ref["cells"])
    assert lp.step(scene, 0, n)["walk_status"] == T.OK
    assert lp.step(scene, 0, n - 1)["walk_status"] == T.E_NO_PATH
    lp.step(scene, 0, ml)
    # a moved goal: the markers lie on the walk to the old goal
    free = np.argwhere(scene.static == 0)
    gy, gx = free[len(free) // 3]
    moved = dataclasses.replace(scene, goal=(int(gx), int(gy)))
    lp.step(moved, 3000, ml)
    lp.step(moved, 100, ml)


def test_spec_walk_unconverged_fields_with_cycles(scene):
    # few sweeps after cold restarts leave 0.5 plateaus: walks cycle (no path) or wander; the
    # speculative walkers must report exactly what the single walk does, tick after tick
    lp = Loop(scene)
    ml = 4 * scene.W
    for tick, (sweeps, warm) in enumerate([(0, 0), (3, 1), (10, 1), (50, 1), (0, 0)]):
        sc = advance_scene(scene, tick + 1)
        lp.step(sc, sweeps, ml, warm=warm)
        ref = lp.step(sc, max_len=ml, **COLD)  # a converged path: markers for the next tick
        assert ref["walk_status"] == T.OK


def test_spec_walk_batch_and_single_scenario_steps():
    # a 3-scenario context: markers are per scenario; plan steps over all scenarios and over one
    # scenario (twg_plan_step with b) alternate
    scs = [scene_random("specb%d" % k, 128, 4, 5, 20 + k) for k in range(3)]
    pl = _planner(scs[0], B=3)
    for b, sc in enumerate(scs):
        pl.set_static(sc.static, b=b)
    wc, ml = warp_cfg(), 2048
    bc = band_cfg(0, ml, 2 * ml)
    prev = [None] * 3
    for tick in range(6):
        cur = [advance_scene(sc, tick) for sc in scs]
        kw = dict(COLD) if tick == 0 else dict(max_sweeps=150)
        rc = relax_cfg(warm_start=1, **kw)
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
            ref = oracle.plan_step(cur[b], max_sweeps=kw["max_sweeps"], check_every=kw.get("check_every"),
                                   tol=kw.get("tol", 0.0), iters=0, max_len=ml, prev=prev[b])
            prev[b] = ref
            assert np.array_equal(pl.get_field(b, 1), ref["u"]), (tick, b)
            assert res[i].walk_status == ref["walk_status"], (tick, b)
            if ref["walk_status"] == T.OK:
                assert np.array_equal(cells[i, : res[i].n_cells], ref["cells"]), (tick, b)


def _descent_properties(raw, cells, start, goal):
    """Eq. 3 / C8 walk properties on the field the walk ran on: starts at the robot cell, ends at
    the goal, every step goes to the first 4-neighbour with the largest |u| (+x, -x, +y, -y)."""
    H, W = raw.shape
    u = np.abs(raw)
    assert tuple(cells[0]) == tuple(start) and tuple(cells[-1]) == tuple(goal)
    for (x, y), (nx, ny) in zip(cells[:-1], cells[1:]):
        best, arg = None, None
        for dx, dy in ((1, 0), (-1, 0), (0, 1), (0, -1)):
            qx, qy = x + dx, y + dy
            if 0 <= qx < W and 0 <= qy < H and (best is None or u[qy, qx] > best):
                best, arg = u[qy, qx], (qx, qy)
        assert (nx, ny) == arg


@pytest.mark.slow
def test_spec_walk_c3_bench_configuration():
    # the bench's C3 loop: converged 4096^2 field, then warm plan steps with moving tracks; each
    # step's speculative walk is the Eq. 3 descent from the robot cell to the goal on its field
    from scenes import scene_c3
    sc0 = scene_c3(0)
    pl = _planner(sc0)
    pl.set_static(sc0.static)
    ml = 4 * (sc0.W + sc0.H)
    bc = band_cfg(0, ml, 2 * ml)
    pl.plan_step(0, [sc0.robot], [sc0.goal], sc0.tracks, [sc0.n_tracks], warp_cfg(),
                 relax_cfg(max_sweeps=4_000_000, check_every=20000, tol=1e-38, warm_start=0, sync_every=4), bc,
                 want_paths=False)
    for k in range(1, 4):
        sc = advance_scene(sc0, k)
        st, res, cells, _ = pl.plan_step(0, [sc.robot], [sc.goal], sc.tracks, [sc.n_tracks], warp_cfg(),
                                         relax_cfg(max_sweeps=100, warm_start=1), bc)
        assert res[0].walk_status == T.OK and res[0].n_cells > 5000
        _descent_properties(pl.get_field(0, 0), cells[0, : res[0].n_cells], oracle.robot_cell(sc), tuple(sc.goal))
