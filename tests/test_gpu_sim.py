"""GPU <-> oracle parity of row f2 (closed-loop simulator) through the C ABI: every tick of
twg_sim_tick (tracker tick, Map Update from resident tracks, relaxation, path, robot and obstacle
motion, status, detections) against oracle.sim_run, bit-exact robot states, statuses, tracks and
turning-angle histograms."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import oracle  # noqa: E402
from paper_1903_07441_b200 import Planner, band_cfg, relax_cfg, warp_cfg, tracker_cfg, sim_cfg  # noqa: E402
from paper_1903_07441_b200 import sim as S  # noqa: E402
from scenes import scene_sim, SimCfg  # noqa: E402


def _stream():
    return torch.cuda.current_stream().cuda_stream


def _cfgs(max_ticks, init_tol=1e-5, seed=5):
    return (sim_cfg(seed=seed, max_ticks=max_ticks, init_tol=init_tol),
            SimCfg(seed=seed, max_ticks=max_ticks, init_tol=init_tol))


@pytest.mark.parametrize("n_obs", [(1, 4, 8), (16, 0, 2)])
def test_sim_ticks_bit_exact(n_obs):
    T = 24
    scs = [scene_sim(10 + k, n) for k, n in enumerate(n_obs)]
    gcfg, ocfg = _cfgs(T)
    pl = Planner(256, 256, len(scs), 0.1, (0.0, 0.0), device=0, stream=_stream())
    for b, sc in enumerate(scs):
        pl.set_static(sc.static, b=b)
        pl.sim_reset(b, sc.robot, sc.goal, sc.truth, gcfg)
    rc, bc = relax_cfg(max_sweeps=100, warm_start=1), band_cfg(20, 4096, 8192)
    gpu = []
    for t in range(T):
        _, trials, running = pl.sim_tick(gcfg, warp_cfg(), rc, bc, tracker_cfg())
        gpu.append([(np.array([tr.x, tr.y, tr.hx, tr.hy, tr.speed, tr.length]), tr.ticks, tr.status)
                    for tr in trials])
        if running == 0:
            break
    for b, sc in enumerate(scs):
        st, recs = oracle.sim_run(sc, ocfg, trial=b, sweeps=100, iters=20, max_len=4096)
        assert len(recs) >= 1
        for t, r in enumerate(recs):
            rob, ticks, status = gpu[t][b]
            assert np.array_equal(rob, r["rob"]), (b, t)
            assert status == r["status"] and ticks == t + 1
        assert np.array_equal(pl.sim_histogram(b), st.hist)
        g, gm = pl.get_tracks(b)
        assert np.array_equal(g, st.tracks) and np.array_equal(gm, st.missed)


def test_sim_reset_validation_and_idle():
    sc = scene_sim(3, 2)
    gcfg, _ = _cfgs(10)
    pl = Planner(256, 256, 2, 0.1, (0.0, 0.0), device=0, stream=_stream())
    pl.set_static(sc.static, b=0)
    pl.set_static(sc.static, b=1)
    from paper_1903_07441_b200 import twg as T
    with pytest.raises(T.TwgError):
        pl.sim_tick(gcfg, warp_cfg(), relax_cfg(), band_cfg(), tracker_cfg())   # before any reset
    with pytest.raises(T.TwgError):
        pl.sim_reset(0, (30.0, 1.0, 0.0, 0.4), sc.goal, sc.truth, gcfg)         # robot outside the grid
    pl.sim_reset(0, sc.robot, sc.goal, sc.truth, gcfg)
    _, trials, running = pl.sim_tick(gcfg, warp_cfg(), relax_cfg(), band_cfg(), tracker_cfg())
    assert trials[1].status == S.IDLE and trials[0].ticks == 1 and running == 1


def test_sim_run_batch_terminates():
    scs = [scene_sim(40 + k, 2) for k in range(6)]
    res, ticks = S.run_batch(scs, cfg=sim_cfg(seed=2, max_ticks=900), stream=_stream())
    assert all(r["outcome"] in ("success", "collision", "timeout") for r in res)
    for r in res:
        assert r["hist"].sum() == r["ticks"]
        if r["outcome"] == "success":
            assert r["length_m"] >= r["straight_m"] - 0.31
    summ = S.summarize(res)
    assert summ["trials"] == 6 and 0.0 <= summ["success_pct"] <= 100.0
