"""Pins of the f2 simulator oracle (no GPU): counter-based generator, robot kinematics, obstacle
motion rules, trial status, turning-angle histogram, and one closed loop (P23; S:395-468,
S:536-562, C31-C36).  Expected values from geometry by hand and stated rules."""
import math
from dataclasses import replace

import numpy as np
import pytest

from scenes import SimCfg, Scene, default_warp_cfg, scene_sim


def _scene(W=64, H=64, static=None, robot=(1.05, 3.25, 0.0, 0.4), goal=(57, 32), truth=None):
    st = np.zeros((H, W), np.uint8) if static is None else static
    tr = np.zeros((0, 4)) if truth is None else np.asarray(truth, np.float64).reshape(-1, 4)
    return Scene("p23", W, H, 0.1, (0.0, 0.0), st, robot, goal, np.zeros((0, 20)), default_warp_cfg(), 0, tr)


def _move(orc, sc, st, wp, cfg):
    orc.sim_move(sc, st, wp, cfg, 0)


def test_p23_rng(orc):
    u = np.array([orc.rng_u01(7, 1, t, e, k) for t in range(20) for e in range(25) for k in range(40)])
    assert u.min() >= 0.0 and u.max() < 1.0 and len(np.unique(u)) == len(u)
    assert abs(u.mean() - 0.5) < 5 * math.sqrt(1 / 12 / len(u))
    assert orc.rng_u01(7, 1, 2, 3, 4) == orc.rng_u01(7, 1, 2, 3, 4)
    z = np.array([orc.rng_normal(3, 0, t, e, 1) for t in range(100) for e in range(100)])
    assert abs(z.mean()) < 5 / math.sqrt(len(z)) and abs(z.var() - 1.0) < 0.05
    assert np.abs(z).max() <= 6.0                         # Irwin-Hall support


def test_p23_sense_zero_noise_is_truth(orc):
    obs = np.array([[1.0, 2.0, 0.3, 0.0], [4.0, 5.0, 0.0, -0.2]])
    assert np.array_equal(orc.sim_sense(obs, 0.0, 1, 0, 0), obs[:, :2])
    z = orc.sim_sense(obs, 0.05, 1, 0, 3)
    assert np.all(np.abs(z - obs[:, :2]) <= 0.3) and not np.array_equal(z, obs[:, :2])


def test_p23_robot_kinematics(orc):
    cfg = SimCfg()
    sc = _scene()
    st = orc.SimState(sc, cfg)
    x0 = st.rob[:2].copy()
    _move(orc, sc, st, (40.5, 32.5), cfg)                  # waypoint straight ahead (+x)
    assert st.rob[2:4].tolist() == [1.0, 0.0] and st.rob[0] - x0[0] == pytest.approx(0.04, abs=1e-15)
    assert st.rob[1] == x0[1] and st.hist[0] == 1
    _move(orc, sc, st, (0.5, 32.5), cfg)                   # behind: saturate at turn_max = 9 degrees
    ang = math.degrees(math.atan2(st.rob[3], st.rob[2]))
    assert abs(abs(ang) - 9.0) < 1e-9 and st.hist[1] == 1
    h = st.rob[2:4].copy()
    _move(orc, sc, st, None, cfg)                          # blocked: straight on (never stops)
    assert np.array_equal(st.rob[2:4], h)
    assert st.rob[5] == pytest.approx(3 * 0.04, abs=1e-15) and st.ticks[0] == 3
    # waypoint exactly at the robot position (0 + 25 * 0.1 = 2.5): heading kept, still advances
    sc = _scene(robot=(2.5, 2.5, 0.3, 0.4))
    st = orc.SimState(sc, cfg)
    h = st.rob[2:4].copy()
    _move(orc, sc, st, (25.0, 25.0), cfg)
    assert np.array_equal(st.rob[2:4], h) and math.hypot(st.rob[0] - 2.5, st.rob[1] - 2.5) == pytest.approx(0.04)


def test_p23_turning_histogram_bin(orc):
    cfg = replace(SimCfg(), turn_max=math.pi)              # unlimited turn: heading = waypoint direction
    sc = _scene()
    st = orc.SimState(sc, cfg)
    a = math.radians(62.0)
    wp = ((st.rob[0] + math.cos(a)) / 0.1, (st.rob[1] + math.sin(a)) / 0.1)
    _move(orc, sc, st, wp, cfg)
    assert st.hist[12] == 1 and st.hist.sum() == 1          # 62 degrees -> bin [60, 65)


def test_p23_obstacle_rules(orc):
    cfg = replace(SimCfg(), heading_sigma=0.0)
    # open space: straight, exactly v dt
    sc = _scene(truth=[[3.0, 3.0, 0.3, 0.1]])
    st = orc.SimState(sc, cfg)
    _move(orc, sc, st, None, cfg)
    assert st.obs[0, 0] == pytest.approx(3.03, abs=1e-15) and st.obs[0, 1] == pytest.approx(3.01, abs=1e-15)
    # heading at a wall 0.4 m ahead (turn_distance 0.5): reflected, i.e. turned by 180 degrees >= 90
    static = np.zeros((64, 64), np.uint8); static[:, 40] = 1
    sc = _scene(static=static, truth=[[3.65, 3.0, 0.3, 0.0]])
    st = orc.SimState(sc, cfg)
    _move(orc, sc, st, None, cfg)
    assert st.obs[0, 2] == pytest.approx(-0.3, abs=1e-15) and st.obs[0, 0] < 3.65
    # two obstacles head-on within 2 r + turn_distance: both reflect about the centre line
    sc = _scene(truth=[[3.0, 3.0, 0.3, 0.0], [3.8, 3.0, -0.3, 0.0]])
    st = orc.SimState(sc, cfg)
    _move(orc, sc, st, None, cfg)
    assert st.obs[0, 2] == pytest.approx(-0.3) and st.obs[1, 2] == pytest.approx(0.3)
    # jitter keeps the speed; obstacles never leave the extent
    cfg2 = replace(SimCfg(), heading_sigma=0.3)
    rng = np.random.default_rng(0)
    tr = np.column_stack([rng.uniform(0.5, 6, 12), rng.uniform(0.5, 6, 12), rng.uniform(-0.5, 0.5, 12),
                          rng.uniform(-0.5, 0.5, 12)])
    sc = _scene(truth=tr, robot=(0.05, 0.05, 0.0, 0.0))
    st = orc.SimState(sc, cfg2)
    sp0 = st.speed.copy()
    for _ in range(300):
        st.status[0] = 0
        _move(orc, sc, st, None, cfg2)
        assert np.all(st.obs[:, :2] >= 0.25 - 1e-12) and np.all(st.obs[:, :2] <= 6.4 - 0.25 + 1e-12)
    assert np.allclose(np.hypot(st.obs[:, 2], st.obs[:, 3]), sp0, rtol=1e-12)


def test_p23_status(orc):
    cfg = SimCfg()
    sc = _scene(robot=(5.70, 3.25, 0.0, 0.4))               # goal cell (57, 32) centre (5.75, 3.25)
    st = orc.SimState(sc, cfg)
    _move(orc, sc, st, None, cfg)
    assert st.status[0] == orc.SIM_SUCCESS
    # obstacle at r_r + r_o - 0.01 from the robot's next position: collision (before success)
    sc = _scene(robot=(2.0, 2.0, 0.0, 0.4), truth=[[2.04 + 0.49, 2.0, 0.0, 1e-9]])
    st = orc.SimState(sc, replace(cfg, heading_sigma=0.0))
    _move(orc, sc, st, None, replace(cfg, heading_sigma=0.0))
    assert st.status[0] == orc.SIM_COLLISION
    static = np.zeros((64, 64), np.uint8); static[20, 23] = 1   # wall cell centre (2.35, 2.05)
    sc = _scene(static=static, robot=(2.06, 2.05, 0.0, 0.4))
    st = orc.SimState(sc, cfg)
    _move(orc, sc, st, None, cfg)                           # robot at (2.10, 2.05): 0.25 from the centre
    assert st.status[0] == orc.SIM_COLLISION
    sc = _scene(robot=(6.38, 3.0, 0.0, 0.4), goal=(5, 5))
    st = orc.SimState(sc, cfg)
    _move(orc, sc, st, None, cfg)                           # leaves the grid
    assert st.status[0] == orc.SIM_COLLISION
    sc = _scene(robot=(1.0, 1.0, 0.0, 0.4))
    st = orc.SimState(sc, replace(cfg, max_ticks=2))
    for _ in range(2):
        _move(orc, sc, st, None, replace(cfg, max_ticks=2))
    assert st.status[0] == orc.SIM_TIMEOUT and st.ticks[0] == 2


def test_p23_closed_loop_empty_room(orc):
    # empty room, goal 5 m ahead, no obstacles -> Success, length within 5 % of 5 m
    sc = _scene(robot=(0.75, 3.25, 0.0, 0.4), goal=(57, 32))
    st, recs = orc.sim_run(sc, SimCfg(max_ticks=400), sweeps=100, iters=50)
    assert st.status[0] == orc.SIM_SUCCESS
    d = math.hypot(5.75 - 0.75, 0.0)
    assert d - 0.3 <= st.rob[5] <= 1.05 * d
    assert all(r["wp"] is not None for r in recs)
