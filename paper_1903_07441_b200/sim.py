"""Batched closed-loop trials: Algorithm 1 driving a
simulated robot among wandering obstacles, every trial of a batch on the GPU at once.

Each tick is one `twg_sim_tick` call (tracker tick, Map Update from the resident tracks,
relaxation, path, robot and obstacle motion, status, next detections -- all in libtwg kernels);
this module only sets the trials up and aggregates their metrics the way the paper reports them:
success rate per obstacle count (Table 1), traversed length (Table 2), and the
turning-angle histogram.
"""
from __future__ import annotations

import numpy as np

from .twg import Planner, band_cfg, relax_cfg, sim_cfg, tracker_cfg, warp_cfg

RUNNING, SUCCESS, COLLISION, TIMEOUT, IDLE = 0, 1, 2, 3, 4
OUTCOME = {SUCCESS: "success", COLLISION: "collision", TIMEOUT: "timeout", RUNNING: "running", IDLE: "idle"}


def run_batch(scenes, cfg=None, wcfg=None, rcfg=None, bcfg=None, tcfg=None, device=0, stream=None, max_ticks=None):
    """Run one trial per scene (all scenes share W, H, cell size, origin) to completion.

    scenes: scenes.Scene objects with `truth` = obstacle states (x, y, vx, vy).  Returns a list of
    per-trial dicts (outcome, ticks, length_m, straight_m, hist[36]) and the tick count."""
    cfg = cfg or sim_cfg()
    wcfg = wcfg or warp_cfg()
    rcfg = rcfg or relax_cfg(max_sweeps=1000, warm_start=1)
    bcfg = bcfg or band_cfg(50, 4096, 8192)
    tcfg = tcfg or tracker_cfg()
    s0 = scenes[0]
    pl = Planner(s0.W, s0.H, len(scenes), s0.cell_size, s0.origin, device=device, stream=stream)
    try:
        for b, sc in enumerate(scenes):
            pl.set_static(np.ascontiguousarray(sc.static, np.uint8), b=b)
            pl.sim_reset(b, sc.robot, sc.goal, sc.truth, cfg)
        ticks = 0
        limit = cfg.max_ticks if max_ticks is None else max_ticks
        trials = None
        while ticks < limit:
            _, trials, running = pl.sim_tick(cfg, wcfg, rcfg, bcfg, tcfg)
            ticks += 1
            if running == 0:
                break
        out = []
        for b, sc in enumerate(scenes):
            t = trials[b]
            gx = sc.origin[0] + (sc.goal[0] + 0.5) * sc.cell_size
            gy = sc.origin[1] + (sc.goal[1] + 0.5) * sc.cell_size
            out.append({"scene": sc.name, "obstacles": int(len(sc.truth)), "outcome": OUTCOME[t.status],
                        "ticks": t.ticks, "length_m": t.length,
                        "straight_m": float(np.hypot(gx - sc.robot[0], gy - sc.robot[1])),
                        "hist": pl.sim_histogram(b)})
        return out, ticks
    finally:
        pl.close()


def summarize(results):
    """Table 1 / Table 2 / histogram analogues of one batch of trials with the same obstacle count."""
    n = len(results)
    succ = [r for r in results if r["outcome"] == "success"]
    hist = np.sum([r["hist"] for r in results], axis=0) if results else np.zeros(36, np.int64)
    tot = max(int(hist.sum()), 1)
    return {"trials": n, "success_pct": 100.0 * len(succ) / max(n, 1),
            "collision_pct": 100.0 * sum(r["outcome"] == "collision" for r in results) / max(n, 1),
            "timeout_pct": 100.0 * sum(r["outcome"] == "timeout" for r in results) / max(n, 1),
            "mean_length_cm": 100.0 * float(np.mean([r["length_m"] for r in succ])) if succ else None,
            "mean_length_over_straight": float(np.mean([r["length_m"] / r["straight_m"] for r in succ])) if succ else None,
            "turns_below_15deg_pct": 100.0 * float(hist[:3].sum()) / tot,
            "hist_5deg": hist.tolist()}
