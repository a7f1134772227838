"""Why do ~7 % of the C5 scenario-steps report NoPath?  For the 1024 C5 scenes (tick 0 relaxed to the
exact fp32 fixed point on the GPU, then warm ticks as in bench.py), classify every NoPath by
  enclosed:   the robot cell is not 4-connected to the goal through free cells (BFS on the class grid
              of the oracle's encode) -- no path exists at all;
  underflow:  connected, but |u| at the robot cell is below 1e-30: the harmonic field has decayed
              below fp32's resolution on the way (narrow passages), so the descent walk meets flat /
              subnormal plateaus and cycles (DESIGN C3);
  unconverged: connected, and the scenario's tick-0 cold solve stopped at the sweep cap with a nonzero
              residual: the cold field (every free cell 0.5) drains through narrow passages so
              slowly that a flat local maximum survives, where the walk cycles;
  other.
Writes profiles/r02_c5_nopath.json."""
import json, os, sys
from collections import deque
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import oracle
from paper_1903_07441_b200 import Planner, band_cfg, relax_cfg, warp_cfg
from scenes import advance_scene, scene_random


def connected(cls, start, goal):
    H, W = cls.shape
    seen = np.zeros_like(cls, bool)
    q = deque([start])
    seen[start[1], start[0]] = True
    while q:
        x, y = q.popleft()
        if (x, y) == goal:
            return True
        for dx, dy in ((1, 0), (-1, 0), (0, 1), (0, -1)):
            nx, ny = x + dx, y + dy
            if 0 <= nx < W and 0 <= ny < H and not seen[ny, nx] and cls[ny, nx] != oracle.OBSTACLE:
                seen[ny, nx] = True
                q.append((nx, ny))
    return False


N = int(os.environ.get("N", "1024"))
ticks = int(os.environ.get("TICKS", "3"))
scs = [scene_random(f"c5_s{s}", 512, 8, 20, s) for s in range(N)]
st = torch.cuda.current_stream().cuda_stream
pl = Planner(512, 512, N, 0.1, (0.0, 0.0), device=0, stream=st)
for b, sc in enumerate(scs):
    pl.set_static(sc.static, b)
wc, bc = warp_cfg(), band_cfg(50, 4096, 8192)
counts = {"steps": 0, "no_path": 0, "enclosed": 0, "underflow": 0, "unconverged": 0, "other": 0,
          "goal_swallowed": 0}
cap = int(os.environ.get("PREP", "100000"))
tick0_unconverged = set()
examples = []
for tick in range(ticks + 1):
    ss = [advance_scene(sc, tick) for sc in scs]
    rob = np.array([s.robot for s in ss], np.float64)
    goals = np.array([s.goal for s in ss], np.int32)
    tr = np.ascontiguousarray(np.vstack([s.tracks for s in ss]))
    nt = np.array([s.n_tracks for s in ss], np.int32)
    rc = (relax_cfg(max_sweeps=cap, check_every=2000, tol=1e-38, warm_start=0, sync_every=4) if tick == 0
          else relax_cfg(max_sweeps=100, warm_start=1))
    _, res, _, _ = pl.plan_step(-1, rob, goals, tr, nt, wc, rc, bc, want_paths=False)
    if tick == 0:
        tick0_unconverged = {b for b, r in enumerate(res) if r.residual > 0.0}
        counts["tick0_unconverged_scenarios"] = len(tick0_unconverged)
        continue
    for b, r in enumerate(res):
        counts["steps"] += 1
        counts["goal_swallowed"] += int(r.status == 1)
        if r.walk_status == 0:
            continue
        counts["no_path"] += 1
        _, cls, *_ = oracle.classify(ss[b])
        start = oracle.robot_cell(ss[b])
        if not connected(cls, start, tuple(ss[b].goal)):
            kind = "enclosed"
        else:
            u = pl.get_field(b, 1)
            kind = ("underflow" if u[start[1], start[0]] < 1e-30 else
                    "unconverged" if b in tick0_unconverged else "other")
            if kind == "other" and len(examples) < 5:
                examples.append({"scenario": b, "tick": tick, "u_robot": float(u[start[1], start[0]])})
        counts[kind] += 1
out = {"config": f"C5: {N} scenes 512^2, tick 0 cold to the fp32 fixed point (cap {cap} sweeps), then {ticks} warm "
                 f"ticks of S = 100",
       "counts": counts, "other_examples": examples}
print(json.dumps(out))
os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
json.dump(out, open(os.path.join(ROOT, "profiles", "r02_c5_nopath.json"), "w"), indent=1)
