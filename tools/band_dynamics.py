"""Rubber-band dynamics on the C3 bench path (diagnostic, GPU box): after the bench's prep and
one warm plan step, run the oracle band for k = 0..iters iterations and report, per iteration,
how many waypoints differ from iteration k-1 and k-2 (fixed points / period-2 oscillations),
and per 64-waypoint chunk (the k_band CTA size) the last iteration in which its local run of
64 + 4 I waypoints changed.  Writes gpurun_out/band_dyn.json."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import oracle
from paper_1903_07441_b200 import Planner, band_cfg, relax_cfg, warp_cfg
from scenes import advance_scene, scene_c3

iters = 50
sc0 = scene_c3(0)
pl = Planner(sc0.W, sc0.H, 1, sc0.cell_size, sc0.origin, 0, torch.cuda.current_stream().cuda_stream)
pl.set_static(sc0.static)
bc = band_cfg(iters, 4 * (sc0.W + sc0.H), 8 * (sc0.W + sc0.H))
wc = warp_cfg()
pl.plan_step(0, [sc0.robot], [sc0.goal], sc0.tracks, [sc0.n_tracks], wc,
             relax_cfg(max_sweeps=4_000_000, check_every=20000, tol=1e-38, warm_start=0, sync_every=4), bc,
             want_paths=False)
s = advance_scene(sc0, 1)
st, res, cells, sm = pl.plan_step(0, [s.robot], [s.goal], s.tracks, [s.n_tracks], wc,
                                  relax_cfg(max_sweeps=100, warm_start=1), bc)
n = res[0].n_cells
raw = pl.get_field(0, 0)
u = np.abs(raw)
cls = np.zeros(raw.shape, np.uint8)
bits = raw.view(np.uint32)
cls[bits == 0] = 1
cls[raw == 1.0] = 2
w0 = oracle.cells_to_waypoints(cells[0, :n])
states = [w0]
for k in range(1, iters + 1):
    states.append(oracle.band(cls, u, w0, iters=k))
out = {"n": int(n), "per_iter": []}
for k in range(1, iters + 1):
    d1 = int(np.any(states[k] != states[k - 1], axis=1).sum())
    d2 = int(np.any(states[k] != states[k - 2], axis=1).sum()) if k >= 2 else -1
    out["per_iter"].append((k, d1, d2))
chg = np.array([np.any(states[k] != states[k - 1], axis=1) for k in range(1, iters + 1)])  # iters x n
C, h = 64, 2 * iters
last = []
for c0 in range(0, n, C):
    lo, hi = max(c0 - h, 0), min(c0 + C + h, n)
    it = np.nonzero(chg[:, lo:hi].any(axis=1))[0]
    last.append(int(it[-1] + 1) if len(it) else 0)
out["chunk_last_change"] = last
# which waypoints still move at the end, and do they cycle
late = np.nonzero(chg[-5:].any(axis=0))[0]
out["late_movers"] = late[:50].tolist()
out["late_traj"] = {int(i): [states[k][i].tolist() for k in range(iters - 6, iters + 1)] for i in late[:5]}
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/band_dyn.json", "w"))
print(json.dumps({"n": n, "tail": out["per_iter"][-8:], "max_last": max(last),
                  "hist": np.bincount(np.array(last) // 10).tolist()}))
# periodicity of each chunk's local run at the end: smallest p with state[iters] == state[iters - p]
per = []
for c0 in range(0, n, C):
    lo, hi = max(c0 - h, 0), min(c0 + C + h, n)
    pp = 0
    for p_ in range(1, 25):
        if np.array_equal(states[iters][lo:hi], states[iters - p_][lo:hi]):
            pp = p_
            break
    # first iteration k at which the local run state repeats with that period
    first = -1
    if pp:
        for k in range(pp, iters + 1):
            if np.array_equal(states[k][lo:hi], states[k - pp][lo:hi]):
                first = k
                break
    per.append((pp, first))
allm = np.nonzero(chg[-10:].any(axis=0))[0]
print(json.dumps({"period_first": [x for x in per if x[1] != 0][-12:], "n_late": int(len(allm)),
                  "late_range": [int(allm.min()), int(allm.max())] if len(allm) else None}))
tr = {int(i): [states[k][i].tolist() for k in range(iters - 12, iters + 1)] for i in (7010, 7020, 7030, 7100, 7200)}
print(json.dumps(tr))
