"""Converge the C3 field, time the path kernels (index + walk + band), optionally save the raw field."""
import sys, os, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1903_07441_b200 import Planner, band_cfg, relax_cfg, warp_cfg
from scenes import scene_c3
sc = scene_c3(0)
st = torch.cuda.current_stream().cuda_stream
pl = Planner(sc.W, sc.H, 1, sc.cell_size, sc.origin, 0, st)
pl.set_static(sc.static)
pl.set_obstacles(0, sc.robot, sc.goal, sc.tracks, warp_cfg(), warm=0)
t0 = time.time()
sw, res = pl.relax(relax_cfg(max_sweeps=4_000_000, check_every=20000, tol=1e-38, sync_every=4))
print("prep", sw, res, time.time() - t0, flush=True)
for it in (0, 50, 50, 50):
    torch.cuda.synchronize(); t1 = time.time()
    s, cells, sm, ns, nxt = pl.extract_path(0, band_cfg(it, 40000, 80000))
    torch.cuda.synchronize(); t2 = time.time()
    print(json.dumps({"iters": it, "walk": s, "n_cells": len(cells), "n_smooth": int(ns), "ms": 1e3 * (t2 - t1),
                      **pl.debug_walk(0)}), flush=True)
if len(sys.argv) > 1:
    np.save(sys.argv[1], pl.get_field(0, 0))
