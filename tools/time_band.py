"""Event-timed twg_extract_path on the converged C3 field with 0 and 50 band iterations (the
difference is the rubber band's share); relaxes to the fp32 fixed point first (~13 s)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1903_07441_b200 import Planner, band_cfg, relax_cfg, warp_cfg
from scenes import scene_c3
sc = scene_c3(0)
st = torch.cuda.current_stream()
pl = Planner(sc.W, sc.H, 1, sc.cell_size, sc.origin, 0, st.cuda_stream)
pl.set_static(sc.static)
pl.set_obstacles(0, sc.robot, sc.goal, sc.tracks, warp_cfg(), warm=0)
pl.relax(relax_cfg(max_sweeps=4_000_000, check_every=20000, tol=1e-38, sync_every=4))
out = {}
for it in (0, 50, 100):
    best = 1e9
    for rep in range(6):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        s, cells, sm, ns, nxt = pl.extract_path(0, band_cfg(it, 40000, 80000))
        e1.record(st)
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    out[it] = {"ms": round(best, 4), "n_cells": len(cells), "n_smooth": int(ns)}
print(json.dumps(out))
