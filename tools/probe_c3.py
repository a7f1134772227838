"""Probe: sweeps needed before the C3 descent walk reaches the goal, and walk/band costs.
usage: probe_c3.py N_SEG N_OBS CHUNK NCHUNK"""
import sys, os, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1903_07441_b200 import Planner, band_cfg, relax_cfg, warp_cfg
from scenes import scene_random

nseg, nobs, chunk, nchunk = (int(a) for a in sys.argv[1:5])
sc = scene_random("p", 4096, nseg, nobs, 0)
st = torch.cuda.current_stream().cuda_stream
pl = Planner(sc.W, sc.H, 1, sc.cell_size, sc.origin, 0, st)
pl.set_static(sc.static)
pl.set_obstacles(0, sc.robot, sc.goal, sc.tracks, warp_cfg(), warm=0)
total = 0
rx, ry = int(sc.robot[0]/0.1), int(sc.robot[1]/0.1)
for k in range(nchunk):
    torch.cuda.synchronize(); t0 = time.time()
    pl.relax(relax_cfg(max_sweeps=chunk), want_result=False)
    torch.cuda.synchronize(); dt = time.time() - t0
    total += chunk
    torch.cuda.synchronize(); t1 = time.time()
    s, cells, sm, ns, nxt = pl.extract_path(0, band_cfg(50, 40000, 80000))
    torch.cuda.synchronize(); t2 = time.time()
    u = pl.get_field(0, 1)
    print(json.dumps({"nseg": nseg, "sweeps": total, "glups": round(sc.W*sc.H*chunk/dt/1e9), "walk": s,
                      "n_cells": len(cells), "n_smooth": int(ns), "path_ms": round(1e3*(t2-t1), 3),
                      "u_robot": float(u[ry, rx]), "n_zero_free": int((u == 0).sum() - (pl.get_field(0,0).view(np.uint32) == 0).sum())}), flush=True)
