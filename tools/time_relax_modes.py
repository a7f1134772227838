"""Time red-black (mode 0) and Jacobi (mode 1) relaxation sweeps on one grid (CUDA events)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1903_07441_b200 import Planner, relax_cfg, warp_cfg
from scenes import scene_random

N = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
S = int(sys.argv[2]) if len(sys.argv) > 2 else 240
sc = scene_random("t", N, 40, 200, 1)
st = torch.cuda.current_stream()
pl = Planner(N, N, 1, sc.cell_size, sc.origin, device=0, stream=st.cuda_stream)
pl.set_static(sc.static)
pl.set_obstacles(0, sc.robot, sc.goal, sc.tracks, warp_cfg(), warm=0)
for mode in (0, 1):
    cfg = relax_cfg(max_sweeps=S, mode=mode)
    pl.relax(cfg, want_result=False)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(5):
        pl.relax(cfg, want_result=False)
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"mode {mode}: {S} sweeps {N}x{N}: {ms:.3f} ms  {N * N * S / ms / 1e6:.1f} GLUP/s  "
          f"{8 * N * N * S / ms / 1e6:.1f} GB/s-equiv")
