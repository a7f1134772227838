"""Sweep temporal depth T and rows per warp for twg_relax on C3 (kernel-only GLUP/s, S sweeps)."""
import sys, os, json, itertools
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1903_07441_b200 import Planner, relax_cfg, warp_cfg
from scenes import scene_c3
sc = scene_c3(0)
st = torch.cuda.current_stream()
pl = Planner(sc.W, sc.H, 1, sc.cell_size, sc.origin, 0, st.cuda_stream)
pl.set_static(sc.static)
pl.set_obstacles(0, sc.robot, sc.goal, sc.tracks, warp_cfg(), warm=0)
S = int(sys.argv[1]) if len(sys.argv) > 1 else 960
Ts = [int(t) for t in sys.argv[2].split(",")] if len(sys.argv) > 2 else [2, 3, 4, 5, 6, 8]
rows = [int(r) for r in sys.argv[3].split(",")] if len(sys.argv) > 3 else [0, 24, 44, 64, 104, 144, 224]
for T, r in itertools.product(Ts, rows):
    cfg = relax_cfg(max_sweeps=S, temporal_depth=T, rows_per_warp=r)
    pl.relax(cfg, want_result=False)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(st)
    for _ in range(3):
        pl.relax(cfg, want_result=False)
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    print(json.dumps({"T": T, "rows": r, "glups": round(sc.W * sc.H * S / ms / 1e6, 1), "us_per_launch": round(1e3 * ms / (S / T), 2)}), flush=True)
