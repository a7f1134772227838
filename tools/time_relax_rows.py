"""Time twg_relax at C3 (T = 6) for several rows-per-warp settings (0 = the library's load model)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1903_07441_b200 import Planner, relax_cfg, warp_cfg  # noqa: E402
from scenes import scene_c3  # noqa: E402

sc = scene_c3(0)
st = torch.cuda.current_stream()
pl = Planner(sc.W, sc.H, 1, sc.cell_size, sc.origin, device=0, stream=st.cuda_stream)
pl.set_static(sc.static)
pl.set_obstacles(0, sc.robot, sc.goal, sc.tracks, warp_cfg(), warm=0)
S = 600
for rows in [0] + [int(a) for a in sys.argv[1:]]:
    cfg = relax_cfg(max_sweeps=S, temporal_depth=6, rows_per_warp=rows)
    pl.relax(cfg, want_result=False)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(5):
        pl.relax(cfg, want_result=False)
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"rows={rows}: {ms:.3f} ms  {4096 * 4096 * S / ms / 1e6:.0f} GLUP/s  {1000 * ms / 100:.2f} us/launch", flush=True)
