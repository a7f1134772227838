"""Time twg_relax at C3 for each temporal depth T (S sweeps, CUDA events): ms, GLUP/s, us per launch."""
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
S = 840
for T in range(1, 9):
    cfg = relax_cfg(max_sweeps=S, temporal_depth=T)
    pl.relax(cfg, want_result=False)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(3):
        pl.relax(cfg, want_result=False)
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    nl = -(-S // T)
    print(f"T={T}: {ms:.3f} ms  {4096 * 4096 * S / ms / 1e6:.0f} GLUP/s  {1000 * ms / nl:.2f} us/launch "
          f"({1000 * ms / S:.2f} us/sweep)", flush=True)
