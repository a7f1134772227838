"""ncu driver: a few tracker ticks at C4 scale (3200 tracks, ~3360 detections)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1903_07441_b200 import Planner, warp_cfg, tracker_cfg  # noqa: E402
from scenes import scene_random, detections  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 3200
sc = scene_random("tk", 16384, 8, n, 2)
st = torch.cuda.current_stream()
pl = Planner(1024, 1024, 1, 0.1, (0.0, 0.0), device=0, stream=st.cuda_stream)
wc = warp_cfg()
pl.set_obstacles(0, (0.55, 0.55, 0.0, 0.4), (3, 3), sc.tracks, wc, warm=0)
for t in range(1, 5):
    z = torch.as_tensor(detections(sc, t, n_clutter=n // 20), device="cuda")
    print(pl.track_update(0, z, [len(z)], wc, tracker_cfg()))
