"""C1 time to tolerance (64^2, tol 1e-6, check every sweep): twg_relax alone and twg_relax + path,
CUDA events, best of 5 (TWG_NO_SMALL=1: the tile kernel with one launch + check per sweep)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1903_07441_b200 import Planner, band_cfg, relax_cfg, warp_cfg
from scenes import scene_c1
sc = scene_c1()
st = torch.cuda.current_stream()
pl = Planner(sc.W, sc.H, 1, sc.cell_size, sc.origin, 0, st.cuda_stream)
pl.set_static(sc.static)
out = {}
for with_path in (False, True):
    best = 1e9
    for _ in range(5):
        pl.set_obstacles(0, sc.robot, sc.goal, sc.tracks, warp_cfg(), warm=0)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        sw, _ = pl.relax(relax_cfg(max_sweeps=10 ** 6, check_every=1, tol=1e-6, warm_start=0), want_result=False)
        if with_path:
            pl.extract_path(0, band_cfg(50, 1000, 4000))
        e1.record(st)
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    out["relax+path" if with_path else "relax"] = round(best, 3)
print(json.dumps({"small": os.environ.get("TWG_NO_SMALL", "0") != "1", "ms": out}))
