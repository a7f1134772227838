"""Relaxation-only timing on C3 (4096^2): twg_relax of S sweeps (T-sweep launches), CUDA events,
both k_rb_tblock paths (packed fast path; TWG_RELAX_SLOW=1 forces the scalar path)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1903_07441_b200 import Planner, relax_cfg, warp_cfg
from scenes import scene_c3
S = int(os.environ.get("S", "600"))
sc = scene_c3(0)
st = torch.cuda.current_stream()
pl = Planner(sc.W, sc.H, 1, sc.cell_size, sc.origin, 0, st.cuda_stream)
pl.set_static(sc.static)
pl.set_obstacles(0, sc.robot, sc.goal, sc.tracks, warp_cfg(), warm=0)
out = {}
ROWS = [int(r) for r in os.environ.get("ROWS", "0").split(",")]
for T, R in [(int(t), r) for t in os.environ.get("TS", "4,6,8").split(",") for r in ROWS]:
    rc = relax_cfg(max_sweeps=S, temporal_depth=T, rows_per_warp=R)
    pl.relax(rc, want_result=False)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        pl.relax(rc, want_result=False)
        e1.record(st)
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    glups = sc.W * sc.H * S / (best * 1e-3) / 1e9
    out[f"T{T}_R{R}"] = {"glups": round(glups, 1), "us_per_launch": round(best * 1e3 / (S / T), 2)}
print(json.dumps({"slow": os.environ.get("TWG_RELAX_SLOW", "0"), "S": S, "res": out}))
