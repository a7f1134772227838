"""Time twg_warp_map (f3) at 4096^2 and 16384^2 through the C ABI (CUDA events, 10 calls each).

Run from the repo root: python tools/time_warp_map.py
"""
import torch, json, sys
sys.path.insert(0, "tools"); sys.path.insert(0, ".")
from paper_1903_07441_b200 import Planner
st = torch.cuda.current_stream()
res = {}
for N in (4096, 16384):
    pl = Planner(N, N, 1, 0.1, (0.0, 0.0), device=0, stream=st.cuda_stream)
    dw = torch.zeros((N, N), dtype=torch.int32, device="cuda")
    robot = (N * 0.05 + 0.0123, N * 0.04 + 0.017, 0.7, 0.4)
    for _ in range(3): pl.warp_map(robot, 1.0, out=dw)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(10): pl.warp_map(robot, 1.0, out=dw)
    e1.record(st); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    res[N] = {"ms": ms, "gcells_s": N * N / ms / 1e6}
    pl.close(); del dw; torch.cuda.empty_cache()
print(json.dumps(res))
