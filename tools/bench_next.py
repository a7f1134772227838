"""Measurement of the SURVEY.md 8(f) rows on one B200 (CUDA events on the library's stream, after
warm-up), each against its roofline; writes one JSON object (stdout and --out).

  f3 Jacobi (k_jacobi):        8 B per cell per sweep (fp32 read + write)      -> HBM roofline
  f3 lexicographic (k_lex):    8 B per cell per sweep; wavefront-latency bound in practice
  f3 index matrix (k_index_dir + 2D copy-out): 4 B read + 1 B written per cell (+1 B D2D copy)
  f3 warp map (k_warp_map):    4 B written per cell (int32), fp64 math per cell
  f1 tracker tick:             latency per tick at 200 (C3) and 3200 (C4) tracks, plus the
                               k_trk_* share; no HBM-relevant traffic (~200 B per track)
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1903_07441_b200 import Planner, relax_cfg, warp_cfg, tracker_cfg  # noqa: E402
from scenes import scene_random, detections  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PEAK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]


def timed(fn, reps, st):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(reps):
        fn()
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    st = torch.cuda.current_stream()
    out = {"peak_hbm_gbs": PEAK}
    for N, S in ((4096, 200), (16384, 40)):
        sc = scene_random("bn", N, N // 8, N // 20, 1)
        pl = Planner(N, N, 1, 0.1, (0.0, 0.0), device=0, stream=st.cuda_stream)
        pl.set_static(sc.static)
        pl.set_obstacles(0, sc.robot, sc.goal, sc.tracks, warp_cfg(), warm=0)
        ms = timed(lambda: pl.relax(relax_cfg(max_sweeps=S, mode=1), want_result=False), 3, st)
        glups = N * N * S / ms / 1e6
        out[f"jacobi_{N}"] = {"sweeps": S, "ms": ms, "glups": glups, "gbs": 8 * glups,
                              "frac_hbm": 8 * glups / PEAK}
        SL = max(S // 10, 4)
        ms = timed(lambda: pl.relax(relax_cfg(max_sweeps=SL, mode=2), want_result=False), 2, st)
        gl = N * N * SL / ms / 1e6
        out[f"lexicographic_{N}"] = {"sweeps": SL, "ms": ms, "glups": gl, "gbs_equiv_8B": 8 * gl,
                                     "frac_hbm_8B": 8 * gl / PEAK}
        ms_rb = timed(lambda: pl.relax(relax_cfg(max_sweeps=S), want_result=False), 3, st)
        out[f"redblack_{N}"] = {"sweeps": S, "ms": ms_rb, "glups": N * N * S / ms_rb / 1e6}
        dm = torch.zeros((N, N), dtype=torch.uint8, device="cuda")
        ms = timed(lambda: pl.index_matrix(0, out=dm), 10, st)
        out[f"index_matrix_{N}"] = {"ms": ms, "gbs": 6 * N * N / ms / 1e6, "frac_hbm": 6 * N * N / ms / 1e6 / PEAK,
                                    "bytes_per_cell": 6}
        dw = torch.zeros((N, N), dtype=torch.int32, device="cuda")
        ms = timed(lambda: pl.warp_map(sc.robot, 1.0, out=dw), 10, st)
        out[f"warp_map_{N}"] = {"ms": ms, "gbs": 4 * N * N / ms / 1e6, "frac_hbm": 4 * N * N / ms / 1e6 / PEAK,
                                "bytes_per_cell": 4}
        pl.close()
        del dm, dw
        torch.cuda.empty_cache()
    # C3 (iii): cold time to tolerance 1e-6 (reported only)
    sc = scene_random("c3_4096_s0", 4096, 512, 200, 0)
    pl = Planner(4096, 4096, 1, 0.1, (0.0, 0.0), device=0, stream=st.cuda_stream)
    pl.set_static(sc.static)
    pl.set_obstacles(0, sc.robot, sc.goal, sc.tracks, warp_cfg(), warm=0)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    sw, res = pl.relax(relax_cfg(max_sweeps=4_000_000, check_every=1000, tol=1e-6, sync_every=8))
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    out["c3_cold_time_to_tol_1e-6"] = {"sweeps": int(sw[0]), "residual": float(res[0]), "ms": ms,
                                       "glups": 4096 * 4096 * int(sw[0]) / ms / 1e6}
    pl.close()
    for name, N, n_obs in (("c3", 4096, 200), ("c4", 16384, 3200)):
        # the tracker is independent of the grid: a small context holds the resident table
        sc = scene_random("tk", N, 8, n_obs, 2)
        pl = Planner(1024, 1024, 1, 0.1, (0.0, 0.0), device=0, stream=st.cuda_stream)
        wc = warp_cfg()
        zs = [torch.as_tensor(detections(sc, t, n_clutter=n_obs // 20), device="cuda") for t in range(1, 12)]
        ticks = []
        for rep in range(2):
            pl.set_obstacles(0, (0.55, 0.55, 0.0, 0.4), (3, 3), sc.tracks, wc, warm=0)
            torch.cuda.synchronize()
            for z in zs:
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st)
                pl.track_update(0, z, [len(z)], wc, tracker_cfg())
                e1.record(st)
                torch.cuda.synchronize()
                if rep == 1:
                    ticks.append(e0.elapsed_time(e1))
        out[f"tracker_{name}"] = {"tracks": n_obs, "detections_per_tick": int(np.mean([len(z) for z in zs])),
                                  "ms_per_tick_median": float(np.median(ticks)),
                                  "ticks_per_s": 1000.0 / float(np.median(ticks)),
                                  "note": "CUDA events around twg_track_update, incl. its host read-back of counts"}
        pl.close()
    print(json.dumps(out, indent=1))
    if a.out:
        with open(a.out, "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
