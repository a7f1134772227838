#!/usr/bin/env python
"""Benchmark of the Time-Warped Grid hot path on B200 (BASELINE.json metric:
"harmonic relaxation GLUP/s and plan steps/sec at 4096^2; % of HBM roofline").

A step = one planning tick of Algorithm 1 through the C ABI:
twg_plan_step = rows a1-a3 (time-warped stamping of 200 Kalman tracks) + a4-a6
(S = 100 red-black sweeps, warm start, Alg. 1) + a7-a9 (descent walk,
50 rubber-band iterations, resampling, next waypoint), on config C3
(4096 x 4096, 200 moving obstacles, BASELINE.json configs[2]).

  value       = 4096^2 * S * K / (device time of K steps), inputs resident in HBM
  e2e         = same metric, tracks copied from pinned host memory and the path
                read back to the host inside every timed step
  relax_glups = kernel-only relaxation throughput (twg_relax, S = 1000)
  roofline    = k_rb_tblock (the dominant kernel): 8 B per cell per launch
                (one fp32 read + one fp32 write; T sweeps fused on chip) over its
                CUDA-event launch time, vs MEASURED_PEAKS.json hbm_gbs
  cpu_baseline= the oracle (oracle/, single thread) on a bounded sample

N > 1 (torchrun): every rank plans its own independent 4096^2 scenario
(seed = rank): the units shard with no data-path collective ("weak").
--impl reference times the CPU oracle (the reference arm of this tier).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "harmonic relaxation GLUP/s and plan steps/sec at 4096^2; % of HBM roofline"
UNIT = "GLUP/s"


def _args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--sweeps", type=int, default=100)
    ap.add_argument("--band-iters", type=int, default=50)
    ap.add_argument("--relax-sweeps", type=int, default=1000)
    ap.add_argument("--T", type=int, default=0, help="temporal depth (0 = library default)")
    ap.add_argument("--rows", type=int, default=0, help="rows per warp (0 = library default)")
    ap.add_argument("--size", type=int, default=4096)
    ap.add_argument("--obstacles", type=int, default=200)
    ap.add_argument("--prep-sweeps", type=int, default=4_000_000,
                    help="untimed cold solve before the timed warm ticks (stops at the exact fp32 fixed point)")
    ap.add_argument("--config", default="c3", choices=["c3", "c4", "c5"],
                    help="c3: 4096^2 plan step (default, headline); c4: 16384^2 row slabs over the ranks; "
                         "c5: 1024 x 512^2 scenarios split over the ranks")
    ap.add_argument("--k", type=int, default=12, help="c4: sweeps between ghost exchanges")
    ap.add_argument("--batch", type=int, default=1024, help="c5: total scenarios")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-clocks", action="store_true")
    ap.add_argument("--no-sub", action="store_true", help="skip the c4_slab / c5_batch sub-results")
    ap.add_argument("--probe", action="store_true", help="launcher check: every rank prints its rank and exits")
    return ap.parse_args()


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def _scene(args, seed):
    from scenes import scene_random
    n_seg = max(1, int(512 * (args.size / 4096) ** 2))
    return scene_random(f"c3_{args.size}_s{seed}", args.size, n_seg, args.obstacles, seed)


class Clocks:
    """nvidia-smi clocks/throttle sampling during the timed region (B200_PROFILING.md)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index, enabled=True):
        self.index, self.enabled, self.proc = index, enabled, None

    def __enter__(self):
        if self.enabled:
            self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
            try:
                self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                              "--format=csv,noheader,nounits", "-lms", "200"],
                                             stdout=self.f, stderr=subprocess.DEVNULL)
                time.sleep(0.3)
            except OSError:
                self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            self.proc.wait()

    def summary(self):
        if self.proc is None:
            return None
        rows = [r.split(",") for r in open(self.f.name).read().strip().splitlines() if r.strip()]
        os.unlink(self.f.name)
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            try:
                sm.append(float(r[1]))
                mx = max(mx, float(r[2]))
                for k, nm in enumerate(names):
                    if r[5 + k].strip().lower() == "active":
                        reasons.add(nm)
            except (ValueError, IndexError):
                continue
        if not sm:
            return None
        load = [v for v in sm if v > 0.5 * mx] or sm
        return {"sm_mhz": float(np.median(load)), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------------------- CPU oracle arm
def _oracle_sample(args, sweeps, steps, seed=0, threads=1):
    """Oracle plan steps (as it stands; its OpenMP variants on `threads` host cores, bit-identical to
    the single-thread oracle, P14) on the same workload; GLUP/s."""
    import oracle
    from scenes import advance_scene
    sc0 = _scene(args, seed)
    prev = None
    t_total, lups = 0.0, 0
    for k in range(steps):
        sc = advance_scene(sc0, k)
        t0 = time.perf_counter()
        prev = oracle.plan_step(sc, max_sweeps=sweeps, iters=args.band_iters, max_len=4 * (sc.W + sc.H), prev=prev,
                                threads=threads)
        t_total += time.perf_counter() - t0
        lups += sc.W * sc.H * sweeps
    return lups / t_total / 1e9, t_total


def run_reference(args):
    ws, rank, _ = _dist()
    if rank != 0:
        return
    import oracle
    oracle.build()
    s = args.sweeps  # the GPU arm's S: same workload, same metric
    cores = oracle.host_cores()
    _oracle_sample(args, s, args.warmup, threads=cores)
    g, t = _oracle_sample(args, s, args.steps, threads=cores)
    line = {"metric": METRIC, "value": g, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * t / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic", "impl": "reference",
            "config": {"workload": f"c3_{args.size}: {args.size}x{args.size} grid, {args.obstacles} moving obstacles, "
                                   f"one plan step per step (oracle sample: S={s} sweeps, I={args.band_iters})",
                       "sweeps": s},
            "cpu_baseline": {"value": g, "unit": UNIT, "cores": cores, "kind": "oracle",
                             "sample": f"{args.steps} oracle plan steps of c3 seed 0 with S={s} sweeps, "
                                       f"I={args.band_iters} (OpenMP variants on {cores} host cores)"},
            "e2e": {"value": g, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------- GPU arm
def run_ours(args):
    import torch
    ws, rank, local = _dist()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    from paper_1903_07441_b200 import Planner, band_cfg, relax_cfg, warp_cfg, lib
    from scenes import advance_scene
    lib()
    stream = torch.cuda.current_stream(dev)
    sc0 = _scene(args, rank)
    N = sc0.W
    wc = warp_cfg()
    bc = band_cfg(args.band_iters, 4 * (sc0.W + sc0.H), 8 * (sc0.W + sc0.H))
    pl = Planner(sc0.W, sc0.H, 1, sc0.cell_size, sc0.origin, device=local, stream=stream.cuda_stream)
    pl.set_static(sc0.static)
    # tick 0 (untimed): cold start, relaxed until the fp32 field stops changing (residual exactly 0)
    # or prep_sweeps, so the timed ticks run in the warm steady state of the plan loop (C7)
    t_prep = time.perf_counter()
    st, res, _, _ = pl.plan_step(0, [sc0.robot], [sc0.goal], sc0.tracks, [sc0.n_tracks], wc,
                                 relax_cfg(max_sweeps=args.prep_sweeps, check_every=20000, tol=1e-38,
                                           warm_start=0, temporal_depth=args.T, rows_per_warp=args.rows,
                                           sync_every=4), bc, want_paths=False)
    prep = {"sweeps": res[0].sweeps, "residual": res[0].residual, "walk_status": res[0].walk_status,
            "n_cells": res[0].n_cells, "s": time.perf_counter() - t_prep}
    rc = relax_cfg(max_sweeps=args.sweeps, warm_start=1, temporal_depth=args.T, rows_per_warp=args.rows)
    n_ticks = args.warmup + args.steps
    scenes = [advance_scene(sc0, 1 + k) for k in range(n_ticks)]
    dev_tracks = [torch.from_numpy(np.ascontiguousarray(s.tracks)).to(dev) for s in scenes]
    pin_tracks = [torch.from_numpy(np.ascontiguousarray(s.tracks)).pin_memory() for s in scenes]
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)  # 256 MiB > L2
    cells_h = np.zeros((1, bc.max_len, 2), np.int32)

    def one(k, host):
        s = scenes[k]
        t = pin_tracks[k] if host else dev_tracks[k]
        return pl.plan_step(0, [s.robot], [s.goal], t, [s.n_tracks], wc, rc, bc, want_paths=host)

    def timed_loop(host, profile=False):
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        for k in range(args.warmup):
            one(k, host)
        if profile:
            pl.profile(1)  # per-launch CUDA events around the relaxation kernel (timed steps only)
        if ws > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize(dev)
        l0 = pl.kernel_launches()
        walk = []
        d2h = []
        torch.cuda.nvtx.range_push("timed_region_host" if host else "timed_region")
        for k in range(args.steps):
            flush.zero_()  # L2 flush between timed steps (outside the events)
            ev[k][0].record(stream)
            _, r, _, _ = one(args.warmup + k, host)
            ev[k][1].record(stream)
            walk.append(r[0].walk_status)
            # read back per step: PathMeta (32 B) + [sweeps|where|res bits|res|flags] (20 B) + the
            # produced cells (8 B each) and smoothed points (8 B each, up to max_smooth)
            d2h.append(52 + 8 * r[0].n_cells + 8 * min(r[0].n_smooth, bc.max_smooth) if host else 52)
        torch.cuda.synchronize(dev)
        torch.cuda.nvtx.range_pop()
        launches = pl.kernel_launches() - l0
        ms = sum(a.elapsed_time(b) for a, b in ev)
        if ws > 1:
            tt = torch.tensor([ms], device=dev, dtype=torch.float64)
            torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
            torch.distributed.barrier()
            ms = float(tt.item())
        timed_loop.d2h = d2h
        return ms, launches, walk

    with Clocks(local, enabled=not args.no_clocks) as clk:
        ms, launches, walk = timed_loop(host=False)
    clocks = clk.summary()
    # roofline pass: the same steps again with CUDA events around every relaxation launch (an event
    # record between two launches also stops the next launch from overlapping the previous one's
    # tail, so this pass is kept out of `value`)
    ms_prof, _, _ = timed_loop(host=False, profile=True)
    rms, rl, rcells = pl.profile_read()
    pl.profile(0)
    ms_e2e, _, _ = timed_loop(host=True)
    d2h_e2e = int(round(sum(timed_loop.d2h) / max(len(timed_loop.d2h), 1)))

    # kernel-only relaxation throughput (S = relax_sweeps), same field
    rc_big = relax_cfg(max_sweeps=args.relax_sweeps, warm_start=1, temporal_depth=args.T, rows_per_warp=args.rows)
    pl.relax(rc_big, want_result=False)
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    flush.zero_()
    e0.record(stream)
    pl.relax(rc_big, want_result=False)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    relax_ms = e0.elapsed_time(e1)

    cells = N * N
    units = cells * args.sweeps * args.steps * ws
    value = units / (ms * 1e-3) / 1e9
    e2e = units / (ms_e2e * 1e-3) / 1e9
    peak, peak_src = _peaks()
    avg_launch_s = (rms / rl) * 1e-3 if rl else float("nan")
    T_eff = rcells / rl / cells if rl else 0
    bytes_per_launch = 8.0 * cells  # one fp32 read + one fp32 write per cell per launch
    achieved = bytes_per_launch / avg_launch_s / 1e9
    # dram__bytes_read.sum + dram__bytes_write.sum of one T = 6 launch at 4096^2: not measured in this run
    # (ncu replays kernels), read from the newest committed `ncu --set full` capture and labelled so
    traffic, traffic_src = None, None
    caps = sorted(f for f in os.listdir(os.path.join(ROOT, "profiles")) if f.endswith("_relax_traffic.json"))
    if caps and N == 4096:
        traffic = json.load(open(os.path.join(ROOT, "profiles", caps[-1]))).get("traffic_bytes_per_launch")
        traffic_src = f"committed ncu capture profiles/{caps[-1]} (not measured in this run)"
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"c3_{N}: {N}x{N} grid, {sc0.n_tracks} moving obstacles (Kalman tracks), warm "
                               f"plan step = stamp + {args.sweeps} red-black sweeps + walk + {args.band_iters} "
                               f"rubber-band iterations", "sweeps": args.sweeps, "band_iters": args.band_iters,
                   "temporal_depth": args.T or 6, "l2": "flushed (256 MiB write) between timed steps",
                   "per_rank": "independent scenario (seed = rank)"},
        "plan_steps_per_s": args.steps * ws / (ms * 1e-3),
        "relax_glups": cells * args.relax_sweeps / (relax_ms * 1e-3) / 1e9,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "traffic_source": traffic_src, "kernel": "k_rb_tblock",
                     "bytes_per_launch": bytes_per_launch,
                     "relax_glups_pct_of_8B_roofline": 100.0 * (cells * args.relax_sweeps / (relax_ms * 1e-3) / 1e9) /
                                                       (peak / 8.0),
                     "sweeps_per_launch": T_eff, "avg_launch_us": avg_launch_s * 1e6, "peak_source": peak_src,
                     "launches_per_step": rl / args.steps if rl else None,
                     "kernel_share_of_step": (rms / ms_prof) if ms_prof else None,
                     "events": "per-launch CUDA events on the library stream, profiled pass of the same steps",
                     "effective_glups_vs_8B_per_LUP": (rcells / (rms * 1e-3) / 1e9) / (peak / 8.0) if rms else None},
        "e2e": {"value": e2e, "unit": UNIT, "h2d_bytes_per_step": int(sc0.n_tracks * 160 + 480),  # tracks + parameter and control blocks
                "d2h_bytes_per_step": d2h_e2e, "ms_per_step": ms_e2e / args.steps},
        "gpu_launches": int(launches),
        "walk_ok_steps": int(sum(1 for w in walk if w == 0)),
        "prep": prep,
        "clocks": clocks,
    }
    if not args.no_sub:
        # the two configurations that shard, measured in the same job at the same N so
        # that the driver's 1/2/4/8 runs carry their scaling too
        def sub(name, fn):  # a failing sub-result is reported in the line, it does not lose the C3 line
            pending[0] = name
            try:
                out[name] = fn()
            except Exception as e:  # noqa: BLE001
                out[name] = {"error": f"{type(e).__name__}: {e}"[:300]}

        # watchdog: a sub-result that does not finish (e.g. a collective that never completes on some
        # multi-GPU topology) must not cost the C3 line -- after SUB_LIMIT_S every rank stops, rank 0
        # first printing the line with the pending sub-result marked
        import threading
        pending = [None]

        def _expired():
            if rank == 0:
                out[pending[0] or "sub"] = {"error": f"did not finish within {SUB_LIMIT_S} s"}
                print(json.dumps(out), flush=True)
            os._exit(0)

        dog = threading.Timer(SUB_LIMIT_S, _expired)
        dog.daemon = True
        dog.start()
        sub("c4_slab", lambda: c4_slab(args, dev, ws, rank, local))
        sub("c5_batch", lambda: c5_batch(args, dev, ws, rank, local))
        if rank == 0:  # single-GPU configurations (BASELINE configs[0], [1])
            sub("c1_solve", lambda: c1_solve(args, dev, not args.no_cpu_baseline))
            sub("c2_loop", lambda: c2_loop(args, dev, not args.no_cpu_baseline))
        dog.cancel()
    if rank == 0 and not args.no_cpu_baseline:
        import oracle
        oracle.build()
        cores = oracle.host_cores()
        g, t = _oracle_sample(args, args.sweeps, 3, threads=cores)
        g1, t1 = _oracle_sample(args, args.sweeps, 1, threads=1)
        out["cpu_baseline"] = {"value": g, "unit": UNIT, "cores": cores, "kind": "oracle",
                               "sample": f"3 oracle plan steps of c3 seed 0 (cold, then warm; S={args.sweeps}, "
                                         f"I={args.band_iters}), {t:.1f} s, OpenMP variants on {cores} host cores "
                                         f"(bit-identical to the single-thread oracle, P14)",
                               "single_thread": {"value": g1, "cores": 1, "sample": f"1 plan step, {t1:.1f} s"}}
    if rank == 0:
        print(json.dumps(out), flush=True)
    pl.close()
    if ws > 1:
        torch.distributed.destroy_process_group()


# ---------------------------------------------------------------------------- C1, C2 sub-results
def c1_solve(args, dev, with_oracle):
    """BASELINE configs[0]: 64^2, one static disk, cold relaxation to residual 1e-6 (check every sweep)
    and path extraction: time to tolerance on the GPU (CUDA events) and for the oracle (one core)."""
    import torch
    from paper_1903_07441_b200 import Planner, band_cfg, relax_cfg, warp_cfg
    from scenes import scene_c1
    sc = scene_c1()
    stream = torch.cuda.current_stream(dev)
    pl = Planner(sc.W, sc.H, 1, sc.cell_size, sc.origin, device=dev.index, stream=stream.cuda_stream)
    pl.set_static(sc.static)
    rc = relax_cfg(max_sweeps=10 ** 6, check_every=1, tol=1e-6, warm_start=0)
    bc = band_cfg(50, 1000, 4000)
    best, sweeps = 1e9, None
    for _ in range(3):
        pl.set_obstacles(0, sc.robot, sc.goal, sc.tracks, warp_cfg(), warm=0)
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        sw, _ = pl.relax(rc)
        pl.extract_path(0, bc)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        best, sweeps = min(best, e0.elapsed_time(e1)), int(sw[0])
    pl.close()
    out = {"workload": "c1_64: cold relax to residual 1e-6 (check every sweep) + walk + 50 band iterations",
           "sweeps": sweeps, "gpu_ms": best}
    if with_oracle:
        import oracle
        t0 = time.perf_counter()
        ref = oracle.plan_step(sc, max_sweeps=10 ** 6, check_every=1, tol=1e-6, iters=50, max_len=1000)
        out.update(oracle_ms=1e3 * (time.perf_counter() - t0), oracle_cores=1, oracle_sweeps=ref["sweeps"])
    return out


def c2_loop(args, dev, with_oracle):
    """BASELINE configs[1]: 512^2, 20 obstacles, the warm plan loop (S = 100, I = 50) after a tick-0
    solve to the exact fp32 fixed point: plan steps/s on the GPU (device-resident tracks, CUDA events)
    and for the oracle (its OpenMP variants on every host core)."""
    import torch
    from paper_1903_07441_b200 import Planner, band_cfg, relax_cfg, warp_cfg
    from scenes import advance_scene, scene_c2
    sc0 = scene_c2(0)
    stream = torch.cuda.current_stream(dev)
    pl = Planner(sc0.W, sc0.H, 1, sc0.cell_size, sc0.origin, device=dev.index, stream=stream.cuda_stream)
    pl.set_static(sc0.static)
    wc, bc = warp_cfg(), band_cfg(args.band_iters, 4096, 8192)
    pl.plan_step(0, [sc0.robot], [sc0.goal], sc0.tracks, [sc0.n_tracks], wc,
                 relax_cfg(max_sweeps=400000, check_every=1000, tol=1e-38, warm_start=0, sync_every=8), bc,
                 want_paths=False)
    n = args.warmup + args.steps
    scs = [advance_scene(sc0, 1 + k) for k in range(n)]
    dtr = [torch.from_numpy(np.ascontiguousarray(s.tracks)).to(dev) for s in scs]
    rc = relax_cfg(max_sweeps=args.sweeps, warm_start=1)
    for k in range(args.warmup):
        pl.plan_step(0, [scs[k].robot], [scs[k].goal], dtr[k], [scs[k].n_tracks], wc, rc, bc, want_paths=False)
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ok = 0
    e0.record(stream)
    for k in range(args.warmup, n):
        _, r, _, _ = pl.plan_step(0, [scs[k].robot], [scs[k].goal], dtr[k], [scs[k].n_tracks], wc, rc, bc,
                                  want_paths=False)
        ok += int(r[0].walk_status == 0)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    ms = e0.elapsed_time(e1)
    pl.close()
    out = {"workload": f"c2_512: warm plan step S={args.sweeps}, I={args.band_iters}, 20 obstacles, after a tick-0 "
                       f"solve to the fp32 fixed point", "plan_steps_per_s": args.steps / (ms * 1e-3),
           "glups": 512 * 512 * args.sweeps * args.steps / (ms * 1e-3) / 1e9, "walk_ok_steps": ok,
           "steps": args.steps}
    if with_oracle:
        import oracle
        cores = oracle.host_cores()
        r0 = oracle.plan_step(sc0, max_sweeps=400000, check_every=1000, tol=1e-38, iters=args.band_iters,
                              max_len=4096, threads=cores)
        t0, prev = time.perf_counter(), r0
        for k in range(2):
            prev = oracle.plan_step(scs[k], max_sweeps=args.sweeps, iters=args.band_iters, max_len=4096, prev=prev,
                                    threads=cores)
        out.update(oracle_plan_steps_per_s=2 / (time.perf_counter() - t0), oracle_cores=cores)
    return out


# ---------------------------------------------------------------------------- C4: row slabs
def c4_slab(args, dev, ws, rank, local):
    """16384^2 relaxation, rows split over the ranks as libtwg sharded contexts (twg_create with an
    NCCL communicator): inside twg_relax the library exchanges the 2k ghost rows every k sweeps
    (ncclSend/ncclRecv on a high-priority stream, overlapped with the interior tiles) and
    max-all-reduces the residual on the device.  Strong scaling.  Returns the sub-result dict."""
    import torch
    from paper_1903_07441_b200 import relax_cfg, warp_cfg
    from paper_1903_07441_b200.slab import make_sharded, nccl_comm_for
    from paper_1903_07441_b200.twg import nccl_comm_destroy
    from scenes import scene_c4
    sc = scene_c4(0)
    stream = torch.cuda.current_stream(dev)
    comm = nccl_comm_for(rank, ws, local)
    pl = make_sharded(sc.W, sc.H, sc.static, sc.robot, sc.goal, sc.tracks, warp_cfg(), args.k, comm, device=local,
                      stream=stream.cuda_stream)
    S = args.relax_sweeps
    rc = relax_cfg(max_sweeps=S, temporal_depth=args.T, rows_per_warp=args.rows)
    for _ in range(args.warmup):
        pl.relax(rc, want_result=False)
    if ws > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0 = pl.kernel_launches()
    e0.record(stream)
    for _ in range(args.steps):
        pl.relax(rc, want_result=False)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    ms_tot = e0.elapsed_time(e1)
    launches = pl.kernel_launches() - l0
    _, res = pl.relax(relax_cfg(max_sweeps=args.k), want_result=True)
    if ws > 1:
        t = torch.tensor([ms_tot], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms_tot = float(t.item())
    out = {"metric": "harmonic relaxation GLUP/s at 16384^2 (row slabs)", "unit": "GLUP/s",
           "value": sc.W * sc.H * S * args.steps / (ms_tot * 1e-3) / 1e9, "scaling": "strong", "n_gpus": ws,
           "ms_per_step": ms_tot / args.steps, "steps": args.steps,
           "config": {"workload": f"c4_16384: {sc.W}x{sc.H} grid, {sc.n_tracks} obstacles, relax {S} red-black "
                                  f"sweeps per step, ghost exchange every k={args.k} sweeps inside twg_relax "
                                  f"(NCCL send/recv; residual all-reduce)",
                      "k": args.k, "ghost_rows": pl.ghost_rows, "rows_per_rank": pl.r1 - pl.r0,
                      "l2": "not flushed: the 16384^2 field (1 GiB, 2 GiB ping-pong) exceeds L2"},
           "gpu_launches": int(launches), "residual_after": float(res[0])}
    pl.close()
    nccl_comm_destroy(comm)
    if rank == 0 and not args.no_cpu_baseline:  # the oracle at S = 8 (every host core)
        import oracle
        _, cls, *_ = oracle.classify(sc)
        u = oracle.init_u32(cls)
        cores = oracle.host_cores()
        t0 = time.perf_counter()
        oracle.relax_f32(cls, u, 8, 8, 0.0, threads=cores)
        dt = time.perf_counter() - t0
        out["cpu_baseline"] = {"value": sc.W * sc.H * 8 / dt / 1e9, "unit": "GLUP/s", "cores": cores, "kind": "oracle",
                               "sample": f"8 red-black sweeps of the whole 16384^2 grid, {dt:.2f} s"}
    return out


def run_c4(args):
    import torch
    ws, rank, local = _dist()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    from paper_1903_07441_b200 import lib
    lib()
    with Clocks(local, enabled=not args.no_clocks) as clk:
        out = c4_slab(args, dev, ws, rank, local)
    if rank == 0:
        out.update({"warmup": args.warmup, "higher_is_better": True, "vs_baseline": None, "dtype": "f32",
                    "data": "synthetic", "clocks": clk.summary()})
        print(json.dumps(out), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()


# ---------------------------------------------------------------------------- C5: batch
def c5_batch(args, dev, ws, rank, local):
    """1024 independent 512^2 scenarios, 1024/N per rank in one batched context (weak in the
    scenarios per rank).  A step = twg_plan_step(b = -1) with S = 100 warm sweeps.  Returns the
    sub-result dict."""
    import torch
    from paper_1903_07441_b200 import Planner, band_cfg, relax_cfg, warp_cfg
    from scenes import scene_random, advance_scene
    per = args.batch // ws
    scs = [scene_random(f"c5_s{s}", 512, 8, 20, s) for s in range(rank * per, (rank + 1) * per)]
    stream = torch.cuda.current_stream(dev)
    pl = Planner(512, 512, per, 0.1, (0.0, 0.0), device=local, stream=stream.cuda_stream)
    for b, sc in enumerate(scs):
        pl.set_static(sc.static, b)
    wc, bc = warp_cfg(), band_cfg(args.band_iters, 4096, 8192)
    ticks = {}

    def inputs(tick):  # scene advance and packing are input generation: done before the timed region
        if tick not in ticks:
            ss = [advance_scene(sc, tick) for sc in scs]
            ticks[tick] = (np.array([s.robot for s in ss], np.float64), np.array([s.goal for s in ss], np.int32),
                           torch.from_numpy(np.ascontiguousarray(np.vstack([s.tracks for s in ss]))).pin_memory(),
                           np.array([s.n_tracks for s in ss], np.int32))
        return ticks[tick]

    def step(tick, rc):
        rob, goals, tr, nt = inputs(tick)
        return pl.plan_step(-1, rob, goals, tr, nt, wc, rc, bc, want_paths=False)

    for k in range(1 + args.warmup + args.steps):
        inputs(k)
    t_prep = time.perf_counter()
    # tick 0: cold solve to the fp32 fixed point; scenes whose cold field drains slowly through narrow
    # passages stop at the cap (profiles/r02_c5_nopath.json)
    step(0, relax_cfg(max_sweeps=300000, check_every=2000, tol=1e-38, warm_start=0, sync_every=4))
    prep_s = time.perf_counter() - t_prep
    rc = relax_cfg(max_sweeps=args.sweeps, warm_start=1)
    for k in range(args.warmup):
        step(1 + k, rc)
    if ws > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize(dev)
    ms_tot, ok = 0.0, 0
    status = {}
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0 = pl.kernel_launches()
    for k in range(args.steps):
        torch.cuda.nvtx.range_push("timed_region")
        e0.record(stream)
        st, res, _, _ = step(1 + args.warmup + k, rc)
        e1.record(stream)
        torch.cuda.nvtx.range_pop()
        torch.cuda.synchronize(dev)
        ms_tot += e0.elapsed_time(e1)
        ok += sum(1 for r in res if r.walk_status == 0)
        for r in res:
            status[int(r.status)] = status.get(int(r.status), 0) + 1
    launches = pl.kernel_launches() - l0
    gathered = per
    if ws > 1:
        t = torch.tensor([ms_tot], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms_tot = float(t.item())
        # the only exchange of the batch mode -- one all-gather of the per-scenario
        # result structs (status, sweeps, path cells, next waypoint) of the last step
        mine = torch.tensor([[r.walk_status, r.sweeps, r.n_cells, r.next_x, r.next_y] for r in res],
                            dtype=torch.float64, device=dev)
        allr = [torch.empty_like(mine) for _ in range(ws)]
        torch.distributed.all_gather(allr, mine)
        gathered = sum(int(a.shape[0]) for a in allr)
        okt = torch.tensor([ok], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(okt)
        ok = int(okt.item())
    out = {"metric": "harmonic relaxation GLUP/s, batch of 512^2 plan steps", "unit": "GLUP/s",
           "value": 512 * 512 * per * ws * args.sweeps * args.steps / (ms_tot * 1e-3) / 1e9, "scaling": "weak",
           "n_gpus": ws, "ms_per_step": ms_tot / args.steps, "steps": args.steps,
           "config": {"workload": f"c5: {args.batch} x 512x512 scenarios (20 obstacles each), {per} per rank, "
                                  f"warm plan step S={args.sweeps}, I={args.band_iters} (host tracks: per-step H2D "
                                  f"inside the timed region)"},
           "scenario_steps_per_s": per * ws * args.steps / (ms_tot * 1e-3),
           "walk_ok_fraction": ok / (args.steps * per * ws), "status_counts_rank0": status, "prep_s": prep_s,
           "results_gathered": gathered, "gpu_launches": int(launches)}
    pl.close()
    if rank == 0 and not args.no_cpu_baseline:  # the oracle's scenario-steps/s on a sample of the scenarios
        import oracle
        cores = oracle.host_cores()
        dt, n = 0.0, 0
        for sc in scs[:4]:  # tick 0 (untimed, 20 000 sweeps) then two timed warm steps each
            prev = oracle.plan_step(advance_scene(sc, 0), max_sweeps=20000, check_every=2000, tol=1e-38,
                                    iters=args.band_iters, max_len=4096, threads=cores)
            for k in range(2):
                t0 = time.perf_counter()
                prev = oracle.plan_step(advance_scene(sc, 1 + k), max_sweeps=args.sweeps, iters=args.band_iters,
                                        max_len=4096, prev=prev, threads=cores)
                dt += time.perf_counter() - t0
                n += 1
        out["cpu_baseline"] = {"value": n / dt, "unit": "scenario-steps/s", "cores": cores, "kind": "oracle",
                               "sample": f"{n} warm oracle plan steps of C5 scenes (S={args.sweeps}, I={args.band_iters})"}
    return out


def run_c5(args):
    import torch
    ws, rank, local = _dist()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    from paper_1903_07441_b200 import lib
    lib()
    with Clocks(local, enabled=not args.no_clocks) as clk:
        out = c5_batch(args, dev, ws, rank, local)
    if rank == 0:
        out.update({"warmup": args.warmup, "higher_is_better": True, "vs_baseline": None, "dtype": "f32",
                    "data": "synthetic", "clocks": clk.summary()})
        print(json.dumps(out), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()


def _launch_ranks(args) -> int:
    """--gpus N > 1 without a torchrun environment: start N ranks (one process per GPU) through
    torch.distributed.run on 127.0.0.1 with this very command line; rank 0 prints the JSON line."""
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


SUB_LIMIT_S = 240  # bound on the sub-results of the default line (normally well under a minute)


def _json_stdout():
    """Keep stdout for the one JSON line: native libraries write to file descriptor 1 (NCCL's version
    banner when the row-slab communicator is created), so fd 1 is pointed at stderr for the run and
    Python's stdout writes to a saved copy of the original descriptor."""
    sys.stdout.flush()
    fd = os.dup(1)
    os.dup2(2, 1)
    sys.stdout = os.fdopen(fd, "w", buffering=1)


def main():
    args = _args()
    ws_env = os.environ.get("WORLD_SIZE")
    if ws_env is None and args.gpus > 1:
        sys.exit(_launch_ranks(args))
    if ws_env is not None and int(ws_env) != args.gpus:
        print(f"bench.py: WORLD_SIZE={ws_env} but --gpus {args.gpus}; refusing to run", file=sys.stderr)
        sys.exit(2)
    if args.probe:
        ws, rank, local = _dist()
        print(json.dumps({"probe": True, "rank": rank, "world_size": ws, "local_rank": local, "pid": os.getpid()}),
              flush=True)
        return
    _json_stdout()
    if args.impl == "reference":
        run_reference(args)
    elif args.config == "c4":
        run_c4(args)
    elif args.config == "c5":
        run_c5(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
