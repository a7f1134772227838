"""Desk-scale analogue of the paper's Table 1 / Table 2 / turning-angle histograms (row f2):
trials per obstacle count on 25.6 m x 25.6 m maps, all trials of all counts in one
batched GPU run.  Writes JSON (stdout and --out)."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1903_07441_b200 import relax_cfg, sim_cfg  # noqa: E402
from paper_1903_07441_b200 import sim as S  # noqa: E402
from scenes import scene_sim  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--trials", type=int, default=40)
    ap.add_argument("--counts", default="1,2,4,8,12,16")
    ap.add_argument("--sweeps", type=int, default=1000)
    ap.add_argument("--max-ticks", type=int, default=1500)
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    counts = [int(c) for c in a.counts.split(",")]
    scs = [scene_sim(1000 * n + k, n) for n in counts for k in range(a.trials)]
    st = torch.cuda.current_stream()
    t0 = time.time()
    res, ticks = S.run_batch(scs, cfg=sim_cfg(seed=7, max_ticks=a.max_ticks),
                             rcfg=relax_cfg(max_sweeps=a.sweeps, warm_start=1), stream=st.cuda_stream)
    torch.cuda.synchronize()
    wall = time.time() - t0
    out = {"trials_per_count": a.trials, "sweeps_per_tick": a.sweeps, "max_ticks": a.max_ticks,
           "batch": len(scs), "ticks_run": ticks, "wall_s": wall,
           "trial_ticks_per_s": sum(r["ticks"] for r in res) / wall, "rows": {}}
    for n in counts:
        out["rows"][str(n)] = S.summarize([r for r in res if r["obstacles"] == n])
    print(json.dumps({k: v for k, v in out.items() if k != "rows"}))
    for n in counts:
        r = out["rows"][str(n)]
        print(n, "success %.1f%% collision %.1f%% timeout %.1f%% length/straight %s turns<15deg %.1f%%" % (
            r["success_pct"], r["collision_pct"], r["timeout_pct"], r["mean_length_over_straight"],
            r["turns_below_15deg_pct"]))
    if a.out:
        with open(a.out, "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
