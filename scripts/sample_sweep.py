"""Timing sweep of bpt_sample on a config (GPU): batch_groups x poll_levels, prints JSON lines.
Usage: python scripts/sample_sweep.py --config C2 --theta 8192 --batches 1,2,4,8 [--profile]"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import graphgen  # noqa: E402
import paper_2311_10201_b200 as bpt  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C2")
ap.add_argument("--theta", type=int, default=0)
ap.add_argument("--colors", default="64")
ap.add_argument("--batches", default="1,2,4,8")
ap.add_argument("--polls", default="0")
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--profile", action="store_true")
ap.add_argument("--select", type=int, default=0)
ap.add_argument("--levels", action="store_true", help="print per-level rows (batch, level, raw, kept, work, vc, coins, atomics)")
ap.add_argument("--flags", default="0", help="comma list of bpt_sample_opts.flags values to sweep (e.g. 0,128)")
a = ap.parse_args()
cfg = graphgen.CONFIGS[a.config]
theta = a.theta or cfg.theta
torch.cuda.set_device(0)
t0 = time.time()
row_ptr, col, thr = graphgen.make_graph(cfg)
print(json.dumps({"gen_s": time.time() - t0}), flush=True)
g = bpt.Graph(row_ptr, col, w_q31=thr, model=bpt.IC if cfg.model == "IC" else bpt.LT)
for F in [int(x, 0) for x in a.flags.split(",")]:
  for C in [int(x) for x in a.colors.split(",")]:
    for B in [int(x) for x in a.batches.split(",")]:
        for P in [int(x) for x in a.polls.split(",")]:
            for r in range(a.reps):
                torch.cuda.synchronize()
                t = time.perf_counter()
                s = g.sample(theta, colors=C, seed=cfg.seed, batch_groups=B, poll_levels=P, profile=a.profile, flags=F)
                dt = time.perf_counter() - t
                info = s.info
                out = {"flags": F, "C": C, "B": B, "P": P, "rep": r, "theta": theta, "s": dt, "sets_per_s": theta / dt,
                       "ms_expand": info["ms_expand"], "e_phys": info["e_phys"], "e_logical": info["e_logical"],
                       "coins": info["coins"], "atomics": info["atomics"], "levels_total": info["levels_total"],
                       "launches": info["kernel_launches"], "expand_GBps": (info["expand_bytes"] / info["ms_expand"] / 1e6) if info["ms_expand"] else None}
                if a.levels:
                    out["levels"] = s.level_stats().tolist()
                if a.select:
                    t = time.perf_counter()
                    s.select_seeds(a.select)
                    out["select_s"] = time.perf_counter() - t
                print(json.dumps(out), flush=True)
                s.close()
