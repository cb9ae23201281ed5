"""One full-size BASELINE config on one GPU: time bpt_sample / bpt_select_seeds and check a
sampled subset of RRR sets (size, digest, list) against the CPU oracle. Prints one JSON line.

  python scripts/config_run.py --config C3 [--theta N] [--colors C] [--check 256] [--reps 2]
"""
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
import oracle  # noqa: E402
import paper_2311_10201_b200 as bpt  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C3")
ap.add_argument("--theta", type=int, default=0)
ap.add_argument("--colors", type=int, default=0)
ap.add_argument("--check", type=int, default=256, help="samples checked against the oracle")
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--k", type=int, default=0)
ap.add_argument("--sparse", action="store_true", help="LT: sorted member lists instead of the dense store")
ap.add_argument("--wide", action="store_true", help="IC: 128 colours per frontier entry")
a = ap.parse_args()
cfg = graphgen.CONFIGS[a.config]
theta = a.theta or cfg.theta
colors = a.colors or cfg.colors
k = a.k or cfg.k
torch.cuda.set_device(0)
t = time.time()
row_ptr, col, thr = graphgen.make_graph(cfg)
gen_s = time.time() - t
model = bpt.IC if cfg.model == "IC" else bpt.LT
g = bpt.Graph(row_ptr, col, w_q31=thr, model=model)
times, sel_times = [], []
s = None
for r in range(a.reps):
    if s is not None:
        s.close()
    torch.cuda.synchronize()
    t = time.perf_counter()
    s = g.sample(theta, colors=colors, seed=cfg.seed, sparse=a.sparse, wide=a.wide)
    times.append(time.perf_counter() - t)
    t = time.perf_counter()
    seeds, gains, sigma = s.select_seeds(k)
    sel_times.append(time.perf_counter() - t)
info = s.info
# sampled parity: strided ids + the first and last 64-sample blocks
ids = np.unique(np.concatenate([np.linspace(0, theta - 1, a.check).astype(np.int64),
                                np.arange(min(64, theta)), np.arange(max(0, theta - 64), theta)])).astype(np.uint64)
og = oracle.Graph(row_ptr, col, w_q31=thr, model=oracle.IC if cfg.model == "IC" else oracle.LT)
t = time.time()
o_sizes, o_dig, _, o_off, o_mem = og.sample_many(cfg.seed, ids, members=True)
oracle_s = time.time() - t
sizes = s.sizes(0, theta)
dig = s.digests(0, theta)
ok_sizes = bool(np.array_equal(sizes[ids.astype(np.int64)], o_sizes))
ok_dig = bool(np.array_equal(dig[ids.astype(np.int64)], o_dig))
ok_lists = True
for j in range(0, len(ids), max(1, len(ids) // 16)):
    off, mem = s.extract(int(ids[j]), 1)
    ok_lists &= bool(np.array_equal(mem, o_mem[o_off[j]:o_off[j + 1]]))
best = min(times)
print(json.dumps({
    "config": cfg.name, "theta": theta, "colors": colors, "model": cfg.model, "n": cfg.n, "m": cfg.m,
    "mode": "sparse lists" if a.sparse else ("wide fusion" if a.wide else "default"),
    "gen_s": gen_s, "sample_s": times, "select_s": sel_times, "rrr_sets_per_s": theta / best,
    "e_phys": info["e_phys"], "e_logical": info["e_logical"], "members": info["members"],
    "edges_per_s": info["e_phys"] / best, "levels_total": info["levels_total"], "levels_max": info["levels_max"],
    "batch_groups": info["batch_groups"], "ms_expand": info["ms_expand"], "store_gb": info["store_bytes"] / 1e9,
    "seeds_head": seeds[:8].tolist(), "gains_head": gains[:8].tolist(), "sigma_hat": sigma,
    "parity_checked_samples": int(len(ids)), "parity_sizes": ok_sizes, "parity_digests": ok_dig,
    "parity_lists": ok_lists, "oracle_s": oracle_s, "invariants": {
        "members_eq_sum_sizes": int(info["members"]) == int(sizes.astype(np.uint64).sum()),
        "gains_nonincreasing": bool(np.all(np.diff(gains.astype(np.int64)) <= 0)),
        "sigma_formula": sigma == cfg.n * int(gains.sum()) / theta}}), flush=True)
