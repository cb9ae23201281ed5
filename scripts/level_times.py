"""Where the expansion time of one C2 sampling call goes (diagnostic only, not a bench number):
per (batch, level) row the edge reads, coins, entries and the CUDA-event time of its expansion
launch (BPT_FLAG_PROFILE, bpt_level_times), aggregated by the level's frontier work relative to
m. Decides where a different formulation of the heavy levels could pay.
python scripts/level_times.py [--config C2] [--theta 65536] [--out rows.npz]"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import graphgen  # noqa: E402
import paper_2311_10201_b200 as bpt  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--theta", type=int, default=0)
    ap.add_argument("--out", default="")
    ap.add_argument("--flags", type=int, default=0)
    ap.add_argument("--print-rows", action="store_true")
    args = ap.parse_args()
    cfg = graphgen.CONFIGS[args.config]
    theta = args.theta or cfg.theta
    row_ptr, col, thr = graphgen.make_graph(cfg)
    dev = torch.device("cuda:0")
    d_row = torch.from_numpy(row_ptr.view(np.int64).copy()).to(dev)
    d_col = torch.from_numpy(col.view(np.int32).copy()).to(dev)
    d_thr = torch.from_numpy(thr.view(np.int32).copy()).to(dev)
    stream = torch.cuda.current_stream()
    g = bpt.Graph(d_row, d_col, w_q31=d_thr, model=bpt.IC, n=cfg.n, m=cfg.m, stream=stream)
    s = g.sample(theta, colors=cfg.colors, seed=cfg.seed, stream=stream, profile=True, flags=args.flags)
    torch.cuda.synchronize()
    st = s.level_stats().astype(np.int64)
    ms = s.level_times().astype(np.float64)
    info = s.info
    s.close()
    batch, level, raw, kept, work, vc, coins, atoms = st.T
    out = {"config": args.config, "theta": theta, "rows": int(len(st)), "ms_expand": float(ms.sum()),
           "edges": int(work.sum()), "coins": int(coins.sum()), "info_ms_expand": info["ms_expand"]}
    frac = work / cfg.m  # frontier work of the level relative to m (4 slots per batch)
    bins = [0, 0.001, 0.01, 0.05, 0.2, 0.5, 1.0, 2.0, 100.0]
    tab = []
    for lo, hi in zip(bins[:-1], bins[1:]):
        sel = (frac >= lo) & (frac < hi)
        if not sel.any():
            continue
        tab.append({"work_over_m": [lo, hi], "levels": int(sel.sum()), "ms": round(float(ms[sel].sum()), 2),
                    "edges": int(work[sel].sum()), "coins": int(coins[sel].sum()),
                    "coins_per_edge": round(float(coins[sel].sum() / max(1, work[sel].sum())), 3),
                    "gedges_per_s": round(float(work[sel].sum() / max(1e-9, ms[sel].sum()) / 1e6), 1),
                    "entries": int(kept[sel].sum())})
    out["by_work_over_m"] = tab
    byb = []
    for b in np.unique(batch)[:: max(1, len(np.unique(batch)) // 16)]:
        sel = batch == b
        byb.append([int(b), int(sel.sum()), round(float(ms[sel].sum()), 3), int(work[sel].sum()), int(coins[sel].sum())])
    out["by_batch_sampled_[batch,levels,ms,edges,coins]"] = byb
    print(json.dumps(out))
    if args.print_rows:
        for r, t in zip(st.tolist(), ms.tolist()):
            print(json.dumps({"row": r, "ms": t}))
    if args.out:
        np.savez_compressed(args.out, stats=st, ms=ms)


if __name__ == "__main__":
    main()
