"""Per-level shape of the fused IC traversal on one BASELINE config (diagnostic only, not a
bench number): how many levels of how much work a batch runs, so the fixed per-level cost
(compaction + expansion launch) can be weighed against the work it carries.
python scripts/level_profile.py --config C2 --theta 8192"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import graphgen  # noqa: E402
import paper_2311_10201_b200 as bpt  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--theta", type=int, default=8192)
    args = ap.parse_args()
    cfg = graphgen.CONFIGS[args.config]
    row_ptr, col, thr = graphgen.make_graph(cfg)
    dev = torch.device("cuda:0")
    d_row = torch.from_numpy(row_ptr.view(np.int64).copy()).to(dev)
    d_col = torch.from_numpy(col.view(np.int32).copy()).to(dev)
    d_thr = torch.from_numpy(thr.view(np.int32).copy()).to(dev)
    model = bpt.LT if cfg.model == "LT" else bpt.IC
    stream = torch.cuda.current_stream()
    g = bpt.Graph(d_row, d_col, w_q31=d_thr, model=model, n=cfg.n, m=cfg.m, stream=stream)
    out = {"config": args.config, "theta": args.theta}
    for mode in ("graph", "graph", "profile"):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        s = g.sample(args.theta, colors=cfg.colors, seed=cfg.seed, stream=stream, profile=(mode == "profile"))
        torch.cuda.synchronize()
        out[f"ms_{mode}"] = (time.perf_counter() - t0) * 1e3
        info = s.info
        out[f"ms_expand_{mode}"] = info["ms_expand"]
        st = s.level_stats()
        s.close()
    st = np.asarray(st, dtype=np.int64).reshape(-1, 8)
    work = st[:, 4]
    raw = st[:, 2]
    out["levels"] = int(len(st))
    out["levels_per_batch"] = float(len(st) / max(1, len(np.unique(st[:, 0]))))
    out["edges_total"] = int(work.sum())
    for lim in (1_000, 10_000, 30_000, 100_000, 300_000, 1_000_000):
        sel = work <= lim
        out[f"levels_work_le_{lim}"] = int(sel.sum())
        out[f"share_work_le_{lim}"] = float(work[sel].sum() / max(1, work.sum()))
    by_level = {}
    for lv in np.unique(st[:, 1]):
        sel = st[:, 1] == lv
        by_level[int(lv)] = [int(sel.sum()), float(work[sel].mean()), float(raw[sel].mean())]
    out["by_level_count_meanwork_meanraw"] = by_level
    print(json.dumps(out))


if __name__ == "__main__":
    main()
