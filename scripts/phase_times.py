"""Wall time of each phase of one bench step (graph_load, sample, extract, select_seeds) on
cuda:0 for one BASELINE config, each phase bracketed by stream synchronisation.
Diagnostic only (not a bench number): python scripts/phase_times.py --config C3 --reps 5"""
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
    ap.add_argument("--config", default="C3")
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    cfg = graphgen.CONFIGS[args.config]
    row_ptr, col, thr = graphgen.make_graph(cfg)
    dev = torch.device("cuda:0")
    d_row = torch.from_numpy(row_ptr.view(np.int64).copy()).to(dev)
    d_col = torch.from_numpy(col.view(np.int32).copy()).to(dev)
    d_thr = torch.from_numpy(thr.view(np.int32).copy()).to(dev)
    model = bpt.LT if cfg.model == "LT" else bpt.IC
    stream = torch.cuda.current_stream()
    rows = []
    for r in range(args.reps):
        t = [time.perf_counter()]
        g = bpt.Graph(d_row, d_col, w_q31=d_thr, model=model, n=cfg.n, m=cfg.m, stream=stream)
        torch.cuda.synchronize(); t.append(time.perf_counter())
        s = g.sample(cfg.theta, colors=cfg.colors, seed=cfg.seed + r % 3, stream=stream)
        torch.cuda.synchronize(); t.append(time.perf_counter())
        cnt = min(64, s.s1 - s.s0)
        sz = int(s.sizes(0, cnt).astype(np.uint64).sum())
        off = torch.empty(cnt + 1, dtype=torch.int64, device=dev)
        mem = torch.empty(max(sz, 1), dtype=torch.int32, device=dev)
        s.extract(0, cnt, offsets=off, members=mem, capacity=sz)
        torch.cuda.synchronize(); t.append(time.perf_counter())
        s.select_seeds(cfg.k)
        torch.cuda.synchronize(); t.append(time.perf_counter())
        s.close(); g.close()
        torch.cuda.synchronize(); t.append(time.perf_counter())
        rows.append(np.diff(t) * 1e3)
    med = np.median(np.array(rows), axis=0)
    print(json.dumps({"config": args.config, "ms_median": dict(zip(
        ["graph_load", "sample", "extract", "select", "close"], [round(float(x), 3) for x in med]))}))


if __name__ == "__main__":
    main()
