"""Load one BASELINE config's graph `--reps` times (diagnostic for ncu launch lists of A0/A1)."""
import argparse
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import graphgen  # noqa: E402
import paper_2311_10201_b200 as bpt  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C3")
ap.add_argument("--reps", type=int, default=3)
args = ap.parse_args()
cfg = graphgen.CONFIGS[args.config]
row_ptr, col, thr = graphgen.make_graph(cfg)
dev = torch.device("cuda:0")
d_row = torch.from_numpy(row_ptr.view(np.int64).copy()).to(dev)
d_col = torch.from_numpy(col.view(np.int32).copy()).to(dev)
d_thr = torch.from_numpy(thr.view(np.int32).copy()).to(dev)
model = bpt.LT if cfg.model == "LT" else bpt.IC
for r in range(args.reps):
    torch.cuda.synchronize()
    t = time.perf_counter()
    g = bpt.Graph(d_row, d_col, w_q31=d_thr, model=model, n=cfg.n, m=cfg.m)
    torch.cuda.synchronize()
    print(f"graph_load {args.config}: {(time.perf_counter() - t) * 1e3:.3f} ms", flush=True)
    g.close()
