"""One C3 (LT) sampling call on cuda:0, printing its info as JSON: the driver for the ncu
capture of k_walk_lt_sparse (profiles/r01_walk_lt_ncu_full.md, walk_lt_traffic.json).
Diagnostic only.  python scripts/lt_walk_once.py [--config C3]"""
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
    ap.add_argument("--config", default="C3")
    ap.add_argument("--reps", type=int, default=1)
    args = ap.parse_args()
    cfg = graphgen.CONFIGS[args.config]
    row_ptr, col, thr = graphgen.make_graph(cfg)
    dev = torch.device("cuda:0")
    d_row = torch.from_numpy(row_ptr.view(np.int64).copy()).to(dev)
    d_col = torch.from_numpy(col.view(np.int32).copy()).to(dev)
    d_thr = torch.from_numpy(thr.view(np.int32).copy()).to(dev)
    stream = torch.cuda.current_stream()
    g = bpt.Graph(d_row, d_col, w_q31=d_thr, model=bpt.LT, n=cfg.n, m=cfg.m, stream=stream)
    keep = ("members", "e_phys", "ms_expand", "expand_bytes", "expand_launches", "store_bytes")
    for _ in range(args.reps):
        s = g.sample(cfg.theta, colors=cfg.colors, seed=cfg.seed, stream=stream)
        torch.cuda.synchronize()
        print(json.dumps({k: s.info[k] for k in keep}))
        s.close()


if __name__ == "__main__":
    main()
