"""Golden values for the batch-wide frontier (include/bpt.h BPT_FLAG_SLOTWISE off, the default):
the oracle's work of sorted C2 batches as ONE 256-sample fused group and as four 64-sample groups
(oracle/ + graphgen/ only; slow: ~7 min per heavy batch on 16 cores, run on the GPU box host).
  python scripts/batch_groups_oracle.py [batch ...]  -> tests/golden/c2_sorted_batch_groups_oracle.json"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import graphgen  # noqa: E402
import oracle  # noqa: E402


def main():
    args = sys.argv[1:]
    group = 256
    if args and args[0].startswith("--group="):
        group = int(args[0].split("=")[1])
        args = args[1:]
    batches = [int(x) for x in args] or [0, 40, 90]
    cfg = graphgen.CONFIGS["C2"]
    row_ptr, col, thr = graphgen.make_graph(cfg)
    og = oracle.Graph(row_ptr, col, w_q31=thr)
    n, theta, seed = cfg.n, cfg.theta, cfg.seed
    ids = np.arange(theta, dtype=np.int64)
    starts = np.array([oracle.start_vertex(int(s), n, seed) for s in ids], dtype=np.int64)
    indeg = np.bincount(col.astype(np.int64), minlength=n)
    order = ids[np.lexsort((ids, starts, -indeg[starts]))]  # reading C-19 (sorted start vertices)
    out = {"citation": "BASELINE.json configs[1] (C2), theta 65,536, sampling seed cfg.seed, sorted start "
                       "vertices (reading C-19, P:430); E_phys of batch b = distinct (v, level) pairs x in-degree "
                       "of the fused traversal of samples order[256 b, 256 b + 256) (SURVEY 8(c), P:239-241); "
                       "written by scripts/batch_groups_oracle.py from oracle/ only",
           "seed": seed, "batches": {}}
    for b in batches:
        t = time.time()
        grp = order[group * b:group * b + group].astype(np.uint64)
        w256 = og.group_work_ids(seed, grp)
        if group != 256:  # exploration of wider batches: the fused group's work and its 256-sample halves
            w4 = [og.group_work_ids(seed, grp[256 * i:256 * i + 256]) for i in range(group // 256)]
            print(b, group, int(w256["e_phys"]), [int(w["e_phys"]) for w in w4], flush=True)
            continue
        w64 = [og.group_work_ids(seed, grp[64 * i:64 * i + 64]) for i in range(4)]
        out["batches"][str(b)] = {"e_phys_256": int(w256["e_phys"]), "levels_256": int(w256["levels"]),
                                  "frontier_256": [int(x) for x in w256["frontier"]],
                                  "e_phys_4x64": [int(w["e_phys"]) for w in w64]}
        print(b, out["batches"][str(b)]["e_phys_256"], sum(out["batches"][str(b)]["e_phys_4x64"]),
              round(time.time() - t, 1), "s", flush=True)
    if group != 256:
        return
    path = os.path.join(ROOT, "tests", "golden", "c2_sorted_batch_groups_oracle.json")
    json.dump(out, open(path, "w"), indent=1)
    print(path)


if __name__ == "__main__":
    main()
