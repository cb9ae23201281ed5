"""Debug: first level where the pull form's level structure departs from the push form's."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import graphgen, oracle  # noqa
import paper_2311_10201_b200 as bpt  # noqa
import torch
torch.cuda.set_device(0)
for name, scale, theta, bg in (("C1", 0, 1024, 1), ("C1", 0, 1024, 0), ("C2", 1 << 12, 256, 1), ("C2", 1 << 15, 2048, 0)):
    cfg = graphgen.CONFIGS[name] if not scale else graphgen.scaled(graphgen.CONFIGS[name], scale, theta=theta)
    row_ptr, col, thr = graphgen.make_graph(cfg)
    g = bpt.Graph(row_ptr, col, w_q31=thr)
    for flags in (0, bpt.FLAG_UNSORTED):
        push = g.sample(theta, seed=cfg.seed, batch_groups=bg, flags=flags)
        pull = g.sample(theta, seed=cfg.seed, batch_groups=bg, flags=flags, pull=True, pull_permille=1)
        a, b = push.level_stats(), pull.level_stats()
        same_sizes = np.array_equal(push.sizes(0, theta), pull.sizes(0, theta))
        print(name, scale, theta, "bg", bg, "flags", flags, "rows", len(a), len(b), "sizes equal", same_sizes,
              "pull levels", pull.info["pull_levels"])
        n = min(len(a), len(b))
        for i in range(n):
            if not np.array_equal(a[i, :6], b[i, :6]):
                print("  first diff row", i, "push", a[i].tolist(), "pull", b[i].tolist())
                if i: print("  prev push", a[i-1].tolist(), "pull", b[i-1].tolist())
                break
        push.close(); pull.close()
