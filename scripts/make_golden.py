"""Expected values of the full-size parity tests, written by the CPU ORACLE ONLY (oracle/ +
graphgen/; nothing here touches the CUDA path). Test infrastructure: the GPU tests compare the
C-ABI results on the same seeded inputs against these files.

  python scripts/make_golden.py C2   -> tests/golden/c2_full_oracle.npz
      all 65,536 samples of BASELINE configs[1] (sizes, digests), the E_phys / level count /
      per-level frontier sizes of every 64-sample traversal group, E_logical, greedy seeds and
      gains for k = 50 at theta = 65,536 and at theta = 2,048 (the first 32 groups), sigma_hat.
      ~40 min on 8 cores, ~20 GB (SURVEY §8(c) oracle step 3 store: lists / bitsets).
  python scripts/make_golden.py C2S  -> tests/golden/c2_sorted_oracle.npz
      per-group E_phys / levels / frontier sizes of the C2 step under sorted start vertices.
  python scripts/make_golden.py C4   -> tests/golden/c4_shard7_oracle.npz
      64 sample ids of the last of 8 rank shards of configs[3] (theta = 131,072), spread over the
      shard and over all 64 colour slots: sizes, digests, and the member lists of two of them.
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import graphgen  # noqa: E402
import oracle  # noqa: E402

GOLD = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "tests", "golden")  # optional output dir


def c2():
    cfg = graphgen.CONFIGS["C2"]
    t0 = time.time()
    row_ptr, col, thr = graphgen.make_graph(cfg)
    g = oracle.Graph(row_ptr, col, w_q31=thr)
    print(f"graph {time.time() - t0:.0f} s", flush=True)
    small = oracle.Store(g, cfg.seed, 0, 2048, 64)
    s_seeds, s_gains = small.greedy(cfg.k)
    del small
    print(f"theta=2048 {time.time() - t0:.0f} s", flush=True)
    S = oracle.Store(g, cfg.seed, 0, cfg.theta, 64)
    print(f"store {time.time() - t0:.0f} s", flush=True)
    seeds, gains = S.greedy(cfg.k)
    print(f"greedy {time.time() - t0:.0f} s", flush=True)
    np.savez_compressed(
        os.path.join(GOLD, "c2_full_oracle.npz"),
        citation=np.array("BASELINE.json configs[1] (C2), graph_seed 2, sampling seed 0x5EED0002, oracle/ only "
                          "(scripts/make_golden.py); RRR sets by Def. 2 (P:115-121), E_phys by P:239-241, "
                          "greedy by P:93-95 with reading C-11, sigma_hat by C-12"),
        theta=cfg.theta, k=cfg.k, seed=cfg.seed, sizes=S.sizes, digests=S.digests, e_phys=S.e_phys,
        levels=S.levels, frontier=S.frontier.astype(np.uint32), e_logical=np.uint64(S.e_logical),
        seeds=seeds, gains=gains, sigma=oracle.sigma_hat(cfg.n, int(gains.sum()), cfg.theta),
        seeds_2048=s_seeds, gains_2048=s_gains, sigma_2048=oracle.sigma_hat(cfg.n, int(s_gains.sum()), 2048))
    print(f"done {time.time() - t0:.0f} s", flush=True)


def c2_sorted():
    """Group work of the C2 step under sorted start vertices (include/bpt.h BPT_FLAG_UNSORTED off):
    the order is start in-degree descending, start id, sample id -- computed from the oracle's
    start vertices and the forward CSR."""
    cfg = graphgen.CONFIGS["C2"]
    t0 = time.time()
    row_ptr, col, thr = graphgen.make_graph(cfg)
    g = oracle.Graph(row_ptr, col, w_q31=thr)
    ids = np.arange(cfg.theta, dtype=np.int64)
    starts = np.array([oracle.start_vertex(int(s), cfg.n, cfg.seed) for s in ids], dtype=np.int64)
    indeg = np.bincount(col.astype(np.int64), minlength=cfg.n)
    order = ids[np.lexsort((ids, starts, -indeg[starts]))]
    S = oracle.Store(g, cfg.seed, 0, cfg.theta, 64, ids=order, keep=False)
    np.savez_compressed(
        os.path.join(GOLD, "c2_sorted_oracle.npz"),
        citation=np.array("BASELINE.json configs[1] (C2) with sorted start vertices (P:430; SURVEY 8(f) NEXT #3): "
                          "E_phys / levels / frontier sizes per 64-sample group of the sorted order, oracle/ only "
                          "(scripts/make_golden.py C2S); P:239-241"),
        order=order.astype(np.uint32), e_phys=S.e_phys, levels=S.levels, frontier=S.frontier.astype(np.uint32))
    print(f"done {time.time() - t0:.0f} s, e_phys {int(S.e_phys.sum())}", flush=True)


def c4_shard_ids(theta=131072, world=8, rank=7, count=64):
    nb = (theta + 63) // 64
    b0, b1 = rank * nb // world, (rank + 1) * nb // world
    s0, s1 = 64 * b0, min(64 * b1, theta)
    span = s1 - s0
    return np.array(sorted({s0 + (j * span) // count // 64 * 64 + j % 64 for j in range(count)} | {s0, s1 - 1}),
                    dtype=np.uint64)


def c4():
    cfg = graphgen.CONFIGS["C4"]
    t0 = time.time()
    row_ptr, col, thr = graphgen.make_graph(cfg)
    g = oracle.Graph(row_ptr, col, w_q31=thr)
    del col
    print(f"graph {time.time() - t0:.0f} s", flush=True)
    ids = c4_shard_ids(cfg.theta)
    sizes, digests, elog = g.sample_many(cfg.seed, ids)
    print(f"samples {time.time() - t0:.0f} s", flush=True)
    lists = {}
    for j in (0, len(ids) - 1):  # two member lists, sampled (every 997th member) to keep the file small
        mem, _, _ = g.sample_one(cfg.seed, int(ids[j]))
        lists[f"list_{int(ids[j])}_len"] = np.array(len(mem), dtype=np.uint64)
        lists[f"list_{int(ids[j])}_every997"] = mem[::997].copy()
    np.savez_compressed(
        os.path.join(GOLD, "c4_shard7_oracle.npz"),
        citation=np.array("BASELINE.json configs[3] (C4), graph_seed 4, sampling seed 0x5EED0004, theta 131072, "
                          "rank 7 of 8 sample shards; oracle/ only (scripts/make_golden.py); Def. 2 (P:115-121)"),
        theta=cfg.theta, seed=cfg.seed, ids=ids, sizes=sizes, digests=digests, elog=elog, **lists)
    print(f"done {time.time() - t0:.0f} s", flush=True)


if __name__ == "__main__":
    {"C2": c2, "C2S": c2_sorted, "C4": c4}[sys.argv[1]]()
