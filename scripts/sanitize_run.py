"""Small end-to-end run of every execution form of the hot path, for compute-sanitizer
(memcheck / racecheck / synccheck, one tool per run):
  compute-sanitizer --tool memcheck --error-exitcode 9 python scripts/sanitize_run.py
C1 (R-MAT scale 10) and a C2-shaped scale-14 graph (IC: batch-wide frontier default, one frontier per
block, pull, first-setter queue, C = 8, wide fusion, profile mode), a C3-shaped scale-12 graph (LT: sparse walks, dense walks, fused
level loop), selection, extraction; every result is checked against the CPU oracle, so a run that
the tool passes is also a correct one."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import graphgen  # noqa: E402
import oracle  # noqa: E402


def main():
    import torch
    torch.cuda.set_device(0)
    import paper_2311_10201_b200 as bpt
    cases = [("C1", None, 512, bpt.IC, [dict(), dict(flags=bpt.FLAG_QUEUE), dict(colors=8), dict(wide=True),
                                         dict(profile=True), dict(batch_groups=3), dict(flags=bpt.FLAG_SLOTWISE),
                                         dict(pull=True, pull_permille=1), dict(batch_groups=8)]),
             ("C2", 1 << 14, 320, bpt.IC, [dict(), dict(flags=bpt.FLAG_QUEUE), dict(wide=True), dict(profile=True),
                                          dict(flags=bpt.FLAG_SLOTWISE | bpt.FLAG_UNSORTED),
                                          dict(pull=True, pull_permille=1)]),
             ("C3", 1 << 12, 400, bpt.LT, [dict(), dict(flags=bpt.FLAG_LT_DENSE), dict(flags=bpt.FLAG_LT_FUSED),
                                          dict(flags=bpt.FLAG_LT_FUSED | bpt.FLAG_LT_LEVELS)])]
    for name, n, theta, model, variants in cases:
        cfg = graphgen.CONFIGS[name] if n is None else graphgen.scaled(graphgen.CONFIGS[name], n, theta=theta)
        row_ptr, col, thr = graphgen.make_graph(cfg)
        og = oracle.Graph(row_ptr, col, w_q31=thr, model=oracle.IC if model == bpt.IC else oracle.LT)
        sizes, digests, _, off, mem = og.sample_many(cfg.seed, np.arange(theta, dtype=np.uint64), members=True)
        seeds, gains = oracle.greedy(cfg.n, off, mem, 5)
        g = bpt.Graph(row_ptr, col, w_q31=thr, model=model)
        for kw in variants:
            s = g.sample(theta, seed=cfg.seed, **kw)
            assert np.array_equal(s.sizes(0, theta), sizes), (name, kw)
            assert np.array_equal(s.digests(0, theta), digests), (name, kw)
            o, m = s.extract(3, 70)
            assert np.array_equal(m, mem[off[3]:off[73]]), (name, kw)
            sd, gn, _ = s.select_seeds(5)
            assert np.array_equal(sd, seeds) and np.array_equal(gn, gains), (name, kw)
            s.close()
            print(f"ok {name} {kw}", flush=True)
        g.close()
    kat = np.array([[0, 0, 0], [0x243F6A88, 0x85A308D3, 0x13198A2E]], np.uint32)
    assert bpt.selftest_philox(kat)[1].tolist() == [0xDD7CE038, 0xF62A4C12]
    print("sanitize_run ok")


if __name__ == "__main__":
    main()
