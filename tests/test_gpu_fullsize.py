"""Full-size parity on the BASELINE.json configs (-m gpu), in the launch configuration bench.py
times. Expected values come from the CPU oracle: precomputed by scripts/make_golden.py (oracle/
only) where the oracle needs tens of minutes (C2 all 65,536 samples, C4), else run here (C3).
Bar (SURVEY §8(c) parity protocol): bit-exact RRR sets (all sizes + digests; member lists where
stored or sampled), seeds, gains; sigma_hat identical (same integers, same f64 formula); exact
E_phys / E_logical / per-level frontier sizes."""
import json
import os

import numpy as np
import pytest

import graphgen
import oracle

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def bpt(cuda_required):
    import torch
    torch.cuda.set_device(0)
    import paper_2311_10201_b200 as b
    return b


@pytest.fixture(scope="module")
def c2(bpt):
    cfg = graphgen.CONFIGS["C2"]
    row_ptr, col, thr = graphgen.make_graph(cfg)
    gold = np.load(os.path.join(GOLD, "c2_full_oracle.npz"))
    assert int(gold["theta"]) == cfg.theta and int(gold["seed"]) == cfg.seed
    g = bpt.Graph(row_ptr, col, w_q31=thr)
    yield cfg, row_ptr, col, thr, gold, g
    g.close()


def _per_batch(rows, col_idx, nb):
    out = np.zeros(nb, np.uint64)
    np.add.at(out, rows[:, 0].astype(np.int64), rows[:, col_idx])
    return out


def test_c2_full_theta(bpt, c2):
    """configs[1] at full size (theta = 2^16, 64 colours, one 64-sample group per batch): every
    sample's size and digest, seeds / gains / sigma_hat of k = 50, E_logical, and per group the
    E_phys and the per-level frontier sizes equal the oracle's."""
    cfg, row_ptr, col, thr, gold, g = c2
    # consecutive-sample groups here (the golden group work is of those groups); the default
    # sorted start vertices are checked in test_c2_full_sorted_start_vertices
    s = g.sample(cfg.theta, colors=64, seed=cfg.seed, flags=bpt.FLAG_UNSORTED | bpt.FLAG_SLOTWISE)
    assert np.array_equal(s.sizes(0, cfg.theta), gold["sizes"])
    assert np.array_equal(s.digests(0, cfg.theta), gold["digests"])
    info = s.info
    assert info["e_logical"] == int(gold["e_logical"])
    assert info["e_phys"] == int(gold["e_phys"].sum())
    assert info["members"] == int(gold["sizes"].astype(np.uint64).sum())
    # per batch of B traversal groups (64-sample blocks in flight together): edge reads, levels and
    # per-level frontier sizes are the sums / maxima of its groups' oracle values
    B = info["batch_groups"]
    ng = cfg.theta // 64
    nb = (ng + B - 1) // B
    grp = np.arange(ng) // B
    rows = s.level_stats()
    want_ephys = np.zeros(nb, np.uint64)
    np.add.at(want_ephys, grp, gold["e_phys"])
    assert np.array_equal(_per_batch(rows, 4, nb), want_ephys)  # edge reads per batch
    want_levels = np.zeros(nb, np.int64)
    np.maximum.at(want_levels, grp, gold["levels"].astype(np.int64))
    assert np.array_equal(np.bincount(rows[:, 0].astype(np.int64), minlength=nb), want_levels)
    want_front = np.zeros((nb, 64), np.uint64)
    np.add.at(want_front, grp, gold["frontier"].astype(np.uint64))
    for b in range(nb):
        r = rows[rows[:, 0] == b]
        assert np.array_equal(r[:, 2], want_front[b, :len(r)]), f"frontier sizes of batch {b}"
    seeds, gains, sigma = s.select_seeds(cfg.k)
    assert np.array_equal(seeds, gold["seeds"]) and np.array_equal(gains, gold["gains"])
    assert sigma == float(gold["sigma"])
    # member lists of groups 0 and G-1 (sampled) against the oracle run here
    og = oracle.Graph(row_ptr, col, w_q31=thr)
    ids = np.array([0, 1, 63, cfg.theta - 64, cfg.theta - 1], dtype=np.uint64)
    _, _, _, off, mem = og.sample_many(cfg.seed, ids, members=True)
    for j, i in enumerate(ids):
        o, m = s.extract(int(i), 1)
        assert np.array_equal(m, mem[off[j]:off[j + 1]])
    s.close()


def test_c2_full_sorted_start_vertices(bpt, c2):
    """The bench's launch configuration (sorted start vertices, the default): all 65,536 sizes and
    digests, seeds, gains, sigma_hat and E_logical equal the oracle's; the groups differ, so E_phys
    equals the oracle's group work of the sorted groups (golden c2_sorted_oracle.npz) and is below
    the consecutive-group value."""
    cfg, row_ptr, col, thr, gold, g = c2
    s = g.sample(cfg.theta, colors=64, seed=cfg.seed)
    assert np.array_equal(s.sizes(0, cfg.theta), gold["sizes"])
    assert np.array_equal(s.digests(0, cfg.theta), gold["digests"])
    info = s.info
    assert info["e_logical"] == int(gold["e_logical"])
    assert info["e_phys"] < int(gold["e_phys"].sum())
    sgold = os.path.join(GOLD, "c2_sorted_oracle.npz")
    if os.path.exists(sgold):
        sg = np.load(sgold)
        assert info["e_phys"] == int(sg["e_phys"].sum())
        B = info["batch_groups"]
        rows = s.level_stats()
        nb = (len(sg["e_phys"]) + B - 1) // B
        want = np.zeros(nb, np.uint64)
        np.add.at(want, np.arange(len(sg["e_phys"])) // B, sg["e_phys"])
        assert np.array_equal(_per_batch(rows, 4, nb), want)
    seeds, gains, sigma = s.select_seeds(cfg.k)
    assert np.array_equal(seeds, gold["seeds"]) and np.array_equal(gains, gold["gains"])
    assert sigma == float(gold["sigma"])
    og = oracle.Graph(row_ptr, col, w_q31=thr)
    ids = np.array([0, 63, 4097, cfg.theta - 1], dtype=np.uint64)
    _, _, _, off, mem = og.sample_many(cfg.seed, ids, members=True)
    for j, i in enumerate(ids):
        o, m = s.extract(int(i), 1)
        assert np.array_equal(m, mem[off[j]:off[j + 1]])
    s.close()


def test_c2_full_batch_wide_frontier(bpt, c2):
    """The bench's launch configuration: sorted start vertices and one frontier per batch of 4
    blocks (the default). The edge reads, level count and per-level frontier sizes of batches 0 and
    90 equal the oracle's fused traversal of their 256 samples, and with one frontier per block
    (BPT_FLAG_SLOTWISE) the edge reads equal the sum of the four 64-sample groups (golden
    c2_sorted_batch_groups_oracle.json, scripts/batch_groups_oracle.py, oracle/ only)."""
    cfg, row_ptr, col, thr, gold, g = c2
    bg = json.load(open(os.path.join(GOLD, "c2_sorted_batch_groups_oracle.json")))
    assert bg["seed"] == cfg.seed
    for flags, key in ((0, "e_phys_256"), (bpt.FLAG_SLOTWISE, "e_phys_4x64")):
        s = g.sample(cfg.theta, colors=64, seed=cfg.seed, flags=flags)
        assert s.info["batch_groups"] == 4
        rows = s.level_stats()
        for b, want in bg["batches"].items():
            r = rows[rows[:, 0] == int(b)]
            exp = want[key] if key == "e_phys_256" else sum(want[key])
            assert int(r[:, 4].sum()) == exp, f"edge reads of batch {b}"
            if not flags:
                assert len(r) == want["levels_256"]
                assert r[:, 2].tolist() == want["frontier_256"], f"frontier sizes of batch {b}"
        assert np.array_equal(s.digests(0, cfg.theta), gold["digests"])
        s.close()


def test_c2_full_graph_theta_2048(bpt, c2):
    """The C2 graph with theta = 2,048 (32 groups): sizes, digests, seeds, gains, sigma_hat."""
    cfg, row_ptr, col, thr, gold, g = c2
    s = g.sample(2048, colors=64, seed=cfg.seed, flags=bpt.FLAG_UNSORTED | bpt.FLAG_SLOTWISE)
    assert np.array_equal(s.sizes(0, 2048), gold["sizes"][:2048])
    assert np.array_equal(s.digests(0, 2048), gold["digests"][:2048])
    assert s.info["e_phys"] == int(gold["e_phys"][:32].sum())
    seeds, gains, sigma = s.select_seeds(cfg.k)
    assert np.array_equal(seeds, gold["seeds_2048"]) and np.array_equal(gains, gold["gains_2048"])
    assert sigma == float(gold["sigma_2048"])
    s.close()


@pytest.mark.parametrize("colors", [1, 8, 32])
def test_c5_colour_sweep_full(bpt, c2, colors):
    """configs[4]: the C2 workload with 1 / 8 / 32 colours per traversal group gives the same
    65,536 RRR sets (sizes, digests), seeds and gains as the oracle (fusion changes only the
    work, reading C-9 / P-4); with one colour the fused reads equal the unfused ones (E_phys =
    E_logical), and fewer colours never read fewer edges (Theorem 1)."""
    cfg, row_ptr, col, thr, gold, g = c2
    # default (1 < C < 64: groups of C samples adjacent in start order) and consecutive groups;
    # the golden E_phys is that of consecutive 64-sample groups, which nest the consecutive C-groups
    for flags in ((0, bpt.FLAG_UNSORTED) if colors > 1 else (0,)):
        s = g.sample(cfg.theta, colors=colors, seed=cfg.seed, flags=flags)
        assert np.array_equal(s.sizes(0, cfg.theta), gold["sizes"])
        assert np.array_equal(s.digests(0, cfg.theta), gold["digests"])
        info = s.info
        assert info["e_logical"] == int(gold["e_logical"])
        assert info["e_phys"] <= info["e_logical"]
        if colors == 1 or flags:
            assert info["e_phys"] >= int(gold["e_phys"].sum())
        if colors == 1:
            assert info["e_phys"] == info["e_logical"]
        seeds, gains, sigma = s.select_seeds(cfg.k)
        assert np.array_equal(seeds, gold["seeds"]) and np.array_equal(gains, gold["gains"])
        s.close()


def test_c2_full_wide_fusion(bpt, c2):
    """BPT_FLAG_WIDE (128 colours per frontier entry) on the full C2 workload: same sets and seeds."""
    cfg, row_ptr, col, thr, gold, g = c2
    s = g.sample(cfg.theta, colors=64, seed=cfg.seed, wide=True)
    assert np.array_equal(s.digests(0, cfg.theta), gold["digests"])
    assert np.array_equal(s.sizes(0, cfg.theta), gold["sizes"])
    seeds, gains, _ = s.select_seeds(cfg.k)
    assert np.array_equal(seeds, gold["seeds"]) and np.array_equal(gains, gold["gains"])
    assert s.info["e_phys"] < int(gold["e_phys"].sum())  # 128-sample groups share more reads
    s.close()


def test_c3_full(bpt):
    """configs[2] (LT, theta = 2^18, k = 100) at full size: every sorted member list, seeds,
    gains and sigma_hat equal the oracle's; the fused level-synchronous form too."""
    cfg = graphgen.CONFIGS["C3"]
    row_ptr, col, thr = graphgen.make_graph(cfg)
    og = oracle.Graph(row_ptr, col, w_q31=thr, model=oracle.LT)
    ids = np.arange(cfg.theta, dtype=np.uint64)
    sizes, digests, elog, off, mem = og.sample_many(cfg.seed, ids, members=True)
    seeds_o, gains_o = oracle.greedy(cfg.n, off, mem, cfg.k, lazy=True)
    sigma_o = oracle.sigma_hat(cfg.n, int(gains_o.sum()), cfg.theta)
    g = bpt.Graph(row_ptr, col, w_q31=thr, model=bpt.LT)
    for flags in (0, bpt.FLAG_LT_FUSED):
        s = g.sample(cfg.theta, colors=64, seed=cfg.seed, flags=flags)
        assert np.array_equal(s.sizes(0, cfg.theta), sizes)
        assert np.array_equal(s.digests(0, cfg.theta), digests)
        o, m = s.extract(0, cfg.theta)
        assert np.array_equal(o, off) and np.array_equal(m, mem)
        seeds, gains, sigma = s.select_seeds(cfg.k)
        assert np.array_equal(seeds, seeds_o) and np.array_equal(gains, gains_o) and sigma == sigma_o
        assert s.info["e_phys"] == s.info["e_logical"] == int(sizes.astype(np.uint64).sum()) == int(elog.sum())
        s.close()


def test_c4_rank_shard(bpt):
    """configs[3] (65.6M vertices, 1.81B edges, theta = 2^17 over 8 GPUs): the last rank's shard
    (16,384 samples, a 134 GB fused store) sampled on this one GPU through the shard hook -- the
    8-GPU per-rank memory plan -- with exact sizes and digests of 66 sample ids spread over the
    shard and all 64 colour slots, and two member lists, against the oracle (golden file)."""
    cfg = graphgen.CONFIGS["C4"]
    gold = np.load(os.path.join(GOLD, "c4_shard7_oracle.npz"))
    assert int(gold["theta"]) == cfg.theta and int(gold["seed"]) == cfg.seed
    row_ptr, col, thr = graphgen.make_graph(cfg)
    g = bpt.Graph(row_ptr, col, w_q31=thr)
    del col, thr
    s = g.sample(cfg.theta, colors=64, seed=cfg.seed, shard=(8, 7))
    g.close()
    assert (s.s0, s.s1) == graphgen.shard_range(cfg.theta, 8, 7)
    assert s.info["store_bytes"] >= 256 * cfg.n * 8  # the rank's dense store is resident
    ids = gold["ids"].astype(np.int64)
    sizes = s.sizes(s.s0, s.s1 - s.s0)
    digests = s.digests(s.s0, s.s1 - s.s0)
    assert np.array_equal(sizes[ids - s.s0], gold["sizes"])
    assert np.array_equal(digests[ids - s.s0], gold["digests"])
    for key in gold.files:
        if key.startswith("list_") and key.endswith("_every997"):
            i = int(key[5:].split("_")[0])
            o, m = s.extract(i, 1)
            assert len(m) == int(gold[f"list_{i}_len"])
            assert np.array_equal(m[::997], gold[key])
    s.close()
    from paper_2311_10201_b200.bpt import bpt_release_cache
    bpt_release_cache()  # return the 134 GB to the device for the tests after this one
