"""GPU parity tests (-m gpu): the CUDA path through the C-ABI vs the CPU oracle on the same
seeded inputs. Bar: bit-exact RRR sets, sizes, digests, seeds and gains; sigma_hat
identical (integers in, same f64 formula); exact E_phys / E_logical / level structure
(DESIGN.md §Parity)."""
import json
import os

import numpy as np
import pytest

import graphgen
import oracle

pytestmark = pytest.mark.gpu
Q31 = 1 << 31
GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def bpt(cuda_required):
    import torch
    torch.cuda.set_device(0)
    import paper_2311_10201_b200 as b
    return b


def oracle_all(row_ptr, col, thr, model, theta, seed, colors=64, k=None, threads=None):
    g = oracle.Graph(row_ptr, col, w_q31=thr, model=model)
    ids = np.arange(theta, dtype=np.uint64)
    sizes, digests, elog, offsets, mem = g.sample_many(seed, ids, threads, members=True)
    out = {"g": g, "sizes": sizes, "digests": digests, "elog": elog, "offsets": offsets, "members": mem}
    if k:
        out["seeds"], out["gains"] = oracle.greedy(g.n, offsets, mem, k)
    return out


def sorted_slots(row_ptr, col, n, theta, seed, s0=0):
    """Traversal order of the samples [s0, theta) under sorted start vertices (include/bpt.h
    BPT_FLAG_UNSORTED): start in-degree descending, then start id, then
    sample id -- computed here from the oracle's start vertices and the forward CSR."""
    ids = np.arange(s0, theta, dtype=np.int64)
    starts = np.array([oracle.start_vertex(int(s), n, seed) for s in ids], dtype=np.int64)
    indeg = np.bincount(col.astype(np.int64), minlength=n)
    return ids[np.lexsort((ids, starts, -indeg[starts]))]


def group_e_phys(og, seed, order, group):
    """E_phys of traversal groups of `group` consecutive samples of `order`."""
    return [og.group_work_ids(seed, order[i:i + group]) for i in range(0, len(order), group)]


def check_full(bpt, s, ref, theta):
    assert np.array_equal(s.sizes(0, theta), ref["sizes"])
    assert np.array_equal(s.digests(0, theta), ref["digests"])
    off, mem = s.extract(0, theta)
    assert np.array_equal(off, ref["offsets"])
    assert np.array_equal(mem, ref["members"])


# ------------------------------------------------------------------ coins (reading C-1), device side

def test_device_philox_kat(bpt):
    """SURVEY §8(c) P-1 on the device: the Philox2x32-10 every coin and start vertex of the CUDA
    path goes through reproduces the Random123 known-answer vectors, and agrees with the oracle's
    independent copy on random counters."""
    kat = json.load(open(os.path.join(GOLD, "philox_kat.json")))["philox2x32_10"]
    rows = np.array([[int(c0, 16), int(c1, 16), int(k, 16)] for c0, c1, k, _, _ in kat], np.uint32)
    want = np.array([[int(o0, 16), int(o1, 16)] for _, _, _, o0, o1 in kat], np.uint32)
    assert np.array_equal(bpt.selftest_philox(rows), want)
    rng = np.random.default_rng(11)
    r = rng.integers(0, 1 << 32, size=(2000, 3), dtype=np.uint64).astype(np.uint32)
    got = bpt.selftest_philox(r)
    for i in range(0, 2000, 97):
        assert tuple(int(x) for x in got[i]) == oracle.philox2x32_10(int(r[i, 0]), int(r[i, 1]), int(r[i, 2]))


def test_launch_evidence_counts(bpt):
    """bpt_kernel_launch_count counts host launches (one per graph launch in graph mode);
    bpt_graph_kernel_count counts the kernels the sampling graph ran, counted on the device:
    per batch init + finalize + next_batch, per level compact + expand."""
    cfg = graphgen.CONFIGS["C1"]
    row_ptr, col, thr = graphgen.make_graph(cfg)
    g = bpt.Graph(row_ptr, col, w_q31=thr)
    h0, d0 = bpt.kernel_launch_count(), bpt.graph_kernel_count()
    s = g.sample(cfg.theta, seed=cfg.seed, batch_groups=1, flags=bpt.FLAG_UNSORTED)
    h1, d1 = bpt.kernel_launch_count(), bpt.graph_kernel_count()
    info = s.info
    assert h1 - h0 == 1  # the graph launch
    assert d1 - d0 == 3 * info["batches"] + 2 * info["levels_total"]
    assert info["kernel_launches"] == (h1 - h0) + (d1 - d0)
    # sorted start vertices add the slot sort: key kernel, log2(N)(log2(N)+1)/2 bitonic steps, maps
    h1, d1 = bpt.kernel_launch_count(), bpt.graph_kernel_count()
    s = g.sample(cfg.theta, seed=cfg.seed, batch_groups=1)
    lg = (cfg.theta - 1).bit_length()
    assert bpt.kernel_launch_count() - h1 == 1 + 2 + lg * (lg + 1) // 2
    assert bpt.graph_kernel_count() - d1 == 3 * s.info["batches"] + 2 * s.info["levels_total"]
    h1, d1 = bpt.kernel_launch_count(), bpt.graph_kernel_count()
    p = g.sample(cfg.theta, seed=cfg.seed, batch_groups=1, profile=True)
    assert bpt.graph_kernel_count() == d1  # profile mode launches directly
    assert bpt.kernel_launch_count() - h1 >= 3 * p.info["batches"] + 2 * p.info["levels_total"]


# ------------------------------------------------------------------ A0/A1 builder

def test_reverse_csr_equals_oracle_transpose(bpt):
    for trial in range(3):
        row_ptr, col = graphgen.random_graph(500 + 97 * trial, 6000, seed=trial, self_loops=True)
        # add parallel edges: duplicate every 7th edge inside its row (stable order matters, C-4)
        rng = np.random.default_rng(trial)
        wf = rng.random(col.shape[0]).astype(np.float32)
        wf[::11] = 1.0
        wf[::13] = 0.0
        g = bpt.Graph(row_ptr, col, w_f32=wf)
        roff, src, thr = g.reverse_csr()
        o_roff, o_src, o_thr = oracle.Graph(row_ptr, col, w_f32=wf).reverse_csr()
        assert np.array_equal(roff.astype(np.uint64), o_roff)
        assert np.array_equal(src, o_src)
        assert np.array_equal(thr, o_thr)


def test_reverse_csr_multigraph_and_lt_prefix(bpt):
    n = 300
    rng = np.random.default_rng(5)
    u = rng.integers(0, n, 5000)
    v = rng.integers(0, n, 5000)
    order = np.argsort(u, kind="stable")
    u, v = u[order], v[order]  # rows by u, destinations unsorted, duplicates kept
    row_ptr = np.zeros(n + 1, np.uint64)
    np.add.at(row_ptr, u + 1, 1)
    row_ptr = np.cumsum(row_ptr).astype(np.uint64)
    col = v.astype(np.uint32)
    thr = graphgen.weights_lt(n, col, seed=9)
    g = bpt.Graph(row_ptr, col, w_q31=thr, model=bpt.LT)
    roff, src, cum = g.reverse_csr()
    o_roff, o_src, o_thr = oracle.Graph(row_ptr, col, w_q31=thr, model=oracle.LT).reverse_csr()
    assert np.array_equal(roff.astype(np.uint64), o_roff)
    assert np.array_equal(src, o_src)
    want = np.zeros_like(o_thr, dtype=np.uint64)
    for x in range(n):
        a, b = int(o_roff[x]), int(o_roff[x + 1])
        want[a:b] = np.cumsum(o_thr[a:b].astype(np.uint64))
    assert np.array_equal(cum.astype(np.uint64), want)


def _hub_graph(n, hubs, others, seed):
    """Forward CSR with `hubs` = {v: in-degree} heavy rows (spanning several 4096-item builder
    tiles) plus `others` random edges; rows by source, duplicates kept."""
    rng = np.random.default_rng(seed)
    v = np.concatenate([np.full(d, h, np.int64) for h, d in hubs.items()] + [rng.integers(0, n, others)])
    u = rng.integers(0, n, v.shape[0])
    order = np.argsort(u, kind="stable")
    u, v = u[order], v[order]
    row_ptr = np.zeros(n + 1, np.uint64)
    np.add.at(row_ptr, u + 1, 1)
    return np.cumsum(row_ptr).astype(np.uint64), v.astype(np.uint32)


def test_reverse_csr_hub_rows_across_tiles(bpt):
    """Three 8-bit radix passes (n > 2^16) and in-degree hubs spanning many builder tiles:
    the payload-carrying sort keeps the stable order (C-4) and the LT segmented scan carries
    row prefixes across tiles (C-6)."""
    n = 70000
    row_ptr, col = _hub_graph(n, {5: 30000, n - 1: 9000, 4097: 4097}, 20000, seed=3)
    rng = np.random.default_rng(4)
    indeg = np.bincount(col, minlength=n)
    thr = (rng.random(col.shape[0]) * (Q31 // np.maximum(indeg[col], 1))).astype(np.uint32)
    for model, omodel in ((bpt.IC, oracle.IC), (bpt.LT, oracle.LT)):
        g = bpt.Graph(row_ptr, col, w_q31=thr, model=model)
        roff, src, got = g.reverse_csr()
        o_roff, o_src, o_thr = oracle.Graph(row_ptr, col, w_q31=thr, model=omodel).reverse_csr()
        assert np.array_equal(roff.astype(np.uint64), o_roff)
        assert np.array_equal(src, o_src)
        if model == bpt.IC:
            assert np.array_equal(got, o_thr)
        else:
            seg = np.repeat(np.arange(n), np.diff(o_roff.astype(np.int64)))
            c = np.cumsum(o_thr.astype(np.uint64))
            start = np.concatenate([[0], c])[o_roff[:-1].astype(np.int64)]
            assert np.array_equal(got.astype(np.uint64), c - start[seg])
        g.close()
    # an LT row whose sum passes 2^31 only in its last tile is rejected with its vertex id
    bad = thr.copy()
    bad[col == 5] = Q31 // 30000 + 1
    with pytest.raises(bpt.BptError) as ei:
        bpt.Graph(row_ptr, col, w_q31=bad, model=bpt.LT)
    assert "vertex 5 " in str(ei.value)


def test_invalid_inputs_rejected(bpt):
    rp = np.array([0, 2, 3], np.uint64)
    col = np.array([1, 0, 1], np.uint32)
    ok = np.array([1, 2, 3], np.uint32)
    cases = [
        (np.array([0, 2, 1, 3], np.uint64), col, dict(w_q31=ok), "decreasing"),
        (np.array([1, 2, 3], np.uint64), col, dict(w_q31=ok), "row_ptr[0]"),
        (rp, np.array([1, 5, 1], np.uint32), dict(w_q31=ok), "col["),
        (rp, col, dict(w_q31=np.array([1, Q31 + 1, 0], np.uint32)), "weight[1]"),
        (rp, col, dict(w_f32=np.array([0.5, np.nan, 0.1], np.float32)), "weight[1]"),
        (rp, col, dict(w_f32=np.array([0.5, 1.5, 0.1], np.float32)), "weight[1]"),
    ]
    for r, c, w, msg in cases:
        with pytest.raises(bpt.BptError) as ei:
            bpt.Graph(r, c, **w)
        assert ei.value.code == bpt.BPT_EINVAL and msg in str(ei.value)
    with pytest.raises(bpt.BptError) as ei:  # LT row sum > 2^31 at vertex 1
        bpt.Graph(rp, col, w_q31=np.array([Q31, 0, 1], np.uint32), model=bpt.LT)
    assert "vertex 1" in str(ei.value)
    g = bpt.Graph(rp, col, w_q31=ok)
    for kw in [dict(theta=0), dict(theta=64, colors=3), dict(theta=64, colors=0), dict(theta=1 << 32)]:
        with pytest.raises(bpt.BptError) as ei:
            g.sample(**kw)
        assert ei.value.code == bpt.BPT_EINVAL
    with pytest.raises(bpt.BptError):
        bpt.bpt_sample(g._h, bpt.LT, 64, 64, 1)  # model mismatch
    s = g.sample(100, seed=1)
    for k in (0, 4):
        with pytest.raises(bpt.BptError):
            s.select_seeds(k)
    with pytest.raises(bpt.BptError):
        s.sizes(90, 20)
    with pytest.raises(bpt.BptError) as ei:
        s.extract(0, 10, members=np.empty(1, np.uint32), capacity=1)
    assert ei.value.code == bpt.BPT_ENOMEM


# ------------------------------------------------------------------ worked example P:139-143

def test_worked_example_on_gpu(bpt):
    fx = json.load(open(os.path.join(GOLD, "fig_fused_example.json")))
    n = fx["n"]
    edges = sorted((tuple(e) for e in fx["edges"]), key=lambda t: (t[0], t[1]))
    row_ptr = np.zeros(n + 1, np.uint64)
    for a, _, _ in edges:
        row_ptr[a + 1] += 1
    row_ptr = np.cumsum(row_ptr).astype(np.uint64)
    col = np.array([b for _, b, _ in edges], np.uint32)
    thr = np.array([t for _, _, t in edges], np.uint32)
    g = bpt.Graph(row_ptr, col, w_q31=thr)
    roff, src, _ = g.reverse_csr()
    assert roff.tolist() == fx["reverse_csr"]["roff"] and src.tolist() == fx["reverse_csr"]["src"]
    s = g.sample(fx["theta"], colors=64, seed=fx["seed"], batch_groups=1)
    off, mem = s.extract(0, 4)
    names = {v: k for k, v in fx["colors"].items()}
    for c in range(4):
        assert mem[off[c]:off[c + 1]].tolist() == fx["rrr"][names[c]]
    assert mem[off[3]:off[4]].tolist() == [4, 5, 6, 7, 8]  # yellow
    rows = s.level_stats()
    # raw entries per level = frontier sizes (a) {1,3,5} (b) {0,4} (c) {3,6,7,8} {4} {6,7,8}
    assert rows[:, 2].tolist() == [len(f) for f in fx["frontiers"]]
    assert rows[:, 5].tolist() == [sum(len(c) for c in f.values()) for f in fx["frontiers"]]


# ------------------------------------------------------------------ degenerate probabilities

def test_p0_and_p1(bpt):
    row_ptr, col = graphgen.random_graph(2000, 16000, seed=3)
    theta, seed = 777, 31
    g0 = bpt.Graph(row_ptr, col, w_q31=np.zeros(col.shape[0], np.uint32))
    s0 = g0.sample(theta, seed=seed)
    assert np.all(s0.sizes(0, theta) == 1)
    off, mem = s0.extract(0, theta)
    assert mem.tolist() == [oracle.start_vertex(s, 2000, seed) for s in range(theta)]
    thr1 = np.full(col.shape[0], Q31, np.uint32)
    g1 = bpt.Graph(row_ptr, col, w_q31=thr1)
    s1 = g1.sample(theta, seed=seed)
    ref = oracle_all(row_ptr, col, thr1, oracle.IC, theta, seed)  # oracle pinned to networkx at p=1
    check_full(bpt, s1, ref, theta)


# ------------------------------------------------------------------ C1 full parity

@pytest.mark.parametrize("colors", [64, 32, 8, 1])
def test_c1_full_parity(bpt, colors):
    cfg = graphgen.CONFIGS["C1"]
    row_ptr, col, thr = graphgen.make_graph(cfg)
    ref = oracle_all(row_ptr, col, thr, oracle.IC, cfg.theta, cfg.seed, k=cfg.k)
    g = bpt.Graph(row_ptr, col, w_q31=thr)
    for batch in (1, 3, 16):
        s = g.sample(cfg.theta, colors=colors, seed=cfg.seed, batch_groups=batch)
        check_full(bpt, s, ref, cfg.theta)
        seeds, gains, sigma = s.select_seeds(cfg.k)
        assert np.array_equal(seeds, ref["seeds"]) and np.array_equal(gains, ref["gains"])
        assert sigma == oracle.sigma_hat(cfg.n, int(ref["gains"].sum()), cfg.theta)
        info = s.info
        # exact work counters: E_phys = sum over traversal groups of the
        # distinct (v, level) pairs weighted by in-degree; E_logical = unfused reads. With 64
        # colours (and 1 < C < 64) the samples are in sorted start order (BPT_FLAG_UNSORTED off); at 64: a batch of
        # <= 4 blocks shares one frontier (BPT_FLAG_SLOTWISE off): one group per batch
        order = (sorted_slots(row_ptr, col, cfg.n, cfg.theta, cfg.seed) if colors > 1  # C = 1: no sort
                 else np.arange(cfg.theta))
        group = 64 * info["batch_groups"] if colors == 64 and info["batch_groups"] <= 4 else colors
        e_phys = sum(w["e_phys"] for w in group_e_phys(ref["g"], cfg.seed, order, group))
        assert info["e_phys"] == e_phys
        assert info["e_logical"] == int(ref["elog"].sum())
        assert info["members"] == int(ref["sizes"].sum())
        assert info["e_phys"] <= info["e_logical"]  # Theorem 1
        if colors == 1:
            assert info["e_phys"] == info["e_logical"]


def test_c1_level_structure_per_group(bpt):
    """batch_groups = 1: each batch is one 64-colour group -- 64 samples in sorted start order by
    default, 64 consecutive samples with BPT_FLAG_UNSORTED; its per-level frontier sizes and edge
    reads equal the oracle's level sets of the same group."""
    cfg = graphgen.CONFIGS["C1"]
    row_ptr, col, thr = graphgen.make_graph(cfg)
    og = oracle.Graph(row_ptr, col, w_q31=thr)
    g = bpt.Graph(row_ptr, col, w_q31=thr)
    order = sorted_slots(row_ptr, col, cfg.n, cfg.theta, cfg.seed)
    for flags, groups in ((0, order), (bpt.FLAG_UNSORTED, np.arange(cfg.theta))):
        s = g.sample(cfg.theta, colors=64, seed=cfg.seed, batch_groups=1, poll_levels=1, flags=flags)
        rows = s.level_stats()
        for b in range(cfg.theta // 64):
            w = og.group_work_ids(cfg.seed, groups[64 * b:64 * b + 64])
            r = rows[rows[:, 0] == b]
            assert r[:, 2].tolist() == w["frontier"].tolist()
            assert int(r[:, 4].sum()) == w["e_phys"]
            assert len(r) == w["levels"]


# ------------------------------------------------------------------ ragged and edge cases

def test_ragged_theta_and_ranges(bpt):
    cfg = graphgen.CONFIGS["C1"]
    row_ptr, col, thr = graphgen.make_graph(cfg)
    g = bpt.Graph(row_ptr, col, w_q31=thr)
    for theta, wide in ((1, False), (63, False), (65, False), (200, False), (1, True), (65, True), (200, True)):
        ref = oracle_all(row_ptr, col, thr, oracle.IC, theta, 99)
        s = g.sample(theta, colors=64, seed=99, wide=wide)
        check_full(bpt, s, ref, theta)
        for first, count in [(0, 1), (theta - 1, 1), (theta // 3, theta - theta // 3)]:
            off, mem = s.extract(first, count)
            a, b = int(ref["offsets"][first]), int(ref["offsets"][first + count])
            assert np.array_equal(mem, ref["members"][a:b])
            assert np.array_equal(off, ref["offsets"][first:first + count + 1] - ref["offsets"][first])
            # pinned host buffers with spare capacity (bench.py's end-to-end path)
            import torch
            pm = torch.full((b - a + 7,), 0xABCD, dtype=torch.int32).pin_memory()
            po = torch.empty(count + 1, dtype=torch.int64).pin_memory()
            s.extract(first, count, offsets=po, members=pm, capacity=pm.numel())
            assert np.array_equal(pm.numpy()[: b - a].view(np.uint32), ref["members"][a:b])
            assert (pm.numpy()[b - a:] == 0xABCD).all()
            assert np.array_equal(po.numpy().view(np.uint64), ref["offsets"][first:first + count + 1] - ref["offsets"][first])


@pytest.mark.parametrize("mode",["ic", "ic_queue", "ic_wide", "lt", "lt_dense", "lt_fused"])
def test_graph_without_edges(bpt, mode):
    n = 10
    flags = {"lt_dense": bpt.FLAG_LT_DENSE, "lt_fused": bpt.FLAG_LT_FUSED, "ic_queue": bpt.FLAG_QUEUE}.get(mode, 0)
    model = bpt.LT if mode.startswith("lt") else bpt.IC
    g = bpt.Graph(np.zeros(n + 1, np.uint64), np.zeros(0, np.uint32), w_q31=np.zeros(0, np.uint32), model=model)
    s = g.sample(100, seed=4, wide=mode == "ic_wide", flags=flags)
    off, mem = s.extract(0, 100)
    assert mem.tolist() == [oracle.start_vertex(i, n, 4) for i in range(100)]
    seeds, gains, sigma = s.select_seeds(n)
    assert sorted(seeds.tolist()) == list(range(n)) and int(gains.sum()) == 100


def test_device_pointers_and_determinism(bpt):
    import torch
    cfg = graphgen.CONFIGS["C1"]
    row_ptr, col, thr = graphgen.make_graph(cfg)
    gh = bpt.Graph(row_ptr, col, w_q31=thr)
    dev = torch.device("cuda")
    gd = bpt.Graph(torch.from_numpy(row_ptr.astype(np.int64)).to(dev), torch.from_numpy(col.astype(np.int32)).to(dev),
                   w_q31=torch.from_numpy(thr.astype(np.int32)).to(dev), n=cfg.n, m=cfg.m)
    a = gh.sample(cfg.theta, seed=cfg.seed)
    b = gd.sample(cfg.theta, seed=cfg.seed)
    c = gh.sample(cfg.theta, seed=cfg.seed, batch_groups=5, poll_levels=7)
    for x in (b, c):
        assert np.array_equal(a.digests(0, cfg.theta), x.digests(0, cfg.theta))
    out = torch.empty(cfg.theta, dtype=torch.int64, device=dev)
    a.digests(0, cfg.theta, out=out)
    assert np.array_equal(out.cpu().numpy().view(np.uint64), a.digests(0, cfg.theta))


# ------------------------------------------------------------------ LT (C3 shape, scaled)

def test_lt_parity_scaled(bpt):
    cfg = graphgen.scaled(graphgen.CONFIGS["C3"], 1 << 13, theta=4096)
    row_ptr, col, thr = graphgen.make_graph(cfg)
    ref = oracle_all(row_ptr, col, thr, oracle.LT, cfg.theta, cfg.seed, k=cfg.k)
    g = bpt.Graph(row_ptr, col, w_q31=thr, model=bpt.LT)
    for colors, batch in ((64, 0), (64, 7), (16, 3)):
        s = g.sample(cfg.theta, colors=colors, seed=cfg.seed, batch_groups=batch)
        check_full(bpt, s, ref, cfg.theta)
        seeds, gains, _ = s.select_seeds(cfg.k)
        assert np.array_equal(seeds, ref["seeds"]) and np.array_equal(gains, ref["gains"])
        assert s.info["e_phys"] == s.info["members"] == int(ref["sizes"].sum())


@pytest.mark.parametrize("model", ["IC", "LT"])
def test_level_loop_variants(bpt, model):
    """The execution forms of the sampling loop give the same RRR sets, seeds and exact work
    counters. IC: the touched-bitmap frontier (default) and the first-setter queue
    (BPT_FLAG_QUEUE), each in the graph's conditional WHILE loop and in the host-driven profiling
    mode. LT: the fused level-synchronous loop (one cooperative launch per batch, or per-level
    launches with BPT_FLAG_LT_LEVELS) and the one-walk-per-thread sampler (default; sparse
    member-list store, lists by a second walk, or the dense store)."""
    if model == "IC":
        cfg = graphgen.CONFIGS["C1"]
        row_ptr, col, thr = graphgen.make_graph(cfg)
        ref = oracle_all(row_ptr, col, thr, oracle.IC, cfg.theta, cfg.seed, k=cfg.k)
        g = bpt.Graph(row_ptr, col, w_q31=thr)
        # consecutive-sample 64-colour groups in both forms (equal work counters), then the default
        # (sorted slots, one frontier per batch)
        variants = [bpt.FLAG_UNSORTED | bpt.FLAG_SLOTWISE, bpt.FLAG_QUEUE | bpt.FLAG_UNSORTED, 0]
    else:
        cfg = graphgen.scaled(graphgen.CONFIGS["C3"], 1 << 12, theta=2048)
        row_ptr, col, thr = graphgen.make_graph(cfg)
        ref = oracle_all(row_ptr, col, thr, oracle.LT, cfg.theta, cfg.seed, k=cfg.k)
        g = bpt.Graph(row_ptr, col, w_q31=thr, model=bpt.LT)
        variants = [bpt.FLAG_LT_FUSED | bpt.FLAG_LT_LEVELS, bpt.FLAG_LT_FUSED,
                    0,                        # walks, sparse store (default)
                    bpt.FLAG_LT_REWALK,       # lists by a 2nd walk
                    bpt.FLAG_LT_DENSE]        # walks, dense store
    infos = []
    for vflags in variants:
        rows = []
        for colors, batch, profile in ((64, 1, False), (64, 5, False), (8, 2, False), (64, 3, True)):
            s = g.sample(cfg.theta, colors=colors, seed=cfg.seed, batch_groups=batch, profile=profile, flags=vflags)
            check_full(bpt, s, ref, cfg.theta)
            seeds, gains, _ = s.select_seeds(cfg.k)
            assert np.array_equal(seeds, ref["seeds"]) and np.array_equal(gains, ref["gains"])
            info = s.info
            walker = model == "LT" and not (vflags & bpt.FLAG_LT_FUSED)
            if walker:
                dense_bytes = (cfg.theta + 63) // 64 * cfg.n * 8
                assert (info["store_bytes"] >= dense_bytes) == bool(vflags & bpt.FLAG_LT_DENSE)
            rows.append((info["e_phys"], info["e_logical"], info["members"]) if walker else
                        (colors, batch, info["e_phys"], info["e_logical"], info["members"], info["levels_total"]))
            s.close()
        infos.append(rows)
    assert infos[0] == infos[1]
    if model == "IC":  # sorted start vertices: other groups, same sets (E_logical, members)
        assert [r[3:5] for r in infos[2]] == [r[3:5] for r in infos[0]]
    if model == "LT":  # walks: same work counters as the fused loop (E_phys = E_logical = sum |RR|)
        for walk in infos[2:]:
            assert [r[2:5] for r in infos[0]] == walk
            assert all(r[0] == r[1] == r[2] == int(ref["sizes"].sum()) for r in walk)


@pytest.mark.parametrize("which", ["C1", "C2s"])
def test_wide_fusion(bpt, which):
    """Wide fusion (BPT_FLAG_WIDE: 2 blocks = 128 colours share one frontier):
    identical RRR sets, seeds and gains; E_phys equals the oracle's group work of the 128-sample
    groups (the same distinct-(v, level) formula), and stays <= E_logical."""
    if which == "C1":
        cfg = graphgen.CONFIGS["C1"]
    else:
        cfg = graphgen.scaled(graphgen.CONFIGS["C2"], 1 << 14, theta=1024 + 64 + 17)  # ragged last batch
    row_ptr, col, thr = graphgen.make_graph(cfg)
    ref = oracle_all(row_ptr, col, thr, oracle.IC, cfg.theta, cfg.seed, k=cfg.k)
    g = bpt.Graph(row_ptr, col, w_q31=thr)
    for profile in (False, True):
        s = g.sample(cfg.theta, colors=64, seed=cfg.seed, profile=profile, wide=True)
        check_full(bpt, s, ref, cfg.theta)
        seeds, gains, _ = s.select_seeds(cfg.k)
        assert np.array_equal(seeds, ref["seeds"]) and np.array_equal(gains, ref["gains"])
        info = s.info
        B = info["batch_groups"]  # blocks sharing one frontier (2 in the product build)
        assert B >= 2
        e_phys = sum(ref["g"].group_work(cfg.seed, a, min(a + 64 * B, cfg.theta))["e_phys"]
                     for a in range(0, cfg.theta, 64 * B))
        assert info["e_phys"] == e_phys
        assert info["e_logical"] == int(ref["elog"].sum())
        assert info["e_phys"] <= info["e_logical"]
        s.close()


def test_lt_sparse_store(bpt):
    """BPT_FLAG_SPARSE (LT): the RRR sets kept as sorted member lists, no dense store; sizes,
    digests, extraction (ragged ranges), occurrences and seeds/gains identical to the oracle."""
    cfg = graphgen.scaled(graphgen.CONFIGS["C3"], 1 << 13, theta=4096 + 64 + 5)
    row_ptr, col, thr = graphgen.make_graph(cfg)
    ref = oracle_all(row_ptr, col, thr, oracle.LT, cfg.theta, cfg.seed, k=cfg.k)
    g = bpt.Graph(row_ptr, col, w_q31=thr, model=bpt.LT)
    s = g.sample(cfg.theta, colors=64, seed=cfg.seed, sparse=True)
    check_full(bpt, s, ref, cfg.theta)
    off, mem = s.extract(77, 300)
    o0 = ref["offsets"]
    assert np.array_equal(mem, ref["members"][o0[77]:o0[377]])
    occ = np.bincount(ref["members"].astype(np.int64), minlength=cfg.n)
    assert np.array_equal(s.occurrences()[:cfg.n], occ)
    seeds, gains, sigma = s.select_seeds(cfg.k)
    assert np.array_equal(seeds, ref["seeds"]) and np.array_equal(gains, ref["gains"])
    assert sigma == oracle.sigma_hat(cfg.n, int(ref["gains"].sum()), cfg.theta)
    info = s.info
    assert info["members"] == info["e_phys"] == int(ref["sizes"].sum())
    assert info["store_bytes"] < (cfg.theta // 64 + 1) * cfg.n * 8 // 4  # lists, not the bitmap
    seeds2, gains2, _ = s.select_seeds(cfg.k)  # the selection does not mutate the store
    assert np.array_equal(seeds2, seeds) and np.array_equal(gains2, gains)
    s.close()


@pytest.mark.parametrize("shape", ["scaled", "skewed"])
def test_lt_sparse_store_row_sums_off_one(bpt, shape):
    """The sparse walks' in-edge pick guesses the position from r / 2^31 and loads one window of
    8 records; row sums well below 2^31 ("scaled": thresholds x 0.37, so ~63% of picks choose no
    edge and the guess lands left of the answer) or weights piled on the last in-edge
    ("skewed": most of each row's mass on its first in-edge, so the guess lands right of the answer) exercise both continuations of the search. Sizes,
    digests and seeds stay identical to the oracle."""
    cfg = graphgen.scaled(graphgen.CONFIGS["C3"], 1 << 13, theta=2048 + 17)
    row_ptr, col, thr = graphgen.make_graph(cfg)
    thr = thr.astype(np.uint64)
    if shape == "scaled":
        thr = (thr * 37) // 100
    else:  # reverse rows keep forward-position order: the first forward edge into v heads v's row
        dst, first = np.unique(col.astype(np.int64), return_index=True)
        thr = thr // 8
        sums = np.bincount(col.astype(np.int64), weights=thr.astype(np.float64), minlength=cfg.n)
        room = np.floor(Q31 - sums[dst]).astype(np.int64) - 64
        thr[first] += np.maximum(room, 0).astype(np.uint64)
    thr = thr.astype(np.uint32)
    ref = oracle_all(row_ptr, col, thr, oracle.LT, cfg.theta, cfg.seed, k=cfg.k)
    g = bpt.Graph(row_ptr, col, w_q31=thr, model=bpt.LT)
    s = g.sample(cfg.theta, colors=64, seed=cfg.seed, sparse=True)
    check_full(bpt, s, ref, cfg.theta)
    seeds, gains, _ = s.select_seeds(cfg.k)
    assert np.array_equal(seeds, ref["seeds"]) and np.array_equal(gains, ref["gains"])
    s.close()


def test_lt_long_walks_fall_back_to_dense(bpt):
    """A chain graph (i -> i+1, LT weight 1): the reverse walk from vertex v has v+1 members, so
    walks outgrow the sparse store's per-thread visited set; by default the call falls back to
    the dense store (same sets as the oracle), with BPT_FLAG_SPARSE it fails with ENOMEM."""
    n = 3000
    row_ptr = np.arange(n + 1, dtype=np.uint64)
    row_ptr[n] = n - 1
    col = np.arange(1, n, dtype=np.uint32)
    thr = np.full(n - 1, Q31, np.uint32)
    theta = 192
    g = bpt.Graph(row_ptr, col, w_q31=thr, model=bpt.LT)
    og = oracle.Graph(row_ptr, col, w_q31=thr, model=oracle.LT)
    sizes, digests, _ = og.sample_many(7, np.arange(theta, dtype=np.uint64))
    assert sizes.max() > 1536  # the case this test is about
    s = g.sample(theta, colors=64, seed=7)
    assert np.array_equal(s.sizes(0, theta), sizes) and np.array_equal(s.digests(0, theta), digests)
    assert s.info["store_bytes"] >= (theta // 64) * n * 8  # the dense store
    s.close()
    with pytest.raises(bpt.BptError) as ei:
        g.sample(theta, colors=64, seed=7, sparse=True)
    assert ei.value.code == bpt.BPT_ENOMEM


def test_lt_sparse_walk_table_epochs(bpt):
    """The sparse walks' visited sets live in per-thread global tables tagged with a walk epoch
    (never cleared between walks): theta > the walk launch's thread count (148 x 8 x 256) makes
    every thread walk twice in one call (two epochs), and repeated calls on the same graph reuse
    the tables with fresh epochs. Sizes and digests stay identical to the oracle each time."""
    cfg = graphgen.scaled(graphgen.CONFIGS["C3"], 1 << 11, theta=64)
    row_ptr, col, thr = graphgen.make_graph(cfg)
    g = bpt.Graph(row_ptr, col, w_q31=thr, model=bpt.LT)
    og = oracle.Graph(row_ptr, col, w_q31=thr, model=oracle.LT)
    for theta, seed in [((1 << 19) + 77, 3), (4096, 4), ((1 << 19) + 77, 3)]:
        sizes, digests, _ = og.sample_many(seed, np.arange(theta, dtype=np.uint64))
        s = g.sample(theta, colors=64, seed=seed, sparse=True)
        assert np.array_equal(s.sizes(0, theta), sizes)
        assert np.array_equal(s.digests(0, theta), digests)
        s.close()


def test_lt_ragged_theta_and_ranges(bpt):
    cfg = graphgen.scaled(graphgen.CONFIGS["C3"], 1 << 11, theta=64)
    row_ptr, col, thr = graphgen.make_graph(cfg)
    g = bpt.Graph(row_ptr, col, w_q31=thr, model=bpt.LT)
    for theta in (1, 63, 65, 200):
        ref = oracle_all(row_ptr, col, thr, oracle.LT, theta, 5)
        s = g.sample(theta, colors=64, seed=5)
        check_full(bpt, s, ref, theta)
        for first, count in [(0, 1), (theta - 1, 1), (theta // 3, theta - theta // 3)]:
            off, mem = s.extract(first, count)
            a, b = int(ref["offsets"][first]), int(ref["offsets"][first + count])
            assert np.array_equal(mem, ref["members"][a:b])
            assert np.array_equal(off, ref["offsets"][first:first + count + 1] - ref["offsets"][first])
        s.close()


# ------------------------------------------------------------------ C2 / C5 shape, scaled

@pytest.fixture(scope="module")
def c2_small():
    cfg = graphgen.scaled(graphgen.CONFIGS["C2"], 1 << 15, theta=2048)
    row_ptr, col, thr = graphgen.make_graph(cfg)
    ref = oracle_all(row_ptr, col, thr, oracle.IC, cfg.theta, cfg.seed, k=cfg.k)
    return cfg, row_ptr, col, thr, ref


def test_c2_shape_parity_and_colour_sweep(bpt, c2_small):
    cfg, row_ptr, col, thr, ref = c2_small
    g = bpt.Graph(row_ptr, col, w_q31=thr)
    prev = None
    for colors in (1, 8, 32, 64):  # C5: fused vs unfused ablation, identical RRR sets
        s = g.sample(cfg.theta, colors=colors, seed=cfg.seed)
        check_full(bpt, s, ref, cfg.theta)
        seeds, gains, sigma = s.select_seeds(cfg.k)
        assert np.array_equal(seeds, ref["seeds"]) and np.array_equal(gains, ref["gains"])
        info = s.info
        assert info["e_logical"] == int(ref["elog"].sum())
        if colors == 1:
            assert info["e_phys"] == info["e_logical"]
        if prev is not None:
            assert info["e_phys"] <= prev  # larger groups fuse more (Theorem 1 per group)
        prev = info["e_phys"]


# ------------------------------------------------------------------ full-size configs (bench launch config)

@pytest.mark.slow
def test_c2_full_size_sampled_parity(bpt):
    """BASELINE configs[1] at full size in bench.py's launch configuration: exact per-sample
    sizes/digests/lists on a strided subset (all of blocks 0 and G-1), plus invariants."""
    cfg = graphgen.CONFIGS["C2"]
    row_ptr, col, thr = graphgen.make_graph(cfg)
    g = bpt.Graph(row_ptr, col, w_q31=thr)
    s = g.sample(cfg.theta, colors=64, seed=cfg.seed)
    ids = np.unique(np.concatenate([np.arange(0, cfg.theta, 257), np.arange(64), np.arange(cfg.theta - 64, cfg.theta)]))
    og = oracle.Graph(row_ptr, col, w_q31=thr)
    o_sizes, o_dig, o_elog, o_off, o_mem = og.sample_many(cfg.seed, ids, members=True)
    sizes = s.sizes(0, cfg.theta)
    dig = s.digests(0, cfg.theta)
    assert np.array_equal(sizes[ids], o_sizes)
    assert np.array_equal(dig[ids], o_dig)
    for j in (0, 1, len(ids) // 2, len(ids) - 1):
        off, mem = s.extract(int(ids[j]), 1)
        assert np.array_equal(mem, o_mem[o_off[j]:o_off[j + 1]])
    info = s.info
    assert info["members"] == int(sizes.astype(np.uint64).sum())
    assert info["e_phys"] <= info["e_logical"]
    seeds, gains, sigma = s.select_seeds(cfg.k)
    assert len(set(seeds.tolist())) == cfg.k
    assert list(gains) == sorted(gains, reverse=True)
    assert int(gains.sum()) <= cfg.theta
    assert sigma == cfg.n * int(gains.sum()) / cfg.theta


# ------------------------------------------------------------------ sharding (P-9) and occurrences (P-8)

def test_shard_invariance_and_occurrences(bpt, c2_small):
    """Every W-way shard reproduces its slice of the W=1 run; shard occurrence counts sum to
    the W=1 counts, which equal sum_s 1[v in RR_s] from the oracle's lists (SURVEY P-8, P-9)."""
    cfg, row_ptr, col, thr, ref = c2_small
    g = bpt.Graph(row_ptr, col, w_q31=thr)
    full = g.sample(cfg.theta, seed=cfg.seed)
    occ = full.occurrences()
    assert np.array_equal(occ, np.bincount(ref["members"], minlength=cfg.n).astype(np.uint32))
    for W in (2, 3, 5):
        acc = np.zeros(cfg.n, np.uint64)
        for r in range(W):
            s = g.sample(cfg.theta, seed=cfg.seed, shard=(W, r))
            s0, s1 = graphgen.shard_range(cfg.theta, W, r)
            assert (s.s0, s.s1) == (s0, s1)
            if s1 > s0:
                assert np.array_equal(s.digests(s0, s1 - s0), ref["digests"][s0:s1])
                assert np.array_equal(s.sizes(s0, s1 - s0), ref["sizes"][s0:s1])
            acc += s.occurrences()
        assert np.array_equal(acc, occ.astype(np.uint64))



def test_empty_rank_shard_selection(bpt):
    """A rank that owns no 64-sample block (ceil(theta/64) < W) still runs the selection: its
    count vector is empty and it marks the chosen vertices (a zero-size grid used to
    fail here). theta = 64 over W = 2: shard 0 owns blocks [0, 0) -- empty -- and shard 1 the
    only block, which alone gives the oracle's seeds."""
    cfg = graphgen.CONFIGS["C1"]
    row_ptr, col, thr = graphgen.make_graph(cfg)
    g = bpt.Graph(row_ptr, col, w_q31=thr)
    ref = oracle_all(row_ptr, col, thr, oracle.IC, 64, cfg.seed, k=cfg.k)
    for flags in (0, bpt.FLAG_QUEUE):
        e = g.sample(64, seed=cfg.seed, shard=(2, 0), flags=flags)
        assert e.s0 == e.s1 == 0
        seeds, gains, _ = e.select_seeds(cfg.k)
        assert int(gains.sum()) == 0 and seeds.tolist() == list(range(cfg.k))
        f = g.sample(64, seed=cfg.seed, shard=(2, 1), flags=flags)
        assert (f.s0, f.s1) == (0, 64)
        seeds, gains, _ = f.select_seeds(cfg.k)
        assert np.array_equal(seeds, ref["seeds"]) and np.array_equal(gains, ref["gains"])
    gl = bpt.Graph(row_ptr, col, w_q31=graphgen.weights_lt(cfg.n, col, seed=3), model=bpt.LT)
    s = gl.sample(64, seed=cfg.seed, shard=(2, 0))
    seeds, gains, _ = s.select_seeds(cfg.k)
    assert int(gains.sum()) == 0


# ------------------------------------------------------------------ sorted start vertices

def test_sorted_start_slots(bpt, c2_small):
    """Samples assigned to traversal slots in start order (in-degree descending, start id, sample
    id): RRR sets, sizes, digests, ragged-range extraction, occurrences, seeds and gains
    are identical to the oracle's (coins keyed by sample id, reading C-1); E_phys equals the
    oracle's group work of the sorted groups and is lower than with consecutive groups; per
    rank shard the samples are sorted inside the shard."""
    cfg, row_ptr, col, thr, ref = c2_small
    g = bpt.Graph(row_ptr, col, w_q31=thr)
    srt = g.sample(cfg.theta, seed=cfg.seed)
    uns = g.sample(cfg.theta, seed=cfg.seed, flags=bpt.FLAG_UNSORTED)
    for s in (srt, uns):
        check_full(bpt, s, ref, cfg.theta)
        for first, count in ((5, 300), (cfg.theta - 77, 77), (1000, 1)):
            off, mem = s.extract(first, count)
            o0 = ref["offsets"]
            assert np.array_equal(mem, ref["members"][o0[first]:o0[first + count]])
        seeds, gains, _ = s.select_seeds(cfg.k)
        assert np.array_equal(seeds, ref["seeds"]) and np.array_equal(gains, ref["gains"])
    assert np.array_equal(srt.occurrences(), uns.occurrences())
    order = sorted_slots(row_ptr, col, cfg.n, cfg.theta, cfg.seed)
    B = srt.info["batch_groups"]
    # the default form: one frontier per batch of B blocks = one fused group of 64 B samples
    ws = group_e_phys(ref["g"], cfg.seed, order, 64 * B)
    assert srt.info["e_phys"] == sum(w["e_phys"] for w in ws)
    assert srt.info["e_phys"] < uns.info["e_phys"]
    assert srt.info["e_logical"] == uns.info["e_logical"] == int(ref["elog"].sum())
    rows = srt.level_stats()
    for b, w in enumerate(ws):  # per batch: edge reads, levels and per-level frontier sizes of its group
        r = rows[rows[:, 0] == b]
        assert int(r[:, 4].sum()) == w["e_phys"]
        assert r[:, 2].tolist() == w["frontier"].tolist()
    # one frontier per block (BPT_FLAG_SLOTWISE): 64-sample groups, summed per batch
    sw = g.sample(cfg.theta, seed=cfg.seed, flags=bpt.FLAG_SLOTWISE)
    check_full(bpt, sw, ref, cfg.theta)
    ws64 = group_e_phys(ref["g"], cfg.seed, order, 64)
    assert sw.info["e_phys"] == sum(w["e_phys"] for w in ws64) > srt.info["e_phys"]
    rows = sw.level_stats()
    for b in range(len(ws64) // B):
        assert int(rows[rows[:, 0] == b][:, 4].sum()) == sum(w["e_phys"] for w in ws64[B * b:B * b + B])
    for W, r in ((3, 1), (3, 2)):
        s0, s1 = graphgen.shard_range(cfg.theta, W, r)
        sh = g.sample(cfg.theta, seed=cfg.seed, shard=(W, r))
        assert np.array_equal(sh.digests(s0, s1 - s0), ref["digests"][s0:s1])
        order = sorted_slots(row_ptr, col, cfg.n, s1, cfg.seed, s0=s0)
        Bs = sh.info["batch_groups"]
        assert sh.info["e_phys"] == sum(w["e_phys"] for w in group_e_phys(ref["g"], cfg.seed, order, 64 * Bs))


# ------------------------------------------------------------------ pull expansion

def _level_cols(s):
    """Per-level structure that does not depend on the expansion direction: batch, level,
    discovered, kept entries, push work, (vertex, colour) pairs."""
    return s.level_stats()[:, :6]


@pytest.mark.parametrize("permille", [1, 300, 0])
def test_pull_levels_parity(bpt, c2_small, permille):
    """BPT_FLAG_PULL (direction switching): levels whose push work reaches
    permille/1000 x m are expanded by streaming every forward edge once for all slots of the batch
    (coins keyed by the edge's canonical reverse id). permille = 1 pulls nearly every level,
    300 mixes both directions inside a batch, 0 is the default threshold. RRR sets, sizes, digests,
    lists, seeds, gains, sigma, E_phys and the per-level structure equal the oracle / the push form."""
    cfg, row_ptr, col, thr, ref = c2_small
    g = bpt.Graph(row_ptr, col, w_q31=thr)
    push = g.sample(cfg.theta, seed=cfg.seed, flags=bpt.FLAG_SLOTWISE)  # the pull form keeps one frontier per block
    s = g.sample(cfg.theta, seed=cfg.seed, pull=True, pull_permille=permille)
    check_full(bpt, s, ref, cfg.theta)
    seeds, gains, sigma = s.select_seeds(cfg.k)
    assert np.array_equal(seeds, ref["seeds"]) and np.array_equal(gains, ref["gains"])
    assert sigma == oracle.sigma_hat(cfg.n, int(ref["gains"].sum()), cfg.theta)
    info, pinfo = s.info, push.info
    assert info["e_phys"] == pinfo["e_phys"] and info["e_logical"] == int(ref["elog"].sum())
    assert info["members"] == pinfo["members"]
    assert np.array_equal(_level_cols(s), _level_cols(push))
    assert np.array_equal(s.occurrences(), push.occurrences())
    if permille == 1:  # every level with >= m / 1000 work
        lim = max(1, int(1 / 1000.0 * cfg.m))
        assert info["pull_levels"] == sum(int(r[4]) >= lim for r in push.level_stats())
    if permille in (1, 300):
        assert 0 < info["pull_levels"] and info["pull_edge_reads"] == info["pull_levels"] * cfg.m
    assert pinfo["pull_levels"] == 0
    s.close()
    push.close()


def test_pull_c1_and_ragged(bpt):
    """Pull on C1 (all 1,024 lists; batches of 4, 3 and 1 slots) and ragged theta, unsorted slots
    and the host-driven profile loop: same sets and seeds as the oracle."""
    cfg = graphgen.CONFIGS["C1"]
    row_ptr, col, thr = graphgen.make_graph(cfg)
    g = bpt.Graph(row_ptr, col, w_q31=thr)
    for theta, bg, flags in ((cfg.theta, 0, 0), (3 * 64 + 5, 3, 0), (cfg.theta, 1, bpt.FLAG_UNSORTED),
                             (200, 0, bpt.FLAG_PROFILE)):
        ref = oracle_all(row_ptr, col, thr, oracle.IC, theta, cfg.seed, k=cfg.k)
        s = g.sample(theta, seed=cfg.seed, batch_groups=bg, flags=flags, pull=True, pull_permille=1)
        check_full(bpt, s, ref, theta)
        seeds, gains, _ = s.select_seeds(cfg.k)
        assert np.array_equal(seeds, ref["seeds"]) and np.array_equal(gains, ref["gains"])
        assert s.info["pull_levels"] > 0
        s.close()
