"""Pins for the CPU oracle (-m "not gpu").

Each test ties an oracle function to something other than itself: published
known-answer vectors, the paper's worked example, a library routine (scipy /
networkx), closed forms, brute-force enumeration, or an independent algorithm
(a pure-Python fused level-synchronous traversal that follows Listing 1).
Citations: P:n = PAPER.md line n; C-k = reading k.
"""
import itertools
import json
import math
import os
from fractions import Fraction

import networkx as nx
import numpy as np
import pytest
import scipy.sparse as sp
from scipy.sparse import csgraph

import graphgen
import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden")
Q31 = 1 << 31


def load(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def csr_from_edges(n, edges):
    """edges: list of (u, v, thr) -> forward CSR sorted by (u, v) with the thr aligned."""
    edges = sorted(edges, key=lambda t: (t[0], t[1]))
    row_ptr = np.zeros(n + 1, dtype=np.uint64)
    for u, _, _ in edges:
        row_ptr[u + 1] += 1
    row_ptr = np.cumsum(row_ptr, dtype=np.uint64)
    col = np.array([v for _, v, _ in edges], dtype=np.uint32)
    thr = np.array([t for _, _, t in edges], dtype=np.uint32)
    return row_ptr, col, thr


def fused_level_sync(g_rev, seed, s0, s1, model=oracle.IC):
    """Independent pure-Python fused BPT (Listing 1), level-synchronous
    (P:239). Masks are Python ints. Coins come from the pinned oracle primitives.
    Returns (visited masks, edge reads, per-level frontier dicts)."""
    roff, src, thr = g_rev
    n = len(roff) - 1
    C = s1 - s0
    visited = [0] * n
    frontier = {}
    for c in range(C):
        v = oracle.start_vertex(s0 + c, n, seed)
        frontier[v] = frontier.get(v, 0) | (1 << c)
    levels = []
    reads = 0
    cum = None
    if model == oracle.LT:
        cum = [0] * len(src)
        for v in range(n):
            run = 0
            for e in range(int(roff[v]), int(roff[v + 1])):
                run += int(thr[e])
                cum[e] = run
    while frontier:
        for v, fr in frontier.items():
            visited[v] |= fr
        levels.append(dict(frontier))
        nxt = {}
        for v, fr in frontier.items():
            a, b = int(roff[v]), int(roff[v + 1])
            if model == oracle.IC:
                for e in range(a, b):
                    reads += 1
                    u = int(src[e])
                    fr_u = fr & ~visited[u]
                    for c in range(C):
                        if fr_u >> c & 1 and not oracle.ic_edge_live(s0 + c, e, int(thr[e]), seed):
                            fr_u &= ~(1 << c)
                    if fr_u:
                        nxt[u] = nxt.get(u, 0) | fr_u
            else:
                for c in range(C):
                    if not fr >> c & 1:
                        continue
                    reads += 1
                    r = oracle.lt_draw(s0 + c, v, seed)
                    lo = 0
                    for e in range(a, b):
                        if lo <= r < cum[e]:
                            u = int(src[e])
                            if not visited[u] >> c & 1:
                                nxt[u] = nxt.get(u, 0) | (1 << c)
                            break
                        lo = cum[e]
        frontier = {u: m & ~visited[u] for u, m in nxt.items() if m & ~visited[u]}
    return visited, reads, levels


# ---------------------------------------------------------------- primitives

def test_philox_kat():
    kat = load("philox_kat.json")
    for c0, c1, k, o0, o1 in kat["philox2x32_10"]:
        assert oracle.philox2x32_10(int(c0, 16), int(c1, 16), int(k, 16)) == (int(o0, 16), int(o1, 16))


def test_digest_mix_is_splitmix64():
    kat = load("philox_kat.json")
    for seed, out in kat["splitmix64_first_output"]:
        assert oracle.digest_mix(int(seed)) == int(out)


def test_q31_conversion_closed_form():
    # reading C-5: thr = floor(p * 2^31); f32 0.1 is 0.100000001490116..., so 214748368
    assert oracle.q31_from_f32(0.0) == 0
    assert oracle.q31_from_f32(1.0) == Q31
    assert oracle.q31_from_f32(0.5) == Q31 // 2
    assert oracle.q31_from_f32(np.float32(0.1)) == 214748368
    assert graphgen.THR_P01 == 214748364 == (Q31 // 10)  # floor(0.1 * 2^31) exactly
    for p in np.random.default_rng(0).random(200).astype(np.float32):
        exact = Fraction(float(p)) * Q31
        assert oracle.q31_from_f32(p) == math.floor(exact)


def test_coin_boundaries_and_rate():
    # C-2: thr = 0 never passes, thr = 2^31 always passes, Pr = thr / 2^31
    seed = 99
    for s in range(50):
        for e in range(20):
            assert not oracle.ic_edge_live(s, e, 0, seed)
            assert oracle.ic_edge_live(s, e, Q31, seed)
    thr = int(0.3 * Q31)
    N = 20000
    hits = sum(oracle.ic_edge_live(s, 7, thr, seed) for s in range(N))
    p = thr / Q31
    assert abs(hits - N * p) < 5 * math.sqrt(N * p * (1 - p))


def test_start_vertex_uniform_and_degenerate():
    assert all(oracle.start_vertex(s, 1, 5) == 0 for s in range(100))
    n, N = 10, 50000
    counts = np.bincount([oracle.start_vertex(s, n, 7) for s in range(N)], minlength=n)
    chi2 = float(((counts - N / n) ** 2 / (N / n)).sum())
    assert chi2 < 33.7  # chi-square(9) at alpha = 1e-4
    # 64-bit counter: s and s + 2^32 are distinct draws
    assert any(oracle.start_vertex(s, 1 << 20, 3) != oracle.start_vertex(s + (1 << 32), 1 << 20, 3) for s in range(8))


# ---------------------------------------------------------------- reverse CSR

def test_reverse_csr_matches_scipy_transpose():
    row_ptr, col = graphgen.random_graph(200, 3000, seed=1)
    # simple graph: dedup
    u = np.repeat(np.arange(200), np.diff(row_ptr).astype(np.int64))
    pairs = np.unique(np.stack([u, col.astype(np.int64)], 1), axis=0)
    row_ptr, col, _ = csr_from_edges(200, [(a, b, 0) for a, b in pairs])
    m = col.shape[0]
    w = np.random.default_rng(2).integers(0, Q31 + 1, size=m).astype(np.uint32)
    g = oracle.Graph(row_ptr, col, w_q31=w)
    roff, src, thr = g.reverse_csr()
    A = sp.csr_matrix((np.arange(m) + 1, col.astype(np.int64), row_ptr.astype(np.int64)), shape=(200, 200))
    T = A.T.tocsr()
    T.sort_indices()
    assert np.array_equal(roff, T.indptr)
    assert np.array_equal(src, T.indices)
    assert np.array_equal(thr, w[T.data - 1])


def test_reverse_csr_parallel_edges_keep_forward_order():
    # multigraph: two 0->2 edges (forward positions 0 and 1) then 1->2; ties by forward position (C-4)
    row_ptr = np.array([0, 2, 3, 3], dtype=np.uint64)
    col = np.array([2, 2, 2], dtype=np.uint32)
    w = np.array([10, 20, 30], dtype=np.uint32)
    roff, src, thr = oracle.Graph(row_ptr, col, w_q31=w).reverse_csr()
    assert list(roff) == [0, 0, 0, 3]
    assert list(src) == [0, 0, 1]
    assert list(thr) == [10, 20, 30]


def test_f32_weights_equal_q31_path():
    row_ptr, col = graphgen.random_graph(50, 400, seed=3)
    wf = np.random.default_rng(4).random(col.shape[0]).astype(np.float32)
    wq = np.array([oracle.q31_from_f32(x) for x in wf], dtype=np.uint32)
    a = oracle.Graph(row_ptr, col, w_f32=wf).reverse_csr()
    b = oracle.Graph(row_ptr, col, w_q31=wq).reverse_csr()
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


# ---------------------------------------------------------------- IC sampling pins

def test_p0_every_rrr_set_is_the_start():
    row_ptr, col = graphgen.random_graph(100, 800, seed=5)
    g = oracle.Graph(row_ptr, col, w_q31=np.zeros(col.shape[0], np.uint32))
    for s in range(64):
        mem, lev, _ = g.sample_one(11, s)
        assert list(mem) == [oracle.start_vertex(s, 100, 11)]
        assert list(lev) == [0]


def test_p1_rrr_set_is_reverse_reachability():
    """p = 1: RR(v) = {u : u ~> v} (Def. 2), compared with networkx.ancestors and the BFS
    levels with scipy's unweighted shortest paths on the transpose."""
    n = 300
    row_ptr, col = graphgen.random_graph(n, 700, seed=6)
    g = oracle.Graph(row_ptr, col, w_q31=np.full(col.shape[0], Q31, np.uint32))
    u = np.repeat(np.arange(n), np.diff(row_ptr).astype(np.int64))
    G = nx.DiGraph()
    G.add_nodes_from(range(n))
    G.add_edges_from(zip(u.tolist(), col.tolist()))
    A = sp.csr_matrix((np.ones(len(u)), (u, col.astype(np.int64))), shape=(n, n))
    for s in range(40):
        start = oracle.start_vertex(s, n, 12)
        mem, lev, _ = g.sample_one(12, s)
        assert set(mem.tolist()) == nx.ancestors(G, start) | {start}
        dist = csgraph.shortest_path(A.T.tocsr(), unweighted=True, indices=start)
        assert np.array_equal(lev, dist[mem].astype(np.uint32))


def test_worked_example_fig_fused_bpt():
    """yellow RRR = {4,5,6,7,8}; frontiers of steps (a)-(c) and after."""
    fx = load("fig_fused_example.json")
    n = fx["n"]
    row_ptr, col, thr = csr_from_edges(n, [tuple(e) for e in fx["edges"]])
    g = oracle.Graph(row_ptr, col, w_q31=thr)
    roff, src, _ = g.reverse_csr()
    assert list(roff) == fx["reverse_csr"]["roff"]
    assert list(src) == fx["reverse_csr"]["src"]
    seed = fx["seed"]
    assert [oracle.start_vertex(s, n, seed) for s in range(fx["theta"])] == fx["starts"]
    names = {v: k for k, v in fx["colors"].items()}
    per_level = {}
    for s in range(fx["theta"]):
        mem, lev, _ = g.sample_one(seed, s)
        assert mem.tolist() == fx["rrr"][names[s]]
        for v, L in zip(mem.tolist(), lev.tolist()):
            per_level.setdefault(L, {}).setdefault(str(v), []).append(names[s])
    got = [dict(sorted((k, sorted(v)) for k, v in per_level[L].items())) for L in sorted(per_level)]
    want = [dict(sorted((k, sorted(v)) for k, v in f.items())) for f in fx["frontiers"]]
    assert got == want
    assert fx["rrr"]["yellow"] == [4, 5, 6, 7, 8]
    # the independent fused simulation agrees level by level
    vis, _, levels = fused_level_sync((roff, src, g.reverse_csr()[2]), seed, 0, 4)
    sim = [{str(v): sorted(names[c] for c in range(4) if m >> c & 1) for v, m in lv.items()} for lv in levels]
    assert [dict(sorted(x.items())) for x in sim] == want
    w = g.group_work(seed, 0, 4)
    assert w["levels"] == 5 and list(w["frontier"]) == [3, 2, 4, 1, 3]


@pytest.mark.parametrize("trial", range(12))
def test_fused_equals_unfused_and_theorem1(trial):
    """Listing 1 fused (independent Python) == one-at-a-time BFS (oracle) per colour;
    E_phys / levels / frontier sizes as the oracle predicts; Theorem 1."""
    rng = np.random.default_rng(100 + trial)
    n = int(rng.integers(5, 60))
    m = int(rng.integers(n, 6 * n))
    row_ptr, col = graphgen.random_graph(n, m, seed=200 + trial, self_loops=bool(trial % 3 == 0))
    mode = trial % 4
    if mode == 0:
        thr = rng.integers(0, Q31 + 1, size=col.shape[0]).astype(np.uint32)
    elif mode == 1:
        thr = np.full(col.shape[0], Q31 // 2, np.uint32)
    elif mode == 2:
        thr = rng.choice([0, Q31 // 4, Q31], size=col.shape[0]).astype(np.uint32)
    else:
        thr = np.full(col.shape[0], Q31, np.uint32)
    g = oracle.Graph(row_ptr, col, w_q31=thr)
    rev = g.reverse_csr()
    seed = 1000 + trial
    for C in (1, 8, 64, 128):  # 128: the wide-fusion groups (two 64-sample blocks)
        for s0 in range(0, 128, C):
            s1 = s0 + C
            vis, reads, levels = fused_level_sync(rev, seed, s0, s1)
            w = g.group_work(seed, s0, s1)
            assert w["e_phys"] == reads
            assert w["levels"] == len(levels)
            assert list(w["frontier"]) == [len(lv) for lv in levels]
            assert w["e_phys"] <= w["e_logical"]
            if C == 1:
                assert w["e_phys"] == w["e_logical"]
            for c in range(C):
                mem, _, _ = g.sample_one(seed, s0 + c)
                assert [v for v in range(n) if vis[v] >> c & 1] == mem.tolist()
            if C >= 64:
                break


@pytest.mark.parametrize("trial", range(6))
def test_lt_fused_equals_walk(trial):
    rng = np.random.default_rng(300 + trial)
    n = int(rng.integers(5, 40))
    row_ptr, col = graphgen.random_graph(n, int(rng.integers(n, 5 * n)), seed=400 + trial)
    thr = graphgen.weights_lt(n, col, seed=trial)
    g = oracle.Graph(row_ptr, col, w_q31=thr, model=oracle.LT)
    rev = g.reverse_csr()
    seed = 77 + trial
    for s0 in (0, 64):
        vis, reads, levels = fused_level_sync(rev, seed, s0, s0 + 64, model=oracle.LT)
        w = g.group_work(seed, s0, s0 + 64)
        total = 0
        for c in range(64):
            mem, lev, el = g.sample_one(seed, s0 + c)
            assert [v for v in range(n) if vis[v] >> c & 1] == mem.tolist()
            # a reverse walk: exactly one vertex per level 0..|RR|-1
            assert sorted(lev.tolist()) == list(range(len(mem)))
            total += len(mem)
        assert w["e_phys"] == total == reads
        assert w["levels"] == len(levels)


def test_lt_chain_and_stop_probability():
    # chain 0 -> 1 -> ... -> 5, every vertex's single in-edge has weight 1 => RR(5) = all
    n = 6
    row_ptr, col, thr = csr_from_edges(n, [(i, i + 1, Q31) for i in range(5)])
    g = oracle.Graph(row_ptr, col, w_q31=thr, model=oracle.LT)
    for s in range(200):
        mem, lev, _ = g.sample_one(3, s)
        start = oracle.start_vertex(s, n, 3)
        assert mem.tolist() == list(range(start + 1))
    g0 = oracle.Graph(row_ptr, col, w_q31=np.zeros_like(thr), model=oracle.LT)
    for s in range(50):
        assert g0.sample_one(3, s)[0].tolist() == [oracle.start_vertex(s, n, 3)]


# ---------------------------------------------------------------- brute force (P-6)

def _reach_sets(n, edges):
    """reach[v] = set of u with a path u ~> v using `edges` (list of (u, v))."""
    radj = [[] for _ in range(n)]
    for a, b in edges:
        radj[b].append(a)
    out = []
    for v in range(n):
        seen = {v}
        st = [v]
        while st:
            x = st.pop()
            for y in radj[x]:
                if y not in seen:
                    seen.add(y)
                    st.append(y)
        out.append(seen)
    return out


def _exact_ic(n, edges_thr):
    """Exact Pr[u in RR(v)] by enumerating all 2^m live-edge graphs (Def. 2)."""
    m = len(edges_thr)
    P = [[Fraction(0)] * n for _ in range(n)]
    for live in itertools.product((0, 1), repeat=m):
        pr = Fraction(1)
        es = []
        for bit, (a, b, t) in zip(live, edges_thr):
            p = Fraction(t, Q31)
            pr *= p if bit else 1 - p
            if bit:
                es.append((a, b))
        if pr == 0:
            continue
        for v, R in enumerate(_reach_sets(n, es)):
            for u in R:
                P[v][u] += pr
    return P


def _exact_lt(n, edges_thr):
    """Exact Pr[u in RR(v)] under LT live-edge semantics (C-6): every vertex keeps at
    most one in-edge j with probability thr_j / 2^31 (none with the leftover mass)."""
    inn = [[] for _ in range(n)]
    for a, b, t in edges_thr:
        inn[b].append((a, t))
    choices = []
    for v in range(n):
        opts = [(a, Fraction(t, Q31)) for a, t in inn[v]]
        rest = 1 - sum((p for _, p in opts), Fraction(0))
        opts.append((None, rest))
        choices.append(opts)
    P = [[Fraction(0)] * n for _ in range(n)]
    for combo in itertools.product(*choices):
        pr = Fraction(1)
        es = []
        for v, (a, p) in enumerate(combo):
            pr *= p
            if a is not None:
                es.append((a, v))
        if pr == 0:
            continue
        for v, R in enumerate(_reach_sets(n, es)):
            for u in R:
                P[v][u] += pr
    return P


@pytest.mark.parametrize("model", [oracle.IC, oracle.LT])
def test_bruteforce_live_edge_enumeration(model):
    n = 6
    rng = np.random.default_rng(7)
    pairs = set()
    while len(pairs) < 11:
        a, b = (int(x) for x in rng.integers(0, n, 2))
        if a != b:
            pairs.add((a, b))
    pairs = sorted(pairs)
    if model == oracle.IC:
        thr_vals = [0, Q31, Q31 // 3, Q31 // 2, 3 * (Q31 // 4)]
        et = [(a, b, thr_vals[i % len(thr_vals)]) for i, (a, b) in enumerate(pairs)]
    else:
        row_ptr, col, _ = csr_from_edges(n, [(a, b, 0) for a, b in pairs])
        w = graphgen.weights_lt(n, col, seed=5)
        w[0] = 0
        et = [(a, b, int(t)) for (a, b), t in zip(pairs, w)]
    row_ptr, col, thr = csr_from_edges(n, et)
    g = oracle.Graph(row_ptr, col, w_q31=thr, model=model)
    exact = _exact_ic(n, et) if model == oracle.IC else _exact_lt(n, et)
    theta = 1 << 16
    seed = 4242
    ids = np.arange(theta, dtype=np.uint64)
    sizes, _, _, offsets, mem = g.sample_many(seed, ids, members=True)
    starts = np.array([oracle.start_vertex(s, n, seed) for s in range(theta)])
    hit = np.zeros((n, n))
    for s in range(theta):
        for u in mem[offsets[s]:offsets[s + 1]]:
            hit[starts[s], u] += 1
    for v in range(n):
        Nv = int((starts == v).sum())
        for u in range(n):
            p = float(exact[v][u])
            if p in (0.0, 1.0):
                assert hit[v, u] == p * Nv
            else:
                z = (hit[v, u] - Nv * p) / math.sqrt(Nv * p * (1 - p))
                assert abs(z) < 5, (v, u, z)
    # RIS identity: sigma(S) = n * Pr[S intersects RR(random v)]; exact vs estimate
    S = {0, 3}
    exact_sigma = sum(1 - _prob_none(exact, v, S, n, et, model) for v in range(n))
    covered = sum(1 for s in range(theta) if S & set(mem[offsets[s]:offsets[s + 1]].tolist()))
    est = oracle.sigma_hat(n, covered, theta)
    p = float(exact_sigma) / n
    assert abs(est - float(exact_sigma)) < 5 * n * math.sqrt(p * (1 - p) / theta)


def _prob_none(exact_unused, v, S, n, et, model):
    """Pr[no vertex of S reaches v] computed exactly by enumeration (joint event)."""
    total = Fraction(0)
    if model == oracle.IC:
        for live in itertools.product((0, 1), repeat=len(et)):
            pr = Fraction(1)
            es = []
            for bit, (a, b, t) in zip(live, et):
                p = Fraction(t, Q31)
                pr *= p if bit else 1 - p
                if bit:
                    es.append((a, b))
            if pr and not (_reach_sets(n, es)[v] & S):
                total += pr
    else:
        inn = [[] for _ in range(n)]
        for a, b, t in et:
            inn[b].append((a, t))
        choices = []
        for x in range(n):
            opts = [(a, Fraction(t, Q31)) for a, t in inn[x]]
            opts.append((None, 1 - sum((p for _, p in opts), Fraction(0))))
            choices.append(opts)
        for combo in itertools.product(*choices):
            pr = Fraction(1)
            es = []
            for x, (a, p) in enumerate(combo):
                pr *= p
                if a is not None:
                    es.append((a, x))
            if pr and not (_reach_sets(n, es)[v] & S):
                total += pr
    return total


def test_sample_many_thread_independent_and_consistent():
    cfg = graphgen.CONFIGS["C1"]
    row_ptr, col, thr = graphgen.make_graph(cfg)
    g = oracle.Graph(row_ptr, col, w_q31=thr)
    ids = np.arange(300, dtype=np.uint64)
    a = g.sample_many(cfg.seed, ids, threads=1, members=True)
    b = g.sample_many(cfg.seed, ids, threads=4, members=True)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)
    sizes, digests, elog, offsets, mem = a
    indeg = np.diff(g.reverse_csr()[0]).astype(np.uint64)
    for i in range(0, 300, 17):
        lst = mem[offsets[i]:offsets[i + 1]]
        assert sizes[i] == len(lst)
        assert int(digests[i]) == sum(oracle.digest_mix(int(v)) for v in lst) % (1 << 64)
        assert int(elog[i]) == int(indeg[lst].sum())
        one, _, _ = g.sample_one(cfg.seed, i)
        assert np.array_equal(one, lst)


# ---------------------------------------------------------------- greedy (P-7)

def _sets_to_csr(sets):
    off = np.zeros(len(sets) + 1, dtype=np.uint64)
    off[1:] = np.cumsum([len(s) for s in sets])
    mem = np.array([v for s in sets for v in sorted(s)], dtype=np.uint32)
    return off, mem


def test_greedy_tie_break_example():
    # {{0,1},{1,2},{2,3}}, k=2 -> [1, 2], covered 3 (smallest id on ties, C-11)
    off, mem = _sets_to_csr([{0, 1}, {1, 2}, {2, 3}])
    for lazy in (False, True):
        seeds, gains = oracle.greedy(4, off, mem, 2, lazy=lazy)
        assert seeds.tolist() == [1, 2] and gains.tolist() == [2, 1]


def test_greedy_exhaustion_picks_smallest_unselected():
    off, mem = _sets_to_csr([{3}, {3}, {5}])
    for lazy in (False, True):
        seeds, gains = oracle.greedy(7, off, mem, 5, lazy=lazy)
        assert seeds.tolist() == [3, 5, 0, 1, 2]
        assert gains.tolist() == [2, 1, 0, 0, 0]


@pytest.mark.parametrize("trial", range(60))
def test_greedy_bruteforce_bound_and_lazy_equals_naive(trial):
    rng = np.random.default_rng(trial)
    n = int(rng.integers(2, 16))
    nsets = int(rng.integers(1, 13))
    k = int(rng.integers(1, min(3, n) + 1))
    sets = [set(rng.choice(n, size=int(rng.integers(1, n + 1)), replace=False).tolist()) for _ in range(nsets)]
    off, mem = _sets_to_csr(sets)
    s_naive, g_naive = oracle.greedy(n, off, mem, k, lazy=False)
    s_lazy, g_lazy = oracle.greedy(n, off, mem, k, lazy=True)
    assert s_naive.tolist() == s_lazy.tolist() and g_naive.tolist() == g_lazy.tolist()
    cov = lambda S: sum(1 for t in sets if t & set(S))
    opt = max(cov(S) for S in itertools.combinations(range(n), k))
    got = int(g_naive.sum())
    assert got == cov(s_naive.tolist())
    assert got >= (1 - 1 / math.e) * opt - 1e-9
    # k = 1 greedy is exact: the first pick maximises coverage, smallest id on ties
    best1 = max(range(n), key=lambda v: (cov([v]), -v))
    assert int(s_naive[0]) == best1
    assert list(g_naive) == sorted(g_naive, reverse=True)  # submodular: gains non-increasing


def test_sigma_hat_closed_forms():
    assert oracle.sigma_hat(1000, 64, 64) == 1000.0
    assert oracle.sigma_hat(1000, 0, 64) == 0.0
    assert oracle.sigma_hat(4847571, 12345, 65536) == 4847571 * 12345 / 65536


# ---------------------------------------------------------------- coin keying, independent (C-1, C-3, C-6)

def _py_philox2x32_10(x0, x1, key):
    """Philox2x32-10 written from Salmon et al. (SC'11) in plain Python integers -- shares no
    code with oracle.c; pinned by the Random123 KAT vectors below before it is used."""
    M, W = 0xD256D193, 0x9E3779B9
    for r in range(10):
        if r:
            key = (key + W) & 0xFFFFFFFF
        p = M * x0
        x0, x1 = ((p >> 32) ^ key ^ x1) & 0xFFFFFFFF, p & 0xFFFFFFFF
    return x0, x1


def _py_key(seed, tag):
    return _py_philox2x32_10(seed & 0xFFFFFFFF, seed >> 32, tag)[0]


def test_python_philox_kat():
    for c0, c1, k, o0, o1 in load("philox_kat.json")["philox2x32_10"]:
        assert _py_philox2x32_10(int(c0, 16), int(c1, 16), int(k, 16)) == (int(o0, 16), int(o1, 16))


def _py_lt_walk(row_ptr, col, thr, seed, s, ctr_order="v_s"):
    """Reverse LT walk of sample s (reading C-6) with coins keyed per reading C-1:
    r = Philox(ctr = {v, lo32(s)}, key = k_LT)[0] >> 1; start per reading C-3. The reverse rows
    are built here from the forward CSR in forward-position order (reading C-4)."""
    n = len(row_ptr) - 1
    rows = [[] for _ in range(n)]
    for u in range(n):
        for ef in range(int(row_ptr[u]), int(row_ptr[u + 1])):
            rows[int(col[ef])].append((u, int(thr[ef])))
    k_lt, k_st = _py_key(seed, oracle.TAG_LT), _py_key(seed, oracle.TAG_START)
    w0, w1 = _py_philox2x32_10(s & 0xFFFFFFFF, s >> 32, k_st)
    v = ((w1 << 32 | w0) * n) >> 64
    seen = [v]
    while True:
        ctr = (v, s & 0xFFFFFFFF) if ctr_order == "v_s" else (s & 0xFFFFFFFF, v)
        r = _py_philox2x32_10(ctr[0], ctr[1], k_lt)[0] >> 1
        lo, nxt = 0, None
        for u, t in rows[v]:
            if lo <= r < lo + t:
                nxt = u
                break
            lo += t
        if nxt is None or nxt in seen:
            return sorted(seen)
        seen.append(nxt)
        v = nxt


@pytest.mark.parametrize("trial", range(4))
def test_lt_coin_keying_independent(trial):
    """The oracle's LT walks equal walks computed with an independent Philox and the coin key
    of reading C-1 (ctr = {v, lo32(s)}, key = k_LT, TAG_LT = 0x4C540001); the swapped counter
    order gives different walks, so the check discriminates the keying, not just the law."""
    rng = np.random.default_rng(900 + trial)
    n = int(rng.integers(20, 60))
    row_ptr, col = graphgen.random_graph(n, int(rng.integers(2 * n, 6 * n)), seed=910 + trial)
    thr = graphgen.weights_lt(n, col, seed=920 + trial)
    g = oracle.Graph(row_ptr, col, w_q31=thr, model=oracle.LT)
    seed = 0x1234_5678_9ABC + trial
    differs = 0
    for s in range(120):
        mem = g.sample_one(seed, s)[0].tolist()
        assert mem == _py_lt_walk(row_ptr, col, thr, seed, s)
        differs += mem != _py_lt_walk(row_ptr, col, thr, seed, s, ctr_order="s_v")
    assert differs > 10


def test_ic_coin_keying_independent():
    """IC coins of the oracle equal Philox(ctr = {e, lo32(s)}, key = k_IC)[0] >> 1 < thr computed
    with the independent Philox (reading C-1/C-2), for random (s, e, thr) incl. 64-bit seeds."""
    rng = np.random.default_rng(5)
    for _ in range(400):
        seed = int(rng.integers(0, 1 << 63))
        s, e, t = int(rng.integers(0, 1 << 32)), int(rng.integers(0, 1 << 32)), int(rng.integers(0, Q31 + 1))
        want = (_py_philox2x32_10(e, s & 0xFFFFFFFF, _py_key(seed, oracle.TAG_IC))[0] >> 1) < t
        assert oracle.ic_edge_live(s, e, t, seed) == want


# ---------------------------------------------------------------- full-size store

@pytest.mark.parametrize("which", ["C1", "C2s"])
def test_store_equals_lists_group_work_and_greedy(which):
    """The list / bitset RRR store gives the same sizes, digests, member lists, E_logical, per-group
    E_phys / levels / frontier sizes (level-mask counting vs or_group_work's sort) and greedy
    seeds / gains (count-maintaining greedy vs the naive recount and CELF) -- whichever
    representation each sample takes (all lists, all bitsets, the n/32 default)."""
    cfg = graphgen.CONFIGS["C1"] if which == "C1" else graphgen.scaled(graphgen.CONFIGS["C2"], 1 << 13, theta=640 + 17)
    row_ptr, col, thr = graphgen.make_graph(cfg)
    g = oracle.Graph(row_ptr, col, w_q31=thr)
    theta = cfg.theta
    sz, dg, el, off, mem = g.sample_many(cfg.seed, np.arange(theta, dtype=np.uint64), members=True)
    ref_seeds, ref_gains = oracle.greedy(cfg.n, off, mem, cfg.k)
    lazy_seeds, lazy_gains = oracle.greedy(cfg.n, off, mem, cfg.k, lazy=True)
    assert np.array_equal(ref_seeds, lazy_seeds) and np.array_equal(ref_gains, lazy_gains)
    works = [g.group_work(cfg.seed, a, min(a + 64, theta)) for a in range(0, theta, 64)]
    for list_max in (0, 1, 1 << 30):
        S = oracle.Store(g, cfg.seed, 0, theta, 64, list_max=list_max)
        assert np.array_equal(S.sizes, sz) and np.array_equal(S.digests, dg) and S.e_logical == int(el.sum())
        for i in (0, 1, theta // 2, theta - 1):
            assert np.array_equal(S.members(i), mem[off[i]:off[i + 1]])
        assert S.e_phys.tolist() == [w["e_phys"] for w in works]
        assert S.levels.tolist() == [w["levels"] for w in works]
        for gi, w in enumerate(works):
            assert S.frontier[gi, :w["levels"]].tolist() == w["frontier"].tolist()
            assert not S.frontier[gi, w["levels"]:].any()
        seeds, gains = S.greedy(cfg.k)
        assert np.array_equal(seeds, ref_seeds) and np.array_equal(gains, ref_gains)
    S = oracle.Store(g, cfg.seed, 0, theta, 64)
    seeds, gains = S.greedy(cfg.n)  # exhaustion: every set covered, then smallest unselected ids
    r_seeds, r_gains = oracle.greedy(cfg.n, off, mem, cfg.n)
    assert np.array_equal(seeds, r_seeds) and np.array_equal(gains, r_gains)


def test_group_work_of_arbitrary_groups():
    """or_group_work_ids (groups of non-consecutive samples) equals the
    contiguous version on contiguous ids, and the store built in a permuted order reproduces it
    group by group (level-mask counting vs the sort), with the per-id sizes and digests."""
    cfg = graphgen.CONFIGS["C1"]
    row_ptr, col, thr = graphgen.make_graph(cfg)
    g = oracle.Graph(row_ptr, col, w_q31=thr)
    for a in (0, 64, 960):
        x, y = g.group_work_ids(cfg.seed, np.arange(a, a + 64)), g.group_work(cfg.seed, a, a + 64)
        assert (x["e_phys"], x["e_logical"], x["levels"]) == (y["e_phys"], y["e_logical"], y["levels"])
        assert np.array_equal(x["frontier"], y["frontier"])
    ids = np.random.default_rng(2).permutation(cfg.theta)
    S = oracle.Store(g, cfg.seed, 0, cfg.theta, 64, ids=ids, keep=False)
    works = [g.group_work_ids(cfg.seed, ids[i:i + 64]) for i in range(0, cfg.theta, 64)]
    assert S.e_phys.tolist() == [w["e_phys"] for w in works]
    assert S.levels.tolist() == [w["levels"] for w in works]
    sz, dg, _ = g.sample_many(cfg.seed, ids.astype(np.uint64))
    assert np.array_equal(S.sizes, sz) and np.array_equal(S.digests, dg)
    # a union bound the sort can only tighten: grouping never reads more than the samples alone
    assert sum(w["e_phys"] for w in works) <= sum(w["e_logical"] for w in works)
