"""World-size-2 gloo tests on CPU (-m "not gpu") for the multi-rank host logic:
64-sample-block sharding and the selection protocol the CUDA path implements with NCCL
(per round: sum-reduce of rank-local occurrence counts, argmax of the packed key
count << 32 | ~v over the rank's vertex shard, max-reduce of the key).
Sampling is by the oracle here; the result must equal the single-process greedy."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import graphgen
import oracle


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, theta, k, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = graphgen.CONFIGS["C1"]
    row_ptr, col, thr = graphgen.make_graph(cfg)
    g = oracle.Graph(row_ptr, col, w_q31=thr)
    s0, s1 = graphgen.shard_range(theta, world, rank)
    ids = np.arange(s0, s1, dtype=np.uint64)
    _, _, _, off, mem = g.sample_many(cfg.seed, ids, threads=2, members=True)
    n = cfg.n
    pad = 64 * world
    n_pad = (n + pad - 1) // pad * pad
    count = np.zeros(n_pad, np.int64)
    np.add.at(count, mem.astype(np.int64), 1)
    covered = np.zeros(len(ids), bool)
    selected = np.zeros(n, bool)
    sets_of = [[] for _ in range(n)]
    for i in range(len(ids)):
        for v in mem[off[i]:off[i + 1]]:
            sets_of[v].append(i)
    seeds, gains = [], []
    shard = n_pad // world
    for _ in range(k):
        tot = torch.from_numpy(count.copy())
        dist.all_reduce(tot)                                   # ReduceScatter emulation
        lo = rank * shard
        best = 0
        for v in range(lo, min(lo + shard, n)):
            if not selected[v]:
                key = (int(tot[v]) << 32) | (~v & 0xFFFFFFFF)
                best = max(best, key)
        kt = torch.tensor([best], dtype=torch.int64)
        dist.all_reduce(kt, op=dist.ReduceOp.MAX)              # AllReduce(max) of the packed key
        key = int(kt.item())
        v = (~key) & 0xFFFFFFFF
        seeds.append(v)
        gains.append(key >> 32)
        selected[v] = True
        for i in sets_of[v]:
            if not covered[i]:
                covered[i] = True
                for u in mem[off[i]:off[i + 1]]:
                    count[u] -= 1
    out_q.put((rank, s0, s1, seeds, gains))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_sharded_selection_protocol_equals_greedy(world):
    theta, k = 640, 8
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, theta, k, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # shards tile [0, theta) in 64-sample blocks
    assert res[0][1] == 0 and res[-1][2] == theta
    assert all(a[2] == b[1] for a, b in zip(res, res[1:]))
    assert all(r[1] % 64 == 0 for r in res)
    # identical seeds on every rank, equal to the single-process greedy
    cfg = graphgen.CONFIGS["C1"]
    row_ptr, col, thr = graphgen.make_graph(cfg)
    g = oracle.Graph(row_ptr, col, w_q31=thr)
    _, _, _, off, mem = g.sample_many(cfg.seed, np.arange(theta, dtype=np.uint64), members=True)
    seeds, gains = oracle.greedy(cfg.n, off, mem, k)
    for r in res:
        assert r[3] == seeds.tolist() and r[4] == gains.tolist()


def test_shard_range_tiles_theta():
    for theta in (1, 63, 64, 65, 1000, 65536):
        for world in (1, 2, 3, 8):
            rs = [graphgen.shard_range(theta, world, r) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == theta
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
            assert all(r[0] % 64 == 0 for r in rs)


def _gather_worker(rank, world, port, theta, k, out_q):
    """Member-list stores (LT): each rank samples its shard, the lists are gathered once
    (sizes, then members, padded to the largest rank and compacted back in rank order) and
    every rank runs the whole greedy locally -- the protocol of k_select.cu gather_lists."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = graphgen.scaled(graphgen.CONFIGS["C3"], 1 << 11, theta=theta)
    row_ptr, col, thr = graphgen.make_graph(cfg)
    g = oracle.Graph(row_ptr, col, w_q31=thr, model=oracle.LT)
    s0, s1 = graphgen.shard_range(theta, world, rank)
    sizes, _, _, off, mem = g.sample_many(cfg.seed, np.arange(s0, s1, dtype=np.uint64), threads=2, members=True)
    hdr = torch.tensor([s1 - s0, len(mem)], dtype=torch.int64)
    hdrs = [torch.zeros(2, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(hdrs, hdr)
    max_n = max(1, max(int(h[0]) for h in hdrs))
    max_t = max(1, max(int(h[1]) for h in hdrs))
    sz = torch.zeros(max_n, dtype=torch.int64)
    sz[: s1 - s0] = torch.from_numpy(sizes.astype(np.int64))
    mm = torch.zeros(max_t, dtype=torch.int64)
    mm[: len(mem)] = torch.from_numpy(mem.astype(np.int64))
    sz_all = [torch.zeros(max_n, dtype=torch.int64) for _ in range(world)]
    mm_all = [torch.zeros(max_t, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(sz_all, sz)
    dist.all_gather(mm_all, mm)
    g_sizes = np.concatenate([sz_all[r][: int(hdrs[r][0])].numpy() for r in range(world)])
    g_mem = np.concatenate([mm_all[r][: int(hdrs[r][1])].numpy() for r in range(world)]).astype(np.uint32)
    g_off = np.concatenate([[0], np.cumsum(g_sizes)]).astype(np.uint64)
    seeds, gains = oracle.greedy(cfg.n, g_off, g_mem, k)
    out_q.put((rank, seeds.tolist(), gains.tolist()))
    dist.destroy_process_group()


def test_gathered_list_selection_equals_greedy():
    world, theta, k = 2, 64 * 9 + 5, 10  # ragged: the ranks own 5 and 5 blocks, the last one partial
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gather_worker, args=(r, world, port, theta, k, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    cfg = graphgen.scaled(graphgen.CONFIGS["C3"], 1 << 11, theta=theta)
    row_ptr, col, thr = graphgen.make_graph(cfg)
    g = oracle.Graph(row_ptr, col, w_q31=thr, model=oracle.LT)
    _, _, _, off, mem = g.sample_many(cfg.seed, np.arange(theta, dtype=np.uint64), members=True)
    seeds, gains = oracle.greedy(cfg.n, off, mem, k)
    for r in res:
        assert r[1] == seeds.tolist() and r[2] == gains.tolist()
