"""Multi-GPU parity (-m gpu, needs >= 2 visible GPUs, skipped otherwise): one process per GPU,
NCCL communicator bootstrapped through torch.distributed (gloo), sample-sharded bpt_sample and
the collective bpt_select_seeds. Seeds, gains and sigma_hat must equal the oracle's on every
rank (integer reductions make the result independent of W)."""
import os
import socket

import numpy as np
import pytest

import graphgen
import oracle

pytestmark = pytest.mark.gpu


def _ngpus():
    try:
        import torch
        return torch.cuda.device_count()
    except Exception:
        return 0


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_main(rank, world, port, cfg_name, n_scaled, theta, q, kw=None):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(rank)
    import paper_2311_10201_b200 as bpt
    cfg = graphgen.CONFIGS[cfg_name]
    if n_scaled:
        cfg = graphgen.scaled(cfg, n_scaled, theta=theta)
    row_ptr, col, thr = graphgen.make_graph(cfg)
    uid = [bpt.Comm.unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    comm = bpt.Comm(world, rank, rank, uid[0])
    kw = dict(kw or {})
    colors = kw.pop("colors", 64)
    model = bpt.IC if cfg.model == "IC" else bpt.LT
    if kw.pop("bcast", False):  # collective load: only rank 0's arrays are read
        g = bpt.Graph(row_ptr if rank == 0 else None, col if rank == 0 else None, w_q31=thr if rank == 0 else None,
                      model=model, comm=comm, n=cfg.n, m=cfg.m, bcast_root=0)
        ref = bpt.Graph(row_ptr, col, w_q31=thr, model=model, comm=comm)
        a, b = g.reverse_csr(), ref.reverse_csr()
        assert all(np.array_equal(x, y) for x, y in zip(a, b))
        ref.close()
    else:
        g = bpt.Graph(row_ptr, col, w_q31=thr, model=model, comm=comm)
    s = g.sample(theta, colors=colors, seed=cfg.seed, **kw)
    sizes = s.sizes(s.s0, s.s1 - s.s0) if s.s1 > s.s0 else np.zeros(0, np.uint32)
    digests = s.digests(s.s0, s.s1 - s.s0) if s.s1 > s.s0 else np.zeros(0, np.uint64)
    seeds, gains, sigma = s.select_seeds(cfg.k)
    q.put((rank, s.s0, s.s1, sizes, digests, seeds, gains, sigma))
    s.close()
    g.close()
    comm.close()
    dist.destroy_process_group()


MODES = {"ic": ("C2", 1 << 14, {}), "ic_wide": ("C2", 1 << 14, {"wide": True}),
         "ic_bcast": ("C2", 1 << 14, {"bcast": True}), "ic_c8": ("C2", 1 << 14, {"colors": 8}),
         "lt": ("C3", 1 << 13, {}), "lt_sparse": ("C3", 1 << 13, {"sparse": True})}


@pytest.mark.skipif(_ngpus() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("mode", list(MODES))
def test_multi_gpu_selection_parity(cuda_required, world, mode):
    if _ngpus() < world:
        pytest.skip(f"needs {world} GPUs")
    import torch.multiprocessing as mp
    name, n_scaled, kw = MODES[mode]
    cfg = graphgen.scaled(graphgen.CONFIGS[name], n_scaled, theta=1024 + 64 * 3)
    theta = cfg.theta
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_rank_main, args=(r, world, port, name, n_scaled, theta, q, kw)) for r in range(world)]
    for p in ps:
        p.start()
    res = sorted((q.get(timeout=600) for _ in range(world)), key=lambda t: t[0])
    for p in ps:
        p.join(timeout=120)
        assert p.exitcode == 0
    row_ptr, col, thr = graphgen.make_graph(cfg)
    g = oracle.Graph(row_ptr, col, w_q31=thr, model=oracle.IC if cfg.model == "IC" else oracle.LT)
    sizes, digests, _, off, mem = g.sample_many(cfg.seed, np.arange(theta, dtype=np.uint64), members=True)
    seeds, gains = oracle.greedy(cfg.n, off, mem, cfg.k)
    sigma = oracle.sigma_hat(cfg.n, int(gains.sum()), theta)
    for rank, s0, s1, sz, dg, sd, gn, sg in res:
        assert (s0, s1) == graphgen.shard_range(theta, world, rank)
        assert np.array_equal(sz, sizes[s0:s1]) and np.array_equal(dg, digests[s0:s1])
        assert np.array_equal(sd, seeds) and np.array_equal(gn, gains) and sg == sigma
