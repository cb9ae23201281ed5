"""Seeded synthetic inputs for the fused-BPT hot path (test and bench infrastructure).

Serves BOTH the CPU oracle (`oracle/`) and the CUDA path (`paper_2311_10201_b200`).
It holds none of the method's arithmetic: it only emits a forward CSR graph and
Q1.31 edge thresholds (p = thr / 2^31), and the per-config
parameters of BASELINE.json's five configs. Recipe: DESIGN.md "Input recipe".

Graphs are Graph500-style R-MAT (initiator 0.57/0.19/0.19/0.05), deduplicated,
self-loop free, label-permuted, rows sorted (graphgen/rmat.c).
"""
from __future__ import annotations

import ctypes
import functools
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "rmat.c")
_LIB = os.path.join(_HERE, "_rmat.so")

# C1: p = 0.1 exactly as a rational threshold: floor(0.1 * 2^31) = 214,748,364 (SURVEY C-5).
THR_P01 = 214748364
Q31_ONE = 1 << 31
SEED_BASE = 0x5EED0000


def build_lib(force: bool = False) -> str:
    """Compile graphgen/_rmat.so with gcc + OpenMP (no GPU needed)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + ".tmp%d" % os.getpid()
        subprocess.check_call(["gcc", "-O3", "-march=x86-64-v2", "-fopenmp", "-shared", "-fPIC",
                               "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


@functools.lru_cache(maxsize=1)
def _lib():
    lib = ctypes.CDLL(build_lib())
    u64, p = ctypes.c_uint64, ctypes.c_void_p
    lib.gg_rmat.argtypes = [u64, u64, u64, p, p]
    lib.gg_rmat.restype = ctypes.c_int
    lib.gg_weights_uniform.argtypes = [u64, u64, p]
    lib.gg_weights_uniform.restype = None
    lib.gg_weights_lt.argtypes = [u64, u64, p, u64, p]
    lib.gg_weights_lt.restype = ctypes.c_int
    return lib


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def rmat(n: int, m: int, seed: int) -> tuple[np.ndarray, np.ndarray]:
    """Forward CSR (row_ptr u64[n+1], col u32[m]) of an R-MAT graph with m unique edges."""
    row_ptr = np.empty(n + 1, dtype=np.uint64)
    col = np.empty(m, dtype=np.uint32)
    rc = _lib().gg_rmat(n, m, seed, _ptr(row_ptr), _ptr(col))
    if rc != 0:
        raise RuntimeError(f"gg_rmat(n={n}, m={m}) failed with code {rc}")
    return row_ptr, col


def weights_uniform(m: int, seed: int) -> np.ndarray:
    """IC weights: Q1.31 thresholds uniform in [0, 2^31), i.e. p ~ U[0,1)."""
    thr = np.empty(m, dtype=np.uint32)
    _lib().gg_weights_uniform(m, seed, _ptr(thr))
    return thr


def weights_const(m: int, thr: int) -> np.ndarray:
    return np.full(m, thr, dtype=np.uint32)


def weights_lt(n: int, col: np.ndarray, seed: int) -> np.ndarray:
    """LT weights: per-destination normalised uniform, sum over in-edges <= 2^31 (SURVEY C-6)."""
    m = col.shape[0]
    thr = np.empty(m, dtype=np.uint32)
    rc = _lib().gg_weights_lt(n, m, _ptr(np.ascontiguousarray(col)), seed, _ptr(thr))
    if rc != 0:
        raise RuntimeError("gg_weights_lt failed")
    return thr


@dataclass(frozen=True)
class Config:
    name: str
    n: int
    m: int
    model: str            # "IC" | "LT"
    weights: str          # "const01" | "uniform" | "lt"
    colors: int
    theta: int
    k: int
    graph_seed: int
    seed: int             # sampling seed

    def describe(self) -> str:
        return (f"{self.name}: R-MAT n={self.n} m={self.m} {self.model} weights={self.weights} "
                f"C={self.colors} theta={self.theta} k={self.k}")


# BASELINE.json configs. graph/weight seed = config index; C5 reuses C2's graph.
CONFIGS = {
    "C1": Config("C1", 1024, 16384, "IC", "const01", 64, 1024, 8, 1, SEED_BASE + 1),
    "C2": Config("C2", 4847571, 68993773, "IC", "uniform", 64, 65536, 50, 2, SEED_BASE + 2),
    "C3": Config("C3", 3072441, 117185083, "LT", "lt", 64, 262144, 100, 3, SEED_BASE + 3),
    "C4": Config("C4", 65608366, 1806067135, "IC", "uniform", 64, 131072, 50, 4, SEED_BASE + 4),
    "C5": Config("C5", 4847571, 68993773, "IC", "uniform", 64, 65536, 50, 2, SEED_BASE + 5),
}


def scaled(cfg: Config, n: int, theta: int | None = None, name: str | None = None) -> Config:
    """Same shape (edge factor, model, weights) at a smaller vertex count."""
    m = int(round(cfg.m / cfg.n * n))
    return Config(name or f"{cfg.name}@n{n}", n, m, cfg.model, cfg.weights, cfg.colors,
                  theta if theta is not None else cfg.theta, cfg.k, cfg.graph_seed, cfg.seed)


@functools.lru_cache(maxsize=4)
def make_graph(cfg: Config) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
    """(row_ptr u64[n+1], col u32[m], thr u32[m]) for a config; cached per process."""
    row_ptr, col = rmat(cfg.n, cfg.m, cfg.graph_seed)
    if cfg.weights == "const01":
        thr = weights_const(cfg.m, THR_P01)
    elif cfg.weights == "uniform":
        thr = weights_uniform(cfg.m, cfg.graph_seed)
    elif cfg.weights == "lt":
        thr = weights_lt(cfg.n, col, cfg.graph_seed)
    else:
        raise ValueError(cfg.weights)
    for a in (row_ptr, col, thr):
        a.setflags(write=False)
    return row_ptr, col, thr


def random_graph(n: int, m: int, seed: int, self_loops: bool = False) -> tuple[np.ndarray, np.ndarray]:
    """Small uniform random multigraph in forward CSR (tests only; numpy RNG)."""
    rng = np.random.default_rng(seed)
    u = rng.integers(0, n, size=m)
    v = rng.integers(0, n, size=m)
    if not self_loops:
        keep = u != v
        u, v = u[keep], v[keep]
    order = np.lexsort((v, u))
    u, v = u[order], v[order]
    row_ptr = np.zeros(n + 1, dtype=np.uint64)
    np.add.at(row_ptr, u + 1, 1)
    row_ptr = np.cumsum(row_ptr, dtype=np.uint64)
    return row_ptr, v.astype(np.uint32)


def shard_range(theta: int, world: int, rank: int) -> tuple[int, int]:
    """Sample range [s0, s1) owned by `rank`: 64-sample blocks split evenly."""
    nb = (theta + 63) // 64
    b0 = rank * nb // world
    b1 = (rank + 1) * nb // world
    return min(64 * b0, theta), min(64 * b1, theta)
