"""CPU oracle for the fused-BPT hot path -- TEST INFRASTRUCTURE ONLY.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py` (its `cpu_baseline` leg and
`--impl reference`) may import this package. The product (`paper_2311_10201_b200`)
never imports it and shares no code with it.

Thin ctypes marshalling over oracle/oracle.c, which holds all the arithmetic, each
function citing the PAPER.md passage / DESIGN.md reading it follows.
"""
from __future__ import annotations

import ctypes
import functools
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "_oracle.so")

IC, LT = 0, 1
_u32, _u64, _p, _i = ctypes.c_uint32, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_int


def build_lib(force: bool = False) -> str:
    """Compile oracle/_oracle.so (plain C, gcc -O2, pthreads)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + ".tmp%d" % os.getpid()
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-shared", "-fPIC", "-pthread", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


@functools.lru_cache(maxsize=1)
def lib():
    L = ctypes.CDLL(build_lib())
    L.or_philox2x32_10.argtypes = [_u32, _u32, _u32, _p]
    L.or_philox2x32_10.restype = None
    L.or_stream_key.argtypes = [_u64, _u32]
    L.or_stream_key.restype = _u32
    L.or_start_vertex.argtypes = [_u64, _u32, _u32]
    L.or_start_vertex.restype = _u32
    L.or_ic_edge_live.argtypes = [_u64, _u32, _u32, _u32]
    L.or_ic_edge_live.restype = _i
    L.or_lt_draw.argtypes = [_u64, _u32, _u32]
    L.or_lt_draw.restype = _u32
    L.or_q31_from_f32.argtypes = [ctypes.c_float]
    L.or_q31_from_f32.restype = _u32
    L.or_digest_mix.argtypes = [_u64]
    L.or_digest_mix.restype = _u64
    L.or_graph_new.argtypes = [_u32, _u64, _p, _p, _p, _p, _i]
    L.or_graph_new.restype = _p
    L.or_graph_free.argtypes = [_p]
    L.or_graph_free.restype = None
    L.or_graph_export.argtypes = [_p, _p, _p, _p]
    L.or_graph_export.restype = None
    L.or_sample_one.argtypes = [_p, _u64, _u64, _p, _p, _p]
    L.or_sample_one.restype = _u32
    L.or_sample_many.argtypes = [_p, _u64, _p, _u64, _i, _p, _p, _p, _p, _p]
    L.or_sample_many.restype = _i
    L.or_group_work.argtypes = [_p, _u64, _u64, _u64, _p, _p, _p, _p, _u32]
    L.or_group_work.restype = _i
    L.or_group_work_ids.argtypes = [_p, _u64, _p, _u64, _p, _p, _p, _p, _u32]
    L.or_group_work_ids.restype = _i
    L.or_greedy.argtypes = [_u32, _u64, _p, _p, _u32, _i, _p, _p]
    L.or_greedy.restype = _i
    L.or_sigma_hat.argtypes = [_u32, _u64, _u64]
    L.or_sigma_hat.restype = ctypes.c_double
    L.or_store_build.argtypes = [_p, _u64, _u64, _u64, _u32, _i, _u32]
    L.or_store_build.restype = _p
    L.or_store_build_ids.argtypes = [_p, _u64, _u64, _p, _u64, _u32, _i, _u32, _i]
    L.or_store_build_ids.restype = _p
    L.or_store_free.argtypes = [_p]
    L.or_store_free.restype = None
    L.or_store_info.argtypes = [_p, _p, _p, _p, _p, _p, _p]
    L.or_store_info.restype = None
    L.or_store_members.argtypes = [_p, _u64, _p]
    L.or_store_members.restype = _u32
    L.or_store_greedy.argtypes = [_p, _u32, _p, _p]
    L.or_store_greedy.restype = _i
    return L


def _ptr(a):
    return None if a is None else a.ctypes.data


def philox2x32_10(x0: int, x1: int, key: int) -> tuple[int, int]:
    out = np.zeros(2, dtype=np.uint32)
    lib().or_philox2x32_10(x0, x1, key, _ptr(out))
    return int(out[0]), int(out[1])


TAG_IC, TAG_LT, TAG_START = 0x49430001, 0x4C540001, 0x53540001


def stream_key(seed: int, tag: int) -> int:
    return lib().or_stream_key(seed, tag)


def start_vertex(s: int, n: int, seed: int) -> int:
    return lib().or_start_vertex(s, n, stream_key(seed, TAG_START))


def ic_edge_live(s: int, e: int, thr: int, seed: int) -> bool:
    return bool(lib().or_ic_edge_live(s, e, thr, stream_key(seed, TAG_IC)))


def lt_draw(s: int, v: int, seed: int) -> int:
    return lib().or_lt_draw(s, v, stream_key(seed, TAG_LT))


def q31_from_f32(p: float) -> int:
    return lib().or_q31_from_f32(p)


def digest_mix(v: int) -> int:
    return lib().or_digest_mix(v)


def default_threads() -> int:
    return max(1, len(os.sched_getaffinity(0)))


class Graph:
    """Oracle's own reverse CSR (stable transpose, reading C-4) of a forward CSR."""

    def __init__(self, row_ptr, col, w_q31=None, w_f32=None, model: int = IC):
        self.row_ptr = np.ascontiguousarray(row_ptr, dtype=np.uint64)
        self.col = np.ascontiguousarray(col, dtype=np.uint32)
        self.n = int(self.row_ptr.shape[0] - 1)
        self.m = int(self.col.shape[0])
        self.model = model
        self._wq = None if w_q31 is None else np.ascontiguousarray(w_q31, dtype=np.uint32)
        self._wf = None if w_f32 is None else np.ascontiguousarray(w_f32, dtype=np.float32)
        assert (self._wq is None) != (self._wf is None)
        h = lib().or_graph_new(self.n, self.m, _ptr(self.row_ptr), _ptr(self.col),
                               _ptr(self._wf), _ptr(self._wq), model)
        if not h:
            raise ValueError("oracle: invalid forward CSR")
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                lib().or_graph_free(h)
            except Exception:  # interpreter shutdown: module globals already cleared
                pass
            self._h = None

    def reverse_csr(self):
        roff = np.empty(self.n + 1, dtype=np.uint64)
        src = np.empty(self.m, dtype=np.uint32)
        thr = np.empty(self.m, dtype=np.uint32)
        lib().or_graph_export(self._h, _ptr(roff), _ptr(src), _ptr(thr))
        return roff, src, thr

    def sample_one(self, seed: int, s: int):
        """(sorted members, their BFS levels, E_logical) of sample s."""
        members = np.empty(self.n, dtype=np.uint32)
        levels = np.empty(self.n, dtype=np.uint32)
        el = np.zeros(1, dtype=np.uint64)
        size = lib().or_sample_one(self._h, seed, s, _ptr(members), _ptr(levels), _ptr(el))
        return members[:size].copy(), levels[:size].copy(), int(el[0])

    def sample_many(self, seed: int, ids, threads: int | None = None, members: bool = False):
        """sizes u32, digests u64, elog u64 per id; with members=True also (offsets, members)."""
        ids = np.ascontiguousarray(ids, dtype=np.uint64)
        cnt = ids.shape[0]
        sizes = np.empty(cnt, dtype=np.uint32)
        digests = np.empty(cnt, dtype=np.uint64)
        elog = np.empty(cnt, dtype=np.uint64)
        t = threads or default_threads()
        lib().or_sample_many(self._h, seed, _ptr(ids), cnt, t, _ptr(sizes), _ptr(digests), _ptr(elog), None, None)
        if not members:
            return sizes, digests, elog
        offsets = np.zeros(cnt + 1, dtype=np.uint64)
        np.cumsum(sizes, out=offsets[1:])
        mem = np.empty(int(offsets[-1]), dtype=np.uint32)
        lib().or_sample_many(self._h, seed, _ptr(ids), cnt, t, None, None, None, _ptr(offsets), _ptr(mem))
        return sizes, digests, elog, offsets, mem

    def group_work_ids(self, seed: int, ids, cap: int = 4096):
        """group_work of a traversal group of arbitrary sample ids."""
        ids = np.ascontiguousarray(ids, dtype=np.uint64)
        ep = np.zeros(1, dtype=np.uint64)
        el = np.zeros(1, dtype=np.uint64)
        lv = np.zeros(1, dtype=np.uint32)
        fr = np.zeros(cap, dtype=np.uint64)
        lib().or_group_work_ids(self._h, seed, _ptr(ids), ids.shape[0], _ptr(ep), _ptr(el), _ptr(lv), _ptr(fr), cap)
        return {"e_phys": int(ep[0]), "e_logical": int(el[0]), "levels": int(lv[0]),
                "frontier": fr[: int(lv[0])].copy()}

    def group_work(self, seed: int, s0: int, s1: int, cap: int = 4096):
        ep = np.zeros(1, dtype=np.uint64)
        el = np.zeros(1, dtype=np.uint64)
        lv = np.zeros(1, dtype=np.uint32)
        fr = np.zeros(cap, dtype=np.uint64)
        lib().or_group_work(self._h, seed, s0, s1, _ptr(ep), _ptr(el), _ptr(lv), _ptr(fr), cap)
        return {"e_phys": int(ep[0]), "e_logical": int(el[0]), "levels": int(lv[0]),
                "frontier": fr[: int(lv[0])].copy()}


class Store:
    """RRR store of samples [s0, s0 + count) (SURVEY §8(c) oracle step 3: sorted lists for small
    sets, n-bit bitsets for large ones), with per-group E_phys / level structure and a greedy
    that runs on it -- so full-size configs fit host memory (C2: ~20 GB instead of ~190 GB)."""

    def __init__(self, graph: "Graph", seed: int, s0: int, count: int, colors: int = 64,
                 threads: int | None = None, list_max: int = 0, ids=None, keep: bool = True):
        """ids: sample ids in traversal order (groups of `colors` consecutive ids; default s0 ...);
        keep=False: sizes, digests and group work only (no sets, no greedy)."""
        self.graph, self.count, self.colors, self.n = graph, count, colors, graph.n
        self.ngroups = (count + colors - 1) // colors
        self._ids = None if ids is None else np.ascontiguousarray(ids, dtype=np.uint64)
        h = lib().or_store_build_ids(graph._h, seed, s0, _ptr(self._ids), count, colors, threads or default_threads(),
                                     list_max, int(keep))
        if not h:
            raise ValueError("oracle store: IC only, and BFS levels must stay below 64")
        self._h = h
        self.sizes = np.empty(count, dtype=np.uint32)
        self.digests = np.empty(count, dtype=np.uint64)
        self.e_phys = np.empty(self.ngroups, dtype=np.uint64)
        self.levels = np.empty(self.ngroups, dtype=np.uint32)
        self.frontier = np.empty((self.ngroups, 64), dtype=np.uint64)
        el = np.zeros(1, dtype=np.uint64)
        lib().or_store_info(h, _ptr(self.sizes), _ptr(self.digests), _ptr(self.e_phys), _ptr(self.levels),
                            _ptr(self.frontier), _ptr(el))
        self.e_logical = int(el[0])

    def members(self, i: int) -> np.ndarray:
        out = np.empty(max(int(self.sizes[i]), 1), dtype=np.uint32)
        c = lib().or_store_members(self._h, i, _ptr(out))
        return out[:c].copy()

    def greedy(self, k: int):
        seeds = np.empty(k, dtype=np.uint32)
        gains = np.empty(k, dtype=np.uint64)
        if lib().or_store_greedy(self._h, k, _ptr(seeds), _ptr(gains)) != 0:
            raise ValueError("oracle store greedy: bad k")
        return seeds, gains

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                lib().or_store_free(h)
            except Exception:
                pass
            self._h = None


def greedy(n: int, set_off, members, k: int, lazy: bool = False):
    """Greedy max-k-cover (reading C-11): seeds u32[k], gains u64[k]."""
    set_off = np.ascontiguousarray(set_off, dtype=np.uint64)
    members = np.ascontiguousarray(members, dtype=np.uint32)
    seeds = np.empty(k, dtype=np.uint32)
    gains = np.empty(k, dtype=np.uint64)
    rc = lib().or_greedy(n, set_off.shape[0] - 1, _ptr(set_off), _ptr(members), k, int(lazy), _ptr(seeds), _ptr(gains))
    if rc != 0:
        raise ValueError("oracle greedy: bad k")
    return seeds, gains


def sigma_hat(n: int, covered: int, theta: int) -> float:
    return lib().or_sigma_hat(n, covered, theta)


def run(row_ptr, col, thr, model: int, theta: int, colors: int, seed: int, k: int, threads: int | None = None):
    """Whole path on a small config: all RRR lists, group work, greedy, sigma_hat."""
    g = Graph(row_ptr, col, w_q31=thr, model=model)
    ids = np.arange(theta, dtype=np.uint64)
    sizes, digests, elog, offsets, mem = g.sample_many(seed, ids, threads, members=True)
    e_phys = 0
    levels = []
    for s0 in range(0, theta, colors):
        w = g.group_work(seed, s0, min(s0 + colors, theta))
        e_phys += w["e_phys"]
        levels.append(w["levels"])
    seeds, gains = greedy(g.n, offsets, mem, k, lazy=False)
    return {"sizes": sizes, "digests": digests, "elog": elog, "offsets": offsets, "members": mem,
            "e_phys": e_phys, "e_logical": int(elog.sum()), "levels": levels,
            "seeds": seeds, "gains": gains, "sigma": sigma_hat(g.n, int(gains.sum()), theta)}
