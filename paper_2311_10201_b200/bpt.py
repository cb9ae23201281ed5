"""ctypes binding of libbpt.so (include/bpt.h). Argument marshalling only: every step of
the hot path runs in the library's CUDA kernels. There is no CPU fallback -- importing
this module fails loudly if libbpt.so has not been built.

Arrays: numpy arrays (host) or any object with `data_ptr()` (e.g. a torch CUDA tensor,
device memory). The library detects host vs device pointers itself.
"""
from __future__ import annotations

import ctypes
import os
import re

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("BPT_LIB") or os.path.join(_HERE, "libbpt.so")  # BPT_LIB: tuning variants only
HEADER = os.path.join(os.path.dirname(_HERE), "include", "bpt.h")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                      "(the CUDA library is the only implementation; there is no fallback)")

_lib = ctypes.CDLL(LIB_PATH)

BPT_OK, BPT_EINVAL, BPT_ENOMEM, BPT_ECUDA, BPT_ENCCL, BPT_ESTATE = 0, -1, -2, -3, -4, -5
IC, LT = 0, 1
FLAG_PROFILE = 1
FLAG_WIDE = 2  # 128 colours per frontier entry (IC, colors=64, batch_groups=0)
FLAG_SPARSE = 4  # LT: sorted member lists instead of the dense store
FLAG_LT_FUSED = 8  # LT: fused level-synchronous loop instead of per-sample walks
FLAG_LT_DENSE = 16  # LT walks: dense store
FLAG_LT_REWALK = 32  # LT sparse store: member lists by a second walk
FLAG_LT_LEVELS = 64  # LT fused: per-level launches instead of one cooperative launch per batch
FLAG_QUEUE = 128  # IC 64 colours: first-setter queue instead of the touched bitmap
FLAG_UNSORTED = 256  # IC, 1 < C <= 64: sample s in slot s (no start-vertex sort)
FLAG_PULL = 512  # IC 64 colours: pull expansion of the heavy levels (direction switching)
FLAG_SLOTWISE = 1024  # IC 64 colours: one frontier per 64-sample block instead of one per batch
_STATUS = {0: "BPT_OK", -1: "BPT_EINVAL", -2: "BPT_ENOMEM", -3: "BPT_ECUDA", -4: "BPT_ENCCL", -5: "BPT_ESTATE"}

_p, _u32, _u64, _i = ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int


class bpt_sample_opts(ctypes.Structure):
    _fields_ = [("batch_groups", _u32), ("poll_levels", _u32), ("flags", _u32), ("shard_world", _u32),
                ("shard_rank", _u32), ("pull_permille", _u32)]


class bpt_samples_info(ctypes.Structure):
    _fields_ = [("theta", _u64), ("seed", _u64), ("s0", _u64), ("s1", _u64),
                ("colors", _u32), ("model", _u32), ("world", _u32), ("rank", _u32),
                ("n", _u32), ("batch_groups", _u32), ("batches", _u32), ("levels_max", _u32),
                ("e_phys", _u64), ("e_logical", _u64), ("members", _u64), ("levels_total", _u64),
                ("frontier_entries", _u64), ("coins", _u64), ("atomics", _u64), ("store_bytes", _u64),
                ("kernel_launches", _u64), ("expand_launches", _u64),
                ("ms_total", ctypes.c_double), ("ms_expand", ctypes.c_double), ("expand_bytes", ctypes.c_double),
                ("pull_levels", _u64), ("pull_edge_reads", _u64)]

    def as_dict(self) -> dict:
        return {name: getattr(self, name) for name, _ in self._fields_}


_SIGS = {
    "bpt_last_error": ([], ctypes.c_char_p),
    "bpt_abi_version": ([], _i),
    "bpt_kernel_launch_count": ([], _u64),
    "bpt_graph_kernel_count": ([], _u64),
    "bpt_comm_unique_id": ([_p], _i),
    "bpt_comm_init": ([_p, _i, _i, _i, ctypes.POINTER(_p)], _i),
    "bpt_comm_free": ([_p], None),
    "bpt_graph_load": ([_p, _p, _p, _u32, _u64, _p, _p, _i, _p, ctypes.POINTER(_p)], _i),
    "bpt_graph_load_bcast": ([_p, _i, _p, _p, _u32, _u64, _p, _p, _i, _p, ctypes.POINTER(_p)], _i),
    "bpt_graph_reverse": ([_p, _p, _p, _p], _i),
    "bpt_graph_dims": ([_p, _p, _p, _p], _i),
    "bpt_graph_free": ([_p], None),
    "bpt_sample": ([_p, _i, _u64, _u32, _u64, _p, ctypes.POINTER(_p)], _i),
    "bpt_sample_ex": ([_p, _i, _u64, _u32, _u64, ctypes.POINTER(bpt_sample_opts), _p, ctypes.POINTER(_p)], _i),
    "bpt_samples_get_info": ([_p, ctypes.POINTER(bpt_samples_info)], _i),
    "bpt_level_stats": ([_p, _p, _u64, _p], _i),
    "bpt_level_times": ([_p, _p, _u64, _p], _i),
    "bpt_occurrences": ([_p, _p], _i),
    "bpt_rrr_sizes": ([_p, _u64, _u64, _p], _i),
    "bpt_rrr_digests": ([_p, _u64, _u64, _p], _i),
    "bpt_rrr_extract": ([_p, _u64, _u64, _p, _p, _u64], _i),
    "bpt_select_seeds": ([_p, _u32, _p, _p, _p], _i),
    "bpt_samples_free": ([_p], None),
    "bpt_release_cache": ([], _i),
    "bpt_selftest_philox": ([_p, _p, _u64], _i),
    "bpt_bench_philox": ([_u64, ctypes.POINTER(_u64), ctypes.POINTER(ctypes.c_double)], _i),
}
for _name, (_args, _res) in _SIGS.items():
    _f = getattr(_lib, _name)
    _f.argtypes = _args
    _f.restype = _res


def header_symbols() -> list[str]:
    """Function names declared in include/bpt.h."""
    with open(HEADER) as f:
        text = f.read()
    return sorted(set(re.findall(r"\b(bpt_[a-z_0-9]+)\s*\(", text)))


class BptError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{_STATUS.get(code, code)}: {msg}")
        self.code = code


def _check(rc: int) -> None:
    if rc != BPT_OK:
        raise BptError(rc, _lib.bpt_last_error().decode(errors="replace"))


def _ptr(a):
    if a is None:
        return None
    if hasattr(a, "data_ptr"):
        return a.data_ptr()
    if isinstance(a, np.ndarray):
        if not a.flags["C_CONTIGUOUS"]:
            raise ValueError("arrays must be C-contiguous")
        return a.ctypes.data
    raise TypeError(f"unsupported array type {type(a)}")


def _stream(stream):
    if stream is None:
        try:
            import torch
            if torch.cuda.is_available():
                return torch.cuda.current_stream().cuda_stream
        except ImportError:
            pass
        return None
    if hasattr(stream, "cuda_stream"):
        return stream.cuda_stream
    return stream


# ------------------------------------------------------------------ raw C-ABI (same names)
def bpt_last_error() -> str:
    return _lib.bpt_last_error().decode(errors="replace")


def bpt_abi_version() -> int:
    return _lib.bpt_abi_version()


def selftest_philox(ctr_key) -> np.ndarray:
    """Device Philox2x32-10 of rows (ctr0, ctr1, key) -> rows (out0, out1) (reading C-1)."""
    a = np.ascontiguousarray(ctr_key, dtype=np.uint32).reshape(-1, 3)
    out = np.zeros((a.shape[0], 2), dtype=np.uint32)
    _check(_lib.bpt_selftest_philox(_ptr(a), _ptr(out), a.shape[0]))
    return out


def bench_philox(iters: int = 64) -> tuple[int, float]:
    """(coin evaluations, device ms) of the Philox throughput kernel."""
    calls, ms = _u64(), ctypes.c_double()
    _check(_lib.bpt_bench_philox(iters, ctypes.byref(calls), ctypes.byref(ms)))
    return int(calls.value), float(ms.value)


def kernel_launch_count() -> int:
    """Kernel launches the host issued (direct launches + one per CUDA-graph launch)."""
    return int(_lib.bpt_kernel_launch_count())


def graph_kernel_count() -> int:
    """Kernel executions inside the sampling graphs, counted on the device by the kernels."""
    return int(_lib.bpt_graph_kernel_count())


def kernels_executed() -> int:
    """Every kernel execution of the library so far (host launches + graph-node executions)."""
    return kernel_launch_count() + graph_kernel_count()


bpt_kernel_launch_count = kernel_launch_count
bpt_graph_kernel_count = graph_kernel_count


def bpt_comm_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(_lib.bpt_comm_unique_id(buf))
    return buf.raw


def bpt_comm_init(uid: bytes | None, world: int, rank: int, device: int):
    h = _p()
    ub = ctypes.create_string_buffer(uid, 128) if uid is not None else None
    _check(_lib.bpt_comm_init(ub, world, rank, device, ctypes.byref(h)))
    return h


def bpt_comm_free(h) -> None:
    _lib.bpt_comm_free(h)


def bpt_graph_load(comm, row_ptr, col, n: int, m: int, w_f32=None, w_q31=None, model: int = IC, stream=None):
    h = _p()
    _check(_lib.bpt_graph_load(comm, _ptr(row_ptr), _ptr(col), n, m, _ptr(w_f32), _ptr(w_q31), model,
                               _stream(stream), ctypes.byref(h)))
    return h


def bpt_graph_load_bcast(comm, root: int, row_ptr, col, n: int, m: int, w_f32=None, w_q31=None, model: int = IC,
                         stream=None):
    h = _p()
    _check(_lib.bpt_graph_load_bcast(comm, root, _ptr(row_ptr), _ptr(col), n, m, _ptr(w_f32), _ptr(w_q31), model,
                                     _stream(stream), ctypes.byref(h)))
    return h


def bpt_graph_free(h) -> None:
    _lib.bpt_graph_free(h)


def bpt_sample(graph, model: int, theta: int, colors: int, seed: int, stream=None, batch_groups: int = 0,
               poll_levels: int = 0, flags: int = 0, shard: tuple[int, int] | None = None, pull_permille: int = 0):
    h = _p()
    sw, sr = shard if shard else (0, 0)
    opts = bpt_sample_opts(batch_groups, poll_levels, flags, sw, sr, pull_permille)
    _check(_lib.bpt_sample_ex(graph, model, theta, colors, seed, ctypes.byref(opts), _stream(stream),
                              ctypes.byref(h)))
    return h


def bpt_samples_get_info(h) -> dict:
    info = bpt_samples_info()
    _check(_lib.bpt_samples_get_info(h, ctypes.byref(info)))
    return info.as_dict()


def bpt_level_stats(h) -> np.ndarray:
    rows = _u64()
    _check(_lib.bpt_level_stats(h, None, 0, ctypes.byref(rows)))
    out = np.zeros((rows.value, 8), dtype=np.uint64)  # batch, level, raw, kept, work, vc, coins, atomics
    if rows.value:
        _check(_lib.bpt_level_stats(h, _ptr(out), rows.value, None))
    return out


def bpt_level_times(h) -> np.ndarray:
    rows = _u64()
    _check(_lib.bpt_level_times(h, None, 0, ctypes.byref(rows)))
    out = np.zeros(rows.value, dtype=np.float32)  # expansion ms per bpt_level_stats row (profile mode)
    if rows.value:
        _check(_lib.bpt_level_times(h, _ptr(out), rows.value, None))
    return out


def bpt_occurrences(h, n: int, out=None):
    out = np.empty(n, dtype=np.uint32) if out is None else out
    _check(_lib.bpt_occurrences(h, _ptr(out)))
    return out


def bpt_rrr_sizes(h, first: int, count: int, out=None):
    out = np.empty(count, dtype=np.uint32) if out is None else out
    _check(_lib.bpt_rrr_sizes(h, first, count, _ptr(out)))
    return out


def bpt_rrr_digests(h, first: int, count: int, out=None):
    out = np.empty(count, dtype=np.uint64) if out is None else out
    _check(_lib.bpt_rrr_digests(h, first, count, _ptr(out)))
    return out


def bpt_rrr_extract(h, first: int, count: int, offsets=None, members=None, capacity: int | None = None):
    if members is None:
        sizes = bpt_rrr_sizes(h, first, count)
        total = int(sizes.astype(np.uint64).sum())
        members = np.empty(max(total, 1), dtype=np.uint32)
        capacity = total
    offsets = np.empty(count + 1, dtype=np.uint64) if offsets is None else offsets
    cap = capacity if capacity is not None else (members.shape[0] if hasattr(members, "shape") else 0)
    _check(_lib.bpt_rrr_extract(h, first, count, _ptr(offsets), _ptr(members), cap))
    if isinstance(members, np.ndarray):
        members = members[: int(offsets[-1])]
    return offsets, members


def bpt_select_seeds(h, k: int, seeds=None, gains=None):
    seeds = np.empty(k, dtype=np.uint32) if seeds is None else seeds
    gains = np.empty(k, dtype=np.uint64) if gains is None else gains
    sigma = ctypes.c_double()
    _check(_lib.bpt_select_seeds(h, k, _ptr(seeds), _ptr(gains), ctypes.byref(sigma)))
    return seeds, gains, sigma.value


def bpt_samples_free(h) -> None:
    _lib.bpt_samples_free(h)


def bpt_release_cache() -> None:
    _check(_lib.bpt_release_cache())


# ------------------------------------------------------------------ object wrappers
class Comm:
    """One process per GPU. world == 1 needs no NCCL id."""

    def __init__(self, world: int = 1, rank: int = 0, device: int = 0, uid: bytes | None = None):
        self.world, self.rank, self.device = world, rank, device
        self._h = bpt_comm_init(uid, world, rank, device)

    @staticmethod
    def unique_id() -> bytes:
        return bpt_comm_unique_id()

    def close(self):
        if getattr(self, "_h", None):
            bpt_comm_free(self._h)
            self._h = None

    def __del__(self):
        self.close()


class Graph:
    """bpt_graph_load: forward CSR + weights -> device reverse CSR."""

    def __init__(self, row_ptr, col, w_f32=None, w_q31=None, model: int = IC, comm: Comm | None = None,
                 n: int | None = None, m: int | None = None, stream=None, bcast_root: int | None = None):
        """bcast_root: collective load (bpt_graph_load_bcast) -- only that rank's arrays are read
        (others may pass None with n and m); the reverse CSR is broadcast over NCCL."""
        self.comm = comm
        self.n = int(n if n is not None else row_ptr.shape[0] - 1)
        self.m = int(m if m is not None else col.shape[0])
        self.model = model
        if bcast_root is not None:
            self._h = bpt_graph_load_bcast(comm._h if comm else None, bcast_root, row_ptr, col, self.n, self.m,
                                           w_f32, w_q31, model, stream)
            return
        if isinstance(row_ptr, np.ndarray):
            row_ptr = np.ascontiguousarray(row_ptr, dtype=np.uint64)
            col = np.ascontiguousarray(col, dtype=np.uint32)
            if w_f32 is not None and isinstance(w_f32, np.ndarray):
                w_f32 = np.ascontiguousarray(w_f32, dtype=np.float32)
            if w_q31 is not None and isinstance(w_q31, np.ndarray):
                w_q31 = np.ascontiguousarray(w_q31, dtype=np.uint32)
        self._h = bpt_graph_load(comm._h if comm else None, row_ptr, col, self.n, self.m, w_f32, w_q31, model,
                                 stream)

    def reverse_csr(self):
        roff = np.empty(self.n + 1, dtype=np.uint32)
        src = np.empty(max(self.m, 1), dtype=np.uint32)
        val = np.empty(max(self.m, 1), dtype=np.uint32)
        _check(_lib.bpt_graph_reverse(self._h, _ptr(roff), _ptr(src), _ptr(val)))
        return roff, src[: self.m], val[: self.m]

    def sample(self, theta: int, colors: int = 64, seed: int = 0, stream=None, batch_groups: int = 0,
               poll_levels: int = 0, profile: bool = False, shard: tuple[int, int] | None = None,
               wide: bool = False, sparse: bool = False, flags: int = 0, pull: bool = False,
               pull_permille: int = 0) -> "Samples":
        flags |= (FLAG_PROFILE if profile else 0) | (FLAG_WIDE if wide else 0) | (FLAG_SPARSE if sparse else 0)
        flags |= FLAG_PULL if pull else 0
        h = bpt_sample(self._h, self.model, theta, colors, seed, stream, batch_groups, poll_levels, flags, shard,
                       pull_permille)
        return Samples(self, h)

    def close(self):
        if getattr(self, "_h", None):
            bpt_graph_free(self._h)
            self._h = None

    def __del__(self):
        self.close()


class Samples:
    """bpt_sample result: fused RRR store of this rank's sample range."""

    def __init__(self, graph: Graph, h):
        self.graph = graph
        self._h = h
        self.info = bpt_samples_get_info(h)
        self.s0, self.s1 = self.info["s0"], self.info["s1"]

    def sizes(self, first: int, count: int, out=None):
        return bpt_rrr_sizes(self._h, first, count, out)

    def digests(self, first: int, count: int, out=None):
        return bpt_rrr_digests(self._h, first, count, out)

    def extract(self, first: int, count: int, offsets=None, members=None, capacity=None):
        return bpt_rrr_extract(self._h, first, count, offsets, members, capacity)

    def occurrences(self, out=None):
        return bpt_occurrences(self._h, self.graph.n, out)

    def level_stats(self) -> np.ndarray:
        return bpt_level_stats(self._h)

    def level_times(self) -> np.ndarray:
        return bpt_level_times(self._h)

    def select_seeds(self, k: int, seeds=None, gains=None):
        return bpt_select_seeds(self._h, k, seeds, gains)

    def close(self):
        if getattr(self, "_h", None):
            bpt_samples_free(self._h)
            self._h = None

    def __del__(self):
        self.close()
