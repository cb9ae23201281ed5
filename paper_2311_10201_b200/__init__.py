"""B200-native fused breadth-first probabilistic traversal (BPT) for IMM RRR sampling.

Paper: arXiv 2311.10201. The hot path lives in libbpt.so (hand-written CUDA
for sm_100a behind the C-ABI of include/bpt.h); this package is its thin ctypes binding.
"""
from .bpt import (  # noqa: F401
    BPT_EINVAL, BPT_ENOMEM, BPT_ECUDA, BPT_ENCCL, BPT_ESTATE, BPT_OK, FLAG_PROFILE, FLAG_SPARSE, FLAG_WIDE, IC, LT, LIB_PATH,
    FLAG_LT_DENSE, FLAG_LT_FUSED, FLAG_LT_LEVELS, FLAG_LT_REWALK, FLAG_QUEUE, FLAG_UNSORTED, FLAG_PULL, FLAG_SLOTWISE,
    BptError, Comm, Graph, Samples, bpt_abi_version, bpt_comm_free, bpt_comm_init, bpt_comm_unique_id,
    bpt_graph_free, bpt_graph_load, bpt_kernel_launch_count, bpt_last_error, bpt_level_stats, bpt_occurrences,
    bpt_rrr_digests, bpt_rrr_extract, bpt_rrr_sizes, bpt_sample, bpt_samples_free, bpt_samples_get_info,
    bpt_select_seeds, header_symbols, kernel_launch_count, graph_kernel_count, kernels_executed, bpt_graph_kernel_count, selftest_philox, bench_philox,
)

__all__ = [n for n in dir() if not n.startswith("_")]
