/*
 * bpt.h -- C-ABI of the B200-native fused breadth-first probabilistic traversal (BPT)
 * library: IMM reverse-reachable (RRR) set sampling with up to 64 fused colours per
 * traversal group, plus greedy max-k-cover seed selection.
 *
 * Paper: "Fused Breadth-First Probabilistic Traversals on Distributed GPU Systems"
 * (arXiv 2311.10201). Citations P:n are lines of its PAPER.md; C-k are the readings
 * listed in DESIGN.md ("Readings of the paper").
 *
 * Conventions (apply to every call):
 *   - Every call returns bpt_status; BPT_OK = 0. On error the outputs are untouched and
 *     bpt_last_error() returns a thread-local, human-readable message.
 *   - Pointer arguments are plain pointers to HOST or DEVICE memory; the library
 *     detects which (cudaPointerGetAttributes). Input arrays are caller-owned and
 *     copied: the library never retains a caller pointer after the call returns.
 *     Host buffers may be pageable; page-locked (pinned) ones are copied at full PCIe /
 *     C2C rate with no staging (large member extractions: pass a reused pinned buffer).
 *   - `stream` is a cudaStream_t passed as void* (NULL = the legacy default stream).
 *     Calls are synchronous with respect to the host on return (results are ready).
 *   - Handles own their device memory until the matching *_free (NULL-safe).
 *   - Sample ids s are GLOBAL: s in [0, theta). Traversal group = C consecutive samples
 *     (s = g*C + c, colour c = bit c mod 64 of the 64-sample block s/64, reading C-9).
 *   - No CPU fallback: if no CUDA device is usable every call fails with BPT_ECUDA.
 */
#ifndef BPT_H
#define BPT_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BPT_ABI_VERSION 2

#if defined(__GNUC__)
#define BPT_API __attribute__((visibility("default")))
#else
#define BPT_API
#endif

typedef enum {
    BPT_OK = 0,
    BPT_EINVAL = -1,   /* invalid argument (message names it) */
    BPT_ENOMEM = -2,   /* device allocation failed, or a caller buffer is too small */
    BPT_ECUDA = -3,    /* CUDA runtime error (message carries cudaGetErrorString) */
    BPT_ENCCL = -4,    /* NCCL error (message carries ncclGetErrorString) */
    BPT_ESTATE = -5    /* call out of order / handle mismatch */
} bpt_status;

/* Diffusion models: independent cascade, linear threshold (reading C-6). */
typedef enum { BPT_IC = 0, BPT_LT = 1 } bpt_model;

typedef struct bpt_comm bpt_comm;
typedef struct bpt_graph bpt_graph;
typedef struct bpt_samples bpt_samples;

/* Thread-local message for the last non-OK status returned on this thread. */
BPT_API const char* bpt_last_error(void);
BPT_API int bpt_abi_version(void);

/* ---------------------------------------------------------------------------------
 * Communicator (one process per GPU). world == 1 needs no NCCL id.
 * bpt_comm_unique_id writes a 128-byte ncclUniqueId (call on rank 0, broadcast it
 * with any transport, e.g. torch.distributed). cuda_device is the device ordinal this
 * rank uses; every later call on handles derived from this comm runs on that device.
 * Errors: EINVAL (world < 1, rank outside [0, world), uid NULL with world > 1),
 * ENCCL, ECUDA.
 * ------------------------------------------------------------------------------- */
BPT_API bpt_status bpt_comm_unique_id(void* uid_out /* 128 bytes, host */);
BPT_API bpt_status bpt_comm_init(const void* nccl_uid, int world, int rank, int cuda_device, bpt_comm** out);
BPT_API void bpt_comm_free(bpt_comm* comm);

/* ---------------------------------------------------------------------------------
 * bpt_graph_load -- A0 + A1: validate a FORWARD CSR with per-edge weights, copy it to
 * the device and build the reverse CSR the BPTs traverse (Def. 2: a BPT
 * from v over the transpose visits exactly the u with a path u ~> v).
 *   row_ptr[n+1] u64: forward rows; col[m] u32: destinations; edge (u, col[e]) for
 *     e in [row_ptr[u], row_ptr[u+1]). Duplicates and self-loops are accepted (each
 *     parallel edge is its own coin, reading C-15).
 *   Weights: exactly one of w_f32[m] (probability in [0,1]; converted to Q1.31 as
 *     floor(p * 2^31), reading C-5) or w_q31[m] (thresholds in [0, 2^31], p = thr/2^31).
 *   model: BPT_IC keeps per-edge thresholds; BPT_LT requires, for every vertex v, the
 *     sum of the thresholds of v's in-edges to be <= 2^31 (reading C-6) and stores
 *     the per-row inclusive prefix instead.
 *   Canonical reverse order (reading C-4): rows by destination; within a row, entries
 *     in forward position order. The edge id used by the coins is the position in
 *     this reverse CSR.
 *   comm may be NULL (single GPU: current device).
 * Errors: EINVAL if n == 0, m >= 2^32, row_ptr[0] != 0, row_ptr not non-decreasing,
 *   row_ptr[n] != m, any col >= n, any weight outside its range (NaN included), both
 *   or neither weight arrays given, or an LT row sum > 2^31 (message names the vertex);
 *   ENOMEM; ECUDA.
 * ------------------------------------------------------------------------------- */
BPT_API bpt_status bpt_graph_load(bpt_comm* comm, const uint64_t* row_ptr, const uint32_t* col, uint32_t n,
                          uint64_t m, const float* w_f32, const uint32_t* w_q31, bpt_model model,
                          void* stream, bpt_graph** out);
/* Collective variant of bpt_graph_load for a communicator of world > 1 (every rank calls it):
 * only the root's row_ptr / col / weights are read (others may pass NULL; n, m and model must
 * be the same on every rank). The root validates and builds the reverse CSR; the result is
 * broadcast over NCCL (NVLink), so the host-to-device copy of the input happens once instead
 * of once per GPU (SURVEY §8(e) "rank 0 builds and ncclBroadcasts"). A validation error on the
 * root fails the call on every rank. world == 1 (or comm NULL): same as bpt_graph_load. */
BPT_API bpt_status bpt_graph_load_bcast(bpt_comm* comm, int root, const uint64_t* row_ptr, const uint32_t* col,
                                        uint32_t n, uint64_t m, const float* w_f32, const uint32_t* w_q31,
                                        bpt_model model, void* stream, bpt_graph** out);
/* Export the reverse CSR (tests): roff[n+1], src[m], val[m] (IC: threshold; LT: cumulative
 * threshold). Any pointer may be NULL. Host or device buffers. */
BPT_API bpt_status bpt_graph_reverse(const bpt_graph* g, uint32_t* roff, uint32_t* src, uint32_t* val);
BPT_API bpt_status bpt_graph_dims(const bpt_graph* g, uint32_t* n, uint64_t* m, int* model);
BPT_API void bpt_graph_free(bpt_graph* g);

/* ---------------------------------------------------------------------------------
 * bpt_sample -- A2..A5: sample theta RRR sets with `colors` BPTs fused per traversal
 * group (Listing 1), level-synchronous (reading C-7).
 *   Start vertex of sample s: reading C-3 ("selected uniformly at random from V").
 *   IC coin of sample s on reverse edge e: Philox2x32-10 keyed by (seed, s, e), edge live
 *     iff (r >> 1) < thr(e) (readings C-1, C-2). LT: one draw per (s, v) picks <= 1
 *     in-edge (reading C-6).
 *   Result: RRR sets stored in fused form (per 64-sample block, a u64 colour mask per
 *     vertex = Listing 1's visited[]), plus per-sample sizes; per-sample digests
 *      are computed from the store on the first bpt_rrr_digests call. RRR sets are identical for any colors, batch size and number
 *     of ranks (readings C-9, C-14).
 *   colors must divide 64 (1, 2, 4, 8, 16, 32, 64). theta in [1, 2^32).
 *   Multi-rank: every rank calls with identical arguments; rank r samples the 64-sample
 *     blocks [floor(r*nb/W), floor((r+1)*nb/W)), nb = ceil(theta/64). No communication.
 * Errors: EINVAL (theta, colors, model != graph model), ENOMEM (store does not fit),
 *   ECUDA.
 * ------------------------------------------------------------------------------- */
typedef struct {
    uint32_t batch_groups;   /* 64-sample blocks traversed concurrently; 0 = automatic */
    uint32_t poll_levels;    /* levels launched between host polls; 0 = automatic */
    uint32_t flags;          /* BPT_FLAG_* */
    uint32_t shard_world;    /* test hook: sample only shard shard_rank of shard_world (0 = use the comm) */
    uint32_t shard_rank;
    uint32_t pull_permille;  /* BPT_FLAG_PULL: levels whose push work is >= pull_permille / 1000 x m
                                are pulled (0 = the default, 1000) */
} bpt_sample_opts;
#define BPT_FLAG_PROFILE 1u  /* time every expansion launch with CUDA events */
/* Wide fusion (the paper fuses up to 1024 colours): IC with
 * colors = 64 and batch_groups = 0 only -- two 64-sample blocks (128 colours) share one
 * frontier, so each reverse edge of a frontier vertex is read once for 128 samples. Same RRR
 * sets (coins are keyed by the global sample id); E_phys counts the 128-sample groups. */
#define BPT_FLAG_WIDE 2u
/* LT only: REQUIRE the sparse store -- the RRR sets kept as member lists instead of the
 * dense n x blocks bitmap (SURVEY A5 "compressed rows": C3 ~0.1 GB instead of 100 GB). LT uses
 * it by default too, falling back to the dense store when a walk outgrows the per-thread
 * visited set (1,536 vertices); with this flag that case fails with ENOMEM instead. Sizes,
 * digests, extraction and selection read whichever form the handle holds. */
#define BPT_FLAG_SPARSE 4u
/* LT samples are drawn as one reverse walk per thread by default (the RRR store is each
 * sample's visited set); batch_groups and BPT_FLAG_PROFILE do not apply to the walks. The
 * flags below select the other execution forms; every form gives the same RRR sets, sizes,
 * digests, seeds and exact work counters (coins are keyed by (sample, edge / vertex) only). */
#define BPT_FLAG_LT_FUSED 8u    /* LT: the fused level-synchronous loop of Listing 1
                                   over 64-colour groups instead of per-sample walks */
#define BPT_FLAG_LT_DENSE 16u   /* LT walks: dense n x blocks store instead of member lists */
#define BPT_FLAG_LT_REWALK 32u  /* LT sparse store: member lists from a second walk */
#define BPT_FLAG_LT_LEVELS 64u  /* LT fused: one launch pair per level instead of one cooperative
                                   launch per batch */
#define BPT_FLAG_QUEUE 128u     /* IC, 64 colours: discovered vertices through a first-setter
                                   queue (atomicOr with return) instead of the touched bitmap */
/* IC, 64 colours (touched-bitmap form) and 1 < C < 64: samples are assigned to the traversal slots in the order
 * of their start vertices (in-degree descending, then start id, then sample id; "sorting the
 * starting vertices"), so samples with large reverse BPTs share groups
 * (a C-colour group = C samples adjacent in that order).
 * On by default; this flag keeps sample s in slot s (groups of consecutive samples, reading C-9).
 * RRR sets, sizes, digests and seeds are identical either way; E_phys / levels differ. */
#define BPT_FLAG_UNSORTED 256u
/* IC, 64 colours (touched-bitmap form): direction switching (P:544-545,
 * P:529-531). A level whose push work (reverse-edge reads of the frontier, all slots of the batch)
 * reaches ~m is expanded by PULL: every forward edge u -> w is read once for all slots of the
 * batch, live = frontier(w) & ~visited(u), with the coin of the edge's canonical reverse id (same
 * RRR sets, sizes, digests, seeds, E_phys and level structure as the push form; coins / merges
 * differ). Needs 16 B per edge of forward records (built on first use, kept with the graph); falls
 * back to push when they do not fit. */
#define BPT_FLAG_PULL 512u
/* IC, 64 colours (touched-bitmap form): by default the <= 4 64-sample blocks of a batch share ONE
 * frontier of vertices (vertex-major working masks; every reverse edge of a frontier vertex is read
 * once for up to 256 colours). This flag keeps one frontier per block
 * (64 colours per entry; implied by BPT_FLAG_PULL). Same RRR sets, sizes, digests and seeds; E_phys
 * and the level structure are those of the 256-sample (resp. 64-sample) fused groups. */
#define BPT_FLAG_SLOTWISE 1024u

BPT_API bpt_status bpt_sample(const bpt_graph* g, bpt_model model, uint64_t theta, uint32_t colors, uint64_t seed,
                      void* stream, bpt_samples** out);
BPT_API bpt_status bpt_sample_ex(const bpt_graph* g, bpt_model model, uint64_t theta, uint32_t colors, uint64_t seed,
                         const bpt_sample_opts* opts, void* stream, bpt_samples** out);

typedef struct {
    uint64_t theta, seed, s0, s1;          /* this rank owns global samples [s0, s1) */
    uint32_t colors, model, world, rank;
    uint32_t n, batch_groups, batches, levels_max;  /* levels_max: deepest batch (LT: longest walk) */
    uint64_t e_phys;        /* IC: reverse-edge records read by the fused expansion;
                               LT: (vertex, colour) expansions = sum |RR_s| */
    uint64_t e_logical;     /* IC: sum_s sum_{v in RR_s} indeg(v) (unfused reads); LT: sum |RR_s| */
    uint64_t members;       /* sum_s |RR_s| over this rank's samples */
    uint64_t levels_total;  /* sum over batches of levels traversed (LT walks: the longest walk) */
    uint64_t frontier_entries; /* (vertex, slice) frontier entries expanded */
    uint64_t coins;         /* coin evaluations (schedule-dependent, informational) */
    uint64_t atomics;       /* atomicOr merges issued (schedule-dependent) */
    uint64_t store_bytes;   /* bytes of the fused RRR store on this rank */
    uint64_t kernel_launches;
    uint64_t expand_launches;
    double ms_total;        /* host wall time of bpt_sample */
    double ms_expand;       /* expansion time: CUDA events per launch (BPT_FLAG_PROFILE), else device
                               %globaltimer spans of the launches; LT walks: the walk kernel */
    double expand_bytes;    /* algorithmic bytes moved by expansion launches */
    uint64_t pull_levels;   /* levels expanded by pull (BPT_FLAG_PULL) */
    uint64_t pull_edge_reads; /* forward-edge records read by those levels (e_phys counts the push
                               form's reads of every level, the work the oracle defines) */
} bpt_samples_info;

BPT_API bpt_status bpt_samples_get_info(const bpt_samples* s, bpt_samples_info* out);

/* A7 round 0: occurrences count[v] = number of this rank's samples whose RRR set contains v,
 * for v in [0, n). counts[n] u32, host or device. */
BPT_API bpt_status bpt_occurrences(const bpt_samples* s, uint32_t* counts);

/* Per level of every batch: {batch, level, raw_entries, kept_entries, edges_or_tasks, vc_pairs,
 * coins, atomics} as 8 u64 per row, host buffer (coins / atomics are schedule-dependent). *rows = number of rows available (written if rows_out != NULL). */
BPT_API bpt_status bpt_level_stats(const bpt_samples* s, uint64_t* out, uint64_t cap_rows, uint64_t* rows_out);
/* Expansion time of every bpt_level_stats row, ms as f32 (CUDA events around each expansion
 * launch), host buffer; only samples drawn with BPT_FLAG_PROFILE have them (*rows = 0 otherwise).
 * Measurement aid for the roofline; *rows = rows available. */
BPT_API bpt_status bpt_level_times(const bpt_samples* s, float* out, uint64_t cap_rows, uint64_t* rows_out);

/* ---------------------------------------------------------------------------------
 * A5/A6: per-sample results for global sample ids [first, first+count), which must lie
 * in this rank's range (else EINVAL).
 *   sizes[count] u32 = |RR_s|; digests[count] u64 = sum over v in RR_s of
 *   splitmix64(v) mod 2^64 (the first digests call on a handle runs
 *   one pass over the local store, later calls read the cached values).
 *   bpt_rrr_extract: Listing 1 lines 18-21 -- RRR lists, sorted ascending,
 *   start included (reading C-10). offsets[count+1] u64 (offsets[0] = 0), members
 *   u32[capacity]. If capacity < offsets[count] -> ENOMEM (message gives the size) and
 *   nothing is written.
 * ------------------------------------------------------------------------------- */
BPT_API bpt_status bpt_rrr_sizes(const bpt_samples* s, uint64_t first, uint64_t count, uint32_t* sizes);
BPT_API bpt_status bpt_rrr_digests(const bpt_samples* s, uint64_t first, uint64_t count, uint64_t* digests);
BPT_API bpt_status bpt_rrr_extract(const bpt_samples* s, uint64_t first, uint64_t count, uint64_t* offsets,
                           uint32_t* members, uint64_t capacity);

/* ---------------------------------------------------------------------------------
 * bpt_select_seeds -- A7/A8: greedy max-k-cover over all theta RRR sets:
 * each round picks the vertex covering the most uncovered sets, smallest id on ties,
 * smallest unselected id once everything is covered (reading C-11).
 *   seeds[k] u32, gains[k] u64 (sets newly covered per round), *sigma_hat =
 *   n * sum(gains) / theta (f64, reading C-12). Any output may be NULL. Host or device.
 *   Collective across the comm (same result on every rank). Does not modify the store:
 *   may be called again with another k.
 * Errors: EINVAL (k == 0 or k > n), ENCCL, ECUDA.
 * ------------------------------------------------------------------------------- */
BPT_API bpt_status bpt_select_seeds(const bpt_samples* s, uint32_t k, uint32_t* seeds, uint64_t* gains,
                            double* sigma_hat);

BPT_API void bpt_samples_free(bpt_samples* s);

/* Device self-test of reading C-1: out[2i], out[2i+1] = Philox2x32-10(ctr = {ctr_key[3i],
 * ctr_key[3i+1]}, key = ctr_key[3i+2]) evaluated by the same device function the coins and start
 * vertices use (checked against the Random123 known-answer vectors). Host or device buffers. */
BPT_API bpt_status bpt_selftest_philox(const uint32_t* ctr_key, uint32_t* out, uint64_t count);
/* Integer-ALU roof of the coin: times `iters` rounds of Philox2x32-10 coin evaluations on every
 * resident thread (CUDA events); *calls = evaluations made, *ms = their device time. */
BPT_API bpt_status bpt_bench_philox(uint64_t iters, uint64_t* calls, double* ms);

/* Release the device blocks the library caches between calls (its memory pool). */
BPT_API bpt_status bpt_release_cache(void);

/* Launch evidence (process-wide counters). bpt_kernel_launch_count: launches the host issued --
 * kernels launched directly plus one per CUDA-graph launch. bpt_graph_kernel_count: kernel
 * executions inside the sampling graphs (its conditional level / batch loops), counted on the
 * device by the kernels themselves. Their sum is every kernel execution of the library. */
BPT_API uint64_t bpt_kernel_launch_count(void);
BPT_API uint64_t bpt_graph_kernel_count(void);

#ifdef __cplusplus
}
#endif
#endif /* BPT_H */
