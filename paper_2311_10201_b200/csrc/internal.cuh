// internal.cuh -- shared declarations of the libbpt CUDA implementation (sm_100a).
// Not part of the ABI; the ABI is include/bpt.h.
#pragma once
#include <cstdint>
#include <mutex>
#include <cstddef>
#include <string>
#include <vector>
#include <cuda_runtime.h>

#include "../../include/bpt.h"

namespace bpt {

// ------------------------------------------------------------------ error plumbing
struct Error {
    bpt_status code;
    std::string msg;
};
[[noreturn]] void fail(bpt_status code, const std::string& msg);
void check_cuda(cudaError_t e, const char* what);
#define BPT_CUDA(x) ::bpt::check_cuda((x), #x)

__host__ __device__ __forceinline__ uint64_t umin64(uint64_t a, uint64_t b) { return a < b ? a : b; }
__host__ __device__ __forceinline__ uint64_t umax64(uint64_t a, uint64_t b) { return a > b ? a : b; }

// Device bounds checks (diagnostic build -DBPT_CHECKS; compute-sanitizer is not available on the
// GPU pool): a failed check records its id in a device flag instead of trapping, and the API call
// that ran the kernels fails with BPT_ECUDA naming the check.
#ifdef BPT_CHECKS
#define BPT_CHECK(cond, id) \
    do { if (!(cond)) ::bpt::check_failed(id); } while (0)
#else
#define BPT_CHECK(cond, id) do { } while (0)
#endif
__device__ void check_failed(uint32_t id);
uint32_t checks_read_reset();  // host: failed-check bits since the last call (0 in normal builds)

extern uint64_t g_launches;        // kernel launches issued by the host (<<<>>> and cudaGraphLaunch)
extern uint64_t g_graph_kernels;   // kernel executions inside CUDA graphs, counted on the device
inline void count_launch(uint64_t k = 1) { g_launches += k; }

// ------------------------------------------------------------------ Philox2x32-10
// Reading C-1: Philox2x32-10 of Salmon et al. (SC'11) with the Random123
// constants. Written here from the definition; the CPU oracle has its own copy.
constexpr uint32_t kPhiloxM = 0xD256D193u;
constexpr uint32_t kPhiloxW = 0x9E3779B9u;
constexpr uint32_t kTagIC = 0x49430001u, kTagLT = 0x4C540001u, kTagStart = 0x53540001u;

__host__ __device__ __forceinline__ uint2 philox2x32_10(uint32_t x0, uint32_t x1, uint32_t key) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        uint64_t p = (uint64_t)kPhiloxM * (uint64_t)x0;
        uint32_t hi = (uint32_t)(p >> 32), lo = (uint32_t)p;
        x0 = hi ^ key ^ x1;
        x1 = lo;
        key += kPhiloxW;
    }
    return make_uint2(x0, x1);
}

// k_tag = Philox(ctr = {lo32(seed), hi32(seed)}, key = tag)[0]
inline uint32_t stream_key(uint64_t seed, uint32_t tag) {
    return philox2x32_10((uint32_t)seed, (uint32_t)(seed >> 32), tag).x;
}

// ------------------------------------------------------------------ handles
struct Comm {
    int world = 1, rank = 0, device = 0;
    void* nccl = nullptr;  // ncclComm_t
};

// The stream the current API call runs on (set by StreamScope at the entry of every call
// that queues work): device blocks are allocated and released in that stream's order.
struct StreamScope {
    explicit StreamScope(cudaStream_t st);
    ~StreamScope();
    StreamScope(const StreamScope&) = delete;
    StreamScope& operator=(const StreamScope&) = delete;
private:
    cudaStream_t prev_;
};

struct DevBuf {  // RAII device allocation from the stream-ordered pool (api.cu)
    void* p = nullptr;
    size_t bytes = 0;
    int device = 0;
    cudaStream_t stream = nullptr;  // last stream that may use the block (release is ordered after it)
    DevBuf() = default;
    explicit DevBuf(size_t b) { alloc(b); }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : p(o.p), bytes(o.bytes), device(o.device), stream(o.stream) { o.p = nullptr; o.bytes = 0; }
    DevBuf& operator=(DevBuf&& o) noexcept {
        reset(); p = o.p; bytes = o.bytes; device = o.device; stream = o.stream; o.p = nullptr; o.bytes = 0; return *this;
    }
    ~DevBuf() { reset(); }
    void alloc(size_t b);
    void reset();
    template <class T> T* as() const { return reinterpret_cast<T*>(p); }
};

struct Graph {
    Comm* comm = nullptr;
    int device = 0;
    uint32_t n = 0;
    uint64_t m = 0;
    int model = 0;
    DevBuf roff;   // u32[n+1]
    DevBuf rec;    // uint2[m] {src, thr (IC) | cum (LT)}
    // LT sparse walks: per-thread visited hash sets in global memory, entries tagged with a walk
    // epoch so no set is ever cleared between walks (zeroed once; re-zeroed when the epochs wrap).
    // Used under `walk_mu`; a call orders itself after the previous user by `walk_ev`.
    mutable DevBuf walk_ht;
    mutable uint32_t walk_epoch = 0;     // last epoch handed out
    mutable std::mutex walk_mu;
    mutable cudaEvent_t walk_ev = nullptr;
    // IC pull expansion: the forward edges with their canonical reverse ids,
    // uint4 {u, w, e, thr} per edge u -> w, grouped by u (built on first use, under pull_mu)
    mutable DevBuf pull_rec;
    // ... and its work list: every row u cut into segments of <= kPullSeg edges, uint4 {u, first
    // record, length, 0}, longest first (a warp's 32 segments have nearly equal lengths)
    mutable DevBuf pull_seg;
    mutable uint64_t pull_nseg = 0;
    mutable std::mutex pull_mu;
    ~Graph() { if (walk_ev) cudaEventDestroy(walk_ev); }
};

// Per-level device record of one batch (zeroed at batch start).
struct LevelRec {
    unsigned long long packed;   // kept entries << 36 | edges (or LT tasks) -- set by compaction
    unsigned long long vc;       // sum popc(mask) over raw entries (vertex-colour pairs)
    unsigned long long coins;    // coin evaluations by the expansion of this level
    unsigned long long atomics;  // atomicOr merges issued by the expansion of this level
    unsigned int raw;            // raw (discovered) entries of THIS level (queue appends, or the
                                 // touched vertices the bitmap compaction found)
    unsigned int overflow;       // set if a queue overflowed
    unsigned long long pad;      // stats copy: batch << 32 | level
    unsigned int any;            // touched-bitmap mode: some colour reached this level
    unsigned int pull;           // 1: this level was expanded by the pull kernel
    unsigned long long pull_reads;  // forward-edge records read by the pull expansion of this level
};
static_assert(sizeof(LevelRec) == 64, "LevelRec layout");
constexpr int kPackShift = 36;
constexpr int kLevelCols = 8;  // bpt_level_stats row width
constexpr unsigned long long kEdgeMask = (1ull << kPackShift) - 1;

struct Samples {
    const Graph* g = nullptr;   // valid only inside bpt_sample; the samples outlive the graph
    uint32_t n = 0;
    int device = 0;
    cudaStream_t stream = nullptr;  // stream of bpt_sample: every later call on the handle runs on it
    Comm* comm = nullptr;       // must outlive the samples (selection collectives)
    int model = 0;
    uint64_t theta = 0, seed = 0, s0 = 0, s1 = 0;
    uint32_t colors = 64;
    uint64_t blocks = 0;        // local 64-sample blocks
    uint64_t gb0 = 0;           // first global block
    DevBuf store;               // u64[blocks][n] visited masks (fused RRR store)
    DevBuf sizes;               // u32[s1 - s0]
    DevBuf digests;             // u64[s1 - s0]
    DevBuf count0;              // u32[n_pad]  occurrences: sum_s 1[v in RR_s] (local)
    uint32_t n_pad = 0;
    bpt_samples_info info{};
    std::vector<uint64_t> level_rows;  // kLevelCols per row (bpt_level_stats)
    std::vector<float> level_ms;       // expansion ms per level row (BPT_FLAG_PROFILE; bpt_level_times)
    // member lists of all local samples (selection on sparse stores), built on demand
    bool lists_built = false, lists_ok = false;
    bool digests_ready = false;
    DevBuf list_off, list_mem;
    // sparse LT store (BPT_FLAG_SPARSE): no dense store; the RRR sets ARE the sorted member
    // lists (list_off, list_mem); the selection uses a vertex -> samples index built on demand
    bool sparse = false;
    DevBuf inv_off, inv_s;
    // sorted start vertices (k_order.cu): the traversal slots (64 * local block + bit) hold the
    // samples in start order; store, per-slot kernels and selection work in slot order, every
    // per-sample output is mapped through these (identity when `sorted` is false)
    bool sorted = false;
    DevBuf slot_sample;   // u32[nlocal]: global sample id of local slot j
    DevBuf sample_slot;   // u32[nlocal]: local slot of local sample i
    std::vector<uint32_t> h_sample_slot;  // host copy, on demand (extraction)
    // batch-wide frontier: the finaliser leaves the per-sample sizes to a pass over the store blocks a
    // sizes / extraction / list request touches (ensure_sizes); blk_sized marks the blocks done
    bool lazy_sizes = false;
    std::vector<uint8_t> blk_sized;
    // multi-rank sparse selection: every rank's lists gathered once (offsets over all ranks'
    // samples, padded members, global occurrence counts)
    DevBuf g_off, g_mem, g_count0;
    uint64_t g_n = 0;
};

// ------------------------------------------------------------------ launchers
// k_build.cu
void build_reverse_csr(Graph& g, const uint64_t* d_row_ptr, const uint32_t* d_col, const float* d_wf,
                       const uint32_t* d_wq, cudaStream_t st);
// k_sample.cu
// Device-resident control block of the level / batch loops (read by every sampling kernel,
// advanced on the device, so the loops need no host round trip).
struct Ctl {
    uint32_t level;          // current level of the current batch
    uint32_t cont;           // 1 while the current batch has a non-empty frontier
    uint64_t blk0;           // first local 64-sample block of the current batch
    uint64_t gblk0;          // its global block index (sample base = 64 * (gblk0 + slot))
    uint32_t slots;          // blocks in the current batch
    uint32_t batch;          // batch index
    uint32_t error;          // 1 queue overflow, 2 too many levels
    uint32_t stats_used;     // level rows written to the stats buffer
    unsigned long long work, vc, coins, atomics, entries, levels_total;
    unsigned long long expand_ns;        // sum over expansion launches of (last end - first start)
    unsigned long long t_start, t_end;   // %globaltimer stamps of the running expansion launch
    unsigned long long c_start, c_end;   // ... of the running compaction launch
    unsigned long long compact_ns;       // sum over compaction launches of (last end - first start)
    uint32_t levels_max;
    uint32_t stats_overflow;
    uint32_t blocks_done;    // expansion blocks finished (the last one advances the level)
    uint32_t bar_count;      // grid barrier of the cooperative LT level loop: arrivals ...
    uint32_t bar_gen;        // ... and generation
    uint32_t pull_levels;    // levels expanded by the pull kernel
    unsigned long long kernels_run;  // kernel executions inside the sampling graph, counted by the
                                     // kernels themselves (block 0, thread 0 of every launch)
    unsigned long long pull_reads;   // forward-edge records read by pull levels
};
static_assert(sizeof(Ctl) % 16 == 0, "Ctl is read with 16-B vector loads");
constexpr int kMaxLevels = 8192;
constexpr uint32_t kPullSeg = 64;  // edges per pull segment (early exit per colour inside a segment)

struct BatchArgs {
    const uint32_t* roff;
    const uint2* rec;
    uint32_t n;
    int model;
    uint32_t colors;
    uint64_t* store;          // the local RRR store V[blocks][n] (written by the finaliser)
    ulonglong2* VN;           // per in-flight block working masks {V visited, N next frontier} [slots][n]:
                              // V[u] and N[u] share one 32-B sector (one gather, one atomic target)
    unsigned long long* raw;  // raw queue entries
    uint64_t raw_cap;
    uint4* q;                 // compacted entries {v, slot, mask lo, mask hi}
    uint32_t* umask;          // IC: bit t set iff a frontier entry's work starts at item t
    uint64_t* qoff;           // exclusive prefix of per-entry work
    uint64_t q_cap;
    LevelRec* lv;             // level records of the current batch (kMaxLevels)
    LevelRec* stats;          // copy of every level record, tagged (batch << 32 | level) in .pad
    uint32_t stats_cap;
    uint32_t slots_max;       // blocks per batch
    uint64_t blocks;          // local blocks of this rank
    Ctl* ctl;
    uint64_t theta;           // global sample count (bits of samples >= theta stay 0)
    uint32_t k_ic, k_lt, k_start;
    uint32_t ic_keys[10];     // Philox key schedule of k_ic: ic_keys[r] = k_ic + r * W (reading C-1)
    // wide fusion (IC, 64 colours): the slots_max = kWide blocks of a
    // batch share one frontier. Working masks vertex-major VN[v * kWide + b]; one frontier entry
    // per vertex with kWide masks; vflag[v] = v already queued for the next level.
    int wide;                 // 0: slot-major layout (one entry per (vertex, block, slice))
    uint32_t* vflag;
    uint32_t* qd;             // entry: rowstart - work offset (edge id = item + qd)
    unsigned long long* qmask;  // entry masks [j * kWide + b]
    // touched-bitmap mode (IC, 64 colours, slot-major): the expansion merges with fire-and-forget
    // ORs and marks every vertex whose N it makes non-empty in touched[slot * tile_words + v / 32];
    // the compaction scans the bitmap (1,024-vertex tiles) instead of a queue of first setters
    uint32_t* touched;        // nullptr: queue mode
    // union layout (bitmap mode): the working masks are U[slot][n] = V | N (gathered by the
    // expansion, 8 B per vertex) followed by V[slot][n] (read / written by the compaction only),
    // in the VN allocation; new colours of a touched vertex = U & ~V
    uint32_t tiles;           // 1,024-vertex tiles per slot (tile_words = 32 * tiles)
    int lt_persist;           // LT fused loop: one cooperative launch per batch
    const uint32_t* slot_sample;  // sorted start vertices: global sample id of each local slot (nullptr:
                                  // slot 64 * local block + bit holds sample 64 * global block + bit)
    uint64_t nlocal;          // local samples
    uint64_t m;               // edges (bounds of rec[], checked in BPT_CHECKS builds)
    uint64_t umask_words;     // words of umask[]
    uint64_t tstart_cap;      // entries of tstart[]
    int lt_blocks_per_sm;     // ... with this many blocks per SM
    // pull expansion (touched-bitmap mode only): levels whose push work
    // (frontier edge reads) is >= pull_min_work are expanded by streaming every forward edge u -> w
    // once for all slots of the batch; the compaction keeps F exact for every level
    const uint4* pull;        // forward records {u, w, e, thr} (nullptr: push only)
    uint64_t pull_edges;      // forward records (= m)
    const uint4* pull_seg;    // row segments {u, first record, length, 0}, longest first
    uint64_t pull_nseg;
    uint64_t pull_min_work;
    unsigned long long* F;    // frontier masks of the current level, vertex-major F[v * slots_max + slot]
    uint32_t* FB;             // touched words of the previous level (same layout as touched)
    // batch-wide frontier (IC, 64 colours, touched-bitmap mode): the slots_max
    // blocks of a batch share ONE frontier. Vertex-major union layout U[v * S + slot] (then V at
    // S * n), one touched bit per vertex, one entry per frontier vertex with S masks (qd, qmask):
    // every reverse edge of a frontier vertex is read once for all 64 S colours
    int vmajor;
};
#ifndef BPT_WIDE_BLOCKS
#define BPT_WIDE_BLOCKS 2
#endif
constexpr uint32_t kWide = BPT_WIDE_BLOCKS;  // blocks (x 64 colours) per wide frontier entry (even)
#ifndef BPT_UNIT_WIDE
#define BPT_UNIT_WIDE 64
#endif
constexpr uint32_t kUnitWide = BPT_UNIT_WIDE;  // work items per wide expansion unit (windows of 32)
// k_store.cu
// per-sample sizes of local samples [first, first + count) present in S.sizes (a no-op unless S.lazy_sizes)
void ensure_sizes(Samples& S, uint64_t first, uint64_t count, cudaStream_t st);
// umode: 0 {V, N} pairs, 1 slot-major union layout, 2 vertex-major union layout (a.vmajor)
void launch_finalize(const Samples& S, ulonglong2* VN, const Ctl* ctl, uint32_t slots_max, const uint32_t* roff,
                     cudaStream_t st, unsigned long long* d_elog, bool wide, int umode);
void add_store_nodes(cudaGraph_t g, cudaGraphNode_t dep, const Samples& S, ulonglong2* VN, const Ctl* ctl,
                     uint32_t slots_max, const uint32_t* roff, unsigned long long* d_elog, cudaGraphNode_t* last,
                     bool wide, int umode);
// k_build.cu: forward records of the pull expansion (Graph::pull_rec), from the reverse CSR
void build_pull_records(const Graph& g, cudaStream_t st);
// k_sample.cu: host-driven level loop (profiling with CUDA events) and the device-resident graph
void launch_init(const BatchArgs& a, cudaStream_t st);
void launch_level(const BatchArgs& a, uint32_t* tstart, uint64_t tstart_cap, cudaStream_t st, cudaEvent_t ev0,
                  cudaEvent_t ev1);
void launch_next_batch(const BatchArgs& a, cudaStream_t st);
struct StoreHook {  // adds the per-batch finalise nodes after the level loop
    const Samples* S;
    ulonglong2* VN;
    const uint32_t* roff;
    unsigned long long* d_elog;
    bool wide;
};
bool level_loop_persistent(const BatchArgs& a);
// LT: every local sample's reverse walk in one launch (store must be zero; sizes written;
// totals[0] += members, totals[1] = max walk length)
void launch_walk_lt(uint64_t* store, uint32_t n, const uint32_t* roff, const uint2* rec, uint64_t s0, uint64_t nlocal,
                    uint32_t k_start, uint32_t k_lt, uint32_t* sizes, uint32_t* count0, unsigned long long* totals,
                    cudaStream_t st);
// LT sparse store: walks with a per-thread visited hash set (no dense store); sizes, count0,
// totals[0..1] as launch_walk_lt, totals[2] = 1 if a walk outgrew the hash set
// `g`'s walk tables (Graph::walk_ht) hold the visited sets
void launch_walk_lt_sparse(const Graph& g, uint64_t s0, uint64_t nlocal,
                           uint32_t k_start, uint32_t k_lt, uint32_t* sizes, uint32_t* count0,
                           unsigned long long* totals, uint32_t* rows, cudaStream_t st);
// walk-order member rows (optional output of the sparse walk: stride walk_row_stride()) -> lists
uint32_t walk_row_stride();
void launch_rows_to_lists(const uint32_t* rows, const uint64_t* off, uint64_t nlists, uint32_t* members, cudaStream_t st);
// sort every list ascending in place (one block per list of <= 4096 members; longer lists set *err)
void launch_sort_lists(const uint64_t* off, uint32_t* members, uint64_t nlists, uint32_t* err, cudaStream_t st);
// LT: re-walk every local sample and write its members at off[i] (unsorted; for the selection)
void launch_walk_lt_lists(uint32_t n, const uint32_t* roff, const uint2* rec, uint32_t m, uint64_t s0, uint64_t nlocal,
                          uint32_t k_start, uint32_t k_lt, const uint32_t* sizes, const uint64_t* off,
                          uint32_t* members, cudaStream_t st);
// k_order.cu: sorted start vertices
void sort_slots(const uint32_t* roff, uint32_t n, uint64_t s0, uint64_t nlocal, uint32_t k_start,
                uint32_t* slot_sample, uint32_t* sample_slot, cudaStream_t st);
cudaGraphExec_t build_sampling_graph(const BatchArgs& a, uint32_t* tstart, uint64_t tstart_cap, const StoreHook& h);
// k_select.cu
void select_seeds(const Samples& S, uint32_t k, uint32_t* h_seeds, uint64_t* h_gains, cudaStream_t st);

int num_sms();
void release_cached_blocks();
size_t cached_bytes();  // bytes held by the device-memory pool of the current device
size_t free_estimate(); // free device memory (cudaMemGetInfo snapshot minus this library's allocations since)

}  // namespace bpt
