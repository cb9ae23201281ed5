// api.cu -- the C-ABI of include/bpt.h and the host orchestration of the hot path:
// argument checks, host/device pointer handling, sample-range sharding, batch planning,
// the device-resident level loop with pipelined polling, and statistics.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>

#include "internal.cuh"

namespace bpt {
#ifndef BPT_PULL_ALPHA
#define BPT_PULL_ALPHA 1.0
#endif
constexpr double kPullAlpha = BPT_PULL_ALPHA;  // pull levels: push work >= kPullAlpha * m

// ------------------------------------------------------------------ errors
thread_local std::string g_last_error;
uint64_t g_launches = 0;
uint64_t g_graph_kernels = 0;

void fail(bpt_status code, const std::string& msg) { throw Error{code, msg}; }

void check_cuda(cudaError_t e, const char* what) {
    if (e == cudaSuccess) return;
    cudaGetLastError();  // clear sticky-free errors
    if (e == cudaErrorMemoryAllocation) fail(BPT_ENOMEM, std::string("device allocation failed: ") + what);
    fail(BPT_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

// ------------------------------------------------------------------ device memory pool
// Freed device blocks are cached per device and reused for later requests of a similar size
// (best fit within +25%), so repeated bpt_graph_load / bpt_sample calls do not pay
// cudaMalloc/cudaFree of multi-GB stores each time. Recycling is stream-ordered: a block
// remembers the stream of the API call that used it (StreamScope); when it is released an
// event is recorded on that stream, and the next call that takes the block makes its own
// stream wait on that event, so a block is never handed out while a kernel queued before
// its release may still touch it (no host synchronisation needed).
// On allocation failure the cache is released (after its events complete) and the
// allocation retried.
thread_local cudaStream_t g_cur_stream = nullptr;

StreamScope::StreamScope(cudaStream_t st) : prev_(g_cur_stream) { g_cur_stream = st; }
StreamScope::~StreamScope() { g_cur_stream = prev_; }

namespace {
struct Cached {
    void* p;
    cudaEvent_t ev;  // recorded on the releasing stream (nullptr: nothing pending)
};
struct Pool {
    std::mutex mu;
    std::multimap<size_t, Cached> free_blocks[64];  // per device: size -> block
    size_t cached[64] = {};
    size_t held[64] = {};   // bytes this library holds from cudaMalloc (in use + cached)
    // free-memory estimate (free_estimate): one cudaMemGetInfo snapshot per device and the bytes
    // held at that moment; the snapshot is refreshed every kMemInfoTtl seconds
    double snap_t[64] = {};
    size_t snap_free[64] = {}, snap_held[64] = {};
};
Pool& pool() {
    static Pool* p = new Pool();  // never destroyed: the CUDA context may be gone at exit
    return *p;
}
size_t round_size(size_t b) {
    if (b < 8) b = 8;
    const size_t g = b >= (64u << 20) ? (2u << 20) : 512;
    return (b + g - 1) / g * g;
}
int current_device() {
    int d = 0;
    cudaGetDevice(&d);
    return d < 0 || d >= 64 ? 0 : d;
}
}  // namespace

// Free device memory, estimated without a cudaMemGetInfo per call (it stalled bpt_sample and the
// selection for 10-40 ms at times, on every rank of a multi-GPU step): the last snapshot's free
// bytes minus what this library allocated since (other allocators are seen at the next refresh)
size_t free_estimate() {
    constexpr double kMemInfoTtl = 30.0;
    Pool& P = pool();
    const int dev = current_device();
    const double now = std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
    std::lock_guard<std::mutex> lk(P.mu);
    if (P.snap_t[dev] == 0.0 || now - P.snap_t[dev] > kMemInfoTtl) {
        size_t f = 0, t = 0;
        if (cudaMemGetInfo(&f, &t) != cudaSuccess) { cudaGetLastError(); f = 0; }
        P.snap_t[dev] = now;
        P.snap_free[dev] = f;
        P.snap_held[dev] = P.held[dev];
    }
    const long long est = (long long)P.snap_free[dev] - ((long long)P.held[dev] - (long long)P.snap_held[dev]);
    return est > 0 ? (size_t)est : 0;
}

size_t cached_bytes() {
    Pool& P = pool();
    std::lock_guard<std::mutex> lk(P.mu);
    return P.cached[current_device()];
}

void release_cached_blocks() {
    Pool& P = pool();
    std::lock_guard<std::mutex> lk(P.mu);
    int cur = current_device();
    for (int d = 0; d < 64; ++d) {
        if (P.free_blocks[d].empty()) continue;
        cudaSetDevice(d);
        for (auto& kv : P.free_blocks[d]) {
            if (kv.second.ev) {
                cudaEventSynchronize(kv.second.ev);
                cudaEventDestroy(kv.second.ev);
            }
            cudaFree(kv.second.p);
            P.held[d] -= kv.first;
        }
        P.free_blocks[d].clear();
        P.cached[d] = 0;
    }
    cudaSetDevice(cur);
}

void DevBuf::alloc(size_t b) {
    reset();
    b = round_size(b);
    const int dev = current_device();
    {
        Pool& P = pool();
        std::lock_guard<std::mutex> lk(P.mu);
        auto it = P.free_blocks[dev].lower_bound(b);
        if (it != P.free_blocks[dev].end() && it->first <= b + b / 4) {
            p = it->second.p;
            bytes = it->first;
            if (it->second.ev) {  // work queued before the release must finish first
                cudaStreamWaitEvent(g_cur_stream, it->second.ev, 0);
                cudaEventDestroy(it->second.ev);
            }
            P.cached[dev] -= bytes;
            P.free_blocks[dev].erase(it);
            device = dev;
            stream = g_cur_stream;
            return;
        }
    }
    cudaError_t e = cudaMalloc(&p, b);
    if (e == cudaErrorMemoryAllocation) {
        cudaGetLastError();
        release_cached_blocks();
        e = cudaMalloc(&p, b);
    }
    if (e != cudaSuccess) {
        p = nullptr;
        cudaGetLastError();
        if (e == cudaErrorMemoryAllocation)
            fail(BPT_ENOMEM, "cudaMalloc of " + std::to_string(b) + " bytes failed (out of device memory)");
        fail(BPT_ECUDA, std::string("cudaMalloc: ") + cudaGetErrorString(e));
    }
    bytes = b;
    device = dev;
    stream = g_cur_stream;
    Pool& P = pool();
    std::lock_guard<std::mutex> lk(P.mu);
    P.held[dev] += b;
}
void DevBuf::reset() {
    if (p) {
        cudaEvent_t ev = nullptr;
        int cur = -1;
        cudaGetDevice(&cur);
        if (cur != device) cudaSetDevice(device);
        if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) == cudaSuccess) {
            if (cudaEventRecord(ev, stream) != cudaSuccess) {  // cannot order: wait for the device
                cudaEventDestroy(ev);
                ev = nullptr;
                cudaDeviceSynchronize();
            }
        } else {
            ev = nullptr;
            cudaDeviceSynchronize();
        }
        cudaGetLastError();
        if (cur != device && cur >= 0) cudaSetDevice(cur);
        Pool& P = pool();
        std::lock_guard<std::mutex> lk(P.mu);
        P.free_blocks[device].emplace(bytes, Cached{p, ev});
        P.cached[device] += bytes;
    }
    p = nullptr;
    bytes = 0;
}

int num_sms() {
    int dev = 0, sms = 0;
    BPT_CUDA(cudaGetDevice(&dev));
    BPT_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    return sms;
}

// launchers defined in other translation units
uint32_t expand_unit(int model, bool bitmap);
void launch_compact(const BatchArgs& a, int level, uint32_t* tstart, uint64_t tstart_cap, cudaStream_t st);
void launch_expand(const BatchArgs& a, int level, const uint32_t* tstart, cudaStream_t st);
void extract_range(const Samples& S, uint64_t first, uint64_t count, const uint64_t* h_offsets, uint32_t* d_members,
                   cudaStream_t st);
void compute_digests(const Samples& S, cudaStream_t st);
void comm_unique_id(void* out);
#ifdef BPT_HIST
void dump_hist();
#endif
void selftest_philox(const uint32_t* d_in, uint32_t* d_out, uint64_t count, cudaStream_t st);
double bench_philox(uint64_t iters, uint64_t* calls_out, cudaStream_t st);
void comm_init(Comm* c, const void* uid);
void comm_destroy(Comm* c);
void comm_broadcast(Comm* c, const void* send, void* recv, uint64_t bytes, int root, cudaStream_t st);
void comm_allreduce_max_u64(Comm* c, unsigned long long* buf, uint64_t count, cudaStream_t st);

namespace {

bool is_device_ptr(const void* p) {
    if (!p) return false;
    cudaPointerAttributes a{};
    cudaError_t e = cudaPointerGetAttributes(&a, p);
    if (e != cudaSuccess) { cudaGetLastError(); return false; }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// device view of a caller array: the pointer itself if on the device, else a copy
struct DevIn {
    DevBuf buf;
    const void* p = nullptr;
    DevIn(const void* src, size_t bytes, cudaStream_t st) {
        if (!src) return;
        if (is_device_ptr(src)) { p = src; return; }
        buf.alloc(bytes);
        BPT_CUDA(cudaMemcpyAsync(buf.p, src, bytes, cudaMemcpyHostToDevice, st));
        p = buf.p;
    }
};

void copy_out(void* dst, const void* dsrc, size_t bytes, cudaStream_t st) {
    if (!dst || !bytes) return;
    BPT_CUDA(cudaMemcpyAsync(dst, dsrc, bytes, is_device_ptr(dst) ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, st));
}

void use_device(int dev) {
    int cur = -1;
    BPT_CUDA(cudaGetDevice(&cur));
    if (cur != dev) BPT_CUDA(cudaSetDevice(dev));
}

// Restores the caller's current device when an API call returns (calls switch to the
// device of the handle they operate on).
struct DeviceGuard {
    int dev = -1;
    DeviceGuard() { if (cudaGetDevice(&dev) != cudaSuccess) { dev = -1; cudaGetLastError(); } }
    ~DeviceGuard() { if (dev >= 0) cudaSetDevice(dev); }
};

template <class F>
bpt_status guarded(F&& f) {
    // a pending error recorded by an earlier (unchecked) runtime call must not be
    // attributed to this call's first launch check; keep it for the message
    const cudaError_t stale = cudaGetLastError();
    DeviceGuard restore_device;
    try {
        f();
        return BPT_OK;
    } catch (const Error& e) {
        g_last_error = e.msg;
        if (stale != cudaSuccess) g_last_error += std::string(" [pending before this call: ") + cudaGetErrorString(stale) + "]";
        return e.code;
    } catch (const std::bad_alloc&) {
        g_last_error = "host allocation failed";
        return BPT_ENOMEM;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return BPT_ECUDA;
    }
}



}  // namespace

using clk_t = std::chrono::steady_clock;

static uint64_t device_total_bytes() {  // cached per device
    static uint64_t total[64] = {};
    int d = 0;
    BPT_CUDA(cudaGetDevice(&d));
    if (d < 0 || d >= 64) d = 0;
    if (!total[d]) {
        cudaDeviceProp p{};
        BPT_CUDA(cudaGetDeviceProperties(&p, d));
        total[d] = p.totalGlobalMem;
    }
    return total[d];
}

// timing of one walk launch (events released on every path)
struct WalkTimer {
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    explicit WalkTimer(cudaStream_t st) {
        BPT_CUDA(cudaEventCreate(&e0));
        BPT_CUDA(cudaEventCreate(&e1));
        BPT_CUDA(cudaEventRecord(e0, st));
    }
    void stop(cudaStream_t st) { BPT_CUDA(cudaEventRecord(e1, st)); }
    float ms() const {
        float t = 0;
        BPT_CUDA(cudaEventElapsedTime(&t, e0, e1));
        return t;
    }
    ~WalkTimer() {
        if (e0) cudaEventDestroy(e0);
        if (e1) cudaEventDestroy(e1);
    }
};

// member lists of the local samples in walk order (a second walk of known length), offsets from
// the sizes the first walk wrote
static void lt_lists_by_rewalk(Samples& S, cudaStream_t st) {
    const Graph& g = *S.g;
    const uint64_t nlocal = S.s1 - S.s0;
    std::vector<uint32_t> sz(nlocal);
    BPT_CUDA(cudaMemcpy(sz.data(), S.sizes.p, nlocal * 4, cudaMemcpyDeviceToHost));
    std::vector<uint64_t> off(nlocal + 1, 0);
    for (uint64_t i = 0; i < nlocal; ++i) off[i + 1] = off[i] + sz[i];
    S.list_off.alloc((nlocal + 1) * 8);
    S.list_mem.alloc(off[nlocal] * 4 + 4);
    BPT_CUDA(cudaMemcpyAsync(S.list_off.p, off.data(), (nlocal + 1) * 8, cudaMemcpyHostToDevice, st));
    launch_walk_lt_lists(g.n, g.roff.as<uint32_t>(), g.rec.as<uint2>(), (uint32_t)g.m, S.s0, nlocal, stream_key(S.seed, kTagStart),
                         stream_key(S.seed, kTagLT), S.sizes.as<uint32_t>(), S.list_off.as<uint64_t>(),
                         S.list_mem.as<uint32_t>(), st);
    S.lists_built = S.lists_ok = true;
}

static void lt_walk_info(Samples& S, const unsigned long long* tot, float ms, uint64_t launches0,
                         clk_t::time_point t_begin, const char* label) {
    bpt_samples_info& I = S.info;
    I.members = I.frontier_entries = tot[0];
    I.coins = tot[0];    // one coinLT draw per member vertex
    I.atomics = tot[0];  // one visited-set insertion per member vertex
    I.e_phys = I.e_logical = tot[0];  // (vertex, colour) expansions, SURVEY §8(d)
    I.levels_total = I.levels_max = tot[1];
    I.batch_groups = (uint32_t)S.blocks;
    I.batches = 1;
    I.store_bytes = S.sparse ? S.list_mem.bytes + S.list_off.bytes : S.store.bytes;
    I.ms_expand = ms;
    I.expand_launches = 1;
    I.expand_bytes = 24.0 * (double)tot[0];  // row bounds 8 + chosen record 8 + visited RMW 8 per member
    S.level_rows.clear();
    I.kernel_launches = g_launches - launches0;
    I.ms_total = std::chrono::duration<double, std::milli>(clk_t::now() - t_begin).count();
    if (getenv("BPT_TRACE"))
        fprintf(stderr, "[bpt] sample (%s): %llu members, longest %llu, walks %.2f ms, total %.2f ms\n", label, tot[0],
                tot[1], ms, I.ms_total);
}

// LT, sparse store: walks with per-thread visited hash sets, sorted member lists as the store.
// Returns false (counts undone) when a walk outgrew the visited set and the flag allows the dense
// store instead.
static bool run_lt_walks_sparse(Samples& S, const bpt_sample_opts& opt, cudaStream_t st, clk_t::time_point t_begin,
                                uint64_t launches0) {
    const Graph& g = *S.g;
    const uint64_t nlocal = S.s1 - S.s0;
    DevBuf totals(24), rows;
    BPT_CUDA(cudaMemsetAsync(totals.p, 0, 24, st));
    auto since = [&]() { return std::chrono::duration<double, std::milli>(clk_t::now() - t_begin).count(); };
    const double t_pre = since();
    if (!(opt.flags & BPT_FLAG_LT_REWALK)) {
        // walk-order rows written during the walk (6 KB per sample) when they fit a quarter of
        // the device memory and the allocation succeeds, else the lists come from a second walk
        // (no cudaMemGetInfo here: it stalled the call for 10-40 ms at times)
        const uint64_t bytes = nlocal * (uint64_t)walk_row_stride() * 4;
        if (bytes < device_total_bytes() / 4) {
            try {
                rows.alloc(bytes);
            } catch (const Error& e) {
                if (e.code != BPT_ENOMEM) throw;
            }
        }
    }
    const double t_alloc = since();
    WalkTimer tm(st);
    launch_walk_lt_sparse(g, S.s0, nlocal, stream_key(S.seed, kTagStart),
                          stream_key(S.seed, kTagLT), S.sizes.as<uint32_t>(), S.count0.as<uint32_t>(),
                          totals.as<unsigned long long>(), rows.p ? rows.as<uint32_t>() : nullptr, st);
    tm.stop(st);
    const double t_launch = since();
    unsigned long long tot[3] = {0, 0, 0};
    BPT_CUDA(cudaMemcpyAsync(tot, totals.p, 24, cudaMemcpyDeviceToHost, st));
    BPT_CUDA(cudaStreamSynchronize(st));
    const double t_walk_ms = std::chrono::duration<double, std::milli>(clk_t::now() - t_begin).count();
    if (tot[2]) {
        if (opt.flags & BPT_FLAG_SPARSE)
            fail(BPT_ENOMEM, "an LT walk is longer than the sparse store's visited set; sample without "
                             "BPT_FLAG_SPARSE");
        BPT_CUDA(cudaMemsetAsync(S.count0.p, 0, (size_t)S.n_pad * 4, st));  // undo this attempt
        BPT_CUDA(cudaMemsetAsync(S.sizes.p, 0, nlocal * 4, st));
        return false;
    }
    if (rows.p) {
        std::vector<uint32_t> sz(nlocal);
        BPT_CUDA(cudaMemcpy(sz.data(), S.sizes.p, nlocal * 4, cudaMemcpyDeviceToHost));
        std::vector<uint64_t> off(nlocal + 1, 0);
        for (uint64_t i = 0; i < nlocal; ++i) off[i + 1] = off[i] + sz[i];
        S.list_off.alloc((nlocal + 1) * 8);
        S.list_mem.alloc(off[nlocal] * 4 + 4);
        BPT_CUDA(cudaMemcpyAsync(S.list_off.p, off.data(), (nlocal + 1) * 8, cudaMemcpyHostToDevice, st));
        launch_rows_to_lists(rows.as<uint32_t>(), S.list_off.as<uint64_t>(), nlocal, S.list_mem.as<uint32_t>(), st);
        S.lists_built = S.lists_ok = true;
    } else {
        lt_lists_by_rewalk(S, st);
    }
    // lists stay in walk order: sizes, digests and the selection do not depend on the order;
    // bpt_rrr_extract sorts the range it returns
    BPT_CUDA(cudaStreamSynchronize(st));
    if (getenv("BPT_TRACE"))
        fprintf(stderr, "[bpt] LT sparse: rows %s, set-up %.2f, rows alloc %.2f, launched %.2f, walk ends %.2f, "
                "lists end %.2f ms after call start\n", rows.p ? "yes" : "no", t_pre, t_alloc, t_launch, t_walk_ms, since());
    S.sparse = true;
    lt_walk_info(S, tot, tm.ms(), launches0, t_begin, "LT sparse walks");
    return true;
}

// LT, dense store: sample s's bit in the RRR store is its visited set; member lists for the
// selection's decrement by re-walking (cheaper than a pass over the dense store)
static void run_lt_walks_dense(Samples& S, cudaStream_t st, clk_t::time_point t_begin, uint64_t launches0) {
    const Graph& g = *S.g;
    const uint64_t nlocal = S.s1 - S.s0;
    S.store.alloc((size_t)S.blocks * g.n * 8);
    BPT_CUDA(cudaMemsetAsync(S.store.p, 0, S.store.bytes, st));
    DevBuf totals(16);
    BPT_CUDA(cudaMemsetAsync(totals.p, 0, 16, st));
    WalkTimer tm(st);
    launch_walk_lt(S.store.as<uint64_t>(), g.n, g.roff.as<uint32_t>(), g.rec.as<uint2>(), S.s0, nlocal,
                   stream_key(S.seed, kTagStart), stream_key(S.seed, kTagLT), S.sizes.as<uint32_t>(),
                   S.count0.as<uint32_t>(), totals.as<unsigned long long>(), st);
    tm.stop(st);
    unsigned long long tot[2] = {0, 0};
    BPT_CUDA(cudaMemcpyAsync(tot, totals.p, 16, cudaMemcpyDeviceToHost, st));
    BPT_CUDA(cudaStreamSynchronize(st));
    lt_lists_by_rewalk(S, st);
    BPT_CUDA(cudaStreamSynchronize(st));
    lt_walk_info(S, tot, tm.ms(), launches0, t_begin, "LT walks");
}

// ------------------------------------------------------------------ sampling driver
static void run_sampling(Samples& S, const bpt_sample_opts& opt, cudaStream_t st) {
    const Graph& g = *S.g;
    const uint32_t n = g.n;
    const uint32_t C = S.colors;
    const uint64_t slices = 64 / C;
    const auto t_begin = std::chrono::steady_clock::now();
    const uint64_t launches0 = g_launches;

    // ---- store + per-sample outputs
    S.count0.alloc((size_t)S.n_pad * 4);
    BPT_CUDA(cudaMemsetAsync(S.count0.p, 0, (size_t)S.n_pad * 4, st));
    if (S.blocks == 0) {  // this rank owns no samples; it still joins the selection collectives
        BPT_CUDA(cudaStreamSynchronize(st));
        return;
    }
    const uint64_t nlocal = S.s1 - S.s0;
    S.sizes.alloc(nlocal * 4);
    S.digests.alloc(nlocal * 8);
    BPT_CUDA(cudaMemsetAsync(S.sizes.p, 0, nlocal * 4, st));

    // ---- LT: one reverse walk per thread (k_sample.cu "LT reverse walks"). Default: the sparse
    //      member-list store, falling back to the dense store when a walk outgrows the per-thread
    //      visited set (BPT_FLAG_SPARSE: fail instead); BPT_LT_DENSE=1 walks into the dense store;
    //      BPT_LT_FUSED=1 runs the level-synchronous fused loop below (same sets).
    if (S.model == BPT_LT) {
        const bool fused = (opt.flags & BPT_FLAG_LT_FUSED) != 0;
        const bool want_sparse = (opt.flags & BPT_FLAG_SPARSE) || (!(opt.flags & BPT_FLAG_LT_DENSE) && !fused);
        if (want_sparse && run_lt_walks_sparse(S, opt, st, t_begin, launches0)) return;
        if (!fused) {
            run_lt_walks_dense(S, st, t_begin, launches0);
            return;
        }
    }
    S.store.alloc((size_t)S.blocks * n * 8);  // fully written by the finaliser, no memset

    // ---- batch plan
    // wide fusion (IC, 64 colours): kWide blocks share one frontier (k_sample.cu "wide fusion")
    const bool wide = S.model == BPT_IC && C == 64 && !opt.batch_groups && (opt.flags & BPT_FLAG_WIDE);
    // touched-bitmap frontier (IC, 64 colours; k_sample.cu "A4: compaction")
    const bool bitmap = S.model == BPT_IC && C == 64 && !wide && !(opt.flags & BPT_FLAG_QUEUE);
    // IC: a few 64-sample blocks per batch -- the union-layout masks U (8 B per vertex and block) of
    // 4 blocks are gathered at ~85% L2 hits, and 4x fewer batches cut the per-level and per-batch
    // fixed costs (C2, theta = 8192: 253 vs 283 ms); the queue form keeps one block
    // ({V, N} pairs, 16 B). LT: as many as fit (fewer, longer levels: LT frontiers are thin).
    uint64_t want = opt.batch_groups ? opt.batch_groups : (S.model == BPT_IC ? (bitmap ? 4 : 1) : 2048);
    if (wide) want = kWide;
    uint64_t slots = wide ? kWide : umin64(umax64(want, 1), S.blocks);
    const uint32_t tile = wide ? kUnitWide : expand_unit(S.model, bitmap);
    const uint64_t tiles = (n + 1023) / 1024;  // bitmap: 1,024-vertex tiles per slot
    // batch-wide frontier (IC, 64 colours, bitmap form, <= 4 blocks per batch; k_sample.cu "Batch-wide
    // frontier"): the default; BPT_FLAG_SLOTWISE (and the pull form) keep one frontier per block
    bool vmajor = bitmap && !(opt.flags & BPT_FLAG_SLOTWISE) && !(opt.flags & BPT_FLAG_PULL);
    auto plan_bytes = [&](uint64_t sl, uint64_t& raw_cap, uint64_t& q_cap, uint64_t& ts_cap) {
        const bool vm = vmajor && sl <= 4;
        raw_cap = umin64(wide || vm ? n : sl * slices * n, (1ull << 28) - 1);  // wide / vmajor: one entry per vertex
        q_cap = raw_cap;
        if (bitmap) raw_cap = 1;  // no queue
        const uint64_t work = S.model == BPT_IC ? umin64((wide || vm ? 1 : sl * slices) * g.m, kEdgeMask)
                                                : umin64(sl * 64 * n, kEdgeMask);
        ts_cap = work / tile + 2;
        return sl * (uint64_t)n * 16 + raw_cap * 8 + q_cap * (vm ? 4 + 8 * sl : 16 + 8) + ts_cap * 20 +
               (bitmap ? (vm ? 1 : sl) * tiles * 128 : 0);
    };
    size_t free_b = free_estimate();
    free_b += cached_bytes();  // the pool's cached blocks are released if an allocation needs them
    // pull expansion of the heavy levels (BPT_FLAG_PULL; touched-bitmap form): forward records
    // (16 B per edge, cached on the graph) + vertex-major frontier masks + the previous level's
    // touched words, when they fit beside the batch (else push only)
    bool pull = bitmap && (opt.flags & BPT_FLAG_PULL) && g.m > 0;
    if (pull) {
        const uint64_t extra = (g.pull_rec.p ? 0 : g.m * 16 + g.m * 24) + (uint64_t)want * n * 8 + want * tiles * 128;
        if (extra > free_b / 2) pull = false;
        else free_b -= extra;
    }
    uint64_t raw_cap = 0, q_cap = 0, ts_cap = 0;
    while (!wide && slots > 1 && plan_bytes(slots, raw_cap, q_cap, ts_cap) > free_b * 0.85) slots /= 2;
    while (!wide && slots > 1 && slots * (uint64_t)n >= (1ull << 32)) slots /= 2;  // 32-bit working-mask indices
    if (wide && (uint64_t)kWide * n >= (1ull << 32)) fail(BPT_EINVAL, "wide fusion needs kWide * n < 2^32");
    if (slots > 4 || n >= (1u << 30)) vmajor = false;  // items pack u | slot << 30
    plan_bytes(slots, raw_cap, q_cap, ts_cap);

    const uint64_t nbatches = (S.blocks + slots - 1) / slots;
    const uint32_t stats_cap = (uint32_t)umin64(nbatches * 64 + 8192, 1ull << 22);
    DevBuf VN((size_t)slots * n * 16), raw(raw_cap * 8), q(vmajor ? 16 : q_cap * 16), qoff(vmajor ? 16 : q_cap * 8),
        tstart(ts_cap * 4),
        umask(S.model == BPT_IC ? (ts_cap * tile / 32 + 4) * 4 : 16),
        lv((size_t)kMaxLevels * sizeof(LevelRec)), stats((size_t)stats_cap * sizeof(LevelRec)), ctl(sizeof(Ctl)),
        elog(8);
    BPT_CUDA(cudaMemsetAsync(VN.p, 0, VN.bytes, st));  // the finaliser re-zeroes it after every batch
    DevBuf vflag, qd, qmask, touched, Fbuf, FBbuf;
    if (vmajor) {
        qd.alloc(q_cap * 4 + 4);
        qmask.alloc(q_cap * slots * 8 + 16);
    }
    if (bitmap) {
        touched.alloc((vmajor ? 1 : slots) * tiles * 128);
        BPT_CUDA(cudaMemsetAsync(touched.p, 0, touched.bytes, st));  // the compaction clears what it reads
    }
    if (pull) {
        build_pull_records(g, st);
        Fbuf.alloc(slots * (uint64_t)n * 8);
        FBbuf.alloc(slots * tiles * 128);
        BPT_CUDA(cudaMemsetAsync(Fbuf.p, 0, Fbuf.bytes, st));  // then kept exact by every compaction
        BPT_CUDA(cudaMemsetAsync(FBbuf.p, 0, FBbuf.bytes, st));
    }
    if (wide) {
        vflag.alloc((uint64_t)n * 4 + 4);
        qd.alloc(q_cap * 4 + 4);
        qmask.alloc(q_cap * kWide * 8 + 16);
        BPT_CUDA(cudaMemsetAsync(vflag.p, 0, vflag.bytes, st));  // the compaction re-zeroes what it reads
    }
    BPT_CUDA(cudaMemsetAsync(lv.p, 0, lv.bytes, st));  // k_next_batch re-zeroes the levels it used
    BPT_CUDA(cudaMemsetAsync(umask.p, 0, umask.bytes, st));  // the expansion re-zeroes every unit it reads
    BPT_CUDA(cudaMemsetAsync(elog.p, 0, 8, st));
    Ctl c0{};
    c0.slots = (uint32_t)umin64(slots, S.blocks);
    c0.gblk0 = S.gb0;
    c0.t_start = ~0ull;
    c0.c_start = ~0ull;
    static thread_local Ctl* c_host = nullptr;
    if (!c_host) BPT_CUDA(cudaMallocHost(&c_host, sizeof(Ctl)));
    *c_host = c0;
    BPT_CUDA(cudaMemcpyAsync(ctl.p, c_host, sizeof(Ctl), cudaMemcpyHostToDevice, st));
    using clk = std::chrono::steady_clock;
    const auto t_alloc = clk::now();

    BatchArgs a{};
    a.roff = g.roff.as<uint32_t>();
    a.rec = g.rec.as<uint2>();
    a.n = n;
    a.model = S.model;
    a.colors = C;
    a.store = S.store.as<uint64_t>();
    a.VN = VN.as<ulonglong2>();
    a.raw = raw.as<unsigned long long>();
    a.raw_cap = raw_cap;
    a.q = q.as<uint4>();
    a.umask = S.model == BPT_IC ? umask.as<uint32_t>() : nullptr;
    a.qoff = qoff.as<uint64_t>();
    a.q_cap = q_cap;
    a.lv = lv.as<LevelRec>();
    a.stats = stats.as<LevelRec>();
    a.stats_cap = stats_cap;
    a.slots_max = (uint32_t)slots;
    a.blocks = S.blocks;
    // sorted start vertices (IC touched-bitmap form; k_order.cu)
    // (and the C < 64 queue form: its C-colour groups become C samples adjacent in start order)
    S.sorted = (bitmap || (S.model == BPT_IC && C > 1 && C < 64 && !wide)) && !(opt.flags & BPT_FLAG_UNSORTED);
    S.lazy_sizes = vmajor;  // k_finalize_v leaves the sizes to ensure_sizes
    if (vmajor) S.blk_sized.assign(S.blocks, 0);
    if (S.sorted) {
        S.slot_sample.alloc(nlocal * 4);
        S.sample_slot.alloc(nlocal * 4);
        sort_slots(g.roff.as<uint32_t>(), n, S.s0, nlocal, stream_key(S.seed, kTagStart), S.slot_sample.as<uint32_t>(),
                   S.sample_slot.as<uint32_t>(), st);
    }
    a.slot_sample = S.sorted ? S.slot_sample.as<uint32_t>() : nullptr;
    a.nlocal = nlocal;
    a.ctl = ctl.as<Ctl>();
    a.theta = S.theta;
    a.k_ic = stream_key(S.seed, kTagIC);
    for (int r = 0; r < 10; ++r) a.ic_keys[r] = a.k_ic + (uint32_t)r * kPhiloxW;
    a.k_lt = stream_key(S.seed, kTagLT);
    a.k_start = stream_key(S.seed, kTagStart);
    a.wide = wide ? 1 : 0;
    a.vflag = wide ? vflag.as<uint32_t>() : nullptr;
    a.qd = wide || vmajor ? qd.as<uint32_t>() : nullptr;
    a.qmask = wide || vmajor ? qmask.as<unsigned long long>() : nullptr;
    a.vmajor = vmajor ? 1 : 0;
    a.touched = bitmap ? touched.as<uint32_t>() : nullptr;
    a.tiles = (uint32_t)tiles;
    a.lt_persist = (opt.flags & BPT_FLAG_LT_LEVELS) ? 0 : 1;
    a.m = g.m;
    a.umask_words = S.model == BPT_IC ? umask.bytes / 4 : 0;
    a.tstart_cap = ts_cap;
    a.lt_blocks_per_sm = 1;
    a.pull = pull ? g.pull_rec.as<uint4>() : nullptr;
    a.pull_edges = pull ? g.m : 0;
    a.pull_seg = pull ? g.pull_seg.as<uint4>() : nullptr;
    a.pull_nseg = pull ? g.pull_nseg : 0;
    // pull when the level's push work reaches kPullAlpha x m (the pull form reads m
    // forward records for all slots of the batch, the push form ~1 record per unit of work)
    a.pull_min_work = (uint64_t)std::max(1.0, (opt.pull_permille ? opt.pull_permille / 1000.0 : kPullAlpha) * (double)g.m);
    a.F = pull ? Fbuf.as<unsigned long long>() : nullptr;
    a.FB = pull ? FBbuf.as<uint32_t>() : nullptr;

    const bool profile = (opt.flags & BPT_FLAG_PROFILE) != 0;
    double ev_ms = 0;
    std::vector<float> ev_each;        // profile mode: ms of every expansion launch, in launch order
    std::vector<uint64_t> ev_batch0;   // ... index of the first launch of every batch
    uint64_t ev_launches = 0, polls = 0;
    double wait_ms = 0;
    if (!profile) {
        // ---- device-resident loops: one graph launch for the whole sample range
        StoreHook hook{&S, a.VN, g.roff.as<uint32_t>(), elog.as<unsigned long long>(), wide};
        cudaGraphExec_t exec = build_sampling_graph(a, tstart.as<uint32_t>(), ts_cap, hook);
        cudaError_t e = cudaGraphLaunch(exec, st);
        cudaGraphExecDestroy(exec);  // deferred by the driver until the launch completes
        BPT_CUDA(e);
    } else {
        // ---- host-driven loop with a CUDA event pair around every expansion launch (roofline
        //      measurement). Same kernels; the host polls the control block every K levels,
        //      pipelined one chunk behind; extra levels launched after the end are no-ops.
        const uint32_t K = opt.poll_levels ? opt.poll_levels : (S.model == BPT_IC ? 3 : 16);
        std::vector<std::pair<cudaEvent_t, cudaEvent_t>> evs;
        struct EvCleanup {
            std::vector<std::pair<cudaEvent_t, cudaEvent_t>>* v;
            ~EvCleanup() { for (auto& e : *v) { cudaEventDestroy(e.first); cudaEventDestroy(e.second); } }
        } evc{&evs};
        cudaEvent_t poll_ev[2];
        BPT_CUDA(cudaEventCreateWithFlags(&poll_ev[0], cudaEventDisableTiming));
        BPT_CUDA(cudaEventCreateWithFlags(&poll_ev[1], cudaEventDisableTiming));
        struct PollCleanup { cudaEvent_t* e; ~PollCleanup() { cudaEventDestroy(e[0]); cudaEventDestroy(e[1]); } } pc{poll_ev};
        static thread_local Ctl* poll_host = nullptr;
        if (!poll_host) BPT_CUDA(cudaMallocHost(&poll_host, 2 * sizeof(Ctl)));
        std::vector<uint64_t> batch_ev0(nbatches);  // first event of every batch
        for (uint64_t b = 0; b < nbatches; ++b) {
            batch_ev0[b] = evs.size();
            launch_init(a, st);
            int cur = 0;
            bool have_prev = false, done = false;
            while (!done) {
                for (uint32_t i = 0; i < K; ++i) {
                    std::pair<cudaEvent_t, cudaEvent_t> e{};
                    BPT_CUDA(cudaEventCreate(&e.first));
                    BPT_CUDA(cudaEventCreate(&e.second));
                    evs.push_back(e);
                    launch_level(a, tstart.as<uint32_t>(), ts_cap, st, e.first, e.second);
                }
                BPT_CUDA(cudaMemcpyAsync(&poll_host[cur], a.ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, st));
                BPT_CUDA(cudaEventRecord(poll_ev[cur], st));
                if (have_prev) {
                    const int prev = cur ^ 1;
                    const auto tw = clk::now();
                    BPT_CUDA(cudaEventSynchronize(poll_ev[prev]));
                    wait_ms += std::chrono::duration<double, std::milli>(clk::now() - tw).count();
                    ++polls;
                    if (poll_host[prev].error || !poll_host[prev].cont) done = true;
                    if (poll_host[prev].level + 2 * K + 2 >= (uint32_t)kMaxLevels) done = true;
                }
                have_prev = true;
                cur ^= 1;
            }
            launch_finalize(S, a.VN, a.ctl, a.slots_max, g.roff.as<uint32_t>(), st, elog.as<unsigned long long>(),
                            a.wide != 0, a.touched ? (a.vmajor ? 2 : 1) : 0);
            launch_next_batch(a, st);
        }
        BPT_CUDA(cudaStreamSynchronize(st));
        ev_each.resize(evs.size());
        for (size_t i = 0; i < evs.size(); ++i) {
            BPT_CUDA(cudaEventElapsedTime(&ev_each[i], evs[i].first, evs[i].second));
            ev_ms += ev_each[i];
        }
        ev_launches = evs.size();
        ev_batch0.swap(batch_ev0);
    }
    const auto t_loop = clk::now();
    unsigned long long h_elog = 0;
    BPT_CUDA(cudaMemcpyAsync(&h_elog, elog.p, 8, cudaMemcpyDeviceToHost, st));
    BPT_CUDA(cudaMemcpyAsync(c_host, ctl.p, sizeof(Ctl), cudaMemcpyDeviceToHost, st));
    BPT_CUDA(cudaStreamSynchronize(st));
    const Ctl cf = *c_host;
    if (const uint32_t bad = checks_read_reset())
        fail(BPT_ECUDA, "device bounds check failed (bits " + std::to_string(bad) + "; k_sample.cu BPT_CHECK ids)");
    if (cf.error == 1) fail(BPT_ENOMEM, "frontier queue overflow; lower batch_groups");
    if (cf.error == 2) fail(BPT_ENOMEM, "level loop exceeded " + std::to_string(kMaxLevels) + " levels");
    const uint32_t rows = (uint32_t)umin64(cf.stats_used, stats_cap);
    std::vector<LevelRec> R(rows);
    if (rows) BPT_CUDA(cudaMemcpy(R.data(), stats.p, (size_t)rows * sizeof(LevelRec), cudaMemcpyDeviceToHost));

    // ---- statistics (exact integers from the device counters)
    bpt_samples_info& I = S.info;
    I.frontier_entries = cf.entries;
    I.members = cf.vc;
    I.coins = cf.coins;
    I.atomics = cf.atomics;
    I.e_phys = S.model == BPT_IC ? cf.work : cf.vc;
    I.e_logical = S.model == BPT_IC ? h_elog : cf.vc;
    I.levels_total = cf.levels_total;
    I.levels_max = cf.levels_max;
    I.pull_levels = cf.pull_levels;
    I.pull_edge_reads = cf.pull_reads;
    I.batch_groups = (uint32_t)slots;
    I.batches = (uint32_t)nbatches;
    I.store_bytes = S.store.bytes;
    S.level_rows.clear();
    S.level_ms.clear();
    double bytes = 0;
    for (uint32_t i = 0; i < rows; ++i) {
        const LevelRec& r = R[i];
        if (profile) {  // batch b's level L ran as launch ev_batch0[b] + L
            const uint64_t b = r.pad >> 32, L = r.pad & 0xffffffffull;
            const uint64_t e = b < ev_batch0.size() ? ev_batch0[b] + L : ~0ull;
            S.level_ms.push_back(e < ev_each.size() ? ev_each[e] : 0.f);
        }
        const uint64_t kept = r.packed >> kPackShift, work = r.packed & kEdgeMask;
        const uint64_t raw_next = (i + 1 < rows && (R[i + 1].pad >> 32) == (r.pad >> 32)) ? R[i + 1].raw : 0;
        if (r.pull)  // 16 B forward record + the slots' F[w] words per edge, U[u] per vertex and slot, merges
            bytes += (16.0 + 8.0 * slots) * (double)r.pull_reads + 8.0 * slots * n + 8.0 * r.atomics + 8.0 * raw_next;
        else if (vmajor)  // record + the S slots' U[u] per edge read, entries {delta, S masks}
            bytes += (8.0 + 8.0 * slots) * work + 8.0 * r.atomics + (4.0 + 8.0 * slots) * kept + 8.0 * raw_next;
        else
            bytes += (S.model == BPT_IC ? 16.0 : 24.0) * work + 8.0 * r.atomics + 24.0 * kept + 8.0 * raw_next;
        const uint64_t row[kLevelCols] = {r.pad >> 32, r.pad & 0xffffffffull, r.raw, kept, work, r.vc, r.coins, r.atomics};
        S.level_rows.insert(S.level_rows.end(), row, row + kLevelCols);
    }
    I.expand_bytes = bytes;
    // expansion time: CUDA events around every launch (profile mode) or the device-side
    // %globaltimer span of every launch (graph mode)
    I.ms_expand = profile ? ev_ms : cf.expand_ns * 1e-6;
    I.expand_launches = profile ? ev_launches : cf.levels_total;
    // graph mode: one host launch (the graph); the kernels it ran counted themselves on the device
    if (!profile) {
        g_launches += 1;
        g_graph_kernels += cf.kernels_run;
    }
    I.kernel_launches = g_launches - launches0 + (profile ? 0 : cf.kernels_run);
#ifdef BPT_HIST
    dump_hist();
#endif
    I.ms_total = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_begin).count();
    if (getenv("BPT_TRACE")) {
        auto ms = [](clk::time_point x, clk::time_point y) { return std::chrono::duration<double, std::milli>(y - x).count(); };
        fprintf(stderr, "[bpt] sample (%s): alloc %.2f ms, loop %.2f ms (polls %llu, wait %.2f ms), drain+stats %.2f ms, "
                        "total %.2f ms, batches %llu, slots %llu, levels %llu, expand %.2f ms, compact %.2f ms\n",
                profile ? "events" : "graph", ms(t_begin, t_alloc), ms(t_alloc, t_loop), (unsigned long long)polls,
                wait_ms, ms(t_loop, clk::now()), I.ms_total, (unsigned long long)nbatches, (unsigned long long)slots,
                (unsigned long long)cf.levels_total, I.ms_expand, cf.compact_ns * 1e-6);
    }
}

}  // namespace bpt

// ==================================================================== C-ABI
using namespace bpt;

struct bpt_comm { Comm c; };
struct bpt_graph { Graph g; };
struct bpt_samples { Samples s; };

extern "C" {

const char* bpt_last_error(void) { return g_last_error.c_str(); }
int bpt_abi_version(void) { return BPT_ABI_VERSION; }
uint64_t bpt_kernel_launch_count(void) { return g_launches; }
uint64_t bpt_graph_kernel_count(void) { return g_graph_kernels; }

bpt_status bpt_release_cache(void) {
    return guarded([&] { release_cached_blocks(); });
}

bpt_status bpt_comm_unique_id(void* uid_out) {
    return guarded([&] {
        if (!uid_out) fail(BPT_EINVAL, "uid_out is NULL");
        comm_unique_id(uid_out);
    });
}

bpt_status bpt_comm_init(const void* nccl_uid, int world, int rank, int cuda_device, bpt_comm** out) {
    return guarded([&] {
        if (!out) fail(BPT_EINVAL, "out is NULL");
        if (world < 1 || rank < 0 || rank >= world) fail(BPT_EINVAL, "need 0 <= rank < world, world >= 1");
        if (world > 1 && !nccl_uid) fail(BPT_EINVAL, "world > 1 needs an NCCL unique id");
        int ndev = 0;
        BPT_CUDA(cudaGetDeviceCount(&ndev));
        if (cuda_device < 0 || cuda_device >= ndev) fail(BPT_EINVAL, "cuda_device out of range");
        BPT_CUDA(cudaSetDevice(cuda_device));
        auto c = std::make_unique<bpt_comm>();
        c->c.world = world;
        c->c.rank = rank;
        c->c.device = cuda_device;
        if (world > 1) comm_init(&c->c, nccl_uid);
        *out = c.release();
    });
}

void bpt_comm_free(bpt_comm* comm) {
    if (!comm) return;
    comm_destroy(&comm->c);
    delete comm;
}

bpt_status bpt_graph_load(bpt_comm* comm, const uint64_t* row_ptr, const uint32_t* col, uint32_t n, uint64_t m,
                          const float* w_f32, const uint32_t* w_q31, bpt_model model, void* stream, bpt_graph** out) {
    return guarded([&] {
        if (!out) fail(BPT_EINVAL, "out is NULL");
        if (n == 0) fail(BPT_EINVAL, "n must be > 0");
        if (m >= (1ull << 32)) fail(BPT_EINVAL, "m must be < 2^32");
        if (!row_ptr || (m && !col)) fail(BPT_EINVAL, "row_ptr / col is NULL");
        if ((w_f32 == nullptr) == (w_q31 == nullptr)) fail(BPT_EINVAL, "give exactly one of w_f32, w_q31");
        if (model != BPT_IC && model != BPT_LT) fail(BPT_EINVAL, "model must be BPT_IC or BPT_LT");
        int dev = 0;
        if (comm) { use_device(comm->c.device); dev = comm->c.device; }
        else BPT_CUDA(cudaGetDevice(&dev));
        cudaStream_t st = (cudaStream_t)stream;
        StreamScope scope(st);
        auto G = std::make_unique<bpt_graph>();
        G->g.comm = comm ? &comm->c : nullptr;
        G->g.device = dev;
        G->g.n = n;
        G->g.m = m;
        G->g.model = model;
        DevIn drp(row_ptr, ((size_t)n + 1) * 8, st);
        DevIn dcol(col, m * 4, st);
        DevIn dwf(w_f32, m * 4, st);
        DevIn dwq(w_q31, m * 4, st);
        build_reverse_csr(G->g, (const uint64_t*)drp.p, (const uint32_t*)dcol.p, (const float*)dwf.p,
                          (const uint32_t*)dwq.p, st);
        *out = G.release();
    });
}

bpt_status bpt_graph_load_bcast(bpt_comm* comm, int root, const uint64_t* row_ptr, const uint32_t* col, uint32_t n,
                                uint64_t m, const float* w_f32, const uint32_t* w_q31, bpt_model model, void* stream,
                                bpt_graph** out) {
    if (!comm || comm->c.world <= 1 || !comm->c.nccl)
        return bpt_graph_load(comm, row_ptr, col, n, m, w_f32, w_q31, model, stream, out);
    return guarded([&] {
        use_device(comm->c.device);
        cudaStream_t st = (cudaStream_t)stream;
        StreamScope scope(st);
        // Every rank takes part in the status exchange whatever its own checks found, so a
        // failure on one rank (its arguments, or the root's validation / build) fails the call
        // on every rank with the same code instead of leaving the others in a broadcast.
        bpt_status local = BPT_OK;
        std::string local_msg;
        auto local_fail = [&](bpt_status c, const char* msg) { if (local == BPT_OK) { local = c; local_msg = msg; } };
        if (!out) local_fail(BPT_EINVAL, "out is NULL");
        if (root < 0 || root >= comm->c.world) local_fail(BPT_EINVAL, "root must be a rank of the communicator");
        if (n == 0) local_fail(BPT_EINVAL, "n must be > 0");
        if (m >= (1ull << 32)) local_fail(BPT_EINVAL, "m must be < 2^32");
        if (model != BPT_IC && model != BPT_LT) local_fail(BPT_EINVAL, "model must be BPT_IC or BPT_LT");
        const bool is_root = comm->c.rank == root;
        bpt_graph* built = nullptr;
        if (is_root && local == BPT_OK) {  // validate + build on the root
            local = bpt_graph_load(comm, row_ptr, col, n, m, w_f32, w_q31, model, stream, &built);
            if (local != BPT_OK) local_msg = g_last_error;
        }
        // status word: (rank-local failure code as a positive number) << 8 | failing rank
        DevBuf status(8);
        const unsigned long long mine =
            local == BPT_OK ? 0ull : ((unsigned long long)(-(int)local) << 8) | (unsigned long long)comm->c.rank;
        BPT_CUDA(cudaMemcpyAsync(status.p, &mine, 8, cudaMemcpyHostToDevice, st));
        comm_allreduce_max_u64(&comm->c, status.as<unsigned long long>(), 1, st);
        unsigned long long got = 0;
        BPT_CUDA(cudaMemcpyAsync(&got, status.p, 8, cudaMemcpyDeviceToHost, st));
        BPT_CUDA(cudaStreamSynchronize(st));
        if (got) {
            if (built) bpt_graph_free(built);
            const bpt_status code = (bpt_status)(-(int)(got >> 8));
            fail(code, local != BPT_OK ? local_msg
                                       : "graph load failed on rank " + std::to_string(got & 0xff) + " (" +
                                             std::to_string((int)code) + ")");
        }
        std::unique_ptr<bpt_graph> G(built ? built : new bpt_graph());
        if (!is_root) {
            G->g.comm = &comm->c;
            G->g.device = comm->c.device;
            G->g.n = n;
            G->g.m = m;
            G->g.model = model;
            G->g.roff.alloc(((size_t)n + 1) * 4);
            G->g.rec.alloc(m * 8 + 8);
        }
        comm_broadcast(&comm->c, G->g.roff.p, G->g.roff.p, ((uint64_t)n + 1) * 4, root, st);
        if (m) comm_broadcast(&comm->c, G->g.rec.p, G->g.rec.p, m * 8, root, st);
        BPT_CUDA(cudaStreamSynchronize(st));
        *out = G.release();
    });
}

bpt_status bpt_graph_reverse(const bpt_graph* g, uint32_t* roff, uint32_t* src, uint32_t* val) {
    return guarded([&] {
        if (!g) fail(BPT_EINVAL, "graph is NULL");
        use_device(g->g.device);
        StreamScope scope(nullptr);
        const Graph& G = g->g;
        copy_out(roff, G.roff.p, ((size_t)G.n + 1) * 4, 0);
        if (src || val) {
            std::vector<uint2> h(G.m);
            if (G.m) BPT_CUDA(cudaMemcpy(h.data(), G.rec.p, G.m * 8, cudaMemcpyDeviceToHost));
            std::vector<uint32_t> a(G.m), b(G.m);
            for (uint64_t i = 0; i < G.m; ++i) { a[i] = h[i].x; b[i] = h[i].y; }
            if (src) BPT_CUDA(cudaMemcpy(src, a.data(), G.m * 4, cudaMemcpyDefault));
            if (val) BPT_CUDA(cudaMemcpy(val, b.data(), G.m * 4, cudaMemcpyDefault));
        }
        BPT_CUDA(cudaDeviceSynchronize());
    });
}

bpt_status bpt_graph_dims(const bpt_graph* g, uint32_t* n, uint64_t* m, int* model) {
    return guarded([&] {
        if (!g) fail(BPT_EINVAL, "graph is NULL");
        if (n) *n = g->g.n;
        if (m) *m = g->g.m;
        if (model) *model = g->g.model;
    });
}

// diagnostic (not in the header): the graph's pull records {u, w, e, thr}, m x 16 B into a host buffer
BPT_API bpt_status bpt_debug_pull_records(const bpt_graph* g, void* host_out) {
    return guarded([&] {
        use_device(g->g.device);
        build_pull_records(g->g, nullptr);
        BPT_CUDA(cudaMemcpy(host_out, g->g.pull_rec.p, g->g.m * 16, cudaMemcpyDeviceToHost));
    });
}

void bpt_graph_free(bpt_graph* g) {
    if (!g) return;
    int cur = -1;
    cudaGetDevice(&cur);
    if (cur != g->g.device) cudaSetDevice(g->g.device);
    delete g;
}

bpt_status bpt_sample_ex(const bpt_graph* g, bpt_model model, uint64_t theta, uint32_t colors, uint64_t seed,
                         const bpt_sample_opts* opts, void* stream, bpt_samples** out) {
    return guarded([&] {
        if (!g || !out) fail(BPT_EINVAL, "graph / out is NULL");
        if ((int)model != g->g.model) fail(BPT_EINVAL, "model does not match the loaded graph");
        if (theta == 0 || theta >= (1ull << 32)) fail(BPT_EINVAL, "theta must be in [1, 2^32)");
        if (colors < 1 || colors > 64 || (64 % colors) != 0) fail(BPT_EINVAL, "colors must divide 64 (1,2,4,...,64)");
        use_device(g->g.device);
        StreamScope scope((cudaStream_t)stream);
        bpt_sample_opts o{};
        if (opts) o = *opts;
        auto S = std::make_unique<bpt_samples>();
        Samples& s = S->s;
        s.g = &g->g;
        s.n = g->g.n;
        s.device = g->g.device;
        s.comm = g->g.comm;
        s.model = model;
        s.theta = theta;
        s.seed = seed;
        s.colors = colors;
        s.stream = (cudaStream_t)stream;
        const Comm* c = g->g.comm;
        uint64_t W = c ? c->world : 1, r = c ? c->rank : 0;
        if (o.shard_world) {  // test hook: one shard of a W-way split, without communication
            if (o.shard_rank >= o.shard_world) fail(BPT_EINVAL, "shard_rank must be < shard_world");
            W = o.shard_world;
            r = o.shard_rank;
        }
        const uint64_t nb = (theta + 63) / 64;
        const uint64_t b0 = r * nb / W, b1 = (r + 1) * nb / W;  // 64-sample blocks of this rank
        s.gb0 = b0;
        s.blocks = b1 - b0;
        s.s0 = umin64(64 * b0, theta);
        s.s1 = umin64(64 * b1, theta);
        const uint64_t pad = 64 * W;
        s.n_pad = (uint32_t)(((uint64_t)g->g.n + pad - 1) / pad * pad);
        bpt_samples_info& I = s.info;
        memset(&I, 0, sizeof(I));
        I.theta = theta; I.seed = seed; I.s0 = s.s0; I.s1 = s.s1;
        I.colors = colors; I.model = model; I.world = (uint32_t)W; I.rank = (uint32_t)r; I.n = g->g.n;
        run_sampling(s, o, (cudaStream_t)stream);
        s.g = nullptr;  // the samples do not depend on the graph after this point
        *out = S.release();
    });
}

bpt_status bpt_sample(const bpt_graph* g, bpt_model model, uint64_t theta, uint32_t colors, uint64_t seed,
                      void* stream, bpt_samples** out) {
    return bpt_sample_ex(g, model, theta, colors, seed, nullptr, stream, out);
}

bpt_status bpt_samples_get_info(const bpt_samples* s, bpt_samples_info* out) {
    return guarded([&] {
        if (!s || !out) fail(BPT_EINVAL, "NULL argument");
        *out = s->s.info;
    });
}

bpt_status bpt_occurrences(const bpt_samples* s, uint32_t* counts) {
    return guarded([&] {
        if (!s || !counts) fail(BPT_EINVAL, "NULL argument");
        use_device(s->s.device);
        StreamScope scope(s->s.stream);
        copy_out(counts, s->s.count0.p, (size_t)s->s.n * 4, s->s.stream);
        BPT_CUDA(cudaStreamSynchronize(s->s.stream));
    });
}

bpt_status bpt_level_stats(const bpt_samples* s, uint64_t* out, uint64_t cap_rows, uint64_t* rows_out) {
    return guarded([&] {
        if (!s) fail(BPT_EINVAL, "samples is NULL");
        const uint64_t rows = s->s.level_rows.size() / kLevelCols;
        if (rows_out) *rows_out = rows;
        if (out) memcpy(out, s->s.level_rows.data(), std::min(rows, cap_rows) * kLevelCols * 8);
    });
}

bpt_status bpt_level_times(const bpt_samples* s, float* out, uint64_t cap_rows, uint64_t* rows_out) {
    return guarded([&] {
        if (!s) fail(BPT_EINVAL, "samples is NULL");
        const uint64_t rows = s->s.level_ms.size();
        if (rows_out) *rows_out = rows;
        if (out) memcpy(out, s->s.level_ms.data(), std::min(rows, cap_rows) * 4);
    });
}

static void check_range(const Samples& S, uint64_t first, uint64_t count) {
    if (count == 0) fail(BPT_EINVAL, "count must be > 0");
    if (first < S.s0 || first + count > S.s1 || first + count < first)
        fail(BPT_EINVAL, "samples [" + std::to_string(first) + ", " + std::to_string(first + count) +
                             ") are not inside this rank's range [" + std::to_string(S.s0) + ", " +
                             std::to_string(S.s1) + ")");
}

bpt_status bpt_rrr_sizes(const bpt_samples* s, uint64_t first, uint64_t count, uint32_t* sizes) {
    return guarded([&] {
        if (!s || !sizes) fail(BPT_EINVAL, "NULL argument");
        check_range(s->s, first, count);
        use_device(s->s.device);
        StreamScope scope(s->s.stream);
        ensure_sizes(const_cast<Samples&>(s->s), first, count, s->s.stream);
        copy_out(sizes, s->s.sizes.as<uint32_t>() + (first - s->s.s0), count * 4, s->s.stream);
        BPT_CUDA(cudaStreamSynchronize(s->s.stream));
    });
}

bpt_status bpt_rrr_digests(const bpt_samples* s, uint64_t first, uint64_t count, uint64_t* digests) {
    return guarded([&] {
        if (!s || !digests) fail(BPT_EINVAL, "NULL argument");
        check_range(s->s, first, count);
        use_device(s->s.device);
        StreamScope scope(s->s.stream);
        Samples& M = const_cast<Samples&>(s->s);
        if (!M.digests_ready) {  // verification checksums: computed on first use
            compute_digests(M, M.stream);
            M.digests_ready = true;
        }
        copy_out(digests, s->s.digests.as<uint64_t>() + (first - s->s.s0), count * 8, M.stream);
        BPT_CUDA(cudaStreamSynchronize(M.stream));
    });
}

bpt_status bpt_rrr_extract(const bpt_samples* s, uint64_t first, uint64_t count, uint64_t* offsets,
                           uint32_t* members, uint64_t capacity) {
    return guarded([&] {
        if (!s || !offsets) fail(BPT_EINVAL, "NULL argument");
        const Samples& S = s->s;
        check_range(S, first, count);
        use_device(S.device);
        const cudaStream_t st = S.stream;
        StreamScope scope(st);
        std::vector<uint32_t> sz(count);
        ensure_sizes(const_cast<Samples&>(S), first, count, st);
        BPT_CUDA(cudaMemcpyAsync(sz.data(), S.sizes.as<uint32_t>() + (first - S.s0), count * 4, cudaMemcpyDeviceToHost, st));
        BPT_CUDA(cudaStreamSynchronize(st));
        std::vector<uint64_t> off(count + 1, 0);
        for (uint64_t i = 0; i < count; ++i) off[i + 1] = off[i] + sz[i];
        const uint64_t total = off[count];
        if (capacity < total)
            fail(BPT_ENOMEM, "members capacity " + std::to_string(capacity) + " < required " + std::to_string(total));
        if (total && !members) fail(BPT_EINVAL, "members is NULL");
        if (total && S.sparse) {  // the store is the member lists: sort the range, one contiguous slice
            DevBuf err(4);
            BPT_CUDA(cudaMemsetAsync(err.p, 0, 4, st));
            launch_sort_lists(S.list_off.as<uint64_t>() + (first - S.s0), const_cast<uint32_t*>(S.list_mem.as<uint32_t>()),
                              count, err.as<uint32_t>(), st);
            uint32_t h_err = 0;
            uint64_t b = 0;
            BPT_CUDA(cudaMemcpyAsync(&h_err, err.p, 4, cudaMemcpyDeviceToHost, st));
            BPT_CUDA(cudaMemcpyAsync(&b, S.list_off.as<uint64_t>() + (first - S.s0), 8, cudaMemcpyDeviceToHost, st));
            BPT_CUDA(cudaStreamSynchronize(st));
            if (h_err) fail(BPT_ESTATE, "member list longer than the list sort");
            BPT_CUDA(cudaMemcpyAsync(members, S.list_mem.as<uint32_t>() + b, total * 4, cudaMemcpyDefault, st));
            BPT_CUDA(cudaStreamSynchronize(st));
        } else if (total) {
            Samples& M = const_cast<Samples&>(S);
            if (M.sorted && M.h_sample_slot.empty()) {  // sample -> slot map on the host, once per handle
                M.h_sample_slot.resize(M.s1 - M.s0);
                BPT_CUDA(cudaMemcpyAsync(M.h_sample_slot.data(), M.sample_slot.p, (M.s1 - M.s0) * 4,
                                         cudaMemcpyDeviceToHost, st));
                BPT_CUDA(cudaStreamSynchronize(st));
            }
            DevBuf tmp;
            uint32_t* dm = members;
            if (!is_device_ptr(members)) { tmp.alloc(total * 4); dm = tmp.as<uint32_t>(); }
            extract_range(S, first, count, off.data(), dm, st);
            if (dm != members) BPT_CUDA(cudaMemcpyAsync(members, dm, total * 4, cudaMemcpyDeviceToHost, st));
            BPT_CUDA(cudaStreamSynchronize(st));
        }
        BPT_CUDA(cudaMemcpyAsync(offsets, off.data(), (count + 1) * 8, cudaMemcpyDefault, st));
        BPT_CUDA(cudaStreamSynchronize(st));
    });
}

bpt_status bpt_select_seeds(const bpt_samples* s, uint32_t k, uint32_t* seeds, uint64_t* gains, double* sigma_hat) {
    return guarded([&] {
        if (!s) fail(BPT_EINVAL, "samples is NULL");
        const Samples& S = s->s;
        if (k == 0 || k > S.n) fail(BPT_EINVAL, "k must be in [1, n]");
        use_device(S.device);
        StreamScope scope(S.stream);
        std::vector<uint32_t> hs(k);
        std::vector<uint64_t> hg(k);
        select_seeds(S, k, hs.data(), hg.data(), S.stream);
        uint64_t covered = 0;
        for (uint32_t i = 0; i < k; ++i) covered += hg[i];
        const double sig = (double)S.n * (double)covered / (double)S.theta;  // reading C-12
        if (seeds) BPT_CUDA(cudaMemcpy(seeds, hs.data(), k * 4, cudaMemcpyDefault));
        if (gains) BPT_CUDA(cudaMemcpy(gains, hg.data(), k * 8, cudaMemcpyDefault));
        if (sigma_hat) {
            if (is_device_ptr(sigma_hat)) BPT_CUDA(cudaMemcpy(sigma_hat, &sig, 8, cudaMemcpyHostToDevice));
            else *sigma_hat = sig;
        }
    });
}

bpt_status bpt_selftest_philox(const uint32_t* ctr_key, uint32_t* out, uint64_t count) {
    return guarded([&] {
        if (count && (!ctr_key || !out)) fail(BPT_EINVAL, "NULL argument");
        StreamScope scope(nullptr);
        DevIn din(ctr_key, count * 12, nullptr);
        DevBuf dout(count * 8 + 8);
        selftest_philox((const uint32_t*)din.p, dout.as<uint32_t>(), count, nullptr);
        copy_out(out, dout.p, count * 8, nullptr);
        BPT_CUDA(cudaStreamSynchronize(nullptr));
    });
}

bpt_status bpt_bench_philox(uint64_t iters, uint64_t* calls, double* ms) {
    return guarded([&] {
        if (!calls || !ms || iters == 0) fail(BPT_EINVAL, "calls / ms NULL or iters == 0");
        StreamScope scope(nullptr);
        *ms = bench_philox(iters, calls, nullptr);
    });
}

void bpt_samples_free(bpt_samples* s) {
    if (!s) return;
    int cur = -1;
    cudaGetDevice(&cur);
    if (cur != s->s.device) cudaSetDevice(s->s.device);
    delete s;
}

}  // extern "C"
