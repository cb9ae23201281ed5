// k_sample.cu -- A2 start/colour assignment, A3/A3' fused frontier expansion (IC / LT),
// A4 frontier compaction.  Listing 1 of the paper, level-synchronous
// (reading C-7), mark-on-discovery.
//
// Data layout per batch of `slots` 64-sample blocks:
//   V[slot][n] u64   visited masks  = the fused RRR store (Listing 1 visited[])
//   N[slot][n] u64   next-frontier accumulators (Listing 1 frontier[u] |= fr_u)
//   raw[]      u64   discovered entries of the next level: v | slot << 32 | slice << 58
//   q[]        uint4 compacted frontier entries {v, slot, mask lo, mask hi}
//   qoff[]     u64   exclusive prefix of per-entry work (IC: in-degree, LT: popcount)
//   tstart[]   u32   first entry of each expansion tile (written by the compaction)
// Level L:  compact(L): raw(L) -> V |= N, q/qoff/tstart      (Listing 1 lines 7-8)
//           expand(L):  q -> N atomicOr, raw(L+1)             (Listing 1 lines 9-15)
#include "internal.cuh"

namespace bpt {
namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kItems = 4;
constexpr uint32_t kTile = kThreads * kItems;   // work items (edges / LT tasks) per tile
constexpr uint32_t kFull = 0xffffffffu;

__device__ __forceinline__ uint64_t raw_pack(uint32_t v, uint32_t slot, uint32_t slice) {
    return (uint64_t)v | ((uint64_t)slot << 32) | ((uint64_t)slice << 58);
}

// slice mask of the traversal group containing bit `bit` (C divides 64)
__device__ __forceinline__ uint64_t slice_mask_of(uint32_t colors, uint32_t slice) {
    return colors == 64 ? ~0ull : (((1ull << colors) - 1ull) << (slice * colors));
}

// position of the r-th (0-based) set bit of x; x must have > r set bits
__device__ __forceinline__ uint32_t nth_set_bit64(uint64_t x, uint32_t r) {
    uint32_t w = (uint32_t)x, base = 0;
    uint32_t p = __popc(w);
    if (r >= p) { r -= p; w = (uint32_t)(x >> 32); base = 32; }
    p = __popc(w & 0xffffu); if (r >= p) { r -= p; w >>= 16; base += 16; }
    p = __popc(w & 0xffu);   if (r >= p) { r -= p; w >>= 8;  base += 8; }
    p = __popc(w & 0xfu);    if (r >= p) { r -= p; w >>= 4;  base += 4; }
    p = __popc(w & 0x3u);    if (r >= p) { r -= p; w >>= 2;  base += 2; }
    if (r >= (w & 1u)) base += 1;
    return base;
}

__device__ __forceinline__ unsigned long long block_sum_ull(unsigned long long x, unsigned long long* sh) {
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) x += __shfl_xor_sync(kFull, x, d);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) sh[w] = x;
    __syncthreads();
    unsigned long long t = 0;
    if (threadIdx.x == 0)
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += sh[i];
    return t;  // valid in thread 0
}

// ------------------------------------------------------------------------ A2: init
// Sample s = 64*(gblk0 + slot) + bit, colour bit of block slot. start(s) per reading C-3.
// Listing 1 lines 1-3: frontier[start].c = 1 -> here N[slot][start] |= bit,
// first setter of the (slot, slice) enqueues the raw entry of level 0.
__global__ void k_init(BatchArgs a) {
    const uint64_t total = (uint64_t)a.slots * 64;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t slot = (uint32_t)(i >> 6), bit = (uint32_t)(i & 63);
        const uint64_t s = 64ull * (a.gblk0 + slot) + bit;
        if (s >= a.theta) continue;
        const uint2 w = philox2x32_10((uint32_t)s, (uint32_t)(s >> 32), a.k_start);
        const uint64_t r64 = ((uint64_t)w.y << 32) | w.x;
        const uint32_t start = (uint32_t)__umul64hi(r64, (uint64_t)a.n);
        const uint32_t slice = bit / a.colors;
        const uint64_t smask = slice_mask_of(a.colors, slice);
        const unsigned long long old = atomicOr((unsigned long long*)&a.N[(size_t)slot * a.n + start], 1ull << bit);
        if ((old & smask) == 0) {
            const unsigned pos = atomicAdd(&a.lv[0].raw, 1u);
            if (pos < a.raw_cap) a.raw[pos] = raw_pack(start, slot, slice);
            else a.lv[0].overflow = 1;
        }
    }
}

// ------------------------------------------------------------------------ A4: compaction
// For each discovered (v, slot, slice) of level L: mask = N & slice; N &= ~slice;
// V |= mask (Listing 1 line 8 "visited[v] = visited[v] | fr_v"); keep the entry if v has
// in-edges (its expansion has work); warp ballot + block prefix give the output slots,
// one packed atomicAdd per block allocates (entries, work) consistently.
__global__ void __launch_bounds__(kThreads) k_compact(BatchArgs a, int level, uint32_t* __restrict__ tstart,
                                                      uint64_t tstart_cap) {
    LevelRec* L = &a.lv[level];
    const uint32_t nraw = min((uint64_t)L->raw, a.raw_cap);
    __shared__ unsigned long long wsum[kWarps];
    __shared__ uint32_t wcnt[kWarps];
    __shared__ unsigned long long blk_base;
    __shared__ unsigned long long vc_acc[kWarps];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const uint32_t lt = (1u << lane) - 1u;
    unsigned long long vc_local = 0;
    for (uint64_t tile0 = (uint64_t)blockIdx.x * kThreads; tile0 < nraw; tile0 += (uint64_t)gridDim.x * kThreads) {
        const uint64_t i = tile0 + threadIdx.x;
        bool keep = false;
        uint32_t v = 0, slot = 0;
        uint64_t mask = 0, work = 0;
        uint32_t rowstart = 0;
        if (i < nraw) {
            const uint64_t r = a.raw[i];
            v = (uint32_t)r;
            slot = (uint32_t)(r >> 32) & ((1u << 26) - 1u);
            const uint32_t slice = (uint32_t)(r >> 58);
            unsigned long long* Np = (unsigned long long*)&a.N[(size_t)slot * a.n + v];
            uint64_t* Vp = &a.store[(size_t)(a.blk0 + slot) * a.n + v];
            if (a.colors == 64) {
                mask = *Np;
                *Np = 0;
                *Vp |= mask;
            } else {
                const uint64_t sm = slice_mask_of(a.colors, slice);
                mask = atomicAnd(Np, ~sm) & sm;
                atomicOr((unsigned long long*)Vp, mask);
            }
            vc_local += __popcll(mask);
            rowstart = a.roff[v];
            const uint32_t deg = a.roff[v + 1] - rowstart;
            work = a.model == BPT_IC ? deg : (deg ? __popcll(mask) : 0);
            keep = work != 0;
        }
        // warp-level ballot + prefix (count) and shuffle prefix (work)
        const uint32_t bal = __ballot_sync(kFull, keep);
        const uint32_t rank = __popc(bal & lt);
        unsigned long long wincl = work;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            unsigned long long y = __shfl_up_sync(kFull, wincl, d);
            if (lane >= d) wincl += y;
        }
        if (lane == 31) { wsum[wid] = wincl; wcnt[wid] = __popc(bal); }
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned long long ts = 0; uint32_t tc = 0;
            for (int w = 0; w < kWarps; ++w) {
                unsigned long long s = wsum[w]; uint32_t c = wcnt[w];
                wsum[w] = ts; wcnt[w] = tc; ts += s; tc += c;
            }
            unsigned long long old = tc ? atomicAdd(&L->packed, ((unsigned long long)tc << kPackShift) + ts) : 0ull;
            if (tc && ((old >> kPackShift) + tc > a.q_cap || (old & kEdgeMask) + ts > kEdgeMask)) {
                L->overflow = 1;
                old = ~0ull;
            }
            blk_base = old;
        }
        __syncthreads();
        const unsigned long long bb = blk_base;
        if (keep && bb != ~0ull) {
            const uint64_t qi = (bb >> kPackShift) + wcnt[wid] + rank;
            const uint64_t off = (bb & kEdgeMask) + wsum[wid] + wincl - work;
            a.q[qi] = make_uint4(v, slot, (uint32_t)mask, (uint32_t)(mask >> 32));
            a.qoff[qi] = off;
            // tiles whose first work item falls inside [off, off + work)
            uint64_t t = (off + kTile - 1) / kTile;
            for (; t * kTile < off + work; ++t) {
                if (t < tstart_cap) tstart[t] = (uint32_t)qi;
                else L->overflow = 1;
            }
        }
        __syncthreads();
    }
    // level statistics
    unsigned long long vc_tot = block_sum_ull(vc_local, vc_acc);
    if (threadIdx.x == 0 && vc_tot) atomicAdd(&L->vc, vc_tot);
}

// ------------------------------------------------------------------------ A3: expansion
struct SmemTile {
    uint32_t rel[kTile + 1];   // max(qoff - t0, 0) per entry of the tile
    uint32_t aux[kTile + 1];   // IC: e - t (mod 2^32); LT: row start
    uint32_t v[kTile + 1];     // LT: vertex
    uint32_t slot[kTile + 1];
    unsigned long long mask[kTile + 1];
    // per-warp coin flattening scratch
    uint32_t f_excl[kWarps][32];
    uint32_t f_e[kWarps][32];
    uint32_t f_thr[kWarps][32];
    uint32_t f_sbase[kWarps][32];
    unsigned long long f_live[kWarps][32];
    unsigned long long f_pass[kWarps][32];
    unsigned long long red[kWarps];
    uint32_t cnt;
};

__device__ __forceinline__ void enqueue_warp(const BatchArgs& a, LevelRec* Lnext, bool first, uint64_t entry) {
    const uint32_t bal = __ballot_sync(kFull, first);
    if (!bal) return;
    const int lane = threadIdx.x & 31;
    const int leader = __ffs(bal) - 1;
    unsigned base = 0;
    if (lane == leader) base = atomicAdd(&Lnext->raw, (unsigned)__popc(bal));
    base = __shfl_sync(kFull, base, leader);
    if (first) {
        const uint64_t pos = (uint64_t)base + __popc(bal & ((1u << lane) - 1u));
        if (pos < a.raw_cap) a.raw[pos] = entry;
        else Lnext->overflow = 1;
    }
}

// IC, Listing 1 lines 9-15: for each frontier entry (v, slot, mask) and each reverse edge e
// of v: u = src[e]; live = mask & ~V[u]; every live colour c keeps its bit iff the coin
// of (sample c, e) passes (reading C-2); surviving bits are OR-merged into N[u] (line 14,
// the fusing step); the first setter of N[u] (per slice) enqueues u for level L+1.
// Each edge record is read once per level for all live colours. The live (edge, colour)
// coin tasks of a warp are flattened and evaluated 32 at a time.
__global__ void __launch_bounds__(kThreads) k_expand_ic(BatchArgs a, int level, const uint32_t* __restrict__ tstart) {
    const LevelRec* L = &a.lv[level];
    LevelRec* Ln = &a.lv[level + 1];
    const unsigned long long packed = L->packed;
    const uint64_t nq = packed >> kPackShift;
    const uint64_t total = packed & kEdgeMask;
    if (nq == 0 || L->overflow) return;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    SmemTile& sm = *reinterpret_cast<SmemTile*>(smem_raw);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const uint32_t lt = (1u << lane) - 1u;
    const uint64_t ntiles = (total + kTile - 1) / kTile;
    unsigned long long coins = 0, atoms = 0;
    for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const uint64_t t0 = tile * kTile;
        const uint32_t j0 = tstart[tile];
        const uint64_t jend = tile + 1 < ntiles ? (uint64_t)tstart[tile + 1] + 1 : nq;  // exclusive
        const uint32_t cnt = (uint32_t)umin64(jend - j0, (uint64_t)kTile + 1);
        __syncthreads();
        for (uint32_t k = threadIdx.x; k < cnt; k += kThreads) {
            const uint64_t j = j0 + k;
            const uint64_t off = a.qoff[j];
            const uint4 ent = a.q[j];
            sm.rel[k] = off <= t0 ? 0u : (uint32_t)(off - t0);
            sm.aux[k] = a.roff[ent.x] - (uint32_t)off;  // e = t + aux  (mod 2^32)
            sm.slot[k] = ent.y;
            sm.mask[k] = (unsigned long long)ent.z | ((unsigned long long)ent.w << 32);
        }
        if (threadIdx.x == 0) sm.cnt = cnt;
        __syncthreads();
#pragma unroll 1
        for (int it = 0; it < kItems; ++it) {
            const uint64_t t = t0 + (uint64_t)it * kThreads + threadIdx.x;
            const bool valid = t < total;
            uint64_t live = 0;
            uint32_t e = 0, thr = 0, u = 0, slot = 0;
            uint64_t emask = 0;
            if (valid) {
                const uint32_t target = (uint32_t)(t - t0);
                uint32_t lo = 0, hi = cnt;  // largest k with rel[k] <= target
                while (hi - lo > 1) {
                    const uint32_t mid = (lo + hi) >> 1;
                    if (sm.rel[mid] <= target) lo = mid; else hi = mid;
                }
                e = (uint32_t)t + sm.aux[lo];
                slot = sm.slot[lo];
                emask = sm.mask[lo];
                const uint2 r = __ldg(&a.rec[e]);
                u = r.x;
                thr = r.y;
                const uint64_t Vu = __ldg((const unsigned long long*)&a.store[(size_t)(a.blk0 + slot) * a.n + u]);
                live = emask & ~Vu;
            }
            // ---- coin-task flattening (warp) ----
            const uint32_t c = __popcll(live);
            uint32_t incl = c;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                uint32_t y = __shfl_up_sync(kFull, incl, d);
                if (lane >= d) incl += y;
            }
            const uint32_t ntask = __shfl_sync(kFull, incl, 31);
            uint64_t pass = 0;
            if (ntask) {
                sm.f_excl[wid][lane] = incl - c;
                sm.f_e[wid][lane] = e;
                sm.f_thr[wid][lane] = thr;
                sm.f_sbase[wid][lane] = (uint32_t)(64ull * (a.gblk0 + slot));
                sm.f_live[wid][lane] = live;
                sm.f_pass[wid][lane] = 0;
                __syncwarp();
                for (uint32_t b = 0; b < ntask; b += 32) {
                    const uint32_t k = b + lane;
                    if (k < ntask) {
                        uint32_t lo = 0;  // owner = largest lane with excl <= k
#pragma unroll
                        for (int step = 16; step > 0; step >>= 1)
                            if (sm.f_excl[wid][lo + step] <= k) lo += step;
                        const uint32_t bit = nth_set_bit64(sm.f_live[wid][lo], k - sm.f_excl[wid][lo]);
                        const uint32_t s = sm.f_sbase[wid][lo] + bit;
                        const uint32_t r = philox2x32_10(sm.f_e[wid][lo], s, a.k_ic).x;
                        if ((r >> 1) < sm.f_thr[wid][lo]) atomicOr(&sm.f_pass[wid][lo], 1ull << bit);
                    }
                }
                __syncwarp();
                pass = sm.f_pass[wid][lane];
                coins += (lane == 0) ? ntask : 0;
            }
            bool first = false;
            uint64_t entry = 0;
            if (pass) {
                ++atoms;
                const unsigned long long old = atomicOr((unsigned long long*)&a.N[(size_t)slot * a.n + u], pass);
                const uint32_t slice = a.colors == 64 ? 0u : (uint32_t)(__ffsll((long long)emask) - 1) / a.colors;
                first = (old & slice_mask_of(a.colors, slice)) == 0;
                entry = raw_pack(u, slot, slice);
            }
            enqueue_warp(a, Ln, first, entry);
        }
    }
    unsigned long long ct = block_sum_ull(coins, sm.red);
    if (threadIdx.x == 0 && ct) atomicAdd(&((LevelRec*)L)->coins, ct);
    unsigned long long at = block_sum_ull(atoms, sm.red);
    if (threadIdx.x == 0 && at) atomicAdd(&((LevelRec*)L)->atomics, at);
}

// LT (reading C-6): work items are (entry, colour) pairs. For colour c at v: r = coinLT(s_c, v)
// >> 1, chosen in-edge j = first with cum[j] > r (binary search of the row, rows are
// cumulative thresholds); none if r >= row sum. If u = src[j] has not been visited by c,
// N[u] |= bit c (fusing) and the first setter enqueues u.
__global__ void __launch_bounds__(kThreads) k_expand_lt(BatchArgs a, int level, const uint32_t* __restrict__ tstart) {
    const LevelRec* L = &a.lv[level];
    LevelRec* Ln = &a.lv[level + 1];
    const unsigned long long packed = L->packed;
    const uint64_t nq = packed >> kPackShift;
    const uint64_t total = packed & kEdgeMask;
    if (nq == 0 || L->overflow) return;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    SmemTile& sm = *reinterpret_cast<SmemTile*>(smem_raw);
    const uint64_t ntiles = (total + kTile - 1) / kTile;
    unsigned long long coins = 0, atoms = 0;
    for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const uint64_t t0 = tile * kTile;
        const uint32_t j0 = tstart[tile];
        const uint64_t jend = tile + 1 < ntiles ? (uint64_t)tstart[tile + 1] + 1 : nq;
        const uint32_t cnt = (uint32_t)umin64(jend - j0, (uint64_t)kTile + 1);
        __syncthreads();
        for (uint32_t k = threadIdx.x; k < cnt; k += kThreads) {
            const uint64_t j = j0 + k;
            const uint64_t off = a.qoff[j];
            const uint4 ent = a.q[j];
            sm.rel[k] = off <= t0 ? 0u : (uint32_t)(off - t0);
            sm.aux[k] = (uint32_t)(t0 > off ? t0 - off : 0);  // tasks of entry k before the tile
            sm.v[k] = ent.x;
            sm.slot[k] = ent.y;
            sm.mask[k] = (unsigned long long)ent.z | ((unsigned long long)ent.w << 32);
        }
        __syncthreads();
#pragma unroll 1
        for (int it = 0; it < kItems; ++it) {
            const uint64_t t = t0 + (uint64_t)it * kThreads + threadIdx.x;
            bool first = false;
            uint64_t entry = 0;
            if (t < total) {
                const uint32_t target = (uint32_t)(t - t0);
                uint32_t lo = 0, hi = cnt;
                while (hi - lo > 1) {
                    const uint32_t mid = (lo + hi) >> 1;
                    if (sm.rel[mid] <= target) lo = mid; else hi = mid;
                }
                const uint32_t v = sm.v[lo], slot = sm.slot[lo];
                const uint64_t emask = sm.mask[lo];
                const uint32_t r_idx = target - sm.rel[lo] + sm.aux[lo];
                const uint32_t bit = nth_set_bit64(emask, r_idx);
                const uint32_t s = (uint32_t)(64ull * (a.gblk0 + slot)) + bit;
                const uint32_t r = philox2x32_10(v, s, a.k_lt).x >> 1;
                ++coins;
                uint32_t lo2 = a.roff[v], hi2 = a.roff[v + 1];  // first j with cum[j] > r
                const uint32_t end = hi2;
                while (lo2 < hi2) {
                    const uint32_t mid = (lo2 + hi2) >> 1;
                    if (__ldg(&a.rec[mid]).y > r) hi2 = mid; else lo2 = mid + 1;
                }
                if (lo2 < end) {
                    const uint32_t u = __ldg(&a.rec[lo2]).x;
                    const uint64_t b = 1ull << bit;
                    const uint64_t Vu = a.store[(size_t)(a.blk0 + slot) * a.n + u];
                    if (!(Vu & b)) {
                        ++atoms;
                        const unsigned long long old = atomicOr((unsigned long long*)&a.N[(size_t)slot * a.n + u], b);
                        const uint32_t slice = bit / a.colors;
                        first = (old & slice_mask_of(a.colors, slice)) == 0;
                        entry = raw_pack(u, slot, slice);
                    }
                }
            }
            enqueue_warp(a, Ln, first, entry);
        }
    }
    unsigned long long ct = block_sum_ull(coins, sm.red);
    if (threadIdx.x == 0 && ct) atomicAdd(&((LevelRec*)L)->coins, ct);
    unsigned long long at = block_sum_ull(atoms, sm.red);
    if (threadIdx.x == 0 && at) atomicAdd(&((LevelRec*)L)->atomics, at);
}

int g_expand_grid = 0;
int g_compact_grid = 0;

}  // namespace

uint32_t expand_tile() { return kTile; }

int expand_grid() {
    if (!g_expand_grid) {
        int per_sm = 0;
        BPT_CUDA(cudaFuncSetAttribute(k_expand_ic, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(SmemTile)));
        BPT_CUDA(cudaFuncSetAttribute(k_expand_lt, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(SmemTile)));
        BPT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_expand_ic, kThreads, sizeof(SmemTile)));
        g_expand_grid = num_sms() * (per_sm > 0 ? per_sm : 1);
        int per_sm_c = 0;
        BPT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_c, k_compact, kThreads, 0));
        g_compact_grid = num_sms() * (per_sm_c > 0 ? per_sm_c : 1);
    }
    return g_expand_grid;
}

void launch_init(const BatchArgs& a, cudaStream_t st) {
    const uint64_t total = (uint64_t)a.slots * 64;
    const unsigned grid = (unsigned)((total + 255) / 256);
    k_init<<<grid, 256, 0, st>>>(a);
    count_launch();
    BPT_CUDA(cudaGetLastError());
}

void launch_compact(const BatchArgs& a, int level, uint32_t* tstart, uint64_t tstart_cap, cudaStream_t st) {
    expand_grid();
    k_compact<<<g_compact_grid, kThreads, 0, st>>>(a, level, tstart, tstart_cap);
    count_launch();
    BPT_CUDA(cudaGetLastError());
}

void launch_expand(const BatchArgs& a, int level, const uint32_t* tstart, cudaStream_t st) {
    const int grid = expand_grid();
    if (a.model == BPT_IC)
        k_expand_ic<<<grid, kThreads, sizeof(SmemTile), st>>>(a, level, tstart);
    else
        k_expand_lt<<<grid, kThreads, sizeof(SmemTile), st>>>(a, level, tstart);
    count_launch();
    BPT_CUDA(cudaGetLastError());
}

}  // namespace bpt
