// k_sample.cu -- A2 start/colour assignment, A3/A3' fused frontier expansion (IC / LT),
// A4 frontier compaction, and the device-resident loops that run them. Listing 1 of the
// paper, level-synchronous (reading C-7), mark-on-discovery.
//
// Data layout per batch of `slots` 64-sample blocks:
//   VN[slot][n] {V, N}  visited masks (Listing 1 visited[]) and next-frontier
//                       accumulators (frontier[u] |= fr_u), one 32-B sector per vertex
//   raw[]      u64      discovered entries of the next level: v | slot << 32 | slice << 58
//   q[]        uint4    compacted frontier entries {rowstart - off (IC) | v (LT), slot, mask}
//   qoff[]     u64      exclusive prefix of per-entry work (LT)
//   tstart[], umask[]   first entry / entry-start bitmap of each expansion unit (IC)
// Level L:  compact(L): raw(L) -> V |= N, q/tstart/umask     (Listing 1 lines 7-8)
//           expand(L):  q -> N atomicOr, raw(L+1)             (Listing 1 lines 9-15)
//
// Sections: helpers; A2 k_init; A4 compaction; level advance; IC expansion (the product's
// dominant kernel); IC wide fusion (2 blocks per frontier entry, §8(f) NEXT #2); LT reverse
// walks (dense and sparse store); LT fused expansion and its cooperative level loop; launchers
// and the CUDA-graph builder.
#include <algorithm>
#include <cstdio>
#include <type_traits>
#include <cstdlib>

#include "internal.cuh"


namespace bpt {
namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
#ifndef BPT_LT_ITEMS
#define BPT_LT_ITEMS 1
#endif
constexpr int kItems = BPT_LT_ITEMS;    // LT tasks per thread per tile (1: thin LT levels spread over all blocks)
constexpr uint32_t kTile = kThreads * kItems;   // LT tasks per tile
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

// Edge records stream through once per level: read them with an evict-first L2 policy so the
// working masks (V, N: 77.6 MB per in-flight block on C2, gathered at random) stay resident in
// the 126 MB L2; the gathers themselves use evict-last.
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ uint2 ld_stream(const uint2* p) {
    uint2 r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.u32 {%0, %1}, [%2], %3;"
                 : "=r"(r.x), "=r"(r.y) : "l"(p), "l"(policy_evict_first()));
    return r;
}
__device__ __forceinline__ uint4 ld_stream4(const uint4* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4], %5;"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p), "l"(policy_evict_first()));
    return r;
}
// coherent (L2) load with evict-last: U is OR-merged by other warps during the same launch (a stale
// value only skips fewer coins)
__device__ __forceinline__ uint2 ld_keep_u64(const unsigned long long* p) {
    uint2 r;
    asm volatile("ld.global.cg.L2::cache_hint.v2.u32 {%0, %1}, [%2], %3;"
                 : "=r"(r.x), "=r"(r.y) : "l"(p), "l"(policy_evict_last()));
    return r;
}
__device__ __forceinline__ ulonglong2 ld_keep(const ulonglong2* p) {
    ulonglong2 r;
    asm volatile("ld.global.nc.L2::cache_hint.v2.u64 {%0, %1}, [%2], %3;"
                 : "=l"(r.x), "=l"(r.y) : "l"(p), "l"(policy_evict_last()));
    return r;
}

// 256-bit loads / stores of a vertex's 4 slot masks (one 32-B sector, LDG/STG.E.ENL2.256)
struct U4 { unsigned long long x, y, z, w; };
__device__ __forceinline__ U4 ld_nc4(const unsigned long long* p) {
    U4 r;
    asm("ld.global.nc.v4.u64 {%0, %1, %2, %3}, [%4];" : "=l"(r.x), "=l"(r.y), "=l"(r.z), "=l"(r.w) : "l"(p));
    return r;
}
__device__ __forceinline__ U4 ld_cg4(const unsigned long long* p) {
    U4 r;
    asm volatile("ld.global.cg.L2::cache_hint.v4.u64 {%0, %1, %2, %3}, [%4], %5;"
                 : "=l"(r.x), "=l"(r.y), "=l"(r.z), "=l"(r.w) : "l"(p), "l"(policy_evict_last()));
    return r;
}
__device__ __forceinline__ U4 ld_plain4(const unsigned long long* p) {
    U4 r;
    asm volatile("ld.global.v4.u64 {%0, %1, %2, %3}, [%4];" : "=l"(r.x), "=l"(r.y), "=l"(r.z), "=l"(r.w) : "l"(p) : "memory");
    return r;
}
__device__ __forceinline__ void st4(unsigned long long* p, unsigned long long x, unsigned long long y,
                                    unsigned long long z, unsigned long long w) {
    asm volatile("st.global.v4.u64 [%0], {%1, %2, %3, %4};" :: "l"(p), "l"(x), "l"(y), "l"(z), "l"(w) : "memory");
}

// coherent (L2) variant for loops that run several levels in one launch
__device__ __forceinline__ ulonglong2 ld_keep_cg(const ulonglong2* p) {
    ulonglong2 r;
    asm volatile("ld.global.cg.L2::cache_hint.v2.u64 {%0, %1}, [%2], %3;"
                 : "=l"(r.x), "=l"(r.y) : "l"(p), "l"(policy_evict_last()));
    return r;
}

__device__ __forceinline__ unsigned long long global_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

}  // namespace

__device__ unsigned int g_check_bits;
__device__ void check_failed(uint32_t id) {
    if (!(atomicOr(&g_check_bits, 1u << (id & 31)) & (1u << (id & 31))))
        printf("[bpt] device bounds check %u failed (block %d thread %d)\n", id, blockIdx.x, threadIdx.x);
}
uint32_t checks_read_reset() {
#ifdef BPT_CHECKS
    unsigned int h = 0, z = 0;
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(&h, g_check_bits, 4);
    cudaMemcpyToSymbol(g_check_bits, &z, 4);
    return h;
#else
    return 0;
#endif
}

namespace {
// every kernel of the sampling graph counts its own execution (launch evidence)
__device__ __forceinline__ void count_self(Ctl* c) {
    if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) atomicAdd(&c->kernels_run, 1ull);
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
// Listing 1 lines 1-3: frontier[start].c = 1 -> here VN[slot][start].N |= bit,
// first setter of the (slot, slice) enqueues the raw entry of level 0.
// bitmap mode: colour `bit` of slot `slot` starts at v (U |= bit, v touched); vertex-major layout
// (a.vmajor): U[v * slots + slot] and one touched bit per vertex for all slots of the batch
__device__ __forceinline__ void mark_start(const BatchArgs& a, uint32_t slot, uint32_t v, uint32_t bit) {
    unsigned long long* U = reinterpret_cast<unsigned long long*>(a.VN);
    if (a.vmajor) {
        atomicOr(U + (size_t)v * a.slots_max + slot, 1ull << bit);
        atomicOr(&a.touched[v >> 5], 1u << (v & 31));
    } else {
        atomicOr(U + (size_t)slot * a.n + v, 1ull << bit);
        atomicOr(&a.touched[(size_t)slot * a.tiles * 32 + (v >> 5)], 1u << (v & 31));
    }
    a.lv[0].any = 1;
}

__global__ void k_init(BatchArgs a, cudaGraphConditionalHandle h_level, int use_cond) {
    count_self(a.ctl);
    const uint64_t total = (uint64_t)a.ctl->slots * 64;
    const uint64_t gblk0 = a.ctl->gblk0;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        a.ctl->cont = 1;
        a.ctl->level = 0;
        if (use_cond) cudaGraphSetConditional(h_level, 1);
    }
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t slot = (uint32_t)(i >> 6), bit = (uint32_t)(i & 63);
        const uint64_t s = 64ull * (gblk0 + slot) + bit;
        if (s >= a.theta) continue;
        const uint2 w = philox2x32_10((uint32_t)s, (uint32_t)(s >> 32), a.k_start);
        const uint64_t r64 = ((uint64_t)w.y << 32) | w.x;
        const uint32_t start = (uint32_t)__umul64hi(r64, (uint64_t)a.n);
        BPT_CHECK(start < a.n, 11);
        if (a.touched && a.slot_sample) {  // sorted start vertices: the slot holds another sample
            const uint64_t li = 64ull * (a.ctl->blk0 + slot) + bit;
            if (li >= a.nlocal) continue;
            const uint32_t ss = a.slot_sample[li];
            const uint2 w2 = philox2x32_10(ss, 0u, a.k_start);
            const uint32_t st2 = (uint32_t)__umul64hi(((uint64_t)w2.y << 32) | w2.x, (uint64_t)a.n);
            BPT_CHECK(st2 < a.n, 12);
            mark_start(a, slot, st2, bit);
            continue;
        }
        if (a.touched) {  // bitmap mode: mark the start, the compaction of level 0 finds it
            mark_start(a, slot, start, bit);
            continue;
        }
        uint32_t st = start;
        if (a.slot_sample) {  // sorted start vertices (C < 64 queue form): the slot holds another sample
            const uint64_t li = 64ull * (a.ctl->blk0 + slot) + bit;
            if (li >= a.nlocal) continue;
            const uint2 w2 = philox2x32_10(a.slot_sample[li], 0u, a.k_start);
            st = (uint32_t)__umul64hi(((uint64_t)w2.y << 32) | w2.x, (uint64_t)a.n);
            BPT_CHECK(st < a.n, 12);
        }
        const uint32_t slice = bit / a.colors;
        const uint64_t smask = slice_mask_of(a.colors, slice);
        const unsigned long long old = atomicOr(&a.VN[(size_t)slot * a.n + st].y, 1ull << bit);
        if ((old & smask) == 0) {
            const unsigned pos = atomicAdd(&a.lv[0].raw, 1u);
            if (pos < a.raw_cap) a.raw[pos] = raw_pack(st, slot, slice);
            else a.lv[0].overflow = 1;
        }
    }
}

// ------------------------------------------------------------------------ A4: compaction
// For each discovered (v, slot, slice) of level L: mask = N & slice; N &= ~slice;
// V |= mask (Listing 1 line 8 "visited[v] = visited[v] | fr_v"); keep the entry if v has
// in-edges (its expansion has work). 4 entries per thread (loads issued together); warp
// shuffle scans + one packed atomicAdd per 1,024-entry block tile allocate (entries, work)
// consistently; every work unit whose first item falls in the entry's range gets its index.
constexpr int kCompItems = 4;
constexpr uint32_t kCompTile = kThreads * kCompItems;

// kCoh: loads of data written earlier in the same launch bypass L1 (the persistent LT level
// loop below runs several levels per launch; separate launches see fresh L1s anyway)
#define LDX(ptr) (kCoh ? __ldcg(ptr) : *(ptr))
// Touched-bitmap mode (IC, 64 colours): the items are the vertices of 1,024-vertex tiles of each
// slot; item i of a tile is discovered iff its bit in the bitmap the expansion set is on (bits
// are cleared as they are read). Same per-item work as a queue entry from then on.
// kUnit: work items per expansion unit (a compile-time constant: the unit divisions below are
// multiplications then -- as a runtime 64-bit divisor they were a quarter of the kernel's instructions)
template <bool kCoh, uint32_t kUnit>
__device__ __forceinline__ void compact_body(const BatchArgs& a, uint32_t* __restrict__ tstart, uint64_t tstart_cap) {
    constexpr uint64_t unit = kUnit;
    LevelRec* L = &a.lv[LDX(&a.ctl->level)];
    const bool bitmap = a.touched != nullptr;
    const uint64_t nraw = bitmap ? (uint64_t)LDX(&a.ctl->slots) * a.tiles * kCompTile : umin64(LDX(&L->raw), a.raw_cap);
    if (blockIdx.x > 0 && (uint64_t)blockIdx.x * kCompTile >= nraw) return;  // no tile of this level
    if (threadIdx.x == 0) atomicMin(&a.ctl->c_start, global_ns());
    __shared__ unsigned long long wsum[kWarps];
    __shared__ uint32_t wcnt[kWarps];
    __shared__ unsigned long long blk_base;
    __shared__ unsigned long long vc_acc[kWarps];
    constexpr uint32_t kBig = 64;
    __shared__ unsigned long long big_u0[kBig], big_u1[kBig];
    __shared__ uint32_t big_q[kBig];
    __shared__ uint32_t big_n;
    if (threadIdx.x == 0) big_n = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    unsigned long long vc_local = 0;
    uint32_t touched_local = 0;
    // bitmap mode: the block's tiles (block b: tiles b, b + G, ...) are first screened with one
    // warp-wide 128-B load per tile, and only the non-empty ones are processed (most tiles of the
    // thin levels are empty: 4 x 4,734 tiles per C2 level)
    constexpr uint32_t kScreen = 256;  // tiles screened per pass
    __shared__ uint32_t nonempty[kScreen];
    __shared__ uint32_t n_nonempty;
    const uint32_t ntiles_all = bitmap ? (uint32_t)(nraw / kCompTile) : 0u;
    uint32_t k0 = 0;       // first screened tile index (in units of the grid stride) of this pass
    uint32_t li = 0;       // next non-empty tile of this pass
    uint64_t tile0 = (uint64_t)blockIdx.x * kCompTile;
    while (true) {
        if (bitmap) {
            if (li == 0 || li >= n_nonempty) {  // screen the next kScreen tiles of this block
                __syncthreads();
                if (li != 0) k0 += kScreen;
                li = 0;
                if (threadIdx.x == 0) n_nonempty = 0;
                __syncthreads();
                if ((uint64_t)blockIdx.x + (uint64_t)k0 * gridDim.x >= ntiles_all) break;
                for (uint32_t k = k0 + wid; k < k0 + kScreen; k += kWarps) {
                    const uint64_t t = (uint64_t)blockIdx.x + (uint64_t)k * gridDim.x;
                    if (t >= ntiles_all) break;
                    uint32_t w = LDX(a.touched + t * 32 + lane);
                    if (a.F) w |= LDX(a.FB + t * 32 + lane);  // pull: leavers of the previous frontier
                    if (__any_sync(kFull, w != 0) && lane == 0) nonempty[atomicAdd(&n_nonempty, 1u)] = (uint32_t)t;
                }
                __syncthreads();
                if (n_nonempty == 0) { li = 1; continue; }  // nothing in this pass: screen the next one
            }
            tile0 = (uint64_t)nonempty[li++] * kCompTile;
        } else {
            if (tile0 >= nraw) break;
        }
        uint64_t r[kCompItems];
        if (bitmap) {
            // tile t of slot t / tiles covers vertices 1024 (t % tiles) + [0, 1024); item it of
            // thread x is vertex it * 256 + x of the tile: bit `lane` of word 8 it + warp
            const uint32_t t = (uint32_t)(tile0 / kCompTile);
            const uint32_t slot = t / a.tiles;
            const uint32_t vbase = (t - slot * a.tiles) * kCompTile;
            uint32_t* wp = a.touched + t * 32 + wid;
            uint32_t wv[kCompItems];
#pragma unroll
            for (int it = 0; it < kCompItems; ++it) wv[it] = LDX(wp + 8 * it);
            if (a.F) {
                // pull: F[v][slot] holds the frontier masks of the current level; the vertices of the
                // previous level's frontier that are not in this one are cleared here (FB = the previous
                // level's touched words), the new ones are written below with their masks
                uint32_t* fp = a.FB + t * 32 + wid;
#pragma unroll
                for (int it = 0; it < kCompItems; ++it) {
                    const uint32_t pv = LDX(fp + 8 * it);
                    if (((pv & ~wv[it]) >> lane) & 1u)
                        a.F[(size_t)(vbase + it * kThreads + threadIdx.x) * a.slots_max + slot] = 0ull;
                    __syncwarp();
                    if (lane == it && pv != wv[it]) fp[8 * it] = wv[it];
                }
            }
#pragma unroll
            for (int it = 0; it < kCompItems; ++it) {
                const bool on = (wv[it] >> lane) & 1u;
                r[it] = on ? raw_pack(vbase + it * kThreads + threadIdx.x, slot, 0) : ~0ull;
                touched_local += on;
            }
            __syncwarp();
#pragma unroll
            for (int it = 0; it < kCompItems; ++it)  // cleared for the next level
                if (lane == it && wv[it]) wp[8 * it] = 0;
        } else {
#pragma unroll
            for (int it = 0; it < kCompItems; ++it) {
                const uint64_t i = tile0 + (uint64_t)it * kThreads + threadIdx.x;
                r[it] = i < nraw ? LDX(&a.raw[i]) : ~0ull;
            }
            tile0 += (uint64_t)gridDim.x * kCompTile;
        }
        uint64_t mask[kCompItems];
        uint32_t rs[kCompItems], re[kCompItems];
#pragma unroll
        for (int it = 0; it < kCompItems; ++it) {
            mask[it] = 0;
            rs[it] = re[it] = 0;
            if (r[it] != ~0ull) {
                const uint32_t v = (uint32_t)r[it];
                const uint32_t slot = (uint32_t)(r[it] >> 32) & ((1u << 26) - 1u);
                ulonglong2* p = &a.VN[(size_t)slot * a.n + v];
                if (bitmap) {  // union layout: new = U & ~V, V = U
                    unsigned long long* U = reinterpret_cast<unsigned long long*>(a.VN);
                    const size_t iu = (size_t)slot * a.n + v, iv = (size_t)a.slots_max * a.n + iu;
                    const unsigned long long u = LDX(&U[iu]);
                    mask[it] = u & ~LDX(&U[iv]);
                    U[iv] = u;
                    if (a.F) a.F[(size_t)v * a.slots_max + slot] = mask[it];
                } else if (a.colors == 64) {
                    const ulonglong2 x = LDX(p);
                    mask[it] = x.y;
                    *p = make_ulonglong2(x.x | x.y, 0ull);
                } else {
                    const uint64_t sm = slice_mask_of(a.colors, (uint32_t)(r[it] >> 58));
                    mask[it] = atomicAnd(&p->y, ~sm) & sm;
                    atomicOr(&p->x, mask[it]);
                }
                rs[it] = __ldg(&a.roff[v]);
                re[it] = __ldg(&a.roff[v + 1]);
            }
        }
        uint32_t cnt = 0;
        unsigned long long work_t = 0;
        uint64_t work[kCompItems];
#pragma unroll
        for (int it = 0; it < kCompItems; ++it) {
            vc_local += __popcll(mask[it]);
            const uint32_t deg = re[it] - rs[it];
            work[it] = a.model == BPT_IC ? deg : (deg ? __popcll(mask[it]) : 0);
            cnt += work[it] != 0;
            work_t += work[it];
        }
        // warp inclusive scans of (count, work)
        uint32_t cincl = cnt;
        unsigned long long wincl = work_t;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t yc = __shfl_up_sync(kFull, cincl, d);
            const unsigned long long yw = __shfl_up_sync(kFull, wincl, d);
            if (lane >= d) { cincl += yc; wincl += yw; }
        }
        if (lane == 31) { wsum[wid] = wincl; wcnt[wid] = cincl; }
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned long long ts = 0;
            uint32_t tc = 0;
            for (int w = 0; w < kWarps; ++w) {
                const unsigned long long s2 = wsum[w];
                const uint32_t c2 = wcnt[w];
                wsum[w] = ts; wcnt[w] = tc; ts += s2; tc += c2;
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
        if (bb != ~0ull && cnt) {
            uint64_t qi = (bb >> kPackShift) + wcnt[wid] + cincl - cnt;
            uint64_t off = (bb & kEdgeMask) + wsum[wid] + wincl - work_t;
            uint64_t mword = ~0ull;  // entry-start bits, merged per 32-item word before the atomic
            uint32_t mbits = 0;
#pragma unroll
            for (int it = 0; it < kCompItems; ++it) {
                if (!work[it]) continue;
                const uint32_t v = (uint32_t)r[it];
                const uint32_t slot = (uint32_t)(r[it] >> 32) & ((1u << 26) - 1u);
                // IC entries carry delta = rowstart - off (mod 2^32): edge id e = t + delta for
                // work item t; LT entries carry the vertex itself
                const uint32_t x = a.model == BPT_IC ? rs[it] - (uint32_t)off : v;
                BPT_CHECK(qi < a.q_cap && v < a.n && slot < a.slots_max, 9);
                a.q[qi] = make_uint4(x, slot, (uint32_t)mask[it], (uint32_t)(mask[it] >> 32));
                if (a.model != BPT_IC) a.qoff[qi] = off;  // IC finds entries via tstart + umask
                if (a.umask && off / unit < tstart_cap) {
                    BPT_CHECK((off >> 5) < a.umask_words, 10);
                    if ((off >> 5) != mword) {
                        if (mbits) atomicOr(&a.umask[mword], mbits);
                        mword = off >> 5;
                        mbits = 0;
                    }
                    mbits |= 1u << (off & 31u);
                }
                // work units whose first item falls inside [off, off + work)
                const uint64_t u0 = (off + unit - 1) / unit, u1 = (off + work[it] + unit - 1) / unit;
                if (u1 > tstart_cap) L->overflow = 1;
                const uint64_t u1c = umin64(u1, tstart_cap);
                if (u1c > u0 + 4) {  // long entry (hub): filled by the whole block below
                    const uint32_t bi = atomicAdd(&big_n, 1u);
                    if (bi < kBig) {
                        big_u0[bi] = u0;
                        big_u1[bi] = u1c;
                        big_q[bi] = (uint32_t)qi;
                    } else {
                        for (uint64_t t = u0; t < u1c; ++t) tstart[t] = (uint32_t)qi;
                    }
                } else {
                    for (uint64_t t = u0; t < u1c; ++t) tstart[t] = (uint32_t)qi;
                }
                ++qi;
                off += work[it];
            }
            if (mbits) atomicOr(&a.umask[mword], mbits);
        }
        __syncthreads();
        const uint32_t nbig = min(big_n, (uint32_t)kBig);
        for (uint32_t bi = 0; bi < nbig; ++bi)
            for (uint64_t t = big_u0[bi] + threadIdx.x; t < big_u1[bi]; t += kThreads) tstart[t] = big_q[bi];
        __syncthreads();
        if (threadIdx.x == 0) big_n = 0;
    }
    // level statistics
    unsigned long long vc_tot = block_sum_ull(vc_local, vc_acc);
    if (threadIdx.x == 0 && vc_tot) atomicAdd(&L->vc, vc_tot);
    if (bitmap) {
        const unsigned long long tt = block_sum_ull(touched_local, vc_acc);
        if (threadIdx.x == 0 && tt) atomicAdd(&L->raw, (unsigned)tt);
    }
    if (threadIdx.x == 0) atomicMax(&a.ctl->c_end, global_ns());
}


template <uint32_t kUnit>
__global__ void __launch_bounds__(kThreads, 5) k_compact(BatchArgs a, uint32_t* __restrict__ tstart,
                                                      uint64_t tstart_cap) {
    count_self(a.ctl);
    if (!a.ctl->cont) return;
    compact_body<false, kUnit>(a, tstart, tstart_cap);
}


// Touched-bitmap compaction (IC, 64 colours), warp-centric: one warp per 1,024-vertex tile of a slot
// (32 bitmap words, one per lane). The touched vertices of the tile are listed in shared memory
// (each lane appends the set bits of its word), then processed 32 at a time with every lane busy:
//   pass 1: kept entries and their work (in-degrees, roff only) -> ONE packed atomicAdd per tile
//           allocates the entries and their work range (Listing 1 lines 7-8 need no order);
//   pass 2: new = U & ~V, V = U (reading C-7), the entry {rowstart - off, slot, new}, its
//           entry-start bit and the first entry of every expansion unit starting inside its range
//           (hub ranges filled by the whole warp).
// No block barriers and one global atomic per non-empty tile (the block-wide form paid three
// barriers and a serialised atomic per tile, ~46 warp-instructions per touched vertex; the
// touched vertices of the heavy levels are spread over every tile of the slot).
constexpr uint32_t kTileV = 1024;  // vertices per bitmap tile (32 words)
template <uint32_t kUnit>
__global__ void __launch_bounds__(kThreads) k_compact_bm(BatchArgs a, uint32_t* __restrict__ tstart,
                                                         uint64_t tstart_cap) {
    count_self(a.ctl);
    if (!a.ctl->cont) return;
    Ctl* ctl = a.ctl;
    LevelRec* L = &a.lv[ctl->level];
    const uint32_t ntiles = ctl->slots * a.tiles;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const uint32_t lt_mask = (1u << lane) - 1u;
    __shared__ uint16_t vlist[kWarps][kTileV];
    __shared__ unsigned long long red[kWarps];
    if (blockIdx.x * kWarps < ntiles && threadIdx.x == 0) atomicMin(&ctl->c_start, global_ns());
    unsigned long long vc_local = 0;
    uint32_t touched_local = 0;
    unsigned long long* U = reinterpret_cast<unsigned long long*>(a.VN);
    for (uint32_t t = blockIdx.x * kWarps + wid; t < ntiles; t += gridDim.x * kWarps) {
        const uint32_t w = a.touched[(size_t)t * 32 + lane];
        const uint32_t pv = a.F ? a.FB[(size_t)t * 32 + lane] : 0u;
        if (!__any_sync(kFull, (w | pv) != 0u)) continue;
        const uint32_t slot = t / a.tiles, vbase = (t - slot * a.tiles) * kTileV;
        if (w) a.touched[(size_t)t * 32 + lane] = 0u;  // cleared for the next level
        if (a.F) {
            // pull: F[v][slot] = the frontier masks of this level; vertices of the previous level's
            // frontier that are not in this one leave it (FB = the previous level's touched words)
            if (pv != w) a.FB[(size_t)t * 32 + lane] = w;
            for (uint32_t x = pv & ~w; x; x &= x - 1u)
                a.F[(size_t)(vbase + 32u * lane + __ffs(x) - 1u) * a.slots_max + slot] = 0ull;
        }
        const uint32_t c = __popc(w);
        uint32_t incl = c;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t y = __shfl_up_sync(kFull, incl, d);
            if (lane >= d) incl += y;
        }
        const uint32_t total = __shfl_sync(kFull, incl, 31);
        touched_local += c;
        if (total == 0) continue;
        {
            uint32_t pos = incl - c;
            for (uint32_t x = w; x; x &= x - 1u) vlist[wid][pos++] = (uint16_t)(32u * lane + __ffs(x) - 1u);
        }
        __syncwarp();
        // pass 1: kept entries (in-degree > 0) and their work
        uint32_t cnt = 0;
        unsigned long long work = 0;
        for (uint32_t j = lane; j < total; j += 32) {
            const uint32_t v = vbase + vlist[wid][j];
            const uint32_t d = __ldg(&a.roff[v + 1]) - __ldg(&a.roff[v]);
            cnt += d != 0u;
            work += d;
        }
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) {
            cnt += __shfl_xor_sync(kFull, cnt, d);
            work += __shfl_xor_sync(kFull, work, d);
        }
        unsigned long long base = ~0ull;
        if (lane == 0 && cnt) {
            const unsigned long long old = atomicAdd(&L->packed, ((unsigned long long)cnt << kPackShift) + work);
            if ((old >> kPackShift) + cnt > a.q_cap || (old & kEdgeMask) + work > kEdgeMask) L->overflow = 1;
            else base = old;
        }
        base = __shfl_sync(kFull, base, 0);
        uint64_t qi = base >> kPackShift, off = base & kEdgeMask;
        // pass 2, 32 touched vertices at a time
        for (uint32_t j0 = 0; j0 < total; j0 += 32) {
            const uint32_t j = j0 + lane;
            const bool has = j < total;
            uint32_t v = 0, rs = 0, d = 0;
            unsigned long long mask = 0ull;
            if (has) {
                v = vbase + vlist[wid][j];
                BPT_CHECK(v < a.n && slot < a.slots_max, 9);
                const size_t iu = (size_t)slot * a.n + v, iv = (size_t)a.slots_max * a.n + iu;
                const unsigned long long uu = U[iu];
                mask = uu & ~U[iv];
                U[iv] = uu;
                if (a.F) a.F[(size_t)v * a.slots_max + slot] = mask;
                rs = __ldg(&a.roff[v]);
                d = __ldg(&a.roff[v + 1]) - rs;
                vc_local += __popcll(mask);
            }
            const bool kept = d != 0u;
            const uint32_t kb = __ballot_sync(kFull, kept);
            uint32_t wx = kept ? d : 0u;  // exclusive scan of the chunk's work
            uint32_t wi = wx;
#pragma unroll
            for (int s2 = 1; s2 < 32; s2 <<= 1) {
                const uint32_t y = __shfl_up_sync(kFull, wi, s2);
                if (lane >= s2) wi += y;
            }
            const uint32_t chunk_work = __shfl_sync(kFull, wi, 31);
            if (base == ~0ull) continue;
            bool longr = false;
            uint64_t u0 = 0, u1c = 0, myq = 0;
            if (kept) {
                myq = qi + __popc(kb & lt_mask);
                const uint64_t myoff = off + (wi - wx);
                BPT_CHECK(myq < a.q_cap, 9);
                // IC entries carry delta = rowstart - off (mod 2^32): edge id e = t + delta for work item t
                a.q[myq] = make_uint4(rs - (uint32_t)myoff, slot, (uint32_t)mask, (uint32_t)(mask >> 32));
                if (myoff / kUnit < tstart_cap) {
                    BPT_CHECK((myoff >> 5) < a.umask_words, 10);
                    atomicOr(&a.umask[myoff >> 5], 1u << (myoff & 31u));
                }
                // expansion units whose first item falls inside [myoff, myoff + d)
                u0 = (myoff + kUnit - 1) / kUnit;
                const uint64_t u1 = (myoff + d + kUnit - 1) / kUnit;
                if (u1 > tstart_cap) L->overflow = 1;
                u1c = umin64(u1, tstart_cap);
                longr = u1c > u0 + 4;
                if (!longr)
                    for (uint64_t x = u0; x < u1c; ++x) tstart[x] = (uint32_t)myq;
            }
            for (uint32_t lb = __ballot_sync(kFull, longr); lb; lb &= lb - 1u) {  // hub ranges: the whole warp
                const int src = __ffs(lb) - 1;
                const uint64_t a0 = __shfl_sync(kFull, u0, src), a1 = __shfl_sync(kFull, u1c, src);
                const uint32_t qv = (uint32_t)__shfl_sync(kFull, myq, src);
                for (uint64_t x = a0 + lane; x < a1; x += 32) tstart[x] = qv;
            }
            qi += __popc(kb);
            off += chunk_work;
        }
        __syncwarp();
    }
    unsigned long long vc_tot = block_sum_ull(vc_local, red);
    if (threadIdx.x == 0 && vc_tot) atomicAdd(&L->vc, vc_tot);
    const unsigned long long tt = block_sum_ull(touched_local, red);
    if (threadIdx.x == 0 && tt) atomicAdd(&L->raw, (unsigned)tt);
    if (blockIdx.x * kWarps < ntiles && threadIdx.x == 0) atomicMax(&ctl->c_end, global_ns());
}


// Batch-wide frontier (a.vmajor; SURVEY §8(f) NEXT #2 with the product's machinery): the S <= 4
// blocks of a batch share one frontier of VERTICES. Tiles are 1,024-vertex tiles of the single
// per-vertex touched bitmap; a touched vertex's new colours of every slot come from one 32-B
// sector of U and of V (vertex-major union layout), and it becomes ONE entry {delta} + S masks.
// Measured with the oracle on C2's sorted groups: one 256-sample fused traversal reads 3.1-3.3x
// fewer reverse edges than its four 64-sample groups (scripts/dbg/overlap.py).
template <uint32_t kUnit>
__global__ void __launch_bounds__(kThreads) k_compact_bmv(BatchArgs a, uint32_t* __restrict__ tstart,
                                                          uint64_t tstart_cap) {
    count_self(a.ctl);
    if (!a.ctl->cont) return;
    Ctl* ctl = a.ctl;
    LevelRec* L = &a.lv[ctl->level];
    const uint32_t ntiles = a.tiles, S = a.slots_max;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const uint32_t lt_mask = (1u << lane) - 1u;
    __shared__ uint16_t vlist[kWarps][kTileV];
    __shared__ unsigned long long red[kWarps];
    if (blockIdx.x * kWarps < ntiles && threadIdx.x == 0) atomicMin(&ctl->c_start, global_ns());
    unsigned long long vc_local = 0;
    uint32_t touched_local = 0;
    unsigned long long* U = reinterpret_cast<unsigned long long*>(a.VN);
    unsigned long long* V = U + (size_t)S * a.n;
    for (uint32_t t = blockIdx.x * kWarps + wid; t < ntiles; t += gridDim.x * kWarps) {
        const uint32_t w = a.touched[(size_t)t * 32 + lane];
        if (!__any_sync(kFull, w != 0u)) continue;
        const uint32_t vbase = t * kTileV;
        if (w) a.touched[(size_t)t * 32 + lane] = 0u;  // cleared for the next level
        const uint32_t c = __popc(w);
        uint32_t incl = c;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t y = __shfl_up_sync(kFull, incl, d);
            if (lane >= d) incl += y;
        }
        const uint32_t total = __shfl_sync(kFull, incl, 31);
        touched_local += c;
        {
            uint32_t pos = incl - c;
            for (uint32_t x = w; x; x &= x - 1u) vlist[wid][pos++] = (uint16_t)(32u * lane + __ffs(x) - 1u);
        }
        __syncwarp();
        uint32_t cnt = 0;
        unsigned long long work = 0;
        for (uint32_t j = lane; j < total; j += 32) {
            const uint32_t v = vbase + vlist[wid][j];
            const uint32_t d = __ldg(&a.roff[v + 1]) - __ldg(&a.roff[v]);
            cnt += d != 0u;
            work += d;
        }
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) {
            cnt += __shfl_xor_sync(kFull, cnt, d);
            work += __shfl_xor_sync(kFull, work, d);
        }
        unsigned long long base = ~0ull;
        if (lane == 0 && cnt) {
            const unsigned long long old = atomicAdd(&L->packed, ((unsigned long long)cnt << kPackShift) + work);
            if ((old >> kPackShift) + cnt > a.q_cap || (old & kEdgeMask) + work > kEdgeMask) L->overflow = 1;
            else base = old;
        }
        base = __shfl_sync(kFull, base, 0);
        uint64_t qi = base >> kPackShift, off = base & kEdgeMask;
        for (uint32_t j0 = 0; j0 < total; j0 += 32) {
            const uint32_t j = j0 + lane;
            const bool has = j < total;
            uint32_t v = 0, rs = 0, d = 0;
            unsigned long long nm[4] = {0ull, 0ull, 0ull, 0ull};
            if (has) {
                v = vbase + vlist[wid][j];
                BPT_CHECK(v < a.n, 9);
                const size_t b = (size_t)v * S;
                if (S == 4) {
                    const U4 uu = ld_plain4(U + b), vv = ld_plain4(V + b);
                    nm[0] = uu.x & ~vv.x; nm[1] = uu.y & ~vv.y; nm[2] = uu.z & ~vv.z; nm[3] = uu.w & ~vv.w;
                    st4(V + b, uu.x, uu.y, uu.z, uu.w);
                } else {
#pragma unroll
                    for (uint32_t sl = 0; sl < 4; ++sl)
                        if (sl < S) {
                            const unsigned long long uu = U[b + sl];
                            nm[sl] = uu & ~V[b + sl];
                            V[b + sl] = uu;
                        }
                }
#pragma unroll
                for (uint32_t sl = 0; sl < 4; ++sl) vc_local += __popcll(nm[sl]);
                rs = __ldg(&a.roff[v]);
                d = __ldg(&a.roff[v + 1]) - rs;
            }
            const bool kept = d != 0u;
            const uint32_t kb = __ballot_sync(kFull, kept);
            uint32_t wx = kept ? d : 0u;
            uint32_t wi = wx;
#pragma unroll
            for (int s2 = 1; s2 < 32; s2 <<= 1) {
                const uint32_t y = __shfl_up_sync(kFull, wi, s2);
                if (lane >= s2) wi += y;
            }
            const uint32_t chunk_work = __shfl_sync(kFull, wi, 31);
            if (base == ~0ull) continue;
            bool longr = false;
            uint64_t u0 = 0, u1c = 0, myq = 0;
            if (kept) {
                myq = qi + __popc(kb & lt_mask);
                const uint64_t myoff = off + (wi - wx);
                BPT_CHECK(myq < a.q_cap, 9);
                a.qd[myq] = rs - (uint32_t)myoff;  // edge id e = work item + delta (mod 2^32)
                unsigned long long* qm = a.qmask + (size_t)myq * S;
                if (S == 4) {
                    st4(qm, nm[0], nm[1], nm[2], nm[3]);
                } else {
#pragma unroll
                    for (uint32_t sl = 0; sl < 4; ++sl)
                        if (sl < S) qm[sl] = nm[sl];
                }
                if (myoff / kUnit < tstart_cap) {
                    BPT_CHECK((myoff >> 5) < a.umask_words, 10);
                    atomicOr(&a.umask[myoff >> 5], 1u << (myoff & 31u));
                }
                u0 = (myoff + kUnit - 1) / kUnit;
                const uint64_t u1 = (myoff + d + kUnit - 1) / kUnit;
                if (u1 > tstart_cap) L->overflow = 1;
                u1c = umin64(u1, tstart_cap);
                longr = u1c > u0 + 4;
                if (!longr)
                    for (uint64_t x = u0; x < u1c; ++x) tstart[x] = (uint32_t)myq;
            }
            for (uint32_t lb = __ballot_sync(kFull, longr); lb; lb &= lb - 1u) {
                const int src = __ffs(lb) - 1;
                const uint64_t a0 = __shfl_sync(kFull, u0, src), a1 = __shfl_sync(kFull, u1c, src);
                const uint32_t qv = (uint32_t)__shfl_sync(kFull, myq, src);
                for (uint64_t x = a0 + lane; x < a1; x += 32) tstart[x] = qv;
            }
            qi += __popc(kb);
            off += chunk_work;
        }
        __syncwarp();
    }
    unsigned long long vc_tot = block_sum_ull(vc_local, red);
    if (threadIdx.x == 0 && vc_tot) atomicAdd(&L->vc, vc_tot);
    const unsigned long long tt = block_sum_ull(touched_local, red);
    if (threadIdx.x == 0 && tt) atomicAdd(&L->raw, (unsigned)tt);
    if (blockIdx.x * kWarps < ntiles && threadIdx.x == 0) atomicMax(&ctl->c_end, global_ns());
}

// ------------------------------------------------------------------------ A3: expansion
struct SmemTile {  // LT expansion tile staging
    uint32_t rel[kTile + 1];   // max(qoff - t0, 0) per entry of the tile
    uint32_t aux[kTile + 1];   // tasks of the entry before the tile
    uint32_t v[kTile + 1];     // LT: vertex
    uint32_t slot[kTile + 1];
    unsigned long long mask[kTile + 1];
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

__device__ __forceinline__ void advance_level(const BatchArgs& a, cudaGraphConditionalHandle h_level, int use_cond) {
    Ctl* c = a.ctl;
    // The counters were updated by other blocks' atomics (and, in the cooperative LT loop, by
    // other blocks' earlier advances): read them from L2 (.cg), all in one batch of vector
    // loads -- this runs on the critical path of every level.
    Ctl C;
    {
        const uint4* src = reinterpret_cast<const uint4*>(c);
        uint4* dst = reinterpret_cast<uint4*>(&C);
#pragma unroll
        for (int i = 0; i < (int)(sizeof(Ctl) / 16); ++i) dst[i] = __ldcg(src + i);
    }
    const uint32_t Lv = C.level;
    LevelRec R;
    {
        const uint4* src = reinterpret_cast<const uint4*>(&a.lv[Lv]);
        uint4* dst = reinterpret_cast<uint4*>(&R);
#pragma unroll
        for (int i = 0; i < (int)(sizeof(LevelRec) / 16); ++i) dst[i] = __ldcg(src + i);
    }
    const uint2 nx = __ldcg(reinterpret_cast<const uint2*>(&a.lv[Lv + 1].raw));  // {raw, overflow}
    R.pad = 0;
    const uint32_t next_raw = a.touched ? __ldcg(&a.lv[Lv + 1].any) : nx.x, next_ovf = nx.y;
    c->work = C.work + (R.packed & kEdgeMask);
    c->entries = C.entries + (R.packed >> kPackShift);
    c->vc = C.vc + R.vc;
    c->coins = C.coins + R.coins;
    c->atomics = C.atomics + R.atomics;
    c->pull_reads = C.pull_reads + R.pull_reads;
    c->pull_levels = C.pull_levels + R.pull;
    if (C.t_start != ~0ull && C.t_end > C.t_start) c->expand_ns = C.expand_ns + (C.t_end - C.t_start);
    if (C.c_start != ~0ull && C.c_end > C.c_start) c->compact_ns = C.compact_ns + (C.c_end - C.c_start);
    c->t_start = ~0ull;
    c->t_end = 0;
    c->c_start = ~0ull;
    c->c_end = 0;
    if (C.stats_used < a.stats_cap) {
        LevelRec row = R;
        row.pad = ((unsigned long long)C.batch << 32) | Lv;
        a.stats[C.stats_used] = row;
        c->stats_used = C.stats_used + 1;
    } else {
        c->stats_overflow = 1;
    }
    const bool ovf = R.overflow || next_ovf;
    if (ovf) c->error = 1;
    bool cont = next_raw != 0 && !ovf;
    if (cont && Lv + 2 >= (uint32_t)kMaxLevels) { c->error = 2; cont = false; }
    c->level = Lv + 1;
    if (!cont) {
        c->cont = 0;
        c->levels_total = C.levels_total + Lv + 1;
        if (Lv + 1 > C.levels_max) c->levels_max = Lv + 1;
    }
    if (use_cond) cudaGraphSetConditional(h_level, cont ? 1u : 0u);
}

// The last block of an expansion launch to finish advances the level (fused, no extra launch).
// nblocks: blocks of this launch that take part (the others left without counting themselves)
__device__ __forceinline__ void finish_expand(const BatchArgs& a, cudaGraphConditionalHandle h_level, int use_cond,
                                              uint32_t nblocks) {
    __syncthreads();
    if (threadIdx.x == 0) {
        atomicMax(&a.ctl->t_end, global_ns());
        __threadfence();
        const unsigned prev = atomicAdd(&a.ctl->blocks_done, 1u);
        if (prev == nblocks - 1) {
            __threadfence();
            a.ctl->blocks_done = 0;
            advance_level(a, h_level, use_cond);
        }
    }
}

// pull or push for this level (both expansion kernels of a level take the same decision)
__device__ __forceinline__ bool pull_level(const BatchArgs& a, const LevelRec* L) {
    return a.pull != nullptr && !L->overflow && (L->packed & kEdgeMask) >= a.pull_min_work;
}

// IC, Listing 1 lines 9-15: for each frontier entry (v, slot, mask) and each reverse edge e
// of v: u = src[e]; live = mask & ~V[u]; every live colour c keeps its bit iff the coin
// of (sample c, e) passes (reading C-2); surviving bits are OR-merged into N[u] (line 14,
// the fusing step); the first setter of N[u] (per slice) enqueues u for level L+1.
//
// Warp-centric and barrier-free: a warp owns units of kUnitIC = 32 * kWinIC (96) consecutive
// work items (reverse edge reads) as kWinIC windows of 32 lanes. The entry of every item comes
// from the unit's first entry (tstart) + a popcount of the entry-start bitmap (no per-edge
// search). The windows' loads are issued together (kWinIC x memory-level parallelism). The
// live colours of all the unit's edges are flattened into one list of
// (edge, colour) coin tasks evaluated 32 at a time (full lanes, no divergence to the
// warp's maximum colour count). Discovered vertices go through a per-warp shared buffer,
// so the global queue counter sees one atomic per >= 32 entries.
#ifndef BPT_WIN_IC
#define BPT_WIN_IC 3
#endif
#ifdef BPT_HIST
__device__ unsigned long long g_hist[16 * 80];
#endif
constexpr int kWinIC = BPT_WIN_IC;       // 32-lane windows per warp work unit
static_assert(kWinIC >= 1 && kWinIC <= 4, "the window search packs <= 3 window prefixes into 8-bit fields");
constexpr int kUnitIC = 32 * kWinIC;
constexpr int kEbuf = 32 + kUnitIC;  // <= 31 pending + one unit's new entries

struct WarpScratch {
    uint32_t excl[32];                  // exclusive prefix of the lanes' task counts
    uint32_t cum[32];                   // per-lane window prefix: c0 | (c0+c1) << 8 | (c0+c1+c2) << 16
    unsigned long long live[kWinIC][32];
    uint32_t e[kWinIC][32];
    uint32_t thr[kWinIC][32];
    uint32_t sbase[kWinIC][32];
    unsigned long long pass[kWinIC][32];  // updated through its 32-bit halves: native ATOMS.OR
    unsigned long long ebuf[kEbuf];
    uint32_t ecount;
};

__device__ __forceinline__ void warp_flush(const BatchArgs& a, LevelRec* Ln, WarpScratch& W, int lane) {
    const uint32_t cnt = W.ecount;
    if (cnt == 0) return;
    unsigned base = 0;
    if (lane == 0) base = atomicAdd(&Ln->raw, cnt);
    base = __shfl_sync(kFull, base, 0);
    for (uint32_t i = lane; i < cnt; i += 32) {
        const uint64_t pos = (uint64_t)base + i;
        if (pos < a.raw_cap) a.raw[pos] = W.ebuf[i];
        else Ln->overflow = 1;
    }
    __syncwarp();
    if (lane == 0) W.ecount = 0;
    __syncwarp();
}

__device__ __forceinline__ uint32_t warp_incl_scan_u32(uint32_t x, int lane) {
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, x, d);
        if (lane >= d) x += y;
    }
    return x;
}

__device__ __forceinline__ void coin_task(const BatchArgs& a, WarpScratch& W, uint32_t o, uint32_t w, uint32_t bit) {
    // sorted start vertices (C < 64): sbase is the slot's local index, mapped to its sample
    const uint32_t sid = a.slot_sample ? __ldg(&a.slot_sample[W.sbase[w][o] + bit]) : W.sbase[w][o] + bit;
    const uint32_t x = philox2x32_10(W.e[w][o], sid, a.k_ic).x;
    if ((x >> 1) < W.thr[w][o])
        atomicOr(reinterpret_cast<uint32_t*>(&W.pass[w][o]) + (bit >> 5), 1u << (bit & 31));
}

// One kUnitIC-item unit. kWhole: all items valid (every unit but the last of a level), so no
// per-lane predication is needed on the loads.
template <bool kWhole, bool kC64, bool kCoh>
__device__ __forceinline__ void expand_unit_ic(const BatchArgs& a, LevelRec* Ln, WarpScratch& W, int lane,
                                               uint32_t le_mask, uint32_t unit, uint32_t rem,
                                               uint32_t jc0, uint64_t gblk0, unsigned long long& coins,
                                               unsigned long long& atoms) {
    const uint32_t t0l = unit * (uint32_t)kUnitIC;  // mod 2^32: edge ids are t + delta (mod 2^32)
    // ---- entry of every item: jc0 contains item 0; the compaction marked every entry start in
    //      the unit's kUnitIC-bit mask (the unit's own mask is cleared here for the next level)
    uint32_t mw[kWinIC];
#pragma unroll
    for (int w = 0; w < kWinIC; ++w) mw[w] = LDX(&a.umask[(size_t)unit * kWinIC + w]);
    __syncwarp();
    if (lane < kWinIC) a.umask[(size_t)unit * kWinIC + lane] = 0;
    mw[0] &= ~1u;  // an entry starting at item 0 is jc0 itself
    uint32_t jl[kWinIC];
    uint32_t before = jc0;
#pragma unroll
    for (int w = 0; w < kWinIC; ++w) {
        jl[w] = before + __popc(mw[w] & le_mask);
        before += __popc(mw[w]);
    }
    // ---- loads of the 4 windows issued together (32-bit index math: slots * n < 2^32).
    //      Invalid items of the last unit re-read a valid item and are masked out below.
    uint4 ent[kWinIC];
    uint2 rc[kWinIC];
    uint32_t vidx[kWinIC];
    uint64_t live[kWinIC];
#pragma unroll
    for (int w = 0; w < kWinIC; ++w) ent[w] = LDX(&a.q[(kWhole || 32u * w + lane < rem) ? jl[w] : jc0]);
#pragma unroll
    for (int w = 0; w < kWinIC; ++w) {
        // an invalid item re-reads item 0 of the unit, which lies in entry jc0
        const uint32_t i = (kWhole || 32u * w + lane < rem) ? 32u * w + lane : 0u;
        rc[w] = ld_stream(&a.rec[t0l + i + ent[w].x]);
    }
#pragma unroll
    for (int w = 0; w < kWinIC; ++w) {
        // {V[u], N[u]}: colours visited, or already merged into u this level by another edge
        // (a possibly stale N only skips fewer coins; the merged result is the same)
        vidx[w] = ent[w].y * a.n + rc[w].x;
        const ulonglong2 vn = kCoh ? ld_keep_cg(&a.VN[vidx[w]]) : ld_keep(&a.VN[vidx[w]]);
        live[w] = (((uint64_t)ent[w].w << 32) | ent[w].z) & ~(vn.x | vn.y);
        if (!kWhole && 32u * w + lane >= rem) live[w] = 0;
    }
    // ---- coin tasks of the whole unit, flattened into one list
    uint32_t c[kWinIC], tot = 0;
#pragma unroll
    for (int w = 0; w < kWinIC; ++w) { c[w] = __popcll(live[w]); tot += c[w]; }
#ifdef BPT_HIST
    {  // diagnostic build only: live-colour histogram per level, and per unit the lane totals' sum / max
        const uint32_t lvl = min(a.ctl->level, 15u);
        for (int w = 0; w < kWinIC; ++w)
            if (c[w]) atomicAdd(&g_hist[lvl * 80 + c[w]], 1ull);
        const uint32_t mx = __reduce_max_sync(kFull, tot), sm = __reduce_add_sync(kFull, tot);
        if (lane == 0) {
            atomicAdd(&g_hist[lvl * 80 + 65], (unsigned long long)sm);
            atomicAdd(&g_hist[lvl * 80 + 66], (unsigned long long)mx);
            atomicAdd(&g_hist[lvl * 80 + 67], 1ull);
            atomicAdd(&g_hist[lvl * 80 + 68], (unsigned long long)((sm + 31) / 32));
        }
    }
#endif
    const uint32_t incl = warp_incl_scan_u32(tot, lane);
    const uint32_t ntask = __shfl_sync(kFull, incl, 31);
    uint64_t pass[kWinIC];
#pragma unroll
    for (int w = 0; w < kWinIC; ++w) pass[w] = 0;
    if (ntask) {
#pragma unroll
        for (int w = 0; w < kWinIC; ++w) {
            W.e[w][lane] = t0l + 32u * w + lane + ent[w].x;
            W.thr[w][lane] = rc[w].y;
            W.sbase[w][lane] = (uint32_t)(64ull * (gblk0 + ent[w].y));
            W.pass[w][lane] = 0;
        }
        {
            // search the owner lane and the colour bit of every task
            W.excl[lane] = incl - tot;
            uint32_t cm = 0, run = 0;  // cumulative task counts of windows 0..2 (0xff: no such window)
#pragma unroll
            for (int w = 0; w < 3; ++w) {
                if (w < kWinIC - 1) run += c[w];
                cm |= (w < kWinIC - 1 ? run : 0xffu) << (8 * w);
            }
            W.cum[lane] = cm;
#pragma unroll
            for (int w = 0; w < kWinIC; ++w) W.live[w][lane] = live[w];
            __syncwarp();
            for (uint32_t b = 0; b < ntask; b += 32) {
                const uint32_t k = b + lane;
                if (k < ntask) {
                    uint32_t o = 0;  // owner lane = largest lane with excl <= k
#pragma unroll
                    for (int step = 16; step > 0; step >>= 1)
                        if (W.excl[o + step] <= k) o += step;
                    uint32_t r = k - W.excl[o];
                    const uint32_t cmo = W.cum[o];
                    uint32_t w = 0, base = 0;  // window of the task: last window whose prefix <= r
#pragma unroll
                    for (int q = 0; q < kWinIC - 1; ++q) {
                        const uint32_t pq = (cmo >> (8 * q)) & 0xffu;
                        if (r >= pq) { w = q + 1; base = pq; }
                    }
                    r -= base;
                    coin_task(a, W, o, w, nth_set_bit64(W.live[w][o], r));
                }
            }
        }
        __syncwarp();
#pragma unroll
        for (int w = 0; w < kWinIC; ++w) pass[w] = W.pass[w][lane];
        __syncwarp();
        if (lane == 0) coins += ntask;
    }
    // ---- merges (Listing 1 line 14) of the windows issued together
    unsigned long long old[kWinIC];
#pragma unroll
    for (int w = 0; w < kWinIC; ++w) {
        old[w] = 0;
        if (pass[w]) {
            ++atoms;
            old[w] = atomicOr(&a.VN[vidx[w]].y, pass[w]);
        }
    }
    // ---- first setters -> per-warp buffer (one scan for the whole unit)
    uint32_t nf = 0;
    bool first[kWinIC];
    uint32_t slice[kWinIC];
#pragma unroll
    for (int w = 0; w < kWinIC; ++w) {
        slice[w] = 0;
        first[w] = false;
        if (pass[w]) {
            const uint64_t emask = ((uint64_t)ent[w].w << 32) | ent[w].z;
            if (kC64) {
                first[w] = old[w] == 0;
            } else {
                slice[w] = (uint32_t)(__ffsll((long long)emask) - 1) / a.colors;
                first[w] = (old[w] & slice_mask_of(a.colors, slice[w])) == 0;
            }
            nf += first[w];
        }
    }
    if (!__any_sync(kFull, nf != 0)) return;
    const uint32_t fincl = warp_incl_scan_u32(nf, lane);
    const uint32_t nfirst = __shfl_sync(kFull, fincl, 31);
    uint32_t pos = W.ecount + fincl - nf;
#pragma unroll
    for (int w = 0; w < kWinIC; ++w)
        if (first[w]) W.ebuf[pos++] = raw_pack(rc[w].x, ent[w].y, slice[w]);
    __syncwarp();
    if (lane == 0) W.ecount += nfirst;
    __syncwarp();
    if (W.ecount >= 32) warp_flush(a, Ln, W, lane);
}

#ifndef BPT_EXPAND_MINB
#define BPT_EXPAND_MINB 5
#endif
template <bool kC64, bool kCoh>
__device__ __forceinline__ void expand_ic_body(const BatchArgs& a, const uint32_t* __restrict__ tstart,
                                               cudaGraphConditionalHandle h_level, int use_cond) {
    Ctl* ctl = a.ctl;
    const uint32_t level = LDX(&ctl->level);
    const uint64_t gblk0 = a.slot_sample ? LDX(&ctl->blk0) : LDX(&ctl->gblk0);  // sorted: local slot base
    const LevelRec* L = &a.lv[level];
    LevelRec* Ln = &a.lv[level + 1];
    const unsigned long long packed = LDX(&L->packed);
    const uint64_t nq = packed >> kPackShift;
    const uint64_t total = packed & kEdgeMask;
    const bool idle = nq == 0 || LDX(&L->overflow);
    // blocks without a unit of this level leave at once (thin levels: a few blocks work); the
    // active ones count themselves out, the last advances the level
    const uint32_t active =
        idle ? 1u : (uint32_t)umin64(gridDim.x, umax64(1, (total + (uint64_t)kUnitIC * kWarps - 1) / ((uint64_t)kUnitIC * kWarps)));
    if (blockIdx.x >= active) return;
    if (threadIdx.x == 0) atomicMin(&ctl->t_start, global_ns());
    if (idle) {
        finish_expand(a, h_level, use_cond, active);
        return;
    }
    extern __shared__ __align__(16) unsigned char smem_raw[];
    WarpScratch* scratch = reinterpret_cast<WarpScratch*>(smem_raw);
    __shared__ unsigned long long red[kWarps];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    WarpScratch& W = scratch[wid];
    if (lane == 0) W.ecount = 0;
    __syncwarp();
    const uint32_t le_mask = lane == 31 ? kFull : ((2u << lane) - 1u);
    // 32-bit unit indices: total < 2^36 work items, so units < 2^30
    const uint32_t nunits = (uint32_t)((total + kUnitIC - 1) / kUnitIC);
    const uint32_t nfull = (uint32_t)(total / kUnitIC);
    const uint32_t nwarps = active * kWarps;
    unsigned long long coins = 0, atoms = 0;
    for (uint32_t unit = blockIdx.x * kWarps + wid; unit < nunits; unit += nwarps) {
        const uint32_t jc0 = LDX(&tstart[unit]);
        if (unit < nfull)
            expand_unit_ic<true, kC64, kCoh>(a, Ln, W, lane, le_mask, unit, kUnitIC, jc0, gblk0, coins, atoms);
        else
            expand_unit_ic<false, kC64, kCoh>(a, Ln, W, lane, le_mask, unit, (uint32_t)(total - (uint64_t)unit * kUnitIC),
                                        jc0, gblk0, coins, atoms);
    }
    warp_flush(a, Ln, W, lane);
    unsigned long long ct = block_sum_ull(coins, red);
    if (threadIdx.x == 0 && ct) atomicAdd(&((LevelRec*)L)->coins, ct);
    unsigned long long at = block_sum_ull(atoms, red);
    if (threadIdx.x == 0 && at) atomicAdd(&((LevelRec*)L)->atomics, at);
    finish_expand(a, h_level, use_cond, active);
}

// the first-setter queue form (BPT_FLAG_QUEUE with 64 colours, and every C < 64 run); C < 64 gets
// 64 registers (4 blocks per SM): its slice handling spills at 48
template <bool kC64>
__global__ void __launch_bounds__(kThreads, kC64 ? BPT_EXPAND_MINB : 4) k_expand_ic(BatchArgs a, const uint32_t* __restrict__ tstart,
                                                              cudaGraphConditionalHandle h_level, int use_cond) {
    count_self(a.ctl);
    if (!a.ctl->cont) return;
    expand_ic_body<kC64, false>(a, tstart, h_level, use_cond);
}

// ------------------------------------------------------------------------ IC expansion (product)
// The product's IC expansion (64 colours, touched-bitmap frontier), Listing 1 lines 9-15
// (P:168-174). Work units of kUnitBm = 32 * kWinBm consecutive reverse-edge reads (items) per
// warp, kWinBm windows of 32 lanes; the entry of every item from the unit's first entry (tstart)
// and a popcount of the entry-start bitmap; the windows' loads (entry, {src, thr} record,
// U[u]) issued together; live = mask & ~U[u] with U = V | N the union of the visited colours and
// the colours another edge already merged into u this level (a stale U only skips fewer coins).
// Union layout: the expansion gathers and ORs 8 B per vertex (U: 38.8 MB per block on C2, so it
// stays L2-resident next to the streamed records); the compaction alone reads V.
// Measured at the heavy levels (C2): ~11% of the items carry a live colour, ~7 live colours each.
// So the live items are first compacted (ballot) into a per-warp list, and everything after the
// gather works on that list, one live item per lane: its (item, colour) coin tasks are flattened
// and evaluated 32 at a time (owner lane by a 5-step search of the exclusive task prefix, colour
// by a rank select in the owner's live mask, one 16-byte shared load per task, the Philox key
// schedule read from the kernel parameters), the passing colours OR-merged per item in shared
// memory and then into U[u] by one fire-and-forget OR per item, and u is marked in the touched
// bitmap (the compaction finds the new colours as U & ~V).
#ifndef BPT_WIN_BM
#define BPT_WIN_BM 4
#endif
constexpr int kWinBm = BPT_WIN_BM;   // 32-lane windows per warp work unit (4: measured 4% faster than 3)
constexpr int kUnitBm = 32 * kWinBm;
#ifndef BPT_HEAVY
#define BPT_HEAVY 32
#endif
constexpr int kHeavy = BPT_HEAVY;  // live colours from which an item's coins are drawn warp-wide
#ifndef BPT_PULL_DEFER
#define BPT_PULL_DEFER 4
#endif
constexpr uint32_t kPullDefer = BPT_PULL_DEFER;  // pull: steps whose live items may wait for one coin call
// Batch-wide frontier (a.vmajor): an item's merge target and colour base follow from (u, slot), so B is
// one word u | slot << 30 (n < 2^30) -- 12 KB less shared memory per block, more L1 for the gathers
struct BmScratchV {
    uint4 A[kUnitBm];
    uint32_t B[kUnitBm];
    unsigned long long pass[32];
    uint2 cum[32];
};
struct BmScratch {
    uint4 A[kUnitBm];                       // live items: {edge id, thr, live lo, live hi}
    uint4 B[kUnitBm];                       // live items: {colour-0 sample id, VN index, touched word | ~0, bit}
    unsigned long long pass[32];            // passing colours of the chunk's live items
    uint2 cum[32];                          // byte prefix popcounts of the chunk's live masks
};

// Philox2x32-10 (reading C-1) with the key schedule k + r * W precomputed in the kernel parameters
__device__ __forceinline__ uint32_t philox_ks0(uint32_t x0, uint32_t x1, const uint32_t (&ks)[10]) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint64_t p = (uint64_t)kPhiloxM * (uint64_t)x0;
        const uint32_t hi = (uint32_t)(p >> 32), lo = (uint32_t)p;
        x0 = hi ^ ks[r] ^ x1;
        x1 = lo;
    }
    return x0;
}

// Philox2x32-10 from round 1 on, round 0 done by the caller: h0 = hi(M * x0) ^ ks[0], l0 = lo(M * x0)
// (x0 = the edge id is shared by all colours of an item, x1 = the sample id is not)
__device__ __forceinline__ uint32_t philox_from1(uint32_t h0, uint32_t l0, uint32_t x1, const uint32_t (&ks)[10]) {
    uint32_t x0 = h0 ^ x1;
    x1 = l0;
#pragma unroll
    for (int r = 1; r < 10; ++r) {
        const uint64_t p = (uint64_t)kPhiloxM * (uint64_t)x0;
        const uint32_t hi = (uint32_t)(p >> 32), lo = (uint32_t)p;
        x0 = hi ^ ks[r] ^ x1;
        x1 = lo;
    }
    return x0;
}

// Sample ids of the colours of the batch's slots in shared memory (the coins' counter word):
// sidt[64 slot + bit] = slot_sample[64 (blk0 + slot) + bit] with sorted start vertices, else the
// global id 64 (gblk0 + slot) + bit; nullptr when the batch has more than kSidSlots slots
constexpr uint32_t kSidSlots = 4;  // the product's batch (1 KB of shared memory: more would cut the L1)
__device__ __forceinline__ const uint32_t* fill_sid_table(const BatchArgs& a, uint32_t* sidt, uint64_t gblk0) {
#ifdef BPT_NO_SIDT
    return nullptr;
#endif
    if (a.slots_max > kSidSlots) return nullptr;
    for (uint32_t i = threadIdx.x; i < a.slots_max * 64; i += blockDim.x) {
        const uint64_t li = 64ull * gblk0 + i;
        sidt[i] = a.slot_sample ? (li < a.nlocal ? __ldg(&a.slot_sample[li]) : 0u) : (uint32_t)li;
    }
    return sidt;
}
// colour 0 of item j in the coins' sample numbering: the global id 64 (gblk0 + slot) (sbase = 64 gblk0)
__device__ __forceinline__ uint32_t item_sample0(const BmScratch& W, uint32_t j, uint32_t) { return W.B[j].x; }
__device__ __forceinline__ uint32_t item_sample0(const BmScratchV& W, uint32_t j, uint32_t sbase) {
    return sbase + 64u * (W.B[j] >> 30);
}
// kTable: the table is known to exist (batch-wide frontier: <= 4 slots), no run-time test
template <bool kTable = false>
__device__ __forceinline__ uint32_t coin_sample(const BatchArgs& a, const uint32_t* sidt, uint32_t sbase, uint32_t sid) {
    if (kTable) return sidt[sid - sbase];
    return sidt ? sidt[sid - sbase] : (a.slot_sample ? __ldg(&a.slot_sample[sid]) : sid);
}

// position of the r-th (0-based) set bit of the 64-bit mask hi:lo: the 32-bit half by one popcount,
// the byte by SWAR byte popcounts and their prefix sums (compared with r in all bytes at once), the
// bit inside the byte from a 256-entry table of packed 3-bit positions (shared memory)
__device__ __forceinline__ uint32_t rank_select64(uint32_t lo, uint32_t hi, uint32_t r, const uint32_t* sel8) {
    const uint32_t c = __popc(lo);
    const bool upper = r >= c;
    const uint32_t w = upper ? hi : lo;
    if (upper) r -= c;
    uint32_t t = w - ((w >> 1) & 0x55555555u);
    t = (t & 0x33333333u) + ((t >> 2) & 0x33333333u);
    t = (t + (t >> 4)) & 0x0f0f0f0fu;
    const uint32_t pre = t * 0x01010101u;                             // byte i: set bits in bytes 0..i
    const uint32_t ge = (((r | 0x80u) * 0x01010101u) - pre) & 0x00808080u;  // bytes i < 3 with pre_i <= r
    const uint32_t byte = __popc(ge);
    const uint32_t before = byte ? (pre >> (8 * byte - 8)) & 0xffu : 0u;
    const uint32_t v = (w >> (8 * byte)) & 0xffu;
    return (upper ? 32u : 0u) + 8u * byte + ((sel8[v] >> (3 * (r - before))) & 7u);
}

// byte prefix popcounts of the 64-bit mask hi:lo -- byte i of .x = set bits in bytes 0..i, of .y =
// set bits in bytes 0..4+i -- computed once per live item, then every rank select of its tasks is a
// SIMD byte compare and one table lookup
__device__ __forceinline__ uint2 byte_prefix64(uint32_t lo, uint32_t hi) {
    auto bytes = [](uint32_t w) {
        uint32_t t = w - ((w >> 1) & 0x55555555u);
        t = (t & 0x33333333u) + ((t >> 2) & 0x33333333u);
        return (t + (t >> 4)) & 0x0f0f0f0fu;
    };
    return make_uint2(bytes(lo) * 0x01010101u, bytes(hi) * 0x01010101u + (uint32_t)__popc(lo) * 0x01010101u);
}
__device__ __forceinline__ uint32_t rank_select_cum(uint32_t lo, uint32_t hi, uint2 cum, uint32_t r,
                                                    const uint32_t* sel8) {
    const uint32_t rr = (r | 0x80u) * 0x01010101u;  // r + 128 in every byte (r < 64, prefixes <= 64)
    const uint32_t byte = __popc((rr - cum.x) & 0x80808080u) + __popc((rr - cum.y) & 0x00808080u);
    const uint64_t c64 = ((uint64_t)cum.y << 32) | cum.x;
    const uint32_t before = byte ? (uint32_t)(c64 >> (8 * byte - 8)) & 0xffu : 0u;
    const uint32_t v = (uint32_t)((((uint64_t)hi << 32) | lo) >> (8 * byte)) & 0xffu;
    return 8u * byte + ((sel8[v] >> (3 * (r - before))) & 7u);
}

// Coins and merges of the live items W.A / W.B[0, nlive) of one warp (shared by the push and the
// pull expansion): item = {edge id, thr, live colours lo, hi} / {colour-0 slot index, U index,
// touched word, bit}. One chunk of <= 32 live items at a time (one live item per lane).
// fold (pull): the passing colours of every item are also OR-ed into fold[slot * 32 + owner lane]
// (W.B.w = bit | owner lane << 8 | slot << 16), the owners' per-colour early exit
template <bool kTable = false, class Scr = BmScratch>
__device__ __forceinline__ void bm_coins_and_merge(const BatchArgs& a, Scr& W, const uint32_t* sel8, int lane,
                                                   uint32_t nlive, unsigned long long& coins,
                                                   unsigned long long& atoms, bool& any_pass,
                                                   const uint32_t* sidt, uint32_t sbase,
                                                   unsigned long long* fold = nullptr) {
    const uint32_t le_mask = lane == 31 ? kFull : ((2u << lane) - 1u);
    for (uint32_t c0 = 0; c0 < nlive; c0 += 32) {
        const uint32_t j = c0 + lane;
        const bool has = j < nlive;
        uint32_t cnt = 0;
        uint4 mine = make_uint4(0, 0, 0, 0);
        if (has) {
            mine = W.A[j];
            cnt = __popc(mine.z) + __popc(mine.w);
        }
        // heavy items (>= kHeavy live colours; the sorted groups' hub rows): the whole warp draws
        // the item's coins by bit POSITION -- lanes l and l + 32 -- with no decode at all, and the
        // passing colours come back as two ballots
        const bool heavy = cnt >= (uint32_t)kHeavy;
        unsigned long long hpass = 0;
        for (uint32_t hb = __ballot_sync(kFull, heavy); hb; hb &= hb - 1) {
            const uint32_t hj = __ffs(hb) - 1;
            const uint4 it = W.A[c0 + hj];  // broadcast
            const uint32_t sb = item_sample0(W, c0 + hj, sbase);
            const uint64_t pe = (uint64_t)kPhiloxM * it.x;  // round 0's product: once for the item's 64 coins
            const uint32_t h0 = (uint32_t)(pe >> 32) ^ a.ic_keys[0], l0 = (uint32_t)pe;
            bool p0 = false, p1 = false;
            if (kTable) {  // both coins of every lane, branch-free (the table covers all 64 colours): two
                           // independent Philox chains interleave, and >= half the bits are live anyway
                const uint32_t x0 = philox_from1(h0, l0, coin_sample<kTable>(a, sidt, sbase, sb + lane), a.ic_keys);
                const uint32_t x1 = philox_from1(h0, l0, coin_sample<kTable>(a, sidt, sbase, sb + 32 + lane), a.ic_keys);
                p0 = ((it.z >> lane) & 1u) && (x0 >> 1) < it.y;
                p1 = ((it.w >> lane) & 1u) && (x1 >> 1) < it.y;
            } else {
                if ((it.z >> lane) & 1u)
                    p0 = (philox_from1(h0, l0, coin_sample<kTable>(a, sidt, sbase, sb + lane), a.ic_keys) >> 1) < it.y;
                if ((it.w >> lane) & 1u)
                    p1 = (philox_from1(h0, l0, coin_sample<kTable>(a, sidt, sbase, sb + 32 + lane), a.ic_keys) >> 1) < it.y;
            }
            const uint32_t lo = __ballot_sync(kFull, p0), hi = __ballot_sync(kFull, p1);
            if (lane == (int)hj) hpass = ((unsigned long long)hi << 32) | lo;
        }
        if (has) {
            W.pass[lane] = hpass;
            W.cum[lane] = byte_prefix64(mine.z, mine.w);
        }
        // light items: their (item, colour) tasks flattened, 32 per round; a heavy item keeps one
        // dummy task so the owners' exclusive prefixes stay strictly increasing
        const uint32_t lcnt = heavy ? 1u : cnt;
        const uint32_t incl = warp_incl_scan_u32(lcnt, lane);
        const uint32_t ntask = __shfl_sync(kFull, incl, 31);
        const uint32_t excl = incl - lcnt;
        __syncwarp();
        uint32_t below = 0;  // live lanes whose tasks start before the window (carried from window to window)
        for (uint32_t b = 0; b < ntask; b += 32) {
            // owner of task b + i = (lanes with excl <= b + i) - 1 (every live item has >= 1 task, so the
            // excl of the live lanes strictly increase): the lanes below the window plus the ranges
            // starting inside it (one OR-reduction) -- no search
            const uint32_t d = excl - b;
            const uint32_t starts = __reduce_or_sync(kFull, (has && d < 32u) ? (1u << d) : 0u);
            const uint32_t o = (below + __popc(starts & le_mask) - 1u) & 31u;
            below += __popc(starts);
            const uint32_t eo = __shfl_sync(kFull, excl, o);
            const bool oheavy = __shfl_sync(kFull, heavy, o);
            const uint32_t k = b + lane;
            if (kTable) {  // branch-free: lanes past the last task compute a coin and drop it (bit < 64 always)
                const bool act = k < ntask && !oheavy;
                const uint4 it = W.A[c0 + o];
                const uint32_t bit = rank_select_cum(it.z, it.w, W.cum[o], k - eo, sel8);
                const uint32_t x = philox_ks0(it.x, coin_sample<kTable>(a, sidt, sbase, item_sample0(W, c0 + o, sbase) + bit), a.ic_keys);
                if (act && (x >> 1) < it.y)
                    atomicOr(reinterpret_cast<uint32_t*>(&W.pass[o]) + (bit >> 5), 1u << (bit & 31));
            } else if (k < ntask && !oheavy) {
                const uint4 it = W.A[c0 + o];
                const uint32_t bit = rank_select_cum(it.z, it.w, W.cum[o], k - eo, sel8);
                const uint32_t x = philox_ks0(it.x, coin_sample<kTable>(a, sidt, sbase, item_sample0(W, c0 + o, sbase) + bit), a.ic_keys);
                if ((x >> 1) < it.y)
                    atomicOr(reinterpret_cast<uint32_t*>(&W.pass[o]) + (bit >> 5), 1u << (bit & 31));
            }
        }
        coins += __reduce_add_sync(kFull, cnt) * (lane == 0);
        __syncwarp();
        if (has) {
            const unsigned long long pass = W.pass[lane];
            if (pass) {
                ++atoms;
                if constexpr (std::is_same<Scr, BmScratchV>::value) {
                    const uint32_t bw = W.B[j], u = bw & ((1u << 30) - 1u), sl = bw >> 30;
                    BPT_CHECK(u < a.n && sl < a.slots_max, 7);
                    atomicOr(reinterpret_cast<unsigned long long*>(a.VN) + (size_t)u * a.slots_max + sl, pass);
                    atomicOr(&a.touched[u >> 5], 1u << (u & 31u));
                } else {
                    const uint4 bb = W.B[j];
                    BPT_CHECK(bb.y < a.slots_max * a.n && bb.z < (uint64_t)a.slots_max * a.tiles * 32, 7);
                    atomicOr(reinterpret_cast<unsigned long long*>(a.VN) + bb.y, pass);
                    atomicOr(&a.touched[bb.z], 1u << (bb.w & 31u));
                    if (fold) atomicOr(&fold[((bb.w >> 16) & 3u) * 32 + ((bb.w >> 8) & 31u)], pass);  // several pending items per owner
                }
                any_pass = true;
            }
        }
        __syncwarp();
    }
}

template <bool kWhole>
__device__ __forceinline__ void expand_unit_bm(const BatchArgs& a, BmScratch& W, const uint32_t* sel8, int lane, uint32_t le_mask,
                                               uint32_t unit, uint32_t rem, uint32_t jc0, uint32_t mword,
                                               uint64_t gblk0, unsigned long long& coins,
                                               unsigned long long& atoms, bool& any_pass,
                                               const uint32_t* sidt, uint32_t sbase) {
    const uint32_t t0l = unit * (uint32_t)kUnitBm;  // mod 2^32: edge ids are t + delta (mod 2^32)
    // entry-start words of the unit (prefetched one unit ahead: lane w holds word w)
    uint32_t mw[kWinBm];
#pragma unroll
    for (int w = 0; w < kWinBm; ++w) mw[w] = __shfl_sync(kFull, mword, w);
    if (lane < kWinBm) a.umask[(size_t)unit * kWinBm + lane] = 0;  // cleared for the next level
    mw[0] &= ~1u;  // an entry starting at item 0 is jc0 itself
    uint32_t jl[kWinBm];
    uint32_t before = jc0;
#pragma unroll
    for (int w = 0; w < kWinBm; ++w) {
        jl[w] = before + __popc(mw[w] & le_mask);
        before += __popc(mw[w]);
    }
    uint4 ent[kWinBm];
    uint2 rc[kWinBm];
    BPT_CHECK((uint64_t)unit * kWinBm + kWinBm <= a.umask_words, 1);
#pragma unroll
    for (int w = 0; w < kWinBm; ++w) {
        BPT_CHECK(((kWhole || 32u * w + lane < rem) ? jl[w] : jc0) < a.q_cap, 2);
        ent[w] = __ldg(&a.q[(kWhole || 32u * w + lane < rem) ? jl[w] : jc0]);
    }
#pragma unroll
    for (int w = 0; w < kWinBm; ++w) {
        const uint32_t i = (kWhole || 32u * w + lane < rem) ? 32u * w + lane : 0u;
        BPT_CHECK((uint32_t)(t0l + i + ent[w].x) < a.m, 3);
        BPT_CHECK(ent[w].y < a.slots_max, 4);
        rc[w] = ld_stream(&a.rec[t0l + i + ent[w].x]);
    }
    // ---- gather of U[u] = V[u] | N[u] (union layout), live colours, compacted list of live items
    const uint32_t lt_mask = le_mask >> 1;  // lanes below this one
    const unsigned long long* U = reinterpret_cast<const unsigned long long*>(a.VN);
    uint32_t nlive = 0;
#pragma unroll
    for (int w = 0; w < kWinBm; ++w) {
        const uint32_t vidx = ent[w].y * a.n + rc[w].x;
        BPT_CHECK(rc[w].x < a.n, 5);
        const uint2 uu = ld_keep_u64(&U[vidx]);
        uint32_t lo = ent[w].z & ~uu.x;
        uint32_t hi = ent[w].w & ~uu.y;
        if (!kWhole && 32u * w + lane >= rem) lo = hi = 0;
        const bool lv = (lo | hi) != 0;
        const uint32_t bal = __ballot_sync(kFull, lv);
        if (lv) {
            const uint32_t pos = nlive + __popc(bal & lt_mask);
            BPT_CHECK(pos < (uint32_t)kUnitBm, 6);
            W.A[pos] = make_uint4(t0l + 32u * w + lane + ent[w].x, rc[w].y, lo, hi);
            W.B[pos] = make_uint4((uint32_t)(64ull * (gblk0 + ent[w].y)), vidx,  // colour-0 sample / slot
                                  ent[w].y * a.tiles * 32 + (rc[w].x >> 5), rc[w].x & 31u);
        }
        nlive += __popc(bal);
    }
    if (nlive == 0) return;
    __syncwarp();
    bm_coins_and_merge(a, W, sel8, lane, nlive, coins, atoms, any_pass, sidt, sbase);
}


// Batch-wide frontier (a.vmajor): the same units of kUnitBm work items, but an item is a reverse
// edge of a frontier VERTEX read once for the S slots of the batch: its source's S masks come
// from one 32-B sector (U[u * S .. u * S + S)), each slot with live colours becomes a live item of
// the coin machinery. The items of a unit are flushed to the coins whenever the next slot's ballot
// would overflow the warp's list.
template <bool kWhole>
__device__ __forceinline__ void expand_unit_bmv(const BatchArgs& a, BmScratchV& W, const uint32_t* sel8, int lane,
                                                uint32_t le_mask, uint32_t unit, uint32_t rem, uint32_t jc0,
                                                uint32_t mword, uint64_t gblk0, uint32_t nslots,
                                                unsigned long long& coins, unsigned long long& atoms,
                                                bool& any_pass, const uint32_t* sidt, uint32_t sbase) {
    const uint32_t t0l = unit * (uint32_t)kUnitBm;
    uint32_t mw[kWinBm];
#pragma unroll
    for (int w = 0; w < kWinBm; ++w) mw[w] = __shfl_sync(kFull, mword, w);
    if (lane < kWinBm) a.umask[(size_t)unit * kWinBm + lane] = 0;  // cleared for the next level
    mw[0] &= ~1u;
    uint32_t jl[kWinBm];
    uint32_t before = jc0;
#pragma unroll
    for (int w = 0; w < kWinBm; ++w) {
        jl[w] = before + __popc(mw[w] & le_mask);
        before += __popc(mw[w]);
        if (!(kWhole || 32u * w + lane < rem)) jl[w] = jc0;
    }
    BPT_CHECK((uint64_t)unit * kWinBm + kWinBm <= a.umask_words, 1);
    uint32_t dl[kWinBm];
#pragma unroll
    for (int w = 0; w < kWinBm; ++w) {
        BPT_CHECK(jl[w] < a.q_cap, 2);
        dl[w] = __ldg(&a.qd[jl[w]]);
    }
    uint2 rc[kWinBm];
#pragma unroll
    for (int w = 0; w < kWinBm; ++w) {
        const uint32_t i = (kWhole || 32u * w + lane < rem) ? 32u * w + lane : 0u;
        BPT_CHECK((uint32_t)(t0l + i + dl[w]) < a.m, 3);
        rc[w] = ld_stream(&a.rec[t0l + i + dl[w]]);
    }
    const uint32_t lt_mask = le_mask >> 1;
    const unsigned long long* U = reinterpret_cast<const unsigned long long*>(a.VN);
    const uint32_t S = a.slots_max;
    uint32_t nlive = 0;
#pragma unroll
    for (int w = 0; w < kWinBm; ++w) {
        const bool valid = kWhole || 32u * w + lane < rem;
        const uint32_t u = rc[w].x;
        BPT_CHECK(u < a.n, 5);
        const unsigned long long* qm = a.qmask + (size_t)jl[w] * S;
        const unsigned long long* Uu = U + (size_t)u * S;
        unsigned long long live[4] = {0ull, 0ull, 0ull, 0ull};
        if (valid) {
            if (S == 4) {
                const U4 mm = ld_nc4(qm), uu = ld_cg4(Uu);
                live[0] = mm.x & ~uu.x; live[1] = mm.y & ~uu.y; live[2] = mm.z & ~uu.z; live[3] = mm.w & ~uu.w;
            } else {
#pragma unroll
                for (uint32_t sl = 0; sl < 4; ++sl)
                    if (sl < S) {
                        const unsigned long long m = __ldg(qm + sl);
                        if (m) {
                            const uint2 uu = ld_keep_u64(Uu + sl);
                            live[sl] = m & ~(((unsigned long long)uu.y << 32) | uu.x);
                        }
                    }
            }
        }
        const uint32_t e = t0l + 32u * w + lane + dl[w];
        // live slots of this lane's edge (slots past the batch's own have no colours, so no mask),
        // one warp scan places the window's items
        uint32_t c = 0;
#pragma unroll
        for (uint32_t sl = 0; sl < 4; ++sl) c += ((uint32_t)live[sl] | (uint32_t)(live[sl] >> 32)) != 0u;
        uint32_t incl = c;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t y = __shfl_up_sync(kFull, incl, d);
            if (lane >= d) incl += y;
        }
        const uint32_t wtot = __shfl_sync(kFull, incl, 31);
        if (wtot == 0) continue;
        if (nlive + wtot > (uint32_t)kUnitBm) {  // the list is full: draw its coins first
            __syncwarp();
            bm_coins_and_merge<true>(a, W, sel8, lane, nlive, coins, atoms, any_pass, sidt, sbase);
            __syncwarp();
            nlive = 0;
        }
        uint32_t pos = nlive + incl - c;
#pragma unroll
        for (uint32_t sl = 0; sl < 4; ++sl) {  // unrolled: live[sl] stays in registers
            if (live[sl] != 0ull) {
                W.A[pos] = make_uint4(e, rc[w].y, (uint32_t)live[sl], (uint32_t)(live[sl] >> 32));
                W.B[pos] = u | (sl << 30);
                ++pos;
            }
        }
        nlive += wtot;
    }
    if (nlive == 0) return;
    __syncwarp();
    bm_coins_and_merge<true>(a, W, sel8, lane, nlive, coins, atoms, any_pass, sidt, sbase);
}

#ifndef BPT_BM_MINB
#define BPT_BM_MINB 4  // 64 registers: no spills; 4 x 8 warps per SM (measured: -4% vs 5 blocks at 48)
#endif
template <bool kVmajor>
__global__ void __launch_bounds__(kThreads, BPT_BM_MINB) k_expand_bm(BatchArgs a, const uint32_t* __restrict__ tstart,
                                                              cudaGraphConditionalHandle h_level, int use_cond) {
    count_self(a.ctl);
    if (!a.ctl->cont) return;
    Ctl* ctl = a.ctl;
    const uint32_t level = ctl->level;
    // colour 0 of slot k is sample 64 * (gblk0 + k) -- or, with sorted start vertices, local slot
    // 64 * (blk0 + k), mapped through slot_sample
    const uint64_t gblk0 = a.slot_sample ? ctl->blk0 : ctl->gblk0;
    const uint32_t nslots = ctl->slots;
    const LevelRec* L = &a.lv[level];
    LevelRec* Ln = &a.lv[level + 1];
    if (pull_level(a, L)) return;  // k_expand_pull expands this level
    const unsigned long long packed = L->packed;
    const uint64_t nq = packed >> kPackShift;
    const uint64_t total = packed & kEdgeMask;
    const bool idle = nq == 0 || L->overflow;
    const uint32_t active =
        idle ? 1u : (uint32_t)umin64(gridDim.x, umax64(1, (total + (uint64_t)kUnitBm * kWarps - 1) / ((uint64_t)kUnitBm * kWarps)));
    if (blockIdx.x >= active) return;
    if (threadIdx.x == 0) atomicMin(&ctl->t_start, global_ns());
    if (idle) {
        finish_expand(a, h_level, use_cond, active);
        return;
    }
    extern __shared__ __align__(16) unsigned char smem_raw[];
    using Scr = std::conditional_t<kVmajor, BmScratchV, BmScratch>;
    Scr& W = reinterpret_cast<Scr*>(smem_raw)[threadIdx.x >> 5];
    __shared__ unsigned long long red[kWarps];
    __shared__ uint32_t sel8[256];  // bit positions of every byte value, 3 bits each (rank_select64)
    __shared__ uint32_t sid_sh[kSidSlots * 64];
    {
        uint32_t t = 0;
        for (uint32_t p = 0, j = 0; p < 8; ++p)
            if ((threadIdx.x >> p) & 1u) t |= p << (3 * j++);
        sel8[threadIdx.x] = t;
    }
    const uint32_t* sidt = fill_sid_table(a, sid_sh, gblk0);
    const uint32_t sbase = (uint32_t)(64ull * gblk0);
    __syncthreads();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const uint32_t le_mask = lane == 31 ? kFull : ((2u << lane) - 1u);
    const uint32_t nunits = (uint32_t)((total + kUnitBm - 1) / kUnitBm);
    const uint32_t nfull = (uint32_t)(total / kUnitBm);
    const uint32_t nwarps = active * kWarps;
    unsigned long long coins = 0, atoms = 0;
    bool any_pass = false;
    // the unit's first entry and entry-start words are loaded one unit ahead (one fewer dependent
    // round trip per unit)
    uint32_t unit = blockIdx.x * kWarps + wid;
    uint32_t nx_t = 0, nx_m = 0;
    if (unit < nunits) {
        nx_t = __ldg(&tstart[unit]);
        nx_m = lane < kWinBm ? a.umask[(size_t)unit * kWinBm + lane] : 0u;
    }
    for (; unit < nunits; unit += nwarps) {
        const uint32_t jc0 = nx_t, mword = nx_m;
        BPT_CHECK(unit < a.tstart_cap, 8);
        const uint32_t nxt = unit + nwarps;
        if (nxt < nunits) {
            nx_t = __ldg(&tstart[nxt]);
            nx_m = lane < kWinBm ? a.umask[(size_t)nxt * kWinBm + lane] : 0u;
        }
        if constexpr (kVmajor) {
            if (unit < nfull)
                expand_unit_bmv<true>(a, W, sel8, lane, le_mask, unit, kUnitBm, jc0, mword, gblk0, nslots, coins, atoms,
                                      any_pass, sidt, sbase);
            else
                expand_unit_bmv<false>(a, W, sel8, lane, le_mask, unit, (uint32_t)(total - (uint64_t)unit * kUnitBm), jc0,
                                       mword, gblk0, nslots, coins, atoms, any_pass, sidt, sbase);
        } else if (unit < nfull) {
            expand_unit_bm<true>(a, W, sel8, lane, le_mask, unit, kUnitBm, jc0, mword, gblk0, coins, atoms, any_pass, sidt,
                                 sbase);
        } else {
            expand_unit_bm<false>(a, W, sel8, lane, le_mask, unit, (uint32_t)(total - (uint64_t)unit * kUnitBm), jc0, mword,
                                  gblk0, coins, atoms, any_pass, sidt, sbase);
        }
    }
    if (__any_sync(kFull, any_pass) && lane == 0) Ln->any = 1;
    unsigned long long ct = block_sum_ull(coins, red);
    if (threadIdx.x == 0 && ct) atomicAdd(&((LevelRec*)L)->coins, ct);
    unsigned long long at = block_sum_ull(atoms, red);
    if (threadIdx.x == 0 && at) atomicAdd(&((LevelRec*)L)->atomics, at);
    finish_expand(a, h_level, use_cond, active);
}


// ------------------------------------------------------------------------ pull expansion (IC)
// SURVEY §8(f) NEXT #1 (direction switching): a level whose push work (the
// frontier's reverse-edge reads, summed over the batch's slots) is >= pull_min_work is expanded
// the other way round, over the forward edges u -> w (Graph::pull_rec {u, w, e, thr}, grouped by
// u): for every vertex u and slot, the colours u does not hold yet are pulled from its frontier
// out-neighbours -- live = F[w][slot] & ~known[slot], F the frontier masks the compaction keeps
// exact (vertex-major: one 32-B sector serves the 4 slots of a batch) -- with the coin of the
// edge's canonical reverse id e (reading C-4), so the RRR sets are those of the push form.
// One lane walks one row segment (<= kPullSeg edges, Graph::pull_seg, longest first so a warp's
// segments have ~equal lengths) edge by edge, and a colour leaves its known mask as soon as one
// coin passes: per-colour early exit, which the push form only gets from the timing of its
// merges. Coins and merges go through the push form's machinery (bm_coins_and_merge); the
// passing colours also come back to the owner lane (fold). Every forward edge is read once per
// pull level for all slots (m per batch level; the push form reads ~3.5 m at C2's heavy levels).
__global__ void __launch_bounds__(kThreads, BPT_BM_MINB) k_expand_pull(BatchArgs a, cudaGraphConditionalHandle h_level,
                                                                int use_cond) {
    count_self(a.ctl);
    if (!a.ctl->cont) return;
    Ctl* ctl = a.ctl;
    const uint32_t level = ctl->level;
    LevelRec* L = &a.lv[level];
    LevelRec* Ln = &a.lv[level + 1];
    if (!pull_level(a, L)) return;  // k_expand_bm expands this level
    if (threadIdx.x == 0) atomicMin(&ctl->t_start, global_ns());
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        L->pull = 1;
        L->pull_reads = a.pull_edges;
    }
    const uint64_t gblk0 = a.slot_sample ? ctl->blk0 : ctl->gblk0;
    const uint32_t nslots = ctl->slots;
    {   // the compaction marked the entry starts of this level's push units; the push kernel, which
        // clears them as it reads them, does not run on a pull level
        const uint64_t words = umin64(((L->packed & kEdgeMask) + 31) / 32 + kWinBm, a.umask_words);
        for (uint64_t i = blockIdx.x * (uint64_t)kThreads + threadIdx.x; i < words; i += (uint64_t)gridDim.x * kThreads)
            a.umask[i] = 0;
    }
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    BmScratch& W = reinterpret_cast<BmScratch*>(smem_raw)[wid];
    __shared__ unsigned long long red[kWarps];
    __shared__ uint32_t sel8[256];
    __shared__ unsigned long long fold_all[kWarps][4 * 32];
    unsigned long long* fold = fold_all[wid];
    {
        uint32_t t = 0;
        for (uint32_t p = 0, j = 0; p < 8; ++p)
            if ((threadIdx.x >> p) & 1u) t |= p << (3 * j++);
        sel8[threadIdx.x] = t;
    }
    for (int i = lane; i < 4 * 32; i += 32) fold[i] = 0ull;
    __shared__ uint32_t sid_sh[kSidSlots * 64];
    const uint32_t* sidt = fill_sid_table(a, sid_sh, gblk0);
    const uint32_t sbase = (uint32_t)(64ull * gblk0);
    __syncthreads();
    const uint32_t lt_mask = (1u << lane) - 1u;
    const unsigned long long* U = reinterpret_cast<const unsigned long long*>(a.VN);
    unsigned long long coins = 0, atoms = 0;
    bool any_pass = false;
    const uint64_t ngroups = (a.pull_nseg + 31) / 32;
    for (uint64_t grp = (uint64_t)blockIdx.x * kWarps + wid; grp < ngroups; grp += (uint64_t)gridDim.x * kWarps) {
        const uint64_t i = grp * 32 + lane;
        const uint4 sg = i < a.pull_nseg ? __ldg(&a.pull_seg[i]) : make_uint4(0, 0, 0, 0);
        const uint32_t u = sg.x, end = sg.y + sg.z;
        uint32_t ptr = sg.y;
        const uint32_t steps = __shfl_sync(kFull, sg.z, 0);  // longest first: lane 0 holds the group's maximum
        BPT_CHECK(sg.z == 0 || (u < a.n && end <= a.m), 13);
        unsigned long long known[4];
#pragma unroll
        for (uint32_t sl = 0; sl < 4; ++sl) {
            known[sl] = ~0ull;
            if (sl < nslots && sg.z) {
                const uint2 uu = ld_keep_u64(&U[sl * a.n + u]);
                known[sl] = ((unsigned long long)uu.y << 32) | uu.x;
            }
        }
        // software pipeline: the record of edge k + 2 and the frontier masks of edge k + 1 are in
        // flight while edge k's coins are drawn (a step is otherwise a chain of two dependent loads)
        auto load_f = [&](const uint4& rr, bool on, unsigned long long (&ff)[4]) {
            ff[0] = ff[1] = ff[2] = ff[3] = 0ull;
            if (!on) return;
            const unsigned long long* Fw = a.F + (size_t)rr.y * a.slots_max;
            if (a.slots_max == 4) {
                const ulonglong2 f01 = ld_keep(reinterpret_cast<const ulonglong2*>(Fw));
                const ulonglong2 f23 = ld_keep(reinterpret_cast<const ulonglong2*>(Fw) + 1);
                ff[0] = f01.x; ff[1] = f01.y; ff[2] = f23.x; ff[3] = f23.y;
            } else {
#pragma unroll
                for (uint32_t sl = 0; sl < 4; ++sl) ff[sl] = sl < nslots ? __ldg(Fw + sl) : 0ull;
            }
        };
        uint32_t nlive = 0, deferred = 0;  // pending live items, steps since the last coin call
        auto flush = [&]() {
            __syncwarp();
            bm_coins_and_merge(a, W, sel8, lane, nlive, coins, atoms, any_pass, sidt, sbase, fold);
            __syncwarp();
#pragma unroll
            for (uint32_t sl = 0; sl < 4; ++sl) {  // early exit: the colours this lane's u just got
                if (sl >= nslots) break;
                known[sl] |= fold[sl * 32 + lane];
                fold[sl * 32 + lane] = 0ull;
            }
            __syncwarp();
            nlive = 0;
            deferred = 0;
        };
        uint4 r1 = ptr < end ? __ldg(&a.pull[ptr]) : make_uint4(0, 0, 0, 0);          // edge k + 1 (k = -1)
        uint4 r2 = ptr + 1 < end ? __ldg(&a.pull[ptr + 1]) : make_uint4(0, 0, 0, 0);  // edge k + 2
        unsigned long long fn[4];
        load_f(r1, ptr < end, fn);
        for (uint32_t k = 0; k < steps; ++k) {
            const uint32_t e_k = r1.z, thr_k = r1.w;
            unsigned long long f[4] = {fn[0], fn[1], fn[2], fn[3]};
            ++ptr;  // now the index of edge k + 1
            r1 = r2;
            if (ptr + 1 < end) r2 = __ldg(&a.pull[ptr + 1]);
            load_f(r1, ptr < end, fn);
            // live (edge, slot) items of this step; they join the warp's pending list, whose coins are
            // drawn once it would overflow (or after kPullDefer steps): the coin machinery has a fixed
            // cost per call, and a step of 32 edges carries few coins at most pull levels
#pragma unroll
            for (uint32_t sl = 0; sl < 4; ++sl) f[sl] &= ~known[sl];
            uint32_t cnt = 0;
#pragma unroll
            for (uint32_t sl = 0; sl < 4; ++sl) cnt += __popc(__ballot_sync(kFull, sl < nslots && f[sl] != 0ull));
            if (nlive && (nlive + cnt > (uint32_t)kUnitBm || deferred >= kPullDefer)) {
                flush();
#pragma unroll
                for (uint32_t sl = 0; sl < 4; ++sl) f[sl] &= ~known[sl];  // colours the flush just delivered
            }
#pragma unroll
            for (uint32_t sl = 0; sl < 4; ++sl) {
                if (sl >= nslots) break;
                const bool lv = f[sl] != 0ull;
                const uint32_t bal = __ballot_sync(kFull, lv);
                if (lv) {
                    const uint32_t pos = nlive + __popc(bal & lt_mask);
                    W.A[pos] = make_uint4(e_k, thr_k, (uint32_t)f[sl], (uint32_t)(f[sl] >> 32));
                    W.B[pos] = make_uint4((uint32_t)(64ull * (gblk0 + sl)), sl * a.n + u, sl * a.tiles * 32 + (u >> 5),
                                          (u & 31u) | ((uint32_t)lane << 8) | (sl << 16));
                }
                nlive += __popc(bal);
            }
            deferred += nlive != 0;
        }
        if (nlive) flush();
    }
    if (__any_sync(kFull, any_pass) && lane == 0) Ln->any = 1;
    unsigned long long ct = block_sum_ull(coins, red);
    if (threadIdx.x == 0 && ct) atomicAdd(&L->coins, ct);
    unsigned long long at = block_sum_ull(atoms, red);
    if (threadIdx.x == 0 && at) atomicAdd(&L->atomics, at);
    finish_expand(a, h_level, use_cond, gridDim.x);
}

// ------------------------------------------------------------------------ wide fusion (IC)
// the kWide = 2 blocks of a batch (128 colours) share one
// frontier. A frontier entry is a vertex with kWide masks; each reverse edge of it is read once
// for all 128 colours, and the working masks are vertex-major, so {V, N}[u] of both blocks is
// one 32-B sector. Measured with the oracle (C2 shape): 1.79x fewer edge reads per sample
// than 64-colour groups. Same coins (keyed by the global sample id), hence the same RRR sets.
constexpr int kWinW = (int)kUnitWide / 32;   // edge windows per unit
constexpr int kVW = kWinW * (int)kWide;      // virtual windows (edge window, block)
static_assert(kVW <= 8 && kWide % 2 == 0, "task prefixes of kVW - 1 virtual windows must fit the cum word");
// per-lane task prefixes of virtual windows 0..kVW-2: 8-bit fields of a u32 (<= 3 x 64) or
// 9-bit fields of a u64 (<= 7 x 64)
using CumW = std::conditional_t<(kVW <= 4), uint32_t, unsigned long long>;
constexpr int kCumBits = kVW <= 4 ? 8 : 9;

__global__ void k_init_w(BatchArgs a, cudaGraphConditionalHandle h_level, int use_cond) {
    count_self(a.ctl);
    const uint64_t total = (uint64_t)a.ctl->slots * 64;
    const uint64_t gblk0 = a.ctl->gblk0;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        a.ctl->cont = 1;
        a.ctl->level = 0;
        if (use_cond) cudaGraphSetConditional(h_level, 1);
    }
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t b = (uint32_t)(i >> 6), bit = (uint32_t)(i & 63);
        const uint64_t s = 64ull * (gblk0 + b) + bit;
        if (s >= a.theta) continue;
        const uint2 w = philox2x32_10((uint32_t)s, (uint32_t)(s >> 32), a.k_start);
        const uint64_t r64 = ((uint64_t)w.y << 32) | w.x;
        const uint32_t start = (uint32_t)__umul64hi(r64, (uint64_t)a.n);
        BPT_CHECK(start < a.n, 11);
        const unsigned long long old = atomicOr(&a.VN[(size_t)start * kWide + b].y, 1ull << bit);
        if (old == 0 && atomicOr(&a.vflag[start], 1u) == 0) {
            const unsigned pos = atomicAdd(&a.lv[0].raw, 1u);
            if (pos < a.raw_cap) a.raw[pos] = start;
            else a.lv[0].overflow = 1;
        }
    }
}

// A4 for wide entries: for each queued vertex v: masks m_b = N_b; V_b |= N_b; N_b = 0; vflag = 0.
__global__ void __launch_bounds__(kThreads, 5) k_compact_w(BatchArgs a, uint32_t* __restrict__ tstart,
                                                        uint64_t tstart_cap) {
    count_self(a.ctl);
    if (!a.ctl->cont) return;
    LevelRec* L = &a.lv[a.ctl->level];
    const uint64_t nraw = umin64(L->raw, a.raw_cap);
    if (blockIdx.x > 0 && (uint64_t)blockIdx.x * kCompTile >= nraw) return;  // no tile of this level
    if (threadIdx.x == 0) atomicMin(&a.ctl->c_start, global_ns());
    constexpr uint32_t unit = kUnitWide;
    __shared__ unsigned long long wsum[kWarps];
    __shared__ uint32_t wcnt[kWarps];
    __shared__ unsigned long long blk_base;
    __shared__ unsigned long long vc_acc[kWarps];
    constexpr uint32_t kBig = 64;
    __shared__ unsigned long long big_u0[kBig], big_u1[kBig];
    __shared__ uint32_t big_q[kBig];
    __shared__ uint32_t big_n;
    if (threadIdx.x == 0) big_n = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    unsigned long long vc_local = 0;
    for (uint64_t tile0 = (uint64_t)blockIdx.x * kCompTile; tile0 < nraw; tile0 += (uint64_t)gridDim.x * kCompTile) {
        uint32_t vv[kCompItems];
#pragma unroll
        for (int it = 0; it < kCompItems; ++it) {
            const uint64_t i = tile0 + (uint64_t)it * kThreads + threadIdx.x;
            vv[it] = i < nraw ? (uint32_t)a.raw[i] : ~0u;
        }
        uint64_t mask[kCompItems][kWide];
        uint32_t rs[kCompItems], re[kCompItems];
#pragma unroll
        for (int it = 0; it < kCompItems; ++it) {
            rs[it] = re[it] = 0;
#pragma unroll
            for (uint32_t b = 0; b < kWide; ++b) mask[it][b] = 0;
            if (vv[it] != ~0u) {
                const uint32_t v = vv[it];
                ulonglong2* p = &a.VN[(size_t)v * kWide];
#pragma unroll
                for (uint32_t b = 0; b < kWide; ++b) {
                    const ulonglong2 x = p[b];
                    mask[it][b] = x.y;
                    if (x.y) p[b] = make_ulonglong2(x.x | x.y, 0ull);
                }
                a.vflag[v] = 0;
                rs[it] = __ldg(&a.roff[v]);
                re[it] = __ldg(&a.roff[v + 1]);
            }
        }
        uint32_t cnt = 0;
        unsigned long long work_t = 0;
        uint64_t work[kCompItems];
#pragma unroll
        for (int it = 0; it < kCompItems; ++it) {
            uint64_t any = 0;
#pragma unroll
            for (uint32_t b = 0; b < kWide; ++b) { vc_local += __popcll(mask[it][b]); any |= mask[it][b]; }
            work[it] = any ? re[it] - rs[it] : 0;
            cnt += work[it] != 0;
            work_t += work[it];
        }
        uint32_t cincl = cnt;
        unsigned long long wincl = work_t;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t yc = __shfl_up_sync(kFull, cincl, d);
            const unsigned long long yw = __shfl_up_sync(kFull, wincl, d);
            if (lane >= d) { cincl += yc; wincl += yw; }
        }
        if (lane == 31) { wsum[wid] = wincl; wcnt[wid] = cincl; }
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned long long ts = 0;
            uint32_t tc = 0;
            for (int w = 0; w < kWarps; ++w) {
                const unsigned long long s2 = wsum[w];
                const uint32_t c2 = wcnt[w];
                wsum[w] = ts; wcnt[w] = tc; ts += s2; tc += c2;
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
        if (bb != ~0ull && cnt) {
            uint64_t qi = (bb >> kPackShift) + wcnt[wid] + cincl - cnt;
            uint64_t off = (bb & kEdgeMask) + wsum[wid] + wincl - work_t;
            uint64_t mword = ~0ull;
            uint32_t mbits = 0;
#pragma unroll
            for (int it = 0; it < kCompItems; ++it) {
                if (!work[it]) continue;
                a.qd[qi] = rs[it] - (uint32_t)off;
#pragma unroll
                for (uint32_t b = 0; b < kWide; ++b) a.qmask[qi * kWide + b] = mask[it][b];
                if (off / unit < tstart_cap) {
                    if ((off >> 5) != mword) {
                        if (mbits) atomicOr(&a.umask[mword], mbits);
                        mword = off >> 5;
                        mbits = 0;
                    }
                    mbits |= 1u << (off & 31u);
                }
                const uint64_t u0 = (off + unit - 1) / unit, u1 = (off + work[it] + unit - 1) / unit;
                if (u1 > tstart_cap) L->overflow = 1;
                const uint64_t u1c = umin64(u1, tstart_cap);
                if (u1c > u0 + 4) {
                    const uint32_t bi = atomicAdd(&big_n, 1u);
                    if (bi < kBig) {
                        big_u0[bi] = u0;
                        big_u1[bi] = u1c;
                        big_q[bi] = (uint32_t)qi;
                    } else {
                        for (uint64_t t = u0; t < u1c; ++t) tstart[t] = (uint32_t)qi;
                    }
                } else {
                    for (uint64_t t = u0; t < u1c; ++t) tstart[t] = (uint32_t)qi;
                }
                ++qi;
                off += work[it];
            }
            if (mbits) atomicOr(&a.umask[mword], mbits);
        }
        __syncthreads();
        const uint32_t nbig = min(big_n, (uint32_t)kBig);
        for (uint32_t bi = 0; bi < nbig; ++bi)
            for (uint64_t t = big_u0[bi] + threadIdx.x; t < big_u1[bi]; t += kThreads) tstart[t] = big_q[bi];
        __syncthreads();
        if (threadIdx.x == 0) big_n = 0;
    }
    unsigned long long vc_tot = block_sum_ull(vc_local, vc_acc);
    if (threadIdx.x == 0 && vc_tot) atomicAdd(&L->vc, vc_tot);
    if (threadIdx.x == 0) atomicMax(&a.ctl->c_end, global_ns());
}

struct WarpScratchW {
    uint32_t excl[32];
    CumW cum[32];                          // field q: tasks of virtual windows 0..q (q < kVW - 1)
    unsigned long long live[kVW][32];
    uint32_t e[kWinW][32];
    uint32_t thr[kWinW][32];
    unsigned long long pass[kVW][32];      // 32-bit halves: native ATOMS.OR
    unsigned long long ebuf[32 + kUnitWide];
    uint32_t ecount;
};

__device__ __forceinline__ void warp_flush_w(const BatchArgs& a, LevelRec* Ln, WarpScratchW& W, int lane) {
    const uint32_t cnt = W.ecount;
    if (cnt == 0) return;
    unsigned base = 0;
    if (lane == 0) base = atomicAdd(&Ln->raw, cnt);
    base = __shfl_sync(kFull, base, 0);
    for (uint32_t i = lane; i < cnt; i += 32) {
        const uint64_t pos = (uint64_t)base + i;
        if (pos < a.raw_cap) a.raw[pos] = W.ebuf[i];
        else Ln->overflow = 1;
    }
    __syncwarp();
    if (lane == 0) W.ecount = 0;
    __syncwarp();
}

template <bool kWhole>
__device__ __forceinline__ void expand_unit_w(const BatchArgs& a, LevelRec* Ln, WarpScratchW& W, int lane,
                                              uint32_t le_mask, uint32_t unit, uint32_t rem, uint32_t jc0,
                                              uint32_t sb0, unsigned long long& coins, unsigned long long& atoms) {
    const uint32_t t0l = unit * kUnitWide;
    uint32_t mw[kWinW];
#pragma unroll
    for (int w = 0; w < kWinW; ++w) mw[w] = a.umask[(size_t)unit * kWinW + w];
    __syncwarp();
    if (lane < kWinW) a.umask[(size_t)unit * kWinW + lane] = 0;
    mw[0] &= ~1u;
    uint32_t jl[kWinW];
    uint32_t before = jc0;
#pragma unroll
    for (int w = 0; w < kWinW; ++w) {
        jl[w] = before + __popc(mw[w] & le_mask);
        before += __popc(mw[w]);
        if (!kWhole && 32u * w + lane >= rem) jl[w] = jc0;
    }
    uint32_t d[kWinW];
    uint2 rc[kWinW];
    uint64_t live[kVW];
    if constexpr (kWide == 2) {
        ulonglong2 M[kWinW];  // {mask of block 0, mask of block 1}
#pragma unroll
        for (int w = 0; w < kWinW; ++w) {
            d[w] = a.qd[jl[w]];
            M[w] = reinterpret_cast<const ulonglong2*>(a.qmask)[jl[w]];
        }
#pragma unroll
        for (int w = 0; w < kWinW; ++w) {
            const uint32_t i = (kWhole || 32u * w + lane < rem) ? 32u * w + lane : 0u;
            rc[w] = ld_stream(&a.rec[t0l + i + d[w]]);
        }
#pragma unroll
        for (int w = 0; w < kWinW; ++w) {
            const ulonglong2* p = &a.VN[(size_t)rc[w].x * kWide];
            const ulonglong2 v0 = ld_keep(p), v1 = ld_keep(p + 1);
            live[w * kWide + 0] = M[w].x & ~(v0.x | v0.y);
            live[w * kWide + 1] = M[w].y & ~(v1.x | v1.y);
            if (!kWhole && 32u * w + lane >= rem) live[w * kWide + 0] = live[w * kWide + 1] = 0;
        }
    } else {
        uint64_t M[kWinW][kWide];  // the entry's mask per block
#pragma unroll
        for (int w = 0; w < kWinW; ++w) {
            d[w] = a.qd[jl[w]];
            const ulonglong2* mp = reinterpret_cast<const ulonglong2*>(a.qmask + (size_t)jl[w] * kWide);
#pragma unroll
            for (uint32_t b = 0; b < kWide; b += 2) {
                const ulonglong2 x = mp[b / 2];
                M[w][b] = x.x;
                M[w][b + 1] = x.y;
            }
        }
#pragma unroll
        for (int w = 0; w < kWinW; ++w) {
            const uint32_t i = (kWhole || 32u * w + lane < rem) ? 32u * w + lane : 0u;
            rc[w] = ld_stream(&a.rec[t0l + i + d[w]]);
        }
#pragma unroll
        for (int w = 0; w < kWinW; ++w) {
            const ulonglong2* p = &a.VN[(size_t)rc[w].x * kWide];
#pragma unroll
            for (uint32_t b = 0; b < kWide; ++b) {
                const ulonglong2 vn = ld_keep(p + b);
                live[w * kWide + b] = (!kWhole && 32u * w + lane >= rem) ? 0ull : M[w][b] & ~(vn.x | vn.y);
            }
        }
    }
    uint32_t c[kVW], tot = 0;
#pragma unroll
    for (int q = 0; q < kVW; ++q) { c[q] = __popcll(live[q]); tot += c[q]; }
    const uint32_t incl = warp_incl_scan_u32(tot, lane);
    const uint32_t ntask = __shfl_sync(kFull, incl, 31);
    uint64_t pass[kVW];
#pragma unroll
    for (int q = 0; q < kVW; ++q) pass[q] = 0;
    if (ntask) {
#pragma unroll
        for (int w = 0; w < kWinW; ++w) {
            W.e[w][lane] = t0l + 32u * w + lane + d[w];
            W.thr[w][lane] = rc[w].y;
        }
#pragma unroll
        for (int q = 0; q < kVW; ++q) { W.pass[q][lane] = 0; W.live[q][lane] = live[q]; }
        W.excl[lane] = incl - tot;
        CumW cm = 0;
        uint32_t run = 0;
#pragma unroll
        for (int q = 0; q < kVW - 1; ++q) { run += c[q]; cm |= (CumW)run << (kCumBits * q); }
        W.cum[lane] = cm;
        __syncwarp();
        for (uint32_t b = 0; b < ntask; b += 32) {
            const uint32_t k = b + lane;
            if (k < ntask) {
                uint32_t o = 0;
#pragma unroll
                for (int step = 16; step > 0; step >>= 1)
                    if (W.excl[o + step] <= k) o += step;
                uint32_t r = k - W.excl[o];
                const CumW cmo = W.cum[o];
                uint32_t q = 0, base = 0;
#pragma unroll
                for (int qq = 0; qq < kVW - 1; ++qq) {
                    const uint32_t pq = (uint32_t)(cmo >> (kCumBits * qq)) & ((1u << kCumBits) - 1u);
                    if (r >= pq) { q = qq + 1; base = pq; }
                }
                r -= base;
                const uint32_t bit = nth_set_bit64(W.live[q][o], r);
                const uint32_t w = q / kWide, blk = q % kWide;
                const uint32_t x = philox2x32_10(W.e[w][o], sb0 + 64u * blk + bit, a.k_ic).x;
                if ((x >> 1) < W.thr[w][o])
                    atomicOr(reinterpret_cast<uint32_t*>(&W.pass[q][o]) + (bit >> 5), 1u << (bit & 31));
            }
        }
        __syncwarp();
#pragma unroll
        for (int q = 0; q < kVW; ++q) pass[q] = W.pass[q][lane];
        __syncwarp();
        if (lane == 0) coins += ntask;
    }
    // merges; a vertex is queued once per level (vflag) by the first setter of any of its words
    unsigned long long old[kVW];
#pragma unroll
    for (int q = 0; q < kVW; ++q) {
        old[q] = ~0ull;
        if (pass[q]) {
            ++atoms;
            old[q] = atomicOr(&a.VN[(size_t)rc[q / kWide].x * kWide + (q % kWide)].y, pass[q]);
        }
    }
    uint32_t nf = 0;
    bool first[kWinW];
#pragma unroll
    for (int w = 0; w < kWinW; ++w) {
        first[w] = false;
        bool fw;
        if constexpr (kWide == 2) {
            fw = old[w * kWide] == 0 || old[w * kWide + 1] == 0;
        } else {
            fw = false;
#pragma unroll
            for (uint32_t b = 0; b < kWide; ++b) fw |= old[w * kWide + b] == 0;
        }
        if (fw && atomicOr(&a.vflag[rc[w].x], 1u) == 0) first[w] = true;
        nf += first[w];
    }
    if (!__any_sync(kFull, nf != 0)) return;
    const uint32_t fincl = warp_incl_scan_u32(nf, lane);
    const uint32_t nfirst = __shfl_sync(kFull, fincl, 31);
    uint32_t pos = W.ecount + fincl - nf;
#pragma unroll
    for (int w = 0; w < kWinW; ++w)
        if (first[w]) W.ebuf[pos++] = rc[w].x;
    __syncwarp();
    if (lane == 0) W.ecount += nfirst;
    __syncwarp();
    if (W.ecount >= 32) warp_flush_w(a, Ln, W, lane);
}

__global__ void __launch_bounds__(kThreads, BPT_EXPAND_MINB) k_expand_w(BatchArgs a, const uint32_t* __restrict__ tstart,
                                                             cudaGraphConditionalHandle h_level, int use_cond) {
    Ctl* ctl = a.ctl;
    count_self(ctl);
    if (!ctl->cont) return;
    const uint32_t level = ctl->level;
    const uint64_t gblk0 = ctl->gblk0;
    const LevelRec* L = &a.lv[level];
    LevelRec* Ln = &a.lv[level + 1];
    const unsigned long long packed = L->packed;
    const uint64_t nq = packed >> kPackShift;
    const uint64_t total = packed & kEdgeMask;
    const bool idle = nq == 0 || L->overflow;
    const uint32_t active =  // blocks with work; the others leave at once
        idle ? 1u : (uint32_t)umin64(gridDim.x, umax64(1, (total + (uint64_t)kUnitWide * kWarps - 1) /
                                                             ((uint64_t)kUnitWide * kWarps)));
    if (blockIdx.x >= active) return;
    if (threadIdx.x == 0) atomicMin(&ctl->t_start, global_ns());
    if (idle) {
        finish_expand(a, h_level, use_cond, active);
        return;
    }
    extern __shared__ __align__(16) unsigned char smem_raw[];
    WarpScratchW* scratch = reinterpret_cast<WarpScratchW*>(smem_raw);
    __shared__ unsigned long long red[kWarps];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    WarpScratchW& W = scratch[wid];
    if (lane == 0) W.ecount = 0;
    __syncwarp();
    const uint32_t le_mask = lane == 31 ? kFull : ((2u << lane) - 1u);
    const uint32_t nunits = (uint32_t)((total + kUnitWide - 1) / kUnitWide);
    const uint32_t nfull = (uint32_t)(total / kUnitWide);
    const uint32_t sb0 = (uint32_t)(64ull * gblk0);
    unsigned long long coins = 0, atoms = 0;
    for (uint32_t unit = blockIdx.x * kWarps + wid; unit < nunits; unit += active * kWarps) {
        const uint32_t jc0 = tstart[unit];
        if (unit < nfull)
            expand_unit_w<true>(a, Ln, W, lane, le_mask, unit, kUnitWide, jc0, sb0, coins, atoms);
        else
            expand_unit_w<false>(a, Ln, W, lane, le_mask, unit, (uint32_t)(total - (uint64_t)unit * kUnitWide), jc0,
                                 sb0, coins, atoms);
    }
    warp_flush_w(a, Ln, W, lane);
    unsigned long long ct = block_sum_ull(coins, red);
    if (threadIdx.x == 0 && ct) atomicAdd(&((LevelRec*)L)->coins, ct);
    unsigned long long at = block_sum_ull(atoms, red);
    if (threadIdx.x == 0 && at) atomicAdd(&((LevelRec*)L)->atomics, at);
    finish_expand(a, h_level, use_cond, active);
}

// ------------------------------------------------------------------------ LT reverse walks
// Under LT (reading C-6) an RRR set is a single reverse walk: each sample is at ONE vertex per
// level, so the 64 colours of a block never share an edge read (E_phys = E_logical = sum |RR|,
// fusion saves nothing -- SURVEY §8(d)), and the level-synchronous fused loop costs ~50 us of
// dependent latency per level for a few thousand walks. Here every thread walks one sample to
// its end: coinLT(s, v) picks the in-edge (interpolation search of the row's cumulative
// thresholds), and the visited set of sample s IS its bit in the RRR store (atomicOr; the walk
// stops at a vertex already in the set, a vertex without in-edges, or on "no edge"). Same coins,
// same sets as the fused loop (tests: BPT_LT_FUSED=1 runs the fused loop).
__device__ __forceinline__ bool lt_pick(const uint32_t* __restrict__ roff, const uint2* __restrict__ rec, uint32_t v,
                                        uint32_t r, uint32_t* u_out) {
    uint32_t lo = __ldg(&roff[v]), hi = __ldg(&roff[v + 1]);
    if (lo >= hi) return false;
    uint2 hit = __ldg(&rec[hi - 1]);  // {src, row sum}
    if (r >= hit.y) return false;
    uint32_t clo = 0, chi = hit.y;
    for (int step = 0; hi - lo > 1; ++step) {
        uint32_t g;
        if (step < 4) {
            // interpolation guess in f32 (any guess inside [lo, hi - 2] is correct; no 64-bit division)
            g = lo + min((uint32_t)(__fdividef((float)(r - clo), (float)(chi - clo)) * (float)(hi - lo)), hi - lo - 2);
        } else {
            g = (lo + hi - 1) >> 1;
        }
        const uint2 x = __ldg(&rec[g]);
        if (x.y > r) { hi = g + 1; chi = x.y; hit = x; }
        else { lo = g + 1; clo = x.y; }
    }
    *u_out = hit.x;
    return true;
}

// The same pick with fewer dependent loads (the walk kernel's time is the critical path of its
// longest walks, a chain of dependent DRAM round trips per step): the first guess assumes the
// row sum is ~2^31 (normalised LT weights; any guess gives the same answer, only the number of
// round trips depends on it) and one 64-B window of 8 records around it is loaded at once. The
// answer is the first j in [lo, hi) with cum[j] > r (none if r >= cum[hi - 1]) exactly as in
// lt_pick; when it is not inside the window the search continues on the side it lies.

// lo, hi: the row bounds roff[v], roff[v + 1], loaded by the caller (ahead of time).
__device__ __forceinline__ bool lt_pick_win(const uint32_t* __restrict__ roff, const uint2* __restrict__ rec,
                                            uint32_t m, uint32_t v, uint32_t lo, uint32_t hi, uint32_t r,
                                            uint32_t* u_out) {
    if (lo >= hi) return false;
    uint32_t g = lo + (uint32_t)(((uint64_t)r * (hi - lo)) >> 31);
    g = min(g, hi - 1);
    const uint32_t w0 = (g >= 3 ? g - 3 : 0u) & ~3u;  // 32-B aligned: the window is two 256-bit loads
    if (w0 + 8 > m) return lt_pick(roff, rec, v, r, u_out);
    uint4 q0, q1, q2, q3;
    asm("ld.global.nc.v8.u32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
        : "=r"(q0.x), "=r"(q0.y), "=r"(q0.z), "=r"(q0.w), "=r"(q1.x), "=r"(q1.y), "=r"(q1.z), "=r"(q1.w)
        : "l"(rec + w0));
    asm("ld.global.nc.v8.u32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
        : "=r"(q2.x), "=r"(q2.y), "=r"(q2.z), "=r"(q2.w), "=r"(q3.x), "=r"(q3.y), "=r"(q3.z), "=r"(q3.w)
        : "l"(rec + w0 + 4));
    const uint32_t xs[8] = {q0.x, q0.z, q1.x, q1.z, q2.x, q2.z, q3.x, q3.z};
    const uint32_t ys[8] = {q0.y, q0.w, q1.y, q1.w, q2.y, q2.w, q3.y, q3.w};
    const uint32_t a = max(lo, w0), b = min(hi, w0 + 8);  // window part inside the row (a < b)
    uint32_t k = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) k += (w0 + j >= a && w0 + j < b && ys[j] <= r) ? 1u : 0u;
    const uint32_t j = a + k;  // first index of [a, b) with cum > r, b if none
    // register selects (no dynamic indexing: that would put the window in local memory) as binary
    // trees over the window offset (3 levels of SEL instead of 8 compares and 8 SELs per value)
    auto pick = [&](const uint32_t (&vals)[8], uint32_t t) -> uint32_t {
        const uint32_t l0 = (t & 1u) ? vals[1] : vals[0], l1 = (t & 1u) ? vals[3] : vals[2];
        const uint32_t l2 = (t & 1u) ? vals[5] : vals[4], l3 = (t & 1u) ? vals[7] : vals[6];
        const uint32_t m0 = (t & 2u) ? l1 : l0, m1 = (t & 2u) ? l3 : l2;
        return (t & 4u) ? m1 : m0;
    };
    const uint32_t xj = pick(xs, (j - w0) & 7u), xa = pick(xs, a - w0), ya = pick(ys, a - w0), yb = pick(ys, b - 1 - w0);
    uint32_t clo, chi;
    uint2 hit;
    if (j < b) {
        if (j > a || a == lo) {  // cum[j - 1] <= r < cum[j] (or j == lo)
            *u_out = xj;
            return true;
        }
        // cum[a] > r, a > lo: the answer is in [lo, a]
        hi = a + 1;
        chi = ya;
        hit = make_uint2(xa, chi);
        clo = 0;
    } else {
        if (b == hi) return false;  // r >= cum[hi - 1]: no in-edge chosen
        clo = yb;                 // cum[b - 1] <= r: the answer is in [b, hi)
        lo = b;
        hit = __ldg(&rec[hi - 1]);
        if (r >= hit.y) return false;
        chi = hit.y;
    }
    for (int step = 0; hi - lo > 1; ++step) {
        uint32_t gg;
        if (step < 4) {  // interpolation guess in f32 (any guess inside [lo, hi - 2] is correct)
            const float f = __fdividef((float)(r - clo), (float)(chi - clo)) * (float)(hi - lo);
            gg = lo + min((uint32_t)f, hi - lo - 2);
        } else {
            gg = (lo + hi - 1) >> 1;
        }
        const uint2 x = __ldg(&rec[gg]);
        if (x.y > r) { hi = gg + 1; chi = x.y; hit = x; }
        else { lo = gg + 1; clo = x.y; }
    }
    *u_out = hit.x;
    return true;
}

__global__ void __launch_bounds__(256) k_walk_lt(uint64_t* __restrict__ store, uint32_t n,
                                                 const uint32_t* __restrict__ roff, const uint2* __restrict__ rec,
                                                 uint64_t s0, uint64_t nlocal, uint32_t k_start, uint32_t k_lt,
                                                 uint32_t* __restrict__ sizes, uint32_t* __restrict__ count0,
                                                 unsigned long long* __restrict__ totals) {
    unsigned long long members = 0;
    uint32_t longest = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nlocal; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t s = s0 + i;  // s0 is block aligned: local block i / 64, colour bit s % 64
        uint64_t* V = store + (i >> 6) * (uint64_t)n;
        const unsigned long long bit = 1ull << (s & 63);
        const uint2 w = philox2x32_10((uint32_t)s, (uint32_t)(s >> 32), k_start);
        uint32_t v = (uint32_t)__umul64hi(((uint64_t)w.y << 32) | w.x, (uint64_t)n);
        atomicOr((unsigned long long*)&V[v], bit);
        atomicAdd(&count0[v], 1u);
        uint32_t size = 1, u = 0;
        while (lt_pick(roff, rec, v, philox2x32_10(v, (uint32_t)s, k_lt).x >> 1, &u)) {
            if (atomicOr((unsigned long long*)&V[u], bit) & bit) break;  // already in RR_s
            atomicAdd(&count0[u], 1u);
            ++size;
            v = u;
        }
        sizes[i] = size;
        members += size;
        longest = max(longest, size);
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
        members += __shfl_xor_sync(kFull, members, d);
        longest = max(longest, __shfl_xor_sync(kFull, longest, d));
    }
    if ((threadIdx.x & 31) == 0 && members) {
        atomicAdd(&totals[0], members);
        atomicMax(&totals[1], (unsigned long long)longest);
    }
}

// Second pass for the selection: re-walk each sample (same coins, same path; the walk length is
// known from pass 1) and write its members to its slot of the member-list buffer.
__global__ void __launch_bounds__(256) k_walk_lt_lists(uint32_t n, const uint32_t* __restrict__ roff,
                                                       const uint2* __restrict__ rec, uint32_t m, uint64_t s0,
                                                       uint64_t nlocal,
                                                       uint32_t k_start, uint32_t k_lt,
                                                       const uint32_t* __restrict__ sizes,
                                                       const uint64_t* __restrict__ off, uint32_t* __restrict__ members) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nlocal; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t s = s0 + i;
        const uint2 w = philox2x32_10((uint32_t)s, (uint32_t)(s >> 32), k_start);
        uint32_t v = (uint32_t)__umul64hi(((uint64_t)w.y << 32) | w.x, (uint64_t)n);
        uint32_t* out = members + off[i];
        const uint32_t size = sizes[i];
        out[0] = v;
        for (uint32_t j = 1; j < size; ++j) {
            uint32_t u = 0;
            lt_pick_win(roff, rec, m, v, __ldg(&roff[v]), __ldg(&roff[v + 1]),
                        philox2x32_10(v, (uint32_t)s, k_lt).x >> 1, &u);
            out[j] = u;
            v = u;
        }
    }
}

// Sparse LT store: the visited set of a walk is a per-thread open-addressing hash set (2,048
// slots; a walk longer than 1,536 vertices is reported, the dense store handles those), so no
// dense n x blocks bitmap exists at all. The sets live in global memory (Graph::walk_ht, one
// 8 KB region per thread, zeroed once) and every entry carries the epoch of the walk that wrote
// it: entry = epoch << shift | (u + 1), n < 2^shift. A slot whose epoch is not the current walk's
// is empty, so a set is never cleared between walks (round 1 cleared a local-memory set of 8 KB
// per walk: 2.1 GB of stores per C3 call, 23x the walk's algorithmic DRAM bytes). Each call
// takes a fresh range of epochs (one per walk of a thread); the host re-zeroes the tables when the
// epochs wrap. shift = 32 (n >= 2^31): epoch 0, empty = 0, the tables cleared per walk.
#ifndef BPT_WALK_HASH_BITS
#define BPT_WALK_HASH_BITS 11
#endif
// per-thread visited set of a walk: 2^bits u32 slots, walks up to 3/4 of that (longer ones move
// the call to the dense-store walks)
constexpr uint32_t kWalkHashBits = BPT_WALK_HASH_BITS;
constexpr uint32_t kWalkHash = 1u << kWalkHashBits, kWalkMax = kWalkHash / 4 * 3;

// Register cap for the sparse walks: at 7 blocks per SM ptxas fits the walk in 32 registers, so
// 8 blocks x 256 threads are resident per SM and C3's 262,144 walks (1,024 blocks) start in ONE
// wave (at 64 registers, 592 resident blocks: the second wave waited for the first wave's
// longest walks). C3 walk 6.6 -> 4.8 ms (warm, CUDA events; 3, 5, 6 blocks/SM: 6.6, 5.4, 5.7).
#ifndef BPT_WALK_MINB
#define BPT_WALK_MINB 7
#endif
struct WalkTab {
    uint32_t* ht;       // [threads][kWalkHash]
    uint32_t shift;     // n < 2^shift (32: no epoch bits)
    uint32_t epoch0;    // epoch of a thread's first walk of this call (walk j: epoch0 + j)
    uint32_t clear;     // 1: clear the thread's set before every walk (no epoch range left)
};
// The visited-set probe *slot (global walk table) and the row bounds roff[u], roff[u + 1] in ONE asm
// statement: the probe decides a branch, and without this the compiler sank the bound loads
// below it (the probe and the bounds then ran as two DRAM round trips in series).
__device__ __forceinline__ void ld_probe_and_bounds_g(const uint32_t* slot, const uint32_t* p, uint32_t& x,
                                                      uint32_t& lo, uint32_t& hi) {
    asm volatile("ld.global.u32 %0, [%3];\n\tld.global.nc.u32 %1, [%4];\n\tld.global.nc.u32 %2, [%4+4];"
                 : "=r"(x), "=r"(lo), "=r"(hi)
                 : "l"(slot), "l"(p)
                 : "memory");
}
__global__ void __launch_bounds__(256, BPT_WALK_MINB) k_walk_lt_sparse(uint32_t n, const uint32_t* __restrict__ roff,
                                                        const uint2* __restrict__ rec, uint32_t m, uint64_t s0,
                                                        uint64_t nlocal,
                                                        uint32_t k_start, uint32_t k_lt,
                                                        uint32_t* __restrict__ sizes, uint32_t* __restrict__ count0,
                                                        unsigned long long* __restrict__ totals,
                                                        uint32_t* __restrict__ rows, WalkTab tab) {
    // rows (optional): member i of local sample l at rows[l * kWalkMax + i], in walk order
    const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    uint32_t* __restrict__ ht = tab.ht + tid * kWalkHash;
    unsigned long long members = 0;
    uint32_t longest = 0, too_long = 0;
    uint32_t epoch = tab.epoch0;
    for (uint64_t i = tid; i < nlocal; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t s = s0 + i;
        if (tab.clear) {
            for (uint32_t h = 0; h < kWalkHash; h += 4) *reinterpret_cast<uint4*>(ht + h) = make_uint4(0, 0, 0, 0);
        }
        // slot value of u in this walk; a slot is empty unless its epoch is this walk's
        const uint32_t etag = epoch << (tab.shift & 31), emask = tab.shift >= 32 ? 0u : ~0u << tab.shift;
        auto empty = [&](uint32_t x) -> bool { return ((x & emask) != etag) | (x == 0u); };
        // insert u, whose home slot h was already read (x); false if u was already in the set
        auto insert_at = [&](uint32_t u, uint32_t h, uint32_t x) -> bool {
            const uint32_t want = etag | (u + 1u);
            while (true) {
                if (x == want) return false;
                if (empty(x)) { ht[h] = want; return true; }
                h = (h + 1) & (kWalkHash - 1);
                x = ht[h];
            }
        };
        auto home = [](uint32_t u) -> uint32_t { return (u * 0x9E3779B1u) >> (32 - kWalkHashBits); };
        auto insert = [&](uint32_t u) -> bool { const uint32_t h = home(u); return insert_at(u, h, ht[h]); };
        const uint2 w = philox2x32_10((uint32_t)s, (uint32_t)(s >> 32), k_start);
        uint32_t v = (uint32_t)__umul64hi(((uint64_t)w.y << 32) | w.x, (uint64_t)n);
        insert(v);
        atomicAdd(&count0[v], 1u);
        uint32_t* row = rows ? rows + i * kWalkMax : nullptr;
        if (row) row[0] = v;
        uint32_t size = 1, u = 0, bad_bounds = 0;
        uint32_t lo = __ldg(&roff[v]), hi = __ldg(&roff[v + 1]);
        uint32_t r = philox2x32_10(v, (uint32_t)s, k_lt).x >> 1;
        while (lt_pick_win(roff, rec, m, v, lo, hi, r, &u)) {
            // u's visited-set probe, its row bounds and its coin do not depend on each other: all
            // three are in flight together (one DRAM round trip per step instead of two in a row;
            // the bounds and coin are wasted only on the step that ends the walk)
            const uint32_t h = home(u);
            uint32_t x;
            ld_probe_and_bounds_g(&ht[h], roff + u, x, lo, hi);
            // consumed on both sides of the branch below (never true for a validated CSR, where
            // roff[u] <= m): keeps the bound loads above the branch
            bad_bounds |= (lo > m) | (hi > m);
            r = philox2x32_10(u, (uint32_t)s, k_lt).x >> 1;
            if (!insert_at(u, h, x)) break;  // already in RR_s
            atomicAdd(&count0[u], 1u);
            if (size >= kWalkMax) { too_long = 1; break; }
            if (row) row[size] = u;
            ++size;
            v = u;
        }
        sizes[i] = size;
        members += size;
        longest = max(longest, size);
        too_long |= bad_bounds;
        if (!tab.clear) ++epoch;
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
        members += __shfl_xor_sync(kFull, members, d);
        longest = max(longest, __shfl_xor_sync(kFull, longest, d));
        too_long |= __shfl_xor_sync(kFull, too_long, d);
    }
    if ((threadIdx.x & 31) == 0) {
        if (members) atomicAdd(&totals[0], members);
        if (longest) atomicMax(&totals[1], (unsigned long long)longest);
        if (too_long) atomicMax(&totals[2], 1ull);
    }
}

// rows (walk order, kWalkMax-strided) -> contiguous member lists at off[l]
__global__ void k_rows_to_lists(const uint32_t* __restrict__ rows, const uint64_t* __restrict__ off, uint64_t nlists,
                                uint32_t* __restrict__ members) {
    const int lane = threadIdx.x & 31;
    for (uint64_t l = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; l < nlists;
         l += ((uint64_t)gridDim.x * blockDim.x) >> 5) {
        const uint64_t b = off[l], len = off[l + 1] - b;
        for (uint64_t j = lane; j < len; j += 32) members[b + j] = rows[l * kWalkMax + j];
    }
}

// Bitonic sort of one member list per block in shared memory (padded to a power of two).
constexpr uint32_t kSortMax = 4096;
__global__ void __launch_bounds__(256) k_sort_lists(const uint64_t* __restrict__ off, uint32_t* __restrict__ members,
                                                    uint64_t nlists, uint32_t* __restrict__ err) {
    __shared__ uint32_t sh[kSortMax];
    for (uint64_t l = blockIdx.x; l < nlists; l += gridDim.x) {
        const uint64_t b = off[l], len = off[l + 1] - b;
        if (len <= 1) continue;
        if (len > kSortMax) {
            if (threadIdx.x == 0) *err = 1;
            continue;
        }
        uint32_t P = 1;
        while (P < len) P <<= 1;
        __syncthreads();
        for (uint32_t i = threadIdx.x; i < P; i += blockDim.x) sh[i] = i < len ? members[b + i] : ~0u;
        __syncthreads();
        for (uint32_t k = 2; k <= P; k <<= 1)
            for (uint32_t j = k >> 1; j > 0; j >>= 1) {
                for (uint32_t i = threadIdx.x; i < P; i += blockDim.x) {
                    const uint32_t ix = i ^ j;
                    if (ix > i) {
                        const uint32_t x = sh[i], y = sh[ix];
                        if (((i & k) == 0) == (x > y)) { sh[i] = y; sh[ix] = x; }
                    }
                }
                __syncthreads();
            }
        for (uint32_t i = threadIdx.x; i < len; i += blockDim.x) members[b + i] = sh[i];
    }
}

// LT (reading C-6): work items are (entry, colour) pairs. For colour c at v: r = coinLT(s_c, v)
// >> 1, chosen in-edge j = first with cum[j] > r (binary search of the row, rows are
// cumulative thresholds); none if r >= row sum. If u = src[j] has not been visited by c,
// N[u] |= bit c (fusing) and the first setter enqueues u.
template <bool kCoh>
__device__ __forceinline__ void expand_lt_body(const BatchArgs& a, const uint32_t* __restrict__ tstart,
                                               cudaGraphConditionalHandle h_level, int use_cond) {
    Ctl* ctl = a.ctl;
    const uint32_t level = LDX(&ctl->level);
    const uint64_t gblk0 = LDX(&ctl->gblk0);
    const LevelRec* L = &a.lv[level];
    LevelRec* Ln = &a.lv[level + 1];
    if (threadIdx.x == 0) atomicMin(&ctl->t_start, global_ns());
    const unsigned long long packed = LDX(&L->packed);
    const uint64_t nq = packed >> kPackShift;
    const uint64_t total = packed & kEdgeMask;
    if (nq == 0 || LDX(&L->overflow)) {
        finish_expand(a, h_level, use_cond, gridDim.x);
        return;
    }
    extern __shared__ __align__(16) unsigned char smem_raw[];
    SmemTile& sm = *reinterpret_cast<SmemTile*>(smem_raw);
    const uint64_t ntiles = (total + kTile - 1) / kTile;
    unsigned long long coins = 0, atoms = 0;
    for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const uint64_t t0 = tile * kTile;
        const uint32_t j0 = LDX(&tstart[tile]);
        const uint64_t jend = tile + 1 < ntiles ? (uint64_t)LDX(&tstart[tile + 1]) + 1 : nq;
        const uint32_t cnt = (uint32_t)umin64(jend - j0, (uint64_t)kTile + 1);
        __syncthreads();
        for (uint32_t k = threadIdx.x; k < cnt; k += kThreads) {
            const uint64_t j = j0 + k;
            const uint64_t off = LDX(&a.qoff[j]);
            const uint4 ent = LDX(&a.q[j]);
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
                const uint32_t s = (uint32_t)(64ull * (gblk0 + slot)) + bit;
                const uint32_t r = philox2x32_10(v, s, a.k_lt).x >> 1;
                ++coins;
                // first j of row v with cum[j] > r (none if r >= the row sum): interpolation
                // search (cum grows ~linearly along a row: ~2-4 dependent probes instead of
                // log2(deg)), bisection after 4 probes
                uint32_t lo2 = a.roff[v], hi2 = a.roff[v + 1];
                bool found = false;
                uint32_t u = 0;
                if (lo2 < hi2) {
                    uint2 hit = __ldg(&a.rec[hi2 - 1]);  // record at hi2 - 1: {src, row sum}
                    if (r < hit.y) {
                        // answer in [lo2, hi2): cum[lo2 - 1] = clo <= r < chi = cum[hi2 - 1]
                        uint32_t clo = 0, chi = hit.y;
                        for (int step = 0; hi2 - lo2 > 1; ++step) {
                            uint32_t g;
                            if (step < 4) {
                                // interpolation guess in f32 (any guess inside [lo, hi - 2] is correct; no 64-bit division)
                                g = lo2 + min((uint32_t)(__fdividef((float)(r - clo), (float)(chi - clo)) * (float)(hi2 - lo2)), hi2 - lo2 - 2);
                            } else {
                                g = (lo2 + hi2 - 1) >> 1;
                            }
                            const uint2 x = __ldg(&a.rec[g]);
                            if (x.y > r) { hi2 = g + 1; chi = x.y; hit = x; }
                            else { lo2 = g + 1; clo = x.y; }
                        }
                        found = true;
                        u = hit.x;
                    }
                }
                if (found) {
                    const uint64_t b = 1ull << bit;
                    const uint64_t Vu = LDX(&a.VN[(size_t)slot * a.n + u].x);
                    if (!(Vu & b)) {
                        ++atoms;
                        const unsigned long long old = atomicOr(&a.VN[(size_t)slot * a.n + u].y, b);
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
    finish_expand(a, h_level, use_cond, gridDim.x);
}

__global__ void __launch_bounds__(kThreads) k_expand_lt(BatchArgs a, const uint32_t* __restrict__ tstart,
                                                      cudaGraphConditionalHandle h_level, int use_cond) {
    count_self(a.ctl);
    if (!a.ctl->cont) return;
    expand_lt_body<false>(a, tstart, h_level, use_cond);
}

// LT levels are thin (a few thousand walks) and many (~700 per batch on C3): one cooperative
// launch runs the whole level loop of a batch, compact(L) -> grid barrier -> expand(L) (its
// last block advances the level) -> grid barrier, instead of two launches per level.
// Grid barrier (all blocks co-resident: cooperative launch): one arrival atomic per block, the
// last arrival bumps the generation the others spin on.
__device__ __forceinline__ void grid_barrier(Ctl* c) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const uint32_t gen = *(volatile uint32_t*)&c->bar_gen;
        __threadfence();
        if (atomicAdd(&c->bar_count, 1u) == gridDim.x - 1) {
            c->bar_count = 0;
            __threadfence();
            atomicAdd(&c->bar_gen, 1u);
        } else {
            while (*(volatile uint32_t*)&c->bar_gen == gen) {
            }
        }
        __threadfence();
    }
    __syncthreads();
}

__global__ void __launch_bounds__(kThreads) k_levels_lt(BatchArgs a, uint32_t* __restrict__ tstart,
                                                      uint64_t tstart_cap) {
    count_self(a.ctl);
    while (__ldcg(&a.ctl->cont)) {
        compact_body<true, kTile>(a, tstart, tstart_cap);
        grid_barrier(a.ctl);
        expand_lt_body<true>(a, tstart, (cudaGraphConditionalHandle)0, 0);
        grid_barrier(a.ctl);
    }
}

// ------------------------------------------------------------------------ level / batch control
// After expand(L): fold level L's record into the totals, keep a tagged copy for the level
// statistics, stop the batch when level L+1 discovered nothing (or a queue overflowed), and
// set the level-loop condition of the graph (device-resident loop, no host round trip).
// After a batch: clear the level records it used, move to the next batch, set the batch-loop
// condition (stop early on an error).
__global__ void k_next_batch(BatchArgs a, cudaGraphConditionalHandle h_batch, int use_cond) {
    Ctl* c = a.ctl;
    count_self(c);
    const uint32_t used = c->level + 2;
    for (uint32_t i = threadIdx.x; i < used && i < (uint32_t)kMaxLevels; i += blockDim.x) {
        LevelRec z{};
        a.lv[i] = z;
    }
    if (threadIdx.x == 0) {
        c->batch += 1;
        c->blk0 += c->slots;
        c->gblk0 += c->slots;
        const uint64_t remaining = a.blocks - c->blk0;
        c->slots = (uint32_t)umin64(a.slots_max, remaining);
        c->level = 0;
        c->cont = 0;
        if (use_cond) cudaGraphSetConditional(h_batch, (remaining > 0 && !c->error) ? 1u : 0u);
    }
}


int g_expand_grid = 0;
int g_expand_grid_w = 0;
int g_expand_grid_b = 0;
int g_expand_grid_p = 0;
int g_expand_grid_lt = 0;
int g_levels_per_sm_lt = 0;  // co-resident blocks per SM of the cooperative LT loop
int g_compact_grid = 0;

}  // namespace

void launch_walk_lt(uint64_t* store, uint32_t n, const uint32_t* roff, const uint2* rec, uint64_t s0, uint64_t nlocal,
                    uint32_t k_start, uint32_t k_lt, uint32_t* sizes, uint32_t* count0, unsigned long long* totals,
                    cudaStream_t st) {
    const unsigned grid = (unsigned)umin64((nlocal + 255) / 256, (uint64_t)num_sms() * 8);
    k_walk_lt<<<grid ? grid : 1, 256, 0, st>>>(store, n, roff, rec, s0, nlocal, k_start, k_lt, sizes, count0, totals);
    count_launch();
    ::bpt::check_cuda(cudaGetLastError(), "launch k_walk_lt");
}

uint32_t walk_row_stride() { return kWalkMax; }

void launch_rows_to_lists(const uint32_t* rows, const uint64_t* off, uint64_t nlists, uint32_t* members, cudaStream_t st) {
    const unsigned grid = (unsigned)umin64((nlists * 32 + 255) / 256, (uint64_t)num_sms() * 16);
    if (!grid) return;
    k_rows_to_lists<<<grid, 256, 0, st>>>(rows, off, nlists, members);
    count_launch();
    ::bpt::check_cuda(cudaGetLastError(), "launch k_rows_to_lists");
}

void launch_walk_lt_sparse(const Graph& g, uint64_t s0, uint64_t nlocal,
                           uint32_t k_start, uint32_t k_lt, uint32_t* sizes, uint32_t* count0,
                           unsigned long long* totals, uint32_t* rows, cudaStream_t st) {
    const unsigned grid = (unsigned)umax64(1, umin64((nlocal + 255) / 256, (uint64_t)num_sms() * 8));
    const uint64_t threads = (uint64_t)grid * 256;
    const uint64_t walks = umax64(1, (nlocal + threads - 1) / threads);  // walks per thread
    std::lock_guard<std::mutex> lock(g.walk_mu);
    if (!g.walk_ev) ::bpt::check_cuda(cudaEventCreateWithFlags(&g.walk_ev, cudaEventDisableTiming), "walk event");
    else ::bpt::check_cuda(cudaStreamWaitEvent(st, g.walk_ev, 0), "walk event wait");  // previous user of the tables
    const size_t bytes = threads * kWalkHash * 4;
    WalkTab tab{};
    tab.shift = 32u - (uint32_t)__builtin_clz(g.n | 1u);  // n < 2^shift
    if (tab.shift >= 31) tab.shift = 32;                    // no room for an epoch field
    const uint64_t max_epoch = tab.shift >= 32 ? 0 : (1ull << (32 - tab.shift)) - 1;
    if (g.walk_ht.bytes < bytes) {
        g.walk_ht.reset();
        g.walk_ht.alloc(bytes);
        ::bpt::check_cuda(cudaMemsetAsync(g.walk_ht.p, 0, g.walk_ht.bytes, st), "walk table zero");
        g.walk_epoch = 0;
    }
    if (max_epoch == 0 || walks > max_epoch) {
        tab.clear = 1;  // every walk clears its set (epoch 0 or a single epoch, re-zeroed below)
        ::bpt::check_cuda(cudaMemsetAsync(g.walk_ht.p, 0, g.walk_ht.bytes, st), "walk table zero");
        g.walk_epoch = 0;
        tab.epoch0 = max_epoch ? 1u : 0u;
    } else {
        if (g.walk_epoch + walks > max_epoch) {  // epochs wrap: stale tags could alias
            ::bpt::check_cuda(cudaMemsetAsync(g.walk_ht.p, 0, g.walk_ht.bytes, st), "walk table zero");
            g.walk_epoch = 0;
        }
        tab.epoch0 = g.walk_epoch + 1;
        g.walk_epoch += (uint32_t)walks;
    }
    tab.ht = g.walk_ht.as<uint32_t>();
    k_walk_lt_sparse<<<grid, 256, 0, st>>>(g.n, g.roff.as<uint32_t>(), g.rec.as<uint2>(), (uint32_t)g.m, s0, nlocal,
                                           k_start, k_lt, sizes, count0, totals, rows, tab);
    count_launch();
    ::bpt::check_cuda(cudaGetLastError(), "launch k_walk_lt_sparse");
    g.walk_ht.stream = st;
    ::bpt::check_cuda(cudaEventRecord(g.walk_ev, st), "walk event record");
}

void launch_sort_lists(const uint64_t* off, uint32_t* members, uint64_t nlists, uint32_t* err, cudaStream_t st) {
    const unsigned grid = (unsigned)umin64(nlists, (uint64_t)num_sms() * 16);
    if (!grid) return;
    k_sort_lists<<<grid, 256, 0, st>>>(off, members, nlists, err);
    count_launch();
    ::bpt::check_cuda(cudaGetLastError(), "launch k_sort_lists");
}

void launch_walk_lt_lists(uint32_t n, const uint32_t* roff, const uint2* rec, uint32_t m, uint64_t s0, uint64_t nlocal,
                          uint32_t k_start, uint32_t k_lt, const uint32_t* sizes, const uint64_t* off,
                          uint32_t* members, cudaStream_t st) {
    const unsigned grid = (unsigned)umin64((nlocal + 255) / 256, (uint64_t)num_sms() * 8);
    k_walk_lt_lists<<<grid ? grid : 1, 256, 0, st>>>(n, roff, rec, m, s0, nlocal, k_start, k_lt, sizes, off, members);
    count_launch();
    ::bpt::check_cuda(cudaGetLastError(), "launch k_walk_lt_lists");
}

// the compaction instance whose unit matches the expansion of this batch
using CompactFn = void (*)(BatchArgs, uint32_t*, uint64_t);
static CompactFn compact_kernel(const BatchArgs& a) {
    if (a.model != BPT_IC) return k_compact<kTile>;
    if (a.touched) return a.vmajor ? k_compact_bmv<kUnitBm> : k_compact_bm<kUnitBm>;
    return k_compact<kUnitIC>;
}

uint32_t expand_unit(int model, bool bitmap) {
    return model == BPT_IC ? (bitmap ? (uint32_t)kUnitBm : (uint32_t)kUnitIC) : kTile;
}

int expand_grid() {
    if (!g_expand_grid) {
        int per_sm = 0;
        BPT_CUDA(cudaFuncSetAttribute(k_expand_lt, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(SmemTile)));
        for (void* f : {(void*)k_expand_ic<true>, (void*)k_expand_ic<false>})
            BPT_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)(sizeof(WarpScratch) * kWarps)));
        BPT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_expand_ic<true>, kThreads,
                                                               sizeof(WarpScratch) * kWarps));
        g_expand_grid = num_sms() * (per_sm > 0 ? per_sm : 1);
        int per_sm_b = 0;
        for (void* f : {(void*)k_expand_bm<false>, (void*)k_expand_bm<true>})
            BPT_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)(sizeof(BmScratch) * kWarps)));
        BPT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_b, k_expand_bm<false>, kThreads,
                                                               sizeof(BmScratch) * kWarps));
        g_expand_grid_b = num_sms() * (per_sm_b > 0 ? per_sm_b : 1);
        int per_sm_p = 0;
        BPT_CUDA(cudaFuncSetAttribute(k_expand_pull, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)(sizeof(BmScratch) * kWarps)));
        BPT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_p, k_expand_pull, kThreads,
                                                               sizeof(BmScratch) * kWarps));
        g_expand_grid_p = num_sms() * (per_sm_p > 0 ? per_sm_p : 1);
        int per_sm_w = 0;
        BPT_CUDA(cudaFuncSetAttribute(k_expand_w, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)(sizeof(WarpScratchW) * kWarps)));
        BPT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_w, k_expand_w, kThreads,
                                                               sizeof(WarpScratchW) * kWarps));
        g_expand_grid_w = num_sms() * (per_sm_w > 0 ? per_sm_w : 1);
        int per_sm_lt = 0;
        BPT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_lt, k_expand_lt, kThreads, sizeof(SmemTile)));
        g_expand_grid_lt = num_sms() * (per_sm_lt > 0 ? per_sm_lt : 1);
        int per_sm_pl = 0;  // the cooperative level loop must be co-resident
        BPT_CUDA(cudaFuncSetAttribute(k_levels_lt, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(SmemTile)));
        BPT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_pl, k_levels_lt, kThreads, sizeof(SmemTile)));
        g_levels_per_sm_lt = per_sm_pl > 0 ? per_sm_pl : 1;
        int per_sm_c = 0;
        BPT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_c, k_compact<kUnitBm>, kThreads, 0));
        g_compact_grid = num_sms() * (per_sm_c > 0 ? per_sm_c : 1);
    }
    return g_expand_grid;
}

// Fused LT batches run their level loop as one cooperative launch (BPT_FLAG_LT_LEVELS: per-level
// launches instead); IC always launches per level (a cooperative IC loop measured slower: its
// same-launch data would have to bypass L1, DESIGN §11 (h))
bool level_loop_persistent(const BatchArgs& a) { return a.model == BPT_LT && !a.wide && a.lt_persist; }

// few blocks: the LT levels are thin, and a grid barrier costs ~ the number of blocks
static unsigned levels_grid_lt(const BatchArgs& a) {
    expand_grid();
    return (unsigned)(num_sms() * std::max(1, std::min(a.lt_blocks_per_sm > 0 ? a.lt_blocks_per_sm : 1, g_levels_per_sm_lt)));
}

static unsigned init_grid(const BatchArgs& a) { return (unsigned)(((uint64_t)a.slots_max * 64 + 255) / 256); }

void launch_init(const BatchArgs& a, cudaStream_t st) {
    if (a.wide) k_init_w<<<init_grid(a), 256, 0, st>>>(a, (cudaGraphConditionalHandle)0, 0);
    else k_init<<<init_grid(a), 256, 0, st>>>(a, (cudaGraphConditionalHandle)0, 0);
    count_launch();
    ::bpt::check_cuda(cudaGetLastError(), "launch k_init");
}

// one level of the host-driven loop: compact(L) -> expand(L) (bracketed by ev0/ev1 if given; its last
// block advances the level)
void launch_level(const BatchArgs& a, uint32_t* tstart, uint64_t tstart_cap, cudaStream_t st, cudaEvent_t ev0,
                  cudaEvent_t ev1) {
    expand_grid();
    const cudaGraphConditionalHandle h0 = 0;
    if (a.wide) {
        k_compact_w<<<g_compact_grid, kThreads, 0, st>>>(a, tstart, tstart_cap);
        if (ev0) BPT_CUDA(cudaEventRecord(ev0, st));
        k_expand_w<<<g_expand_grid_w, kThreads, sizeof(WarpScratchW) * kWarps, st>>>(a, tstart, h0, 0);
        if (ev1) BPT_CUDA(cudaEventRecord(ev1, st));
        count_launch(2);
        ::bpt::check_cuda(cudaGetLastError(), "launch wide level kernels");
        return;
    }
    compact_kernel(a)<<<g_compact_grid, kThreads, 0, st>>>(a, tstart, tstart_cap);
    if (ev0) BPT_CUDA(cudaEventRecord(ev0, st));
    if (a.model == BPT_IC && a.touched) {
        if (a.vmajor) k_expand_bm<true><<<g_expand_grid_b, kThreads, sizeof(BmScratchV) * kWarps, st>>>(a, tstart, h0, 0);
        else k_expand_bm<false><<<g_expand_grid_b, kThreads, sizeof(BmScratch) * kWarps, st>>>(a, tstart, h0, 0);
        if (a.pull) {
            k_expand_pull<<<g_expand_grid_p, kThreads, sizeof(BmScratch) * kWarps, st>>>(a, h0, 0);
            count_launch();
        }
    }
    else if (a.model == BPT_IC && a.colors == 64)
        k_expand_ic<true><<<g_expand_grid, kThreads, sizeof(WarpScratch) * kWarps, st>>>(a, tstart, h0, 0);
    else if (a.model == BPT_IC)
        k_expand_ic<false><<<g_expand_grid, kThreads, sizeof(WarpScratch) * kWarps, st>>>(a, tstart, h0, 0);
    else
        k_expand_lt<<<g_expand_grid_lt, kThreads, sizeof(SmemTile), st>>>(a, tstart, h0, 0);
    if (ev1) BPT_CUDA(cudaEventRecord(ev1, st));
    count_launch(2);
    ::bpt::check_cuda(cudaGetLastError(), "launch level kernels");
}

void launch_next_batch(const BatchArgs& a, cudaStream_t st) {
    k_next_batch<<<1, 256, 0, st>>>(a, (cudaGraphConditionalHandle)0, 0);
    count_launch();
    ::bpt::check_cuda(cudaGetLastError(), "launch k_next_batch");
}

// The whole bpt_sample loop as one CUDA graph with two nested conditional WHILE nodes:
//   while (batches remain) { init -> while (frontier non-empty) { compact -> expand }
//                            -> finalize -> count -> next_batch }
// Conditions are set on the device (cudaGraphSetConditional) by the expansion / k_next_batch, so
// the host launches the graph once and never polls (SURVEY §8(a) kernel note 4).
cudaGraphExec_t build_sampling_graph(const BatchArgs& a, uint32_t* tstart, uint64_t tstart_cap, const StoreHook& h) {
    expand_grid();
    cudaGraph_t root;
    BPT_CUDA(cudaGraphCreate(&root, 0));
    cudaGraphConditionalHandle h_batch, h_level;
    BPT_CUDA(cudaGraphConditionalHandleCreate(&h_batch, root, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams cb{};
    cb.type = cudaGraphNodeTypeConditional;
    cb.conditional.handle = h_batch;
    cb.conditional.type = cudaGraphCondTypeWhile;
    cb.conditional.size = 1;
    cudaGraphNode_t n_batch;
    BPT_CUDA(cudaGraphAddNode(&n_batch, root, nullptr, 0, &cb));
    cudaGraph_t body = cb.conditional.phGraph_out[0];
    const bool lt_persist = level_loop_persistent(a);
    h_level = 0;
    if (!lt_persist) BPT_CUDA(cudaGraphConditionalHandleCreate(&h_level, body, 1, cudaGraphCondAssignDefault));

    BatchArgs args = a;
    int one = 1;
    auto add_kernel = [&](cudaGraph_t g, const cudaGraphNode_t* dep, void* fn, dim3 grid, dim3 block, size_t smem,
                          void** params) {
        cudaKernelNodeParams p{};
        p.func = fn;
        p.gridDim = grid;
        p.blockDim = block;
        p.sharedMemBytes = (unsigned)smem;
        p.kernelParams = params;
        cudaGraphNode_t node;
        BPT_CUDA(cudaGraphAddKernelNode(&node, g, dep, dep ? 1 : 0, &p));
        return node;
    };
    int zero = 0;
    // batch body: init
    void* init_args[] = {&args, &h_level, lt_persist ? &zero : &one};
    cudaGraphNode_t n_init =
        add_kernel(body, nullptr, a.wide ? (void*)k_init_w : (void*)k_init, dim3(init_grid(a)), dim3(256), 0, init_args);
    if (lt_persist) {
        // the whole level loop as one cooperative launch (grid barriers between phases)
        void* lv_args[] = {&args, &tstart, &tstart_cap};
        cudaGraphNode_t n_lv = add_kernel(body, &n_init, (void*)k_levels_lt, dim3(levels_grid_lt(a)), dim3(kThreads),
                                          sizeof(SmemTile), lv_args);
        cudaLaunchAttributeValue coop{};
        coop.cooperative = 1;
        BPT_CUDA(cudaGraphKernelNodeSetAttribute(n_lv, cudaLaunchAttributeCooperative, &coop));
        cudaGraphNode_t n_store;
        add_store_nodes(body, n_lv, *h.S, h.VN, a.ctl, a.slots_max, h.roff, h.d_elog, &n_store, a.wide != 0, a.touched ? (a.vmajor ? 2 : 1) : 0);
        void* nb_args[] = {&args, &h_batch, &one};
        add_kernel(body, &n_store, (void*)k_next_batch, dim3(1), dim3(256), 0, nb_args);
        cudaGraphExec_t exec;
        BPT_CUDA(cudaGraphInstantiate(&exec, root, 0));
        BPT_CUDA(cudaGraphDestroy(root));
        return exec;
    }
    // level loop
    cudaGraphNodeParams cl{};
    cl.type = cudaGraphNodeTypeConditional;
    cl.conditional.handle = h_level;
    cl.conditional.type = cudaGraphCondTypeWhile;
    cl.conditional.size = 1;
    cudaGraphNode_t n_level;
    BPT_CUDA(cudaGraphAddNode(&n_level, body, &n_init, 1, &cl));
    cudaGraph_t lbody = cl.conditional.phGraph_out[0];
    void* cmp_args[] = {&args, &tstart, &tstart_cap};
    void* cmpw_args[] = {&args, &tstart, &tstart_cap};
    cudaGraphNode_t n_cmp = a.wide
        ? add_kernel(lbody, nullptr, (void*)k_compact_w, dim3(g_compact_grid), dim3(kThreads), 0, cmpw_args)
        : add_kernel(lbody, nullptr, (void*)compact_kernel(a), dim3(g_compact_grid), dim3(kThreads), 0, cmp_args);
    void* exp_args[] = {&args, &tstart, &h_level, &one};
    cudaGraphNode_t n_exp = a.wide
        ? add_kernel(lbody, &n_cmp, (void*)k_expand_w, dim3(g_expand_grid_w), dim3(kThreads),
                     sizeof(WarpScratchW) * kWarps, exp_args)
        : a.model == BPT_IC && a.touched
        ? add_kernel(lbody, &n_cmp, a.vmajor ? (void*)k_expand_bm<true> : (void*)k_expand_bm<false>,
                     dim3(g_expand_grid_b), dim3(kThreads),
                     a.vmajor ? sizeof(BmScratchV) * kWarps : sizeof(BmScratch) * kWarps, exp_args)
        : a.model == BPT_IC
        ? add_kernel(lbody, &n_cmp, a.colors == 64 ? (void*)k_expand_ic<true> : (void*)k_expand_ic<false>,
                     dim3(g_expand_grid), dim3(kThreads), sizeof(WarpScratch) * kWarps, exp_args)
        : add_kernel(lbody, &n_cmp, (void*)k_expand_lt, dim3(g_expand_grid_lt), dim3(kThreads), sizeof(SmemTile), exp_args);
    if (a.model == BPT_IC && a.touched && a.pull) {  // pull levels: the push kernel returns at once
        void* pull_args[] = {&args, &h_level, &one};
        add_kernel(lbody, &n_exp, (void*)k_expand_pull, dim3(g_expand_grid_p), dim3(kThreads), sizeof(BmScratch) * kWarps,
                   pull_args);
    }
    // the expansion's last block advances the level and sets the loop condition
    // finalize + count, then next batch
    cudaGraphNode_t n_store;
    add_store_nodes(body, n_level, *h.S, h.VN, a.ctl, a.slots_max, h.roff, h.d_elog, &n_store, a.wide != 0, a.touched ? (a.vmajor ? 2 : 1) : 0);
    void* nb_args[] = {&args, &h_batch, &one};
    add_kernel(body, &n_store, (void*)k_next_batch, dim3(1), dim3(256), 0, nb_args);

    cudaGraphExec_t exec;
    BPT_CUDA(cudaGraphInstantiate(&exec, root, 0));
    BPT_CUDA(cudaGraphDestroy(root));
    return exec;
}

}  // namespace bpt

#ifdef BPT_HIST
namespace bpt {
void dump_hist() {  // diagnostic build only
    unsigned long long h[16 * 80];
    cudaMemcpyFromSymbol(h, g_hist, sizeof(h));
    fprintf(stderr, "{\"hist\": [");
    for (int i = 0; i < 16 * 80; ++i) fprintf(stderr, "%s%llu", i ? "," : "", h[i]);
    fprintf(stderr, "]}\n");
    unsigned long long z[16 * 80] = {};
    cudaMemcpyToSymbol(g_hist, z, sizeof(z));
}
}  // namespace bpt
#endif
