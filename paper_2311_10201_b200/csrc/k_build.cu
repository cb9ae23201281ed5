// k_build.cu -- A0 validation + A1 reverse-CSR builder.
//
// The BPTs traverse the transpose (Def. 2; Listing 1's mate(e,v)).
// Canonical order (reading C-4): rows by destination v, entries in forward-CSR position
// order inside a row. That is a STABLE sort of the forward edge list by destination,
// done here as an LSD radix sort (8-bit digits; per-warp ballot ranking keeps
// it stable; the {src, thr} payload travels with the key), then:
//   roff[v]  = lower_bound(sorted destinations, v)
//   rec[i]   = {src(e_fwd), thr(e_fwd)}, thr = Q1.31 (reading C-5: floor(p * 2^31))
//   LT       : rec[i].y = inclusive prefix of thr within the row, row sum <= 2^31 (C-6)
#include "internal.cuh"

namespace bpt {

size_t scan_temp_bytes(uint64_t count);
void exclusive_scan_u32(const uint32_t* in, uint32_t* out, uint64_t count, void* temp, cudaStream_t st);

namespace {

constexpr int kRsThreads = 256;
constexpr int kRsWarps = kRsThreads / 32;
#ifndef BPT_RS_ROUNDS
#define BPT_RS_ROUNDS 12
#endif
#ifndef BPT_RS_MINB
#define BPT_RS_MINB 3
#endif
constexpr int kRsRounds = BPT_RS_ROUNDS;                       // 32-item rounds per warp
constexpr uint64_t kRsTile = (uint64_t)kRsThreads * kRsRounds; // 4096 items per tile
constexpr int kRadix = 256;

struct BuildErr {
    unsigned long long bad_row, bad_col, bad_w, bad_lt, bad_ends;
};

__global__ void k_validate_rows(const uint64_t* __restrict__ row_ptr, uint32_t n, uint64_t m, BuildErr* err) {
    for (uint64_t u = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; u < n; u += (uint64_t)gridDim.x * blockDim.x) {
        if (row_ptr[u] > row_ptr[u + 1]) atomicMin(&err->bad_row, (unsigned long long)u);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0 && (row_ptr[0] != 0 || row_ptr[n] != m))
        err->bad_ends = 1;
}

__global__ void k_validate_edges(const uint32_t* __restrict__ col, uint32_t n, uint64_t m,
                                 const float* __restrict__ wf, const uint32_t* __restrict__ wq, BuildErr* err) {
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < m; e += (uint64_t)gridDim.x * blockDim.x) {
        if (col[e] >= n) atomicMin(&err->bad_col, (unsigned long long)e);
        bool ok;
        if (wf) {
            float p = wf[e];
            ok = p >= 0.0f && p <= 1.0f;  // false for NaN
        } else {
            ok = wq[e] <= 0x80000000u;
        }
        if (!ok) atomicMin(&err->bad_w, (unsigned long long)e);
    }
}

// srcof[e] = u for every forward edge e of row u (warp per row, coalesced writes)
__global__ void k_expand_rows(const uint64_t* __restrict__ row_ptr, uint32_t n, uint32_t* __restrict__ srcof) {
    const int lane = threadIdx.x & 31;
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t u = warp; u < n; u += nwarps) {
        uint64_t a = row_ptr[u], b = row_ptr[u + 1];
        for (uint64_t e = a + lane; e < b; e += 32) srcof[e] = (uint32_t)u;
    }
}

// lanes of the warp holding the same digit d in [0, kRadix] (kRadix = past the end): nine
// ballots, a constant cost; __match_any_sync costs grow with the number of distinct values
// per warp (measured 3.6x slower on the low digits of R-MAT destinations)
__device__ __forceinline__ uint32_t digit_peers(uint32_t d) {
    uint32_t p = 0xffffffffu;
#pragma unroll
    for (int b = 0; b < 9; ++b) {
        const bool on = (d >> b) & 1u;
        const uint32_t bal = __ballot_sync(0xffffffffu, on);
        p &= on ? bal : ~bal;
    }
    return p;
}

// Per-tile digit counts need no stable ranks: one shared-memory atomic per item into the
// warp's own histogram (the ballot ranking costs ~30 instructions per 32 items)
__global__ void __launch_bounds__(kRsThreads) k_radix_hist(const uint32_t* __restrict__ keys, uint64_t m, int shift,
                                                           uint32_t* __restrict__ hist, uint64_t ntiles) {
    __shared__ uint32_t cnt[kRsWarps][kRadix];
    for (int i = threadIdx.x; i < kRsWarps * kRadix; i += kRsThreads) (&cnt[0][0])[i] = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const uint64_t base = (uint64_t)blockIdx.x * kRsTile + (uint64_t)w * (32 * kRsRounds);
    uint32_t key[kRsRounds];
#pragma unroll
    for (int r = 0; r < kRsRounds; ++r) {
        const uint64_t i = base + (uint64_t)r * 32 + lane;
        key[r] = i < m ? keys[i] : 0u;
    }
#pragma unroll
    for (int r = 0; r < kRsRounds; ++r)
        if (base + (uint64_t)r * 32 + lane < m) atomicAdd(&cnt[w][(key[r] >> shift) & (kRadix - 1)], 1u);
    __syncthreads();
    uint32_t s = 0;
    for (int q = 0; q < kRsWarps; ++q) s += cnt[q][threadIdx.x];
    hist[(uint64_t)threadIdx.x * ntiles + blockIdx.x] = s;  // digit-major
}

// One stable LSD pass over a 3072-item tile, the (src, thr) payload carried with the key so
// the sorted records need no gather through a permutation afterwards. The tile is ranked in
// registers (per-warp ballot rounds), reordered by digit in shared memory, and
// written out in that order: the items of one digit leave as one contiguous run (12 items on
// average at 8-bit digits) instead of 32 scattered 4-byte stores per warp round.
// kFirst: payload read from (srcof, weights); kLast: records written as uint2 {src, thr}.
constexpr size_t kPassSmem = (size_t)kRsTile * 12 + (size_t)kRsWarps * kRadix * 4 + kRadix * 8;

template <bool kFirst, bool kLast>
__global__ void __launch_bounds__(kRsThreads, BPT_RS_MINB) k_radix_pass(const uint32_t* __restrict__ keys,
                                                           const uint32_t* __restrict__ src,
                                                           const float* __restrict__ wf,
                                                           const uint32_t* __restrict__ wq, uint64_t m, int shift,
                                                           const uint32_t* __restrict__ hist_scan, uint64_t ntiles,
                                                           uint32_t* __restrict__ keys_out,
                                                           uint32_t* __restrict__ src_out,
                                                           uint32_t* __restrict__ w_out, uint2* __restrict__ rec_out) {
    extern __shared__ uint4 smem_raw[];
    uint32_t* sk = reinterpret_cast<uint32_t*>(smem_raw);
    uint32_t* ss = sk + kRsTile;
    uint32_t* sw = ss + kRsTile;
    uint32_t (*cnt)[kRadix] = reinterpret_cast<uint32_t (*)[kRadix]>(sw + kRsTile);
    uint32_t* toff = &cnt[kRsWarps][0];  // [kRadix] tile-local digit offsets
    uint32_t* gdel = toff + kRadix;      // [kRadix] global position - local position (mod 2^32)
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < kRsWarps * kRadix; i += kRsThreads) (&cnt[0][0])[i] = 0;
    __syncthreads();
    const uint64_t tile0 = (uint64_t)blockIdx.x * kRsTile;
    const uint64_t base = tile0 + (uint64_t)w * (32 * kRsRounds);
    const uint32_t lt = (1u << lane) - 1u;
    uint32_t key[kRsRounds], sv[kRsRounds], wv[kRsRounds], rank[kRsRounds];
#pragma unroll
    for (int r = 0; r < kRsRounds; ++r) {  // the whole tile in flight before the ranking
        const uint64_t i = base + (uint64_t)r * 32 + lane;
        key[r] = sv[r] = wv[r] = 0u;
        if (i < m) {
            key[r] = keys[i];
            sv[r] = src[i];
            wv[r] = kFirst && wf ? (uint32_t)floor((double)wf[i] * 2147483648.0) : wq[i];  // reading C-5
        }
    }
#pragma unroll
    for (int r = 0; r < kRsRounds; ++r) {
        const uint64_t i = base + (uint64_t)r * 32 + lane;
        const uint32_t d = i < m ? (key[r] >> shift) & (kRadix - 1) : kRadix;
        const uint32_t peers = digit_peers(d);
        rank[r] = 0;
        if (d < kRadix) rank[r] = cnt[w][d] + __popc(peers & lt);
        __syncwarp();
        if (d < kRadix && lane == __ffs(peers) - 1) cnt[w][d] += __popc(peers);
        __syncwarp();
    }
    __syncthreads();
    {   // thread d: tile total of digit d, exclusive scan over digits, per-warp bases
        const int d = threadIdx.x;
        uint32_t tot = 0;
        for (int q = 0; q < kRsWarps; ++q) tot += cnt[q][d];
        uint32_t x = tot;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        toff[d] = x;  // inclusive within the warp, fixed up below
        __syncthreads();
        uint32_t carry = 0;
        for (int q = 0; q < w; ++q) carry += toff[q * 32 + 31];
        __syncthreads();
        const uint32_t off = carry + x - tot;
        toff[d] = off;
        gdel[d] = hist_scan[(uint64_t)d * ntiles + blockIdx.x] - off;
        uint32_t run = off;
        for (int q = 0; q < kRsWarps; ++q) { const uint32_t c = cnt[q][d]; cnt[q][d] = run; run += c; }
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kRsRounds; ++r) {
        const uint64_t i = base + (uint64_t)r * 32 + lane;
        if (i < m) {
            const uint32_t d = (key[r] >> shift) & (kRadix - 1);
            const uint32_t lp = cnt[w][d] + rank[r];
            sk[lp] = key[r];
            ss[lp] = sv[r];
            sw[lp] = wv[r];
        }
    }
    __syncthreads();
    const uint32_t count = (uint32_t)(m - tile0 < kRsTile ? m - tile0 : kRsTile);
    for (uint32_t j = threadIdx.x; j < count; j += kRsThreads) {
        const uint32_t k = sk[j];
        const uint32_t pos = gdel[(k >> shift) & (kRadix - 1)] + j;
        if (kLast) {
            rec_out[pos] = make_uint2(ss[j], sw[j]);
            keys_out[pos] = k;
        } else {
            keys_out[pos] = k;
            src_out[pos] = ss[j];
            w_out[pos] = sw[j];
        }
    }
}

// roff[v] = first index i with sorted_dst[i] >= v, v in [0, n]
__global__ void k_row_offsets(const uint32_t* __restrict__ sorted_dst, uint64_t m, uint32_t n, uint32_t* __restrict__ roff) {
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v <= n; v += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t lo = 0, hi = m;
        while (lo < hi) {
            uint64_t mid = (lo + hi) >> 1;
            if (sorted_dst[mid] < v) lo = mid + 1; else hi = mid;
        }
        roff[v] = (uint32_t)lo;
    }
}

// LT: rec[i].y <- inclusive prefix of thr over the row, row sum must be <= 2^31 (reading C-6).
// A flat segmented scan over the sorted records (segments = equal destination keys), so
// the work is coalesced and independent of the degree distribution:
//   k_lt_scan_tiles : per 4096-item tile, in-tile segmented scan (the tile start counts as a
//                     segment head); tail[t] = local sum of the tile's last segment; checks
//                     the row sums of the segments that start inside the tile
//   k_lt_fix_tiles  : per tile, the carry of its first segment from the tiles before it
//                     (walking back while the key continues), added to that segment; checks
//                     its row sum where it ends
constexpr int kLtThreads = 256;
#ifndef BPT_LT_ROUNDS
#define BPT_LT_ROUNDS 8
#endif
constexpr int kLtRounds = BPT_LT_ROUNDS;  // consecutive items per thread (multiple of 4)
constexpr uint64_t kLtTile = (uint64_t)kLtThreads * kLtRounds;

__device__ __forceinline__ uint32_t sat32(unsigned long long x) { return x > 0xFFFFFFFFull ? 0xFFFFFFFFu : (uint32_t)x; }

__global__ void __launch_bounds__(kLtThreads) k_lt_scan_tiles(const uint32_t* __restrict__ keys, uint64_t m,
                                                              uint2* __restrict__ rec,
                                                              unsigned long long* __restrict__ tail, BuildErr* err) {
    // thread t owns the kLtRounds consecutive items i0 .. i0 + 15 (vector loads), a sequential
    // segmented scan over them, then one block-wide segmented scan of the thread aggregates
    __shared__ unsigned long long wsum[kLtThreads / 32];
    __shared__ uint32_t wflag[kLtThreads / 32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const uint64_t tile0 = (uint64_t)blockIdx.x * kLtTile;
    const uint64_t i0 = tile0 + (uint64_t)threadIdx.x * kLtRounds;
    const uint32_t key0 = keys[tile0];
    uint32_t k[kLtRounds + 1];
    uint2 r2[kLtRounds];
    if (i0 + kLtRounds <= m) {
#pragma unroll
        for (int j = 0; j < kLtRounds; j += 4) {
            const uint4 q = *reinterpret_cast<const uint4*>(keys + i0 + j);
            k[j] = q.x; k[j + 1] = q.y; k[j + 2] = q.z; k[j + 3] = q.w;
        }
#pragma unroll
        for (int j = 0; j < kLtRounds; j += 2) {
            const uint4 q = *reinterpret_cast<const uint4*>(rec + i0 + j);
            r2[j] = make_uint2(q.x, q.y); r2[j + 1] = make_uint2(q.z, q.w);
        }
    } else {
#pragma unroll
        for (int j = 0; j < kLtRounds; ++j) {
            const bool in = i0 + j < m;
            k[j] = in ? keys[i0 + j] : 0xFFFFFFFFu;
            r2[j] = in ? rec[i0 + j] : make_uint2(0u, 0u);
        }
    }
    k[kLtRounds] = i0 + kLtRounds < m ? keys[i0 + kLtRounds] : 0xFFFFFFFFu;  // for the segment-end test
    const uint32_t kprev = i0 > tile0 && i0 <= m ? keys[i0 - 1] : 0u;
    unsigned long long x[kLtRounds];
    unsigned long long run = 0;
    int first_head = kLtRounds;  // index of the first segment head among the thread's items
#pragma unroll
    for (int j = kLtRounds - 1; j >= 0; --j) {
        const uint64_t i = i0 + j;
        const bool head = i < m && (i == tile0 || k[j] != (j ? k[j - 1] : kprev));
        if (head) first_head = j;
    }
#pragma unroll
    for (int j = 0; j < kLtRounds; ++j) {
        const uint64_t i = i0 + j;
        const bool head = i < m && (i == tile0 || k[j] != (j ? k[j - 1] : kprev));
        if (head) run = 0;
        run += i < m ? r2[j].y : 0u;
        x[j] = run;
    }
    // block-wide exclusive segmented scan of (has head, run)
    uint32_t f = first_head < kLtRounds;
    unsigned long long agg = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(0xffffffffu, agg, o);
        const uint32_t fy = __shfl_up_sync(0xffffffffu, f, o);
        if (lane >= o) { if (!f) agg += y; f |= fy; }
    }
    if (lane == 31) { wsum[w] = agg; wflag[w] = f; }
    const unsigned long long ex = __shfl_up_sync(0xffffffffu, agg, 1);
    const uint32_t exf = __shfl_up_sync(0xffffffffu, f, 1);
    __syncthreads();
    unsigned long long pre = 0;  // exclusive prefix of the earlier warps
    for (int q = 0; q < w; ++q) pre = wflag[q] ? wsum[q] : pre + wsum[q];
    const unsigned long long carry = lane == 0 ? pre : (exf ? ex : pre + ex);
    const uint64_t last = (m - tile0 < kLtTile ? m : tile0 + kLtTile) - 1;
#pragma unroll
    for (int j = 0; j < kLtRounds; ++j) {
        const uint64_t i = i0 + j;
        if (j < first_head) x[j] += carry;
        if (i < m) {
            const bool end = i + 1 == m || k[j + 1] != k[j];
            if (end && k[j] != key0 && x[j] > 0x80000000ull) atomicMin(&err->bad_lt, (unsigned long long)k[j]);
            if (i == last) tail[blockIdx.x] = x[j];  // local sum of the tile's last segment
            r2[j].y = sat32(x[j]);
        }
    }
    if (i0 + kLtRounds <= m) {
#pragma unroll
        for (int j = 0; j < kLtRounds; j += 2)
            *reinterpret_cast<uint4*>(rec + i0 + j) = make_uint4(r2[j].x, r2[j].y, r2[j + 1].x, r2[j + 1].y);
    } else {
        for (int j = 0; j < kLtRounds; ++j)
            if (i0 + j < m) rec[i0 + j] = r2[j];
    }
}

__global__ void __launch_bounds__(kLtThreads) k_lt_fix_tiles(const uint32_t* __restrict__ keys, uint64_t m,
                                                             uint2* __restrict__ rec,
                                                             const unsigned long long* __restrict__ tail,
                                                             BuildErr* err) {
    __shared__ unsigned long long carry_s;
    const uint64_t t = blockIdx.x, tile0 = t * kLtTile;
    const uint64_t tile1 = m - tile0 < kLtTile ? m : tile0 + kLtTile;
    const uint32_t key0 = keys[tile0];
    if (threadIdx.x == 0) {
        unsigned long long c = 0;
        for (uint64_t q = t; q > 0; --q) {  // tile q-1 ends with key0?
            if (keys[q * kLtTile - 1] != key0) break;
            c += tail[q - 1];
            if (keys[(q - 1) * kLtTile] != key0) break;  // its last segment starts inside it
        }
        carry_s = c;
    }
    __syncthreads();
    const unsigned long long c = carry_s;
    for (uint64_t i = tile0 + threadIdx.x; i < tile1; i += kLtThreads) {
        if (keys[i] != key0) break;  // keys are sorted: the first segment is a prefix of the tile
        unsigned long long x = rec[i].y;
        if (c) { x += c; rec[i].y = sat32(x); }
        const bool end = i + 1 == m || keys[i + 1] != key0;
        if (end && x > 0x80000000ull) atomicMin(&err->bad_lt, (unsigned long long)key0);
    }
}

// Pull records: per reverse record e (row w): its source, its own index
// and its row, the sort keys / payloads that regroup the edges by source u
__global__ void k_pull_keys(const uint2* __restrict__ rec, const uint32_t* __restrict__ roff, uint32_t n, uint64_t m,
                            uint32_t* __restrict__ src, uint32_t* __restrict__ eid, uint32_t* __restrict__ row) {
    const int lane = threadIdx.x & 31;
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t w = warp; w < n; w += nwarps)
        for (uint64_t e = roff[w] + lane; e < roff[w + 1]; e += 32) {
            src[e] = rec[e].x;
            eid[e] = (uint32_t)e;
            row[e] = (uint32_t)w;
        }
}

// pull[i] = {u, w, e, thr(e)} from the records sorted by u ({e, w}) and the sorted keys (u)
__global__ void k_pull_pack(const uint32_t* __restrict__ u_sorted, const uint2* __restrict__ ew, const uint2* __restrict__ rec,
                            uint64_t m, uint4* __restrict__ pull) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint2 x = ew[i];
        pull[i] = make_uint4(u_sorted[i], x.y, x.x, rec[x.x].y);
    }
}

// Pull work list: row u of the grouped records cut into ceil(d / kPullSeg) segments
__global__ void k_seg_count(const uint32_t* __restrict__ off, uint32_t n, uint32_t* __restrict__ cnt) {
    for (uint64_t u = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; u <= n; u += (uint64_t)gridDim.x * blockDim.x)
        cnt[u] = u < n ? (off[u + 1] - off[u] + kPullSeg - 1) / kPullSeg : 0u;
}
__global__ void k_seg_write(const uint32_t* __restrict__ off, const uint32_t* __restrict__ pos, uint32_t n,
                            uint32_t* __restrict__ key, uint32_t* __restrict__ su, uint32_t* __restrict__ sst) {
    for (uint64_t u = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; u < n; u += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t a = off[u], d = off[u + 1] - a;
        for (uint32_t k = 0, p = pos[u]; k * kPullSeg < d; ++k, ++p) {
            key[p] = kPullSeg - min(kPullSeg, d - k * kPullSeg);  // longest first
            su[p] = (uint32_t)u;
            sst[p] = a + k * kPullSeg;
        }
    }
}
__global__ void k_seg_pack(const uint32_t* __restrict__ key, const uint2* __restrict__ us, uint64_t nseg,
                           uint4* __restrict__ seg) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nseg; i += (uint64_t)gridDim.x * blockDim.x)
        seg[i] = make_uint4(us[i].x, us[i].y, kPullSeg - key[i], 0u);
}

inline unsigned grid_for(uint64_t work, int threads) {
    uint64_t g = (work + threads - 1) / threads;
    uint64_t cap = (uint64_t)num_sms() * 16;
    if (g > cap) g = cap;
    return (unsigned)(g ? g : 1);
}

}  // namespace

// Stable LSD radix sort of m items by key (keys < key_bound), carrying two u32 payloads: the
// sorted records {a, b} go to rec_out, the sorted keys to keys_out (returned). b comes from wq,
// or from wf as Q1.31 thresholds (reading C-5) when wf is given.
static const uint32_t* radix_sort_records(const uint32_t* keys, const uint32_t* pa, const float* wf, const uint32_t* wq,
                                          uint64_t m, uint64_t key_bound, uint32_t* keys_out, uint2* rec_out,
                                          cudaStream_t st) {
    int bits = 0;
    while (bits < 32 && (1ull << bits) < key_bound) ++bits;
    const int passes = bits <= 8 ? 1 : (bits + 7) / 8;
    const uint64_t ntiles = (m + kRsTile - 1) / kRsTile;
    DevBuf hist(ntiles * kRadix * 4), tmp(scan_temp_bytes(ntiles * kRadix));
    DevBuf k1(m * 4 + 4), s1(m * 4 + 4), s0(m * 4 + 4), w0(m * 4 + 4), w1(m * 4 + 4);
    for (auto fn : {k_radix_pass<true, false>, k_radix_pass<false, false>, k_radix_pass<true, true>,
                    k_radix_pass<false, true>})
        BPT_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kPassSmem));
    const uint32_t* kin = keys;
    const uint32_t* sin = pa;
    const uint32_t* win = wq;
    uint32_t* sbuf[2] = {s1.as<uint32_t>(), s0.as<uint32_t>()};
    uint32_t* wbuf[2] = {w1.as<uint32_t>(), w0.as<uint32_t>()};
    for (int p = 0; p < passes; ++p) {
        const int shift = 8 * p;
        const bool first = p == 0, last = p == passes - 1;
        k_radix_hist<<<(unsigned)ntiles, kRsThreads, 0, st>>>(kin, m, shift, hist.as<uint32_t>(), ntiles);
        count_launch();
        exclusive_scan_u32(hist.as<uint32_t>(), hist.as<uint32_t>(), ntiles * kRadix, tmp.p, st);
        // keys ping-pong between k1 and keys_out so that the last pass writes keys_out
        uint32_t *ko = ((passes - 1 - p) % 2 == 0) ? keys_out : k1.as<uint32_t>(), *so = sbuf[p & 1], *wo = wbuf[p & 1];
        const float* wfi = first ? wf : nullptr;
        auto* fn = first ? (last ? k_radix_pass<true, true> : k_radix_pass<true, false>)
                         : (last ? k_radix_pass<false, true> : k_radix_pass<false, false>);
        fn<<<(unsigned)ntiles, kRsThreads, kPassSmem, st>>>(kin, sin, wfi, win, m, shift, hist.as<uint32_t>(), ntiles, ko,
                                                           so, wo, rec_out);
        count_launch();
        ::bpt::check_cuda(cudaGetLastError(), "launch k_radix_pass");
        kin = ko;
        sin = so;
        win = wo;
    }
    BPT_CUDA(cudaStreamSynchronize(st));  // temporaries are freed on return
    return kin;
}

void build_reverse_csr(Graph& g, const uint64_t* d_row_ptr, const uint32_t* d_col, const float* d_wf,
                       const uint32_t* d_wq, cudaStream_t st) {
    const uint32_t n = g.n;
    const uint64_t m = g.m;
    DevBuf err_buf(sizeof(BuildErr));
    BuildErr* err = err_buf.as<BuildErr>();
    BPT_CUDA(cudaMemsetAsync(err, 0xff, sizeof(BuildErr), st));
    BPT_CUDA(cudaMemsetAsync(&err->bad_ends, 0, sizeof(unsigned long long), st));
    k_validate_rows<<<grid_for(n, 256), 256, 0, st>>>(d_row_ptr, n, m, err);
    k_validate_edges<<<grid_for(m, 256), 256, 0, st>>>(d_col, n, m, d_wf, d_wq, err);
    count_launch(2);
    ::bpt::check_cuda(cudaGetLastError(), "launch k_validate_edges");
    BuildErr h{};
    BPT_CUDA(cudaMemcpyAsync(&h, err, sizeof(BuildErr), cudaMemcpyDeviceToHost, st));
    BPT_CUDA(cudaStreamSynchronize(st));
    if (h.bad_ends) fail(BPT_EINVAL, "row_ptr[0] must be 0 and row_ptr[n] must equal m");
    if (h.bad_row != ~0ull) fail(BPT_EINVAL, "row_ptr is decreasing at row " + std::to_string(h.bad_row));
    if (h.bad_col != ~0ull) fail(BPT_EINVAL, "col[" + std::to_string(h.bad_col) + "] >= n");
    if (h.bad_w != ~0ull)
        fail(BPT_EINVAL, std::string("weight[") + std::to_string(h.bad_w) + "] outside " +
                             (d_wf ? "[0, 1]" : "[0, 2^31]"));

    g.roff.alloc(((size_t)n + 1) * sizeof(uint32_t));
    g.rec.alloc((m ? m : 1) * sizeof(uint2));

    // stable LSD radix sort of the forward edges by dst, carrying {src, thr}
    DevBuf s0(m * 4 + 4), k2(m * 4 + 4);
    const uint32_t* sorted_keys = d_col;
    if (m) {
        k_expand_rows<<<grid_for((uint64_t)n * 32, 256), 256, 0, st>>>(d_row_ptr, n, s0.as<uint32_t>());
        count_launch();
        sorted_keys = radix_sort_records(d_col, s0.as<uint32_t>(), d_wf, d_wq, m, n, k2.as<uint32_t>(), g.rec.as<uint2>(), st);
    }
    k_row_offsets<<<grid_for((uint64_t)n + 1, 256), 256, 0, st>>>(sorted_keys, m, n, g.roff.as<uint32_t>());
    count_launch();
    ::bpt::check_cuda(cudaGetLastError(), "launch k_row_offsets");
    if (g.model == BPT_LT && m) {
        const uint64_t nt = (m + kLtTile - 1) / kLtTile;
        DevBuf tail(nt * 8);
        k_lt_scan_tiles<<<(unsigned)nt, kLtThreads, 0, st>>>(sorted_keys, m, g.rec.as<uint2>(),
                                                            tail.as<unsigned long long>(), err);
        k_lt_fix_tiles<<<(unsigned)nt, kLtThreads, 0, st>>>(sorted_keys, m, g.rec.as<uint2>(),
                                                           tail.as<unsigned long long>(), err);
        count_launch(2);
        ::bpt::check_cuda(cudaGetLastError(), "launch k_lt_fix_tiles");
        BPT_CUDA(cudaMemcpyAsync(&h, err, sizeof(BuildErr), cudaMemcpyDeviceToHost, st));
        BPT_CUDA(cudaStreamSynchronize(st));
        if (h.bad_lt != ~0ull)
            fail(BPT_EINVAL, "LT: sum of in-edge thresholds of vertex " + std::to_string(h.bad_lt) + " exceeds 2^31");
    }
    BPT_CUDA(cudaStreamSynchronize(st));  // temporaries are freed on return
}


// The forward edges regrouped by source with their canonical reverse ids (reading C-4): a stable
// radix sort of the reverse records by source u, so inside a group the edges keep reverse-CSR
// order. Built once per graph, on first use by a pull-enabled bpt_sample (Graph::pull_rec).
void build_pull_records(const Graph& g, cudaStream_t st) {
    std::lock_guard<std::mutex> lock(g.pull_mu);
    if (g.pull_rec.p || !g.m) return;
    const uint64_t m = g.m;
    DevBuf src(m * 4), eid(m * 4), row(m * 4), us(m * 4), ew(m * 8);
    k_pull_keys<<<grid_for((uint64_t)g.n * 32, 256), 256, 0, st>>>(g.rec.as<uint2>(), g.roff.as<uint32_t>(), g.n, m,
                                                                 src.as<uint32_t>(), eid.as<uint32_t>(), row.as<uint32_t>());
    count_launch();
    ::bpt::check_cuda(cudaGetLastError(), "launch k_pull_keys");
    radix_sort_records(src.as<uint32_t>(), eid.as<uint32_t>(), nullptr, row.as<uint32_t>(), m, g.n, us.as<uint32_t>(),
                       ew.as<uint2>(), st);
    DevBuf out(m * 16);
    k_pull_pack<<<grid_for(m, 256), 256, 0, st>>>(us.as<uint32_t>(), ew.as<uint2>(), g.rec.as<uint2>(), m, out.as<uint4>());
    count_launch();
    ::bpt::check_cuda(cudaGetLastError(), "launch k_pull_pack");
    // the segment work list: row offsets of the grouped records, segments per row, their positions
    const uint32_t n = g.n;
    DevBuf off(((uint64_t)n + 1) * 4), cnt(((uint64_t)n + 1) * 4), pos(((uint64_t)n + 1) * 4),
        tmp(scan_temp_bytes((uint64_t)n + 1));
    k_row_offsets<<<grid_for((uint64_t)n + 1, 256), 256, 0, st>>>(us.as<uint32_t>(), m, n, off.as<uint32_t>());
    k_seg_count<<<grid_for((uint64_t)n + 1, 256), 256, 0, st>>>(off.as<uint32_t>(), n, cnt.as<uint32_t>());
    count_launch(2);
    exclusive_scan_u32(cnt.as<uint32_t>(), pos.as<uint32_t>(), (uint64_t)n + 1, tmp.p, st);
    uint32_t nseg = 0;
    BPT_CUDA(cudaMemcpyAsync(&nseg, pos.as<uint32_t>() + n, 4, cudaMemcpyDeviceToHost, st));
    BPT_CUDA(cudaStreamSynchronize(st));
    DevBuf key(nseg * 4ull + 4), su(nseg * 4ull + 4), sst(nseg * 4ull + 4), skey(nseg * 4ull + 4), sus(nseg * 8ull + 8);
    k_seg_write<<<grid_for(n, 256), 256, 0, st>>>(off.as<uint32_t>(), pos.as<uint32_t>(), n, key.as<uint32_t>(),
                                                 su.as<uint32_t>(), sst.as<uint32_t>());
    count_launch();
    radix_sort_records(key.as<uint32_t>(), su.as<uint32_t>(), nullptr, sst.as<uint32_t>(), nseg, kPullSeg + 1,
                       skey.as<uint32_t>(), sus.as<uint2>(), st);
    DevBuf seg(nseg * 16ull + 16);
    k_seg_pack<<<grid_for(nseg, 256), 256, 0, st>>>(skey.as<uint32_t>(), sus.as<uint2>(), nseg, seg.as<uint4>());
    count_launch();
    ::bpt::check_cuda(cudaGetLastError(), "launch k_seg_pack");
    BPT_CUDA(cudaStreamSynchronize(st));
    g.pull_seg = std::move(seg);
    g.pull_nseg = nseg;
    g.pull_rec = std::move(out);
}

}  // namespace bpt
