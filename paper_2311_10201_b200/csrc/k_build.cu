// k_build.cu -- A0 validation + A1 reverse-CSR builder.
//
// The BPTs traverse the transpose (Def. 2; Listing 1's mate(e,v)).
// Canonical order (reading C-4): rows by destination v, entries in forward-CSR position
// order inside a row. That is a STABLE sort of the forward edge list by destination,
// done here as an LSD radix sort (8-bit digits; per-warp __match_any_sync ranking keeps
// it stable), then:
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
constexpr int kRsRounds = 16;                                  // 32-item rounds per warp
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

__global__ void k_iota(uint32_t* __restrict__ v, uint64_t m) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x)
        v[i] = (uint32_t)i;
}

// per-warp digit counts of one tile into smem cnt[warp][digit]
__device__ __forceinline__ void tile_warp_counts(const uint32_t* __restrict__ keys, uint64_t m, int shift,
                                                 uint32_t (*cnt)[kRadix]) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const uint64_t base = (uint64_t)blockIdx.x * kRsTile + (uint64_t)w * (32 * kRsRounds);
    for (int r = 0; r < kRsRounds; ++r) {
        uint64_t i = base + (uint64_t)r * 32 + lane;
        uint32_t d = i < m ? (keys[i] >> shift) & (kRadix - 1) : kRadix;
        uint32_t peers = __match_any_sync(0xffffffffu, d);
        if (d < kRadix && lane == __ffs(peers) - 1) cnt[w][d] += __popc(peers);
    }
}

__global__ void __launch_bounds__(kRsThreads) k_radix_hist(const uint32_t* __restrict__ keys, uint64_t m, int shift,
                                                           uint32_t* __restrict__ hist, uint64_t ntiles) {
    __shared__ uint32_t cnt[kRsWarps][kRadix];
    for (int i = threadIdx.x; i < kRsWarps * kRadix; i += kRsThreads) (&cnt[0][0])[i] = 0;
    __syncthreads();
    tile_warp_counts(keys, m, shift, cnt);
    __syncthreads();
    uint32_t s = 0;
    for (int w = 0; w < kRsWarps; ++w) s += cnt[w][threadIdx.x];
    hist[(uint64_t)threadIdx.x * ntiles + blockIdx.x] = s;  // digit-major
}

__global__ void __launch_bounds__(kRsThreads) k_radix_scatter(const uint32_t* __restrict__ keys,
                                                              const uint32_t* __restrict__ vals, uint64_t m,
                                                              int shift, const uint32_t* __restrict__ hist_scan,
                                                              uint64_t ntiles, uint32_t* __restrict__ keys_out,
                                                              uint32_t* __restrict__ vals_out) {
    __shared__ uint32_t cnt[kRsWarps][kRadix];
    for (int i = threadIdx.x; i < kRsWarps * kRadix; i += kRsThreads) (&cnt[0][0])[i] = 0;
    __syncthreads();
    tile_warp_counts(keys, m, shift, cnt);
    __syncthreads();
    {   // cnt[w][d] <- global position of warp w's first item with digit d
        const int d = threadIdx.x;
        uint32_t run = hist_scan[(uint64_t)d * ntiles + blockIdx.x];
        for (int w = 0; w < kRsWarps; ++w) { uint32_t c = cnt[w][d]; cnt[w][d] = run; run += c; }
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const uint64_t base = (uint64_t)blockIdx.x * kRsTile + (uint64_t)w * (32 * kRsRounds);
    const uint32_t lt = (1u << lane) - 1u;
    for (int r = 0; r < kRsRounds; ++r) {
        uint64_t i = base + (uint64_t)r * 32 + lane;
        uint32_t key = 0, val = 0, d = kRadix;
        if (i < m) { key = keys[i]; val = vals[i]; d = (key >> shift) & (kRadix - 1); }
        uint32_t peers = __match_any_sync(0xffffffffu, d);
        uint32_t pos = 0;
        if (d < kRadix) pos = cnt[w][d] + __popc(peers & lt);
        __syncwarp();
        if (d < kRadix && lane == __ffs(peers) - 1) cnt[w][d] += __popc(peers);
        __syncwarp();
        if (d < kRadix) { keys_out[pos] = key; vals_out[pos] = val; }
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

__device__ __forceinline__ uint32_t q31_of(const float* wf, const uint32_t* wq, uint32_t ef) {
    if (wf) return (uint32_t)floor((double)wf[ef] * 2147483648.0);  // reading C-5, exact in f64
    return wq[ef];
}

__global__ void k_gather_records(const uint32_t* __restrict__ order, const uint32_t* __restrict__ srcof,
                                 const float* __restrict__ wf, const uint32_t* __restrict__ wq, uint64_t m,
                                 uint2* __restrict__ rec) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t ef = order[i];
        rec[i] = make_uint2(srcof[ef], q31_of(wf, wq, ef));
    }
}

// LT: rec[i].y <- inclusive prefix of thr over the row (warp per row); row sum must be <= 2^31
__global__ void k_lt_prefix(const uint32_t* __restrict__ roff, uint32_t n, uint2* __restrict__ rec, BuildErr* err) {
    const int lane = threadIdx.x & 31;
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t v = warp; v < n; v += nwarps) {
        uint32_t a = roff[v], b = roff[v + 1];
        unsigned long long carry = 0;
        for (uint32_t base = a; base < b; base += 32) {
            uint32_t i = base + lane;
            unsigned long long x = i < b ? rec[i].y : 0ull;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                unsigned long long y = __shfl_up_sync(0xffffffffu, x, d);
                if (lane >= d) x += y;
            }
            unsigned long long c = carry + x;
            if (i < b) rec[i].y = c > 0xFFFFFFFFull ? 0xFFFFFFFFu : (uint32_t)c;
            carry += __shfl_sync(0xffffffffu, x, 31);
        }
        if (lane == 0 && carry > 0x80000000ull) atomicMin(&err->bad_lt, (unsigned long long)v);
    }
}

inline unsigned grid_for(uint64_t work, int threads) {
    uint64_t g = (work + threads - 1) / threads;
    uint64_t cap = (uint64_t)num_sms() * 16;
    if (g > cap) g = cap;
    return (unsigned)(g ? g : 1);
}

}  // namespace

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

    // stable LSD radix sort of (dst, forward position) by dst
    DevBuf k0(m * 4 + 4), k1(m * 4 + 4), v0(m * 4 + 4), v1(m * 4 + 4), srcof(m * 4 + 4);
    uint32_t *ka = k0.as<uint32_t>(), *kb = k1.as<uint32_t>(), *va = v0.as<uint32_t>(), *vb = v1.as<uint32_t>();
    if (m) {
        BPT_CUDA(cudaMemcpyAsync(ka, d_col, m * 4, cudaMemcpyDeviceToDevice, st));
        k_iota<<<grid_for(m, 256), 256, 0, st>>>(va, m);
        k_expand_rows<<<grid_for((uint64_t)n * 32, 256), 256, 0, st>>>(d_row_ptr, n, srcof.as<uint32_t>());
        count_launch(2);
        int bits = 0;
        while (bits < 32 && (1ull << bits) < (uint64_t)n) ++bits;
        const uint64_t ntiles = (m + kRsTile - 1) / kRsTile;
        DevBuf hist(ntiles * kRadix * 4), tmp(scan_temp_bytes(ntiles * kRadix));
        for (int shift = 0; shift < bits; shift += 8) {
            k_radix_hist<<<(unsigned)ntiles, kRsThreads, 0, st>>>(ka, m, shift, hist.as<uint32_t>(), ntiles);
            count_launch();
            exclusive_scan_u32(hist.as<uint32_t>(), hist.as<uint32_t>(), ntiles * kRadix, tmp.p, st);
            k_radix_scatter<<<(unsigned)ntiles, kRsThreads, 0, st>>>(ka, va, m, shift, hist.as<uint32_t>(), ntiles,
                                                                     kb, vb);
            count_launch();
            std::swap(ka, kb);
            std::swap(va, vb);
        }
        k_gather_records<<<grid_for(m, 256), 256, 0, st>>>(va, srcof.as<uint32_t>(), d_wf, d_wq, m,
                                                            g.rec.as<uint2>());
        count_launch();
    }
    k_row_offsets<<<grid_for((uint64_t)n + 1, 256), 256, 0, st>>>(ka, m, n, g.roff.as<uint32_t>());
    count_launch();
    ::bpt::check_cuda(cudaGetLastError(), "launch k_row_offsets");
    if (g.model == BPT_LT && m) {
        k_lt_prefix<<<grid_for((uint64_t)n * 32, 256), 256, 0, st>>>(g.roff.as<uint32_t>(), n, g.rec.as<uint2>(), err);
        count_launch();
        ::bpt::check_cuda(cudaGetLastError(), "launch k_lt_prefix");
        BPT_CUDA(cudaMemcpyAsync(&h, err, sizeof(BuildErr), cudaMemcpyDeviceToHost, st));
        BPT_CUDA(cudaStreamSynchronize(st));
        if (h.bad_lt != ~0ull)
            fail(BPT_EINVAL, "LT: sum of in-edge thresholds of vertex " + std::to_string(h.bad_lt) + " exceeds 2^31");
    }
    BPT_CUDA(cudaStreamSynchronize(st));  // temporaries are freed on return
}

}  // namespace bpt
