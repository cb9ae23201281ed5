// k_scan.cu -- device-wide exclusive prefix sum (reduce-then-scan, 3 launches).
// Used by the reverse-CSR builder (radix-sort digit offsets) and the RRR extraction.
#include "internal.cuh"

namespace bpt {
namespace {

constexpr int kScanThreads = 512;
constexpr int kScanItems = 8;
constexpr uint64_t kScanTile = (uint64_t)kScanThreads * kScanItems;

template <class T>
__device__ __forceinline__ T warp_incl_scan(T x) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        T y = __shfl_up_sync(0xffffffffu, x, d);
        if (lane >= d) x += y;
    }
    return x;
}

// block-wide exclusive scan of one value per thread; returns the block total in *total
template <class T>
__device__ __forceinline__ T block_excl_scan(T x, T* total) {
    __shared__ T warp_sums[kScanThreads / 32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    T incl = warp_incl_scan(x);
    if (lane == 31) warp_sums[w] = incl;
    __syncthreads();
    if (w == 0) {
        T s = lane < kScanThreads / 32 ? warp_sums[lane] : T(0);
        s = warp_incl_scan(s);
        if (lane < kScanThreads / 32) warp_sums[lane] = s;
    }
    __syncthreads();
    T base = w > 0 ? warp_sums[w - 1] : T(0);
    *total = warp_sums[kScanThreads / 32 - 1];
    __syncthreads();
    return base + incl - x;
}

template <class T>
__global__ void __launch_bounds__(kScanThreads) k_tile_sums(const T* __restrict__ in, uint64_t count,
                                                            T* __restrict__ sums) {
    const uint64_t base = (uint64_t)blockIdx.x * kScanTile + (uint64_t)threadIdx.x * kScanItems;
    T s = 0;
#pragma unroll
    for (int i = 0; i < kScanItems; ++i)
        if (base + i < count) s += in[base + i];
    T total;
    block_excl_scan<T>(s, &total);
    if (threadIdx.x == 0) sums[blockIdx.x] = total;
}

// single block: exclusive scan of the tile sums in place
template <class T>
__global__ void __launch_bounds__(kScanThreads) k_scan_sums(T* sums, uint64_t ntiles) {
    T carry = 0;
    for (uint64_t b = 0; b < ntiles; b += kScanThreads) {
        uint64_t i = b + threadIdx.x;
        T x = i < ntiles ? sums[i] : T(0);
        T total;
        T ex = block_excl_scan<T>(x, &total);
        if (i < ntiles) sums[i] = carry + ex;
        carry += total;
    }
}

template <class T>
__global__ void __launch_bounds__(kScanThreads) k_tile_scan(const T* in, T* out, uint64_t count,
                                                           const T* __restrict__ sums) {
    const uint64_t base = (uint64_t)blockIdx.x * kScanTile + (uint64_t)threadIdx.x * kScanItems;
    T v[kScanItems];
    T s = 0;
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
        v[i] = base + i < count ? in[base + i] : T(0);
        s += v[i];
    }
    T total;
    T ex = block_excl_scan<T>(s, &total) + sums[blockIdx.x];
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
        if (base + i < count) out[base + i] = ex;
        ex += v[i];
    }
}

template <class T>
void scan_impl(const T* in, T* out, uint64_t count, void* temp, cudaStream_t st) {
    if (count == 0) return;
    uint64_t ntiles = (count + kScanTile - 1) / kScanTile;
    T* sums = reinterpret_cast<T*>(temp);
    k_tile_sums<T><<<(unsigned)ntiles, kScanThreads, 0, st>>>(in, count, sums);
    k_scan_sums<T><<<1, kScanThreads, 0, st>>>(sums, ntiles);
    k_tile_scan<T><<<(unsigned)ntiles, kScanThreads, 0, st>>>(in, out, count, sums);
    count_launch(3);
    ::bpt::check_cuda(cudaGetLastError(), "launch k_tile_scan");
}

}  // namespace

size_t scan_temp_bytes(uint64_t count) { return ((count + kScanTile - 1) / kScanTile + 1) * sizeof(uint64_t); }

void exclusive_scan_u32(const uint32_t* in, uint32_t* out, uint64_t count, void* temp, cudaStream_t st) {
    scan_impl<uint32_t>(in, out, count, temp, st);
}
void exclusive_scan_u64(const uint64_t* in, uint64_t* out, uint64_t count, void* temp, cudaStream_t st) {
    scan_impl<uint64_t>(in, out, count, temp, st);
}

}  // namespace bpt
