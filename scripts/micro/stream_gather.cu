// Micro-benchmark (not part of the product): the expansion's memory pattern without its
// arithmetic -- a coalesced stream of 8-B edge records {u, thr} (552 MB, C2-sized) and, per
// record, a dependent random 16-B gather of {V,N}[u] from a 78 MB table. Prints G records/s.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t pol_first() { uint64_t p; asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p)); return p; }
__device__ __forceinline__ uint64_t pol_last() { uint64_t p; asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p)); return p; }

template <int W, int RECMODE, int VNMODE>
__global__ void k(const uint2* __restrict__ rec, const ulonglong2* __restrict__ tab, uint64_t m, unsigned long long* out) {
    unsigned long long acc = 0;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i0 = blockIdx.x * (uint64_t)blockDim.x * W + threadIdx.x; i0 < m; i0 += stride * W) {
        uint2 r[W];
#pragma unroll
        for (int w = 0; w < W; ++w) {
            const uint64_t i = i0 + (uint64_t)w * blockDim.x;
            const uint2* p = rec + (i < m ? i : 0);
            if (RECMODE == 0) r[w] = *p;
            else asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.u32 {%0,%1}, [%2], %3;" : "=r"(r[w].x), "=r"(r[w].y) : "l"(p), "l"(pol_first()));
        }
#pragma unroll
        for (int w = 0; w < W; ++w) {
            ulonglong2 v;
            const ulonglong2* p = tab + r[w].x;
            if (VNMODE == 0) v = *p;
            else asm volatile("ld.global.nc.L2::cache_hint.v2.u64 {%0,%1}, [%2], %3;" : "=l"(v.x), "=l"(v.y) : "l"(p), "l"(pol_last()));
            acc += (v.x ^ v.y) + r[w].y;
        }
    }
    if (acc == 0x123456789ull) out[0] = acc;
}

template <int W, int RM, int VM>
void run(const uint2* rec, const ulonglong2* tab, uint64_t m, unsigned long long* out, int sms) {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaFuncSetAttribute(k<W, RM, VM>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    for (int smem_kb : {0, 16, 33, 40}) for (int bps : {4, 5}) {
        const size_t sm = (size_t)smem_kb * 1024;
        k<W, RM, VM><<<sms * bps, 256, sm>>>(rec, tab, m, out);
        cudaEventRecord(e0);
        for (int rr = 0; rr < 3; ++rr) k<W, RM, VM><<<sms * bps, 256, sm>>>(rec, tab, m, out);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        printf("W=%d rec%d vn%d blocks/SM %d smem %d KB/block: %.1f G records/s\n", W, RM, VM, bps, smem_kb, 3.0 * m / (ms * 1e-3) / 1e9);
    }
}

#include <cmath>
int main(int argc, char** argv) {
    const double skew = argc > 1 ? atof(argv[1]) : 1.0;  // u = n * r^skew (skew > 1: hub-heavy)
    const uint64_t m = 69000000, n = 4850000;
    uint2* rec; ulonglong2* tab; unsigned long long* out;
    cudaMalloc(&rec, m * 8); cudaMalloc(&tab, n * 16); cudaMalloc(&out, 8);
    cudaMemset(tab, 1, n * 16);
    uint2* h = new uint2[m];
    uint64_t x = 88172645463325252ull;
    for (uint64_t i = 0; i < m; ++i) { x ^= x << 13; x ^= x >> 7; x ^= x << 17; const double r = (double)(x >> 11) / 9007199254740992.0; h[i] = make_uint2((uint32_t)fmin((double)(n - 1), n * pow(r, skew)), (uint32_t)x); }
    if (argc > 2) {  // real reverse-CSR sources (u32 per edge, in reverse-CSR order)
        FILE* f = fopen(argv[2], "rb");
        uint32_t* src = new uint32_t[m];
        const size_t got = fread(src, 4, m, f);
        fclose(f);
        for (uint64_t i = 0; i < m; ++i) h[i].x = src[i % got] % n;
        printf("real sources from %s (%zu)\n", argv[2], got);
    }
    cudaMemcpy(rec, h, m * 8, cudaMemcpyHostToDevice);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    printf("skew %.1f\n", skew);
    run<3, 1, 1>(rec, tab, m, out, sms);
    return 0;
}
