// Micro-benchmark (not part of the product): random 16-B gathers from a table of S bytes,
// the access pattern of the expansion's {V,N}[u] reads. Prints G gathers/s per configuration.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void k_gather(const uint32_t* __restrict__ idx, const ulonglong2* __restrict__ tab, uint64_t n_idx,
                         unsigned long long* out, int mode) {
    unsigned long long acc = 0;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n_idx; i += 3 * stride) {
        uint32_t j0 = idx[i], j1 = i + stride < n_idx ? idx[i + stride] : 0, j2 = i + 2 * stride < n_idx ? idx[i + 2 * stride] : 0;
        ulonglong2 a, b, c;
        if (mode == 0) { a = tab[j0]; b = tab[j1]; c = tab[j2]; }
        else {
            asm volatile("ld.global.nc.L1::no_allocate.v2.u64 {%0,%1}, [%2];" : "=l"(a.x), "=l"(a.y) : "l"(tab + j0));
            asm volatile("ld.global.nc.L1::no_allocate.v2.u64 {%0,%1}, [%2];" : "=l"(b.x), "=l"(b.y) : "l"(tab + j1));
            asm volatile("ld.global.nc.L1::no_allocate.v2.u64 {%0,%1}, [%2];" : "=l"(c.x), "=l"(c.y) : "l"(tab + j2));
        }
        acc += a.x ^ b.y ^ c.x;
    }
    if (acc == 0x123456789ull) out[0] = acc;
}

int main() {
    const uint64_t n_idx = 1ull << 27;  // 134M gathers
    uint32_t* idx; ulonglong2* tab; unsigned long long* out;
    const uint64_t max_entries = (1ull << 30) / 16;  // up to 1 GB table
    cudaMalloc(&idx, n_idx * 4); cudaMalloc(&tab, max_entries * 16); cudaMalloc(&out, 8);
    cudaMemset(tab, 1, max_entries * 16);
    uint32_t* h = new uint32_t[n_idx];
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (uint64_t mb : {8ull, 32ull, 78ull, 128ull, 512ull, 1024ull}) {
        const uint64_t ent = mb * (1ull << 20) / 16;
        uint64_t x = 88172645463325252ull;
        for (uint64_t i = 0; i < n_idx; ++i) { x ^= x << 13; x ^= x >> 7; x ^= x << 17; h[i] = (uint32_t)(x % ent); }
        cudaMemcpy(idx, h, n_idx * 4, cudaMemcpyHostToDevice);
        for (int mode = 0; mode < 2; ++mode)
        for (int bps : {2, 4, 5, 6, 8}) {
            const int grid = sms * bps;
            k_gather<<<grid, 256>>>(idx, tab, n_idx, out, mode);
            cudaEventRecord(e0);
            for (int r = 0; r < 3; ++r) k_gather<<<grid, 256>>>(idx, tab, n_idx, out, mode);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            printf("table %5llu MB mode %d blocks/SM %d: %.1f G gathers/s\n", (unsigned long long)mb, mode, bps, 3.0 * n_idx / (ms * 1e-3) / 1e9);
        }
    }
    return 0;
}
