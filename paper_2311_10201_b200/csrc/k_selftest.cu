// k_selftest.cu -- device self-tests and the integer-ALU roof of the coin (reading C-1).
//   bpt_selftest_philox: the product's own device Philox2x32-10 (internal.cuh, the function every
//     coin and start vertex goes through) evaluated on caller-given (ctr, key) triples, so the
//     Random123 known-answer vectors can be checked ON THE DEVICE.
//   bpt_bench_philox: Philox2x32-10 calls per second of the device (the co-binding ALU roof of the
//     fused expansion, SURVEY §8(d) "measure it first"): every thread evaluates a chain of
//     independent coins keyed like the expansion's (ctr = {e, s}, one stream key) and folds the
//     pass bits into a checksum so nothing is eliminated.
#include "internal.cuh"

namespace bpt {
namespace {

__global__ void k_philox_kat(const uint32_t* __restrict__ in, uint32_t* __restrict__ out, uint64_t count) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint2 r = philox2x32_10(in[3 * i], in[3 * i + 1], in[3 * i + 2]);
        out[2 * i] = r.x;
        out[2 * i + 1] = r.y;
    }
}

constexpr int kChain = 16;  // independent coins per thread per iteration (ILP, like a flattened round)

__global__ void __launch_bounds__(256) k_philox_rate(uint64_t iters, uint32_t key, uint32_t thr,
                                                     unsigned long long* __restrict__ sink) {
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t acc = 0;
    for (uint64_t it = 0; it < iters; ++it) {
#pragma unroll
        for (int c = 0; c < kChain; ++c) {
            const uint32_t e = tid * kChain + c;
            const uint32_t x = philox2x32_10(e, (uint32_t)it, key).x;
            acc += (x >> 1) < thr;
        }
    }
    if (acc == 0xffffffffu) atomicAdd(sink, 1ull);  // never true; keeps the chain live
    if (threadIdx.x == 0 && blockIdx.x == 0) atomicAdd(sink + 1, (unsigned long long)acc);
}

}  // namespace

void selftest_philox(const uint32_t* d_in, uint32_t* d_out, uint64_t count, cudaStream_t st) {
    if (!count) return;
    const unsigned grid = (unsigned)umin64((count + 255) / 256, 1024);
    k_philox_kat<<<grid, 256, 0, st>>>(d_in, d_out, count);
    count_launch();
    ::bpt::check_cuda(cudaGetLastError(), "launch k_philox_kat");
}

double bench_philox(uint64_t iters, uint64_t* calls_out, cudaStream_t st) {
    const int sms = num_sms();
    int per_sm = 0;
    BPT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_philox_rate, 256, 0));
    const unsigned grid = (unsigned)(sms * (per_sm > 0 ? per_sm : 1));
    DevBuf sink(16);
    BPT_CUDA(cudaMemsetAsync(sink.p, 0, 16, st));
    cudaEvent_t e0, e1;
    BPT_CUDA(cudaEventCreate(&e0));
    BPT_CUDA(cudaEventCreate(&e1));
    k_philox_rate<<<grid, 256, 0, st>>>(2, 0x1234567u, 1u << 30, sink.as<unsigned long long>());  // warm-up
    BPT_CUDA(cudaEventRecord(e0, st));
    k_philox_rate<<<grid, 256, 0, st>>>(iters, 0x1234567u, 1u << 30, sink.as<unsigned long long>());
    BPT_CUDA(cudaEventRecord(e1, st));
    count_launch(2);
    ::bpt::check_cuda(cudaGetLastError(), "launch k_philox_rate");
    BPT_CUDA(cudaEventSynchronize(e1));
    float ms = 0;
    BPT_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    *calls_out = (uint64_t)grid * 256 * kChain * iters;
    return ms;
}

}  // namespace bpt
