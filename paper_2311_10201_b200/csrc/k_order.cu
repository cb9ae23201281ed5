// k_order.cu -- sorted start vertices ("sorting the starting
// vertices", P:298-313 locality / degree-based sorting): the local samples are assigned to the
// traversal slots (64-sample blocks x colour bits) in the order of their start vertices --
// in-degree descending, then start id, then sample id -- so samples whose reverse BPTs are large
// (high in-degree starts) share traversal groups, and the many samples whose start has no
// in-edge (a singleton RRR set) fill groups that finish after one level. Coins and starts stay
// keyed by the sample id (readings C-1, C-3), so every RRR set, size, digest and seed is
// unchanged; only which samples are fused together (E_phys, levels) changes.
//   slot_sample[slot] = global sample id traversed in local slot `slot` (slot = 64 * block + bit)
//   sample_slot[i]    = local slot of local sample i
// The order is a bitonic sort of (key, sample) pairs on the device (unique keys, so stable).
#include "internal.cuh"

namespace bpt {
namespace {

// key of local sample i: (~indeg(start)) << 32 | start, low 32 bits of the value = i
__global__ void k_order_keys(const uint32_t* __restrict__ roff, uint32_t n, uint64_t s0, uint64_t nlocal,
                             uint64_t npow2, uint32_t k_start, unsigned long long* __restrict__ key,
                             uint32_t* __restrict__ val) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < npow2; i += (uint64_t)gridDim.x * blockDim.x) {
        if (i < nlocal) {
            const uint64_t s = s0 + i;
            const uint2 w = philox2x32_10((uint32_t)s, (uint32_t)(s >> 32), k_start);  // reading C-3
            const uint64_t r64 = ((uint64_t)w.y << 32) | w.x;
            const uint32_t start = (uint32_t)__umul64hi(r64, (uint64_t)n);
            const uint32_t indeg = roff[start + 1] - roff[start];
            key[i] = ((unsigned long long)(~indeg) << 32) | start;
            val[i] = (uint32_t)i;
        } else {
            key[i] = ~0ull;
            val[i] = ~0u;
        }
    }
}

// one bitonic compare-exchange step over (key, val) pairs, ascending
__global__ void k_bitonic_step(unsigned long long* __restrict__ key, uint32_t* __restrict__ val, uint64_t npow2,
                               uint64_t j, uint64_t k) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < npow2; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t p = i ^ j;
        if (p <= i) continue;
        const bool up = (i & k) == 0;
        const unsigned long long ki = key[i], kp = key[p];
        const uint32_t vi = val[i], vp = val[p];
        const bool gt = ki > kp || (ki == kp && vi > vp);
        if (gt == up) {
            key[i] = kp; key[p] = ki;
            val[i] = vp; val[p] = vi;
        }
    }
}

__global__ void k_order_maps(const uint32_t* __restrict__ val, uint64_t s0, uint64_t nlocal,
                             uint32_t* __restrict__ slot_sample, uint32_t* __restrict__ sample_slot) {
    for (uint64_t slot = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; slot < nlocal;
         slot += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t i = val[slot];
        slot_sample[slot] = (uint32_t)(s0 + i);
        sample_slot[i] = (uint32_t)slot;
    }
}

}  // namespace

void sort_slots(const uint32_t* roff, uint32_t n, uint64_t s0, uint64_t nlocal, uint32_t k_start,
                uint32_t* slot_sample, uint32_t* sample_slot, cudaStream_t st) {
    if (nlocal == 0) return;
    uint64_t npow2 = 1;
    while (npow2 < nlocal) npow2 <<= 1;
    DevBuf key(npow2 * 8), val(npow2 * 4);
    const unsigned grid = (unsigned)umin64((npow2 + 255) / 256, (uint64_t)num_sms() * 8);
    k_order_keys<<<grid, 256, 0, st>>>(roff, n, s0, nlocal, npow2, k_start, key.as<unsigned long long>(),
                                       val.as<uint32_t>());
    count_launch();
    for (uint64_t k = 2; k <= npow2; k <<= 1)
        for (uint64_t j = k >> 1; j > 0; j >>= 1) {
            k_bitonic_step<<<grid, 256, 0, st>>>(key.as<unsigned long long>(), val.as<uint32_t>(), npow2, j, k);
            count_launch();
        }
    k_order_maps<<<grid, 256, 0, st>>>(val.as<uint32_t>(), s0, nlocal, slot_sample, sample_slot);
    count_launch();
    ::bpt::check_cuda(cudaGetLastError(), "launch sort_slots");
}

}  // namespace bpt
