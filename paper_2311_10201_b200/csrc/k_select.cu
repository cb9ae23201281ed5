// k_select.cu -- A7 greedy max-k-cover seed selection over the fused RRR store.
//
// State (device): count[v] = uncovered samples containing v (this rank's; with W > 1 ranks and a
// dense store the GLOBAL count, see below); cov[g] = covered samples of local 64-sample block g;
// selected[v].
// Round r:  (1) key[v] = selected ? 0 : count[v] << 32 | ~v   (max gain, smallest id, reading C-11)
//           multi-rank dense stores: the counts are AllReduce'd once, every
//           rank takes the same argmax, round 0's decrements are AllReduce'd densely and later
//           rounds' (few covered samples) are exchanged as AllGathered (vertex, decrement) pairs;
//           if a rank's pairs overflow, the selection is redone with the per-round ReduceScatter of
//           the counts and AllReduce(max) of the per-rank maxima.
//           (2) new_g = V_g[v*] & ~cov_g ; cov_g |= new_g ; list the blocks with new_g != 0
//           (3) count[v] -= sum over listed g of popcount(V_g[v] & new_g)
// Each sample leaves `count` exactly once, so the decrements over all rounds cost at most one
// pass over the store plus the few blocks touched by later rounds.
// Member-list stores (LT): the same greedy through a vertex -> samples index; with W > 1 ranks
// every rank gathers all ranks' lists once (AllGather) and runs the rounds
// locally, so the k rounds need no collective at all.
#include <chrono>
#include <cstdio>
#include <cstdlib>

#include "internal.cuh"

namespace bpt {

size_t scan_temp_bytes(uint64_t count);
void exclusive_scan_u64(const uint64_t* in, uint64_t* out, uint64_t count, void* temp, cudaStream_t st);
void comm_reduce_scatter_u32(Comm* c, const uint32_t* send, uint32_t* recv, uint64_t recv_count, cudaStream_t st);
void comm_allreduce_max_u64(Comm* c, unsigned long long* buf, uint64_t count, cudaStream_t st);
void comm_allreduce_sum_u32(Comm* c, uint32_t* buf, uint64_t count, cudaStream_t st);
void comm_allgather_u32(Comm* c, const uint32_t* send, uint32_t* recv, uint64_t count, cudaStream_t st);
void comm_allgather_u64(Comm* c, const uint64_t* send, uint64_t* recv, uint64_t count, cudaStream_t st);

namespace {

constexpr int kSelThreads = 512;

__global__ void __launch_bounds__(kSelThreads) k_argmax(const uint32_t* __restrict__ count, uint64_t len, uint64_t vbase,
                                                        uint32_t n, const uint8_t* __restrict__ selected,
                                                        unsigned long long* __restrict__ key_out,
                                                        uint32_t* __restrict__ nlist) {
    if (blockIdx.x == 0 && threadIdx.x == 0) *nlist = 0;
    unsigned long long best = 0;
    // four vertices per thread: one 16-B load of counts, one 4-B load of selected flags
    // (vbase is a multiple of 64; count and selected are padded to a multiple of 4)
    const uint4* c4 = reinterpret_cast<const uint4*>(count);
    const uint32_t* s4 = reinterpret_cast<const uint32_t*>(selected + vbase);
    for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; 4 * q < len; q += (uint64_t)gridDim.x * blockDim.x) {
        const uint4 c = c4[q];
        const uint32_t sl = s4[q];
        const uint32_t cv[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const uint64_t v = vbase + 4 * q + e;
            if (v >= n || 4 * q + e >= len || ((sl >> (8 * e)) & 0xffu)) continue;
            const unsigned long long k = ((unsigned long long)cv[e] << 32) | (unsigned long long)(~(uint32_t)v);
            best = k > best ? k : best;
        }
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
        unsigned long long o = __shfl_xor_sync(0xffffffffu, best, d);
        best = o > best ? o : best;
    }
    __shared__ unsigned long long wb[kSelThreads / 32];
    if ((threadIdx.x & 31) == 0) wb[threadIdx.x >> 5] = best;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < kSelThreads / 32; ++w) best = wb[w] > best ? wb[w] : best;
        if (best) atomicMax(key_out, best);
    }
}

__global__ void k_cover(const uint64_t* __restrict__ store, uint32_t n, uint64_t blocks,
                        const unsigned long long* __restrict__ key, uint64_t* __restrict__ cov,
                        uint8_t* __restrict__ selected, uint32_t* __restrict__ nlist, uint32_t* __restrict__ list,
                        uint64_t* __restrict__ newm) {
    const uint32_t vstar = ~(uint32_t)(*key);
    if (blockIdx.x == 0 && threadIdx.x == 0) selected[vstar] = 1;
    for (uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; g < blocks; g += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t nw = store[(size_t)g * n + vstar] & ~cov[g];
        if (nw) {
            cov[g] |= nw;
            const uint32_t i = atomicAdd(nlist, 1u);
            list[i] = (uint32_t)g;
            newm[i] = nw;
        }
    }
}

__global__ void k_decrement(const uint64_t* __restrict__ store, uint32_t n, const uint32_t* __restrict__ nlist,
                            const uint32_t* __restrict__ list, const uint64_t* __restrict__ newm,
                            uint32_t* __restrict__ count) {
    const uint32_t L = *nlist;
    if (L == 0) return;
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n; v += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t d = 0;
        for (uint32_t i = 0; i < L; ++i) d += __popcll(store[(size_t)list[i] * n + v] & newm[i]);
        if (d) count[v] -= d;
    }
}

// Multi-rank dense stores, rounds >= 1: every rank keeps the GLOBAL counts,
// so the argmax needs no collective; a round's decrements are sparse after round 0 (the later
// seeds cover few samples), so each rank lists its nonzero decrements as (v | d << 32) pairs
// (warp-aggregated appends, at most cap; more sets *overflow and the selection is redone with the
// per-round ReduceScatter) and the pairs of all ranks are AllGathered and applied.
__global__ void k_decrement_pairs(const uint64_t* __restrict__ store, uint32_t n, const uint32_t* __restrict__ nlist,
                                  const uint32_t* __restrict__ list, const uint64_t* __restrict__ newm,
                                  unsigned long long* __restrict__ pairs, uint32_t cap, uint32_t* __restrict__ npairs,
                                  uint32_t* __restrict__ overflow) {
    const uint32_t L = *nlist;
    if (L == 0) return;
    const int lane = threadIdx.x & 31;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t v0 = blockIdx.x * (uint64_t)blockDim.x; v0 < n; v0 += stride) {  // whole warps per pass
        const uint64_t v = v0 + threadIdx.x;
        uint32_t d = 0;
        if (v < n)
            for (uint32_t i = 0; i < L; ++i) d += __popcll(store[(size_t)list[i] * n + v] & newm[i]);
        const uint32_t bal = __ballot_sync(0xffffffffu, d != 0);
        if (!bal) continue;
        uint32_t base = 0;
        if (lane == __ffs(bal) - 1) base = atomicAdd(npairs, (uint32_t)__popc(bal));
        base = __shfl_sync(0xffffffffu, base, __ffs(bal) - 1);
        if (d) {
            const uint32_t pos = base + __popc(bal & ((1u << lane) - 1u));
            if (pos < cap) pairs[pos] = (unsigned long long)v | ((unsigned long long)d << 32);
            else *overflow = 1;
        }
    }
}

__global__ void k_apply_pairs(const unsigned long long* __restrict__ pairs, uint64_t total, uint32_t* __restrict__ count) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total; i += (uint64_t)gridDim.x * blockDim.x) {
        const unsigned long long p = pairs[i];
        if (p != ~0ull) atomicSub(&count[(uint32_t)p], (uint32_t)(p >> 32));
    }
}

__global__ void k_widen_flag(const uint32_t* __restrict__ flag, unsigned long long* __restrict__ out) {
    if (threadIdx.x == 0) *out = *flag ? 1ull : 0ull;
}

__global__ void k_add_u32(uint32_t* __restrict__ a, const uint32_t* __restrict__ b, uint64_t len) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < len; i += (uint64_t)gridDim.x * blockDim.x) a[i] += b[i];
}

// sparse stores (e.g. LT): decrement through the members of the newly covered samples,
// read from their extracted RRR lists (one block per listed 64-sample block)
__global__ void k_decrement_lists(const uint32_t* __restrict__ nlist, const uint32_t* __restrict__ list,
                                  const uint64_t* __restrict__ newm, const uint64_t* __restrict__ off,
                                  const uint32_t* __restrict__ members, uint64_t nlocal,
                                  uint32_t* __restrict__ count) {
    const uint32_t L = *nlist;
    for (uint32_t i = blockIdx.x; i < L; i += gridDim.x) {
        uint64_t m = newm[i];
        const uint64_t base = 64ull * list[i];
        while (m) {
            const uint32_t c = __ffsll((long long)m) - 1;
            m &= m - 1;
            const uint64_t s = base + c;
            if (s >= nlocal) break;
            for (uint64_t j = off[s] + threadIdx.x; j < off[s + 1]; j += blockDim.x) atomicSub(&count[members[j]], 1u);
        }
    }
}

// One pass over the store: every set bit (block g, vertex v, colour c) appends v to the list of
// sample 64 g + c through that sample's cursor. Lists come out unsorted -- the selection's
// decrement only needs the member sets (bpt_rrr_extract has its own ordered path).
__global__ void k_lists_scatter(const uint64_t* __restrict__ store, uint32_t n, uint64_t blocks, uint64_t nlocal,
                                const uint64_t* __restrict__ off, uint32_t* __restrict__ cursor,
                                uint32_t* __restrict__ members) {
    for (uint64_t g = blockIdx.y; g < blocks; g += gridDim.y) {
        const uint64_t* V = store + g * n;
        for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
            uint64_t m = V[v];
            while (m) {
                const uint32_t c = __ffsll((long long)m) - 1;
                m &= m - 1;
                const uint64_t s = 64 * g + c;
                if (s >= nlocal) break;
                members[off[s] + atomicAdd(&cursor[s], 1u)] = v;
            }
        }
    }
}

__global__ void k_widen_u32(const uint32_t* __restrict__ in, uint64_t* __restrict__ out, uint64_t count) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count; i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = in[i];
}

// sparse store: vertex -> local samples index (inv_off = exclusive scan of the occurrence counts)
__global__ void k_inv_scatter(const uint64_t* __restrict__ off, const uint32_t* __restrict__ members, uint64_t nlists,
                              const uint64_t* __restrict__ inv_off, uint32_t* __restrict__ cursor,
                              uint32_t* __restrict__ inv_s) {
    const int lane = threadIdx.x & 31;  // one warp per list, lanes over its members
    for (uint64_t l = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; l < nlists;
         l += ((uint64_t)gridDim.x * blockDim.x) >> 5)
        for (uint64_t j = off[l] + lane; j < off[l + 1]; j += 32) {
            const uint32_t w = members[j];
            inv_s[inv_off[w] + atomicAdd(&cursor[w], 1u)] = (uint32_t)l;
        }
}

// sparse store, one round: the samples containing v* that are not covered yet become covered
// and leave the counts of all their members
__global__ void k_cover_sparse(const unsigned long long* __restrict__ key, const uint64_t* __restrict__ inv_off,
                               const uint32_t* __restrict__ inv_s, const uint64_t* __restrict__ off,
                               const uint32_t* __restrict__ members, uint32_t* __restrict__ covered,
                               uint8_t* __restrict__ selected, uint32_t* __restrict__ count) {
    const uint32_t vstar = ~(uint32_t)(*key);
    if (blockIdx.x == 0 && threadIdx.x == 0) selected[vstar] = 1;
    if (*key == 0) return;  // no gain left on any rank's shard: nothing to cover
    const uint64_t b = inv_off[vstar], e = inv_off[vstar + 1];
    const int lane = threadIdx.x & 31;  // one warp per sample containing v*, lanes over its members
    for (uint64_t j = b + ((blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5); j < e;
         j += ((uint64_t)gridDim.x * blockDim.x) >> 5) {
        const uint32_t l = inv_s[j];
        uint32_t was = 0;
        if (lane == 0) was = atomicExch(&covered[l], 1u);
        if (__shfl_sync(0xffffffffu, was, 0)) continue;
        for (uint64_t t = off[l] + lane; t < off[l + 1]; t += 32) atomicSub(&count[members[t]], 1u);
    }
}

}  // namespace

// Member lists of all local samples, if they are small enough to keep (sparse stores); cached.
static bool build_lists(const Samples& S, cudaStream_t st) {
    if (S.lists_built) return S.lists_ok;
    Samples& M = const_cast<Samples&>(S);
    M.lists_built = true;
    const uint64_t nlocal = S.s1 - S.s0;
    const uint64_t bytes = S.info.members * 4 + (nlocal + 1) * 8;
    const size_t free_b = free_estimate() + cached_bytes();
    // lists pay off when they are much smaller than one pass over the store
    if (nlocal == 0 || bytes > free_b / 4 || bytes * 8 > S.store.bytes) return M.lists_ok = false;
    std::vector<uint32_t> sz(nlocal);
    ensure_sizes(M, S.s0, nlocal, st);
    BPT_CUDA(cudaStreamSynchronize(st));
    BPT_CUDA(cudaMemcpy(sz.data(), S.sizes.p, nlocal * 4, cudaMemcpyDeviceToHost));
    if (S.sorted) {  // the lists follow the store: one per slot (the slot's sample's size)
        std::vector<uint32_t> slot_sample(nlocal), by_slot(nlocal);
        BPT_CUDA(cudaMemcpy(slot_sample.data(), S.slot_sample.p, nlocal * 4, cudaMemcpyDeviceToHost));
        for (uint64_t j = 0; j < nlocal; ++j) by_slot[j] = sz[slot_sample[j] - S.s0];
        sz.swap(by_slot);
    }
    std::vector<uint64_t> off(nlocal + 1, 0);
    for (uint64_t i = 0; i < nlocal; ++i) off[i + 1] = off[i] + sz[i];
    M.list_off.alloc((nlocal + 1) * 8);
    M.list_mem.alloc(off[nlocal] * 4 + 4);
    BPT_CUDA(cudaMemcpyAsync(M.list_off.p, off.data(), (nlocal + 1) * 8, cudaMemcpyHostToDevice, st));
    if (off[nlocal]) {
        DevBuf cursor(nlocal * 4);
        BPT_CUDA(cudaMemsetAsync(cursor.p, 0, nlocal * 4, st));
        const dim3 grid((unsigned)umin64((S.n + 255) / 256, 64), (unsigned)umin64(S.blocks, (uint64_t)num_sms() * 4));
        k_lists_scatter<<<grid, 256, 0, st>>>(S.store.as<uint64_t>(), S.n, S.blocks, nlocal,
                                                       M.list_off.as<uint64_t>(), cursor.as<uint32_t>(),
                                                       M.list_mem.as<uint32_t>());
        count_launch();
        ::bpt::check_cuda(cudaGetLastError(), "launch k_lists_scatter");
        BPT_CUDA(cudaStreamSynchronize(st));
    }
    BPT_CUDA(cudaStreamSynchronize(st));
    return M.lists_ok = true;
}

// Sparse stores (member lists, e.g. LT): the selection index over a list collection -- the
// vertex -> samples inverted index and, per round, the samples containing v* leave the counts of
// all their members (each sample leaves once: total work = one pass over the lists).
struct ListIndex {
    const uint64_t* off = nullptr;   // [nlists + 1]
    const uint32_t* mem = nullptr;
    uint64_t nlists = 0;
    const uint32_t* count0 = nullptr;  // occurrences over these lists, [n_pad]
};

static void build_inverted(Samples& M, const ListIndex& L, uint32_t n, cudaStream_t st) {
    M.inv_off.alloc((uint64_t)(n + 1) * 8);
    DevBuf wide((uint64_t)(n + 1) * 8), temp(scan_temp_bytes(n + 1));
    BPT_CUDA(cudaMemsetAsync(wide.p, 0, wide.bytes, st));
    k_widen_u32<<<num_sms() * 4, 256, 0, st>>>(L.count0, wide.as<uint64_t>(), n);
    exclusive_scan_u64(wide.as<uint64_t>(), M.inv_off.as<uint64_t>(), n + 1, temp.p, st);
    count_launch();
    uint64_t total = 0;
    BPT_CUDA(cudaMemcpyAsync(&total, M.inv_off.as<uint64_t>() + n, 8, cudaMemcpyDeviceToHost, st));
    BPT_CUDA(cudaStreamSynchronize(st));
    M.inv_s.alloc(total * 4 + 4);
    DevBuf cursor((uint64_t)n * 4);
    BPT_CUDA(cudaMemsetAsync(cursor.p, 0, cursor.bytes, st));
    const unsigned g = (unsigned)umin64((L.nlists * 32 + 255) / 256, (uint64_t)num_sms() * 16);
    if (g) k_inv_scatter<<<g, 256, 0, st>>>(L.off, L.mem, L.nlists, M.inv_off.as<uint64_t>(), cursor.as<uint32_t>(),
                                            M.inv_s.as<uint32_t>());
    count_launch();
    ::bpt::check_cuda(cudaGetLastError(), "launch k_inv_scatter");
    BPT_CUDA(cudaStreamSynchronize(st));
}

// Multi-rank sparse store: every rank gathers all ranks' member lists once (one AllGather of the
// list sizes and one of the members) and then runs the whole greedy
// locally -- no collective per round; every rank computes the same seeds from the same data.
static void gather_lists(Samples& M, cudaStream_t st) {
    Comm* c = M.comm;
    const int W = c->world;
    const uint64_t nlocal = M.s1 - M.s0;
    const uint64_t total = M.info.members;
    DevBuf hdr(16), hdr_all((uint64_t)W * 16);
    const uint64_t mine[2] = {nlocal, total};
    BPT_CUDA(cudaMemcpyAsync(hdr.p, mine, 16, cudaMemcpyHostToDevice, st));
    comm_allgather_u64(c, hdr.as<uint64_t>(), hdr_all.as<uint64_t>(), 2, st);
    std::vector<uint64_t> h((size_t)W * 2);
    BPT_CUDA(cudaMemcpyAsync(h.data(), hdr_all.p, (size_t)W * 16, cudaMemcpyDeviceToHost, st));
    BPT_CUDA(cudaStreamSynchronize(st));
    uint64_t max_n = 1, max_t = 1;
    for (int r = 0; r < W; ++r) { max_n = umax64(max_n, h[2 * r]); max_t = umax64(max_t, h[2 * r + 1]); }
    // local sizes and members, padded to the largest rank's
    DevBuf sz(max_n * 4), mem(max_t * 4), sz_all((uint64_t)W * max_n * 4), mem_all((uint64_t)W * max_t * 4);
    BPT_CUDA(cudaMemsetAsync(sz.p, 0, sz.bytes, st));
    if (nlocal) BPT_CUDA(cudaMemcpyAsync(sz.p, M.sizes.p, nlocal * 4, cudaMemcpyDeviceToDevice, st));
    if (total) BPT_CUDA(cudaMemcpyAsync(mem.p, M.list_mem.p, total * 4, cudaMemcpyDeviceToDevice, st));
    comm_allgather_u32(c, sz.as<uint32_t>(), sz_all.as<uint32_t>(), max_n, st);
    comm_allgather_u32(c, mem.as<uint32_t>(), mem_all.as<uint32_t>(), max_t, st);
    // drop the padding: rank r's members (gathered at r * max_t) move to one contiguous array
    uint64_t tall = 0;
    for (int r = 0; r < W; ++r) tall += h[2 * r + 1];
    M.g_mem.alloc(tall * 4 + 4);
    for (int r = 0; r < W; ++r) {
        uint64_t before = 0;
        for (int q = 0; q < r; ++q) before += h[2 * q + 1];
        if (h[2 * r + 1])
            BPT_CUDA(cudaMemcpyAsync(M.g_mem.as<uint32_t>() + before, mem_all.as<uint32_t>() + (uint64_t)r * max_t,
                                     h[2 * r + 1] * 4, cudaMemcpyDeviceToDevice, st));
    }
    // global list offsets over all ranks' samples, in rank order
    std::vector<uint32_t> hs((size_t)W * max_n);
    BPT_CUDA(cudaMemcpyAsync(hs.data(), sz_all.p, hs.size() * 4, cudaMemcpyDeviceToHost, st));
    BPT_CUDA(cudaStreamSynchronize(st));
    uint64_t nall = 0;
    for (int r = 0; r < W; ++r) nall += h[2 * r];
    std::vector<uint64_t> off(nall + 1);
    uint64_t i = 0, o = 0;
    for (int r = 0; r < W; ++r)
        for (uint64_t j = 0; j < h[2 * r]; ++j) { off[i++] = o; o += hs[(size_t)r * max_n + j]; }
    off[nall] = o;
    M.g_off.alloc((nall + 1) * 8);
    BPT_CUDA(cudaMemcpyAsync(M.g_off.p, off.data(), (nall + 1) * 8, cudaMemcpyHostToDevice, st));
    M.g_n = nall;
    // occurrences over all ranks' samples
    M.g_count0.alloc((uint64_t)M.n_pad * 4);
    BPT_CUDA(cudaMemcpyAsync(M.g_count0.p, M.count0.p, (uint64_t)M.n_pad * 4, cudaMemcpyDeviceToDevice, st));
    comm_allreduce_sum_u32(c, M.g_count0.as<uint32_t>(), M.n_pad, st);
    BPT_CUDA(cudaStreamSynchronize(st));
}

static void select_rounds(const Samples& S, uint32_t k, uint32_t* h_seeds, uint64_t* h_gains, cudaStream_t st,
                          bool pair_exchange, bool* overflowed);

void select_seeds(const Samples& S, uint32_t k, uint32_t* h_seeds, uint64_t* h_gains, cudaStream_t st) {
    const int world = S.comm ? S.comm->world : 1;
    bool ovf = false;
    // multi-rank dense stores: global counts + sparse decrement exchange; if any rank's decrements of
    // some round outgrew the pair buffer, every rank redoes the selection with the per-round ReduceScatter
    select_rounds(S, k, h_seeds, h_gains, st, world > 1 && !S.sparse, &ovf);
    if (ovf) select_rounds(S, k, h_seeds, h_gains, st, false, &ovf);
}

static void select_rounds(const Samples& S, uint32_t k, uint32_t* h_seeds, uint64_t* h_gains, cudaStream_t st,
                          bool pair_exchange, bool* overflowed) {
    *overflowed = false;
    const uint32_t n = S.n;
    Comm* comm = S.comm;
    const int world = comm ? comm->world : 1, rank = comm ? comm->rank : 0;
    const uint64_t blocks = S.blocks;
    DevBuf count((uint64_t)S.n_pad * 4), shard(world > 1 ? (uint64_t)S.n_pad / world * 4 : 4), sel(S.n_pad),
        cov(blocks * 8 + 8), list(blocks * 4 + 4), newm(blocks * 8 + 8), nlist(4), keys((uint64_t)k * 8);
    BPT_CUDA(cudaMemcpyAsync(count.p, S.count0.p, (uint64_t)S.n_pad * 4, cudaMemcpyDeviceToDevice, st));
    BPT_CUDA(cudaMemsetAsync(sel.p, 0, S.n_pad, st));
    BPT_CUDA(cudaMemsetAsync(cov.p, 0, blocks * 8 + 8, st));
    BPT_CUDA(cudaMemsetAsync(keys.p, 0, (uint64_t)k * 8, st));
    const unsigned vgrid = (unsigned)umin64(((uint64_t)n + 4 * kSelThreads - 1) / (4 * kSelThreads), (uint64_t)num_sms() * 4);
    // >= 1 block: a rank without local blocks still marks v* selected (and joins every collective)
    const unsigned ggrid = (unsigned)umax64(1, umin64((blocks + 255) / 256, (uint64_t)num_sms() * 4));
    const unsigned dgrid = (unsigned)umin64(((uint64_t)n + 255) / 256, (uint64_t)num_sms() * 8);
    const uint64_t shard_len = (uint64_t)S.n_pad / world;
    using clk = std::chrono::steady_clock;
    const auto t0 = clk::now();
    const bool lists = build_lists(S, st);
    // sparse stores: the lists the selection runs on (all ranks' lists, gathered once, if W > 1)
    ListIndex L;
    if (S.sparse) {
        Samples& M = const_cast<Samples&>(S);
        if (world > 1 && !M.g_off.p) gather_lists(M, st);
        L = world > 1 ? ListIndex{M.g_off.as<uint64_t>(), M.g_mem.as<uint32_t>(), M.g_n, M.g_count0.as<uint32_t>()}
                      : ListIndex{S.list_off.as<uint64_t>(), S.list_mem.as<uint32_t>(), S.s1 - S.s0,
                                  S.count0.as<uint32_t>()};
        if (!S.inv_off.p) build_inverted(M, L, n, st);  // vertex -> samples index, once per handle
        BPT_CUDA(cudaMemcpyAsync(count.p, L.count0, (uint64_t)S.n_pad * 4, cudaMemcpyDeviceToDevice, st));
    }
    DevBuf covered(S.sparse ? L.nlists * 4 + 4 : 4);
    if (S.sparse) BPT_CUDA(cudaMemsetAsync(covered.p, 0, covered.bytes, st));
    const auto t1 = clk::now();
    // pair exchange (multi-rank dense stores): the counts become global once
#ifndef BPT_PAIR_CAP
#define BPT_PAIR_CAP (1u << 16)
#endif
    constexpr uint32_t kPairCap = BPT_PAIR_CAP;  // decrement pairs per rank and round (-D for the overflow test build)
    DevBuf pairs(pair_exchange ? kPairCap * 8ull : 8), pairs_all(pair_exchange ? (uint64_t)world * kPairCap * 8 : 8),
        npairs(8), tmp(pair_exchange ? (uint64_t)S.n_pad * 4 : 4);
    if (pair_exchange) {
        comm_allreduce_sum_u32(comm, count.as<uint32_t>(), S.n_pad, st);
        BPT_CUDA(cudaMemsetAsync(npairs.p, 0, 8, st));  // [0] pairs of the round, [1] overflow
    }
    for (uint32_t r = 0; r < k; ++r) {
        unsigned long long* key = keys.as<unsigned long long>() + r;
        if (pair_exchange) {
            // identical global counts on every rank: the same argmax everywhere, no collective
            k_argmax<<<vgrid, kSelThreads, 0, st>>>(count.as<uint32_t>(), n, 0, n, sel.as<uint8_t>(), key,
                                                    nlist.as<uint32_t>());
            k_cover<<<ggrid, 256, 0, st>>>(S.store.as<uint64_t>(), n, blocks, key, cov.as<uint64_t>(), sel.as<uint8_t>(),
                                           nlist.as<uint32_t>(), list.as<uint32_t>(), newm.as<uint64_t>());
            count_launch(2);
            if (r == 0) {  // the first seed covers a large share of the samples: one dense exchange
                BPT_CUDA(cudaMemsetAsync(tmp.p, 0, tmp.bytes, st));
                k_decrement<<<dgrid, 256, 0, st>>>(S.store.as<uint64_t>(), n, nlist.as<uint32_t>(), list.as<uint32_t>(),
                                                   newm.as<uint64_t>(), tmp.as<uint32_t>());  // tmp = -d (mod 2^32)
                comm_allreduce_sum_u32(comm, tmp.as<uint32_t>(), S.n_pad, st);
                k_add_u32<<<dgrid, 256, 0, st>>>(count.as<uint32_t>(), tmp.as<uint32_t>(), S.n_pad);
            } else {
                BPT_CUDA(cudaMemsetAsync(pairs.p, 0xff, pairs.bytes, st));
                BPT_CUDA(cudaMemsetAsync(npairs.p, 0, 4, st));
                k_decrement_pairs<<<dgrid, 256, 0, st>>>(S.store.as<uint64_t>(), n, nlist.as<uint32_t>(), list.as<uint32_t>(),
                                                         newm.as<uint64_t>(), pairs.as<unsigned long long>(), kPairCap,
                                                         npairs.as<uint32_t>(), npairs.as<uint32_t>() + 1);
                comm_allgather_u64(comm, pairs.as<uint64_t>(), pairs_all.as<uint64_t>(), kPairCap, st);
                k_apply_pairs<<<num_sms() * 4, 256, 0, st>>>(pairs_all.as<unsigned long long>(),
                                                             (uint64_t)world * kPairCap, count.as<uint32_t>());
            }
            count_launch(2);
            ::bpt::check_cuda(cudaGetLastError(), "launch selection pair exchange");
            continue;
        }
        if (world > 1 && !S.sparse) {
            comm_reduce_scatter_u32(comm, count.as<uint32_t>(), shard.as<uint32_t>(), shard_len, st);
            k_argmax<<<vgrid, kSelThreads, 0, st>>>(shard.as<uint32_t>(), shard_len, (uint64_t)rank * shard_len, n,
                                                    sel.as<uint8_t>(), key, nlist.as<uint32_t>());
            count_launch();
            comm_allreduce_max_u64(comm, key, 1, st);
        } else {
            k_argmax<<<vgrid, kSelThreads, 0, st>>>(count.as<uint32_t>(), n, 0, n, sel.as<uint8_t>(), key,
                                                    nlist.as<uint32_t>());
            count_launch();
        }
        if (S.sparse) {
            k_cover_sparse<<<num_sms() * 4, 256, 0, st>>>(key, S.inv_off.as<uint64_t>(), S.inv_s.as<uint32_t>(),
                                                           L.off, L.mem, covered.as<uint32_t>(), sel.as<uint8_t>(),
                                                           count.as<uint32_t>());
            count_launch();
            ::bpt::check_cuda(cudaGetLastError(), "launch k_cover_sparse");
            continue;
        }
        k_cover<<<ggrid, 256, 0, st>>>(S.store.as<uint64_t>(), n, blocks, key, cov.as<uint64_t>(), sel.as<uint8_t>(),
                                       nlist.as<uint32_t>(), list.as<uint32_t>(), newm.as<uint64_t>());
        if (lists)
            k_decrement_lists<<<num_sms() * 4, 256, 0, st>>>(nlist.as<uint32_t>(), list.as<uint32_t>(),
                                                             newm.as<uint64_t>(), S.list_off.as<uint64_t>(),
                                                             S.list_mem.as<uint32_t>(), S.s1 - S.s0,
                                                             count.as<uint32_t>());
        else
            k_decrement<<<dgrid, 256, 0, st>>>(S.store.as<uint64_t>(), n, nlist.as<uint32_t>(), list.as<uint32_t>(),
                                               newm.as<uint64_t>(), count.as<uint32_t>());
        count_launch(2);
        ::bpt::check_cuda(cudaGetLastError(), "launch k_decrement");
    }
    std::vector<unsigned long long> hk(k);
    BPT_CUDA(cudaMemcpyAsync(hk.data(), keys.p, (uint64_t)k * 8, cudaMemcpyDeviceToHost, st));
    if (pair_exchange) {  // did any rank's pairs of any round overflow? (the same answer on every rank)
        unsigned long long* f = reinterpret_cast<unsigned long long*>(npairs.p);
        // [1] (the overflow word) -> a u64 for the max-reduction
        k_widen_flag<<<1, 32, 0, st>>>(npairs.as<uint32_t>() + 1, f);
        comm_allreduce_max_u64(comm, f, 1, st);
        unsigned long long hf = 0;
        BPT_CUDA(cudaMemcpyAsync(&hf, f, 8, cudaMemcpyDeviceToHost, st));
        BPT_CUDA(cudaStreamSynchronize(st));
        if (hf) { *overflowed = true; return; }
    }
    BPT_CUDA(cudaStreamSynchronize(st));
    if (getenv("BPT_TRACE")) {
        auto ms = [](clk::time_point x, clk::time_point y) { return std::chrono::duration<double, std::milli>(y - x).count(); };
        fprintf(stderr, "[bpt] select k=%u: lists %s %.2f ms, rounds %.2f ms (world %d, blocks %llu)\n", k,
                lists ? "on" : "off", ms(t0, t1), ms(t1, clk::now()), world, (unsigned long long)blocks);
    }
    for (uint32_t r = 0; r < k; ++r) {
        h_seeds[r] = ~(uint32_t)hk[r];
        h_gains[r] = hk[r] >> 32;
    }
}

}  // namespace bpt
