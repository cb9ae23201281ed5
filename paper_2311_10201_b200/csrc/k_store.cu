// k_store.cu -- A5 RRR store finalisation (sizes, digests, E_logical, occurrence counts)
// and A6 RRR extraction (Listing 1 lines 18-21: "for vertex v, for colour c,
// if visited[v].c: RRRset(c).add(v)") as an ordered, atomic-free mask -> list transpose.
#include <cstring>
#include <map>

#include "internal.cuh"

namespace bpt {

void exclusive_scan_u32(const uint32_t* in, uint32_t* out, uint64_t count, void* temp, cudaStream_t st);
void exclusive_scan_u64(const uint64_t* in, uint64_t* out, uint64_t count, void* temp, cudaStream_t st);
size_t scan_temp_bytes(uint64_t count);

namespace {

constexpr uint32_t kFull = 0xffffffffu;

// SplitMix64 output function of v + gamma (digest definition)
__device__ __forceinline__ uint64_t digest_mix(uint64_t v) {
    uint64_t z = v + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

constexpr int kFinThreads = 256;

// 256-bit load / store of a vertex's 4 slot masks (one 32-B sector)
__device__ __forceinline__ void ld4(const unsigned long long* p, unsigned long long (&m)[4]) {
    asm volatile("ld.global.v4.u64 {%0, %1, %2, %3}, [%4];" : "=l"(m[0]), "=l"(m[1]), "=l"(m[2]), "=l"(m[3]) : "l"(p) : "memory");
}
__device__ __forceinline__ void st4z(unsigned long long* p) {
    asm volatile("st.global.v4.u64 [%0], {%1, %1, %1, %1};" :: "l"(p), "l"(0ull) : "memory");
}

// grid (ranges, slots). Block (r, slot) scans vertices [r*chunk, (r+1)*chunk) of the working
// masks of in-flight block `slot` (= local block blk0+slot): writes V to the RRR store, clears
// the working pair for the next batch and adds the occurrences. Each warp walks its own
// 32-vertex tiles; lane l accumulates colours l and l+32 over the tile's non-zero masks
// (broadcast from shared memory), so the per-colour sums cost O(non-zero vertices).
__global__ void __launch_bounds__(kFinThreads) k_finalize(ulonglong2* __restrict__ VN, uint64_t* __restrict__ store,
                                                          uint32_t n, const Ctl* __restrict__ ctl,
                                                          uint64_t chunk, const uint32_t* __restrict__ roff,
                                                          uint64_t nlocal, uint32_t* __restrict__ sizes,
                                                          unsigned long long* __restrict__ elog_total,
                                                          uint32_t* __restrict__ count0, int single_slot,
                                                          uint32_t vstride, uint64_t sstride, int umode,
                                                          const uint32_t* __restrict__ slot_sample, uint64_t s0) {
    constexpr int kW = kFinThreads / 32;
    __shared__ unsigned long long s_mask[kW][32];
    __shared__ uint32_t s_size[kW][64];
    __shared__ unsigned long long s_el[kW];
    if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0)  // launch evidence (Ctl::kernels_run)
        atomicAdd(&const_cast<Ctl*>(ctl)->kernels_run, 1ull);
    if (blockIdx.y >= ctl->slots) return;
    const uint64_t blk = ctl->blk0 + blockIdx.y;
    uint64_t* V = store + (size_t)blk * n;
    // working mask of vertex v of this block: W[v * vstride] (slot-major: vstride 1, sstride n;
    // wide vertex-major: vstride kWide, sstride 1)
    ulonglong2* W = VN + (size_t)blockIdx.y * sstride;
    // union layout: U[slot][n] then V[slot][n]; sstride = n, gridDim.y = slots_max
    unsigned long long* UV = reinterpret_cast<unsigned long long*>(VN) + (size_t)blockIdx.y * n;
    const size_t slots_max_n = (size_t)gridDim.y * n;
    // vertex-major union layout (umode 2): U[v * slots_max + slot], V after slots_max * n words
    unsigned long long* UVm = reinterpret_cast<unsigned long long*>(VN);
    const uint64_t v_begin = (uint64_t)blockIdx.x * chunk;
    const uint64_t v_end = umin64(v_begin + chunk, n);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint32_t sz_lo = 0, sz_hi = 0;
    unsigned long long el = 0;
    constexpr int kU = 4;  // tiles per warp iteration: their loads are issued together
    for (uint64_t base = v_begin + 32ull * kU * wid; base < v_end; base += 32ull * kU * kW) {
        uint64_t m[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const uint64_t v = base + 32ull * u + lane;
            // N is 0 after the last level (union layout: U == V, V after the U block)
            m[u] = v < v_end ? (umode == 2 ? UVm[slots_max_n + v * gridDim.y + blockIdx.y]
                                : umode ? UV[slots_max_n + v] : W[v * vstride].x) : 0ull;
        }
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const uint64_t v = base + 32ull * u + lane;
            if (v < v_end) {
                V[v] = m[u];
                if (m[u]) {
                    if (umode == 2) {
                        UVm[v * gridDim.y + blockIdx.y] = 0ull;
                        UVm[slots_max_n + v * gridDim.y + blockIdx.y] = 0ull;
                    } else if (umode) {
                        UV[v] = 0ull;
                        UV[slots_max_n + v] = 0ull;
                    } else {
                        W[v * vstride] = make_ulonglong2(0ull, 0ull);
                    }
                    const uint32_t pc = __popcll(m[u]);
                    // occurrences (A7 round 0): one block owns v when the batch has one slot
                    if (single_slot) count0[v] += pc;
                    else atomicAdd(&count0[v], pc);
                    el += (unsigned long long)pc * (roff[v + 1] - roff[v]);  // E_logical: unfused reads
                }
            }
        }
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            uint32_t b = __ballot_sync(kFull, m[u] != 0);
            if (!b) continue;
            s_mask[wid][lane] = m[u];
            __syncwarp();
            while (b) {
                const int j = __ffs(b) - 1;
                b &= b - 1;
                const unsigned long long mj = s_mask[wid][j];
                sz_lo += (uint32_t)(mj >> lane) & 1u;
                sz_hi += (uint32_t)(mj >> (lane + 32)) & 1u;
            }
            __syncwarp();
        }
    }
    s_size[wid][lane] = sz_lo;
    s_size[wid][lane + 32] = sz_hi;
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) el += __shfl_xor_sync(kFull, el, d);
    if (lane == 0) s_el[wid] = el;
    __syncthreads();
    if (threadIdx.x < 64) {
        const int c = threadIdx.x;
        uint32_t S = 0;
        for (int q = 0; q < kW; ++q) S += s_size[q][c];
        const uint64_t li = 64ull * blk + c;  // local slot = local sample index unless start-sorted
        if (li < nlocal && S) atomicAdd(&sizes[slot_sample ? slot_sample[li] - s0 : li], S);
    }
    if (threadIdx.x == 0) {
        unsigned long long E = 0;
        for (int q = 0; q < kW; ++q) E += s_el[q];
        if (E) atomicAdd(elog_total, E);
    }
}


// Vertex-major finaliser (batch-wide frontier, umode 2): one thread per vertex handles the S <= 4
// slots of the batch -- one 32-B read of V[v][0..S), S coalesced store writes, U / V re-zeroed with
// 16-B stores, occurrences without atomics (one writer per vertex), per-colour sizes of every slot
// (lane l counts colours l and l + 32 of the warp's non-zero masks, broadcast from shared memory).
__global__ void __launch_bounds__(kFinThreads) k_finalize_v(unsigned long long* __restrict__ UV, uint64_t* __restrict__ store,
                                                            uint32_t n, const Ctl* __restrict__ ctl, uint64_t chunk,
                                                            const uint32_t* __restrict__ roff, uint64_t nlocal,
                                                            uint32_t* __restrict__ sizes,
                                                            unsigned long long* __restrict__ elog_total,
                                                            uint32_t* __restrict__ count0, uint32_t S,
                                                            const uint32_t* __restrict__ slot_sample, uint64_t s0) {
    constexpr int kW = kFinThreads / 32;
    __shared__ unsigned long long s_el[kW];
    if (blockIdx.x == 0 && threadIdx.x == 0)  // launch evidence (Ctl::kernels_run)
        atomicAdd(&const_cast<Ctl*>(ctl)->kernels_run, 1ull);
    const uint32_t nsl = ctl->slots;
    const uint64_t blk0 = ctl->blk0;
    unsigned long long* V = UV + (size_t)S * n;
    const uint64_t v_begin = (uint64_t)blockIdx.x * chunk;
    const uint64_t v_end = umin64(v_begin + chunk, n);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    unsigned long long el = 0;
    for (uint64_t base = v_begin + 32ull * wid; base < v_end; base += 32ull * kW) {
        const uint64_t v = base + lane;
        unsigned long long m[4] = {0ull, 0ull, 0ull, 0ull};
        if (v < v_end) {
            if (S == 4) {
                ld4(V + v * 4, m);
            } else {
#pragma unroll
                for (uint32_t s = 0; s < 4; ++s) m[s] = s < S ? V[v * S + s] : 0ull;
            }
#pragma unroll
            for (uint32_t s = 0; s < 4; ++s)
                if (s < nsl) store[(size_t)(blk0 + s) * n + v] = m[s];
            const bool any = (m[0] | m[1] | m[2] | m[3]) != 0ull;
            if (any) {
                if (S == 4) {
                    st4z(V + v * 4);
                    st4z(UV + v * 4);
                } else {
                    for (uint32_t s = 0; s < S; ++s) { V[v * S + s] = 0ull; UV[v * S + s] = 0ull; }
                }
                const uint32_t pc = __popcll(m[0]) + __popcll(m[1]) + __popcll(m[2]) + __popcll(m[3]);
                count0[v] += pc;  // occurrences (A7 round 0); one writer per vertex
                el += (unsigned long long)pc * (roff[v + 1] - roff[v]);  // E_logical: unfused reads
            }
        }
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) el += __shfl_xor_sync(0xffffffffu, el, d);
    if (lane == 0) s_el[wid] = el;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long E = 0;
        for (int q = 0; q < kW; ++q) E += s_el[q];
        if (E) atomicAdd(elog_total, E);
    }
}


// Per-sample sizes of listed store blocks (the batch-wide frontier's finaliser leaves them to the
// requests that need them, see ensure_sizes): block (r, j) counts, per colour, the set bits of
// vertices [r chunk, (r + 1) chunk) of store block blk[j] (lane l counts colours l and l + 32 of the
// warp's non-zero masks, broadcast from shared memory).
__global__ void __launch_bounds__(kFinThreads) k_block_sizes(const uint64_t* __restrict__ store, uint32_t n,
                                                             uint64_t chunk, const uint64_t* __restrict__ blk,
                                                             uint64_t nlocal, const uint32_t* __restrict__ slot_sample,
                                                             uint64_t s0, uint32_t* __restrict__ sizes) {
    constexpr int kW = kFinThreads / 32;
    __shared__ unsigned long long s_mask[kW][32];
    __shared__ uint32_t s_size[kW][64];
    const uint64_t b = blk[blockIdx.y];
    const uint64_t* V = store + (size_t)b * n;
    const uint64_t v_begin = (uint64_t)blockIdx.x * chunk;
    const uint64_t v_end = umin64(v_begin + chunk, n);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint32_t sz_lo = 0, sz_hi = 0;
    for (uint64_t base = v_begin + 32ull * wid; base < v_end; base += 32ull * kW) {
        const uint64_t v = base + lane;
        const uint64_t m = v < v_end ? V[v] : 0ull;
        uint32_t bl = __ballot_sync(kFull, m != 0);
        if (!bl) continue;
        s_mask[wid][lane] = m;
        __syncwarp();
        while (bl) {
            const int j = __ffs(bl) - 1;
            bl &= bl - 1;
            const unsigned long long mj = s_mask[wid][j];
            sz_lo += (uint32_t)(mj >> lane) & 1u;
            sz_hi += (uint32_t)(mj >> (lane + 32)) & 1u;
        }
        __syncwarp();
    }
    s_size[wid][lane] = sz_lo;
    s_size[wid][lane + 32] = sz_hi;
    __syncthreads();
    if (threadIdx.x < 64) {
        const int c = threadIdx.x;
        uint32_t T = 0;
        for (int q = 0; q < kW; ++q) T += s_size[q][c];
        const uint64_t li = 64ull * b + c;  // local slot
        if (li < nlocal && T) atomicAdd(&sizes[slot_sample ? slot_sample[li] - s0 : li], T);
    }
}

// Per-sample digests, computed on demand from the store (verification
// checksums, not part of the method): block (r, g) accumulates colour sums of splitmix64(v)
// over vertices [r*chunk, (r+1)*chunk) of local block g.
__global__ void __launch_bounds__(kFinThreads) k_digests(const uint64_t* __restrict__ store, uint32_t n,
                                                         uint64_t chunk, uint64_t nlocal,
                                                         unsigned long long* __restrict__ digests,
                                                         const uint32_t* __restrict__ slot_sample, uint64_t s0) {
    constexpr int kW = kFinThreads / 32;
    __shared__ unsigned long long s_mask[kW][32];
    __shared__ unsigned long long s_mix[kW][32];
    __shared__ unsigned long long s_dig[kW][64];
    const uint64_t blk = blockIdx.y;
    const uint64_t* V = store + (size_t)blk * n;
    const uint64_t v_begin = (uint64_t)blockIdx.x * chunk;
    const uint64_t v_end = umin64(v_begin + chunk, n);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    unsigned long long dg_lo = 0, dg_hi = 0;
    for (uint64_t base = v_begin + 32ull * wid; base < v_end; base += 32ull * kW) {
        const uint64_t v = base + lane;
        const uint64_t m = v < v_end ? V[v] : 0ull;
        uint32_t b = __ballot_sync(kFull, m != 0);
        if (!b) continue;
        s_mask[wid][lane] = m;
        s_mix[wid][lane] = digest_mix(v);
        __syncwarp();
        while (b) {
            const int j = __ffs(b) - 1;
            b &= b - 1;
            const unsigned long long mj = s_mask[wid][j], xj = s_mix[wid][j];
            if ((mj >> lane) & 1ull) dg_lo += xj;
            if ((mj >> (lane + 32)) & 1ull) dg_hi += xj;
        }
        __syncwarp();
    }
    s_dig[wid][lane] = dg_lo;
    s_dig[wid][lane + 32] = dg_hi;
    __syncthreads();
    if (threadIdx.x < 64) {
        const int c = threadIdx.x;
        unsigned long long D = 0;
        for (int q = 0; q < kW; ++q) D += s_dig[q][c];
        const uint64_t li = 64ull * blk + c;  // local slot (relative to this launch's first block)
        if (li < nlocal && D) atomicAdd(&digests[slot_sample ? slot_sample[li] - s0 : li], D);
    }
}

// ---------------------------------------------------------------------------- extraction
// One warp owns a tile of kExRounds*32 consecutive vertices of block `blk`.
constexpr int kExRounds = 32;
constexpr uint32_t kExTile = 32 * kExRounds;

// All requested store blocks in one launch: grid.y = j-th requested block (blk[j], colour set
// cms[j]); its counts / positions are the j-th [64][ntiles] slab of tcnt / tpos, its colours'
// output offsets cbase[64 j + c].
// pass 1: per-(colour, tile) member counts, colour-major; colours outside the requested set cm = 0
__global__ void k_extract_count(const uint64_t* __restrict__ store, uint32_t n, const uint64_t* __restrict__ blk,
                                const uint64_t* __restrict__ cms, uint32_t ntiles, uint32_t* __restrict__ tcnt_all) {
    const uint64_t* V = store + (size_t)blk[blockIdx.y] * n;
    const uint64_t cm = cms[blockIdx.y];
    uint32_t* tcnt = tcnt_all + (uint64_t)blockIdx.y * 64 * ntiles;
    const int lane = threadIdx.x & 31;
    const uint64_t tile = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    if (tile >= ntiles) return;
    uint32_t cnt_lo = 0, cnt_hi = 0;  // lane l counts colours l and l + 32
    for (int r = 0; r < kExRounds; ++r) {
        const uint64_t v = tile * kExTile + (uint64_t)r * 32 + lane;
        const uint64_t m = v < n ? V[v] : 0ull;
        if (!__any_sync(kFull, m != 0)) continue;
        for (uint64_t mm = cm; mm; mm &= mm - 1) {
            const uint32_t c = __ffsll((long long)mm) - 1;
            const uint32_t b = __ballot_sync(kFull, (m >> c) & 1ull);
            if (lane == (int)(c & 31)) { if (c < 32) cnt_lo += __popc(b); else cnt_hi += __popc(b); }
        }
    }
    tcnt[(uint64_t)lane * ntiles + tile] = ((cm >> lane) & 1ull) ? cnt_lo : 0;
    const uint32_t c2 = lane + 32;
    tcnt[(uint64_t)c2 * ntiles + tile] = ((cm >> c2) & 1ull) ? cnt_hi : 0;
}

// pass 2: ordered scatter; tpos = exclusive colour-major scan of tcnt; colour c's members go to
// cbase[c] + (its members in earlier tiles) + rank, vertices ascending (reading C-10)
__global__ void k_extract_write(const uint64_t* __restrict__ store, uint32_t n, const uint64_t* __restrict__ blk,
                                const uint64_t* __restrict__ cms, uint32_t ntiles, const uint32_t* __restrict__ tpos_all,
                                const uint64_t* __restrict__ cbase_all, uint32_t* __restrict__ members) {
    const uint64_t* V = store + (size_t)blk[blockIdx.y] * n;
    const uint64_t cm = cms[blockIdx.y];
    const uint32_t* tpos = tpos_all + (uint64_t)blockIdx.y * 64 * ntiles;
    const uint64_t* cbase = cbase_all + 64ull * blockIdx.y;
    const int lane = threadIdx.x & 31;
    const uint64_t tile = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    if (tile >= ntiles) return;
    // positions relative to the colour's first tile, plus the caller's offset of that colour's sample
    uint64_t pos_lo = ((cm >> lane) & 1ull) ? cbase[lane] + tpos[(uint64_t)lane * ntiles + tile] -
                                                  tpos[(uint64_t)lane * ntiles] : 0;
    uint64_t pos_hi = ((cm >> (lane + 32)) & 1ull) ? cbase[lane + 32] + tpos[(uint64_t)(lane + 32) * ntiles + tile] -
                                                         tpos[(uint64_t)(lane + 32) * ntiles] : 0;
    const uint32_t lt = (1u << lane) - 1u;
    for (int r = 0; r < kExRounds; ++r) {
        const uint64_t v = tile * kExTile + (uint64_t)r * 32 + lane;
        const uint64_t m = v < n ? V[v] : 0ull;
        if (!__any_sync(kFull, m != 0)) continue;
        for (uint64_t mm = cm; mm; mm &= mm - 1) {
            const uint32_t c = __ffsll((long long)mm) - 1;
            const bool has = (m >> c) & 1ull;
            const uint32_t b = __ballot_sync(kFull, has);
            if (!b) continue;
            const uint32_t src_lane = c & 31;
            const uint64_t p = __shfl_sync(kFull, c < 32 ? pos_lo : pos_hi, src_lane);
            if (has) members[p + __popc(b & lt)] = (uint32_t)v;
            if (lane == (int)src_lane) { if (c < 32) pos_lo += __popc(b); else pos_hi += __popc(b); }
        }
    }
}

}  // namespace

// launch configuration of the finaliser for batches of `slots_max` blocks
static dim3 finalize_grid(uint32_t n, uint32_t slots_max, uint64_t* chunk_out) {
    uint64_t ranges = (uint64_t)num_sms() * 4 / (slots_max ? slots_max : 1);
    if (ranges < 1) ranges = 1;
    uint64_t chunk = (n + ranges - 1) / ranges;
    chunk = (chunk + kFinThreads - 1) / kFinThreads * kFinThreads;
    if (chunk == 0) chunk = kFinThreads;
    ranges = (n + chunk - 1) / chunk;
    *chunk_out = chunk;
    return dim3((unsigned)ranges, slots_max);
}

namespace {
// sparse store: digest of list l = sum of splitmix64 over its members
__global__ void k_digests_lists(const uint64_t* __restrict__ off, const uint32_t* __restrict__ members, uint64_t nlists,
                                unsigned long long* __restrict__ digests) {
    for (uint64_t l = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; l < nlists; l += (uint64_t)gridDim.x * blockDim.x) {
        unsigned long long d = 0;
        for (uint64_t j = off[l]; j < off[l + 1]; ++j) d += digest_mix(members[j]);
        digests[l] = d;
    }
}
}  // namespace

void compute_digests(const Samples& S, cudaStream_t st) {
    const uint64_t nlocal = S.s1 - S.s0;
    if (S.sparse) {
        const unsigned grid = (unsigned)umin64((nlocal + 255) / 256, (uint64_t)num_sms() * 8);
        if (grid) k_digests_lists<<<grid, 256, 0, st>>>(S.list_off.as<uint64_t>(), S.list_mem.as<uint32_t>(), nlocal,
                                                        S.digests.as<unsigned long long>());
        count_launch();
        ::bpt::check_cuda(cudaGetLastError(), "launch k_digests_lists");
        return;
    }
    BPT_CUDA(cudaMemsetAsync(S.digests.p, 0, nlocal * 8, st));
    uint64_t ranges = (uint64_t)num_sms() * 4 / umax64(S.blocks, 1);
    if (ranges < 1) ranges = 1;
    uint64_t chunk = (S.n + ranges - 1) / ranges;
    chunk = (chunk + 255) / 256 * 256;
    ranges = (S.n + chunk - 1) / chunk;
    for (uint64_t b0 = 0; b0 < S.blocks; b0 += 65535) {
        const uint64_t nb = umin64(65535, S.blocks - b0);
        k_digests<<<dim3((unsigned)ranges, (unsigned)nb), kFinThreads, 0, st>>>(
            S.store.as<uint64_t>() + (size_t)b0 * S.n, S.n, chunk, nlocal - 64 * b0,
            S.sorted ? S.digests.as<unsigned long long>() : S.digests.as<unsigned long long>() + 64 * b0,
            S.sorted ? S.slot_sample.as<uint32_t>() + 64 * b0 : nullptr, S.s0);
        count_launch();
    }
    ::bpt::check_cuda(cudaGetLastError(), "launch k_digests");
}

void launch_finalize(const Samples& S, ulonglong2* VN, const Ctl* ctl, uint32_t slots_max, const uint32_t* roff,
                     cudaStream_t st, unsigned long long* d_elog, bool wide, int umode) {
    uint64_t chunk = 0;
    if (umode == 2) {
        const dim3 grid = finalize_grid(S.n, 1, &chunk);
        k_finalize_v<<<grid.x, kFinThreads, 0, st>>>(reinterpret_cast<unsigned long long*>(VN), S.store.as<uint64_t>(),
                                                     S.n, ctl, chunk, roff, S.s1 - S.s0, S.sizes.as<uint32_t>(), d_elog,
                                                     S.count0.as<uint32_t>(), slots_max,
                                                     S.sorted ? S.slot_sample.as<uint32_t>() : nullptr, S.s0);
        count_launch();
        ::bpt::check_cuda(cudaGetLastError(), "launch k_finalize_v");
        return;
    }
    const dim3 grid = finalize_grid(S.n, slots_max, &chunk);
    k_finalize<<<grid, kFinThreads, 0, st>>>(VN, S.store.as<uint64_t>(), S.n, ctl, chunk, roff, S.s1 - S.s0,
                                             S.sizes.as<uint32_t>(), d_elog,
                                             S.count0.as<uint32_t>(), slots_max == 1 ? 1 : 0,
                                             wide ? kWide : 1u, wide ? (uint64_t)1 : (uint64_t)S.n, umode,
                                             S.sorted ? S.slot_sample.as<uint32_t>() : nullptr, S.s0);
    count_launch();
    ::bpt::check_cuda(cudaGetLastError(), "launch k_finalize");
}

// graph node for the finaliser (device-resident batch loop)
void add_store_nodes(cudaGraph_t g, cudaGraphNode_t dep, const Samples& S, ulonglong2* VN, const Ctl* ctl,
                     uint32_t slots_max, const uint32_t* roff, unsigned long long* d_elog, cudaGraphNode_t* last,
                     bool wide, int umode) {
    uint64_t chunk = 0;
    if (umode == 2) {
        const dim3 grid = finalize_grid(S.n, 1, &chunk);
        unsigned long long* UV = reinterpret_cast<unsigned long long*>(VN);
        uint64_t* store = S.store.as<uint64_t>();
        uint32_t n = S.n, Sl = slots_max;
        uint64_t nlocal = S.s1 - S.s0, s0 = S.s0;
        uint32_t* sizes = S.sizes.as<uint32_t>();
        uint32_t* count0 = S.count0.as<uint32_t>();
        const uint32_t* slot_sample = S.sorted ? S.slot_sample.as<uint32_t>() : nullptr;
        void* args[] = {&UV, &store, &n, (void*)&ctl, &chunk, (void*)&roff, &nlocal, &sizes, &d_elog, &count0, &Sl,
                        (void*)&slot_sample, &s0};
        cudaKernelNodeParams p{};
        p.func = (void*)k_finalize_v;
        p.gridDim = dim3(grid.x);
        p.blockDim = dim3(kFinThreads);
        p.kernelParams = args;
        BPT_CUDA(cudaGraphAddKernelNode(last, g, &dep, 1, &p));
        return;
    }
    const dim3 grid = finalize_grid(S.n, slots_max, &chunk);
    uint64_t* store = S.store.as<uint64_t>();
    uint32_t n = S.n;
    uint64_t nlocal = S.s1 - S.s0;
    uint32_t* sizes = S.sizes.as<uint32_t>();
    uint32_t* count0 = S.count0.as<uint32_t>();
    int single = slots_max == 1 ? 1 : 0;
    uint32_t vstride = wide ? kWide : 1u;
    uint64_t sstride = wide ? 1 : (uint64_t)n;
    int um = umode;
    const uint32_t* slot_sample = S.sorted ? S.slot_sample.as<uint32_t>() : nullptr;
    uint64_t s0 = S.s0;
    void* fin_args[] = {&VN, &store, &n, (void*)&ctl, &chunk, (void*)&roff, &nlocal, &sizes, &d_elog,
                        &count0, &single, &vstride, &sstride, &um, (void*)&slot_sample, &s0};
    cudaKernelNodeParams p{};
    p.func = (void*)k_finalize;
    p.gridDim = grid;
    p.blockDim = dim3(kFinThreads);
    p.kernelParams = fin_args;
    BPT_CUDA(cudaGraphAddKernelNode(last, g, &dep, 1, &p));
}

// d_offsets[count+1] must already hold the exclusive scan of sizes (offsets[count] = total)
void ensure_sizes(Samples& S, uint64_t first, uint64_t count, cudaStream_t st) {
    if (!S.lazy_sizes || count == 0) return;
    const uint64_t lfirst = first - S.s0;
    if (S.sorted && S.h_sample_slot.empty()) {
        S.h_sample_slot.resize(S.s1 - S.s0);
        BPT_CUDA(cudaMemcpyAsync(S.h_sample_slot.data(), S.sample_slot.p, (S.s1 - S.s0) * 4, cudaMemcpyDeviceToHost, st));
        BPT_CUDA(cudaStreamSynchronize(st));
    }
    std::vector<uint64_t> need;
    for (uint64_t i = 0; i < count; ++i) {
        const uint64_t slot = S.sorted ? S.h_sample_slot[lfirst + i] : lfirst + i;
        const uint64_t b = slot / 64;
        if (!S.blk_sized[b]) { S.blk_sized[b] = 1; need.push_back(b); }
    }
    if (need.empty()) return;
    uint64_t chunk = 0;
    const dim3 grid = finalize_grid(S.n, 1, &chunk);
    constexpr uint64_t kGroup = 1024;
    DevBuf dblk(umin64(need.size(), kGroup) * 8);
    for (uint64_t g0 = 0; g0 < need.size(); g0 += kGroup) {
        const uint64_t nb = umin64(kGroup, need.size() - g0);
        BPT_CUDA(cudaMemcpyAsync(dblk.p, need.data() + g0, nb * 8, cudaMemcpyHostToDevice, st));
        k_block_sizes<<<dim3(grid.x, (unsigned)nb), kFinThreads, 0, st>>>(
            S.store.as<uint64_t>(), S.n, chunk, dblk.as<uint64_t>(), S.s1 - S.s0,
            S.sorted ? S.slot_sample.as<uint32_t>() : nullptr, S.s0, S.sizes.as<uint32_t>());
        count_launch();
        ::bpt::check_cuda(cudaGetLastError(), "launch k_block_sizes");
    }
}

void extract_range(const Samples& S, uint64_t first, uint64_t count, const uint64_t* h_offsets, uint32_t* d_members,
                   cudaStream_t st) {
    const uint32_t n = S.n;
    const uint32_t ntiles = (uint32_t)((n + kExTile - 1) / kExTile);
    const uint64_t lfirst = first - S.s0;  // local sample index of `first`
    // the store's blocks holding the requested samples: per block the colour (slot bit) set and
    // each colour's output offset (slots are the samples themselves unless start-sorted)
    struct Blk { uint64_t mask = 0; uint64_t base[64]; };
    std::map<uint64_t, Blk> blocks;
    for (uint64_t i = 0; i < count; ++i) {
        const uint64_t slot = S.sorted ? S.h_sample_slot[lfirst + i] : lfirst + i;
        Blk& b = blocks[slot / 64];
        b.mask |= 1ull << (slot % 64);
        b.base[slot % 64] = h_offsets[i];
    }
    // one slab per requested block: [blk ids | colour sets | colour offsets (64 per block)]; up to
    // kExGroup blocks share the same three launches (with sorted start vertices 64 consecutive samples
    // sit in up to 64 blocks; the group bounds the count slabs to kExGroup x 1.2 MB on C2)
    constexpr uint64_t kExGroup = 64;
    const uint64_t slab = (uint64_t)64 * ntiles;
    std::vector<std::pair<uint64_t, const Blk*>> all;
    for (auto& kv : blocks) all.emplace_back(kv.first, &kv.second);
    const uint64_t gmax = umin64(kExGroup, all.size());
    DevBuf tcnt(gmax * slab * 4), tmp(scan_temp_bytes(gmax * slab)), dhdr(gmax * (2 + 64) * 8);
    for (uint64_t g0 = 0; g0 < all.size(); g0 += kExGroup) {
        const uint64_t nb = umin64(kExGroup, all.size() - g0);
        std::vector<uint64_t> hdr(nb * (2 + 64), 0);
        for (uint64_t bi = 0; bi < nb; ++bi) {
            hdr[bi] = all[g0 + bi].first;
            hdr[nb + bi] = all[g0 + bi].second->mask;
            memcpy(&hdr[2 * nb + 64 * bi], all[g0 + bi].second->base, sizeof(all[g0 + bi].second->base));
        }
        BPT_CUDA(cudaMemcpyAsync(dhdr.p, hdr.data(), hdr.size() * 8, cudaMemcpyHostToDevice, st));
        const uint64_t* dblk = dhdr.as<uint64_t>();
        const uint64_t* dcm = dblk + nb;
        const uint64_t* dbase = dblk + 2 * nb;
        const dim3 grid((unsigned)(((uint64_t)ntiles * 32 + 255) / 256), (unsigned)nb);
        k_extract_count<<<grid, 256, 0, st>>>(S.store.as<uint64_t>(), n, dblk, dcm, ntiles, tcnt.as<uint32_t>());
        count_launch();
        exclusive_scan_u32(tcnt.as<uint32_t>(), tcnt.as<uint32_t>(), nb * slab, tmp.p, st);
        k_extract_write<<<grid, 256, 0, st>>>(S.store.as<uint64_t>(), n, dblk, dcm, ntiles, tcnt.as<uint32_t>(), dbase,
                                              d_members);
        count_launch();  // the next group's header copy is stream-ordered after these kernels
    }
    ::bpt::check_cuda(cudaGetLastError(), "launch k_extract_write");
}

}  // namespace bpt
