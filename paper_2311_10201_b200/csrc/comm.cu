// comm.cu -- NCCL plumbing for multi-GPU seed selection: one process per GPU,
// a 128-byte ncclUniqueId bootstrapped by the caller (e.g. torch.distributed). Sampling
// itself never communicates. Selection over dense stores issues one ReduceScatter(count, sum)
// and one 8-byte AllReduce(max) per greedy round; over member-list stores it gathers all
// lists once (AllGather) and needs no collective per round. Enqueued on the caller's stream.
#include <nccl.h>

#include "internal.cuh"

namespace bpt {

static void check_nccl(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) fail(BPT_ENCCL, std::string(what) + ": " + ncclGetErrorString(r));
}

void comm_unique_id(void* out) {
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
    ncclUniqueId id;
    check_nccl(ncclGetUniqueId(&id), "ncclGetUniqueId");
    memcpy(out, &id, sizeof(id));
}

void comm_init(Comm* c, const void* uid) {
    ncclUniqueId id;
    memcpy(&id, uid, sizeof(id));
    ncclComm_t nc = nullptr;
    check_nccl(ncclCommInitRank(&nc, c->world, id, c->rank), "ncclCommInitRank");
    c->nccl = nc;
}

void comm_destroy(Comm* c) {
    if (c && c->nccl) {
        ncclCommDestroy((ncclComm_t)c->nccl);
        c->nccl = nullptr;
    }
}

void comm_reduce_scatter_u32(Comm* c, const uint32_t* send, uint32_t* recv, uint64_t recv_count, cudaStream_t st) {
    check_nccl(ncclReduceScatter(send, recv, recv_count, ncclUint32, ncclSum, (ncclComm_t)c->nccl, st),
               "ncclReduceScatter");
}

void comm_broadcast(Comm* c, const void* send, void* recv, uint64_t bytes, int root, cudaStream_t st) {
    check_nccl(ncclBroadcast(send, recv, bytes, ncclUint8, root, (ncclComm_t)c->nccl, st), "ncclBroadcast");
}

void comm_allreduce_sum_u32(Comm* c, uint32_t* buf, uint64_t count, cudaStream_t st) {
    check_nccl(ncclAllReduce(buf, buf, count, ncclUint32, ncclSum, (ncclComm_t)c->nccl, st), "ncclAllReduce");
}

void comm_allgather_u32(Comm* c, const uint32_t* send, uint32_t* recv, uint64_t count, cudaStream_t st) {
    check_nccl(ncclAllGather(send, recv, count, ncclUint32, (ncclComm_t)c->nccl, st), "ncclAllGather");
}

void comm_allgather_u64(Comm* c, const uint64_t* send, uint64_t* recv, uint64_t count, cudaStream_t st) {
    check_nccl(ncclAllGather(send, recv, count, ncclUint64, (ncclComm_t)c->nccl, st), "ncclAllGather");
}

void comm_allreduce_max_u64(Comm* c, unsigned long long* buf, uint64_t count, cudaStream_t st) {
    check_nccl(ncclAllReduce(buf, buf, count, ncclUint64, ncclMax, (ncclComm_t)c->nccl, st), "ncclAllReduce");
}

}  // namespace bpt
