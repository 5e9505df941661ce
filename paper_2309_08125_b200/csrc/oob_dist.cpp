// Single-profile multi-GPU sharding of the template DP.
//
// Every rank runs oob_dp_run on the same profile.  The W-cell work of each wavefront is
// split across ranks (rank r takes units r, r + world, ... of every range's queue); after
// the wavefront one ncclAllGather of the per-rank partial argmins (16 bytes per output)
// lets every rank take the lexicographic minimum and finalize the whole wavefront, so all
// tables stay bit-identical.  The communicator is created here from a unique id the
// caller broadcasts (e.g. with torch.distributed); NCCL runs over NVLink inside the box.
#include <nccl.h>

#include <cstring>
#include <string>

#include "oob_internal.h"

namespace oob {

static oob_status nccl_fail(ncclResult_t r, const char *what) {
    return fail(OOB_E_NCCL, std::string(what) + ": " + ncclGetErrorString(r));
}

oob_status nccl_allgather_bytes(void *comm, const void *send, void *recv, size_t bytes, size_t /*recv_cap*/,
                                int /*world*/, void *stream) {
    ncclResult_t r = ncclAllGather(send, recv, bytes, ncclInt8, (ncclComm_t)comm, (cudaStream_t)stream);
    if (r != ncclSuccess) return nccl_fail(r, "ncclAllGather (wavefront partials)");
    return OOB_OK;
}

}  // namespace oob

using namespace oob;

extern "C" oob_status oob_nccl_unique_id(void *id_out) {
    if (!id_out) return fail(OOB_E_INVALID, "oob_nccl_unique_id: NULL");
    ncclUniqueId id;
    ncclResult_t r = ncclGetUniqueId(&id);
    if (r != ncclSuccess) return nccl_fail(r, "ncclGetUniqueId");
    static_assert(sizeof(ncclUniqueId) == OOB_NCCL_ID_BYTES, "unique id size");
    std::memcpy(id_out, &id, sizeof(id));
    return OOB_OK;
}

extern "C" oob_status oob_nccl_comm_create(const void *id, int32_t world, int32_t rank, int32_t device,
                                           void **comm_out) {
    if (!id || !comm_out || world < 1 || rank < 0 || rank >= world)
        return fail(OOB_E_INVALID, "oob_nccl_comm_create: bad argument");
    if (device >= 0) {
        cudaError_t e = cudaSetDevice(device);
        if (e != cudaSuccess) return fail(OOB_E_CUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(e));
    }
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof(uid));
    ncclComm_t comm;
    ncclResult_t r = ncclCommInitRank(&comm, world, uid, rank);
    if (r != ncclSuccess) return nccl_fail(r, "ncclCommInitRank");
    *comm_out = comm;
    return OOB_OK;
}

extern "C" void oob_nccl_comm_destroy(void *comm) {
    if (comm) ncclCommDestroy((ncclComm_t)comm);
}

extern "C" oob_status oob_nccl_allgather(void *comm, const void *d_send, void *d_recv, size_t bytes_per_rank,
                                         void *stream) {
    if (!comm || !d_send || !d_recv) return fail(OOB_E_INVALID, "oob_nccl_allgather: NULL argument");
    ncclResult_t r = ncclAllGather(d_send, d_recv, bytes_per_rank, ncclInt8, (ncclComm_t)comm, (cudaStream_t)stream);
    if (r != ncclSuccess) return nccl_fail(r, "ncclAllGather (packed template sets)");
    return OOB_OK;
}
