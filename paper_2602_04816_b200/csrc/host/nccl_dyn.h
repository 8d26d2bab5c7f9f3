// NCCL loaded at run time (dlopen "libnccl.so.2") so single-GPU use carries no
// NCCL dependency. Types come from the system header /usr/include/nccl.h.
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

namespace hlm {
inline namespace b200 {

struct NcclApi {
    ncclResult_t (*GetUniqueId)(ncclUniqueId*);
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
    ncclResult_t (*CommDestroy)(ncclComm_t);
    ncclResult_t (*ReduceScatter)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t);
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t);
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t);
    const char* (*GetErrorString)(ncclResult_t);
};

// Throws CudaError when libnccl.so.2 or a symbol is missing.
const NcclApi& nccl();
void nccl_check(ncclResult_t r, const char* what);

}  // inline namespace b200
}  // namespace hlm
