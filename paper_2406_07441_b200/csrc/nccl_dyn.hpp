// NCCL entry points resolved at run time (dlopen), so libkf.so has no hard
// dependency on a particular libnccl: inside a PyTorch process it binds to the
// NCCL torch already loaded; elsewhere to the system libnccl.so.2.
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

namespace kfb {

struct NcclApi {
    ncclResult_t (*GetUniqueId)(ncclUniqueId*);
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
    ncclResult_t (*CommDestroy)(ncclComm_t);
    ncclResult_t (*GroupStart)();
    ncclResult_t (*GroupEnd)();
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t);
    const char* (*GetErrorString)(ncclResult_t);
};

// Throws SolverError(KF_CUDA) when no libnccl can be loaded.
const NcclApi& nccl();
void nccl_check(ncclResult_t r, const char* what);

}  // namespace kfb
