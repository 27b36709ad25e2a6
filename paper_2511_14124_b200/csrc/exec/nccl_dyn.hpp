// NCCL, loaded at run time. The process may already hold torch's libnccl.so.2
// (torch.distributed); dlopen by soname then returns that same copy, so our
// communicator and torch's never come from two different NCCL builds. Only
// the handful of entry points the ZeRO-3 exchange needs are resolved.
#pragma once

#include <nccl.h>

#include <string>

namespace tcb {

struct Nccl {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*ReduceScatter)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                                cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*GetVersion)(int*) = nullptr;
};

// Throws DeviceError(TC_ENCCL) when no libnccl.so.2 can be loaded.
const Nccl& nccl();
void nccl_check(ncclResult_t r, const char* what);

}  // namespace tcb
