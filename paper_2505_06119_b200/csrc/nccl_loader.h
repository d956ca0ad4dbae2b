// Lazy NCCL binding. The library must load on boxes without NCCL and must not
// pin a second libnccl next to the one torch already loaded, so the symbols are
// resolved with dlopen/dlsym on first use (prefer an already-loaded
// libnccl.so.2, RTLD_NOLOAD).
#pragma once

#include <nccl.h>

namespace qtnhb {

struct Nccl {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*);
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
  ncclResult_t (*CommDestroy)(ncclComm_t);
  ncclResult_t (*CommAbort)(ncclComm_t);
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*);
  // non-blocking initialisation (NCCL >= 2.14); null when absent
  ncclResult_t (*CommInitRankConfig)(ncclComm_t*, int, ncclUniqueId, int, ncclConfig_t*);
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*GroupStart)();
  ncclResult_t (*GroupEnd)();
  const char* (*GetErrorString)(ncclResult_t);
};

// Throws Status(QTNH_E_RUNTIME) when NCCL cannot be loaded.
const Nccl& nccl();
void nccl_check(ncclResult_t r, const char* what);

}  // namespace qtnhb
