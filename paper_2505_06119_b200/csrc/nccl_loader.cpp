#include "nccl_loader.h"

#include <dlfcn.h>

#include <cstdlib>
#include <mutex>
#include <string>

#include "common.h"

namespace qtnhb {

namespace {
Nccl g_nccl{};
bool g_loaded = false;
std::mutex g_mu;

void* sym(void* h, const char* name) {
  void* p = dlsym(h, name);
  if (!p) throw_runtime(std::string("NCCL symbol missing: ") + name);
  return p;
}
}  // namespace

const Nccl& nccl() {
  std::lock_guard<std::mutex> lk(g_mu);
  if (g_loaded) return g_nccl;
  // QTNH_NCCL_LIB names a specific build; otherwise the libnccl.so.2 already in
  // the process (torch's) is reused, and only then one is loaded by soname.
  void* h = nullptr;
  if (const char* lib = std::getenv("QTNH_NCCL_LIB")) h = dlopen(lib, RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) throw_runtime("cannot load libnccl.so.2");
  g_nccl.GetUniqueId = reinterpret_cast<decltype(g_nccl.GetUniqueId)>(sym(h, "ncclGetUniqueId"));
  g_nccl.CommInitRank = reinterpret_cast<decltype(g_nccl.CommInitRank)>(sym(h, "ncclCommInitRank"));
  g_nccl.CommDestroy = reinterpret_cast<decltype(g_nccl.CommDestroy)>(sym(h, "ncclCommDestroy"));
  g_nccl.CommAbort = reinterpret_cast<decltype(g_nccl.CommAbort)>(sym(h, "ncclCommAbort"));
  g_nccl.CommGetAsyncError =
      reinterpret_cast<decltype(g_nccl.CommGetAsyncError)>(sym(h, "ncclCommGetAsyncError"));
  g_nccl.CommInitRankConfig = reinterpret_cast<decltype(g_nccl.CommInitRankConfig)>(dlsym(h, "ncclCommInitRankConfig"));
  g_nccl.Send = reinterpret_cast<decltype(g_nccl.Send)>(sym(h, "ncclSend"));
  g_nccl.Recv = reinterpret_cast<decltype(g_nccl.Recv)>(sym(h, "ncclRecv"));
  g_nccl.GroupStart = reinterpret_cast<decltype(g_nccl.GroupStart)>(sym(h, "ncclGroupStart"));
  g_nccl.GroupEnd = reinterpret_cast<decltype(g_nccl.GroupEnd)>(sym(h, "ncclGroupEnd"));
  g_nccl.GetErrorString = reinterpret_cast<decltype(g_nccl.GetErrorString)>(sym(h, "ncclGetErrorString"));
  g_loaded = true;
  return g_nccl;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw_runtime(std::string("NCCL ") + what + ": " + nccl().GetErrorString(r));
}

}  // namespace qtnhb
