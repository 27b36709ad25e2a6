#include "nccl_dyn.hpp"

#include <dlfcn.h>

#include <mutex>

#include "capi_common.hpp"

namespace tcb {

namespace {

template <typename F>
void bind(void* h, F& fn, const char* name) {
  fn = reinterpret_cast<F>(dlsym(h, name));
  if (fn == nullptr) throw DeviceError(TC_ENCCL, std::string("libnccl: missing symbol ") + name);
}

}  // namespace

const Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  static std::string err;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (h == nullptr) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (h == nullptr) {
      err = std::string("cannot load libnccl.so.2: ") + dlerror();
      return;
    }
    try {
      bind(h, n.GetUniqueId, "ncclGetUniqueId");
      bind(h, n.CommInitRank, "ncclCommInitRank");
      bind(h, n.CommDestroy, "ncclCommDestroy");
      bind(h, n.AllGather, "ncclAllGather");
      bind(h, n.ReduceScatter, "ncclReduceScatter");
      bind(h, n.GetErrorString, "ncclGetErrorString");
      bind(h, n.GetVersion, "ncclGetVersion");
    } catch (const std::exception& e) {
      err = e.what();
      n = Nccl{};
    }
  });
  if (n.AllGather == nullptr) throw DeviceError(TC_ENCCL, err);
  return n;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) throw DeviceError(TC_ENCCL, std::string(what) + ": " + nccl().GetErrorString(r));
}

}  // namespace tcb
