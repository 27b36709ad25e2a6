#include "gds.hpp"

#include <cufile.h>
#include <dlfcn.h>
#include <sys/stat.h>

#include <map>
#include <mutex>

#include "capi_common.hpp"

namespace tcb {

namespace {

struct CuFile {
  CUfileError_t (*DriverOpen)() = nullptr;
  CUfileError_t (*HandleRegister)(CUfileHandle_t*, CUfileDescr_t*) = nullptr;
  void (*HandleDeregister)(CUfileHandle_t) = nullptr;
  ssize_t (*Read)(CUfileHandle_t, void*, size_t, off_t, off_t) = nullptr;
  ssize_t (*Write)(CUfileHandle_t, const void*, size_t, off_t, off_t) = nullptr;
};

struct State {
  std::once_flag once;
  bool ok = false;
  std::string why;
  CuFile f;
  std::mutex mu;
  std::map<int, CUfileHandle_t> handles;
};

State& state() {
  static State s;
  return s;
}

bool path_exists(const char* p) {
  struct stat st;
  return stat(p, &st) == 0;
}

void probe(State& s) {
  const char* env = std::getenv("TC_GDS");
  if (env && std::string(env) == "0") {
    s.why = "disabled (TC_GDS=0)";
    return;
  }
  if (!path_exists("/proc/driver/nvidia-fs")) {  // compatibility mode only: not GDS (and hangs on this pool)
    s.why = "no nvidia-fs kernel driver (/proc/driver/nvidia-fs absent)";
    return;
  }
  void* h = dlopen("libcufile.so.0", RTLD_NOW | RTLD_GLOBAL);
  if (h == nullptr) {
    s.why = std::string("cannot load libcufile.so.0: ") + dlerror();
    return;
  }
  auto sym = [&](const char* n) { return dlsym(h, n); };
  s.f.DriverOpen = reinterpret_cast<decltype(s.f.DriverOpen)>(sym("cuFileDriverOpen"));
  s.f.HandleRegister = reinterpret_cast<decltype(s.f.HandleRegister)>(sym("cuFileHandleRegister"));
  s.f.HandleDeregister = reinterpret_cast<decltype(s.f.HandleDeregister)>(sym("cuFileHandleDeregister"));
  s.f.Read = reinterpret_cast<decltype(s.f.Read)>(sym("cuFileRead"));
  s.f.Write = reinterpret_cast<decltype(s.f.Write)>(sym("cuFileWrite"));
  if (!s.f.DriverOpen || !s.f.HandleRegister || !s.f.Read || !s.f.Write) {
    s.why = "libcufile.so.0: missing symbols";
    return;
  }
  const CUfileError_t e = s.f.DriverOpen();
  if (e.err != CU_FILE_SUCCESS) {
    s.why = "cuFileDriverOpen failed (" + std::to_string(static_cast<int>(e.err)) + ")";
    return;
  }
  s.ok = true;
}

}  // namespace

bool Gds::available(std::string* why) {
  State& s = state();
  std::call_once(s.once, [&] { probe(s); });
  if (why) *why = s.ok ? "" : s.why;
  return s.ok;
}

Gds& Gds::get() {
  static Gds g;
  if (!available()) throw DeviceError(TC_ECONFIG, "GPUDirect Storage unavailable: " + state().why);
  return g;
}

void* Gds::handle(int fd) {
  State& s = state();
  std::lock_guard<std::mutex> g(s.mu);
  auto it = s.handles.find(fd);
  if (it != s.handles.end()) return it->second;
  CUfileDescr_t d{};
  d.handle.fd = fd;
  d.type = CU_FILE_HANDLE_TYPE_OPAQUE_FD;
  CUfileHandle_t h = nullptr;
  const CUfileError_t e = s.f.HandleRegister(&h, &d);
  if (e.err != CU_FILE_SUCCESS)
    throw DeviceError(TC_EIO, "cuFileHandleRegister failed (" + std::to_string(static_cast<int>(e.err)) + ")");
  s.handles[fd] = h;
  return h;
}

void Gds::release(int fd) {
  State& s = state();
  if (!s.ok) return;
  std::lock_guard<std::mutex> g(s.mu);
  auto it = s.handles.find(fd);
  if (it == s.handles.end()) return;
  if (s.f.HandleDeregister) s.f.HandleDeregister(it->second);
  s.handles.erase(it);
}

bool Gds::read(void* fh, void* dev, std::uint64_t bytes, std::uint64_t file_off) {
  for (std::uint64_t done = 0; done < bytes;) {
    const ssize_t r = state().f.Read(static_cast<CUfileHandle_t>(fh), dev, bytes - done,
                                     static_cast<off_t>(file_off + done), static_cast<off_t>(done));
    if (r <= 0) return false;
    done += static_cast<std::uint64_t>(r);
  }
  return true;
}

bool Gds::write(void* fh, const void* dev, std::uint64_t bytes, std::uint64_t file_off) {
  for (std::uint64_t done = 0; done < bytes;) {
    const ssize_t r = state().f.Write(static_cast<CUfileHandle_t>(fh), dev, bytes - done,
                                      static_cast<off_t>(file_off + done), static_cast<off_t>(done));
    if (r <= 0) return false;
    done += static_cast<std::uint64_t>(r);
  }
  return true;
}

}  // namespace tcb
