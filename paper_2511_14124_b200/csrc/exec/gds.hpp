// GPUDirect Storage (cuFile) for the NVMe tier: tier
// bytes move between the striped files and HBM directly, without the pinned
// bounce buffer the reference models as a second leg (machine.cpp:104-107,
// the staging slot of engine.cpp:214-221).
//
// Runtime-gated: libcufile is loaded by soname, and only when the nvidia-fs
// kernel driver is present (/proc/driver/nvidia-fs). Without it cuFile runs
// in compatibility mode — a POSIX read into its own bounce buffer plus a
// copy, i.e. the path the executor already has — and on this pool's boxes
// cuFileDriverOpen does not return in that mode (profiles/r01_gds_probe*),
// so it is never called there. TC_GDS=0 turns it off.
#pragma once

#include <cstdint>
#include <string>

namespace tcb {

class Gds {
 public:
  // True when nvidia-fs is loaded, libcufile resolves and the driver opened
  // (once per process); `why` says what is missing otherwise.
  static bool available(std::string* why = nullptr);
  static Gds& get();  // requires available()

  // A registered handle for an O_DIRECT file descriptor (idempotent per fd).
  void* handle(int fd);
  // Deregister the handle of `fd` before the descriptor is closed (a later
  // file may reuse the number). No-op when GDS never ran or fd has none.
  static void release(int fd);
  // Whole transfer between HBM and a registered file; false on an I/O error.
  bool read(void* fh, void* dev, std::uint64_t bytes, std::uint64_t file_off);
  bool write(void* fh, const void* dev, std::uint64_t bytes, std::uint64_t file_off);
  // (Buffers are not cuFileBufRegister'ed: pieces start at arbitrary slot
  // offsets, and registration would pin devPtr_base to one region base.)

 private:
  Gds() = default;
};

}  // namespace tcb
