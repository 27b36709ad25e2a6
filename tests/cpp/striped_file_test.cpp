// NVMe tier backing store (csrc/exec/nvme_io.hpp StripedFile): a logical byte
// range striped over K files in 16 MiB stripes. Writes random extents that
// cross stripe and file boundaries through io(), reads them back through io()
// and through the raw per-file layout (file = stripe % K, offset = (stripe / K)
// * stripe + within), and prints "ok". CPU only (no CUDA call).
#include <cstdio>
#include <cstring>
#include <random>
#include <vector>

#include "nvme_io.hpp"

using tcb::StripedFile;

int main(int argc, char** argv) {
  const std::string dir = argc > 1 ? argv[1] : "/tmp";
  const std::uint64_t S = StripedFile::kStripe;
  for (int files : {1, 3, 16}) {
    const std::uint64_t total = 40 * S + 12345;
    StripedFile f(dir, total, files, false);
    if (f.files() != files) return 1;
    std::mt19937_64 rng(files);
    std::vector<std::uint8_t> shadow(total, 0);
    for (int k = 0; k < 40; ++k) {
      const std::uint64_t off = rng() % (total - 1), len = 1 + rng() % std::min<std::uint64_t>(3 * S, total - off);
      std::vector<std::uint8_t> buf(len);
      for (auto& b : buf) b = static_cast<std::uint8_t>(rng());
      if (!f.io(true, buf.data(), len, off)) return 2;
      std::memcpy(shadow.data() + off, buf.data(), len);
    }
    std::vector<std::uint8_t> back(total);
    if (!f.io(false, back.data(), total, 0)) return 3;
    if (back != shadow) {
      std::printf("mismatch with %d files\n", files);
      return 4;
    }
  }
  std::printf("ok\n");
  return 0;
}
