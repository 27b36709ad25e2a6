// Pinned-memory setup cost on this host: cudaHostAlloc vs mmap + transparent
// huge pages + parallel first touch + cudaHostRegister, for one region size.
// Build: g++ -O2 -std=c++17 tools/pin_probe.cpp -I/usr/local/cuda/include
//        -L/usr/local/cuda/lib64 -lcudart -lpthread -o gpurun_out/pin_probe
#include <sys/mman.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

#include <cuda_runtime.h>

static double now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int main(int argc, char** argv) {
  const size_t gib = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : 16;
  const size_t bytes = gib << 30;
  const int threads = argc > 2 ? std::atoi(argv[2]) : 16;
  cudaFree(nullptr);
  double t0 = now();
  void* a = nullptr;
  if (cudaHostAlloc(&a, bytes, cudaHostAllocPortable) != cudaSuccess) return 1;
  const double t_alloc = now() - t0;
  cudaFreeHost(a);

  for (int huge = 0; huge < 2; ++huge) {
    t0 = now();
    void* p = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
    if (p == MAP_FAILED) return 2;
    if (huge) madvise(p, bytes, MADV_HUGEPAGE);
    std::vector<std::thread> th;
    for (int k = 0; k < threads; ++k)
      th.emplace_back([&, k] {
        const size_t per = bytes / threads, b = k * per, e = k + 1 == threads ? bytes : b + per;
        std::memset(static_cast<char*>(p) + b, 0, e - b);
      });
    for (auto& t : th) t.join();
    const double t_touch = now() - t0;
    t0 = now();
    const cudaError_t r = cudaHostRegister(p, bytes, cudaHostRegisterPortable);
    const double t_reg = now() - t0;
    std::printf("{\"gib\": %zu, \"cudaHostAlloc_s\": %.3f, \"thp\": %d, \"touch_s\": %.3f, \"register_s\": %.3f, "
                "\"register_ok\": %d}\n",
                gib, t_alloc, huge, t_touch, t_reg, r == cudaSuccess);
    if (r == cudaSuccess) cudaHostUnregister(p);
    munmap(p, bytes);
  }
  return 0;
}
