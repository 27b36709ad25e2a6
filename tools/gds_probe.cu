// GDS probe for the NVMe tier (§8f-2): can cuFile move tier bytes straight
// between a file and HBM on these boxes, and how fast? Writes GB GiB from a
// device buffer with cuFileWrite over T threads (disjoint 16 MiB pieces),
// reads them back into a second device buffer with cuFileRead, compares the
// two buffers on the device, and prints one JSON line. Reports the cuFile
// driver properties (nvidia-fs present or compatibility mode).
//   nvcc -O2 -std=c++17 -gencode arch=compute_100a,code=sm_100a tools/gds_probe.cu -o gpurun_out/gds_probe -lcufile -lcuda
//   gds_probe DIR [GB] [THREADS] [direct 0/1]
#include <cuda.h>
#include <cuda_runtime.h>
#include <cufile.h>
#include <fcntl.h>
#include <unistd.h>

#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <thread>
#include <vector>

static void stage(const char* m) {  // progress on stderr (where a hang sits)
  std::fprintf(stderr, "[gds_probe] %s\n", m);
  std::fflush(stderr);
}

static double now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

__global__ void fill(unsigned* p, size_t n) {
  for (size_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
    p[i] = unsigned(i * 2654435761u) ^ 0x5bd1e995u;
}
__global__ void diff(const unsigned* a, const unsigned* b, size_t n, unsigned long long* bad) {
  for (size_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
    if (a[i] != b[i]) atomicAdd(bad, 1ull);
}

int main(int argc, char** argv) {
  const std::string dir = argc > 1 ? argv[1] : "/tmp";
  const size_t bytes = size_t(argc > 2 ? atoi(argv[2]) : 4) << 30;
  const int threads = argc > 3 ? atoi(argv[3]) : 8;
  const bool direct = argc > 4 ? atoi(argv[4]) != 0 : true;
  const size_t piece = 16ull << 20;
  cudaSetDevice(0);
  stage("cuFileDriverOpen");
  CUfileError_t st = cuFileDriverOpen();
  if (st.err != CU_FILE_SUCCESS) {
    std::printf("{\"gds\": \"cuFileDriverOpen failed\", \"err\": %d}\n", int(st.err));
    return 0;
  }
  CUfileDrvProps_t props{};
  cuFileDriverGetProperties(&props);
  const std::string path = dir + "/gds_probe.bin";
  const int fd = open(path.c_str(), O_RDWR | O_CREAT | O_TRUNC | (direct ? O_DIRECT : 0), 0600);
  if (fd < 0) {
    std::printf("{\"gds\": \"open failed\"}\n");
    return 0;
  }
  if (ftruncate(fd, off_t(bytes)) != 0) return 1;
  CUfileDescr_t d{};
  d.handle.fd = fd;
  d.type = CU_FILE_HANDLE_TYPE_OPAQUE_FD;
  CUfileHandle_t h;
  stage("cuFileHandleRegister");
  st = cuFileHandleRegister(&h, &d);
  if (st.err != CU_FILE_SUCCESS) {
    std::printf("{\"gds\": \"cuFileHandleRegister failed\", \"err\": %d}\n", int(st.err));
    unlink(path.c_str());
    return 0;
  }
  void *a = nullptr, *b = nullptr;
  cudaMalloc(&a, bytes);
  cudaMalloc(&b, bytes);
  cudaMemset(b, 0, bytes);
  fill<<<148 * 8, 256>>>(static_cast<unsigned*>(a), bytes / 4);
  cudaDeviceSynchronize();
  stage("cuFileBufRegister");
  const bool reg_a = cuFileBufRegister(a, bytes, 0).err == CU_FILE_SUCCESS;
  const bool reg_b = cuFileBufRegister(b, bytes, 0).err == CU_FILE_SUCCESS;
  auto run = [&](bool write, void* buf) {
    std::atomic<size_t> next{0};
    std::atomic<long> errors{0};
    std::vector<std::thread> ts;
    const double t0 = now();
    for (int t = 0; t < threads; ++t)
      ts.emplace_back([&] {
        cudaSetDevice(0);
        for (size_t off; (off = next.fetch_add(piece)) < bytes;) {
          const size_t n = std::min(piece, bytes - off);
          const ssize_t r = write ? cuFileWrite(h, buf, n, off_t(off), off_t(off))
                                  : cuFileRead(h, buf, n, off_t(off), off_t(off));
          if (r != ssize_t(n)) errors.fetch_add(1);
        }
      });
    for (auto& t : ts) t.join();
    return std::make_pair(bytes / (now() - t0) / 1e9, errors.load());
  };
  stage("cuFileWrite");
  const auto w = run(true, a);
  stage("cuFileRead");
  const auto r = run(false, b);
  unsigned long long* bad;
  cudaMallocManaged(&bad, 8);
  *bad = 0;
  diff<<<148 * 8, 256>>>(static_cast<unsigned*>(a), static_cast<unsigned*>(b), bytes / 4, bad);
  cudaDeviceSynchronize();
  std::printf(
      "{\"gds\": \"ok\", \"nvfs_major\": %u, \"nvfs_minor\": %u, \"compat_mode_hint\": \"%s\", \"bytes\": %zu, "
      "\"threads\": %d, \"o_direct\": %s, \"buf_registered\": %s, \"write_GBps\": %.2f, \"read_GBps\": %.2f, "
      "\"io_errors\": %ld, \"mismatched_words\": %llu}\n",
      props.nvfs.major_version, props.nvfs.minor_version,
      props.nvfs.major_version == 0 ? "nvidia-fs absent: cuFile compatibility mode (POSIX I/O + bounce)" : "nvidia-fs",
      bytes, threads, direct ? "true" : "false", reg_a && reg_b ? "true" : "false", w.first, r.first,
      w.second + r.second, *bad);
  cuFileBufDeregister(a);
  cuFileBufDeregister(b);
  cuFileHandleDeregister(h);
  close(fd);
  unlink(path.c_str());
  cuFileDriverClose();
  return 0;
}
