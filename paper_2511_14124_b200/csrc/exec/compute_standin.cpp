#include "compute_standin.hpp"

#include <cublas_v2.h>
#include <dlfcn.h>

#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <mutex>
#include <vector>

#include "capi_common.hpp"
#include "dataplane.cuh"

namespace tcb {

namespace {

struct Cublas {
  cublasStatus_t (*Create)(cublasHandle_t*) = nullptr;
  cublasStatus_t (*Destroy)(cublasHandle_t) = nullptr;
  cublasStatus_t (*SetStream)(cublasHandle_t, cudaStream_t) = nullptr;
  cublasStatus_t (*SetWorkspace)(cublasHandle_t, void*, size_t) = nullptr;
  cublasStatus_t (*GemmEx)(cublasHandle_t, cublasOperation_t, cublasOperation_t, int, int, int, const void*,
                           const void*, cudaDataType, int, const void*, cudaDataType, int, const void*, void*,
                           cudaDataType, int, cublasComputeType_t, cublasGemmAlgo_t) = nullptr;
};

const Cublas& cublas() {
  static Cublas c;
  static std::once_flag once;
  static std::string err;
  std::call_once(once, [] {
    void* h = dlopen("libcublas.so.12", RTLD_NOW | RTLD_NOLOAD);
    if (h == nullptr) h = dlopen("libcublas.so.12", RTLD_NOW | RTLD_GLOBAL);
    if (h == nullptr) {
      err = std::string("cannot load libcublas.so.12: ") + dlerror();
      return;
    }
    c.Create = reinterpret_cast<decltype(c.Create)>(dlsym(h, "cublasCreate_v2"));
    c.Destroy = reinterpret_cast<decltype(c.Destroy)>(dlsym(h, "cublasDestroy_v2"));
    c.SetStream = reinterpret_cast<decltype(c.SetStream)>(dlsym(h, "cublasSetStream_v2"));
    c.SetWorkspace = reinterpret_cast<decltype(c.SetWorkspace)>(dlsym(h, "cublasSetWorkspace_v2"));
    c.GemmEx = reinterpret_cast<decltype(c.GemmEx)>(dlsym(h, "cublasGemmEx"));
    if (!c.Create || !c.Destroy || !c.SetStream || !c.GemmEx) {
      err = "libcublas.so.12: missing symbols";
      c = Cublas{};
    }
  });
  if (c.GemmEx == nullptr) throw DeviceError(TC_ECUDA, err);
  return c;
}

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw DeviceError(TC_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

void bk(cublasStatus_t s, const char* what) {
  if (s != CUBLAS_STATUS_SUCCESS) throw DeviceError(TC_ECUDA, std::string(what) + ": cublas status " + std::to_string(s));
}

constexpr std::uint64_t kWorkspace = 32ull << 20;

}  // namespace

// W = the chunk's first K*N bf16 elements, K the largest of 4096..128 with
// at least 128 columns, N rounded down to a multiple of 64 (the tail bytes are
// still read by the checksum that precedes the GEMMs).
GemmStandin::GemmStandin(int device, std::uint64_t chunk_bytes, double max_us) : device_(device) {
  const std::uint64_t elems = chunk_bytes / 2;
  for (int k = 4096; k >= 128; k /= 2)
    if (elems / static_cast<std::uint64_t>(k) >= 128) {
      K_ = k;
      break;
    }
  if (K_ == 0) throw DeviceError(TC_ECONFIG, "GEMM stand-in: chunk too small (< 32 KiB)");
  N_ = static_cast<int>(std::min<std::uint64_t>(elems / K_ / 64 * 64, 1u << 20));
  ck(cudaSetDevice(device_), "cudaSetDevice");
  const Cublas& c = cublas();
  cublasHandle_t h = nullptr;
  bk(c.Create(&h), "cublasCreate");
  handle_ = h;
  ck(cudaMalloc(&ws_, kWorkspace), "cudaMalloc(workspace)");
  if (c.SetWorkspace) bk(c.SetWorkspace(h, ws_, kWorkspace), "cublasSetWorkspace");
  max_m_ = 16384;
  ck(cudaMalloc(&x_, static_cast<std::uint64_t>(max_m_) * K_ * 2), "cudaMalloc(X)");
  ck(cudaMalloc(&y_, static_cast<std::uint64_t>(max_m_) * N_ * 2), "cudaMalloc(Y)");
  ck(launch_fill_normal_bf16(static_cast<std::uint16_t*>(x_), static_cast<std::uint64_t>(max_m_) * K_, 1.0f, 7, 0,
                             nullptr), "fill X");
  // calibration alone on a private stream against a scratch weight matrix
  void* w = nullptr;
  ck(cudaMalloc(&w, static_cast<std::uint64_t>(K_) * N_ * 2), "cudaMalloc(W)");
  ck(launch_fill_normal_bf16(static_cast<std::uint16_t*>(w), static_cast<std::uint64_t>(K_) * N_, 0.02f, 8, 0,
                             nullptr), "fill W");
  cudaStream_t s = nullptr;
  ck(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "stream");
  cudaEvent_t e0, e1;
  ck(cudaEventCreate(&e0), "event");
  ck(cudaEventCreate(&e1), "event");
  for (int i = 0; i < 3; ++i) gemm(s, w, max_m_);
  float best = 1e30f;
  for (int i = 0; i < 5; ++i) {
    ck(cudaEventRecord(e0, s), "record");
    gemm(s, w, max_m_);
    ck(cudaEventRecord(e1, s), "record");
    ck(cudaEventSynchronize(e1), "sync");
    float ms = 0;
    ck(cudaEventElapsedTime(&ms, e0, e1), "elapsed");
    best = std::min(best, ms);
  }
  tflops_ = 2.0 * max_m_ * K_ * static_cast<double>(N_) / (best * 1e-3) / 1e12;
  rate_tflops_ = tflops_;
  // TC_STANDIN_OPEN_LOOP=1: keep the alone rate (under a profiler, event
  // times are serialised replays and would shrink the GEMMs)
  open_loop_ = std::getenv("TC_STANDIN_OPEN_LOOP") && std::atoi(std::getenv("TC_STANDIN_OPEN_LOOP")) != 0;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaStreamDestroy(s);
  cudaFree(w);
  flops_ = 0;
  (void)max_us;
}

GemmStandin::~GemmStandin() {
  cudaSetDevice(device_);
  for (const Sample& s : inflight_) {
    cudaEventSynchronize(s.e1);
    cudaEventDestroy(s.e0);
    cudaEventDestroy(s.e1);
  }
  for (cudaEvent_t e : spare_events_) cudaEventDestroy(e);
  if (handle_) cublas().Destroy(static_cast<cublasHandle_t>(handle_));
  for (void* p : {x_, y_, ws_})
    if (p) cudaFree(p);
}

// Row-major Y[M,N] = X[M,K] * W[K,N] is column-major Y^T = W^T X^T.
void GemmStandin::gemm(cudaStream_t s, const void* w, int M) {
  const Cublas& c = cublas();
  auto h = static_cast<cublasHandle_t>(handle_);
  bk(c.SetStream(h, s), "cublasSetStream");
  const float alpha = 1.0f, beta = 0.0f;
  bk(c.GemmEx(h, CUBLAS_OP_N, CUBLAS_OP_N, N_, M, K_, &alpha, w, CUDA_R_16BF, N_, x_, CUDA_R_16BF, K_, &beta, y_,
              CUDA_R_16BF, N_, CUBLAS_COMPUTE_32F, CUBLAS_GEMM_DEFAULT),
     "cublasGemmEx");
  flops_ += 2.0 * M * K_ * static_cast<double>(N_);
}

cudaEvent_t GemmStandin::event() {
  if (!spare_events_.empty()) {
    cudaEvent_t e = spare_events_.front();
    spare_events_.pop_front();
    return e;
  }
  cudaEvent_t e = nullptr;
  ck(cudaEventCreate(&e), "cudaEventCreate");
  return e;
}

// Fold completed steps into the rate window (the last 256 steps); block on
// the oldest only when too many are in flight.
void GemmStandin::poll(bool block_oldest) {
  constexpr std::size_t kWindow = 256, kMaxInflight = 4096;
  while (!inflight_.empty()) {
    Sample& f = inflight_.front();
    if (block_oldest && inflight_.size() > kMaxInflight) ck(cudaEventSynchronize(f.e1), "cudaEventSynchronize");
    const cudaError_t q = cudaEventQuery(f.e1);
    if (q == cudaErrorNotReady) break;
    ck(q, "cudaEventQuery");
    float ms = 0;
    ck(cudaEventElapsedTime(&ms, f.e0, f.e1), "cudaEventElapsedTime");
    if (ms > 0) {
      window_.emplace_back(f.flops, ms * 1e-3);
      win_flops_ += f.flops;
      win_s_ += ms * 1e-3;
      while (window_.size() > kWindow) {
        win_flops_ -= window_.front().first;
        win_s_ -= window_.front().second;
        window_.pop_front();
      }
    }
    spare_events_.push_back(f.e0);
    spare_events_.push_back(f.e1);
    inflight_.pop_front();
  }
  if (window_.size() >= 8 && win_s_ > 0 && !open_loop_) rate_tflops_ = win_flops_ / win_s_ / 1e12;
}

// The FLOPs that occupy the GPU for `us` at the rate measured under load, in
// GEMMs of at most max_M rows (multiples of 64, at least 64).
int GemmStandin::run(cudaStream_t s, const void* weights, double us) {
  if (us <= 0) return 0;
  poll(true);
  const double per_row = 2.0 * K_ * static_cast<double>(N_);
  const double rows = us * 1e-6 * rate_tflops_ * 1e12 / per_row;
  const int n = std::max(1, static_cast<int>(std::ceil(rows / max_m_)));
  const int M = std::clamp(static_cast<int>(std::lround(rows / n / 64.0)) * 64, 64, max_m_);
  Sample smp{event(), event(), 0.0};
  ck(cudaEventRecord(smp.e0, s), "cudaEventRecord");
  const double f0 = flops_;
  for (int i = 0; i < n; ++i) gemm(s, weights, M);
  ck(cudaEventRecord(smp.e1, s), "cudaEventRecord");
  smp.flops = flops_ - f0;
  inflight_.push_back(smp);
  return n;
}

std::string GemmStandin::describe() const {
  return "{\"kind\":\"cuBLAS bf16 GEMM, fp32 accumulate: Y[M,N] = X[M,K] * W[K,N], W = the migrated chunk\","
         "\"K\":" + std::to_string(K_) + ",\"N\":" + std::to_string(N_) + ",\"max_M\":" + std::to_string(max_m_) +
         ",\"calibrated_tflops_alone\":" + std::to_string(tflops_) +
         ",\"tflops_under_load\":" + std::to_string(rate_tflops_) +
         ",\"sizing\":\"closed loop: each step's GEMM rows = compute_us x the GEMM rate measured in this run "
         "(CUDA events, last 256 steps)\"}";
}

}  // namespace tcb
