// The layer compute the migration path does not own, as real tensor-core
// work: bf16 GEMMs Y[M,N] = X[M,K] * W[K,N] whose weight matrix W is the
// migrated parameter chunk itself, with M chosen so the GEMMs occupy the GPU
// for the trace step's compute_us (trace.hpp:38). This loads SMs, tensor
// cores and HBM the way a layer's forward/backward would, so migration
// overlap and the in-step AdamW are measured under contention (a nanosleep
// spin occupies nothing). cuBLAS (a plain library GEMM) is loaded at run
// time by soname, so the process shares torch's copy when one is loaded.
//
// Closed loop: the rows per step come from the GEMM rate measured in the run
// itself (CUDA events around each step's GEMMs, read back without blocking a
// few steps later), not from the rate alone at full clocks. Under concurrent
// PCIe DMA, the AdamW kernels and the power cap that dense GEMMs drive the
// B200 into, the alone rate would overshoot compute_us by ~30 %; the loop
// keeps the GPU busy for the modelled compute_us.
#pragma once

#include <cstdint>
#include <deque>
#include <string>

#include <cuda_runtime.h>

namespace tcb {

class GemmStandin {
 public:
  GemmStandin(int device, std::uint64_t chunk_bytes, double max_us);
  ~GemmStandin();
  GemmStandin(const GemmStandin&) = delete;
  GemmStandin& operator=(const GemmStandin&) = delete;

  // Enqueue GEMMs reading `weights` (>= chunk_bytes) on `s` for ~us microseconds.
  // Returns the number of GEMM launches.
  int run(cudaStream_t s, const void* weights, double us);
  double flops_issued() const { return flops_; }
  double calibrated_tflops() const { return tflops_; }
  double loaded_tflops() const { return rate_tflops_; }
  int K() const { return K_; }
  int N() const { return N_; }
  int max_M() const { return max_m_; }
  std::string describe() const;

 private:
  void gemm(cudaStream_t s, const void* w, int M);
  int device_ = 0;
  void* handle_ = nullptr;  // cublasHandle_t
  void* x_ = nullptr;       // X [max_M x K] bf16
  void* y_ = nullptr;       // Y [max_M x N] bf16
  void* ws_ = nullptr;      // cuBLAS workspace
  int K_ = 0, N_ = 0, max_m_ = 0;
  double tflops_ = 0;       // measured alone at construction
  double flops_ = 0;
  // closed loop: (start, end, flops) of recent steps; the rate over the
  // completed window sizes the next steps
  struct Sample {
    cudaEvent_t e0, e1;
    double flops;
  };
  std::deque<Sample> inflight_;
  std::deque<std::pair<double, double>> window_;  // (flops, seconds) of completed steps
  double win_flops_ = 0, win_s_ = 0;
  double rate_tflops_ = 0;  // current estimate under load (starts at the alone rate)
  bool open_loop_ = false;
  std::deque<cudaEvent_t> spare_events_;
  void poll(bool block_oldest);
  cudaEvent_t event();
};

}  // namespace tcb
