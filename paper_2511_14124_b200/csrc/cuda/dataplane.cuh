// Device-side declarations of the data-plane kernels (sm_100a). Host
// launchers are in dataplane.cu; the C-ABI wrappers in capi/dataplane_capi.cpp.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace tcb {

struct PackSeg {  // device-side fragment with its start in the virtual stream
  std::uint64_t src_off, dst_off, bytes, vstart;
};

struct AdamScalars {
  float b1, b2, omb1, omb2, eps, step_size, inv_sqrt_bc2, decay;
};

AdamScalars adam_scalars(double lr, double b1, double b2, double eps, double wd, std::int64_t step);

// All launchers return cudaGetLastError() of the launch.
cudaError_t launch_adamw(float* p, float* m, float* v, const std::uint16_t* g, std::uint16_t* pout, std::uint64_t n,
                         const AdamScalars& s, float grad_scale, cudaStream_t st);
cudaError_t launch_cast_bf16_to_f32(const std::uint16_t* in, float* out, std::uint64_t n, cudaStream_t st);
cudaError_t launch_cast_f32_to_bf16(const float* in, std::uint16_t* out, std::uint64_t n, cudaStream_t st);
// inverse = false: dst[dst_off..] <- src[src_off..]; true: dst[src_off..] <- src[dst_off..]
cudaError_t launch_pack(const PackSeg* segs, std::uint32_t n, std::uint64_t total, const void* src, void* dst,
                        bool inverse, bool aligned16, cudaStream_t st);
// max_ctas > 0 caps the grid (the forward/backward stand-in leaves SMs to concurrent kernels).
cudaError_t launch_checksum(const void* data, std::uint64_t bytes, unsigned long long* out, cudaStream_t st,
                            int max_ctas = 0);
cudaError_t launch_spin(std::uint64_t ns, int ctas, cudaStream_t st);
// Deterministic N(0, sigma) bf16 fill (counter-based RNG keyed by seed, stream).
cudaError_t launch_fill_normal_bf16(std::uint16_t* out, std::uint64_t n, float sigma, std::uint64_t seed,
                                    std::uint64_t stream_id, cudaStream_t st);
// Optimizer-state init from bf16 params: p32 = float(param), m = v = 0.
cudaError_t launch_init_state(const std::uint16_t* param, float* state, std::uint64_t n, cudaStream_t st);

int num_sms();
// AdamW kernel variant: 0 register-unrolled, 1 register-lean one wave, 2 TMA bulk pipeline.
void set_adamw_variant(int v);
int adamw_variant();

}  // namespace tcb
