// extern "C" surface of the sm_100a data-plane kernels (include/tencache_c.h,
// "data plane" block). No CPU fallback: without a device every call returns
// TC_ECUDA.
#include <vector>

#include <cuda_runtime.h>

#include "capi_common.hpp"
#include "dataplane.cuh"

using namespace tcb;

struct tc_pack_plan {
  PackSeg* dev = nullptr;
  std::uint32_t n = 0;
  std::uint64_t total = 0;
  bool vec16 = true;
};

namespace {

int cuda_status(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return TC_OK;
  return set_error(TC_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }

}  // namespace

extern "C" {

int tc_pack_plan_create(const tc_segment* segs, uint32_t n, tc_pack_plan** out) {
  TC_GUARD({
    if (out == nullptr || (n && segs == nullptr)) return set_error(TC_EARG, "tc_pack_plan_create: null argument");
    auto plan = std::make_unique<tc_pack_plan>();
    std::vector<PackSeg> host(n);
    std::uint64_t v = 0;
    for (uint32_t k = 0; k < n; ++k) {
      host[k] = PackSeg{segs[k].src_off, segs[k].dst_off, segs[k].bytes, v};
      v += segs[k].bytes;
      plan->vec16 = plan->vec16 && ((segs[k].src_off | segs[k].dst_off | segs[k].bytes) % 16 == 0);
    }
    plan->n = n;
    plan->total = v;
    if (n) {
      if (int rc = cuda_status(cudaMalloc(&plan->dev, sizeof(PackSeg) * n), "cudaMalloc(pack plan)")) return rc;
      if (int rc = cuda_status(cudaMemcpy(plan->dev, host.data(), sizeof(PackSeg) * n, cudaMemcpyHostToDevice),
                               "cudaMemcpy(pack plan)")) {
        cudaFree(plan->dev);
        return rc;
      }
    }
    *out = plan.release();
    return TC_OK;
  })
}

void tc_pack_plan_destroy(tc_pack_plan* plan) {
  if (plan == nullptr) return;
  if (plan->dev) cudaFree(plan->dev);
  delete plan;
}

uint64_t tc_pack_plan_bytes(const tc_pack_plan* plan) { return plan ? plan->total : 0; }

int tc_pack(const tc_pack_plan* plan, const void* src_base, void* dst_base, void* stream) {
  if (plan == nullptr) return set_error(TC_EARG, "tc_pack: null plan");
  return cuda_status(launch_pack(plan->dev, plan->n, plan->total, src_base, dst_base, false, plan->vec16,
                                 as_stream(stream)),
                     "tc_pack");
}

int tc_unpack(const tc_pack_plan* plan, const void* src_base, void* dst_base, void* stream) {
  if (plan == nullptr) return set_error(TC_EARG, "tc_unpack: null plan");
  return cuda_status(launch_pack(plan->dev, plan->n, plan->total, src_base, dst_base, true, plan->vec16,
                                 as_stream(stream)),
                     "tc_unpack");
}

int tc_cast_bf16_to_f32(const void* in, float* out, uint64_t n, void* stream) {
  return cuda_status(launch_cast_bf16_to_f32(static_cast<const std::uint16_t*>(in), out, n, as_stream(stream)),
                     "tc_cast_bf16_to_f32");
}

int tc_cast_f32_to_bf16(const float* in, void* out, uint64_t n, void* stream) {
  return cuda_status(launch_cast_f32_to_bf16(in, static_cast<std::uint16_t*>(out), n, as_stream(stream)),
                     "tc_cast_f32_to_bf16");
}

int tc_adamw_split(float* p32, float* m, float* v, const void* grad, void* param_out, uint64_t n, double lr,
                   double beta1, double beta2, double eps, double weight_decay, int64_t step, float grad_scale,
                   void* stream) {
  if (step < 1) return set_error(TC_EARG, "tc_adamw: step must be >= 1");
  if (n == 0) return TC_OK;
  if (!p32 || !m || !v || !grad) return set_error(TC_EARG, "tc_adamw: null buffer");
  const AdamScalars s = adam_scalars(lr, beta1, beta2, eps, weight_decay, step);
  return cuda_status(launch_adamw(p32, m, v, static_cast<const std::uint16_t*>(grad),
                                  static_cast<std::uint16_t*>(param_out), n, s, grad_scale, as_stream(stream)),
                     "tc_adamw");
}

int tc_adamw(float* state, const void* grad, void* param_out, uint64_t n, double lr, double beta1, double beta2,
             double eps, double weight_decay, int64_t step, float grad_scale, void* stream) {
  return tc_adamw_split(state, state + n, state + 2 * n, grad, param_out, n, lr, beta1, beta2, eps, weight_decay,
                        step, grad_scale, stream);
}

int tc_adamw_batch(const tc_adam_chunk* chunks, uint32_t count, double lr, double beta1, double beta2, double eps,
                   double weight_decay, int64_t step, float grad_scale, void* stream) {
  if (count > static_cast<uint32_t>(kMaxAdamChunks) || (count && chunks == nullptr))
    return set_error(TC_EARG, "tc_adamw_batch: 0..8 chunks");
  AdamChunk c[kMaxAdamChunks];
  for (uint32_t k = 0; k < count; ++k) {
    const std::uint64_t n = chunks[k].n;
    c[k] = AdamChunk{chunks[k].state, chunks[k].state + n, chunks[k].state + 2 * n,
                     static_cast<const std::uint16_t*>(chunks[k].grad), static_cast<std::uint16_t*>(chunks[k].param_out), n};
  }
  const cudaError_t e = launch_adamw_batch(c, static_cast<int>(count), adam_scalars(lr, beta1, beta2, eps, weight_decay, step),
                                           grad_scale, as_stream(stream));
  if (e == cudaErrorInvalidValue) {
    cudaGetLastError();
    return set_error(TC_EARG, "tc_adamw_batch: every chunk needs n % 8 == 0 and 16-byte aligned pointers");
  }
  return cuda_status(e, "tc_adamw_batch");
}

uint64_t tc_split_state_bytes(uint64_t n) { return packed_layout(n).bytes; }

int tc_adamw_split_master(void* split_state, const void* grad, void* param, uint64_t n, double lr, double beta1,
                          double beta2, double eps, double weight_decay, int64_t step, float grad_scale,
                          void* stream) {
  if (step < 1) return set_error(TC_EARG, "tc_adamw_split_master: step must be >= 1");
  if (n % kSplitTile) return set_error(TC_EARG, "tc_adamw_split_master: n must be a multiple of 2048");
  if (n == 0) return TC_OK;
  if (!split_state || !grad || !param) return set_error(TC_EARG, "tc_adamw_split_master: null buffer");
  auto* b = static_cast<std::uint8_t*>(split_state);
  AdamChunk c{nullptr, nullptr, nullptr, static_cast<const std::uint16_t*>(grad), static_cast<std::uint16_t*>(param), n,
              b, b + packed_layout(n).ovf};
  const cudaError_t e = launch_adamw_batch(&c, 1, adam_scalars(lr, beta1, beta2, eps, weight_decay, step), grad_scale,
                                           as_stream(stream));
  if (e == cudaErrorInvalidValue) {
    cudaGetLastError();
    return set_error(TC_EARG, "tc_adamw_split_master: buffers must be 16-byte aligned");
  }
  return cuda_status(e, "tc_adamw_split_master");
}

int tc_state_expand(const void* split_state, const void* param, float* full_state, uint64_t n, void* stream) {
  if (n % kSplitTile) return set_error(TC_EARG, "tc_state_expand: n must be a multiple of 2048");
  return cuda_status(launch_state_expand(static_cast<const std::uint8_t*>(split_state),
                                         static_cast<const std::uint16_t*>(param), full_state, n, as_stream(stream)),
                     "tc_state_expand");
}

int tc_state_compress(const float* full_state, const void* param, void* split_state, uint64_t n,
                      uint32_t* d_mismatch, void* stream) {
  if (n % kSplitTile || d_mismatch == nullptr)
    return set_error(TC_EARG, "tc_state_compress: n must be a multiple of 2048 and d_mismatch non-null");
  return cuda_status(launch_state_compress(full_state, static_cast<const std::uint16_t*>(param),
                                           static_cast<std::uint8_t*>(split_state), n, d_mismatch, as_stream(stream)),
                     "tc_state_compress");
}

int tc_adamw_scalars(double lr, double beta1, double beta2, double eps, double weight_decay, int64_t step,
                     float out[8]) {
  const AdamScalars s = adam_scalars(lr, beta1, beta2, eps, weight_decay, step);
  const float v[8] = {s.b1, s.b2, s.omb1, s.omb2, s.eps, s.step_size, s.inv_sqrt_bc2, s.decay};
  for (int i = 0; i < 8; ++i) out[i] = v[i];
  return TC_OK;
}

int tc_checksum(const void* data, uint64_t bytes, uint64_t* out, void* stream) {
  if (bytes % 4) return set_error(TC_EARG, "tc_checksum: bytes must be a multiple of 4");
  return cuda_status(launch_checksum(data, bytes, reinterpret_cast<unsigned long long*>(out), as_stream(stream)),
                     "tc_checksum");
}

int tc_fill_normal_bf16(void* out, uint64_t n, float sigma, uint64_t seed, uint64_t stream_id, void* stream) {
  return cuda_status(launch_fill_normal_bf16(static_cast<std::uint16_t*>(out), n, sigma, seed, stream_id,
                                             as_stream(stream)),
                     "tc_fill_normal_bf16");
}

int tc_spin(double us, int ctas, void* stream) {
  return cuda_status(launch_spin(static_cast<std::uint64_t>(us * 1000.0), ctas, as_stream(stream)), "tc_spin");
}

}  // extern "C"
