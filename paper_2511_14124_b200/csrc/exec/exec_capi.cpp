// C-ABI of the migration executor (include/tencache_c.h, tc_engine_*).
#include "executor.hpp"
#include "gds.hpp"

#include <algorithm>
#include <string>

#include <cstring>

// ------------------------------------------------------------------ C-ABI
struct tc_engine {
  std::unique_ptr<tcb::Executor> ex;
};

using namespace tcb;

extern "C" {

int tc_engine_create(const char* trace_path, const char* machine_path, const char* cfg_json,
                     const tc_engine_options* opts, tc_engine** out) {
  TC_GUARD({
    if (out == nullptr || trace_path == nullptr) return set_error(TC_EARG, "tc_engine_create: null argument");
    tc_engine_options o{};
    o.gpu_spare_slots = 16;
    o.host_spare_slots = 1;
    o.opt_stage_slots = 0;  // auto (Executor::auto_stage_slots)
    o.grad_bytes_per_param_byte = 1;
    if (opts) o = *opts;
    auto e = std::make_unique<tc_engine>();
    e->ex = std::make_unique<Executor>(trace_path, machine_path ? machine_path : "", cfg_json ? cfg_json : "", o);
    *out = e.release();
    return TC_OK;
  })
}

void tc_engine_destroy(tc_engine* e) { delete e; }

int tc_engine_seed(tc_engine* e, uint64_t seed) {
  TC_GUARD({
    e->ex->seed(seed);
    return TC_OK;
  })
}

int tc_engine_read_tensor(tc_engine* e, uint32_t tensor, void* host_dst, uint64_t bytes) {
  TC_GUARD({
    e->ex->read_tensor(tensor, host_dst, bytes);
    return TC_OK;
  })
}

int tc_engine_write_tensor(tc_engine* e, uint32_t tensor, const void* host_src, uint64_t bytes) {
  TC_GUARD({
    e->ex->write_tensor(tensor, host_src, bytes);
    return TC_OK;
  })
}

int tc_engine_read_grad(tc_engine* e, uint32_t tensor, void* host_dst, uint64_t bytes) {
  TC_GUARD({
    void* g = e->ex->grad_ptr(tensor);
    if (g == nullptr) return set_error(TC_EARG, "tensor has no gradient");
    if (bytes != e->ex->tensor_bytes(tensor))
      return set_error(TC_EARG, "tc_engine_read_grad: size mismatch (the gradient has the parameter's size)");
    e->ex->sync();
    TCB_CK(cudaMemcpy(host_dst, g, bytes, cudaMemcpyDeviceToHost));
    return TC_OK;
  })
}

void* tc_engine_gpu_ptr(tc_engine* e, uint32_t tensor) {
  try {
    return e->ex->gpu_ptr(tensor);
  } catch (...) {
    return nullptr;
  }
}

void* tc_engine_grad_ptr(tc_engine* e, uint32_t tensor) {
  try {
    return e->ex->grad_ptr(tensor);
  } catch (...) {
    return nullptr;
  }
}

namespace {
StepOptions step_options(const tc_step_options* so) {
  StepOptions o;
  if (so) {
    o.lr = so->lr;
    o.beta1 = so->beta1;
    o.beta2 = so->beta2;
    o.eps = so->eps;
    o.weight_decay = so->weight_decay;
    o.grad_scale = so->grad_scale;
    o.compute_mode = so->compute_mode;
    o.spin_ctas = so->spin_ctas;
    o.hoist_optimizer = (so->flags & 1) == 0;
    o.prestage = (so->flags & 2) == 0;
    o.prologue = (so->flags & 4) == 0;
  }
  return o;
}
}  // namespace

int tc_engine_iteration(tc_engine* e, const tc_step_options* so, void* compute_stream) {
  TC_GUARD({
    if (!e) return set_error(TC_EARG, "null engine");
    e->ex->iteration(step_options(so), static_cast<cudaStream_t>(compute_stream));
    return TC_OK;
  })
}

int tc_engine_iteration_begin(tc_engine* e, const tc_step_options* so, void* compute_stream) {
  TC_GUARD({
    if (!e) return set_error(TC_EARG, "null engine");
    e->ex->iteration_begin(step_options(so), static_cast<cudaStream_t>(compute_stream), true);
    return TC_OK;
  })
}

int tc_engine_step_begin(tc_engine* e, uint32_t step, void** ptrs, size_t cap, size_t* n) {
  TC_GUARD({
    if (!e) return set_error(TC_EARG, "null engine");
    const std::vector<void*> v = e->ex->step_begin(step);
    if (n) *n = v.size();
    if (v.size() > cap || (!v.empty() && ptrs == nullptr))
      return set_error(TC_ERANGE, "tc_engine_step_begin: the step has " + std::to_string(v.size()) +
                                      " tensors; the step is open, read them with tc_engine_gpu_ptr");
    for (std::size_t i = 0; i < v.size(); ++i) ptrs[i] = v[i];
    return TC_OK;
  })
}

int tc_engine_step_end(tc_engine* e, uint32_t step) {
  TC_GUARD({
    if (!e) return set_error(TC_EARG, "null engine");
    e->ex->step_end(step);
    return TC_OK;
  })
}

int tc_engine_iteration_end(tc_engine* e) {
  TC_GUARD({
    if (!e) return set_error(TC_EARG, "null engine");
    e->ex->iteration_end();
    return TC_OK;
  })
}

int tc_engine_iteration_abort(tc_engine* e) {
  TC_GUARD({
    if (!e) return set_error(TC_EARG, "null engine");
    e->ex->iteration_abort();
    return TC_OK;
  })
}

int tc_engine_regions(tc_engine* e, void** hbm_pool, uint64_t* hbm_pool_bytes, void** grads, uint64_t* grad_bytes) {
  TC_GUARD({
    if (!e) return set_error(TC_EARG, "null engine");
    void* pb = nullptr;
    void* gb = nullptr;
    std::uint64_t pn = 0, gn = 0;
    e->ex->regions(&pb, &pn, &gb, &gn);
    if (hbm_pool) *hbm_pool = pb;
    if (hbm_pool_bytes) *hbm_pool_bytes = pn;
    if (grads) *grads = gb;
    if (grad_bytes) *grad_bytes = gn;
    return TC_OK;
  })
}

int tc_engine_zero3_views(tc_engine* e, void** params, void** grads, uint64_t* layer_bytes) {
  TC_GUARD({
    if (!e) return set_error(TC_EARG, "null engine");
    void* pb = nullptr;
    void* gb = nullptr;
    std::uint64_t n = 0;
    e->ex->zero3_views(&pb, &gb, &n);
    if (params) *params = pb;
    if (grads) *grads = gb;
    if (layer_bytes) *layer_bytes = n;
    return TC_OK;
  })
}

int tc_engine_sync(tc_engine* e) {
  TC_GUARD({
    e->ex->sync();
    return TC_OK;
  })
}

int tc_nccl_unique_id(uint8_t out[128]) {
  TC_GUARD({
    ncclUniqueId id;
    nccl_check(nccl().GetUniqueId(&id), "ncclGetUniqueId");
    std::memcpy(out, id.internal, sizeof(id.internal));
    return TC_OK;
  })
}

int tc_engine_enable_zero3(tc_engine* e, int world, int rank, const uint8_t id[128], const uint64_t* layer_elems,
                           const uint64_t* layer_per, uint32_t n_layers) {
  TC_GUARD({
    if (!e || world < 1 || rank < 0 || rank >= world) return set_error(TC_EARG, "tc_engine_enable_zero3: bad arguments");
    ncclUniqueId nid;
    std::memcpy(nid.internal, id, sizeof(nid.internal));
    e->ex->enable_zero3(world, rank, nid, layer_elems, layer_per, n_layers);
    return TC_OK;
  })
}

uint64_t tc_engine_exchanged_bytes(tc_engine* e) { return e ? e->ex->exchanged_bytes() : 0; }

int tc_gds_available(char* why, size_t cap) {
  std::string w;
  const bool ok = tcb::Gds::available(&w);
  if (why && cap) {
    const size_t n = std::min(cap - 1, w.size());
    std::memcpy(why, w.data(), n);
    why[n] = 0;
  }
  return ok ? 1 : 0;
}

int tc_engine_gds(tc_engine* e) { return e && e->ex->gds() ? 1 : 0; }

int tc_engine_p2p_handles(tc_engine* e, uint8_t* out, size_t cap, size_t* n) {
  TC_GUARD({
    if (!e) return set_error(TC_EARG, "null engine");
    const std::vector<std::uint8_t> b = e->ex->p2p_handles();
    if (n) *n = b.size();
    if (out && cap >= b.size()) std::memcpy(out, b.data(), b.size());
    return TC_OK;
  })
}

int tc_engine_enable_p2p(tc_engine* e, const uint8_t* all_blobs) {
  TC_GUARD({
    if (!e || !all_blobs) return set_error(TC_EARG, "null argument");
    e->ex->enable_p2p(all_blobs);
    return TC_OK;
  })
}

int tc_engine_event_log(tc_engine* e, const char* path) {
  TC_GUARD({
    if (!e) return set_error(TC_EARG, "null engine");
    e->ex->set_event_log(path ? path : "");
    return TC_OK;
  })
}

int tc_engine_stats_get(tc_engine* e, tc_engine_stats* out) {
  TC_GUARD({
    if (!e || !out) return set_error(TC_EARG, "null argument");
    e->ex->sync();
    *out = e->ex->stats();
    return TC_OK;
  })
}

int tc_engine_phase_ms(tc_engine* e, double* out, size_t cap, size_t* n) {
  if (!e) return set_error(TC_EARG, "null argument");
  try {
    e->ex->sync();
  } catch (const std::exception& ex) {
    return set_error(TC_ECUDA, ex.what());
  }
  const auto& v = e->ex->phase_ms();
  for (std::size_t i = 0; i < v.size() && i < cap; ++i) out[i] = v[i];
  if (n) *n = v.size();
  return TC_OK;
}

int tc_engine_standin_info(tc_engine* e, char* out, size_t cap) {
  TC_GUARD({
    if (!e || !out || cap == 0) return set_error(TC_EARG, "null argument");
    const std::string s = e->ex->standin_info();
    if (s.size() + 1 > cap) return set_error(TC_EARG, "tc_engine_standin_info: buffer too small");
    std::memcpy(out, s.c_str(), s.size() + 1);
    return TC_OK;
  })
}

int tc_engine_stats_reset(tc_engine* e) {
  TC_GUARD({
    if (!e) return set_error(TC_EARG, "null argument");
    e->ex->sync();
    e->ex->reset_stats();
    return TC_OK;
  })
}

int tc_engine_step_result(tc_engine* e, uint64_t* out, size_t cap, size_t* n) {
  TC_GUARD({
    if (!e) return set_error(TC_EARG, "null argument");
    if (out == nullptr || cap == 0) {  // size query: no wait
      if (n) *n = e->ex->n_accesses();
      return TC_OK;
    }
    const auto v = e->ex->step_result();
    for (std::size_t i = 0; i < v.size() && i < cap; ++i) out[i] = v[i];
    if (n) *n = v.size();
    return TC_OK;
  })
}

int tc_engine_access_checksums(tc_engine* e, uint64_t* out, size_t cap, size_t* n) {
  TC_GUARD({
    const auto& v = e->ex->access_checksums();
    for (std::size_t i = 0; i < v.size() && i < cap; ++i) out[i] = v[i];
    if (n) *n = v.size();
    return TC_OK;
  })
}

}  // extern "C"
