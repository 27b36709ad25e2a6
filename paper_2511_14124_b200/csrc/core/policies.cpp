// Policy plug-ins behind IPolicy (reference counterpart: policies.cpp:27-265,
// baselines.cpp:1-190). TenCache is the product path; the comparison
// policies (ZeRO-Infinity-like, L2L-like, NoOffload) keep the paper's
// relative claims reproducible on the same executor.
#include <algorithm>

#include "tencache/tencache.hpp"

namespace tencache {

PolicyKind policy_from_string(const std::string& name) {
  static const std::pair<const char*, PolicyKind> kNames[] = {
      {"tencache", PolicyKind::TenCache},          {"tencache+opt", PolicyKind::TenCachePlusOpt},
      {"zero-infinity", PolicyKind::ZeroInfinityLike}, {"l2l", PolicyKind::L2LLike},
      {"no-offload", PolicyKind::NoOffload}};
  for (const auto& [n, k] : kNames)
    if (name == n) return k;
  throw ConfigError("unknown policy: " + name);
}

const char* to_string(PolicyKind kind) {
  switch (kind) {
    case PolicyKind::TenCache: return "tencache";
    case PolicyKind::TenCachePlusOpt: return "tencache+opt";
    case PolicyKind::ZeroInfinityLike: return "zero-infinity";
    case PolicyKind::L2LLike: return "l2l";
    case PolicyKind::NoOffload: return "no-offload";
  }
  return "?";
}

namespace {

using Req = TransferRequest;

std::vector<TensorDescriptor> states_by_update_order(const ExecutionTrace& trace) {
  std::vector<TensorDescriptor> out;
  for (const auto& pr : trace.optimizer_pairs()) out.push_back(trace.tensor(pr.first));
  return out;
}

// Home copy of a baseline parameter is fetched and later dropped for free.
Req home_fetch(const ExecutionTrace& trace, TensorId id, Tier home) {
  Req r;
  r.tensor_id = id;
  r.src = home;
  r.dst = Tier::Gpu;
  r.size_bytes = trace.tensor(id).size_bytes;
  r.kind = Req::Kind::Prefetch;
  r.via_cpu_staging = home == Tier::Nvme;
  r.src_retains = true;
  return r;
}

Req home_drop(const ExecutionTrace& trace, TensorId id, Tier home) {
  Req r;
  r.tensor_id = id;
  r.src = Tier::Gpu;
  r.dst = home;
  r.size_bytes = trace.tensor(id).size_bytes;
  r.kind = Req::Kind::Evict;
  r.instant = true;
  r.dst_has_copy = true;
  return r;
}

void index_param_steps(const ExecutionTrace& trace, std::vector<std::size_t>& order,
                       std::map<std::size_t, std::size_t>& pos) {
  for (std::size_t i = 0; i < trace.steps.size(); ++i)
    if (trace.steps[i].phase != Phase::OptimizerUpdate) {
      pos[i] = order.size();
      order.push_back(i);
    }
}

// ----------------------------------------------------------------- TenCache
class TenCache final : public IPolicy {
 public:
  TenCache(const ExecutionTrace& t, const MachineConfig& m, const RunConfig& c) : trace_(t), machine_(m), cfg_(c) {}

  InitInfo init() override {
    // Alg. 1 + Alg. 2 over the parameter census.
    const TensorCensus census = tensor_census(trace_, TensorKind::ParamFP16);
    BufferPlan plan;
    if (!census.empty())
      plan = plan_buffers(census, size_distribution(census), machine_.gpu_capacity_bytes, machine_.cpu_capacity_bytes);
    check_steps_fit(plan);

    PrefetchTable table = build_prefetch_table(trace_);
    PlacementState params = place_parameters(table, trace_, plan);

    // Optimizer states get what host memory the parameter plan leaves. The
    // base TenCache posture keeps them all in NVMe (synchronous write-back)
    // unless every state fits; +Opt fills the remainder.
    const std::vector<TensorDescriptor> states = states_by_update_order(trace_);
    const std::uint64_t remaining = machine_.cpu_capacity_bytes - plan.cpu_planned_bytes();
    std::uint64_t state_bytes = 0;
    for (const auto& s : states) state_bytes += s.size_bytes;
    const bool base_posture = cfg_.policy == PolicyKind::TenCache;
    const std::uint64_t budget = (base_posture && state_bytes > remaining) ? 0 : remaining;
    PlacementState opt = place_optimizer_states(states, budget);
    sync_writeback_ = budget == 0 && !states.empty();

    std::map<std::uint64_t, std::uint64_t> opt_slots;
    for (const auto& s : states)
      if (opt.location_of.at(s.id) == Tier::Cpu) ++opt_slots[s.size_bytes];

    InitInfo info;
    info.fp16_in_nvme_count = params.gpu_param_count_nvme;
    auto account = [&](const std::map<TensorId, Tier>& where) {
      for (const auto& [id, tier] : where) {
        const std::uint64_t sz = trace_.tensor(id).size_bytes;
        (tier == Tier::Gpu ? info.gpu_resident_bytes
                           : tier == Tier::Cpu ? info.cpu_resident_bytes : info.nvme_resident_bytes) += sz;
      }
    };
    account(params.location_of);
    account(opt.location_of);  // states are never GPU-placed

    state_ = make_scheduler_state(trace_, std::move(table), std::move(params), std::move(opt),
                                  BufferPool::build(Tier::Gpu, plan.gpu_counts),
                                  BufferPool::build(Tier::Cpu, plan.cpu_counts), BufferPool::build(Tier::Cpu, opt_slots));
    return info;
  }

  std::vector<Req> on_step_begin(const TraceStep& step) override { return on_step_start(state_, step); }

  std::vector<Req> on_step_end(const TraceStep& step) override {
    if (step.phase == Phase::OptimizerUpdate) {
      std::vector<Req> r = optimizer_on_update_end(state_, step.tensor_ids.front());
      if (sync_writeback_)
        for (Req& q : r)
          if (q.kind == Req::Kind::Evict && !q.instant) q.blocking = true;
      return r;
    }
    if (state_.halted) return {};
    return prefetch_tensor(state_, step.tensor_ids);
  }

  std::vector<Req> on_param_restore_point() override { return restore_final_locations(state_, RestoreScope::Parameters); }
  std::vector<Req> on_iteration_end() override { return restore_final_locations(state_, RestoreScope::OptimizerStates); }
  void reset_iteration() override { tencache::reset_iteration(state_); }
  const SchedulerState* scheduler_state() const override { return &state_; }
  std::optional<Tier> initial_tier(TensorId id) const override { return state_.final_loc(id); }

 private:
  // Every forward/backward step must be servable from the planned GPU slots.
  void check_steps_fit(const BufferPlan& plan) const {
    for (const TraceStep& s : trace_.steps) {
      if (s.phase == Phase::OptimizerUpdate) continue;
      std::map<std::uint64_t, std::uint64_t> need;
      for (TensorId id : s.tensor_ids) ++need[trace_.tensor(id).size_bytes];
      for (const auto& [size, n] : need) {
        auto it = plan.gpu_counts.find(size);
        if (it == plan.gpu_counts.end() || it->second < n)
          throw ConfigError("GPU capacity cannot hold step " + std::to_string(s.step_index) + ": needs " +
                            std::to_string(n) + " buffer(s) of " + std::to_string(size) + " bytes");
      }
    }
  }

  const ExecutionTrace& trace_;
  const MachineConfig& machine_;
  RunConfig cfg_;
  SchedulerState state_;
  bool sync_writeback_ = false;
};

// ------------------------------------------------------- ZeRO-Infinity-like
class ZeroInfinity final : public IPolicy {
 public:
  ZeroInfinity(const ExecutionTrace& t, const MachineConfig& m, const RunConfig& c) : trace_(t), machine_(m), cfg_(c) {}

  InitInfo init() override {
    st_ = make_zero_infinity_state(trace_, machine_, cfg_.zero_lookahead_k);
    InitInfo info;
    if (st_.fits_gpu) {
      for (const auto& t : trace_.tensors)
        if (t.kind == TensorKind::ParamFP16) info.gpu_resident_bytes += t.size_bytes;
    } else {
      for (const auto& [id, home] : st_.param_home) {
        const std::uint64_t sz = trace_.tensor(id).size_bytes;
        if (home == Tier::Cpu) info.cpu_resident_bytes += sz;
        if (home == Tier::Nvme) {
          info.nvme_resident_bytes += sz;
          ++info.fp16_in_nvme_count;
        }
      }
    }
    for (const auto& s : states_by_update_order(trace_)) info.nvme_resident_bytes += s.size_bytes;
    return info;
  }

  std::vector<Req> on_step_begin(const TraceStep& step) override {
    if (step.phase != Phase::OptimizerUpdate) return zero_infinity_step_begin(st_, step);
    Req r;  // synchronous swap-in of the state under update
    r.tensor_id = step.tensor_ids.front();
    r.src = Tier::Nvme;
    r.dst = Tier::Cpu;
    r.size_bytes = trace_.tensor(r.tensor_id).size_bytes;
    r.kind = Req::Kind::Prefetch;
    return {r};
  }

  std::vector<Req> on_step_end(const TraceStep& step) override {
    if (step.phase != Phase::OptimizerUpdate) return zero_infinity_step_end(st_, step);
    Req r;  // synchronous swap-out; the next update waits for it
    r.tensor_id = step.tensor_ids.front();
    r.src = Tier::Cpu;
    r.dst = Tier::Nvme;
    r.size_bytes = trace_.tensor(r.tensor_id).size_bytes;
    r.kind = Req::Kind::Evict;
    r.blocking = true;
    return {r};
  }

  std::vector<Req> on_param_restore_point() override { return {}; }
  std::vector<Req> on_iteration_end() override { return {}; }
  void reset_iteration() override { st_ = make_zero_infinity_state(trace_, machine_, cfg_.zero_lookahead_k); }
  std::optional<Tier> initial_tier(TensorId id) const override {
    if (trace_.tensor(id).kind == TensorKind::OptStateFP32) return Tier::Nvme;  // states all in NVMe
    if (st_.fits_gpu) return Tier::Gpu;
    return st_.param_home.at(id);
  }

 private:
  const ExecutionTrace& trace_;
  const MachineConfig& machine_;
  RunConfig cfg_;
  ZeroInfinityState st_;
};

// ------------------------------------------------------------------- L2L
class LayerToLayer final : public IPolicy {
 public:
  explicit LayerToLayer(const ExecutionTrace& t) : trace_(t) {}
  InitInfo init() override {
    st_ = make_l2l_state(trace_);
    InitInfo info;
    for (const auto& t : trace_.tensors) info.cpu_resident_bytes += t.size_bytes;
    return info;
  }
  std::vector<Req> on_step_begin(const TraceStep& s) override { return l2l_step_begin(st_, s); }
  std::vector<Req> on_step_end(const TraceStep& s) override { return l2l_step_end(st_, s); }
  std::vector<Req> on_param_restore_point() override { return {}; }
  std::vector<Req> on_iteration_end() override { return {}; }
  void reset_iteration() override { st_ = make_l2l_state(trace_); }
  std::optional<Tier> initial_tier(TensorId) const override { return Tier::Cpu; }

 private:
  const ExecutionTrace& trace_;
  L2LState st_;
};

// ------------------------------------------------------------- NoOffload
class NoOffload final : public IPolicy {
 public:
  NoOffload(const ExecutionTrace& t, const MachineConfig& m) : trace_(t), machine_(m) {}
  InitInfo init() override {
    InitInfo info;
    info.gpu_resident_bytes = no_offload_check(trace_, machine_);
    return info;
  }
  std::vector<Req> on_step_begin(const TraceStep&) override { return {}; }
  std::vector<Req> on_step_end(const TraceStep&) override { return {}; }
  std::vector<Req> on_param_restore_point() override { return {}; }
  std::vector<Req> on_iteration_end() override { return {}; }
  void reset_iteration() override {}
  std::optional<Tier> initial_tier(TensorId) const override { return Tier::Gpu; }

 private:
  const ExecutionTrace& trace_;
  const MachineConfig& machine_;
};

}  // namespace

// --------------------------------------------------- baseline free functions
ZeroInfinityState make_zero_infinity_state(const ExecutionTrace& trace, const MachineConfig& machine, int lookahead_k) {
  ZeroInfinityState st;
  st.trace = &trace;
  st.lookahead_k = lookahead_k;
  index_param_steps(trace, st.param_step_order, st.param_step_pos);
  std::vector<const TensorDescriptor*> params;
  std::uint64_t bytes = 0;
  for (const auto& t : trace.tensors)
    if (t.kind == TensorKind::ParamFP16) {
      params.push_back(&t);
      bytes += t.size_bytes;
    }
  if (bytes <= machine.gpu_capacity_bytes) {  // degenerates to no offload
    st.fits_gpu = true;
    for (const auto* t : params) st.gpu_resident.insert(t->id);
    return st;
  }
  // Largest parameters claim host memory first; the overflow lives in NVMe.
  std::sort(params.begin(), params.end(), [](const TensorDescriptor* a, const TensorDescriptor* b) {
    return a->size_bytes != b->size_bytes ? a->size_bytes > b->size_bytes : a->id < b->id;
  });
  std::uint64_t used = 0;
  for (const auto* t : params) {
    const bool fits = used + t->size_bytes <= machine.cpu_capacity_bytes;
    if (fits) used += t->size_bytes;
    st.param_home[t->id] = fits ? Tier::Cpu : Tier::Nvme;
  }
  return st;
}

std::vector<TransferRequest> zero_infinity_step_begin(ZeroInfinityState& st, const TraceStep& step) {
  std::vector<Req> out;
  if (st.fits_gpu || step.phase == Phase::OptimizerUpdate) return out;
  auto fetch = [&](const TraceStep& s) {
    for (TensorId id : s.tensor_ids)
      if (st.gpu_resident.insert(id).second) out.push_back(home_fetch(*st.trace, id, st.param_home.at(id)));
  };
  fetch(step);
  const std::size_t pos = st.param_step_pos.at(step.step_index);
  for (int k = 1; k <= st.lookahead_k && pos + static_cast<std::size_t>(k) < st.param_step_order.size(); ++k)
    fetch(st.trace->steps[st.param_step_order[pos + static_cast<std::size_t>(k)]]);
  return out;
}

std::vector<TransferRequest> zero_infinity_step_end(ZeroInfinityState& st, const TraceStep& step) {
  std::vector<Req> out;
  if (st.fits_gpu || step.phase == Phase::OptimizerUpdate) return out;
  for (TensorId id : step.tensor_ids)
    if (st.gpu_resident.erase(id)) out.push_back(home_drop(*st.trace, id, st.param_home.at(id)));
  return out;
}

L2LState make_l2l_state(const ExecutionTrace& trace) {
  L2LState st;
  st.trace = &trace;
  index_param_steps(trace, st.param_step_order, st.param_step_pos);
  for (const auto& t : trace.tensors)
    if (t.kind == TensorKind::ParamFP16) st.layer_tensors[t.layer].push_back(t.id);
  return st;
}

std::vector<TransferRequest> l2l_step_begin(L2LState& st, const TraceStep& step) {
  std::vector<Req> out;
  if (step.phase == Phase::OptimizerUpdate) return out;
  const std::uint32_t layer = st.trace->tensor(step.tensor_ids.front()).layer;
  if (st.loaded_layer == static_cast<std::int64_t>(layer)) return out;
  for (TensorId id : st.gpu_resident) out.push_back(home_drop(*st.trace, id, Tier::Cpu));
  st.gpu_resident.clear();
  for (TensorId id : st.layer_tensors.at(layer)) {
    st.gpu_resident.insert(id);
    out.push_back(home_fetch(*st.trace, id, Tier::Cpu));
  }
  st.loaded_layer = layer;
  return out;
}

std::vector<TransferRequest> l2l_step_end(L2LState& st, const TraceStep& step) {
  std::vector<Req> out;
  if (step.phase == Phase::OptimizerUpdate) return out;
  const std::size_t pos = st.param_step_pos.at(step.step_index);
  const std::uint32_t layer = st.trace->tensor(step.tensor_ids.front()).layer;
  bool last = true;  // the layer's last consecutive parameter step
  if (pos + 1 < st.param_step_order.size())
    last = st.trace->tensor(st.trace->steps[st.param_step_order[pos + 1]].tensor_ids.front()).layer != layer;
  if (last) {
    for (TensorId id : st.gpu_resident) out.push_back(home_drop(*st.trace, id, Tier::Cpu));
    st.gpu_resident.clear();
    st.loaded_layer = -1;
  }
  return out;
}

std::uint64_t no_offload_check(const ExecutionTrace& trace, const MachineConfig& machine) {
  std::uint64_t bytes = 0;
  for (const auto& t : trace.tensors) bytes += t.size_bytes;
  if (bytes > machine.gpu_capacity_bytes)
    throw OomError("model requires " + std::to_string(bytes) + " bytes but GPU capacity is " +
                   std::to_string(machine.gpu_capacity_bytes));
  return bytes;
}

std::unique_ptr<IPolicy> make_policy(const ExecutionTrace& trace, const MachineConfig& machine, const RunConfig& config) {
  switch (config.policy) {
    case PolicyKind::TenCache:
    case PolicyKind::TenCachePlusOpt: return std::make_unique<TenCache>(trace, machine, config);
    case PolicyKind::ZeroInfinityLike: return std::make_unique<ZeroInfinity>(trace, machine, config);
    case PolicyKind::L2LLike: return std::make_unique<LayerToLayer>(trace);
    case PolicyKind::NoOffload: return std::make_unique<NoOffload>(trace, machine);
  }
  throw ConfigError("unknown policy");
}

}  // namespace tencache
