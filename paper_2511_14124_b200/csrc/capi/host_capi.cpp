// extern "C" surface of the host decision engine (include/tencache_c.h,
// "decision engine" block). Exceptions are mapped to status codes here and
// never cross the boundary.
#include <chrono>
#include <cstdio>
#include <cstring>
#include <fstream>

#include <json.hpp>

#include "capi_common.hpp"
#include "tencache/tencache.hpp"
#include "tencache_c.h"

using namespace tencache;
using nlohmann::json;

namespace tcb {

thread_local std::string g_last_error;

int set_error(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

RunConfig parse_run_config(const char* cfg_json) {
  RunConfig c;
  if (cfg_json == nullptr || *cfg_json == 0) return c;
  const json j = json::parse(cfg_json);
  if (auto it = j.find("policy"); it != j.end()) c.policy = policy_from_string(it->get<std::string>());
  if (auto it = j.find("thresholds_us"); it != j.end()) c.thresholds_us = it->get<std::vector<double>>();
  if (auto it = j.find("restore_overlap"); it != j.end()) c.restore_overlap = it->get<bool>();
  if (auto it = j.find("batch_scale"); it != j.end()) c.batch_scale = it->get<double>();
  if (auto it = j.find("zero_lookahead_k"); it != j.end()) c.zero_lookahead_k = it->get<int>();
  if (auto it = j.find("seed"); it != j.end()) c.seed = it->get<std::uint64_t>();
  return c;
}

MachineConfig machine_from(const char* path) {
  return (path == nullptr || *path == 0) ? default_machine() : load_machine(path);
}

tc_request to_c(const TransferRequest& r) {
  tc_request c{};
  c.tensor_id = r.tensor_id;
  c.src = static_cast<std::uint8_t>(r.src);
  c.dst = static_cast<std::uint8_t>(r.dst);
  c.kind = static_cast<std::uint8_t>(r.kind);
  c.flags = static_cast<std::uint8_t>((r.via_cpu_staging ? 1 : 0) | (r.instant ? 2 : 0) | (r.src_retains ? 4 : 0) |
                                      (r.dst_has_copy ? 8 : 0) | (r.blocking ? 16 : 0));
  c.size_bytes = r.size_bytes;
  return c;
}

std::size_t first_optimizer_step(const ExecutionTrace& t) {
  for (std::size_t i = 0; i < t.steps.size(); ++i)
    if (t.steps[i].phase == Phase::OptimizerUpdate) return i;
  return t.steps.size();
}

}  // namespace tcb

using namespace tcb;

struct tc_policy {
  ExecutionTrace trace;
  MachineConfig machine;
  RunConfig cfg;
  std::unique_ptr<IPolicy> policy;
  std::vector<TransferRequest> overflow;  // requests of the last call that did not fit the caller's buffer
};

namespace {

const BufferPool* pool_of(const tc_policy* p, int which) {
  const SchedulerState* st = p->policy->scheduler_state();
  if (st == nullptr) return nullptr;
  switch (which) {
    case 0: return &st->gpu_pool;
    case 1: return &st->cpu_pool;
    case 2: return &st->cpu_opt_pool;
    default: return nullptr;
  }
}

json occupants_json(const BufferPool& pool) {
  json a = json::array();
  for (const Chunk& c : pool.chunks()) {
    std::int64_t v = c.occupant ? static_cast<std::int64_t>(*c.occupant) : 0;
    a.push_back(c.gpu_designated ? -v : v);
  }
  return a;
}

json layout_json(const BufferPool& pool) {
  json a = json::array();
  for (const Chunk& c : pool.chunks()) a.push_back(json::array({c.offset, c.size}));
  return a;
}

json request_json(const TransferRequest& r) {
  const tc_request c = to_c(r);
  return json::array({c.tensor_id, c.src, c.dst, c.size_bytes, c.kind, c.flags});
}

json report_json(const SimReport& r) {
  auto S = [](const Rat& x) { return rat_to_string(x); };
  json j;
  j["total_time_us"] = S(r.total_time_us);
  j["total_time_us_f"] = to_double(r.total_time_us);
  json per = json::array();
  for (const Rat& x : r.per_iteration_us) per.push_back(S(x));
  j["per_iteration_us"] = per;
  j["hit_rate"] = S(r.hit_rate);
  j["param_accesses"] = r.param_accesses;
  j["param_hits"] = r.param_hits;
  json waits = json::array();
  for (const Rat& w : r.param_wait_us) waits.push_back(S(w));
  j["param_wait_us"] = waits;
  json pct = json::array();
  for (const auto& [thr, p] : r.pct_wait_below) pct.push_back(json::array({thr, S(p)}));
  j["pct_wait_below"] = pct;
  j["optimizer_miss_rate"] = S(r.optimizer_miss_rate);
  j["opt_accesses"] = r.opt_accesses;
  j["opt_misses"] = r.opt_misses;
  j["gpu_utilization_timeavg"] = S(r.gpu_utilization_timeavg);
  j["cpu_utilization_timeavg"] = S(r.cpu_utilization_timeavg);
  j["fp16_in_nvme_count"] = r.fp16_in_nvme_count;
  j["transfer_bytes"] = r.transfer_bytes;
  j["profile_overhead_us"] = S(r.profile_overhead_us);
  return j;
}

}  // namespace

std::string tcb::report_json_text(const SimReport& r) { return report_json(r).dump(); }

extern "C" {

const char* tc_last_error(void) { return g_last_error.c_str(); }
const char* tc_version(void) { return "b200-tencache 0.1 (sm_100a)"; }

int tc_policy_create(const char* trace_path, const char* machine_path, const char* cfg_json, tc_policy** out,
                     uint64_t info[4]) {
  TC_GUARD({
    if (out == nullptr) return set_error(TC_EARG, "tc_policy_create: null out");
    auto p = std::make_unique<tc_policy>();
    p->trace = load_trace(trace_path);
    p->machine = machine_from(machine_path);
    p->cfg = parse_run_config(cfg_json);
    p->policy = make_policy(p->trace, p->machine, p->cfg);
    const IPolicy::InitInfo ii = p->policy->init();
    if (info) {
      info[0] = ii.gpu_resident_bytes;
      info[1] = ii.cpu_resident_bytes;
      info[2] = ii.nvme_resident_bytes;
      info[3] = ii.fp16_in_nvme_count;
    }
    *out = p.release();
    return TC_OK;
  })
}

void tc_policy_destroy(tc_policy* p) { delete p; }

int tc_policy_call(tc_policy* p, int hook, uint32_t step, tc_request* out, size_t cap, size_t* n) {
  TC_GUARD({
    if (p == nullptr) return set_error(TC_EARG, "null policy");
    std::vector<TransferRequest> reqs;
    if (hook != 5 && !p->overflow.empty())
      return set_error(TC_ERANGE, "tc_policy_call: the previous call's requests were not drained (hook 5)");
    switch (hook) {
      case 0: reqs = p->policy->on_step_begin(p->trace.steps.at(step)); break;
      case 1: reqs = p->policy->on_step_end(p->trace.steps.at(step)); break;
      case 2: reqs = p->policy->on_param_restore_point(); break;
      case 3: reqs = p->policy->on_iteration_end(); break;
      case 4: p->policy->reset_iteration(); break;
      case 5: reqs = std::move(p->overflow); p->overflow.clear(); break;  // drain, no state change
      default: return set_error(TC_EARG, "unknown hook " + std::to_string(hook));
    }
    if (n) *n = reqs.size();
    if (reqs.size() > cap) {  // the policy state has advanced: keep the requests for a hook-5 drain
      p->overflow = std::move(reqs);
      return set_error(TC_ERANGE, "tc_policy_call: " + std::to_string(*n) + " requests, buffer holds " +
                                      std::to_string(cap) + "; drain them with hook 5");
    }
    for (std::size_t k = 0; k < reqs.size(); ++k) out[k] = to_c(reqs[k]);
    return TC_OK;
  })
}

int tc_policy_pool(const tc_policy* p, int which, int64_t* occupant, size_t cap, size_t* n) {
  TC_GUARD({
    const BufferPool* pool = p ? pool_of(p, which) : nullptr;
    if (pool == nullptr) return set_error(TC_EARG, "no such pool");
    const auto& ch = pool->chunks();
    for (std::size_t i = 0; i < ch.size() && i < cap; ++i) {
      std::int64_t v = ch[i].occupant ? static_cast<std::int64_t>(*ch[i].occupant) : 0;
      occupant[i] = ch[i].gpu_designated ? -v : v;
    }
    if (n) *n = ch.size();
    return TC_OK;
  })
}

int tc_policy_layout(const tc_policy* p, int which, uint64_t* offset_size, size_t cap, size_t* n) {
  TC_GUARD({
    const BufferPool* pool = p ? pool_of(p, which) : nullptr;
    if (pool == nullptr) return set_error(TC_EARG, "no such pool");
    const auto& ch = pool->chunks();
    for (std::size_t i = 0; i < ch.size() && i < cap; ++i) {
      offset_size[2 * i] = ch[i].offset;
      offset_size[2 * i + 1] = ch[i].size;
    }
    if (n) *n = ch.size();
    return TC_OK;
  })
}

int64_t tc_policy_buffer_of(const tc_policy* p, int which, uint32_t tensor) {
  const BufferPool* pool = p ? pool_of(p, which) : nullptr;
  if (pool == nullptr) return -1;
  auto b = pool->buffer_of(tensor);
  return b ? static_cast<int64_t>(*b) : -1;
}

int tc_policy_shape(const tc_policy* p, uint32_t* steps, uint32_t* iterations, uint32_t* first_opt_step) {
  if (p == nullptr) return set_error(TC_EARG, "null policy");
  if (steps) *steps = static_cast<uint32_t>(p->trace.steps.size());
  if (iterations) *iterations = p->trace.iterations;
  if (first_opt_step) *first_opt_step = static_cast<uint32_t>(first_optimizer_step(p->trace));
  return TC_OK;
}

int tc_run(const char* trace_path, const char* machine_path, const char* cfg_json, const char* report_path,
           const char* events_path, int reference_guard) {
  TC_GUARD({
    const ExecutionTrace trace = load_trace(trace_path);
    const MachineConfig m = machine_from(machine_path);
    RunConfig c = parse_run_config(cfg_json);
    std::ofstream ev;
    if (events_path && *events_path) {
      ev.open(events_path);
      c.event_log = &ev;
    }
    const SimReport r = reference_guard ? run_reference(trace, m, c) : run(trace, m, c);
    std::ofstream(report_path) << report_json(r).dump() << "\n";
    return TC_OK;
  })
}

int tc_decisions(const char* trace_path, const char* machine_path, const char* cfg_json, const char* out_path,
                 int with_pools) {
  TC_GUARD({
    const ExecutionTrace trace = load_trace(trace_path);
    const MachineConfig m = machine_from(machine_path);
    const RunConfig c = parse_run_config(cfg_json);
    std::unique_ptr<IPolicy> policy = make_policy(trace, m, c);
    const IPolicy::InitInfo ii = policy->init();
    const SchedulerState* st = policy->scheduler_state();
    json init;
    init["info"] = json::array({ii.gpu_resident_bytes, ii.cpu_resident_bytes, ii.nvme_resident_bytes,
                                ii.fp16_in_nvme_count});
    if (st) {
      // The Alg. 2 plan (policies.cpp:34-39), zero-count classes included.
      json g = json::object(), cc = json::object();
      const TensorCensus census = tensor_census(trace, TensorKind::ParamFP16);
      if (!census.empty()) {
        const BufferPlan plan =
            plan_buffers(census, size_distribution(census), m.gpu_capacity_bytes, m.cpu_capacity_bytes);
        for (const auto& [s, n] : plan.gpu_counts) g[std::to_string(s)] = n;
        for (const auto& [s, n] : plan.cpu_counts) cc[std::to_string(s)] = n;
      }
      init["plan"] = {{"gpu", g}, {"cpu", cc}};
      init["layout"] = {{"gpu", layout_json(st->gpu_pool)},
                        {"cpu", layout_json(st->cpu_pool)},
                        {"cpu_opt", layout_json(st->cpu_opt_pool)}};
      init["pools"] = {{"gpu", occupants_json(st->gpu_pool)},
                       {"cpu", occupants_json(st->cpu_pool)},
                       {"cpu_opt", occupants_json(st->cpu_opt_pool)}};
      json pl = json::object(), ol = json::object();
      for (const auto& [id, t] : st->placement.location_of) pl[std::to_string(id)] = static_cast<int>(t);
      for (const auto& [id, t] : st->opt_placement.location_of) ol[std::to_string(id)] = static_cast<int>(t);
      init["placement"] = {{"params", pl}, {"opt", ol}};
      json tab = json::array();
      for (const PrefetchRow& r : st->table.rows)
        tab.push_back(json::array({r.order, r.tensor_id, rat_to_string(r.activation_us),
                                   static_cast<int>(r.current_loc), static_cast<int>(r.final_loc)}));
      init["table"] = tab;
      init["mode"] = static_cast<int>(st->mode);
    }
    json calls = json::array();
    auto emit = [&](std::uint32_t it, long step, const char* hook, const std::vector<TransferRequest>& reqs) {
      json rq = json::array();
      for (const auto& r : reqs) rq.push_back(request_json(r));
      json call = json::array({it, step, hook, rq});
      if (st && with_pools) {
        call.push_back(occupants_json(st->gpu_pool));
        call.push_back(occupants_json(st->cpu_pool));
        call.push_back(occupants_json(st->cpu_opt_pool));
      }
      calls.push_back(std::move(call));
    };
    const std::size_t first_opt = first_optimizer_step(trace);
    if (!trace.steps.empty())
      for (std::uint32_t it = 0; it < trace.iterations; ++it) {
        bool restored = false;
        for (std::size_t i = 0; i < trace.steps.size(); ++i) {
          if (c.restore_overlap && i == first_opt && !restored) {
            restored = true;
            emit(it, static_cast<long>(i), "R", policy->on_param_restore_point());
          }
          emit(it, static_cast<long>(i), "B", policy->on_step_begin(trace.steps[i]));
          emit(it, static_cast<long>(i), "E", policy->on_step_end(trace.steps[i]));
        }
        if (!restored) emit(it, -1, "R", policy->on_param_restore_point());
        emit(it, -1, "I", policy->on_iteration_end());
        policy->reset_iteration();
        emit(it, -1, "Z", {});
      }
    json out;
    out["init"] = init;
    out["calls"] = calls;
    std::ofstream(out_path) << out.dump() << "\n";
    return TC_OK;
  })
}

int tc_sweep(const char* trace_path, const char* machine_path, const char* cfg_json, const char* axis,
             const double* values, uint32_t n, uint32_t threads, const char* out_path) {
  TC_GUARD({
    const ExecutionTrace trace = load_trace(trace_path);
    const MachineConfig m = machine_from(machine_path);
    const RunConfig c = parse_run_config(cfg_json);
    const std::vector<SimReport> reps =
        sweep(trace, m, c, sweep_axis_from_string(axis), std::vector<double>(values, values + n), threads);
    json arr = json::array();
    for (const SimReport& r : reps) arr.push_back(report_json(r));
    std::ofstream(out_path) << arr.dump() << "\n";
    return TC_OK;
  })
}

int tc_synthesize(uint32_t layers, uint32_t tensors_per_layer, const uint64_t* sizes, int nsizes,
                  double compute_us_per_byte, uint64_t seed, uint32_t iterations, double opt_us_per_byte,
                  int optimizer_steps, const char* out_path) {
  TC_GUARD({
    SizeProfile prof;
    prof.choices.assign(sizes, sizes + nsizes);
    save_trace(synthesize_transformer_trace(layers, tensors_per_layer, prof, compute_us_per_byte, seed, iterations,
                                            opt_us_per_byte, optimizer_steps != 0),
               out_path);
    return TC_OK;
  })
}

int tc_trace_roundtrip(const char* in_path, const char* out_path) {
  TC_GUARD({
    save_trace(load_trace(in_path), out_path);
    return TC_OK;
  })
}

int tc_transfer_time(const char* machine_path, int src, int dst, uint64_t bytes, char* out, size_t out_len) {
  TC_GUARD({
    if (src < 0 || src > 2 || dst < 0 || dst > 2) return set_error(TC_EARG, "bad tier");
    const std::string s =
        rat_to_string(transfer_time_us(machine_from(machine_path), static_cast<Tier>(src), static_cast<Tier>(dst), bytes));
    std::snprintf(out, out_len, "%s", s.c_str());
    return TC_OK;
  })
}

int tc_time_decisions(const char* trace_path, const char* machine_path, const char* cfg_json, int iterations,
                      double* ns_per_iteration, double* init_ns) {
  TC_GUARD({
    const ExecutionTrace trace = load_trace(trace_path);
    const MachineConfig m = machine_from(machine_path);
    const RunConfig c = parse_run_config(cfg_json);
    using clk = std::chrono::steady_clock;
    const auto t0 = clk::now();
    std::unique_ptr<IPolicy> policy = make_policy(trace, m, c);
    policy->init();
    const auto t1 = clk::now();
    const std::size_t first_opt = first_optimizer_step(trace);
    std::size_t sink = 0;
    for (int it = 0; it < iterations; ++it) {
      bool restored = false;
      for (std::size_t i = 0; i < trace.steps.size(); ++i) {
        if (c.restore_overlap && i == first_opt && !restored) {
          restored = true;
          sink += policy->on_param_restore_point().size();
        }
        sink += policy->on_step_begin(trace.steps[i]).size();
        sink += policy->on_step_end(trace.steps[i]).size();
      }
      if (!restored) sink += policy->on_param_restore_point().size();
      sink += policy->on_iteration_end().size();
      policy->reset_iteration();
    }
    const auto t2 = clk::now();
    if (init_ns) *init_ns = std::chrono::duration<double, std::nano>(t1 - t0).count();
    if (ns_per_iteration)
      *ns_per_iteration = std::chrono::duration<double, std::nano>(t2 - t1).count() / std::max(iterations, 1) +
                          0.0 * static_cast<double>(sink);
    return TC_OK;
  })
}

int tc_time_run(const char* trace_path, const char* machine_path, const char* cfg_json, int repeats,
                double* ns_per_run) {
  TC_GUARD({
    const ExecutionTrace trace = load_trace(trace_path);
    const MachineConfig m = machine_from(machine_path);
    const RunConfig c = parse_run_config(cfg_json);
    const auto t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < repeats; ++i) (void)run(trace, m, c);
    const auto t1 = std::chrono::steady_clock::now();
    *ns_per_run = std::chrono::duration<double, std::nano>(t1 - t0).count() / std::max(repeats, 1);
    return TC_OK;
  })
}

}  // extern "C"
