// ORACLE TEST INFRASTRUCTURE — not product code. Only tests/, smoke() and
// bench.py's cpu_baseline / --impl reference legs may load this library.
//
// A thin extern "C" driver over the UNMODIFIED reference simulator
// (/root/reference/proj/src/*.cpp, compiled by oracle/Makefile into
// oracle/_ref/libtencache_ref.so). It exposes:
//   * tcref_run            — reference run() / run_reference() → SimReport JSON
//                            (exact rationals as "num/den" strings) + event log
//   * tcref_decisions      — the policy call sequence of engine.cpp:363-431
//                            (begin/end per step, restore point, iteration end,
//                            reset) through the public IPolicy (engine.hpp:52-74),
//                            with the pool contents after every call
//   * tcref_synthesize     — synthesize_transformer_trace (trace.cpp:239-307)
//   * tcref_replay_*       — step-by-step IPolicy driving for the CPU baseline
// Pool snapshots need the SchedulerState, which TenCachePolicy keeps private
// (policies.cpp:121); this driver therefore rebuilds the same state from the
// reference's public free functions (the init sequence of policies.cpp:33-93)
// and asserts that its request stream equals the IPolicy stream call by call.
#include <chrono>
#include <cstring>
#include <fstream>
#include <memory>
#include <sstream>
#include <string>
#include <vector>

#include <json.hpp>

#include "tencache/analyzer.hpp"
#include "tencache/baselines.hpp"
#include "tencache/bufpool.hpp"
#include "tencache/engine.hpp"
#include "tencache/machine.hpp"
#include "tencache/placement.hpp"
#include "tencache/scheduler.hpp"
#include "tencache/trace.hpp"

using namespace tencache;
using nlohmann::json;

namespace {

thread_local std::string g_err;

int fail(const std::exception& e, const char* kind) {
  g_err = std::string(kind) + ": " + e.what();
  return -1;
}

#define GUARD(...)                                         \
  try {                                                    \
    __VA_ARGS__                                            \
  } catch (const ConfigError& e) {                         \
    g_err = std::string("ConfigError: ") + e.what();       \
    return 2;                                              \
  } catch (const OomError& e) {                            \
    g_err = std::string("OomError: ") + e.what();          \
    return 3;                                              \
  } catch (const TraceError& e) {                          \
    g_err = std::string("TraceError: ") + e.what();        \
    return 4;                                              \
  } catch (const PoolError& e) {                           \
    g_err = std::string("PoolError: ") + e.what();         \
    return 5;                                              \
  } catch (const std::exception& e) {                      \
    return fail(e, "Error");                               \
  }

RunConfig parse_cfg(const char* cfg_json) {
  RunConfig c;
  if (!cfg_json || !*cfg_json) return c;
  json j = json::parse(cfg_json);
  if (j.contains("policy")) c.policy = policy_from_string(j.at("policy").get<std::string>());
  if (j.contains("thresholds_us")) c.thresholds_us = j.at("thresholds_us").get<std::vector<double>>();
  if (j.contains("restore_overlap")) c.restore_overlap = j.at("restore_overlap").get<bool>();
  if (j.contains("batch_scale")) c.batch_scale = j.at("batch_scale").get<double>();
  if (j.contains("zero_lookahead_k")) c.zero_lookahead_k = j.at("zero_lookahead_k").get<int>();
  if (j.contains("seed")) c.seed = j.at("seed").get<std::uint64_t>();
  return c;
}

MachineConfig get_machine(const char* path) {
  if (!path || !*path) return default_machine();
  return load_machine(path);
}

std::string R(const Rat& r) { return rat_to_string(r); }

json report_json(const SimReport& r) {
  json j;
  j["total_time_us"] = R(r.total_time_us);
  j["total_time_us_f"] = to_double(r.total_time_us);
  json per = json::array();
  for (const auto& x : r.per_iteration_us) per.push_back(R(x));
  j["per_iteration_us"] = per;
  j["hit_rate"] = R(r.hit_rate);
  j["param_accesses"] = r.param_accesses;
  j["param_hits"] = r.param_hits;
  json waits = json::array();
  for (const auto& w : r.param_wait_us) waits.push_back(R(w));
  j["param_wait_us"] = waits;
  json pct = json::array();
  for (const auto& [thr, p] : r.pct_wait_below) pct.push_back(json::array({thr, R(p)}));
  j["pct_wait_below"] = pct;
  j["optimizer_miss_rate"] = R(r.optimizer_miss_rate);
  j["opt_accesses"] = r.opt_accesses;
  j["opt_misses"] = r.opt_misses;
  j["gpu_utilization_timeavg"] = R(r.gpu_utilization_timeavg);
  j["cpu_utilization_timeavg"] = R(r.cpu_utilization_timeavg);
  j["fp16_in_nvme_count"] = r.fp16_in_nvme_count;
  j["transfer_bytes"] = r.transfer_bytes;
  j["profile_overhead_us"] = R(r.profile_overhead_us);
  return j;
}

json req_json(const TransferRequest& q) {
  int flags = (q.via_cpu_staging ? 1 : 0) | (q.instant ? 2 : 0) | (q.src_retains ? 4 : 0) |
              (q.dst_has_copy ? 8 : 0) | (q.blocking ? 16 : 0);
  return json::array({q.tensor_id, static_cast<int>(q.src), static_cast<int>(q.dst), q.size_bytes,
                      static_cast<int>(q.kind), flags});
}

bool same_req(const TransferRequest& a, const TransferRequest& b) {
  return a.tensor_id == b.tensor_id && a.src == b.src && a.dst == b.dst &&
         a.size_bytes == b.size_bytes && a.kind == b.kind &&
         a.via_cpu_staging == b.via_cpu_staging && a.instant == b.instant &&
         a.src_retains == b.src_retains && a.dst_has_copy == b.dst_has_copy &&
         a.blocking == b.blocking;
}

// occupant per buffer id; 0 = free; negative = GPU-designated CPU chunk
json pool_occ(const BufferPool& p) {
  json a = json::array();
  for (const Chunk& c : p.chunks()) {
    std::int64_t v = c.occupant ? static_cast<std::int64_t>(*c.occupant) : 0;
    if (c.gpu_designated) v = -v;
    a.push_back(v);
  }
  return a;
}

json pool_layout(const BufferPool& p) {
  json a = json::array();
  for (const Chunk& c : p.chunks()) a.push_back(json::array({c.offset, c.size}));
  return a;
}

std::vector<TensorDescriptor> states_in_order(const ExecutionTrace& t) {
  std::vector<TensorDescriptor> s;
  for (const auto& [sid, pid] : t.optimizer_pairs()) s.push_back(t.tensor(sid));
  return s;
}

// Mirror of the TenCache init sequence (policies.cpp:33-93) over the
// reference's public functions, so pool contents can be observed.
struct Shadow {
  SchedulerState st;
  bool sync_posture = false;
  BufferPlan plan;
};

Shadow build_shadow(const ExecutionTrace& trace, const MachineConfig& m, const RunConfig& cfg) {
  Shadow sh;
  TensorCensus tc = tensor_census(trace, TensorKind::ParamFP16);
  if (!tc.empty()) sh.plan = plan_buffers(tc, size_distribution(tc), m.gpu_capacity_bytes, m.cpu_capacity_bytes);
  PrefetchTable table = build_prefetch_table(trace);
  PlacementState params = place_parameters(table, trace, sh.plan);
  auto states = states_in_order(trace);
  std::uint64_t rem = m.cpu_capacity_bytes - sh.plan.cpu_planned_bytes();
  std::uint64_t sb = 0;
  for (auto& s : states) sb += s.size_bytes;
  std::uint64_t budget = rem;
  if (cfg.policy == PolicyKind::TenCache && sb > rem) budget = 0;
  PlacementState opt = place_optimizer_states(states, budget);
  sh.sync_posture = budget == 0 && !states.empty();
  std::map<std::uint64_t, std::uint64_t> oc;
  for (auto& s : states)
    if (opt.location_of.at(s.id) == Tier::Cpu) ++oc[s.size_bytes];
  sh.st = make_scheduler_state(trace, std::move(table), std::move(params), std::move(opt),
                               BufferPool::build(Tier::Gpu, sh.plan.gpu_counts),
                               BufferPool::build(Tier::Cpu, sh.plan.cpu_counts),
                               BufferPool::build(Tier::Cpu, oc));
  return sh;
}

std::vector<TransferRequest> shadow_end(Shadow& sh, const TraceStep& step) {
  if (step.phase == Phase::OptimizerUpdate) {
    auto reqs = optimizer_on_update_end(sh.st, step.tensor_ids.front());
    if (sh.sync_posture)
      for (auto& r : reqs)
        if (r.kind == TransferRequest::Kind::Evict && !r.instant) r.blocking = true;
    return reqs;
  }
  if (sh.st.halted) return {};
  return prefetch_tensor(sh.st, step.tensor_ids);
}

}  // namespace

extern "C" {

const char* tcref_last_error() { return g_err.c_str(); }

int tcref_run(const char* trace_path, const char* machine_path, const char* cfg_json,
              const char* out_report, const char* out_events, int use_reference_engine) {
  GUARD({
    ExecutionTrace trace = load_trace(trace_path);
    MachineConfig m = get_machine(machine_path);
    RunConfig c = parse_cfg(cfg_json);
    std::ofstream ev;
    if (out_events && *out_events) {
      ev.open(out_events);
      c.event_log = &ev;
    }
    SimReport r = use_reference_engine ? run_reference(trace, m, c) : run(trace, m, c);
    std::ofstream(out_report) << report_json(r).dump() << "\n";
    return 0;
  })
}

// Wall-clock cost of the reference run() (model clock + decisions), ns.
int tcref_time_run(const char* trace_path, const char* machine_path, const char* cfg_json,
                   int repeats, double* out_ns_per_run) {
  GUARD({
    ExecutionTrace trace = load_trace(trace_path);
    MachineConfig m = get_machine(machine_path);
    RunConfig c = parse_cfg(cfg_json);
    auto t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < repeats; ++i) (void)run(trace, m, c);
    auto t1 = std::chrono::steady_clock::now();
    *out_ns_per_run = std::chrono::duration<double, std::nano>(t1 - t0).count() / repeats;
    return 0;
  })
}

// The reference's sweep() (engine.cpp:334-384) over one axis on `threads`
// threads: reports as a JSON array (same schema as tcref_run) and the
// wall-clock cost in ns.
int tcref_sweep(const char* trace_path, const char* machine_path, const char* cfg_json, const char* axis,
                const double* values, unsigned n, unsigned threads, const char* out_path, double* out_ns) {
  GUARD({
    ExecutionTrace trace = load_trace(trace_path);
    MachineConfig m = get_machine(machine_path);
    RunConfig c = parse_cfg(cfg_json);
    const std::vector<double> v(values, values + n);
    auto t0 = std::chrono::steady_clock::now();
    std::vector<SimReport> reps = sweep(trace, m, c, sweep_axis_from_string(axis), v, threads);
    auto t1 = std::chrono::steady_clock::now();
    if (out_ns) *out_ns = std::chrono::duration<double, std::nano>(t1 - t0).count();
    if (out_path && *out_path) {
      nlohmann::json arr = nlohmann::json::array();
      for (const SimReport& r : reps) arr.push_back(report_json(r));
      std::ofstream(out_path) << arr.dump() << "\n";
    }
    return 0;
  })
}

int tcref_decisions(const char* trace_path, const char* machine_path, const char* cfg_json,
                    const char* out_path, int with_pools) {
  GUARD({
    ExecutionTrace trace = load_trace(trace_path);
    MachineConfig m = get_machine(machine_path);
    RunConfig c = parse_cfg(cfg_json);
    auto policy = make_policy(trace, m, c);
    IPolicy::InitInfo info = policy->init();
    bool tencache = c.policy == PolicyKind::TenCache || c.policy == PolicyKind::TenCachePlusOpt;
    std::unique_ptr<Shadow> sh;
    if (tencache) sh = std::make_unique<Shadow>(build_shadow(trace, m, c));

    json out;
    json jinit;
    jinit["info"] = json::array({info.gpu_resident_bytes, info.cpu_resident_bytes,
                                 info.nvme_resident_bytes, info.fp16_in_nvme_count});
    if (sh) {
      json plan;
      json g = json::object(), cc = json::object();
      for (auto& [s, n] : sh->plan.gpu_counts) g[std::to_string(s)] = n;
      for (auto& [s, n] : sh->plan.cpu_counts) cc[std::to_string(s)] = n;
      plan["gpu"] = g;
      plan["cpu"] = cc;
      jinit["plan"] = plan;
      jinit["layout"] = {{"gpu", pool_layout(sh->st.gpu_pool)},
                         {"cpu", pool_layout(sh->st.cpu_pool)},
                         {"cpu_opt", pool_layout(sh->st.cpu_opt_pool)}};
      jinit["pools"] = {{"gpu", pool_occ(sh->st.gpu_pool)},
                        {"cpu", pool_occ(sh->st.cpu_pool)},
                        {"cpu_opt", pool_occ(sh->st.cpu_opt_pool)}};
      json pl = json::object(), ol = json::object();
      for (auto& [id, t] : sh->st.placement.location_of) pl[std::to_string(id)] = static_cast<int>(t);
      for (auto& [id, t] : sh->st.opt_placement.location_of) ol[std::to_string(id)] = static_cast<int>(t);
      jinit["placement"] = {{"params", pl}, {"opt", ol}};
      json tab = json::array();
      for (auto& r : sh->st.table.rows)
        tab.push_back(json::array({r.order, r.tensor_id, R(r.activation_us),
                                   static_cast<int>(r.current_loc), static_cast<int>(r.final_loc)}));
      jinit["table"] = tab;
      jinit["mode"] = static_cast<int>(sh->st.mode);
    }
    out["init"] = jinit;

    std::size_t first_opt = trace.steps.size();
    for (std::size_t i = 0; i < trace.steps.size(); ++i)
      if (trace.steps[i].phase == Phase::OptimizerUpdate) {
        first_opt = i;
        break;
      }

    json calls = json::array();
    auto emit = [&](std::uint32_t iter, long step, const char* hook,
                    const std::vector<TransferRequest>& reqs,
                    const std::vector<TransferRequest>* shadow) {
      if (shadow) {
        bool ok = shadow->size() == reqs.size();
        for (std::size_t k = 0; ok && k < reqs.size(); ++k) ok = same_req(reqs[k], (*shadow)[k]);
        if (!ok) throw std::logic_error("shadow scheduler diverged from IPolicy at hook " + std::string(hook));
      }
      json rq = json::array();
      for (auto& q : reqs) rq.push_back(req_json(q));
      json call = json::array({iter, step, hook, rq});
      if (sh && with_pools) {
        call.push_back(pool_occ(sh->st.gpu_pool));
        call.push_back(pool_occ(sh->st.cpu_pool));
        call.push_back(pool_occ(sh->st.cpu_opt_pool));
      }
      calls.push_back(call);
    };

    if (!trace.steps.empty()) {
      for (std::uint32_t it = 0; it < trace.iterations; ++it) {
        bool restored = false;
        for (std::size_t i = 0; i < trace.steps.size(); ++i) {
          const TraceStep& s = trace.steps[i];
          if (c.restore_overlap && i == first_opt && !restored) {
            restored = true;
            auto r = policy->on_param_restore_point();
            std::vector<TransferRequest> s2;
            if (sh) s2 = restore_final_locations(sh->st, RestoreScope::Parameters);
            emit(it, static_cast<long>(i), "R", r, sh ? &s2 : nullptr);
          }
          auto b = policy->on_step_begin(s);
          std::vector<TransferRequest> b2;
          if (sh) b2 = on_step_start(sh->st, s);
          emit(it, static_cast<long>(i), "B", b, sh ? &b2 : nullptr);
          auto e = policy->on_step_end(s);
          std::vector<TransferRequest> e2;
          if (sh) e2 = shadow_end(*sh, s);
          emit(it, static_cast<long>(i), "E", e, sh ? &e2 : nullptr);
        }
        if (!restored) {
          auto r = policy->on_param_restore_point();
          std::vector<TransferRequest> s2;
          if (sh) s2 = restore_final_locations(sh->st, RestoreScope::Parameters);
          emit(it, -1, "R", r, sh ? &s2 : nullptr);
        }
        auto ie = policy->on_iteration_end();
        std::vector<TransferRequest> ie2;
        if (sh) ie2 = restore_final_locations(sh->st, RestoreScope::OptimizerStates);
        emit(it, -1, "I", ie, sh ? &ie2 : nullptr);
        policy->reset_iteration();
        if (sh) reset_iteration(sh->st);
        emit(it, -1, "Z", {}, nullptr);
      }
    }
    out["calls"] = calls;
    std::ofstream(out_path) << out.dump() << "\n";
    return 0;
  })
}

// Decisions-only cost of one iteration through IPolicy (no model clock), ns.
int tcref_time_decisions(const char* trace_path, const char* machine_path, const char* cfg_json,
                         int iterations, double* out_ns_per_iter, double* out_init_ns) {
  GUARD({
    ExecutionTrace trace = load_trace(trace_path);
    MachineConfig m = get_machine(machine_path);
    RunConfig c = parse_cfg(cfg_json);
    auto t0 = std::chrono::steady_clock::now();
    auto policy = make_policy(trace, m, c);
    policy->init();
    auto t1 = std::chrono::steady_clock::now();
    std::size_t first_opt = trace.steps.size();
    for (std::size_t i = 0; i < trace.steps.size(); ++i)
      if (trace.steps[i].phase == Phase::OptimizerUpdate) {
        first_opt = i;
        break;
      }
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
    auto t2 = std::chrono::steady_clock::now();
    *out_init_ns = std::chrono::duration<double, std::nano>(t1 - t0).count();
    *out_ns_per_iter = std::chrono::duration<double, std::nano>(t2 - t1).count() / iterations +
                       static_cast<double>(sink % 2) * 0.0;
    return 0;
  })
}

int tcref_synthesize(unsigned layers, unsigned tensors_per_layer, const unsigned long long* sizes,
                     int nsizes, double compute_us_per_byte, unsigned long long seed,
                     unsigned iterations, double opt_us_per_byte, int optimizer_steps,
                     const char* out_path) {
  GUARD({
    SizeProfile p;
    for (int i = 0; i < nsizes; ++i) p.choices.push_back(sizes[i]);
    ExecutionTrace t = synthesize_transformer_trace(layers, tensors_per_layer, p, compute_us_per_byte,
                                                    seed, iterations, opt_us_per_byte,
                                                    optimizer_steps != 0);
    save_trace(t, out_path);
    return 0;
  })
}

int tcref_roundtrip(const char* in_path, const char* out_path) {
  GUARD({
    save_trace(load_trace(in_path), out_path);
    return 0;
  })
}

int tcref_transfer_time(const char* machine_path, int src, int dst, unsigned long long bytes,
                        char* out, int out_len) {
  GUARD({
    MachineConfig m = get_machine(machine_path);
    std::string s = rat_to_string(transfer_time_us(m, static_cast<Tier>(src), static_cast<Tier>(dst), bytes));
    std::snprintf(out, static_cast<std::size_t>(out_len), "%s", s.c_str());
    return 0;
  })
}

// ---- step-by-step IPolicy replay (CPU reference arm of bench.py) -----------
struct tcref_replay {
  ExecutionTrace trace;
  MachineConfig machine;
  RunConfig cfg;
  std::unique_ptr<IPolicy> policy;
  std::vector<TransferRequest> last;
};

void* tcref_replay_open(const char* trace_path, const char* machine_path, const char* cfg_json) {
  try {
    auto* r = new tcref_replay;
    r->trace = load_trace(trace_path);
    r->machine = get_machine(machine_path);
    r->cfg = parse_cfg(cfg_json);
    r->policy = make_policy(r->trace, r->machine, r->cfg);
    r->policy->init();
    return r;
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

void tcref_replay_close(void* h) { delete static_cast<tcref_replay*>(h); }

// hook: 0 begin, 1 end, 2 restore point, 3 iteration end, 4 reset.
// Writes up to cap requests as 6 u64 each (tensor, src, dst, size, kind, flags).
int tcref_replay_call(void* h, int hook, int step, unsigned long long* out, int cap) {
  auto* r = static_cast<tcref_replay*>(h);
  try {
    std::vector<TransferRequest> reqs;
    switch (hook) {
      case 0: reqs = r->policy->on_step_begin(r->trace.steps.at(step)); break;
      case 1: reqs = r->policy->on_step_end(r->trace.steps.at(step)); break;
      case 2: reqs = r->policy->on_param_restore_point(); break;
      case 3: reqs = r->policy->on_iteration_end(); break;
      case 4: r->policy->reset_iteration(); break;
      default: return -1;
    }
    int n = static_cast<int>(reqs.size());
    for (int k = 0; k < n && k < cap; ++k) {
      const auto& q = reqs[k];
      out[6 * k + 0] = q.tensor_id;
      out[6 * k + 1] = static_cast<unsigned long long>(q.src);
      out[6 * k + 2] = static_cast<unsigned long long>(q.dst);
      out[6 * k + 3] = q.size_bytes;
      out[6 * k + 4] = static_cast<unsigned long long>(q.kind);
      out[6 * k + 5] = (q.via_cpu_staging ? 1 : 0) | (q.instant ? 2 : 0) | (q.src_retains ? 4 : 0) |
                       (q.dst_has_copy ? 8 : 0) | (q.blocking ? 16 : 0);
    }
    return n;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

}  // extern "C"
