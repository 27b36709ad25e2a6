// Written against the REFERENCE's C++ API only (proj/include/tencache/*.hpp).
// tests/test_cpp_dropin.py compiles it twice — against the reference headers +
// the compiled reference, and against our include/ + libtencache_b200.so —
// and requires byte-identical output: the drop-in claim at source level.
#include <iostream>
#include <sstream>

#include "tencache/analyzer.hpp"
#include "tencache/baselines.hpp"
#include "tencache/bufpool.hpp"
#include "tencache/engine.hpp"
#include "tencache/machine.hpp"
#include "tencache/placement.hpp"
#include "tencache/rational.hpp"
#include "tencache/scheduler.hpp"
#include "tencache/trace.hpp"
#include "tencache/types.hpp"

using namespace tencache;

static void report(const char* tag, const SimReport& r) {
  std::cout << tag << " total=" << rat_to_string(r.total_time_us) << " hit=" << rat_to_string(r.hit_rate)
            << " acc=" << r.param_accesses << " hits=" << r.param_hits
            << " optmiss=" << rat_to_string(r.optimizer_miss_rate) << " gpu_util=" << rat_to_string(r.gpu_utilization_timeavg)
            << " cpu_util=" << rat_to_string(r.cpu_utilization_timeavg) << " nvme16=" << r.fp16_in_nvme_count
            << " prof=" << rat_to_string(r.profile_overhead_us);
  for (const auto& [k, v] : r.transfer_bytes) std::cout << " " << k << "=" << v;
  for (const auto& [t, p] : r.pct_wait_below) std::cout << " <" << t << ":" << rat_to_string(p);
  std::cout << "\n";
}

static void reqs(const std::vector<TransferRequest>& v) {
  for (const auto& q : v)
    std::cout << " [" << q.tensor_id << " " << to_string(q.src) << "->" << to_string(q.dst) << " " << q.size_bytes
              << " k" << static_cast<int>(q.kind) << " " << q.via_cpu_staging << q.instant << q.src_retains
              << q.dst_has_copy << q.blocking << "]";
  std::cout << "\n";
}

int main(int argc, char** argv) {
  const std::string dir = argc > 1 ? argv[1] : ".";
  SizeProfile prof{{4096, 8192, 12288, 1000}};
  ExecutionTrace t = synthesize_transformer_trace(9, 2, prof, kDefaultComputeUsPerByte, 7, 3);
  save_trace(t, dir + "/t.jsonl");
  ExecutionTrace t2 = load_trace(dir + "/t.jsonl");
  std::cout << "roundtrip " << (t == t2) << " tensors=" << t.tensors.size() << " steps=" << t.steps.size() << "\n";

  // Rational surface
  Rat a = rat_from_double(0.1), b = rat_decimal(2474, -2);
  std::cout << "rat " << rat_to_string(a) << " " << rat_to_string(a * b + Rat(3)) << " " << to_double(a / b) << " "
            << (a < b) << " " << rat_to_string(rat_of(std::uint64_t(12)) - b) << "\n";
  BigInt big = BigInt(1) << 200;
  std::cout << "big " << big << " " << (big / BigInt(3)) << " " << (big % BigInt(1000007)) << "\n";

  // profiler / planner / pool / placement
  TensorCensus tc = tensor_census(t, TensorKind::ParamFP16);
  SizeDistribution sd = size_distribution(tc);
  for (const auto& [s, r] : sd.ratios) std::cout << "tsd " << s << " " << rat_to_string(r) << " " << sd.ratio_as_double(s) << "\n";
  BufferPlan plan = plan_buffers(tc, sd, 60000, 50000);
  std::cout << "plan gpu=" << plan.gpu_planned_bytes() << " cpu=" << plan.cpu_planned_bytes() << "\n";
  PrefetchTable table = build_prefetch_table(t);
  std::ostringstream csv;
  dump_prefetch_table_csv(table, csv);
  PlacementState ps = place_parameters(table, t, plan);
  dump_placement_csv(ps, t, csv);
  std::map<std::uint64_t, std::uint64_t> counts{{1000, 2}, {4096, 3}, {8192, 1}};
  BufferPool gp = BufferPool::build(Tier::Cpu, counts);
  auto b1 = gp.acquire(4096, 1);
  auto b2 = gp.acquire(4096, 2);
  auto b3 = gp.acquire(8192, 3);
  auto b4 = gp.acquire(8192, 4);
  std::cout << "acq " << (b1 ? *b1 : 99) << " " << (b2 ? *b2 : 99) << " " << (b3 ? *b3 : 99) << " "
            << (b4 ? *b4 : 99) << "\n";
  gp.set_designated(*b2, true);
  gp.release(*gp.buffer_of(1));
  gp.dump_csv(csv);
  auto v = gp.find_victim(4096, false);
  auto vd = gp.find_victim(4096, true);
  std::cout << "victim " << (v ? static_cast<long>(v->second) : -1L) << " " << (vd ? static_cast<long>(vd->second) : -1L)
            << " free=" << gp.free_count(4096) << " region=" << gp.region_bytes() << " occ=" << gp.occupied_bytes()
            << " has " << gp.has_class(4096) << gp.has_class(5) << "\n";
  for (auto [id, t] : gp.occupants(4096, false)) std::cout << "occ " << id << " " << t << "\n";
  try {
    gp.release(0);
  } catch (const PoolError& e) {
    std::cout << "PoolError " << e.what() << "\n";
  }
  try {
    gp.acquire(5, 9);
  } catch (const PoolError& e) {
    std::cout << "PoolError " << e.what() << "\n";
  }
  std::cout << csv.str();
  std::cout << "overhead " << rat_to_string(profile_overhead(t)) << "\n";

  // machine
  MachineConfig m = default_machine();
  m.gpu_capacity_bytes = 120000;
  m.cpu_capacity_bytes = 200000;
  for (auto [s, d] : {std::pair{Tier::Cpu, Tier::Gpu}, {Tier::Gpu, Tier::Cpu}, {Tier::Nvme, Tier::Gpu}, {Tier::Cpu, Tier::Nvme}})
    std::cout << "tt " << rat_to_string(transfer_time_us(m, s, d, 123456789)) << "\n";

  // policy plug-in through IPolicy, the engine's call order
  for (PolicyKind k : {PolicyKind::TenCache, PolicyKind::TenCachePlusOpt, PolicyKind::ZeroInfinityLike,
                       PolicyKind::L2LLike}) {
    RunConfig cfg;
    cfg.policy = k;
    std::ostringstream events;
    cfg.event_log = &events;
    try {
      auto pol = make_policy(t, m, cfg);
      auto info = pol->init();
      std::cout << to_string(k) << " init " << info.gpu_resident_bytes << " " << info.cpu_resident_bytes << " "
                << info.nvme_resident_bytes << " " << info.fp16_in_nvme_count << "\n";
      for (const auto& s : t.steps) {
        reqs(pol->on_step_begin(s));
        reqs(pol->on_step_end(s));
      }
      reqs(pol->on_param_restore_point());
      reqs(pol->on_iteration_end());
      pol->reset_iteration();
      report(to_string(k), run(t, m, cfg));
      std::cout << events.str().size() << " event bytes\n" << events.str().substr(0, 2000);
    } catch (const ConfigError& e) {
      std::cout << to_string(k) << " ConfigError " << e.what() << "\n";
    }
  }

  // free scheduler API: state built from the public pieces, halt check, optimizer schedule, restore
  for (std::uint64_t gcap : {std::uint64_t(60000), std::uint64_t(90000), std::uint64_t(150000)}) try {
    BufferPlan p2 = plan_buffers(tc, sd, gcap, 50000);
    PrefetchTable tb = build_prefetch_table(t);
    PlacementState params = place_parameters(tb, t, p2);
    std::vector<TensorDescriptor> states;
    for (const auto& [sid, pid] : t.optimizer_pairs()) states.push_back(t.tensor(sid));
    PlacementState opt = place_optimizer_states(states, 100000);
    std::map<std::uint64_t, std::uint64_t> oc;
    for (const auto& s : states)
      if (opt.location_of.at(s.id) == Tier::Cpu) ++oc[s.size_bytes];
    SchedulerState st = make_scheduler_state(t, tb, params, opt, BufferPool::build(Tier::Gpu, p2.gpu_counts),
                                             BufferPool::build(Tier::Cpu, p2.cpu_counts), BufferPool::build(Tier::Cpu, oc));
    std::cout << "mode " << static_cast<int>(st.mode) << " halt " << halt_check(st) << "\n";
    for (const auto& s : t.steps) {
      if (s.phase == Phase::OptimizerUpdate) break;
      reqs(on_step_start(st, s));
      if (!st.halted) reqs(prefetch_tensor(st, s.tensor_ids));
      std::cout << "halt " << halt_check(st) << " cursor " << st.table.cursor << "\n";
    }
    reqs(optimizer_step_schedule(st));
    reqs(restore_final_locations(st, RestoreScope::All));
    reset_iteration(st);
    std::cout << "after reset cursor " << st.table.cursor << " window " << st.active_window.size() << "\n";
  } catch (const std::logic_error& e) {
    std::cout << "logic_error " << e.what() << "\n";
  }

  // sweep (thread pool), deterministic order
  RunConfig cfg;
  cfg.policy = PolicyKind::TenCachePlusOpt;
  try {
    auto reps = sweep(t, m, cfg, SweepAxis::GpuCapacity, {90000, 120000, 200000, 400000}, 3);
    for (const auto& r : reps) report("sweep", r);
    auto reps2 = sweep(t, m, cfg, sweep_axis_from_string("batch_scale"), {0.5, 1.0, 2.0}, 1);
    for (const auto& r : reps2) report("sweep_bs", r);
    auto reps3 = sweep(t, m, cfg, SweepAxis::Pinned, {0, 1}, 2);
    for (const auto& r : reps3) report("sweep_pin", r);
  } catch (const ConfigError& e) {
    std::cout << "sweep ConfigError " << e.what() << "\n";
  }
  try {
    (void)no_offload_check(t, m);
  } catch (const OomError& e) {
    std::cout << "OomError " << e.what() << "\n";
  }
  try {
    (void)load_trace(dir + "/missing.jsonl");
  } catch (const TraceError& e) {
    std::cout << "TraceError " << e.what() << "\n";
  }
  std::cout << "policy names " << to_string(policy_from_string("l2l")) << " " << to_string(Tier::Nvme) << " "
            << to_string(Phase::Backward) << "\n";
  return 0;
}
