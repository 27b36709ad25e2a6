// Model-clock executor: a deterministic discrete-event replay of the policy's
// request stream over serialised links (reference counterpart: engine.cpp:17-384
// and engine_internal.hpp:35-142). The CUDA executor replaces this at run time;
// it is kept as the exact prediction the real run is reported beside, and the
// bit-exact parity target for waits, stalls and the optimizer miss rate.
//
// Semantics (all from the reference): one sequential step chain; a step whose
// tensors still have transfers in flight waits; its wait is measured from the
// step's FIRST attempt; nine directed link slots serve one transfer at a time
// in (arrival, seq) order; NVMe->GPU transfers are two legs through a
// per-size-class host staging slot; `blocking` transfers hold the next step;
// the iteration ends when every transfer has drained.
#include <array>
#include <atomic>
#include <queue>
#include <thread>

#include <json.hpp>

#include "tencache/tencache.hpp"

namespace tencache {

namespace {

std::string link_label(Tier s, Tier d) { return std::string(to_string(s)) + "->" + to_string(d); }

const char* request_tag(TransferRequest::Kind k) {
  switch (k) {
    case TransferRequest::Kind::Prefetch: return "prefetch";
    case TransferRequest::Kind::Evict: return "evict";
    case TransferRequest::Kind::Restore: return "restore";
  }
  return "?";
}

void check_config(const RunConfig& c) {
  if (c.batch_scale <= 0) throw ConfigError("batch_scale must be positive");
  if (c.zero_lookahead_k < 0) throw ConfigError("lookahead must be non-negative");
  double prev = 0;
  for (double t : c.thresholds_us) {
    if (t <= prev) throw ConfigError("thresholds must be positive and strictly increasing");
    prev = t;
  }
}

// Ids whose residency gates a step: all of a parameter step, the state(s) of
// an optimizer step.
std::vector<TensorId> gating_ids(const std::unordered_map<TensorId, TensorKind>& kind, const TraceStep& s) {
  if (s.phase != Phase::OptimizerUpdate) return s.tensor_ids;
  std::vector<TensorId> out;
  for (TensorId id : s.tensor_ids)
    if (kind.at(id) == TensorKind::OptStateFP32) out.push_back(id);
  return out;
}

// Time integral of bytes resident in one tier (piecewise constant).
struct Occupancy {
  std::int64_t bytes = 0;
  Rat area{0};
  Rat since{0};
  void add(std::int64_t delta, const Rat& now) {
    area += Rat(BigInt(bytes)) * (now - since);
    since = now;
    bytes += delta;
  }
  void set(std::int64_t v, const Rat& now) { add(v - bytes, now); }
};

struct Ledger {
  std::uint64_t param_accesses = 0, param_hits = 0, opt_accesses = 0, opt_misses = 0;
  std::vector<Rat> waits;
  std::map<std::string, std::uint64_t> bytes;
  std::array<Occupancy, 3> occ;

  Occupancy& tier(Tier t) { return occ[static_cast<std::size_t>(t)]; }

  void issued(const TransferRequest& r, const Rat& now) {
    if (!r.instant) {
      if (r.via_cpu_staging) {
        bytes[link_label(Tier::Nvme, Tier::Cpu)] += r.size_bytes;
        bytes[link_label(Tier::Cpu, Tier::Gpu)] += r.size_bytes;
      } else {
        bytes[link_label(r.src, r.dst)] += r.size_bytes;
      }
    }
    const auto sz = static_cast<std::int64_t>(r.size_bytes);
    if (!r.src_retains) tier(r.src).add(-sz, now);
    if (r.instant && !r.dst_has_copy) tier(r.dst).add(sz, now);
  }
  void completed(const TransferRequest& r, const Rat& now) {
    if (!r.dst_has_copy) tier(r.dst).add(static_cast<std::int64_t>(r.size_bytes), now);
  }

  SimReport report(const ExecutionTrace& trace, const MachineConfig& m, const RunConfig& cfg, const Rat& total,
                   std::vector<Rat> per_iter, std::uint64_t fp16_nvme) {
    SimReport r;
    r.total_time_us = total;
    r.per_iteration_us = std::move(per_iter);
    r.param_accesses = param_accesses;
    r.param_hits = param_hits;
    r.opt_accesses = opt_accesses;
    r.opt_misses = opt_misses;
    if (param_accesses) r.hit_rate = Rat(BigInt(param_hits), BigInt(param_accesses));
    if (opt_accesses) r.optimizer_miss_rate = Rat(BigInt(opt_misses), BigInt(opt_accesses));
    r.param_wait_us = std::move(waits);
    for (double thr : cfg.thresholds_us) {
      const Rat lim = rat_from_double(thr);
      std::uint64_t below = 0;
      for (const Rat& w : r.param_wait_us) below += w < lim ? 1 : 0;
      r.pct_wait_below.emplace_back(
          thr, param_accesses ? Rat(BigInt(below * 100), BigInt(param_accesses)) : Rat(0));
    }
    if (total > Rat(0)) {
      tier(Tier::Gpu).add(0, total);
      tier(Tier::Cpu).add(0, total);
      r.gpu_utilization_timeavg = tier(Tier::Gpu).area / (total * Rat(BigInt(m.gpu_capacity_bytes)));
      r.cpu_utilization_timeavg = tier(Tier::Cpu).area / (total * Rat(BigInt(m.cpu_capacity_bytes)));
    }
    r.fp16_in_nvme_count = fp16_nvme;
    r.transfer_bytes = std::move(bytes);
    r.profile_overhead_us = profile_overhead(trace);
    return r;
  }
};

class ModelClock {
 public:
  ModelClock(const ExecutionTrace& t, const MachineConfig& m, const RunConfig& c) : trace_(t), machine_(m), cfg_(c) {
    for (const auto& d : t.tensors) kind_[d.id] = d.kind;
  }

  SimReport execute() {
    check_config(cfg_);
    std::unique_ptr<IPolicy> policy = make_policy(trace_, machine_, cfg_);
    policy_ = policy.get();
    info_ = policy->init();
    ledger_.tier(Tier::Gpu).set(static_cast<std::int64_t>(info_.gpu_resident_bytes), Rat(0));
    ledger_.tier(Tier::Cpu).set(static_cast<std::int64_t>(info_.cpu_resident_bytes), Rat(0));
    ledger_.tier(Tier::Nvme).set(static_cast<std::int64_t>(info_.nvme_resident_bytes), Rat(0));
    first_opt_ = trace_.steps.size();
    for (std::size_t i = 0; i < trace_.steps.size(); ++i)
      if (trace_.steps[i].phase == Phase::OptimizerUpdate) {
        first_opt_ = i;
        break;
      }
    if (trace_.steps.empty())
      return ledger_.report(trace_, machine_, cfg_, Rat(0), std::vector<Rat>(trace_.iterations, Rat(0)),
                            info_.fp16_in_nvme_count);
    for (std::size_t i = 0; i < trace_.steps.size(); ++i) gates_.push_back(gating_ids(kind_, trace_.steps[i]));
    attempt_at_.assign(trace_.steps.size(), std::nullopt);
    post(Rat(0), Ev::StepStart, 0);
    while (!queue_.empty()) {
      Event e = queue_.top();
      queue_.pop();
      now_ = e.at;
      switch (e.kind) {
        case Ev::StepStart: try_start(e.arg); break;
        case Ev::StepEnd: end_step(e.arg); break;
        case Ev::LegDone: leg_done(e.arg); break;
        case Ev::IterEnd: end_iteration(); break;
      }
    }
    return ledger_.report(trace_, machine_, cfg_, total_, std::move(per_iter_), info_.fp16_in_nvme_count);
  }

 private:
  enum class Ev : std::uint8_t { StepStart, StepEnd, LegDone, IterEnd };
  struct Event {
    Rat at;
    std::uint64_t seq;
    Ev kind;
    std::size_t arg;
  };
  struct Later {
    bool operator()(const Event& a, const Event& b) const { return a.at != b.at ? a.at > b.at : a.seq > b.seq; }
  };
  struct Flight {
    TransferRequest req;
    std::uint64_t seq = 0;
    Rat arrived;
    bool second_leg = false;
  };
  struct LinkSlot {
    std::optional<std::size_t> busy;
    std::vector<std::size_t> queue;
  };
  struct Staging {
    bool busy = false;
    std::deque<std::size_t> queue;
  };
  struct TensorTrack {
    int in_flight = 0;
    int issued_since_access = 0;
    Rat ready{0};
  };

  static std::size_t link_of(Tier s, Tier d) { return static_cast<std::size_t>(s) * 3 + static_cast<std::size_t>(d); }
  std::size_t leg_link(const Flight& f) const {
    if (!f.req.via_cpu_staging) return link_of(f.req.src, f.req.dst);
    return f.second_leg ? link_of(Tier::Cpu, Tier::Gpu) : link_of(Tier::Nvme, Tier::Cpu);
  }
  Rat leg_time(const Flight& f) const {
    if (!f.req.via_cpu_staging) return transfer_time_us(machine_, f.req.src, f.req.dst, f.req.size_bytes);
    return f.second_leg ? transfer_time_us(machine_, Tier::Cpu, Tier::Gpu, f.req.size_bytes)
                        : transfer_time_us(machine_, Tier::Nvme, Tier::Cpu, f.req.size_bytes);
  }

  void post(const Rat& at, Ev k, std::size_t arg) { queue_.push(Event{at, seq_++, k, arg}); }

  void log(const char* kind, TensorId id, Tier s, Tier d) {
    if (!cfg_.event_log) return;
    nlohmann::json j = {{"us", to_double(now_)}, {"kind", kind}, {"tensor", id}, {"src", to_string(s)},
                        {"dst", to_string(d)}};
    *cfg_.event_log << j.dump() << "\n";
  }

  void try_start(std::size_t i) {
    if (barriers_ > 0) {
      parked_ = i;
      return;
    }
    if (!attempt_at_[i]) {
      attempt_at_[i] = now_;
      if (cfg_.restore_overlap && i == first_opt_ && !restored_) {
        restored_ = true;
        issue(policy_->on_param_restore_point());
      }
      issue(policy_->on_step_begin(trace_.steps[i]));
    }
    for (TensorId id : gates_[i])
      if (tracks_[id].in_flight > 0) {
        parked_ = i;
        return;
      }
    parked_.reset();
    const TraceStep& step = trace_.steps[i];
    const Rat& first = *attempt_at_[i];
    for (TensorId id : gates_[i]) {
      TensorTrack& tr = tracks_[id];
      const Rat wait = tr.ready > first ? tr.ready - first : Rat(0);
      if (step.phase == Phase::OptimizerUpdate) {
        ++ledger_.opt_accesses;
        if (wait > Rat(0)) ++ledger_.opt_misses;
      } else {
        ++ledger_.param_accesses;
        if (wait == Rat(0) && tr.issued_since_access == 0) ++ledger_.param_hits;
        ledger_.waits.push_back(wait);
      }
      tr.issued_since_access = 0;
      if (wait > Rat(0)) log("stall", id, Tier::Gpu, Tier::Gpu);
    }
    post(now_ + rat_from_double(step.compute_us) * rat_from_double(cfg_.batch_scale), Ev::StepEnd, i);
  }

  void end_step(std::size_t i) {
    issue(policy_->on_step_end(trace_.steps[i]));
    if (i + 1 < trace_.steps.size()) {
      post(now_, Ev::StepStart, i + 1);
      return;
    }
    if (!restored_) {
      restored_ = true;
      issue(policy_->on_param_restore_point());
    }
    issue(policy_->on_iteration_end());
    draining_ = true;
    maybe_drained();
  }

  void end_iteration() {
    draining_ = false;
    per_iter_.push_back(now_ - iter_start_);
    iter_start_ = now_;
    ledger_.tier(Tier::Nvme).set(static_cast<std::int64_t>(info_.nvme_resident_bytes), now_);
    policy_->reset_iteration();
    restored_ = false;
    if (++iter_ < trace_.iterations) {
      std::fill(attempt_at_.begin(), attempt_at_.end(), std::nullopt);
      post(now_, Ev::StepStart, 0);
    } else {
      total_ = now_;
    }
  }

  void maybe_drained() {
    if (draining_ && in_flight_ == 0) post(now_, Ev::IterEnd, 0);
  }

  void issue(const std::vector<TransferRequest>& reqs) {
    for (const TransferRequest& r : reqs) {
      log(request_tag(r.kind), r.tensor_id, r.src, r.dst);
      ledger_.issued(r, now_);
      if (r.instant) continue;
      const std::size_t idx = flights_.size();
      flights_.push_back(Flight{r, seq_++, now_, false});
      ++in_flight_;
      TensorTrack& tr = tracks_[r.tensor_id];
      ++tr.in_flight;
      ++tr.issued_since_access;
      if (r.blocking) ++barriers_;
      if (r.via_cpu_staging) {
        Staging& s = staging_[r.size_bytes];
        if (s.busy) {
          s.queue.push_back(idx);
          continue;
        }
        s.busy = true;
      }
      enqueue(idx);
    }
  }

  void enqueue(std::size_t idx) {
    flights_[idx].arrived = now_;
    LinkSlot& l = links_[leg_link(flights_[idx])];
    l.queue.push_back(idx);
    dispatch(l);
  }

  // Serve the earliest (arrival, seq) waiter when the link is idle.
  void dispatch(LinkSlot& l) {
    if (l.busy || l.queue.empty()) return;
    std::size_t pick = 0;
    for (std::size_t k = 1; k < l.queue.size(); ++k) {
      const Flight& a = flights_[l.queue[k]];
      const Flight& b = flights_[l.queue[pick]];
      if (a.arrived < b.arrived || (a.arrived == b.arrived && a.seq < b.seq)) pick = k;
    }
    const std::size_t idx = l.queue[pick];
    l.queue.erase(l.queue.begin() + static_cast<std::ptrdiff_t>(pick));
    l.busy = idx;
    post(now_ + leg_time(flights_[idx]), Ev::LegDone, idx);
  }

  void leg_done(std::size_t idx) {
    Flight& f = flights_[idx];
    LinkSlot& l = links_[leg_link(f)];
    l.busy.reset();
    dispatch(l);
    if (f.req.via_cpu_staging && !f.second_leg) {
      f.second_leg = true;
      enqueue(idx);
      return;
    }
    --in_flight_;
    ledger_.completed(f.req, now_);
    TensorTrack& tr = tracks_[f.req.tensor_id];
    --tr.in_flight;
    if (now_ > tr.ready) tr.ready = now_;
    if (f.req.blocking) --barriers_;
    if (f.req.via_cpu_staging) {
      Staging& s = staging_[f.req.size_bytes];
      s.busy = false;
      if (!s.queue.empty()) {
        const std::size_t nxt = s.queue.front();
        s.queue.pop_front();
        s.busy = true;
        enqueue(nxt);
      }
    }
    if (parked_) try_start(*parked_);
    maybe_drained();
  }

  const ExecutionTrace& trace_;
  const MachineConfig& machine_;
  RunConfig cfg_;
  std::unordered_map<TensorId, TensorKind> kind_;
  std::vector<std::vector<TensorId>> gates_;
  IPolicy* policy_ = nullptr;
  IPolicy::InitInfo info_;
  Ledger ledger_;

  std::priority_queue<Event, std::vector<Event>, Later> queue_;
  std::uint64_t seq_ = 0;
  Rat now_{0};
  std::vector<Flight> flights_;
  std::array<LinkSlot, 9> links_;
  std::map<std::uint64_t, Staging> staging_;
  std::unordered_map<TensorId, TensorTrack> tracks_;
  std::size_t in_flight_ = 0;
  int barriers_ = 0;
  std::optional<std::size_t> parked_;
  std::vector<std::optional<Rat>> attempt_at_;
  std::size_t first_opt_ = 0;
  bool restored_ = false;
  bool draining_ = false;
  std::uint32_t iter_ = 0;
  Rat iter_start_{0};
  std::vector<Rat> per_iter_;
  Rat total_{0};
};

}  // namespace

SimReport run(const ExecutionTrace& trace, const MachineConfig& machine, const RunConfig& config) {
  validate_trace(trace);
  return ModelClock(trace, machine, config).execute();
}

SimReport run_reference(const ExecutionTrace& trace, const MachineConfig& machine, const RunConfig& config) {
  if (trace.tensors.size() > kReferenceTensorGuard)
    throw ConfigError("run_reference: trace exceeds the " + std::to_string(kReferenceTensorGuard) + "-tensor guard");
  return run(trace, machine, config);
}

SweepAxis sweep_axis_from_string(const std::string& name) {
  for (SweepAxis a : {SweepAxis::BatchScale, SweepAxis::GpuCapacity, SweepAxis::CpuCapacity, SweepAxis::Pinned})
    if (name == to_string(a)) return a;
  throw ConfigError("unknown sweep axis: " + name);
}

const char* to_string(SweepAxis axis) {
  switch (axis) {
    case SweepAxis::BatchScale: return "batch_scale";
    case SweepAxis::GpuCapacity: return "gpu_capacity";
    case SweepAxis::CpuCapacity: return "cpu_capacity";
    case SweepAxis::Pinned: return "pinned";
  }
  return "?";
}

std::vector<SimReport> sweep(const ExecutionTrace& trace, const MachineConfig& machine, const RunConfig& config,
                             SweepAxis axis, const std::vector<double>& values, unsigned threads) {
  std::vector<SimReport> out(values.size());
  auto one = [&](std::size_t i) {
    MachineConfig m = machine;
    RunConfig c = config;
    c.event_log = nullptr;  // interleaved per-run logs would be meaningless
    const double v = values[i];
    switch (axis) {
      case SweepAxis::BatchScale: c.batch_scale = v; break;
      case SweepAxis::GpuCapacity: m.gpu_capacity_bytes = static_cast<std::uint64_t>(v); break;
      case SweepAxis::CpuCapacity: m.cpu_capacity_bytes = static_cast<std::uint64_t>(v); break;
      case SweepAxis::Pinned: m.cpu_memory_class = v != 0 ? CpuMemoryClass::Pinned : CpuMemoryClass::Pageable; break;
    }
    out[i] = run(trace, m, c);
  };
  if (threads <= 1) {
    for (std::size_t i = 0; i < values.size(); ++i) one(i);
    return out;
  }
  std::atomic<std::size_t> next{0};
  std::vector<std::thread> pool;
  for (unsigned t = 0; t < threads; ++t)
    pool.emplace_back([&] {
      for (std::size_t i = next++; i < values.size(); i = next++) one(i);
    });
  for (auto& th : pool) th.join();
  return out;
}

}  // namespace tencache
