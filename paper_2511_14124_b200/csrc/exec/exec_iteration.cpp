// Iteration pipeline of the per-GPU executor: the whole iteration's decisions
// made ahead, optimizer hoisting and pre-staging, the forward/backward
// stand-in, the fused AdamW data path, and the harvest of per-iteration
// timing records (executor.hpp has the physical layout).
#include "executor.hpp"

#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <thread>

namespace tcb {

using namespace tencache;

// A forward/backward step's tensors become readable on the compute stream:
// wait for their slots' writers (arrivals) and pending barriers, count hits
// (engine_internal.hpp:98-102), and run the access-side data work (ZeRO-3
// gather, or the checksum of the migrated bytes when compute_mode is 0).
void Executor::param_enter(const TraceStep& step, cudaStream_t cs, bool external) {
  cudaEvent_t reach = events_.get(true), go = events_.get(true);
  TCB_CK(cudaEventRecord(reach, cs));
  for (TensorId id : step.tensor_ids) {
    TensorRec& x = rec(id);
    if (x.tier != PTier::Gpu) throw DeviceError(TC_EINTERNAL, "step tensor " + std::to_string(id) + " not GPU-resident");
    wait_for_read(cs, slot_of(x).sync);
    // the caller writes this step's gradients: not before the previous
    // update that read them is done
    if (external && step.phase == Phase::Backward && x.grad_reader) TCB_CK(cudaStreamWaitEvent(cs, x.grad_reader, 0));
  }
  if (z3_ && external) {  // the caller reads the gathered layer (and, backward, writes its gradient view)
    const std::uint32_t layer = z3_->plans.at(index_of(step.tensor_ids.front())).layer;
    for (TensorId id : step.tensor_ids)
      if (z3_->plans.at(index_of(id)).layer != layer)
        throw DeviceError(TC_ECONFIG, "ZeRO-3 per-step execution needs every step to access one layer's chunks");
    z3_->open_layer = layer;
    if (step.phase == Phase::Backward) zero3_grad_fence(cs);
  }
  wait_barriers(cs);
  TCB_CK(cudaEventRecord(go, cs));
  stalls_.push_back(Stall{reach, go, step.tensor_ids.front()});
  for (TensorId id : step.tensor_ids) {
    TensorRec& x = rec(id);
    ++stats_.param_accesses;
    if (x.issued_since_access == 0)
      ++stats_.param_hits;
    else if (x.arrival)
      ontime_.emplace_back(reach, x.arrival);
    x.issued_since_access = 0;
    if (z3_ && external) {
      zero3_gather(x, cs);
    } else if (z3_) {
      zero3_access(x, step.phase == Phase::Backward, cs);
    } else if (access_cursor_ < n_accesses_) {
      if (so_.compute_mode == 0 || !external)
        TCB_CK(launch_checksum(where(x), x.bytes & ~3ull,
                               reinterpret_cast<unsigned long long*>(cks_base_ + access_cursor_), cs));
      ++stats_.kernel_launches;
      ++access_cursor_;
    }
  }
}

// The layer-compute stand-in of iteration(): a 1-CTA spin or bf16 GEMMs over
// the migrated chunk for the step's compute_us (trace.hpp:38).
void Executor::param_compute(const TraceStep& step, cudaStream_t cs) {
  const double us = step.compute_us * cfg_.batch_scale;
  if (so_.compute_mode == 1) {
    TCB_CK(launch_spin(static_cast<std::uint64_t>(us * 1000.0), so_.spin_ctas, cs));
    ++stats_.kernel_launches;
  } else if (so_.compute_mode == 2 && us > 0) {
    if (!standin_) {  // one weight shape for the trace: the smallest parameter chunk
      std::uint64_t smallest = ~0ull;
      for (const auto& r : recs_)
        if (!r.is_state) smallest = std::min(smallest, r.bytes);
      standin_ = std::make_unique<GemmStandin>(device_, smallest, us);
    }
    const double f0 = standin_->flops_issued();
    stats_.compute_gemms += static_cast<std::uint64_t>(standin_->run(cs, where(rec(step.tensor_ids.front())), us));
    stats_.compute_flops += standin_->flops_issued() - f0;
  }
}

// Everything the step computes is enqueued: its slots are read until here,
// and a caller-computed backward step's gradients are final here.
void Executor::param_exit(const TraceStep& step, cudaStream_t cs, bool external) {
  if (z3_ && external) {  // the caller's full-layer gradient is summed into this rank's chunks
    if (step.phase == Phase::Backward)
      for (TensorId id : step.tensor_ids) zero3_reduce(rec(id), cs, false);
    z3_->open_layer = -1;
  }
  cudaEvent_t done = events_.get(false);
  TCB_CK(cudaEventRecord(done, cs));
  for (TensorId id : step.tensor_ids) {
    TensorRec& x = rec(id);
    slot_of(x).sync.readers.push_back(done);
    if (external && step.phase == Phase::Backward) x.grad_ready = done;
  }
}

// One optimizer update, data side: state chunk H2D into an HBM stage, fused
// AdamW on the optimizer stream (bf16 result straight into the parameter's
// HBM slot when resident, else a scratch buffer), updated state D2H back to
// its pinned slot, and the parameter write-back when it lives off-GPU.
// Issue the H2D of a host-resident optimizer state into a free HBM stage.
std::size_t Executor::stage_state(TensorRec& s) {
  if (s.tier != PTier::HostOpt) throw DeviceError(TC_EINTERNAL, "optimizer state not in host memory when staged");
  if (stage_free_.empty()) throw DeviceError(TC_EINTERNAL, "no free optimizer stage");
  const std::size_t b = stage_free_.front();
  stage_free_.pop_front();
  Slot& h = slot_of(s);
  tag_ = CopyTag{"opt_load", s.id, 1, 0};
  wait_for_write(h2d_opt_, stage_sync_[b]);
  wait_for_read(h2d_opt_, h.sync);
  cudaEvent_t e1 = copy(h2d_opt_, stage_[b], h.ptr, state_xfer_bytes(s), true);
  h.sync.readers.push_back(e1);
  stage_sync_[b] = SlotSync{e1, {}};
  staged_[index_of(s.id)] = b;
  return b;
}

// Keep up to `want_staged` states staged ahead of their updates, in update order.
void Executor::refill_stages(std::size_t want_staged) {
  while (prestage_next_ < prestage_order_.size() && staged_.size() < want_staged && stage_free_.size() > 1) {
    TensorRec& s = recs_[static_cast<std::size_t>(prestage_order_[prestage_next_++])];
    if (!staged_.count(index_of(s.id)) && s.tier == PTier::HostOpt) stage_state(s);
  }
}

// One optimizer update, data side, in three parts so that consecutive
// hoisted updates share one fused AdamW launch: prepare (the state's HBM
// stage and the bf16 destination, every wait on the optimizer stream), one
// launch for the batch, then per update the state's write-back and the
// parameter's.
Executor::UpdateJob Executor::prepare_update(TensorRec& s, TensorRec& p) {
  cudaStream_t ost = adam_stream();
  UpdateJob j;
  j.s = &s;
  j.p = &p;
  j.state_on_gpu = s.tier == PTier::Gpu;  // no-offload posture: update in place in HBM
  if (!j.state_on_gpu && s.tier != PTier::HostOpt)
    throw DeviceError(TC_EINTERNAL, "optimizer state not in host memory at its update");
  j.n = p.bytes / 2;
  if (j.state_on_gpu) {
    Slot& gs = slot_of(s);
    j.stg = gs.ptr;
    wait_for_write(ost, gs.sync);
  } else {
    auto it = staged_.find(index_of(s.id));
    j.b = it != staged_.end() ? it->second : stage_state(s);
    staged_.erase(index_of(s.id));
    stats_.opt_h2d_bytes += state_xfer_bytes(s);  // counted at the update it feeds (staging may be a prologue)
    stats_.opt_logical_bytes += s.bytes;
    j.split = s.split;
    j.stg = stage_[j.b];
    // (null once a drain between the prologue's staging and this update completed it)
    if (stage_sync_[j.b].writer) TCB_CK(cudaStreamWaitEvent(ost, stage_sync_[j.b].writer, 0));
  }
  if (p.grad_ready) TCB_CK(cudaStreamWaitEvent(ost, p.grad_ready, 0));
  j.on_gpu = p.tier == PTier::Gpu;
  if (j.on_gpu) {
    Slot& g = slot_of(p);
    j.pout = g.ptr;
    j.psync = &g.sync;
  } else {  // a ring of at least the batch size: a batch never reuses a buffer
    std::size_t& k = pout_next_[p.bytes];
    j.pout = pout_scratch_[p.bytes][k];
    j.psync = &pout_sync_[p.bytes][k];
    k = (k + 1) % pout_scratch_[p.bytes].size();
  }
  if (j.state_on_gpu && s.split) throw DeviceError(TC_EINTERNAL, "split optimizer state moved into HBM");
  if (j.split) {  // the kernel reads and writes the overflow area in the state's pinned slot directly
    Slot& h = slot_of(s);
    j.ovf = h.dptr + packed_layout(j.n).ovf;
    wait_for_write(ost, h.sync);
  }
  if (j.split && !j.on_gpu) {  // the master's high half: the parameter's bytes from its host slot into the scratch
    if (p.tier != PTier::HostParam)
      throw DeviceError(TC_EINTERNAL, "split optimizer state " + std::to_string(s.id) + ": parameter in NVMe");
    Slot& ph = slot_of(p);
    wait_for_write(h2d_opt_, *j.psync);
    wait_for_read(h2d_opt_, ph.sync);
    tag_ = CopyTag{"param_hi", p.id, 1, 0};
    cudaEvent_t e = copy(h2d_opt_, j.pout, ph.ptr, p.bytes, true);
    ph.sync.readers.push_back(e);
    *j.psync = SlotSync{e, {}};
    stats_.opt_h2d_bytes += p.bytes;
  }
  wait_for_write(ost, *j.psync);
  return j;
}

void Executor::run_updates(std::vector<UpdateJob>& jobs) {
  if (jobs.empty()) return;
  cudaStream_t ost = adam_stream();
  cudaEvent_t a0 = events_.get(true), a1 = events_.get(true);
  TCB_CK(cudaEventRecord(a0, ost));
  const AdamScalars sc = adam_scalars(so_.lr, so_.beta1, so_.beta2, so_.eps, so_.weight_decay, adam_step_);
  unsigned long long *smin = nullptr, *smax = nullptr;
  const std::size_t cap = std::max<std::size_t>(recs_.size(), 1);
  if (span_cursor_ < cap) {  // in-kernel resident span of this launch
    smin = span_base_ + span_cursor_;
    smax = span_base_ + cap + span_cursor_;
    ++span_cursor_;
  }
  if (adam_stamps_ && smin) TCB_CK(launch_stamp(smin + 2 * cap, ost));
  std::vector<AdamChunk> chunks;
  for (const UpdateJob& j : jobs) {
    auto* st = reinterpret_cast<float*>(j.stg);
    const auto* g = reinterpret_cast<const std::uint16_t*>(j.p->grad);
    auto* pout = reinterpret_cast<std::uint16_t*>(j.pout);
    if (j.split) {
      chunks.push_back(AdamChunk{nullptr, nullptr, nullptr, g, pout, j.n, j.stg, j.ovf});
      ++stats_.split_updates;
      stats_.split_elems += j.n;
    } else {
      chunks.push_back(AdamChunk{st, st + j.n, st + 2 * j.n, g, pout, j.n});
    }
    stats_.adam_elems += j.n;
  }
  TCB_CK(launch_adamw_batch(chunks.data(), static_cast<int>(chunks.size()), sc, so_.grad_scale, ost, smin, smax));
  if (adam_stamps_ && smin) TCB_CK(launch_stamp(smin + 3 * cap, ost));
  TCB_CK(cudaEventRecord(a1, ost));
  adam_.emplace_back(a0, a1);
  ++stats_.kernel_launches;
  ++stats_.adam_launches;
  for (UpdateJob& j : jobs) finish_update(j, a1);
}

void Executor::finish_update(UpdateJob& j, cudaEvent_t a1) {
  TensorRec& s = *j.s;
  TensorRec& p = *j.p;
  *j.psync = SlotSync{a1, {}};
  p.grad_reader = a1;
  p.nvme_valid = false;  // any NVMe replica of the parameter is now stale
  if (p.has_home) p.home_valid = false;
  if (j.on_gpu) p.arrival = nullptr;

  if (j.state_on_gpu) {
    slot_of(s).sync = SlotSync{a1, {}};
  } else {
    Slot& h = slot_of(s);
    stage_sync_[j.b].readers.push_back(a1);
    wait_for_read(d2h_opt_, stage_sync_[j.b]);
    wait_for_write(d2h_opt_, h.sync);
    TCB_CK(cudaStreamWaitEvent(d2h_opt_, a1, 0));
    tag_ = CopyTag{"opt_store", s.id, 0, 1};
    cudaEvent_t e3 = copy(d2h_opt_, h.ptr, j.stg, state_xfer_bytes(s), false);
    h.sync = SlotSync{e3, {}};
    stage_sync_[j.b].readers.push_back(e3);
    stage_free_.push_back(j.b);
    stats_.opt_d2h_bytes += state_xfer_bytes(s);
    stats_.opt_logical_bytes += s.bytes;
  }

  if (!j.on_gpu) {  // updated-parameter write-back to its home tier (category iii)
    tag_ = CopyTag{"writeback", p.id, 0, static_cast<std::uint8_t>(p.tier == PTier::Nvme ? 2 : 1)};
    if (p.tier == PTier::Nvme) {
      std::uint8_t* bb = bounce_.at(p.bytes);
      SlotSync& bs = bounce_sync_[p.bytes];
      if (io_) {
        wait_for_write(d2h_opt_, bs);
        TCB_CK(cudaStreamWaitEvent(d2h_opt_, a1, 0));
        cudaEvent_t e4 = copy(d2h_opt_, bb, j.pout, p.bytes, false);
        j.psync->readers.push_back(e4);
        bs = SlotSync{e4, {}};
        nvme_write_async(p, bb, bs);
      } else {
        TCB_CK(cudaEventSynchronize(a1));
        host_wait_all(bs);
        TCB_CK(cudaMemcpy(bb, j.pout, p.bytes, cudaMemcpyDeviceToHost));
        bs = SlotSync{};
        nvme_write(p, bb);
      }
    } else {
      Slot& ph = slot_of(p);
      wait_for_write(d2h_opt_, ph.sync);
      TCB_CK(cudaStreamWaitEvent(d2h_opt_, a1, 0));
      cudaEvent_t e4 = copy(d2h_opt_, ph.ptr, j.pout, p.bytes, false);
      ph.sync = SlotSync{e4, {}};
      j.psync->readers.push_back(e4);
    }
    stats_.writeback_bytes += p.bytes;
  }
}

void Executor::optimizer_work(TensorRec& s, TensorRec& p) {
  std::vector<UpdateJob> one{prepare_update(s, p)};
  run_updates(one);
}

// A hoisted update waits in the batch until adam_batch() are ready or
// anything could observe its results (a decision moving its tensors, an
// in-place update, the end of the iteration): the data dependencies are all
// event-based, so deferring within those bounds changes no result.
void Executor::defer_update(TensorRec& s, TensorRec& p) {
  deferred_.emplace_back(index_of(s.id), index_of(p.id));
  if (deferred_.size() >= adam_batch()) flush_updates();
}

void Executor::flush_updates() {
  if (deferred_.empty()) return;
  std::vector<UpdateJob> jobs;
  for (const auto& [si, pi] : deferred_) {
    TensorRec& s = recs_[static_cast<std::size_t>(si)];
    const bool needs_stage = s.tier == PTier::HostOpt && !staged_.count(si);
    if (needs_stage && stage_free_.empty() && !jobs.empty()) {  // the batch so far frees its stages first
      run_updates(jobs);
      jobs.clear();
    }
    jobs.push_back(prepare_update(s, recs_[static_cast<std::size_t>(pi)]));
  }
  deferred_.clear();
  run_updates(jobs);
  if (so_.prestage) refill_stages(prestage_lookahead_ + adam_batch());
}

// Flush before `reqs` run if any of them moves a tensor of a deferred update.
void Executor::flush_if_touched(const std::vector<Req>& reqs) {
  if (deferred_.empty()) return;
  for (const Req& r : reqs)
    for (const auto& [si, pi] : deferred_)
      if (recs_[static_cast<std::size_t>(si)].id == r.tensor_id || recs_[static_cast<std::size_t>(pi)].id == r.tensor_id) {
        flush_updates();
        return;
      }
}

// The whole iteration's decisions, made up front in the reference's call
// order (engine.cpp:363-431). Legal because the request stream is a pure
// function of (trace, capacities, policy) and independent of timing
// (engine.hpp:49-51); it lets the executor see every future
// move when it schedules the data work.
std::vector<Executor::Hook> Executor::decide_iteration() {
  std::vector<Hook> hooks;
  std::size_t first_opt = trace_.steps.size();
  for (std::size_t i = 0; i < trace_.steps.size(); ++i)
    if (trace_.steps[i].phase == Phase::OptimizerUpdate) {
      first_opt = i;
      break;
    }
  bool restored = false;
  for (std::size_t i = 0; i < trace_.steps.size(); ++i) {
    if (cfg_.restore_overlap && i == first_opt && !restored) {
      restored = true;
      hooks.push_back({2, i, policy_->on_param_restore_point()});
    }
    hooks.push_back({0, i, policy_->on_step_begin(trace_.steps[i])});
    hooks.push_back({1, i, policy_->on_step_end(trace_.steps[i])});
  }
  if (!restored) hooks.push_back({2, trace_.steps.size(), policy_->on_param_restore_point()});
  hooks.push_back({3, trace_.steps.size(), policy_->on_iteration_end()});
  policy_->reset_iteration();
  return hooks;
}

// For each step, the optimizer steps whose data work runs right after that
// step's compute (before its end-hook moves): the parameter's last forward /
// backward access has happened, its gradient is final, and no decision
// touches the state until the update's own step. hoist_at[i] lists opt step
// indexes to run after step i; an opt step not listed runs in place.
std::vector<std::size_t> Executor::plan_hoisting(const std::vector<Hook>& hooks) {
  const std::size_t n = trace_.steps.size();
  std::vector<std::size_t> at(n, n);  // opt step -> host step (n = in place)
  if (!so_.hoist_optimizer) return at;
  std::unordered_map<TensorId, std::size_t> last_access;
  for (std::size_t i = 0; i < n; ++i)
    if (trace_.steps[i].phase != Phase::OptimizerUpdate)
      for (TensorId id : trace_.steps[i].tensor_ids) last_access[id] = i;
  // position of each begin hook, and the hooks touching each tensor
  std::vector<std::size_t> begin_pos(n, 0), end_pos(n, 0);
  std::unordered_map<TensorId, std::vector<std::size_t>> touched;
  for (std::size_t k = 0; k < hooks.size(); ++k) {
    if (hooks[k].kind == 0) begin_pos[hooks[k].step] = k;
    if (hooks[k].kind == 1) end_pos[hooks[k].step] = k;
    for (const Req& r : hooks[k].reqs) touched[r.tensor_id].push_back(k);
  }
  // the state's residency at iteration start = the policy's placement
  for (std::size_t j = 0; j < n; ++j) {
    const TraceStep& os = trace_.steps[j];
    if (os.phase != Phase::OptimizerUpdate) continue;
    const TensorId sid = os.tensor_ids.front();
    const TensorRec& s = rec(sid);
    if (!s.is_state || s.partner < 0) continue;
    const TensorId pid = recs_[static_cast<std::size_t>(s.partner)].id;
    auto la = last_access.find(pid);
    if (la == last_access.end()) continue;
    const std::size_t a = la->second;
    const Tier home = policy_->initial_tier(sid).value_or(Tier::Nvme);
    if (home != Tier::Cpu && home != Tier::Gpu) continue;
    // any decision moving the state before its update has run; its own end
    // hook's moves (the +Opt rotation evicts the updated state to NVMe there,
    // scheduler.cpp:338-370) come after the hoisted update anyway: requests
    // touching a deferred update's tensors flush it first (flush_if_touched)
    // and wait on its write-back through the slot's events
    bool moved = false;
    auto t = touched.find(sid);
    if (t != touched.end())
      for (std::size_t k : t->second) moved = moved || k < end_pos[j];
    if (moved) continue;
    at[j] = a;
  }
  return at;
}

// How many optimizer states fit through the H2D link during the forward
// pass on top of the forward's own parameter prefetches, by the machine's
// bandwidth model (machine.cpp:101-111) and the trace's compute time. With no
// forward prefetches to protect (every parameter resident: C3, C5's cached
// shard) the whole stage ring is filled: the loads only queue behind each
// other, and the forward under load runs longer than the model says (C3:
// ~360 vs 313 ms), so a model-sized budget left the link idle ~100 ms per
// step before the backward freed its first stage.
std::size_t Executor::forward_prestage_budget(const std::vector<Hook>& hooks) const {
  double fwd_us = 0, fwd_h2d = 0;
  for (const Hook& h : hooks) {
    if ((h.kind == 0 || h.kind == 1) && trace_.steps[h.step].phase == Phase::Forward) {
      if (h.kind == 0) fwd_us += trace_.steps[h.step].compute_us * cfg_.batch_scale;
      for (const Req& r : h.reqs)
        if (!r.instant && r.dst == Tier::Gpu) fwd_h2d += static_cast<double>(r.size_bytes);
    }
  }
  double bw;
  try {
    bw = to_double(machine_.effective_bandwidth(Tier::Cpu, Tier::Gpu)) * 1e3;  // bytes per us
  } catch (...) {
    return 0;
  }
  if (fwd_h2d == 0 && !prestage_order_.empty()) return stage_.size() > 2 ? stage_.size() - 2 : 1;
  const double spare = fwd_us * bw - fwd_h2d;
  if (spare <= 0 || prestage_order_.empty()) return std::min<std::size_t>(1, prestage_order_.size());
  const double sbytes =
      static_cast<double>(state_xfer_bytes(recs_[static_cast<std::size_t>(prestage_order_.front())]));
  return std::max<std::size_t>(1, static_cast<std::size_t>(spare / sbytes));
}

// An iteration is opened (decisions, hoisting plan, pre-staging), then driven
// step by step -- by iteration() itself, or by a training loop through
// tc_engine_step_begin / tc_engine_step_end, which run the same hooks at the
// reference's fixed call points (engine.cpp:119-131 begin, :157-168 end) --
// and closed (restore point, iteration end, harvest).
void Executor::iteration(const StepOptions& so, cudaStream_t compute) {
  iteration_begin(so, compute, false);
  for (std::size_t i = 0; i < trace_.steps.size(); ++i) {
    step_begin(i);
    step_end(i);
  }
  iteration_end();
}

void Executor::iteration_begin(const StepOptions& so, cudaStream_t compute, bool external) {
  TCB_CK(cudaSetDevice(device_));
  if (open_) throw DeviceError(TC_EARG, "iteration_begin: an iteration is already open");
  if (compute == nullptr) {
    if (!compute_owned_) TCB_CK(cudaStreamCreateWithFlags(&compute_owned_, cudaStreamNonBlocking));
    compute = compute_owned_;
  }
  compute_ = compute;
  if (io_) io_->check();  // a failed NVMe job of an earlier iteration fails the next call
  so_ = so;
  ++adam_step_;
  access_cursor_ = 0;
  if (!ahead_) events_.next_generation();  // else the prologue already opened this generation
  cks_base_ = d_checksums_ + (events_.generation() % 2) * std::max<std::size_t>(n_accesses_, 1);
  {  // per-launch AdamW spans: mins start at UINT64_MAX (0xff bytes), maxes at 0
    const std::size_t cap = std::max<std::size_t>(recs_.size(), 1);
    span_base_ = d_span_ + (events_.generation() % 2) * 4 * cap;  // [min | max | pre stamp | post stamp]
    span_cursor_ = 0;
    TCB_CK(launch_fill_u64(span_base_, ~0ull, cap, adam_stream()));  // same stream as the updates
    TCB_CK(launch_fill_u64(span_base_ + cap, 0ull, cap, adam_stream()));
  }
  TCB_CK(launch_fill_u64(reinterpret_cast<unsigned long long*>(cks_base_), 0ull, std::max<std::size_t>(n_accesses_, 1),
                         compute));
  OpenIter it;
  it.external = external;
  if (ahead_) {  // decided (and its first states staged) at the end of the previous iteration
    it.hooks = std::move(*ahead_);
    ahead_.reset();
  } else {
    nvtxRangePushA("tencache.decide");
    it.hooks = decide_iteration();
    nvtxRangePop();
    drop_staged();
  }
  it.hoist = plan_hoisting(it.hooks);
  const std::size_t n = trace_.steps.size();
  it.after.assign(n, {});
  for (std::size_t j = 0; j < n; ++j)
    if (it.hoist[j] < n) it.after[it.hoist[j]].push_back(j);
  // Hoisted updates in execution order; their states can be staged any time
  // (no decision touches them before their update, plan_hoisting). States
  // staged by the prologue are skipped by refill_stages.
  set_prestage_order(it.hooks, it.hoist);
  set_early_order(it.hooks);
  refill_early();
  // states the prologue staged come first in the order: continue after them
  while (prestage_next_ < prestage_order_.size() && staged_.count(prestage_order_[prestage_next_])) ++prestage_next_;
  if (so_.prestage) {
    refill_stages(prestage_fwd_override_ >= 0 ? static_cast<std::size_t>(prestage_fwd_override_)
                                              : forward_prestage_budget(it.hooks));
  }
  open_ = std::move(it);
  mark_phase();
}

void Executor::mark_phase() {
  cudaEvent_t e = events_.get(true);
  TCB_CK(cudaEventRecord(e, compute_));
  phase_marks_.push_back(e);
}

// Hooks up to and including step i's begin hook (a restore point placed
// before the first optimizer step runs here, engine.cpp:125-131), then the
// compute stream is ordered after the step's tensors' arrivals. Returns the
// device address of every tensor of a forward/backward step, in step order.
std::vector<void*> Executor::step_begin(std::size_t i) {
  if (!open_) throw DeviceError(TC_EARG, "step_begin: no open iteration (call iteration_begin)");
  OpenIter& it = *open_;
  if (it.in_step || i != it.next)
    throw DeviceError(TC_EARG, "step_begin(" + std::to_string(i) + "): steps run in trace order, begin then end; expected " +
                                   (it.in_step ? "step_end(" : "step_begin(") +
                                   std::to_string(it.in_step ? it.next - 1 : it.next) + ")");
  TCB_CK(cudaSetDevice(device_));
  while (it.hk < it.hooks.size() && it.hooks[it.hk].kind == 2) {
    flush_updates();  // the restore point moves tensors wholesale
    execute(it.hooks[it.hk++].reqs);
  }
  if (it.hk >= it.hooks.size() || it.hooks[it.hk].kind != 0 || it.hooks[it.hk].step != i)
    throw DeviceError(TC_EINTERNAL, "step_begin: hook sequence out of step");
  const TraceStep& step = trace_.steps[i];
  if (step.phase != it.prev) {
    mark_phase();
    it.prev = step.phase;
  }
  nvtxRangePushA(step.phase == Phase::Forward ? "tencache.fwd" : step.phase == Phase::Backward ? "tencache.bwd"
                                                                                               : "tencache.opt");
  if (step.phase == Phase::OptimizerUpdate) flush_updates();
  flush_if_touched(it.hooks[it.hk].reqs);
  execute(it.hooks[it.hk++].reqs);
  it.in_step = true;
  ++it.next;
  std::vector<void*> ptrs;
  if (step.phase != Phase::OptimizerUpdate) {
    param_enter(step, compute_, it.external);
    if (!it.external) param_compute(step, compute_);
    for (TensorId id : step.tensor_ids) ptrs.push_back(where(rec(id)));
  }
  return ptrs;
}

// The step's compute is enqueued (by the caller, on the compute stream): its
// tensors' slots are read until here, a backward step's gradients are final,
// the updates hoisted behind this step run, then the step's end hook.
void Executor::step_end(std::size_t i) {
  if (!open_ || !open_->in_step || open_->next != i + 1)
    throw DeviceError(TC_EARG, "step_end(" + std::to_string(i) + "): no such open step");
  OpenIter& it = *open_;
  TCB_CK(cudaSetDevice(device_));
  const TraceStep& step = trace_.steps[i];
  const std::size_t n = trace_.steps.size();
  if (step.phase == Phase::OptimizerUpdate) {
    if (it.hoist[i] == n) {  // in place: waits for the state's decisions
      TensorRec& s = rec(step.tensor_ids.front());
      if (s.partner < 0) throw DeviceError(TC_EINTERNAL, "optimizer step without a paired state");
      wait_barriers(adam_stream());
      optimizer_work(s, recs_[static_cast<std::size_t>(s.partner)]);
    }
  } else {
    param_exit(step, compute_, it.external);
    for (std::size_t j : it.after[i]) {
      TensorRec& s = rec(trace_.steps[j].tensor_ids.front());
      defer_update(s, recs_[static_cast<std::size_t>(s.partner)]);
    }
  }
  nvtxRangePop();
  if (it.hk >= it.hooks.size() || it.hooks[it.hk].kind != 1 || it.hooks[it.hk].step != i)
    throw DeviceError(TC_EINTERNAL, "step_end: hook sequence out of step");
  flush_if_touched(it.hooks[it.hk].reqs);
  execute(it.hooks[it.hk++].reqs);
  it.in_step = false;
}

void Executor::iteration_end() {
  if (!open_) throw DeviceError(TC_EARG, "iteration_end: no open iteration");
  if (open_->in_step || open_->next != trace_.steps.size())
    throw DeviceError(TC_EARG, "iteration_end: " + std::to_string(trace_.steps.size() - open_->next) +
                                   " step(s) not run" + (open_->in_step ? " (a step is still open)" : ""));
  TCB_CK(cudaSetDevice(device_));
  OpenIter& it = *open_;
  flush_updates();
  while (it.hk < it.hooks.size()) execute(it.hooks[it.hk++].reqs);  // restore point (if not yet), iteration end
  open_.reset();
  mark_phase();
  finish_iteration();
  if (lookahead_ && so_.prestage && so_.prologue) prologue_next();
}

// Abandon an open iteration (the caller's step failed): the remaining hooks
// still run so that tensors end at the policy's final placement and the
// next iteration's decisions hold; no further compute is ordered.
void Executor::iteration_abort() {
  if (!open_) return;
  if (open_->in_step) {
    nvtxRangePop();
    open_->in_step = false;
  }
  deferred_.clear();  // abandoned with the rest of the iteration's updates
  while (open_->hk < open_->hooks.size()) execute(open_->hooks[open_->hk++].reqs);
  open_.reset();
  mark_phase();
  finish_iteration();
}

// Hoisted updates of an iteration in execution order = the order their
// states are staged.
void Executor::set_prestage_order(const std::vector<Hook>& hooks, const std::vector<std::size_t>& hoist) {
  const std::size_t n = trace_.steps.size();
  std::vector<std::vector<std::size_t>> after(n);
  for (std::size_t j = 0; j < n; ++j)
    if (hoist[j] < n) after[hoist[j]].push_back(j);
  prestage_order_.clear();
  prestage_next_ = 0;
  for (std::size_t i = 0; i < n; ++i)
    for (std::size_t j : after[i]) prestage_order_.push_back(index_of(trace_.steps[j].tensor_ids.front()));
}

// Release stages holding pre-staged states (their bytes may be stale: the
// caller wrote or re-seeded tensors); the decisions made ahead stay valid.
void Executor::drop_staged() {
  for (auto& [idx, b] : staged_) stage_free_.push_back(b);
  staged_.clear();
  drop_early();
}

// The iteration's NVMe -> pinned state fetches, in decision order.
void Executor::set_early_order(const std::vector<Hook>& hooks) {
  drop_early();  // (empty here: every read-ahead of an iteration is bound by its own decision)
  if (nvme_ahead_ == 0 || !io_) return;
  for (const Hook& h : hooks)
    for (const Req& r : h.reqs)
      if (r.src == Tier::Nvme && r.dst == Tier::Cpu && !r.instant && rec(r.tensor_id).is_state)
        early_order_.push_back(index_of(r.tensor_id));
}

// Keep up to nvme_ahead_ of the upcoming fetches read into spare pinned
// slots. An entry whose state is not in the NVMe tier now (an earlier fetch
// of the same state in this iteration comes first) is left to its decision.
void Executor::refill_early() {
  while (early_.size() < nvme_ahead_ && early_next_ < early_order_.size()) {
    const std::int32_t xi = early_order_[early_next_];
    TensorRec& x = recs_[static_cast<std::size_t>(xi)];
    if (x.tier != PTier::Nvme || !x.nvme_valid || early_.count(xi)) {
      ++early_next_;
      continue;
    }
    if (!host_opt_.has_free(x.bytes)) return;  // every spare slot holds a read-ahead: wait for a bind
    ++early_next_;
    const std::uint32_t hs = take_slot(PTier::HostOpt, x.bytes, xi);
    Slot& h = host_opt_.cls(x.bytes).slots[hs];
    tag_ = CopyTag{"nvme_ahead", x.id, 2, 1};
    nvme_read_async(x, h.ptr, h.sync);
    early_[xi] = EarlyFetch{hs};
  }
}

// Give read-ahead slots back (their pending reads stay ordered before any
// later writer of the slot through its SlotSync).
void Executor::drop_early() {
  for (auto& [xi, ef] : early_) free_slot(PTier::HostOpt, recs_[static_cast<std::size_t>(xi)].bytes, ef.slot);
  early_.clear();
  early_order_.clear();
  early_next_ = 0;
}

// Prologue of iteration t+1, run at the end of iteration t's enqueue: its
// decisions are made now (the request stream is timing-independent,
// engine.hpp:49-51) and its first optimizer states are staged right behind
// t's last state loads, so the H2D link works through t's write-back tail
// whether or not the caller waits for t's result before calling iteration()
// again (tc_engine_step_result waits for t's compute stream).
void Executor::prologue_next() {
  events_.next_generation();
  nvtxRangePushA("tencache.decide");
  std::vector<Hook> hooks = decide_iteration();
  nvtxRangePop();
  set_prestage_order(hooks, plan_hoisting(hooks));
  refill_stages(prestage_fwd_override_ >= 0 ? static_cast<std::size_t>(prestage_fwd_override_)
                                            : forward_prestage_budget(hooks));
  ahead_ = std::move(hooks);
}

// The iteration is enqueued; nothing waits for it here. Its timing records
// and a fence per stream are parked; the previous iteration is harvested
// (fences awaited, timings summed, its events recycled) so that iteration
// t+1's forward pass overlaps iteration t's optimizer write-back tail.
void Executor::finish_iteration() {
  {  // the step's result (per-access checksums) to pinned host memory, on the
     // compute stream: step_result() waits for this, not for the optimizer tail
    const std::size_t k = static_cast<std::size_t>(events_.generation() % 2), na = std::max<std::size_t>(n_accesses_, 1);
    // a kernel storing into mapped pinned memory: a cudaMemcpyAsync here would
    // queue on the D2H copy engine behind the iteration's bulk state stores
    // and hold the next iteration's compute stream until they drain
    TCB_CK(launch_copy_u64(reinterpret_cast<unsigned long long*>(d_result_) + k * na,
                           reinterpret_cast<const unsigned long long*>(cks_base_), n_accesses_, compute_));
    TCB_CK(cudaEventRecord(result_ev_[k], compute_));
    result_gen_ = events_.generation();
    have_result_ = true;
  }
  {  // this iteration's AdamW spans/stamps to mapped host memory, behind its last update
    const std::size_t cap = std::max<std::size_t>(recs_.size(), 1);
    TCB_CK(launch_copy_u64(reinterpret_cast<unsigned long long*>(d_span_host_) + (events_.generation() % 2) * 4 * cap,
                           span_base_, 4 * cap, adam_stream()));
  }
  IterRecord rec;
  rec.gen = events_.generation();
  rec.copies = std::move(copies_);
  rec.stalls = std::move(stalls_);
  rec.ontime = std::move(ontime_);
  rec.adam = std::move(adam_);
  rec.marks = std::move(phase_marks_);
  for (cudaStream_t x : {h2d_, d2h_, opt_, h2d_opt_, d2h_opt_, compute_}) {
    cudaEvent_t e = events_.get(true);
    TCB_CK(cudaEventRecord(e, x));
    rec.fences.push_back(e);
  }
  rec.cks_buf = static_cast<std::size_t>(events_.generation() % 2);
  rec.io_seq = io_ ? io_->submitted() : 0;
  rec.spans = span_cursor_;
  copies_.clear();
  stalls_.clear();
  ontime_.clear();
  adam_.clear();
  phase_marks_.clear();
  if (!staged_.empty()) {  // defensive: a staged state whose update did not run
    for (auto& [idx, b] : staged_) stage_free_.push_back(b);
    staged_.clear();
  }
  pending_.push_back(std::move(rec));
  while (pending_.size() > 1) harvest_front();
}

void Executor::harvest_front() {
  IterRecord rec = std::move(pending_.front());
  pending_.pop_front();
  {  // fences, with a diagnostic if an iteration does not drain
    static const char* const kStreams[] = {"h2d", "d2h", "opt", "h2d_opt", "d2h_opt", "compute"};
    const auto t0 = std::chrono::steady_clock::now();
    for (bool reported = false;;) {
      bool all = true;
      std::string pending;
      for (std::size_t i = 0; i < rec.fences.size(); ++i) {
        const cudaError_t q = cudaEventQuery(rec.fences[i]);
        if (q == cudaErrorNotReady) {
          all = false;
          pending += std::string(" ") + (i < 6 ? kStreams[i] : "?");
        } else if (q != cudaSuccess) {
          TCB_CK(q);
        }
      }
      if (all) break;
      if (!reported && std::chrono::steady_clock::now() - t0 > std::chrono::seconds(30)) {
        reported = true;
        std::fprintf(stderr, "[executor] iteration %llu not drained after 30 s; streams pending:%s; %s\n",
                     static_cast<unsigned long long>(rec.gen), pending.c_str(),
                     io_ ? io_->describe().c_str() : "no nvme queue");
      }
      std::this_thread::sleep_for(std::chrono::microseconds(50));
    }
  }
  if (io_) io_->wait_upto(rec.io_seq);  // no queued job may still name an event we recycle
  float ms = 0;
  phase_ms_.clear();
  for (std::size_t i = 0; i + 1 < rec.marks.size(); ++i) {
    TCB_CK(cudaEventElapsedTime(&ms, rec.marks[i], rec.marks[i + 1]));
    phase_ms_.push_back(ms);
  }
  if (!rec.marks.empty()) {  // whole iteration: start mark -> last fence
    float end = 0;
    for (cudaEvent_t f : rec.fences) {
      TCB_CK(cudaEventElapsedTime(&ms, rec.marks.front(), f));
      end = std::max(end, ms);
    }
    phase_ms_.push_back(end);
  }
  for (const Copy& c : rec.copies) {
    TCB_CK(cudaEventElapsedTime(&ms, c.start, c.end));
    (c.h2d ? stats_.h2d_busy_ms : stats_.d2h_busy_ms) += ms;
  }
  for (const Stall& st : rec.stalls) {
    TCB_CK(cudaEventElapsedTime(&ms, st.reach, st.go));
    stats_.stall_ms += ms;
  }
  if (event_log_ && !rec.marks.empty()) {  // measured timeline in the reference's event-log schema
    static const char* const kTiers[] = {"gpu", "cpu", "nvme"};
    float t0 = 0, t1 = 0;
    for (std::size_t k = 0; k < rec.marks.size(); ++k) {  // phase boundaries of this iteration
      TCB_CK(cudaEventElapsedTime(&t0, rec.marks.front(), rec.marks[k]));
      *event_log_ << "{\"iter\":" << rec.gen << ",\"kind\":\"mark\",\"k\":" << k << ",\"us\":" << t0 * 1e3 << "}\n";
    }
    if (!pending_.empty() && !pending_.front().marks.empty()) {  // where the next iteration starts
      TCB_CK(cudaEventSynchronize(pending_.front().marks.front()));
      TCB_CK(cudaEventElapsedTime(&t0, rec.marks.front(), pending_.front().marks.front()));
      *event_log_ << "{\"iter\":" << rec.gen << ",\"kind\":\"next_iter\",\"us\":" << t0 * 1e3 << "}\n";
    }
    for (const Copy& c : rec.copies) {
      TCB_CK(cudaEventElapsedTime(&t0, rec.marks.front(), c.start));
      TCB_CK(cudaEventElapsedTime(&t1, rec.marks.front(), c.end));
      *event_log_ << "{\"bytes\":" << c.bytes << ",\"dst\":\"" << kTiers[c.tag.dst] << "\",\"end_us\":" << t1 * 1e3
                  << ",\"iter\":" << rec.gen << ",\"kind\":\"" << c.tag.kind << "\",\"src\":\"" << kTiers[c.tag.src]
                  << "\",\"tensor\":" << c.tag.tensor << ",\"us\":" << t0 * 1e3 << "}\n";
    }
    for (const Stall& st : rec.stalls) {
      TCB_CK(cudaEventElapsedTime(&ms, st.reach, st.go));
      if (ms <= 0.0005f) continue;
      TCB_CK(cudaEventElapsedTime(&t0, rec.marks.front(), st.reach));
      *event_log_ << "{\"dst\":\"gpu\",\"iter\":" << rec.gen << ",\"kind\":\"stall\",\"src\":\"gpu\",\"tensor\":"
                  << st.tensor << ",\"us\":" << t0 * 1e3 << ",\"wait_us\":" << ms * 1e3 << "}\n";
    }
    event_log_->flush();
  }
  for (const auto& [reach, arrival] : rec.ontime) {
    TCB_CK(cudaEventElapsedTime(&ms, reach, arrival));
    if (ms <= 0.0f) ++stats_.ontime_accesses;
  }
  for (const auto& [a0, a1] : rec.adam) {
    TCB_CK(cudaEventElapsedTime(&ms, a0, a1));
    stats_.adam_ms += ms;
  }
  // from the mapped copies written by kernels at the iteration's end: a
  // synchronous cudaMemcpy here would enter the legacy stream (often the
  // caller's compute stream) and queue on the D2H copy engine behind the
  // next iteration's bulk state stores, stalling that stream until they drain
  std::memcpy(h_checksums_.data(), h_result_ + rec.cks_buf * std::max<std::size_t>(n_accesses_, 1),
              n_accesses_ * sizeof(std::uint64_t));
  if (rec.spans) {
    const std::size_t cap = std::max<std::size_t>(recs_.size(), 1);
    const unsigned long long* sp = h_span_ + rec.cks_buf * 4 * cap;
    for (std::size_t k = 0; k < rec.spans; ++k)
      if (sp[cap + k] > sp[k]) {
        stats_.adam_span_ms += static_cast<double>(sp[cap + k] - sp[k]) * 1e-6;
        ++stats_.adam_spans;
        if (adam_stamps_ && sp[2 * cap + k] && sp[3 * cap + k] >= sp[cap + k]) {
          stamp_pre_ns_ += static_cast<double>(sp[k]) - static_cast<double>(sp[2 * cap + k]);
          stamp_post_ns_ += static_cast<double>(sp[3 * cap + k] - sp[cap + k]);
          ++stamps_;
        }
      }
  }
  scrub(rec.gen);
  events_.recycle_upto(rec.gen);
}

// Drop every reference to events of generations <= gen (all complete).
void Executor::scrub(std::uint64_t gen) {
  const std::uint64_t io_done = io_ ? io_->done() : 0;
  auto clean = [&](SlotSync& y) {
    if (y.writer && events_.done_by(y.writer, gen)) y.writer = nullptr;
    std::erase_if(y.readers, [&](cudaEvent_t e) { return events_.done_by(e, gen); });
    if (y.io_read <= io_done) y.io_read = 0;
    if (y.io_write <= io_done) y.io_write = 0;
  };
  for (SlotPool* p : {&gpu_, &host_param_, &host_opt_})
    for (auto& [size, c] : p->classes())
      for (Slot& s : c.slots) clean(s.sync);
  for (auto& [k, v] : bounce_sync_) clean(v);
  for (auto& v : stage_sync_) clean(v);
  for (auto& [k, v] : pout_sync_)
    for (auto& y : v) clean(y);
  for (auto& r : recs_) {
    if (r.arrival && events_.done_by(r.arrival, gen)) r.arrival = nullptr;
    if (r.grad_ready && events_.done_by(r.grad_ready, gen)) r.grad_ready = nullptr;
    if (r.grad_reader && events_.done_by(r.grad_reader, gen)) r.grad_reader = nullptr;
  }
  std::erase_if(barriers_, [&](cudaEvent_t e) { return events_.done_by(e, gen); });
}

void Executor::drain() {
  while (!pending_.empty()) harvest_front();
  if (io_) io_->wait_all();
  TCB_CK(cudaDeviceSynchronize());
  scrub(events_.generation());
  events_.recycle_all();
}

}  // namespace tcb
