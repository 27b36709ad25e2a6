// Per-GPU migration executor (see executor.hpp for the physical layout).
#include "executor.hpp"

#include <nvtx3/nvToolsExt.h>

#include <fcntl.h>
#include <sys/mman.h>
#include <unistd.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>

namespace tcb {

using namespace tencache;

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw DeviceError(TC_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

// ------------------------------------------------------------ EventArena
EventArena::~EventArena() {
  for (auto* v : {&free_, &free_timed_})
    for (cudaEvent_t e : *v) cudaEventDestroy(e);
  for (const Used& u : used_) cudaEventDestroy(u.e);
}

cudaEvent_t EventArena::get(bool timing) {
  auto& fr = timing ? free_timed_ : free_;
  cudaEvent_t e;
  if (fr.empty()) {
    TCB_CK(cudaEventCreateWithFlags(&e, timing ? cudaEventDefault : cudaEventDisableTiming));
  } else {
    e = fr.back();
    fr.pop_back();
  }
  used_.push_back(Used{e, timing, gen_});
  gen_of_[e] = gen_;
  return e;
}

bool EventArena::done_by(cudaEvent_t e, std::uint64_t gen) const {
  auto it = gen_of_.find(e);
  return it == gen_of_.end() || it->second <= gen;
}

void EventArena::recycle_upto(std::uint64_t gen) {
  while (!used_.empty() && used_.front().gen <= gen) {
    const Used u = used_.front();
    used_.pop_front();
    gen_of_.erase(u.e);
    (u.timed ? free_timed_ : free_).push_back(u.e);
  }
}

void EventArena::recycle_all() { recycle_upto(~0ull); }

// -------------------------------------------------------------- SlotPool
// Pinned host memory for the pools: anonymous mmap backed by transparent huge
// pages, first-touched by all host threads, then cudaHostRegister. Measured
// on the B200 boxes (tools/pin_probe.cpp, 16 GiB): cudaHostAlloc 7.0 s, this
// 0.72 s (4 KiB pages: 2.4 s) — pinning cost is per page. Returns null (the
// caller falls back to cudaHostAlloc) if the registration is refused.
static std::uint8_t* pin_region(std::uint64_t bytes, std::uint64_t* mapped_len) {
  void* p = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
  if (p == MAP_FAILED) return nullptr;
  madvise(p, bytes, MADV_HUGEPAGE);
  const unsigned nt = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  std::vector<std::thread> th;
  for (unsigned k = 0; k < nt; ++k)
    th.emplace_back([=] {
      const std::uint64_t per = (bytes / nt) & ~((2ull << 20) - 1), b = k * per, e = k + 1 == nt ? bytes : b + per;
      std::memset(static_cast<char*>(p) + b, 0, e - b);
    });
  for (auto& t : th) t.join();
  if (cudaHostRegister(p, bytes, cudaHostRegisterPortable) != cudaSuccess) {
    cudaGetLastError();
    munmap(p, bytes);
    return nullptr;
  }
  *mapped_len = bytes;
  return static_cast<std::uint8_t*>(p);
}

// One region per tier carved in ascending class order (bufpool.cpp:47-66).
// Host regions are pinned in pieces of at most 16 GiB (whole slots each): a
// single ~80 GB cudaHostAlloc is fragile on VMs, slots never straddle pieces.
void SlotPool::allocate(bool device, int dev) {
  device_ = device;
  bytes_ = 0;
  for (const auto& [size, n] : want_) bytes_ += size * n;
  if (bytes_ == 0) return;
  constexpr std::uint64_t kRegion = 16ull << 30;
  std::vector<std::pair<std::uint64_t, std::uint32_t>> slots;  // (size, class) in carving order
  for (const auto& [size, n] : want_)
    for (std::uint32_t i = 0; i < n; ++i) slots.emplace_back(size, i);
  // region plan: whole slots per piece
  std::vector<std::pair<std::size_t, std::size_t>> ranges;  // [begin, end) of slots
  std::vector<std::uint64_t> pieces;
  for (std::size_t k = 0; k < slots.size();) {
    std::uint64_t piece = 0;
    std::size_t end = k;
    while (end < slots.size() && (piece == 0 || piece + slots[end].first <= kRegion || device)) piece += slots[end++].first;
    ranges.emplace_back(k, end);
    pieces.push_back(piece);
    k = end;
  }
  regions_.assign(pieces.size(), nullptr);
  if (device) {
    for (std::size_t r = 0; r < pieces.size(); ++r) TCB_CK(cudaMalloc(&regions_[r], pieces[r]));
  } else {
    mapped_.assign(pieces.size(), 0);
    for (std::size_t r = 0; r < pieces.size(); ++r) {
      regions_[r] = pin_region(pieces[r], &mapped_[r]);
      if (!regions_[r]) TCB_CK(cudaHostAlloc(reinterpret_cast<void**>(&regions_[r]), pieces[r], cudaHostAllocPortable));
    }
  }
  for (std::size_t r = 0; r < pieces.size(); ++r) {
    std::uint64_t off = 0;
    for (std::size_t k = ranges[r].first; k < ranges[r].second; ++k) {
      SlotClass& c = classes_[slots[k].first];
      c.size = slots[k].first;
      Slot sl;
      sl.ptr = regions_[r] + off;
      off += slots[k].first;
      c.free_fifo.push_back(static_cast<std::uint32_t>(c.slots.size()));
      c.slots.push_back(sl);
    }
  }
}

void SlotPool::release_memory() {
  for (std::size_t i = 0; i < regions_.size(); ++i) {
    std::uint8_t* r = regions_[i];
    if (device_) {
      cudaFree(r);
    } else if (i < mapped_.size() && mapped_[i]) {
      cudaHostUnregister(r);
      munmap(r, mapped_[i]);
    } else {
      cudaFreeHost(r);
    }
  }
  regions_.clear();
  mapped_.clear();
}

SlotClass& SlotPool::cls(std::uint64_t size) {
  auto it = classes_.find(size);
  if (it == classes_.end()) throw DeviceError(TC_EINTERNAL, "no physical slot class of " + std::to_string(size) + " bytes");
  return it->second;
}

bool SlotPool::has_free(std::uint64_t size) const {
  auto it = classes_.find(size);
  return it != classes_.end() && !it->second.free_fifo.empty();
}

// -------------------------------------------------------------- Executor
namespace {

constexpr std::uint64_t kAlign = 4096;
std::uint64_t round_up(std::uint64_t x, std::uint64_t a) { return (x + a - 1) / a * a; }

}  // namespace


Executor::Executor(const std::string& trace_path, const std::string& machine_path, const std::string& cfg_json,
                   const tc_engine_options& opts)
    : opts_(opts) {
  const bool timing = std::getenv("TC_SETUP_TIMING") != nullptr;  // diagnostic: setup phases to stderr
  auto t_last = std::chrono::steady_clock::now();
  auto lap = [&](const char* what) {
    if (!timing) return;
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[tencache setup] %-28s %8.3f s\n", what, std::chrono::duration<double>(now - t_last).count());
    t_last = now;
  };
  device_ = opts.device;
  TCB_CK(cudaSetDevice(device_));
  lap("cuda context");
  trace_ = load_trace(trace_path);
  machine_ = machine_from(machine_path.c_str());
  cfg_ = parse_run_config(cfg_json.c_str());
  policy_ = make_policy(trace_, machine_, cfg_);
  policy_->init();
  lap("trace + policy init");

  // tensor table
  recs_.reserve(trace_.tensors.size());
  for (const auto& t : trace_.tensors) {
    index_[t.id] = static_cast<std::int32_t>(recs_.size());
    TensorRec r;
    r.id = t.id;
    r.bytes = t.size_bytes;
    r.is_state = t.kind == TensorKind::OptStateFP32;
    recs_.push_back(r);
  }
  for (const TraceStep& st : trace_.steps)  // decisions key the update on the first id (scheduler.cpp:321)
    if (st.phase == Phase::OptimizerUpdate && trace_.tensor(st.tensor_ids.front()).kind != TensorKind::OptStateFP32)
      throw ConfigError("executor: optimizer step " + std::to_string(st.step_index) + " must list its state first");
  for (const auto& [sid, pid] : trace_.optimizer_pairs()) {
    if (pid == 0) continue;
    TensorRec& s = rec(sid);
    TensorRec& p = rec(pid);
    if (s.bytes != 6 * p.bytes || p.bytes % 16 != 0)
      throw ConfigError("optimizer state " + std::to_string(sid) + " must be 6x its bf16 parameter (16-byte multiple)");
    s.partner = index_.at(pid);
    p.partner = index_.at(sid);
  }

  // physical pools: the peak number of tensors of each (tier, class) holding
  // a slot over the policy's decisions (dry run), at least the policy's own
  // logical pool sizes, plus spare slots per class.
  const int gspare = std::max(opts.gpu_spare_slots, 1), hspare = std::max(opts.host_spare_slots, 1);
  double fwd_h2d = 0;
  std::map<std::pair<int, std::uint64_t>, std::uint32_t> need = simulate_occupancy(&fwd_h2d);
  lap("occupancy dry run");
  if (const SchedulerState* st = policy_->scheduler_state()) {
    std::map<std::pair<int, std::uint64_t>, std::uint32_t> logical;
    for (const Chunk& c : st->gpu_pool.chunks()) ++logical[{0, c.size}];
    for (const Chunk& c : st->cpu_pool.chunks()) ++logical[{1, c.size}];
    for (const Chunk& c : st->cpu_opt_pool.chunks()) ++logical[{2, c.size}];
    for (const auto& [k, v] : logical) need[k] = std::max(need[k], v);
  }
  std::map<std::uint64_t, bool> pclass, sclass;
  for (const auto& r : recs_) (r.is_state ? sclass : pclass)[r.bytes] = true;
  for (const auto& [size, _] : pclass) {
    gpu_.plan(size, need[{0, size}] + gspare);
    host_param_.plan(size, need[{1, size}] + hspare);
  }
  for (const auto& [size, _] : sclass) {
    if (need[{0, size}]) gpu_.plan(size, need[{0, size}] + 1);  // GPU-resident states (no offload)
    host_opt_.plan(size, need[{2, size}] + hspare + 1);          // +1 transient
  }
  gpu_.allocate(true, device_);
  lap("HBM pool");
  host_param_.allocate(false, device_);
  host_opt_.allocate(false, device_);
  lap("pinned host pools");
  if (timing) {  // how much of the process is backed by transparent huge pages (DMA-friendly)
    std::ifstream sm("/proc/self/smaps_rollup");
    for (std::string line; std::getline(sm, line);)
      if (line.rfind("AnonHugePages", 0) == 0 || line.rfind("Rss:", 0) == 0)
        std::fprintf(stderr, "[tencache setup] %s\n", line.c_str());
  }

  // NVMe tier: one sparse file, a 4 KiB-aligned extent per tensor
  std::uint64_t off = 0;
  bool all_aligned = true;
  for (auto& r : recs_) {
    r.nvme_off = off;
    off += round_up(r.bytes, kAlign);
    all_aligned = all_aligned && r.bytes % kAlign == 0;
  }
  std::string dir = opts.nvme_dir && *opts.nvme_dir ? opts.nvme_dir : "";
  if (dir.empty()) dir = std::getenv("TMPDIR") ? std::getenv("TMPDIR") : "/tmp";
  {
    const char* nf = std::getenv("TC_NVME_FILES");
    nvme_ = std::make_unique<StripedFile>(dir, off, nf ? std::atoi(nf) : 16, opts.direct_io && all_aligned);
  }
  if (const char* c = std::getenv("TC_OPT_YIELD")) opt_yield_ = std::atoi(c) != 0;
  if (const char* c = std::getenv("TC_PRESTAGE_FWD")) prestage_fwd_override_ = std::atoi(c);
  if (const char* c = std::getenv("TC_PRESTAGE_GATE")) prestage_gate_ = std::atoi(c) != 0;
  if (const char* c = std::getenv("TC_EDGE_FILL")) edge_fill_ = std::atoi(c) != 0;
  if (const char* c = std::getenv("TC_LOOKAHEAD")) lookahead_ = std::atoi(c) != 0;
  if (const char* c = std::getenv("TC_ADAM_STAMPS")) adam_stamps_ = std::atoi(c) != 0;
  {  // migration-bound? trace compute time vs the optimizer states' H2D time alone (machine.cpp:101-111)
    double compute_us = 0, state_bytes = 0;
    for (const TraceStep& st : trace_.steps)
      if (st.phase != Phase::OptimizerUpdate) compute_us += st.compute_us * cfg_.batch_scale;
    for (const auto& r : recs_)
      if (r.is_state) state_bytes += static_cast<double>(r.bytes);
    try {
      const double bw = to_double(machine_.effective_bandwidth(Tier::Cpu, Tier::Gpu)) * 1e3;  // bytes per us
      adam_on_compute_ = bw > 0 && compute_us < state_bytes / bw;
    } catch (...) {
      adam_on_compute_ = false;
    }
  }
  if (const char* c = std::getenv("TC_ADAM_ON_COMPUTE")) adam_on_compute_ = std::atoi(c) != 0;
  if (!std::getenv("TC_SYNC_NVME")) {
    try {
      io_ = std::make_unique<NvmeQueue>(device_, nvme_.get());
      TCB_CK(cudaStreamCreateWithFlags(&io_join_, cudaStreamNonBlocking));
    } catch (const std::exception&) {
      io_.reset();  // no stream memory operations: synchronous NVMe I/O
    }
  }

  lap("NVMe tier files + I/O pool");
  for (const auto& [size, _] : pclass) {
    void* p = nullptr;
    TCB_CK(cudaHostAlloc(&p, size, cudaHostAllocPortable));
    bounce_[size] = static_cast<std::uint8_t*>(p);
    bounce_sync_[size] = SlotSync{};
  }
  std::uint64_t max_state = 0;
  for (const auto& [size, _] : sclass) max_state = std::max(max_state, size);
  for (const auto& [size, _] : pclass) max_state = std::max(max_state, 6 * size);  // seed scratch
  stage_bytes_ = max_state;
  const int nstage = opts.opt_stage_slots > 0 ? std::max(opts.opt_stage_slots, 2) : auto_stage_slots(fwd_h2d);
  if (timing) std::fprintf(stderr, "[tencache setup] optimizer stage ring: %d stages\n", nstage);
  for (int i = 0; i < nstage; ++i) {
    void* p = nullptr;
    TCB_CK(cudaMalloc(&p, stage_bytes_));
    stage_.push_back(static_cast<std::uint8_t*>(p));
    stage_sync_.emplace_back();
    stage_free_.push_back(static_cast<std::size_t>(i));
  }
  for (const auto& [size, _] : pclass) {
    for (int i = 0; i < 2; ++i) {
      void* p = nullptr;
      TCB_CK(cudaMalloc(&p, size));
      pout_scratch_[size].push_back(static_cast<std::uint8_t*>(p));
      pout_sync_[size].emplace_back();
    }
    pout_next_[size] = 0;
  }
  lap("bounce + HBM stages");
  std::uint64_t gbytes = 0;
  for (const auto& r : recs_)
    if (!r.is_state) gbytes += r.bytes;
  if (gbytes) TCB_CK(cudaMalloc(&grads_, gbytes));
  gbytes = 0;
  for (auto& r : recs_)
    if (!r.is_state) {
      r.grad = grads_ + gbytes;
      gbytes += r.bytes;
    }
  for (const auto& s : trace_.steps)
    if (s.phase != Phase::OptimizerUpdate) n_accesses_ += s.tensor_ids.size();
  TCB_CK(cudaMalloc(&d_checksums_, 2 * std::max<std::size_t>(n_accesses_, 1) * sizeof(std::uint64_t)));
  TCB_CK(cudaMalloc(&d_span_, 2 * 4 * std::max<std::size_t>(recs_.size(), 1) * sizeof(unsigned long long)));
  h_checksums_.assign(n_accesses_, 0);
  TCB_CK(cudaHostAlloc(&h_result_, 2 * std::max<std::size_t>(n_accesses_, 1) * sizeof(std::uint64_t),
                       cudaHostAllocMapped));
  TCB_CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&d_result_), h_result_, 0));
  TCB_CK(cudaHostAlloc(reinterpret_cast<void**>(&h_span_), 2 * 4 * std::max<std::size_t>(recs_.size(), 1) *
                       sizeof(unsigned long long), cudaHostAllocMapped));
  TCB_CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&d_span_host_), h_span_, 0));
  for (auto& e : result_ev_) TCB_CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  TCB_CK(cudaStreamCreateWithFlags(&h2d_, cudaStreamNonBlocking));
  TCB_CK(cudaStreamCreateWithFlags(&d2h_, cudaStreamNonBlocking));
  int lo_prio = 0, hi_prio = 0;  // the fused AdamW gets the highest stream priority
  TCB_CK(cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio));
  const char* op = std::getenv("TC_OPT_PRIORITY");  // diagnostic: 0 = default priority for the AdamW stream
  TCB_CK(cudaStreamCreateWithPriority(&opt_, cudaStreamNonBlocking, (op && std::atoi(op) == 0) ? lo_prio : hi_prio));
  TCB_CK(cudaStreamCreateWithFlags(&h2d_opt_, cudaStreamNonBlocking));
  TCB_CK(cudaStreamCreateWithFlags(&d2h_opt_, cudaStreamNonBlocking));

  // initial physical placement = the policy's placement
  for (auto& r : recs_) {
    const Tier t = policy_->initial_tier(r.id).value_or(Tier::Cpu);
    if (t == Tier::Gpu) {
      r.tier = PTier::Gpu;
      r.slot = take_slot(PTier::Gpu, r.bytes, index_of(r.id));
    } else if (t == Tier::Cpu) {
      r.tier = host_tier(r);
      r.slot = take_slot(r.tier, r.bytes, index_of(r.id));
    } else {
      r.tier = PTier::Nvme;
    }
    r.nvme_valid = t == Tier::Nvme;
  }
}

Executor::~Executor() {
  if (adam_stamps_ && stamps_)
    std::fprintf(stderr, "[tencache] AdamW launches: %.0f: stream reaches it -> first CTA %.2f us, "
                 "last CTA end -> next op %.2f us (avg)\n",
                 static_cast<double>(stamps_), stamp_pre_ns_ / stamps_ * 1e-3, stamp_post_ns_ / stamps_ * 1e-3);
  cudaSetDevice(device_);
  try {
    drain();
  } catch (...) {
  }
  io_.reset();
  if (h2d_) cudaStreamSynchronize(h2d_);
  if (d2h_) cudaStreamSynchronize(d2h_);
  cudaDeviceSynchronize();
  gpu_.release_memory();
  host_param_.release_memory();
  host_opt_.release_memory();
  for (auto& [s, p] : bounce_) cudaFreeHost(p);
  for (auto* p : stage_) cudaFree(p);
  for (auto& [s, v] : pout_scratch_)
    for (auto* p : v) cudaFree(p);
  if (grads_) cudaFree(grads_);
  if (d_checksums_) cudaFree(d_checksums_);
  if (h_result_) cudaFreeHost(h_result_);
  if (h_span_) cudaFreeHost(h_span_);
  for (auto& e : result_ev_)
    if (e) cudaEventDestroy(e);
  if (d_span_) cudaFree(d_span_);
  if (h2d_) cudaStreamDestroy(h2d_);
  if (d2h_) cudaStreamDestroy(d2h_);
  if (opt_) cudaStreamDestroy(opt_);
  if (h2d_opt_) cudaStreamDestroy(h2d_opt_);
  if (d2h_opt_) cudaStreamDestroy(d2h_opt_);
  if (io_join_) cudaStreamDestroy(io_join_);
  if (compute_owned_) cudaStreamDestroy(compute_owned_);
  if (z3_) {
    for (auto& [k, cp] : z3_->plans)
      if (cp.segs) cudaFree(cp.segs);
    for (void* p : z3_->opened) cudaIpcCloseMemHandle(p);
    if (z3_->ctl) cudaFree(z3_->ctl);
    for (std::uint8_t* p : {z3_->gather, z3_->view, z3_->gview, z3_->gpad})
      if (p) cudaFree(p);
    if (z3_->comm) nccl().CommDestroy(z3_->comm);
  }
}

// Dry run of one iteration of decisions on a fresh policy: the peak number
// of tensors per (tier, size) that must hold a slot at once. Tier keys: 0 GPU,
// 1 host parameter cache, 2 host optimizer-state cache. A retained source
// (src_retains) keeps its slot; a destination that already has the bytes
// (dst_has_copy) takes none.
std::map<std::pair<int, std::uint64_t>, std::uint32_t> Executor::simulate_occupancy(double* fwd_h2d) const {
  std::unique_ptr<IPolicy> pol = make_policy(trace_, machine_, cfg_);
  pol->init();
  std::unordered_map<TensorId, std::set<Tier>> where;
  std::unordered_map<TensorId, std::pair<std::uint64_t, bool>> info;  // size, is_state
  std::map<std::pair<int, std::uint64_t>, std::int64_t> cur;
  std::map<std::pair<int, std::uint64_t>, std::uint32_t> peak;
  auto key = [&](TensorId id, Tier t) -> std::pair<int, std::uint64_t> {
    const auto& [size, st] = info.at(id);
    return {t == Tier::Gpu ? 0 : (st ? 2 : 1), size};
  };
  auto add = [&](TensorId id, Tier t, int d) {
    if (t == Tier::Nvme) return;
    auto k = key(id, t);
    cur[k] += d;
    if (cur[k] > 0) peak[k] = std::max<std::uint32_t>(peak[k], static_cast<std::uint32_t>(cur[k]));
  };
  for (const auto& t : trace_.tensors) {
    info[t.id] = {t.size_bytes, t.kind == TensorKind::OptStateFP32};
    const Tier tier = pol->initial_tier(t.id).value_or(Tier::Cpu);
    where[t.id] = {tier};
    add(t.id, tier, +1);
  }
  auto apply_reqs = [&](const std::vector<TransferRequest>& reqs) {
    for (const TransferRequest& r : reqs) {
      auto& w = where[r.tensor_id];
      if (!r.src_retains && w.erase(r.src)) add(r.tensor_id, r.src, -1);
      if (w.insert(r.dst).second) add(r.tensor_id, r.dst, +1);
    }
  };
  std::size_t first_opt = trace_.steps.size();
  for (std::size_t i = 0; i < trace_.steps.size(); ++i)
    if (trace_.steps[i].phase == Phase::OptimizerUpdate) {
      first_opt = i;
      break;
    }
  double fwd = 0;
  auto fwd_bytes = [&](const std::vector<TransferRequest>& reqs, std::size_t i) {
    if (trace_.steps[i].phase != Phase::Forward) return;
    for (const TransferRequest& r : reqs)
      if (!r.instant && r.dst == Tier::Gpu) fwd += static_cast<double>(r.size_bytes);
  };
  for (int it = 0; it < 2; ++it) {
    bool restored = false;
    fwd = 0;  // the second (steady-state) iteration's value is kept
    for (std::size_t i = 0; i < trace_.steps.size(); ++i) {
      if (cfg_.restore_overlap && i == first_opt && !restored) {
        restored = true;
        apply_reqs(pol->on_param_restore_point());
      }
      const auto b = pol->on_step_begin(trace_.steps[i]);
      fwd_bytes(b, i);
      apply_reqs(b);
      const auto e = pol->on_step_end(trace_.steps[i]);
      fwd_bytes(e, i);
      apply_reqs(e);
    }
    if (!restored) apply_reqs(pol->on_param_restore_point());
    apply_reqs(pol->on_iteration_end());
    pol->reset_iteration();
  }
  if (fwd_h2d) *fwd_h2d = fwd;
  return peak;
}

// opt_stage_slots <= 0: size the HBM stage ring so the forward pass can
// pre-stage as many optimizer states as its spare H2D time carries (trace
// compute time x the machine model's CPU->GPU bandwidth minus the forward's
// own cache prefetches), plus the backward's lookahead; at least 12, at most
// half the free HBM. Measured optima it reproduces: 12 on C2 at 16k tokens,
// ~118 on C5 (profiles/r01_stage_sweep.json).
int Executor::auto_stage_slots(double fwd_h2d) const {
  double fwd_us = 0, sbytes = 0;
  std::size_t nstates = 0;
  for (const TraceStep& st : trace_.steps)
    if (st.phase == Phase::Forward) fwd_us += st.compute_us * cfg_.batch_scale;
  for (const auto& r : recs_)
    if (r.is_state) {
      sbytes = std::max(sbytes, static_cast<double>(r.bytes));
      ++nstates;
    }
  if (nstates == 0 || sbytes == 0) return 12;
  double bw = 0;
  try {
    bw = to_double(machine_.effective_bandwidth(Tier::Cpu, Tier::Gpu)) * 1e3;  // bytes per us
  } catch (...) {
    return 12;
  }
  const double spare = std::max(0.0, fwd_us * bw - fwd_h2d);
  std::size_t n = static_cast<std::size_t>(spare / sbytes) + 4;
  std::size_t free_b = 0, total_b = 0;
  if (cudaMemGetInfo(&free_b, &total_b) == cudaSuccess)
    n = std::min<std::size_t>(n, static_cast<std::size_t>(0.5 * static_cast<double>(free_b) / sbytes));
  n = std::min(n, nstates + 2);
  return static_cast<int>(std::max<std::size_t>(n, 12));
}

std::int32_t Executor::index_of(TensorId id) const {
  auto it = index_.find(id);
  if (it == index_.end()) throw TraceError("unknown tensor id " + std::to_string(id));
  return it->second;
}

TensorRec& Executor::rec(TensorId id) { return recs_[static_cast<std::size_t>(index_of(id))]; }

SlotPool& Executor::pool(PTier t) {
  switch (t) {
    case PTier::Gpu: return gpu_;
    case PTier::HostParam: return host_param_;
    case PTier::HostOpt: return host_opt_;
    default: throw DeviceError(TC_EINTERNAL, "NVMe has no slot pool");
  }
}

Slot& Executor::slot_of(const TensorRec& r) { return pool(r.tier).cls(r.bytes).slots.at(r.slot); }
std::uint8_t* Executor::where(const TensorRec& r) { return slot_of(r).ptr; }

std::uint32_t Executor::take_slot(PTier t, std::uint64_t size, std::int32_t occupant) {
  SlotClass& c = pool(t).cls(size);
  if (c.free_fifo.empty()) throw DeviceError(TC_EINTERNAL, "physical slot pool exhausted (class " + std::to_string(size) + ")");
  const std::uint32_t s = c.free_fifo.front();
  c.free_fifo.pop_front();
  c.slots[s].occupant = occupant;
  return s;
}

void Executor::free_slot(PTier t, std::uint64_t size, std::uint32_t s) {
  SlotClass& c = pool(t).cls(size);
  c.slots[s].occupant = -1;
  c.free_fifo.push_back(s);
}

void Executor::wait_for_read(cudaStream_t s, const SlotSync& y) {
  if (y.writer) TCB_CK(cudaStreamWaitEvent(s, y.writer, 0));
  if (y.io_write && io_) io_->stream_wait(s, y.io_write);
}

void Executor::wait_for_write(cudaStream_t s, const SlotSync& y) {
  if (y.writer) TCB_CK(cudaStreamWaitEvent(s, y.writer, 0));
  for (cudaEvent_t e : y.readers) TCB_CK(cudaStreamWaitEvent(s, e, 0));
  if (io_) {
    io_->stream_wait(s, y.io_read);
    io_->stream_wait(s, y.io_write);
  }
  if (y.peer_cnt && y.peer_target) stream_wait_value32(s, y.peer_cnt, y.peer_target);
}

void Executor::host_wait_all(const SlotSync& y) {
  if (y.writer) TCB_CK(cudaEventSynchronize(y.writer));
  for (cudaEvent_t e : y.readers) TCB_CK(cudaEventSynchronize(e));
  if (io_) {
    io_->wait(y.io_read);
    io_->wait(y.io_write);
  }
}

// The I/O worker waits on events later, on its own thread; an event it names
// could meanwhile be recycled and re-recorded behind GPU work that waits on
// that very job. So a job never names slot events directly: they are joined
// on a side stream into ONE fresh event of the current generation, which is
// harvested only after all of that generation's jobs completed.
std::vector<cudaEvent_t> Executor::io_deps(std::vector<cudaEvent_t> deps) {
  std::erase(deps, nullptr);
  if (deps.empty()) return {};
  for (cudaEvent_t e : deps) TCB_CK(cudaStreamWaitEvent(io_join_, e, 0));
  cudaEvent_t j = events_.get(false);
  TCB_CK(cudaEventRecord(j, io_join_));
  return {j};
}

// NVMe -> host buffer once every GPU op touching `target` is done; returns the
// job (GPU consumers wait on it through target.io_write).
std::uint64_t Executor::nvme_read_async(TensorRec& r, void* dst, SlotSync& target) {
  std::vector<cudaEvent_t> waits(target.readers.begin(), target.readers.end());
  if (target.writer) waits.push_back(target.writer);
  // after: the buffer's previous job and the extent's previous job (a pending
  // write of the same tensor must land before it is read back)
  const std::uint64_t k = io_->submit_read(dst, r.bytes, r.nvme_off, io_deps(std::move(waits)),
                                           {target.io_read, target.io_write, r.nvme_job});
  r.nvme_job = k;
  target = SlotSync{};
  target.io_write = k;
  stats_.nvme_read_bytes += r.bytes;
  return k;
}

// host buffer -> NVMe once the copy that filled `source` is done; later writers
// of the buffer wait on source.io_read.
std::uint64_t Executor::nvme_write_async(TensorRec& r, const void* src, SlotSync& source) {
  std::vector<cudaEvent_t> waits;
  if (source.writer) waits.push_back(source.writer);
  const std::uint64_t k =
      io_->submit_write(src, r.bytes, r.nvme_off, io_deps(std::move(waits)),
                        // the buffer's previous reader too: source.io_read must keep naming a job
                        // whose completion implies every earlier read of the buffer finished
                        {source.io_write, source.io_read, r.nvme_job});
  r.nvme_job = k;
  source.io_read = k;
  r.nvme_valid = true;
  stats_.nvme_write_bytes += r.bytes;
  return k;
}

cudaEvent_t Executor::copy(cudaStream_t s, void* dst, const void* src, std::uint64_t n, bool h2d) {
  Copy c;
  c.start = events_.get(true);
  c.end = events_.get(true);
  c.h2d = h2d;
  c.bytes = n;
  c.tag = tag_;
  TCB_CK(cudaEventRecord(c.start, s));
  TCB_CK(cudaMemcpyAsync(dst, src, n, h2d ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost, s));
  TCB_CK(cudaEventRecord(c.end, s));
  copies_.push_back(c);
  ++stats_.copies;
  return c.end;
}

void Executor::nvme_read(const TensorRec& r, void* dst) {
  if (!nvme_->io(false, static_cast<std::uint8_t*>(dst), r.bytes, r.nvme_off))
    throw DeviceError(TC_EIO, "NVMe tier read failed for tensor " + std::to_string(r.id));
  stats_.nvme_read_bytes += r.bytes;
}

void Executor::nvme_write(TensorRec& r, const void* src) {
  if (!nvme_->io(true, const_cast<std::uint8_t*>(static_cast<const std::uint8_t*>(src)), r.bytes, r.nvme_off))
    throw DeviceError(TC_EIO, "NVMe tier write failed for tensor " + std::to_string(r.id));
  r.nvme_valid = true;
  stats_.nvme_write_bytes += r.bytes;
}

// An "instant" move to NVMe claims a clean replica. After an optimizer update
// the replica is stale, so the executor writes the current bytes first
// (SURVEY.md §7 traffic category iii).
void Executor::ensure_nvme_fresh(TensorRec& r) {
  if (r.nvme_valid) return;
  tag_ = CopyTag{"writeback", r.id, 0, 2};
  if (r.tier == PTier::Gpu) {
    Slot& g = slot_of(r);
    std::uint8_t* b = bounce_.at(r.bytes);
    SlotSync& bs = bounce_sync_[r.bytes];
    if (!io_) host_wait_all(bs);
    wait_for_read(d2h_, g.sync);
    wait_for_write(d2h_, bs);
    cudaEvent_t e = copy(d2h_, b, g.ptr, r.bytes, false);
    g.sync.readers.push_back(e);
    if (io_) {
      bs = SlotSync{e, {}};
      nvme_write_async(r, b, bs);
    } else {
      TCB_CK(cudaEventSynchronize(e));
      bs = SlotSync{};
      nvme_write(r, b);
    }
  } else {
    Slot& h = slot_of(r);
    if (io_) {
      nvme_write_async(r, h.ptr, h.sync);
    } else {
      host_wait_all(h.sync);
      nvme_write(r, h.ptr);
    }
  }
  stats_.writeback_bytes += r.bytes;
}

bool Executor::dest_available(const Req& r) const {
  if (r.instant || r.dst == Tier::Nvme) return true;
  const TensorRec& x = recs_[static_cast<std::size_t>(index_of(r.tensor_id))];
  if (r.dst == Tier::Gpu) return gpu_.has_free(x.bytes);
  return (x.is_state ? host_opt_ : host_param_).has_free(x.bytes);
}

// Requests run in order, except that one whose destination class has no free
// physical slot yet waits for a later departure from that class (never past
// an earlier request for the same tensor).
void Executor::execute(std::vector<Req> reqs) {
  while (!reqs.empty()) {
    std::size_t pick = reqs.size();
    for (std::size_t i = 0; i < reqs.size() && pick == reqs.size(); ++i) {
      bool blocked = false;
      for (std::size_t j = 0; j < i && !blocked; ++j) blocked = reqs[j].tensor_id == reqs[i].tensor_id;
      if (!blocked && dest_available(reqs[i])) pick = i;
    }
    if (pick == reqs.size()) throw DeviceError(TC_EINTERNAL, "no physical slot for any pending transfer");
    apply(reqs[pick]);
    reqs.erase(reqs.begin() + static_cast<std::ptrdiff_t>(pick));
  }
}

void Executor::apply(const Req& r) {
  TensorRec& x = rec(r.tensor_id);
  ++stats_.requests;
  if (!r.instant) ++x.issued_since_access;
  const bool src_ok = (r.src == Tier::Gpu && x.tier == PTier::Gpu) ||
                      (r.src == Tier::Cpu && (x.tier == PTier::HostParam || x.tier == PTier::HostOpt)) ||
                      (r.src == Tier::Nvme && x.tier == PTier::Nvme);
  if (!src_ok)
    throw DeviceError(TC_EINTERNAL, "executor/policy desync: tensor " + std::to_string(x.id) + " not in " + to_string(r.src));
  const std::int32_t xi = index_of(x.id);
  cudaEvent_t done = nullptr;
  static const char* const kKinds[] = {"prefetch", "evict", "restore"};
  tag_ = CopyTag{kKinds[static_cast<int>(r.kind)], r.tensor_id, static_cast<std::uint8_t>(r.src),
                 static_cast<std::uint8_t>(r.dst)};

  if (r.src == Tier::Gpu && r.dst == Tier::Cpu && r.instant) {  // drop: the retained home copy is primary again
    if (!x.has_home) throw DeviceError(TC_EINTERNAL, "instant GPU->CPU drop without a retained home copy");
    Slot& g = slot_of(x);
    Slot& h = pool(x.home_tier).cls(x.bytes).slots[x.home_slot];
    if (!x.home_valid) {  // updated on the GPU since the fetch: write the bytes home first
      wait_for_read(d2h_, g.sync);
      wait_for_write(d2h_, h.sync);
      done = copy(d2h_, h.ptr, g.ptr, x.bytes, false);
      g.sync.readers.push_back(done);
      h.sync = SlotSync{done, {}};
      stats_.writeback_bytes += x.bytes;
    }
    free_slot(PTier::Gpu, x.bytes, x.slot);
    x.tier = x.home_tier;
    x.slot = x.home_slot;
    x.has_home = x.home_valid = false;
  } else if (r.src == Tier::Gpu && r.dst == Tier::Cpu) {  // evict / restore, D2H
    Slot& g = slot_of(x);
    const PTier ht = host_tier(x);
    const std::uint32_t hs = take_slot(ht, x.bytes, xi);
    Slot& h = pool(ht).cls(x.bytes).slots[hs];
    wait_for_read(d2h_, g.sync);
    wait_for_write(d2h_, h.sync);
    done = copy(d2h_, h.ptr, g.ptr, x.bytes, false);
    g.sync.readers.push_back(done);
    h.sync.writer = done;
    h.sync.readers.clear();
    free_slot(PTier::Gpu, x.bytes, x.slot);
    x.tier = ht;
    x.slot = hs;
    stats_.d2h_bytes += x.bytes;
  } else if (r.src == Tier::Cpu && r.dst == Tier::Gpu) {  // prefetch / restore, H2D
    Slot& h = slot_of(x);
    const std::uint32_t gs = take_slot(PTier::Gpu, x.bytes, xi);
    Slot& g = gpu_.cls(x.bytes).slots[gs];
    wait_for_read(h2d_, h.sync);
    wait_for_write(h2d_, g.sync);
    done = copy(h2d_, g.ptr, h.ptr, x.bytes, true);
    h.sync.readers.push_back(done);
    g.sync.writer = done;
    g.sync.readers.clear();
    if (r.src_retains) {  // comparison policies: the home copy stays valid and allocated
      x.has_home = true;
      x.home_valid = true;
      x.home_tier = x.tier;
      x.home_slot = x.slot;
    } else {
      free_slot(x.tier, x.bytes, x.slot);
    }
    x.tier = PTier::Gpu;
    x.slot = gs;
    x.arrival = done;
    stats_.h2d_bytes += x.bytes;
  } else if (r.src == Tier::Nvme && r.dst == Tier::Gpu) {  // staged: NVMe -> bounce -> HBM
    const std::uint32_t gs = take_slot(PTier::Gpu, x.bytes, xi);
    Slot& g = gpu_.cls(x.bytes).slots[gs];
    std::uint8_t* b = bounce_.at(x.bytes);
    SlotSync& bs = bounce_sync_[x.bytes];
    if (io_) {
      nvme_read_async(x, b, bs);
    } else {
      host_wait_all(bs);
      nvme_read(x, b);
      bs = SlotSync{};
    }
    wait_for_write(h2d_, g.sync);
    wait_for_read(h2d_, bs);
    done = copy(h2d_, g.ptr, b, x.bytes, true);
    bs.readers.push_back(done);
    g.sync.writer = done;
    g.sync.readers.clear();
    if (!r.src_retains) x.nvme_valid = false;
    x.tier = PTier::Gpu;
    x.slot = gs;
    x.arrival = done;
    stats_.h2d_bytes += x.bytes;
  } else if (r.src == Tier::Nvme && r.dst == Tier::Cpu) {  // state (or param) read into host memory
    const PTier ht = host_tier(x);
    const std::uint32_t hs = take_slot(ht, x.bytes, xi);
    Slot& h = pool(ht).cls(x.bytes).slots[hs];
    if (io_) {
      nvme_read_async(x, h.ptr, h.sync);
    } else {
      host_wait_all(h.sync);
      nvme_read(x, h.ptr);
      h.sync = SlotSync{};
    }
    if (!r.src_retains) x.nvme_valid = false;
    x.tier = ht;
    x.slot = hs;
  } else if (r.src == Tier::Cpu && r.dst == Tier::Nvme) {  // spill / state write-back
    Slot& h = slot_of(x);
    if (!r.instant || !x.nvme_valid) {
      if (io_) {
        const std::uint64_t k = nvme_write_async(x, h.ptr, h.sync);  // later writers of the slot wait on the job
        if (r.blocking) barrier_io_ = std::max(barrier_io_, k);
      } else {
        host_wait_all(h.sync);
        nvme_write(x, h.ptr);
        h.sync = SlotSync{};
      }
    }
    free_slot(x.tier, x.bytes, x.slot);
    x.tier = PTier::Nvme;
  } else if (r.src == Tier::Gpu && r.dst == Tier::Nvme) {  // drop (replica authoritative) or write-back
    ensure_nvme_fresh(x);
    free_slot(PTier::Gpu, x.bytes, x.slot);
    x.tier = PTier::Nvme;
  } else {
    throw DeviceError(TC_EINTERNAL, "unsupported transfer direction");
  }
  if (r.blocking && done) barriers_.push_back(done);
  if (done && !r.instant) (r.dst == Tier::Gpu ? last_h2d_ : last_d2h_) = done;
}

void Executor::wait_barriers(cudaStream_t cs) {
  for (cudaEvent_t e : barriers_) TCB_CK(cudaStreamWaitEvent(cs, e, 0));
  barriers_.clear();
  if (barrier_io_ && io_) io_->stream_wait_upto(cs, barrier_io_);
  barrier_io_ = 0;
}

void Executor::param_step(const TraceStep& step, std::size_t, cudaStream_t cs) {
  cudaEvent_t reach = events_.get(true), go = events_.get(true);
  TCB_CK(cudaEventRecord(reach, cs));
  for (TensorId id : step.tensor_ids) {
    TensorRec& x = rec(id);
    if (x.tier != PTier::Gpu) throw DeviceError(TC_EINTERNAL, "step tensor " + std::to_string(id) + " not GPU-resident");
    wait_for_read(cs, slot_of(x).sync);
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
    if (z3_) {
      zero3_access(x, step.phase == Phase::Backward, cs);
    } else if (access_cursor_ < n_accesses_) {
      TCB_CK(launch_checksum(where(x), x.bytes & ~3ull,
                             reinterpret_cast<unsigned long long*>(cks_base_ + access_cursor_), cs));
      ++stats_.kernel_launches;
      ++access_cursor_;
    }
  }
  if (so_.compute_mode == 1) {
    const double us = step.compute_us * cfg_.batch_scale;
    TCB_CK(launch_spin(static_cast<std::uint64_t>(us * 1000.0), so_.spin_ctas, cs));
    ++stats_.kernel_launches;
  }
  cudaEvent_t done = events_.get(false);
  TCB_CK(cudaEventRecord(done, cs));
  for (TensorId id : step.tensor_ids) slot_of(rec(id)).sync.readers.push_back(done);
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
  if (opt_yield_ && last_h2d_) TCB_CK(cudaStreamWaitEvent(h2d_opt_, last_h2d_, 0));
  wait_for_write(h2d_opt_, stage_sync_[b]);
  wait_for_read(h2d_opt_, h.sync);
  cudaEvent_t e1 = copy(h2d_opt_, stage_[b], h.ptr, s.bytes, true);
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

void Executor::optimizer_work(TensorRec& s, TensorRec& p) {
  cudaStream_t ost = adam_stream();
  const bool state_on_gpu = s.tier == PTier::Gpu;  // no-offload posture: update in place in HBM
  if (!state_on_gpu && s.tier != PTier::HostOpt)
    throw DeviceError(TC_EINTERNAL, "optimizer state not in host memory at its update");
  const std::uint64_t n = p.bytes / 2;
  std::uint8_t* stg;
  std::size_t b = 0;
  if (state_on_gpu) {
    Slot& gs = slot_of(s);
    stg = gs.ptr;
    wait_for_write(ost, gs.sync);
  } else {
    auto it = staged_.find(index_of(s.id));
    b = it != staged_.end() ? it->second : stage_state(s);
    staged_.erase(index_of(s.id));
    stats_.opt_h2d_bytes += s.bytes;  // counted at the update it feeds (staging may be a prologue)
    stg = stage_[b];
    // (null once a drain between the prologue's staging and this update completed it)
    if (stage_sync_[b].writer) TCB_CK(cudaStreamWaitEvent(ost, stage_sync_[b].writer, 0));
  }
  if (p.grad_ready) TCB_CK(cudaStreamWaitEvent(ost, p.grad_ready, 0));
  std::uint8_t* pout;
  SlotSync* psync;
  const bool on_gpu = p.tier == PTier::Gpu;
  if (on_gpu) {
    Slot& g = slot_of(p);
    pout = g.ptr;
    psync = &g.sync;
  } else {
    std::size_t& k = pout_next_[p.bytes];
    pout = pout_scratch_[p.bytes][k];
    psync = &pout_sync_[p.bytes][k];
    k = (k + 1) % pout_scratch_[p.bytes].size();
  }
  wait_for_write(ost, *psync);
  cudaEvent_t a0 = events_.get(true), a1 = events_.get(true);
  TCB_CK(cudaEventRecord(a0, ost));
  auto* st = reinterpret_cast<float*>(stg);
  const AdamScalars sc = adam_scalars(so_.lr, so_.beta1, so_.beta2, so_.eps, so_.weight_decay, adam_step_);
  unsigned long long *smin = nullptr, *smax = nullptr;
  const std::size_t cap = std::max<std::size_t>(recs_.size(), 1);
  if (span_cursor_ < cap && adamw_variant() >= 2) {  // in-kernel resident span (TMA variants)
    smin = span_base_ + span_cursor_;
    smax = span_base_ + cap + span_cursor_;
    ++span_cursor_;
  }
  if (adam_stamps_ && smin) TCB_CK(launch_stamp(smin + 2 * cap, ost));
  TCB_CK(launch_adamw(st, st + n, st + 2 * n, reinterpret_cast<const std::uint16_t*>(p.grad),
                      reinterpret_cast<std::uint16_t*>(pout), n, sc, so_.grad_scale, ost, smin, smax));
  if (adam_stamps_ && smin) TCB_CK(launch_stamp(smin + 3 * cap, ost));
  TCB_CK(cudaEventRecord(a1, ost));
  adam_.emplace_back(a0, a1);
  ++stats_.kernel_launches;
  stats_.adam_elems += n;
  *psync = SlotSync{a1, {}};
  p.nvme_valid = false;  // any NVMe replica of the parameter is now stale
  if (p.has_home) p.home_valid = false;
  if (on_gpu) p.arrival = nullptr;

  if (state_on_gpu) {
    slot_of(s).sync = SlotSync{a1, {}};
  } else {
    Slot& h = slot_of(s);
    stage_sync_[b].readers.push_back(a1);
    wait_for_read(d2h_opt_, stage_sync_[b]);
    wait_for_write(d2h_opt_, h.sync);
    TCB_CK(cudaStreamWaitEvent(d2h_opt_, a1, 0));
    if (opt_yield_ && last_d2h_) TCB_CK(cudaStreamWaitEvent(d2h_opt_, last_d2h_, 0));
    tag_ = CopyTag{"opt_store", s.id, 0, 1};
    cudaEvent_t e3 = copy(d2h_opt_, h.ptr, stg, s.bytes, false);
    h.sync = SlotSync{e3, {}};
    stage_sync_[b].readers.push_back(e3);
    stage_free_.push_back(b);
    stats_.opt_d2h_bytes += s.bytes;
  }

  if (!on_gpu) {  // updated-parameter write-back to its home tier (category iii)
    tag_ = CopyTag{"writeback", p.id, 0, static_cast<std::uint8_t>(p.tier == PTier::Nvme ? 2 : 1)};
    if (p.tier == PTier::Nvme) {
      std::uint8_t* bb = bounce_.at(p.bytes);
      SlotSync& bs = bounce_sync_[p.bytes];
      if (io_) {
        wait_for_write(d2h_opt_, bs);
        TCB_CK(cudaStreamWaitEvent(d2h_opt_, a1, 0));
        cudaEvent_t e4 = copy(d2h_opt_, bb, pout, p.bytes, false);
        psync->readers.push_back(e4);
        bs = SlotSync{e4, {}};
        nvme_write_async(p, bb, bs);
      } else {
        TCB_CK(cudaEventSynchronize(a1));
        host_wait_all(bs);
        TCB_CK(cudaMemcpy(bb, pout, p.bytes, cudaMemcpyDeviceToHost));
        bs = SlotSync{};
        nvme_write(p, bb);
      }
    } else {
      Slot& ph = slot_of(p);
      wait_for_write(d2h_opt_, ph.sync);
      TCB_CK(cudaStreamWaitEvent(d2h_opt_, a1, 0));
      cudaEvent_t e4 = copy(d2h_opt_, ph.ptr, pout, p.bytes, false);
      ph.sync = SlotSync{e4, {}};
      psync->readers.push_back(e4);
    }
    stats_.writeback_bytes += p.bytes;
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
    bool moved = false;  // any decision moving the state before its update's end
    auto t = touched.find(sid);
    if (t != touched.end())
      for (std::size_t k : t->second) moved = moved || k <= end_pos[j];
    if (moved) continue;
    at[j] = a;
  }
  return at;
}

// How many optimizer states fit through the H2D link during the forward
// pass on top of the forward's own parameter prefetches, by the machine's
// bandwidth model (machine.cpp:101-111) and the trace's compute time.
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
  const double spare = fwd_us * bw - fwd_h2d;
  if (spare <= 0 || prestage_order_.empty()) return std::min<std::size_t>(1, prestage_order_.size());
  const double sbytes = static_cast<double>(recs_[static_cast<std::size_t>(prestage_order_.front())].bytes);
  return std::max<std::size_t>(1, static_cast<std::size_t>(spare / sbytes));
}

void Executor::iteration(const StepOptions& so, cudaStream_t compute) {
  TCB_CK(cudaSetDevice(device_));
  if (compute == nullptr) {
    if (!compute_owned_) TCB_CK(cudaStreamCreateWithFlags(&compute_owned_, cudaStreamNonBlocking));
    compute = compute_owned_;
  }
  compute_ = compute;
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
  std::vector<Hook> hooks;
  if (ahead_) {  // decided (and its first states staged) at the end of the previous iteration
    hooks = std::move(*ahead_);
    ahead_.reset();
  } else {
    nvtxRangePushA("tencache.decide");
    hooks = decide_iteration();
    nvtxRangePop();
    drop_staged();
  }
  const std::vector<std::size_t> hoist = plan_hoisting(hooks);
  const std::size_t n = trace_.steps.size();
  std::vector<std::vector<std::size_t>> after(n);
  for (std::size_t j = 0; j < n; ++j)
    if (hoist[j] < n) after[hoist[j]].push_back(j);
  // Hoisted updates in execution order; their states can be staged any time
  // (no decision touches them before their update, plan_hoisting). States
  // staged by the prologue are skipped by refill_stages.
  set_prestage_order(hooks, hoist);
  // states the prologue staged come first in the order: continue after them
  while (prestage_next_ < prestage_order_.size() && staged_.count(prestage_order_[prestage_next_])) ++prestage_next_;
  if (so_.prestage) {
    // The forward refill of iteration t+1 is issued while iteration t's tail
    // may still be moving; gated, it starts only after t's last cache
    // prefetch so it never competes with t's critical H2D traffic.
    if (prestage_gate_ && last_h2d_) TCB_CK(cudaStreamWaitEvent(h2d_opt_, last_h2d_, 0));
    refill_stages(prestage_fwd_override_ >= 0 ? static_cast<std::size_t>(prestage_fwd_override_)
                                              : forward_prestage_budget(hooks));
  }
  auto mark = [&] {
    cudaEvent_t e = events_.get(true);
    TCB_CK(cudaEventRecord(e, compute));
    phase_marks_.push_back(e);
  };
  mark();
  Phase prev = Phase::Forward;
  for (const Hook& h : hooks) {
    if (h.kind == 0) {
      const TraceStep& step = trace_.steps[h.step];
      if (step.phase != prev) {
        mark();
        if (prev == Phase::Forward && so_.prestage && edge_fill_) {
          // Forward -> backward edge: the forward's cache prefetches are all
          // issued and no backward prefetch exists yet, so the H2D link
          // would idle until the first update frees a stage. Fill the rest
          // of the ring, starting when the forward's last prefetch lands.
          if (last_h2d_) TCB_CK(cudaStreamWaitEvent(h2d_opt_, last_h2d_, 0));
          refill_stages(stage_.size());
        }
        prev = step.phase;
      }
      nvtxRangePushA(step.phase == Phase::Forward ? "tencache.fwd" : step.phase == Phase::Backward ? "tencache.bwd"
                                                                                                   : "tencache.opt");
      execute(h.reqs);
      if (step.phase == Phase::OptimizerUpdate) {
        if (hoist[h.step] == n) {  // in place: waits for the state's decisions
          TensorRec& s = rec(step.tensor_ids.front());
          if (s.partner < 0) throw DeviceError(TC_EINTERNAL, "optimizer step without a paired state");
          wait_barriers(adam_stream());
          optimizer_work(s, recs_[static_cast<std::size_t>(s.partner)]);
        }
      } else {
        param_step(step, h.step, compute);
        for (std::size_t j : after[h.step]) {
          TensorRec& s = rec(trace_.steps[j].tensor_ids.front());
          optimizer_work(s, recs_[static_cast<std::size_t>(s.partner)]);
          if (so_.prestage) refill_stages(prestage_lookahead_);
        }
      }
      nvtxRangePop();
    } else {
      execute(h.reqs);
    }
  }
  mark();
  finish_iteration();
  if (lookahead_ && so_.prestage && so_.prologue) prologue_next();
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
  if (prestage_gate_ && last_h2d_) TCB_CK(cudaStreamWaitEvent(h2d_opt_, last_h2d_, 0));
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
  }
  std::erase_if(barriers_, [&](cudaEvent_t e) { return events_.done_by(e, gen); });
  if (last_h2d_ && events_.done_by(last_h2d_, gen)) last_h2d_ = nullptr;
  if (last_d2h_ && events_.done_by(last_d2h_, gen)) last_d2h_ = nullptr;
}

void Executor::drain() {
  while (!pending_.empty()) harvest_front();
  if (io_) io_->wait_all();
  TCB_CK(cudaDeviceSynchronize());
  scrub(events_.generation());
  events_.recycle_all();
}

// ZeRO-3: attach a NCCL communicator and precompute, per parameter chunk, the
// fragment list between the rank-major gathered buffer [r0 S | r1 S | ...] and
// the flat layer view (same list reversed packs the full-layer gradient for
// the reduce-scatter).
void Executor::enable_zero3(int world, int rank, const ncclUniqueId& id, const std::uint64_t* layer_elems,
                            const std::uint64_t* layer_per, std::uint32_t n_layers) {
  TCB_CK(cudaSetDevice(device_));
  auto z = std::make_unique<Zero3>();
  z->world = world;
  z->rank = rank;
  z->layer_elems.assign(layer_elems, layer_elems + n_layers);
  z->layer_per.assign(layer_per, layer_per + n_layers);
  std::map<std::uint32_t, std::vector<std::int32_t>> by_layer;
  std::uint64_t S = 0;
  for (const auto& t : trace_.tensors)
    if (t.kind == TensorKind::ParamFP16) {
      if (S != 0 && t.size_bytes != S) throw ConfigError("ZeRO-3 exchange needs uniform parameter chunks");
      S = t.size_bytes;
      if (t.layer >= n_layers) throw ConfigError("ZeRO-3 layer table shorter than the trace's layers");
      by_layer[t.layer].push_back(index_of(t.id));
    }
  z->S = S;
  std::uint64_t max_layer = 0;
  for (std::uint32_t l = 0; l < n_layers; ++l) max_layer = std::max(max_layer, 2 * layer_elems[l]);
  for (auto& [layer, idxs] : by_layer) {
    std::sort(idxs.begin(), idxs.end(), [&](std::int32_t a, std::int32_t b) { return recs_[a].id < recs_[b].id; });
    const std::uint64_t E = layer_elems[layer], per = layer_per[layer];
    if (per * static_cast<std::uint64_t>(world) < E) throw ConfigError("ZeRO-3: per * world < layer elements");
    for (std::size_t c = 0; c < idxs.size(); ++c) {
      Zero3::ChunkPlan cp;
      cp.layer = layer;
      cp.rank_bytes.assign(world, 0);
      cp.rank_view_off.assign(world, 0);
      std::vector<PackSeg> segs;
      std::uint64_t v = 0;
      for (int r = 0; r < world; ++r) {
        const std::uint64_t lo = std::min<std::uint64_t>(static_cast<std::uint64_t>(r) * per, E);
        const std::uint64_t shard = 2 * (std::min<std::uint64_t>(lo + per, E) - lo);
        const std::uint64_t start = c * S;
        if (shard <= start) continue;
        const std::uint64_t nb = std::min<std::uint64_t>(S, shard - start);
        segs.push_back(PackSeg{static_cast<std::uint64_t>(r) * S, 2 * lo + start, nb, v});
        cp.pieces.emplace_back(2 * lo + start, nb);
        cp.rank_bytes[r] = nb;
        cp.rank_view_off[r] = 2 * lo + start;
        cp.vec = cp.vec && ((2 * lo + start) % 16 == 0) && nb % 16 == 0;
        v += nb;
      }
      cp.nseg = static_cast<std::uint32_t>(segs.size());
      cp.total = v;
      if (!segs.empty()) {
        TCB_CK(cudaMalloc(&cp.segs, sizeof(PackSeg) * segs.size()));
        TCB_CK(cudaMemcpy(cp.segs, segs.data(), sizeof(PackSeg) * segs.size(), cudaMemcpyHostToDevice));
      }
      z->plans[idxs[c]] = std::move(cp);
    }
  }
  {
    std::vector<std::int32_t> order;
    for (auto& [idx, cp] : z->plans) order.push_back(idx);
    std::sort(order.begin(), order.end(), [&](std::int32_t a, std::int32_t b) { return recs_[a].id < recs_[b].id; });
    for (std::size_t k = 0; k < order.size(); ++k) z->plans[order[k]].chunk = static_cast<std::uint32_t>(k);
    if (order.size() > static_cast<std::size_t>(P2PCtl::kMaxChunks))
      throw ConfigError("ZeRO-3: more chunks than the p2p control block holds");
    z->access_epoch.assign(order.size(), 0);
  }
  TCB_CK(cudaMalloc(&z->gather, world * S));
  TCB_CK(cudaMalloc(&z->view, std::max<std::uint64_t>(max_layer, 16)));
  TCB_CK(cudaMalloc(&z->gview, std::max<std::uint64_t>(max_layer, 16)));
  TCB_CK(cudaMalloc(&z->gpad, world * S));
  TCB_CK(cudaMemset(z->gpad, 0, world * S));
  bool id_zero = true;  // an all-zero id: p2p-only exchange, no NCCL communicator
  for (char ch : id.internal) id_zero = id_zero && ch == 0;
  if (!id_zero) nccl_check(nccl().CommInitRank(&z->comm, world, id, rank), "ncclCommInitRank");
  z3_ = std::move(z);
}

// One parameter access under ZeRO-3, on the compute stream: all-gather the
// chunk from every rank, unpack into the flat layer view, checksum the view's
// pieces (the layer compute reads exactly those). Backward also produces the
// full-layer gradient of those pieces (stand-in: seeded per rank), packs it
// rank-major and reduce-scatters it (sum) into this rank's gradient chunk.
void Executor::zero3_access(TensorRec& x, bool backward, cudaStream_t cs) {
  Zero3& z = *z3_;
  const Zero3::ChunkPlan& cp = z.plans.at(index_of(x.id));
  const unsigned peers_n = static_cast<unsigned>(z.world - 1);
  if (z.p2p) {  // fused all-gather + unpack straight from the peers' HBM slots
    const std::uint32_t a = ++z.access_epoch[cp.chunk];
    Slot& sl = slot_of(x);
    TCB_CK(launch_p2p_publish(z.ctl, cp.chunk, static_cast<std::uint64_t>(sl.ptr - gpu_.base()), a, cs));
    TCB_CK(launch_p2p_gather_unpack(z.peers, cp.chunk, a, cp.rank_bytes.data(), cp.rank_view_off.data(), z.view, cs));
    stats_.kernel_launches += 2;
    // peers read the slot from now on: its next writer waits for all of them
    sl.sync.peer_cnt = &z.ctl->cnt[cp.chunk];
    sl.sync.peer_target = a * peers_n;
  } else {
    nccl_check(nccl().AllGather(where(x), z.gather, z.S, ncclUint8, z.comm, cs), "ncclAllGather");
    TCB_CK(launch_pack(cp.segs, cp.nseg, cp.total, z.gather, z.view, false, cp.vec, cs));
    stats_.kernel_launches += 1;
  }
  z.gathered_bytes += z.S * static_cast<std::uint64_t>(z.world);
  if (access_cursor_ < n_accesses_) {
    for (const auto& [off, nb] : cp.pieces) {
      TCB_CK(launch_checksum(z.view + off, nb & ~3ull, reinterpret_cast<unsigned long long*>(cks_base_ + access_cursor_),
                             cs));
      ++stats_.kernel_launches;
    }
    ++access_cursor_;
  }
  if (!backward) return;
  if (z.p2p) {  // my gradient view is refilled only after every peer pulled the previous one
    const std::uint32_t g = ++z.grad_epoch;
    if (peers_n && g > 1) stream_wait_value32(cs, &z.ctl->gcnt, (g - 1) * peers_n);
  }
  for (const auto& [off, nb] : cp.pieces) {
    TCB_CK(launch_fill_normal_bf16(reinterpret_cast<std::uint16_t*>(z.gview + off), nb / 2, 1e-3f,
                                   static_cast<std::uint64_t>(adam_step_) * 1000003ull + static_cast<std::uint64_t>(z.rank),
                                   (static_cast<std::uint64_t>(cp.layer) << 40) + off / 2, cs));
    ++stats_.kernel_launches;
  }
  if (z.p2p) {  // fused pack + reduce-scatter: pull my piece from every rank's view and sum
    TCB_CK(launch_p2p_publish_grad(z.ctl, z.grad_epoch, cs));
    TCB_CK(launch_p2p_pull_reduce(z.peers, z.grad_epoch, cp.rank_view_off[z.rank], cp.rank_bytes[z.rank], z.S,
                                  reinterpret_cast<std::uint16_t*>(x.grad), cs));
    stats_.kernel_launches += 2;
  } else {
    if (cp.total < z.S * static_cast<std::uint64_t>(z.world))  // padded chunk: padding gradient is zero
      TCB_CK(cudaMemsetAsync(z.gpad, 0, z.S * static_cast<std::uint64_t>(z.world), cs));
    TCB_CK(launch_pack(cp.segs, cp.nseg, cp.total, z.gview, z.gpad, true, cp.vec, cs));
    ++stats_.kernel_launches;
    nccl_check(nccl().ReduceScatter(z.gpad, x.grad, z.S / 2, ncclBfloat16, ncclSum, z.comm, cs),
               "ncclReduceScatter");
  }
  z.reduced_bytes += z.S * static_cast<std::uint64_t>(z.world);
  cudaEvent_t e = events_.get(false);
  TCB_CK(cudaEventRecord(e, cs));
  x.grad_ready = e;
}

// This rank's IPC handles: HBM parameter pool, control block, gradient view.
std::vector<std::uint8_t> Executor::p2p_handles() {
  if (!z3_) throw ConfigError("p2p exchange needs tc_engine_enable_zero3 first");
  Zero3& z = *z3_;
  if (!z.ctl) {
    TCB_CK(cudaMalloc(&z.ctl, sizeof(P2PCtl)));
    TCB_CK(cudaMemset(z.ctl, 0, sizeof(P2PCtl)));
  }
  std::vector<std::uint8_t> blob(3 * sizeof(cudaIpcMemHandle_t));
  cudaIpcMemHandle_t h[3];
  TCB_CK(cudaIpcGetMemHandle(&h[0], gpu_.base()));
  TCB_CK(cudaIpcGetMemHandle(&h[1], z.ctl));
  TCB_CK(cudaIpcGetMemHandle(&h[2], z.gview));
  std::memcpy(blob.data(), h, sizeof(h));
  return blob;
}

// Map every peer's pool, control block and gradient view (self: local
// pointers) and switch the exchange to the fused p2p kernels.
void Executor::enable_p2p(const std::uint8_t* all_blobs) {
  if (!z3_) throw ConfigError("p2p exchange needs tc_engine_enable_zero3 first");
  Zero3& z = *z3_;
  if (z.world > kMaxPeers) throw ConfigError("p2p exchange supports up to 8 ranks");
  if (!z.ctl) p2p_handles();
  z.peers.world = z.world;
  z.peers.rank = z.rank;
  for (int q = 0; q < z.world; ++q) {
    if (q == z.rank) {
      z.peers.pool[q] = gpu_.base();
      z.peers.ctl[q] = z.ctl;
      z.peers.gview[q] = z.gview;
      continue;
    }
    cudaIpcMemHandle_t h[3];
    std::memcpy(h, all_blobs + static_cast<std::size_t>(q) * sizeof(h), sizeof(h));
    void* ptr[3];
    for (int k = 0; k < 3; ++k) {
      TCB_CK(cudaIpcOpenMemHandle(&ptr[k], h[k], cudaIpcMemLazyEnablePeerAccess));
      z.opened.push_back(ptr[k]);
    }
    z.peers.pool[q] = static_cast<const std::uint8_t*>(ptr[0]);
    z.peers.ctl[q] = static_cast<P2PCtl*>(ptr[1]);
    z.peers.gview[q] = static_cast<const std::uint8_t*>(ptr[2]);
  }
  z.p2p = true;
}

void Executor::set_event_log(const std::string& path) {
  drain();
  if (path.empty()) {
    event_log_.reset();
    return;
  }
  event_log_ = std::make_unique<std::ofstream>(path);
  if (!*event_log_) throw DeviceError(TC_EIO, "cannot open event log " + path);
}

void Executor::sync() {
  TCB_CK(cudaSetDevice(device_));
  drain();
}

const std::vector<std::uint64_t>& Executor::access_checksums() {
  drain();
  return h_checksums_;
}

std::vector<std::uint64_t> Executor::step_result() {
  TCB_CK(cudaSetDevice(device_));
  if (!have_result_) throw DeviceError(TC_EARG, "no iteration has been run");
  const std::size_t k = static_cast<std::size_t>(result_gen_ % 2);
  TCB_CK(cudaEventSynchronize(result_ev_[k]));
  const std::uint64_t* r = h_result_ + k * std::max<std::size_t>(n_accesses_, 1);
  return std::vector<std::uint64_t>(r, r + n_accesses_);
}

void Executor::seed(std::uint64_t seed) {
  TCB_CK(cudaSetDevice(device_));
  sync();
  drop_staged();  // stages 0/1 are scratch below, and every state changes
  std::uint8_t* tmp = stage_[0];  // >= 6x the largest parameter
  for (auto& p : recs_) {
    if (p.is_state) continue;
    const std::uint64_t n = p.bytes / 2;
    std::uint8_t* dst = p.tier == PTier::Gpu ? where(p) : tmp;
    TCB_CK(launch_fill_normal_bf16(reinterpret_cast<std::uint16_t*>(dst), n, 0.02f, seed, p.id, nullptr));
    TCB_CK(launch_fill_normal_bf16(reinterpret_cast<std::uint16_t*>(p.grad), n, 1e-3f, seed + 1, p.id, nullptr));
    if (p.tier != PTier::Gpu) {
      TCB_CK(cudaDeviceSynchronize());
      if (p.tier == PTier::Nvme) {
        std::uint8_t* b = bounce_.at(p.bytes);
        TCB_CK(cudaMemcpy(b, tmp, p.bytes, cudaMemcpyDeviceToHost));
        nvme_write(p, b);
      } else {
        TCB_CK(cudaMemcpy(where(p), tmp, p.bytes, cudaMemcpyDeviceToHost));
      }
    }
    if (p.partner >= 0) {  // master copy = the bf16 value, moments zero
      TensorRec& s = recs_[static_cast<std::size_t>(p.partner)];
      std::uint8_t* pv = p.tier == PTier::Gpu ? where(p) : tmp;
      std::uint8_t* sdst = stage_[1];
      TCB_CK(launch_init_state(reinterpret_cast<const std::uint16_t*>(pv), reinterpret_cast<float*>(sdst), n, nullptr));
      TCB_CK(cudaDeviceSynchronize());
      if (s.tier == PTier::Nvme) {
        std::vector<std::uint8_t> hb(s.bytes);
        void* pin = nullptr;
        TCB_CK(cudaMallocHost(&pin, s.bytes));
        TCB_CK(cudaMemcpy(pin, sdst, s.bytes, cudaMemcpyDeviceToHost));
        nvme_write(s, pin);
        cudaFreeHost(pin);
      } else {
        TCB_CK(cudaMemcpy(where(s), sdst, s.bytes, cudaMemcpyDeviceToHost));
      }
    }
  }
  TCB_CK(cudaDeviceSynchronize());
  adam_step_ = 0;
  stats_.nvme_write_bytes = 0;
  for (auto& r : recs_) r.issued_since_access = 0;
}

void Executor::read_tensor(TensorId id, void* dst, std::uint64_t bytes) {
  TCB_CK(cudaSetDevice(device_));
  sync();
  TensorRec& r = rec(id);
  if (bytes != r.bytes) throw std::invalid_argument("read_tensor: size mismatch");
  if (r.tier == PTier::Gpu) {
    TCB_CK(cudaMemcpy(dst, where(r), bytes, cudaMemcpyDeviceToHost));
  } else if (r.tier == PTier::Nvme) {
    if (!r.nvme_valid) throw DeviceError(TC_EINTERNAL, "NVMe replica of tensor is stale");
    std::uint8_t* tmp = nullptr;  // pinned and page-aligned (O_DIRECT tiers)
    TCB_CK(cudaMallocHost(reinterpret_cast<void**>(&tmp), bytes));
    const bool ok = nvme_->io(false, tmp, bytes, r.nvme_off);
    if (ok) std::memcpy(dst, tmp, bytes);
    cudaFreeHost(tmp);
    if (!ok) throw DeviceError(TC_EIO, "read_tensor: NVMe read failed");
  } else {
    std::memcpy(dst, where(r), bytes);
  }
}

void Executor::write_tensor(TensorId id, const void* src, std::uint64_t bytes) {
  TCB_CK(cudaSetDevice(device_));
  sync();
  TensorRec& r = rec(id);
  if (bytes != r.bytes) throw std::invalid_argument("write_tensor: size mismatch");
  if (r.is_state) drop_staged();
  if (r.tier == PTier::Gpu) {
    TCB_CK(cudaMemcpy(where(r), src, bytes, cudaMemcpyHostToDevice));
    r.nvme_valid = false;
  } else if (r.tier == PTier::Nvme) {
    std::uint8_t* tmp = nullptr;
    TCB_CK(cudaMallocHost(reinterpret_cast<void**>(&tmp), bytes));
    std::memcpy(tmp, src, bytes);
    nvme_write(r, tmp);
    cudaFreeHost(tmp);
  } else {
    std::memcpy(where(r), src, bytes);
    r.nvme_valid = false;
  }
}

void* Executor::gpu_ptr(TensorId id) {
  TensorRec& r = rec(id);
  return r.tier == PTier::Gpu ? where(r) : nullptr;
}

void* Executor::grad_ptr(TensorId id) { return rec(id).grad; }

}  // namespace tcb

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

int tc_engine_iteration(tc_engine* e, const tc_step_options* so, void* compute_stream) {
  TC_GUARD({
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
    e->ex->iteration(o, static_cast<cudaStream_t>(compute_stream));
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
