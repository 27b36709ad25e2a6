// Per-GPU migration executor (see executor.hpp for the physical layout).
#include "executor.hpp"
#include "gds.hpp"

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
  if (cudaHostRegister(p, bytes, cudaHostRegisterPortable | cudaHostRegisterMapped) != cudaSuccess) {
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
      if (!regions_[r])
        TCB_CK(cudaHostAlloc(reinterpret_cast<void**>(&regions_[r]), pieces[r], cudaHostAllocPortable | cudaHostAllocMapped));
    }
  }
  std::vector<std::uint8_t*> dev_base(pieces.size(), nullptr);  // host regions: device-side alias (kernels' zero-copy)
  for (std::size_t r = 0; r < pieces.size(); ++r) {
    if (device) {
      dev_base[r] = regions_[r];
    } else {
      void* d = nullptr;
      TCB_CK(cudaHostGetDevicePointer(&d, regions_[r], 0));
      dev_base[r] = static_cast<std::uint8_t*>(d);
    }
  }
  for (std::size_t r = 0; r < pieces.size(); ++r) {
    std::uint64_t off = 0;
    for (std::size_t k = ranges[r].first; k < ranges[r].second; ++k) {
      SlotClass& c = classes_[slots[k].first];
      c.size = slots[k].first;
      Slot sl;
      sl.ptr = regions_[r] + off;
      sl.dptr = dev_base[r] + off;
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
  std::set<TensorId> in_nvme, to_gpu;
  std::map<std::pair<int, std::uint64_t>, std::uint32_t> need = simulate_occupancy(&fwd_h2d, &in_nvme, &to_gpu);
  {  // NVMe lookahead window: only when optimizer states live in the NVMe tier
    bool states_in_nvme = false;
    for (const auto& r : recs_) states_in_nvme = states_in_nvme || (r.is_state && in_nvme.count(r.id));
    const char* na = std::getenv("TC_NVME_AHEAD");
    nvme_ahead_ = states_in_nvme ? (na ? static_cast<std::size_t>(std::max(0, std::atoi(na))) : 16) : 0;
  }
  lap("occupancy dry run");
  {  // split-master eligibility (TensorRec::split_ok)
    const char* fm = std::getenv("TC_FULL_MASTER");
    const bool full_master = opts.full_master != 0 || (fm && std::atoi(fm) != 0);
    for (auto& s : recs_) {
      if (!s.is_state || s.partner < 0 || full_master) continue;
      const TensorRec& p = recs_[static_cast<std::size_t>(s.partner)];
      s.split_ok = !in_nvme.count(p.id) && policy_->initial_tier(s.id).value_or(Tier::Cpu) != Tier::Gpu &&
                   !to_gpu.count(s.id) && (p.bytes / 2) % kSplitTile == 0;
    }
  }
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
    host_opt_.plan(size, need[{2, size}] + hspare + 1 + nvme_ahead_);  // +1 transient, + NVMe lookahead
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
    // 32 files x 32 I/O threads: C4 648 vs 660 ms/step with 16 x 16, two interleaved repeats
    // (profiles/r02_c4_hoist_readahead.json)
    const char* nf = std::getenv("TC_NVME_FILES");
    nvme_ = std::make_unique<StripedFile>(dir, off, nf ? std::atoi(nf) : 32, opts.direct_io && all_aligned);
  }
  if (const char* c = std::getenv("TC_PRESTAGE_FWD")) prestage_fwd_override_ = std::atoi(c);
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

  // GPUDirect Storage for the NVMe tier when O_DIRECT was asked for and the
  // nvidia-fs driver is present (never probed otherwise: gds.hpp)
  gds_ = io_ != nullptr && nvme_->direct() && Gds::available();
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
  if (const char* c = std::getenv("TC_ADAM_BATCH"))
    adam_batch_env_ = static_cast<std::size_t>(std::clamp(std::atoi(c), 1, kMaxAdamChunks));
  for (const auto& [size, _] : pclass) {
    for (std::size_t i = 0; i < std::max<std::size_t>({2, adam_batch_env_, kAdamBatchConcurrent}); ++i) {
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
  TCB_CK(cudaStreamCreateWithPriority(&opt_, cudaStreamNonBlocking, hi_prio));
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
  TCB_CK(cudaMalloc(&codec_flag_, sizeof(unsigned)));
}

Executor::~Executor() {
  if (adam_stamps_ && stamps_)
    std::fprintf(stderr, "[tencache] AdamW launches: %.0f: stream reaches it -> first CTA %.2f us, "
                 "last CTA end -> next op %.2f us (avg)\n",
                 static_cast<double>(stamps_), stamp_pre_ns_ / stamps_ * 1e-3, stamp_post_ns_ / stamps_ * 1e-3);
  cudaSetDevice(device_);
  try {
    iteration_abort();
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
  if (codec_flag_) cudaFree(codec_flag_);
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
    if (z3_->peers.scratch) cudaFree(z3_->peers.scratch);
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
std::map<std::pair<int, std::uint64_t>, std::uint32_t> Executor::simulate_occupancy(double* fwd_h2d,
                                                                                    std::set<TensorId>* in_nvme,
                                                                                    std::set<TensorId>* to_gpu) const {
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
    if (in_nvme && tier == Tier::Nvme) in_nvme->insert(t.id);
    add(t.id, tier, +1);
  }
  auto apply_reqs = [&](const std::vector<TransferRequest>& reqs) {
    for (const TransferRequest& r : reqs) {
      if (in_nvme && r.dst == Tier::Nvme) in_nvme->insert(r.tensor_id);
      if (to_gpu && r.dst == Tier::Gpu) to_gpu->insert(r.tensor_id);
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
// ~118 on C5 (profiles/r01_stage_sweep.json). Without forward prefetches the
// forward's time is taken 2x the model's (it runs longer under load — at
// 1.5x the C3 H2D link still idled ~35 ms per step before the backward freed
// a stage, profiles/r02_timeline_c3.json — and the prologue then fills the
// ring: forward_prestage_budget).
int Executor::auto_stage_slots(double fwd_h2d) const {
  double fwd_us = 0, sbytes = 0, alloc = 0;
  std::size_t nstates = 0;
  for (const TraceStep& st : trace_.steps)
    if (st.phase == Phase::Forward) fwd_us += st.compute_us * cfg_.batch_scale;
  for (const auto& r : recs_)
    if (r.is_state) {  // bytes a load moves (split-master prefix where eligible)
      sbytes = std::max(sbytes, static_cast<double>(r.split_ok ? packed_layout(r.bytes / 12).bytes : r.bytes));
      alloc = std::max(alloc, static_cast<double>(r.bytes));
      ++nstates;
    }
  if (nstates == 0 || sbytes == 0) return 12;
  double bw = 0;
  try {
    bw = to_double(machine_.effective_bandwidth(Tier::Cpu, Tier::Gpu)) * 1e3;  // bytes per us
  } catch (...) {
    return 12;
  }
  const double spare = std::max(0.0, (fwd_h2d == 0 ? 2.0 : 1.0) * fwd_us * bw - fwd_h2d);
  std::size_t n = static_cast<std::size_t>(spare / sbytes) + 4;
  std::size_t free_b = 0, total_b = 0;
  if (cudaMemGetInfo(&free_b, &total_b) == cudaSuccess)
    n = std::min<std::size_t>(n, static_cast<std::size_t>(0.5 * static_cast<double>(free_b) / alloc));
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
std::uint64_t Executor::nvme_read_async(TensorRec& r, void* dst, SlotSync& target, bool device) {
  std::vector<cudaEvent_t> waits(target.readers.begin(), target.readers.end());
  if (target.writer) waits.push_back(target.writer);
  // after: the buffer's previous job and the extent's previous job (a pending
  // write of the same tensor must land before it is read back)
  std::vector<std::uint64_t> after{target.io_read, target.io_write, r.nvme_job};
  const std::uint64_t pn = r.is_state && r.split ? r.bytes / 12 : 0;  // packed: what the last write moved
  const std::uint64_t k = device ? io_->submit_read_device(dst, r.bytes, r.nvme_off, io_deps(std::move(waits)), after)
                                 : io_->submit_read(dst, r.bytes, r.nvme_off, io_deps(std::move(waits)), after, pn);
  r.nvme_job = k;
  target = SlotSync{};
  target.io_write = k;
  stats_.nvme_read_bytes += r.bytes;
  return k;
}

// host buffer -> NVMe once the copy that filled `source` is done; later writers
// of the buffer wait on source.io_read.
std::uint64_t Executor::nvme_write_async(TensorRec& r, const void* src, SlotSync& source, bool device) {
  std::vector<cudaEvent_t> waits;
  if (source.writer) waits.push_back(source.writer);
  // the buffer's previous reader too: source.io_read must keep naming a job
  // whose completion implies every earlier read of the buffer finished
  std::vector<std::uint64_t> after{source.io_write, source.io_read, r.nvme_job};
  const std::uint64_t pn = r.is_state && r.split ? r.bytes / 12 : 0;  // packed: prefix (+ overflow area)
  const std::uint64_t k = device ? io_->submit_write_device(src, r.bytes, r.nvme_off, io_deps(std::move(waits)), after)
                                 : io_->submit_write(src, r.bytes, r.nvme_off, io_deps(std::move(waits)), after, pn);
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
  if (io_) io_->forget_extent(r.nvme_off);  // the whole slot lands outside the queue
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
  if (r.tier == PTier::Gpu && gds_) {  // HBM -> file directly (GPUDirect Storage)
    Slot& g = slot_of(r);
    nvme_write_async(r, g.ptr, g.sync, true);
  } else if (r.tier == PTier::Gpu) {
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
  const std::int32_t xi = index_of(r.tensor_id);
  if (r.src == Tier::Nvme && early_.count(xi)) return true;  // its slot is already taken (read ahead)
  const TensorRec& x = recs_[static_cast<std::size_t>(xi)];
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
  } else if (r.src == Tier::Nvme && r.dst == Tier::Gpu && gds_) {  // GPUDirect Storage: file -> HBM, one leg
    const std::uint32_t gs = take_slot(PTier::Gpu, x.bytes, xi);
    Slot& g = gpu_.cls(x.bytes).slots[gs];
    const std::uint64_t k = nvme_read_async(x, g.ptr, g.sync, true);
    io_->stream_wait(h2d_, k);
    done = events_.get(true);
    TCB_CK(cudaEventRecord(done, h2d_));
    g.sync = SlotSync{done, {}};
    if (!r.src_retains) x.nvme_valid = false;
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
  } else if (r.src == Tier::Nvme && r.dst == Tier::Cpu && early_.count(xi)) {  // read ahead: bind its slot
    x.slot = early_.at(xi).slot;
    early_.erase(xi);
    if (!r.src_retains) x.nvme_valid = false;
    x.tier = host_tier(x);
    refill_early();
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
}

void Executor::wait_barriers(cudaStream_t cs) {
  for (cudaEvent_t e : barriers_) TCB_CK(cudaStreamWaitEvent(cs, e, 0));
  barriers_.clear();
  if (barrier_io_ && io_) io_->stream_wait_upto(cs, barrier_io_);
  barrier_io_ = 0;
}

void Executor::set_event_log(const std::string& path) {
  sync();
  if (path.empty()) {
    event_log_.reset();
    return;
  }
  event_log_ = std::make_unique<std::ofstream>(path);
  if (!*event_log_) throw DeviceError(TC_EIO, "cannot open event log " + path);
}

void Executor::sync() {
  TCB_CK(cudaSetDevice(device_));
  if (open_) throw DeviceError(TC_EARG, "an iteration is open: finish it with iteration_end (or abort it) first");
  drain();
}

const std::vector<std::uint64_t>& Executor::access_checksums() {
  sync();
  return h_checksums_;
}

std::vector<std::uint64_t> Executor::step_result() {
  TCB_CK(cudaSetDevice(device_));
  if (!have_result_) throw DeviceError(TC_EARG, "no iteration has been run");
  const std::size_t k = static_cast<std::size_t>(result_gen_ % 2);
  TCB_CK(cudaEventSynchronize(result_ev_[k]));
  if (io_) io_->check();  // the result may have consumed bytes of a failed NVMe job
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
      s.split = s.split_ok;
      if (s.split)  // master = float(param): low halves, round bits, moments, codes, flags all zero
        TCB_CK(cudaMemset(sdst, 0, s.bytes));
      else
        TCB_CK(launch_init_state(reinterpret_cast<const std::uint16_t*>(pv), reinterpret_cast<float*>(sdst), n, nullptr));
      TCB_CK(cudaDeviceSynchronize());
      if (s.tier == PTier::Nvme) {
        std::vector<std::uint8_t> hb(s.bytes);
        void* pin = nullptr;
        TCB_CK(cudaMallocHost(&pin, s.bytes));
        TCB_CK(cudaMemcpy(pin, sdst, s.bytes, cudaMemcpyDeviceToHost));
        nvme_write(s, pin);
        cudaFreeHost(pin);
      } else if (s.tier == PTier::Gpu) {
        TCB_CK(cudaMemcpy(where(s), sdst, s.bytes, cudaMemcpyDeviceToDevice));
      } else {
        TCB_CK(cudaMemcpy(where(s), sdst, state_xfer_bytes(s), cudaMemcpyDeviceToHost));
      }
    }
  }
  TCB_CK(cudaDeviceSynchronize());
  adam_step_ = 0;
  stats_.nvme_write_bytes = 0;
  for (auto& r : recs_) r.issued_since_access = 0;
}

// A tensor's stored bytes from / to wherever it lives (states: as stored,
// split or full).
void Executor::load_state_host(TensorRec& r, void* dst) {
  if (r.tier == PTier::Gpu) {
    TCB_CK(cudaMemcpy(dst, where(r), r.bytes, cudaMemcpyDeviceToHost));
  } else if (r.tier == PTier::Nvme) {
    if (!r.nvme_valid) throw DeviceError(TC_EINTERNAL, "NVMe replica of tensor is stale");
    std::uint8_t* tmp = nullptr;  // pinned and page-aligned (O_DIRECT tiers)
    TCB_CK(cudaMallocHost(reinterpret_cast<void**>(&tmp), r.bytes));
    const bool ok = nvme_->io(false, tmp, r.bytes, r.nvme_off);
    if (ok) std::memcpy(dst, tmp, r.bytes);
    cudaFreeHost(tmp);
    if (!ok) throw DeviceError(TC_EIO, "read_tensor: NVMe read failed");
  } else {
    std::memcpy(dst, where(r), r.bytes);
  }
}

void Executor::store_state_host(TensorRec& r, const void* src) {
  if (r.tier == PTier::Gpu) {
    TCB_CK(cudaMemcpy(where(r), src, r.bytes, cudaMemcpyHostToDevice));
    r.nvme_valid = false;
  } else if (r.tier == PTier::Nvme) {
    std::uint8_t* tmp = nullptr;
    TCB_CK(cudaMallocHost(reinterpret_cast<void**>(&tmp), r.bytes));
    std::memcpy(tmp, src, r.bytes);
    nvme_write(r, tmp);
    cudaFreeHost(tmp);
  } else {
    std::memcpy(where(r), src, r.bytes);
    r.nvme_valid = false;
  }
}

// Split state -> full [p32|m|v] layout, on the GPU (stages 0/1 as scratch;
// the caller has synced). The master's high half is the partner's bf16 value.
void Executor::state_to_full(TensorRec& s, const void* stored_host, void* full_host) {
  TensorRec& p = recs_[static_cast<std::size_t>(s.partner)];
  drop_staged();
  const std::uint16_t* B = param_bits_dev(p);
  TCB_CK(cudaMemcpy(stage_[0], stored_host, s.bytes, cudaMemcpyHostToDevice));  // prefix + overflow area
  TCB_CK(launch_state_expand(stage_[0], B, reinterpret_cast<float*>(stage_[1]), p.bytes / 2, nullptr));
  TCB_CK(cudaMemcpy(full_host, stage_[1], s.bytes, cudaMemcpyDeviceToHost));
}

// Full layout -> packed split (prefix + overflow area), on the GPU, into
// stage 1; false when some master does not round to the parameter's bf16
// value (not representable split).
bool Executor::state_from_full(TensorRec& s, const void* full_host, std::uint8_t* stored_dev) {
  TensorRec& p = recs_[static_cast<std::size_t>(s.partner)];
  drop_staged();
  const std::uint16_t* B = param_bits_dev(p);
  TCB_CK(cudaMemcpy(stage_[0], full_host, s.bytes, cudaMemcpyHostToDevice));
  TCB_CK(cudaMemset(codec_flag_, 0, sizeof(unsigned)));
  TCB_CK(launch_state_compress(reinterpret_cast<const float*>(stage_[0]), B, stored_dev, p.bytes / 2, codec_flag_,
                               nullptr));
  unsigned flag = 1;
  TCB_CK(cudaMemcpy(&flag, codec_flag_, sizeof(unsigned), cudaMemcpyDeviceToHost));
  return flag == 0;
}

// The parameter's current bf16 bytes in HBM: its GPU slot, else a copy in its
// first update scratch buffer (callers have synced: nothing uses it).
const std::uint16_t* Executor::param_bits_dev(TensorRec& p) {
  if (p.tier == PTier::Gpu) return reinterpret_cast<const std::uint16_t*>(where(p));
  std::vector<std::uint8_t> hb(p.bytes);
  load_state_host(p, hb.data());
  std::uint8_t* d = pout_scratch_.at(p.bytes).front();
  TCB_CK(cudaMemcpy(d, hb.data(), p.bytes, cudaMemcpyHostToDevice));
  return reinterpret_cast<const std::uint16_t*>(d);
}

// Back to the full layout in place (its parameter is about to change).
void Executor::unsplit(TensorRec& s) {
  if (!s.split) return;
  std::vector<std::uint8_t> stored(s.bytes), full(s.bytes);
  load_state_host(s, stored.data());
  state_to_full(s, stored.data(), full.data());
  s.split = false;
  store_state_host(s, full.data());
}

void Executor::read_tensor(TensorId id, void* dst, std::uint64_t bytes) {
  TCB_CK(cudaSetDevice(device_));
  sync();
  TensorRec& r = rec(id);
  if (bytes != r.bytes) throw std::invalid_argument("read_tensor: size mismatch");
  if (r.is_state && r.split) {
    std::vector<std::uint8_t> stored(r.bytes);
    load_state_host(r, stored.data());
    state_to_full(r, stored.data(), dst);
  } else {
    load_state_host(r, dst);
  }
}

void Executor::write_tensor(TensorId id, const void* src, std::uint64_t bytes) {
  TCB_CK(cudaSetDevice(device_));
  sync();
  TensorRec& r = rec(id);
  if (bytes != r.bytes) throw std::invalid_argument("write_tensor: size mismatch");
  if (r.is_state) drop_staged();
  if (!r.is_state && r.partner >= 0) unsplit(recs_[static_cast<std::size_t>(r.partner)]);  // its high halves change
  if (r.is_state && r.split_ok) {
    if (state_from_full(r, src, stage_[1])) {
      std::vector<std::uint8_t> stored(r.bytes, 0);
      TCB_CK(cudaMemcpy(stored.data(), stage_[1], r.bytes, cudaMemcpyDeviceToHost));  // prefix + overflow area
      r.split = true;
      store_state_host(r, stored.data());
      return;
    }
    r.split = false;
  }
  store_state_host(r, src);
}

void* Executor::gpu_ptr(TensorId id) {
  TensorRec& r = rec(id);
  return r.tier == PTier::Gpu ? where(r) : nullptr;
}

void* Executor::grad_ptr(TensorId id) { return rec(id).grad; }

void Executor::regions(void** pool, std::uint64_t* pool_bytes, void** grads, std::uint64_t* grad_bytes) {
  *pool = gpu_.base();
  *pool_bytes = gpu_.bytes();
  *grads = grads_;
  std::uint64_t g = 0;
  for (const auto& r : recs_)
    if (!r.is_state) g += r.bytes;
  *grad_bytes = g;
}

}  // namespace tcb
