// Per-GPU migration executor: replays the TenCache policy's TransferRequests
// (scheduler.hpp:20-33) as real data movement on a B200.
//
// Physical layout (one set per GPU):
//   * HBM parameter pool   — one cudaMalloc region carved into size classes
//                            exactly like the policy's GPU BufferPool
//                            (bufpool.cpp:47-66), plus `spare` slots/class;
//   * pinned host pools    — parameter cache and optimizer-state cache, each
//                            one cudaHostAlloc region carved the same way;
//   * NVMe tier            — one sparse file, a fixed 4 KiB-aligned extent per
//                            tensor, reached through per-class pinned bounce
//                            buffers (the staging slot of engine.cpp:214-221);
//   * HBM optimizer stages — a ring of state-chunk buffers for the
//                            H2D -> fused AdamW -> D2H pipeline;
//   * HBM gradients        — one bf16 buffer per parameter (ZeRO-3 keeps the
//                            reduce-scattered shard on GPU for GPU Adam).
// Logical buffer ids of the policy stay logical: physical
// slots are chosen from per-class FIFO free lists, so an evict+prefetch pair
// lands in slots freed a step earlier and both copy directions run at once.
// Hazards are tracked per physical slot with CUDA events (last writer + the
// readers since), never by stream-wide synchronisation.
#pragma once

#include <cstdint>
#include <deque>
#include <map>
#include <memory>
#include <optional>
#include <set>
#include <string>
#include <fstream>
#include <unordered_map>
#include <vector>

#include <cuda_runtime.h>

#include "capi_common.hpp"
#include "compute_standin.hpp"
#include "dataplane.cuh"
#include "nccl_dyn.hpp"
#include "nvme_io.hpp"
#include "tencache/tencache.hpp"
#include "tencache_c.h"

namespace tcb {

void cuda_check(cudaError_t e, const char* what);
#define TCB_CK(x) ::tcb::cuda_check((x), #x)

// Events are tagged with the iteration (generation) that recorded them and
// recycled only once that iteration's fences have completed, after every slot
// reference to them has been scrubbed — a recorded event is never re-recorded
// underneath a waiter.
class EventArena {
 public:
  ~EventArena();
  cudaEvent_t get(bool timing = false);
  std::uint64_t generation() const { return gen_; }
  void next_generation() { ++gen_; }
  bool done_by(cudaEvent_t e, std::uint64_t gen) const;  // recorded in a generation <= gen
  void recycle_upto(std::uint64_t gen);
  void recycle_all();

 private:
  struct Used {
    cudaEvent_t e;
    bool timed;
    std::uint64_t gen;
  };
  std::vector<cudaEvent_t> free_, free_timed_;
  std::deque<Used> used_;
  std::unordered_map<cudaEvent_t, std::uint64_t> gen_of_;
  std::uint64_t gen_ = 0;
};

struct SlotSync {
  cudaEvent_t writer = nullptr;         // last op that wrote the slot
  std::vector<cudaEvent_t> readers;     // ops that read it since
  std::uint64_t io_write = 0;           // NVMe job that filled it (host buffers)
  std::uint64_t io_read = 0;            // NVMe job that last read it
  const unsigned* peer_cnt = nullptr;   // ZeRO-3 p2p: peers' reads of the occupant (device word)
  unsigned peer_target = 0;             // ... writers wait until *peer_cnt >= peer_target
};

enum class PTier : std::uint8_t { Gpu, HostParam, HostOpt, Nvme };

struct Slot {
  std::uint8_t* ptr = nullptr;
  std::uint8_t* dptr = nullptr;  // the same bytes as seen by kernels (host slots: mapped pinned memory)
  SlotSync sync;
  std::int32_t occupant = -1;  // tensor index
};

struct SlotClass {
  std::uint64_t size = 0;
  std::vector<Slot> slots;
  std::deque<std::uint32_t> free_fifo;
};

class SlotPool {
 public:
  void plan(std::uint64_t size, std::uint32_t count) { want_[size] += count; }
  void allocate(bool device, int dev);
  void release_memory();
  SlotClass& cls(std::uint64_t size);
  bool has_free(std::uint64_t size) const;
  std::uint64_t bytes() const { return bytes_; }
  std::map<std::uint64_t, SlotClass>& classes() { return classes_; }
  std::uint8_t* base() const { return regions_.empty() ? nullptr : regions_.front(); }  // device pools: one region

 private:
  std::map<std::uint64_t, std::uint32_t> want_;
  std::map<std::uint64_t, SlotClass> classes_;
  std::vector<std::uint8_t*> regions_;  // contiguous carving, split into <= kRegion pieces for pinning
  std::vector<std::uint64_t> mapped_;   // host regions: mmap length (0: cudaHostAlloc fallback)
  bool device_ = false;
  std::uint64_t bytes_ = 0;
};

struct TensorRec {
  tencache::TensorId id = 0;
  std::uint64_t bytes = 0;
  bool is_state = false;
  std::int32_t partner = -1;       // state <-> param index
  PTier tier = PTier::Nvme;
  std::uint32_t slot = 0;          // physical slot index within its class
  std::uint64_t nvme_off = 0;
  bool nvme_valid = false;         // NVMe extent holds the current bytes
  std::uint64_t nvme_job = 0;      // last async job on its NVMe extent (file-side ordering)
  std::uint8_t* grad = nullptr;    // params: bf16 gradient in HBM
  int issued_since_access = 0;     // P7b hit definition
  cudaEvent_t arrival = nullptr;   // last H2D into its GPU slot (for on-time)
  cudaEvent_t grad_ready = nullptr;  // producer of its gradient (ZeRO-3 reduce-scatter, or the caller's backward step)
  cudaEvent_t grad_reader = nullptr; // last fused AdamW that read its gradient
  // A retained home copy (comparison policies fetch with src_retains and drop
  // instantly): the host slot stays allocated while the GPU copy is primary.
  bool has_home = false, home_valid = false;
  PTier home_tier = PTier::HostParam;
  std::uint32_t home_slot = 0;
  // States: held split on the host (dataplane.cuh PackedLayout: the master's
  // high half is the partner parameter's bf16 value, which only the update
  // writes; the moments' exponents coded per 32-element group). split_ok (dry run of the policy's decisions): the partner never
  // lives in NVMe (its bytes are in HBM or pinned memory at every update),
  // the state never moves into HBM, and the chunk is whole AdamW tiles.
  bool split = false, split_ok = false;
};

// ZeRO-3 exchange state of one rank. Chunk c of layer L holds
// bytes [c*S, (c+1)*S) of this rank's shard of the layer's flat parameters;
// rank r's shard starts at byte 2*r*per_L of the flat layer.
struct Zero3 {
  int world = 1, rank = 0;
  ncclComm_t comm = nullptr;
  std::uint64_t S = 0;
  std::vector<std::uint64_t> layer_elems, layer_per;
  struct ChunkPlan {
    PackSeg* segs = nullptr;  // gathered (rank-major, r*S) <-> flat layer view
    std::uint32_t nseg = 0;
    std::uint64_t total = 0;
    bool vec = true;
    std::vector<std::pair<std::uint64_t, std::uint64_t>> pieces;  // (view offset, bytes)
    std::vector<std::uint64_t> rank_bytes, rank_view_off;          // per rank (zero-byte ranks included)
    std::uint32_t layer = 0;
    std::uint32_t chunk = 0;                                       // dense chunk index (p2p control block)
  };
  std::unordered_map<std::int32_t, ChunkPlan> plans;  // by parameter rec index
  std::uint8_t* gather = nullptr;  // world * S
  std::uint8_t* view = nullptr;    // flat parameters of the largest layer
  std::uint8_t* gview = nullptr;   // full-layer gradient of the current chunk's pieces
  std::uint8_t* gpad = nullptr;    // world * S rank-major padded gradient (padding zero)
  std::uint64_t gathered_bytes = 0, reduced_bytes = 0;
  // p2p fused exchange (no NCCL): peer table over CUDA IPC mappings
  bool p2p = false;
  PeerTable peers{};
  P2PCtl* ctl = nullptr;
  std::vector<void*> opened;               // IPC mappings to close
  std::vector<std::uint32_t> access_epoch;  // per chunk
  std::uint32_t grad_epoch = 0;
  std::int64_t open_layer = -1;  // layer in the views during a caller-computed step
};

struct StepOptions {
  double lr = 1e-4, beta1 = 0.9, beta2 = 0.999, eps = 1e-8, weight_decay = 0.01;
  float grad_scale = 1.0f;
  int compute_mode = 0;
  int spin_ctas = 1;
  bool hoist_optimizer = true;  // run each update right after its parameter's last fwd/bwd access
  bool prestage = true;         // stage optimizer states into HBM ahead of their updates
  bool prologue = true;         // enqueue the next iteration's decisions + first state loads at the end
};

class Executor {
 public:
  Executor(const std::string& trace_path, const std::string& machine_path, const std::string& cfg_json,
           const tc_engine_options& opts);
  ~Executor();

  void seed(std::uint64_t seed);
  void iteration(const StepOptions& so, cudaStream_t compute);
  // per-step execution (tc_engine_iteration_begin / step_begin / step_end / iteration_end)
  void iteration_begin(const StepOptions& so, cudaStream_t compute, bool external);
  std::vector<void*> step_begin(std::size_t i);
  void step_end(std::size_t i);
  void iteration_end();
  void iteration_abort();
  bool iteration_open() const { return open_.has_value(); }
  void sync();
  void read_tensor(tencache::TensorId id, void* dst, std::uint64_t bytes);
  void write_tensor(tencache::TensorId id, const void* src, std::uint64_t bytes);
  void* gpu_ptr(tencache::TensorId id);
  void* grad_ptr(tencache::TensorId id);
  void regions(void** pool, std::uint64_t* pool_bytes, void** grads, std::uint64_t* grad_bytes);
  // ZeRO-3, inside a caller-computed step: the gathered layer and its gradient view
  void zero3_views(void** params, void** grads, std::uint64_t* layer_bytes);
  std::uint64_t tensor_bytes(tencache::TensorId id) { return rec(id).bytes; }
  void enable_zero3(int world, int rank, const ncclUniqueId& id, const std::uint64_t* layer_elems,
                    const std::uint64_t* layer_per, std::uint32_t n_layers);
  std::uint64_t exchanged_bytes() const { return z3_ ? z3_->gathered_bytes + z3_->reduced_bytes : 0; }
  std::vector<std::uint8_t> p2p_handles();
  void enable_p2p(const std::uint8_t* all_blobs);
  tc_engine_stats stats() const { return stats_; }
  void reset_stats() { stats_ = tc_engine_stats{}; }
  const std::vector<std::uint64_t>& access_checksums();
  // The last enqueued iteration's per-access checksums; waits only for its
  // compute stream (forward/backward), not its optimizer write-back tail.
  std::vector<std::uint64_t> step_result();
  std::size_t n_accesses() const { return n_accesses_; }
  const std::vector<double>& phase_ms() const { return phase_ms_; }
  const tencache::IPolicy& policy() const { return *policy_; }

 private:
  using Req = tencache::TransferRequest;
  struct CopyTag {  // what a copy is, for the measured event log
    const char* kind = "";
    tencache::TensorId tensor = 0;
    std::uint8_t src = 0, dst = 0;
  };
  struct Copy {
    cudaEvent_t start = nullptr, end = nullptr;
    bool h2d = true;
    std::uint64_t bytes = 0;
    CopyTag tag;
  };
  struct Stall {
    cudaEvent_t reach = nullptr, go = nullptr;
    tencache::TensorId tensor = 0;
  };
  CopyTag tag_;

  TensorRec& rec(tencache::TensorId id);
  std::int32_t index_of(tencache::TensorId id) const;
  SlotPool& pool(PTier t);
  PTier host_tier(const TensorRec& r) const { return r.is_state ? PTier::HostOpt : PTier::HostParam; }
  Slot& slot_of(const TensorRec& r);
  std::uint8_t* where(const TensorRec& r);

  // request execution
  void execute(std::vector<Req> reqs);
  bool dest_available(const Req& r) const;
  void apply(const Req& r);
  std::uint32_t take_slot(PTier t, std::uint64_t size, std::int32_t occupant);
  void free_slot(PTier t, std::uint64_t size, std::uint32_t s);
  void wait_for_write(cudaStream_t s, const SlotSync& y);
  void wait_for_read(cudaStream_t s, const SlotSync& y);
  void host_wait_all(const SlotSync& y);
  cudaEvent_t copy(cudaStream_t s, void* dst, const void* src, std::uint64_t n, bool h2d);
  void nvme_read(const TensorRec& r, void* dst);
  void nvme_write(TensorRec& r, const void* src);
  void ensure_nvme_fresh(TensorRec& r);

  // compute
  struct Hook {
    int kind;           // 0 begin, 1 end, 2 restore point, 3 iteration end
    std::size_t step;   // trace step (begin/end)
    std::vector<Req> reqs;
  };
  std::vector<Hook> decide_iteration();
  std::vector<std::size_t> plan_hoisting(const std::vector<Hook>& hooks);
  void param_enter(const tencache::TraceStep& step, cudaStream_t cs, bool external);
  void param_compute(const tencache::TraceStep& step, cudaStream_t cs);
  void param_exit(const tencache::TraceStep& step, cudaStream_t cs, bool external);
  void mark_phase();
  struct OpenIter {  // the iteration between iteration_begin and iteration_end
    std::vector<Hook> hooks;
    std::vector<std::size_t> hoist;
    std::vector<std::vector<std::size_t>> after;  // hoisted updates run after each step
    std::size_t hk = 0;    // next hook
    std::size_t next = 0;  // next step to begin
    bool in_step = false;
    bool external = false;  // the caller computes between step_begin and step_end
    tencache::Phase prev = tencache::Phase::Forward;
  };
  std::optional<OpenIter> open_;
  void zero3_access(TensorRec& x, bool backward, cudaStream_t cs);
  void zero3_gather(TensorRec& x, cudaStream_t cs);
  void zero3_grad_fence(cudaStream_t cs);
  void zero3_reduce(TensorRec& x, cudaStream_t cs, bool stand_in);
  void optimizer_work(TensorRec& s, TensorRec& p);
  struct UpdateJob {
    TensorRec* s = nullptr;
    TensorRec* p = nullptr;
    bool state_on_gpu = false, on_gpu = false;
    std::uint64_t n = 0;
    std::uint8_t* stg = nullptr;  // [p32 | m | v] in HBM (stage or GPU slot)
    std::size_t b = 0;            // stage index (host-resident states)
    std::uint8_t* pout = nullptr;  // bf16 result (the parameter's GPU slot or a scratch buffer)
    SlotSync* psync = nullptr;
    bool split = false;            // stg holds the PackedLayout prefix; pout is also the master's high half
    std::uint8_t* ovf = nullptr;   // split: the overflow area (tail of the state's pinned slot, mapped)
  };
  // bytes of a host-resident state that cross PCIe (its packed prefix or all of it)
  std::uint64_t state_xfer_bytes(const TensorRec& s) const {
    return s.split ? packed_layout(s.bytes / 12).bytes : s.bytes;
  }
  // state bytes as stored (split or full) <-> the full [p32|m|v] layout, on the GPU
  void state_to_full(TensorRec& s, const void* stored_host, void* full_host);
  const std::uint16_t* param_bits_dev(TensorRec& p);  // the parameter's bf16 bytes in HBM (synchronous)
  bool state_from_full(TensorRec& s, const void* full_host, std::uint8_t* stored_dev);
  void unsplit(TensorRec& s);
  void load_state_host(TensorRec& s, void* host_dst);          // the state's stored bytes, any host tier
  void store_state_host(TensorRec& s, const void* host_src);   // ... written back
  unsigned* codec_flag_ = nullptr;  // device word: compress mismatch
  UpdateJob prepare_update(TensorRec& s, TensorRec& p);
  void run_updates(std::vector<UpdateJob>& jobs);
  void finish_update(UpdateJob& j, cudaEvent_t a1);
  void defer_update(TensorRec& s, TensorRec& p);
  void flush_updates();
  void flush_if_touched(const std::vector<Req>& reqs);
  std::vector<std::pair<std::int32_t, std::int32_t>> deferred_;  // hoisted updates waiting for a batch
  // Hoisted updates per fused AdamW launch: 8 on either stream (one launch's
  // front-end latency and ramp instead of 8). On its own stream (compute-
  // bound traces, ZeRO-3 at world > 1) each launch waits for SMs behind the
  // concurrent layer compute (C3, packed states: event-timed 0.34 / 0.42 /
  // 0.49 / 0.54 of the HBM peak at 1 / 2 / 4 / 8, step time unchanged,
  // profiles/r02_adam_batch_packed.json); on the compute stream (migration-
  // bound traces, world-1 ZeRO-3) C3 0.44 -> 0.59, C5 0.49 -> 0.65, C2 0.49 ->
  // 0.56 with steps within 0.5 % (profiles/r02_adam_placement_c3.json,
  // r02_adam_batch_compute.json). TC_ADAM_BATCH overrides (1..8).
  static constexpr std::size_t kAdamBatchConcurrent = 8;
  std::size_t adam_batch_env_ = 0;
  std::size_t adam_batch() const { return adam_batch_env_ ? adam_batch_env_ : kAdamBatchConcurrent; }
  std::size_t stage_state(TensorRec& s);
  void refill_stages(std::size_t want_staged);
  // NVMe lookahead: the iteration's NVMe -> pinned fetches of optimizer states
  // (the +Opt rotation, scheduler.cpp:320-370) are known when it is decided;
  // up to nvme_ahead_ of them are read into spare pinned slots early, and the
  // decision's fetch then binds the slot instead of starting the read. The
  // state's NVMe bytes cannot change in between (only its fetch moves it), and
  // the read is ordered after the extent's last write (nvme_read_async).
  struct EarlyFetch {
    std::uint32_t slot = 0;  // physical slot in the state's pinned class
  };
  std::unordered_map<std::int32_t, EarlyFetch> early_;
  std::vector<std::int32_t> early_order_;  // state fetches NVMe -> CPU in decision order
  std::size_t early_next_ = 0, nvme_ahead_ = 0;
  void set_early_order(const std::vector<Hook>& hooks);
  void refill_early();
  void drop_early();
  std::size_t forward_prestage_budget(const std::vector<Hook>& hooks) const;
  void set_prestage_order(const std::vector<Hook>& hooks, const std::vector<std::size_t>& hoist);
  void drop_staged();
  void prologue_next();
  void wait_barriers(cudaStream_t cs);
  void finish_iteration();
  struct IterRecord {
    std::uint64_t gen = 0;
    std::vector<Copy> copies;
    std::vector<Stall> stalls;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ontime, adam;
    std::vector<cudaEvent_t> marks, fences;
    std::size_t cks_buf = 0;
    std::uint64_t io_seq = 0;  // last NVMe job submitted in the iteration
    std::size_t spans = 0;     // AdamW launches with a recorded span
  };
  void harvest_front();
  void drain();
  void scrub(std::uint64_t gen);

  tencache::ExecutionTrace trace_;
  tencache::MachineConfig machine_;
  tencache::RunConfig cfg_;
  std::unique_ptr<tencache::IPolicy> policy_;
  tc_engine_options opts_;
  int device_ = 0;

  std::vector<TensorRec> recs_;
  std::unordered_map<tencache::TensorId, std::int32_t> index_;
  SlotPool gpu_, host_param_, host_opt_;
  std::map<std::uint64_t, std::uint8_t*> bounce_;  // pinned NVMe staging per class
  std::map<std::uint64_t, SlotSync> bounce_sync_;
  // HBM optimizer-state stages: a state is staged (H2D) ahead of its update,
  // updated in place, written back (D2H); the stage is then free again.
  std::vector<std::uint8_t*> stage_;
  std::vector<SlotSync> stage_sync_;
  std::deque<std::size_t> stage_free_;
  std::unordered_map<std::int32_t, std::size_t> staged_;  // state index -> stage
  std::vector<std::int32_t> prestage_order_;              // states in update (hoist) order
  std::size_t prestage_next_ = 0;
  std::size_t prestage_lookahead_ = 2;
  int prestage_fwd_override_ = -1;  // TC_PRESTAGE_FWD: states staged for the forward (-1: bandwidth model)
  bool adam_stamps_ = false;        // TC_ADAM_STAMPS: %globaltimer stamps around each AdamW (diagnostic)
  // Updates on the compute stream when the trace is migration-bound (the
  // compute stream idles on copies anyway, and a same-stream launch skips the
  // cross-stream scheduling latency); on the opt stream when compute-bound, to
  // overlap. TC_ADAM_ON_COMPUTE=0/1 overrides.
  bool adam_on_compute_ = false;
  // never with a ZeRO-3 exchange between ranks: an in-place update may wait
  // for peers' reads of its slot, which must not stall this rank's compute
  // stream. World 1 has no peers: C3 at N=1 (migration-bound) runs its
  // updates between the layers' GEMMs, on the whole GPU instead of beside
  // them (event-timed 0.55 -> 0.59 of the HBM peak, migration hidden 0.95 ->
  // 0.99, profiles/r02_adam_placement_c3.json)
  cudaStream_t adam_stream() const {
    return adam_on_compute_ && compute_ && (!z3_ || z3_->world == 1) ? compute_ : opt_;
  }
  double stamp_pre_ns_ = 0, stamp_post_ns_ = 0, stamps_ = 0;
  bool lookahead_ = true;           // TC_LOOKAHEAD: decide + pre-stage iteration t+1 at the end of t
  std::optional<std::vector<Hook>> ahead_;
  std::uint64_t stage_bytes_ = 0;
  std::map<std::uint64_t, std::vector<std::uint8_t*>> pout_scratch_;  // HBM updated-param scratch
  std::map<std::uint64_t, std::vector<SlotSync>> pout_sync_;
  std::map<std::uint64_t, std::size_t> pout_next_;
  std::uint8_t* grads_ = nullptr;
  std::uint64_t* d_checksums_ = nullptr;  // two buffers of n_accesses_ (iteration parity)
  std::vector<std::uint64_t> h_checksums_;
  std::uint64_t* h_result_ = nullptr;  // pinned + mapped, two buffers of n_accesses_ (iteration parity)
  std::uint64_t* d_result_ = nullptr;  // device alias of h_result_
  unsigned long long* h_span_ = nullptr;       // pinned + mapped copy of the AdamW span buffers (parity)
  unsigned long long* d_span_host_ = nullptr;  // device alias of h_span_
  cudaEvent_t result_ev_[2] = {nullptr, nullptr};
  std::uint64_t result_gen_ = 0;
  bool have_result_ = false;
  std::uint64_t* cks_base_ = nullptr;
  unsigned long long* d_span_ = nullptr;  // 2 parities x n_params x (min, max) AdamW kernel spans
  unsigned long long* span_base_ = nullptr;
  std::size_t span_cursor_ = 0;
  std::size_t n_accesses_ = 0, access_cursor_ = 0;
  std::unique_ptr<StripedFile> nvme_;  // NVMe tier backing files
  std::unique_ptr<NvmeQueue> io_;  // async NVMe tier I/O (null: synchronous fallback)
  cudaStream_t io_join_ = nullptr;  // joins a job's dependencies into one event of the submitting generation
  std::vector<cudaEvent_t> io_deps(std::vector<cudaEvent_t> deps);
  std::uint64_t nvme_read_async(TensorRec& r, void* dst, SlotSync& target, bool device = false);
  std::uint64_t nvme_write_async(TensorRec& r, const void* src, SlotSync& source, bool device = false);
  bool gds_ = false;  // NVMe <-> HBM through GPUDirect Storage (direct_io, nvidia-fs present: gds.hpp)
 public:
  bool gds() const { return gds_; }
 private:

  // h2d_/d2h_: cache decisions (prefetch, evict, restore); h2d_opt_/d2h_opt_:
  // optimizer-state staging and write-back, so evictions never queue behind
  // state traffic; opt_: the fused AdamW.
  cudaStream_t h2d_ = nullptr, d2h_ = nullptr, opt_ = nullptr, h2d_opt_ = nullptr, d2h_opt_ = nullptr;
  std::deque<IterRecord> pending_;
  std::vector<cudaEvent_t> phase_marks_;  // compute-stream timing marks: start, fwd end, bwd end, end
  cudaStream_t compute_ = nullptr;
  cudaStream_t compute_owned_ = nullptr;
  EventArena events_;
  std::vector<cudaEvent_t> barriers_;
  std::uint64_t barrier_io_ = 0;  // NVMe job a blocking request ended with
  // peak slots per (tier, class) over two iterations of decisions; also the
  // steady-state forward pass's non-instant H2D bytes (*fwd_h2d)
  std::map<std::pair<int, std::uint64_t>, std::uint32_t> simulate_occupancy(
      double* fwd_h2d = nullptr, std::set<tencache::TensorId>* in_nvme = nullptr,
      std::set<tencache::TensorId>* to_gpu = nullptr) const;
  int auto_stage_slots(double fwd_h2d) const;
  std::vector<Copy> copies_;
  std::vector<Stall> stalls_;                                      // (reach, go) on compute
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ontime_;        // (reach, arrival)
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> adam_;          // kernel start/end
  std::int64_t adam_step_ = 0;
  std::unique_ptr<std::ofstream> event_log_;  // measured per-copy JSONL (reference event-log schema + timings)
 public:
  void set_event_log(const std::string& path);
 private:
  std::unique_ptr<Zero3> z3_;
  std::unique_ptr<GemmStandin> standin_;  // compute_mode 2 (created on first use)
 public:
  std::string standin_info() const { return standin_ ? standin_->describe() : "{}"; }
 private:
  std::vector<double> phase_ms_;
  StepOptions so_;
  tc_engine_stats stats_{};
};

}  // namespace tcb
