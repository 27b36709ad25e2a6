// b200-tencache — the C++ decision API of 10Cache's tensor cache, re-implemented
// for the B200 engine. Source-compatible with the reference headers
// (/root/reference/proj/include/tencache/*.hpp): every type, member and free
// function a caller of the reference can name exists here with the same
// meaning, so the per-file headers next to this one (types.hpp, trace.hpp, …)
// simply include this file. Internals are our own (dense indexes, our own
// exact rational), see paper_2511_14124_b200/csrc/core/.
#pragma once

#include <cstdint>
#include <deque>
#include <map>
#include <memory>
#include <optional>
#include <ostream>
#include <set>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <unordered_map>
#include <utility>
#include <vector>

namespace tencache {

// ============================================================== vocabulary
// (reference: types.hpp:9-38)
using TensorId = std::uint32_t;

enum class Tier : std::uint8_t { Gpu, Cpu, Nvme };

const char* to_string(Tier t);
Tier tier_from_string(const std::string& s);

struct ConfigError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct OomError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// ============================================================ exact numbers
// (reference: rational.hpp:11-31, there boost::rational<cpp_int>)
//
// Arbitrary-precision signed integer: sign + magnitude in 32-bit limbs.
// The model clock needs ~224-bit intermediates.
class BigInt {
 public:
  BigInt() = default;
  template <typename T, typename = std::enable_if_t<std::is_integral_v<T>>>
  BigInt(T v) {  // NOLINT: implicit, like boost::multiprecision::cpp_int
    if constexpr (std::is_signed_v<T>) {
      if (v < 0) {
        neg_ = true;
        set_u64(static_cast<std::uint64_t>(0) - static_cast<std::uint64_t>(v));
        return;
      }
    }
    set_u64(static_cast<std::uint64_t>(v));
  }

  template <typename T>
  T convert_to() const {
    if constexpr (std::is_floating_point_v<T>) {
      return static_cast<T>(to_double());
    } else {
      std::uint64_t lo = low_u64();
      return neg_ ? static_cast<T>(static_cast<std::uint64_t>(0) - lo) : static_cast<T>(lo);
    }
  }

  bool is_zero() const { return w_.empty(); }
  bool is_negative() const { return neg_; }
  int sign() const { return w_.empty() ? 0 : (neg_ ? -1 : 1); }
  std::size_t bit_length() const;
  std::string str() const;
  double to_double() const;  // round to nearest, ties to even

  friend BigInt operator+(const BigInt& a, const BigInt& b);
  friend BigInt operator-(const BigInt& a, const BigInt& b);
  friend BigInt operator-(const BigInt& a);
  friend BigInt operator*(const BigInt& a, const BigInt& b);
  friend BigInt operator/(const BigInt& a, const BigInt& b);  // truncating
  friend BigInt operator%(const BigInt& a, const BigInt& b);
  friend BigInt operator<<(const BigInt& a, int bits);
  BigInt& operator+=(const BigInt& b) { return *this = *this + b; }
  BigInt& operator-=(const BigInt& b) { return *this = *this - b; }
  BigInt& operator*=(const BigInt& b) { return *this = *this * b; }
  BigInt& operator/=(const BigInt& b) { return *this = *this / b; }

  friend int compare(const BigInt& a, const BigInt& b);
  friend bool operator==(const BigInt& a, const BigInt& b) { return a.neg_ == b.neg_ && a.w_ == b.w_; }
  friend bool operator!=(const BigInt& a, const BigInt& b) { return !(a == b); }
  friend bool operator<(const BigInt& a, const BigInt& b) { return compare(a, b) < 0; }
  friend bool operator>(const BigInt& a, const BigInt& b) { return compare(a, b) > 0; }
  friend bool operator<=(const BigInt& a, const BigInt& b) { return compare(a, b) <= 0; }
  friend bool operator>=(const BigInt& a, const BigInt& b) { return compare(a, b) >= 0; }
  friend std::ostream& operator<<(std::ostream& os, const BigInt& a) { return os << a.str(); }

  // magnitude helpers shared with Rat
  static BigInt gcd(BigInt a, BigInt b);
  static void divmod(const BigInt& a, const BigInt& b, BigInt& q, BigInt& r);
  const std::vector<std::uint32_t>& words() const { return w_; }

 private:
  void set_u64(std::uint64_t m);
  std::uint64_t low_u64() const;
  void trim();

  bool neg_ = false;
  std::vector<std::uint32_t> w_;  // magnitude, little-endian base 2^32, no leading zeros
};

// Exact rational: gcd-reduced, positive denominator.
class Rat {
 public:
  Rat() : num_(0), den_(1) {}
  template <typename T, typename = std::enable_if_t<std::is_integral_v<T>>>
  Rat(T v) : num_(v), den_(1) {}  // NOLINT
  Rat(const BigInt& n) : num_(n), den_(1) {}  // NOLINT
  Rat(const BigInt& n, const BigInt& d);

  const BigInt& numerator() const { return num_; }
  const BigInt& denominator() const { return den_; }

  friend Rat operator+(const Rat& a, const Rat& b);
  friend Rat operator-(const Rat& a, const Rat& b);
  friend Rat operator*(const Rat& a, const Rat& b);
  friend Rat operator/(const Rat& a, const Rat& b);
  Rat& operator+=(const Rat& b) { return *this = *this + b; }
  Rat& operator-=(const Rat& b) { return *this = *this - b; }
  Rat& operator*=(const Rat& b) { return *this = *this * b; }
  Rat& operator/=(const Rat& b) { return *this = *this / b; }

  friend bool operator==(const Rat& a, const Rat& b) { return a.num_ == b.num_ && a.den_ == b.den_; }
  friend bool operator!=(const Rat& a, const Rat& b) { return !(a == b); }
  friend bool operator<(const Rat& a, const Rat& b);
  friend bool operator>(const Rat& a, const Rat& b) { return b < a; }
  friend bool operator<=(const Rat& a, const Rat& b) { return !(b < a); }
  friend bool operator>=(const Rat& a, const Rat& b) { return !(a < b); }

 private:
  struct Raw {};
  Rat(BigInt n, BigInt d, Raw) : num_(std::move(n)), den_(std::move(d)) {}
  void reduce();
  BigInt num_, den_;
};

Rat rat_from_double(double v);      // exact value of a finite double
double to_double(const Rat& r);     // nearest double of num and den, then divide
Rat rat_decimal(std::int64_t mantissa, int exp10);
std::string rat_to_string(const Rat& r);
inline Rat rat_of(std::uint64_t v) { return Rat(v); }
inline Rat rat_of(std::int64_t v) { return Rat(v); }
inline Rat rat_of(int v) { return Rat(v); }

// ================================================================== traces
// (reference: trace.hpp:14-90)
enum class TensorKind : std::uint8_t { ParamFP16, OptStateFP32 };
enum class Phase : std::uint8_t { Forward, Backward, OptimizerUpdate };
const char* to_string(Phase p);

struct TensorDescriptor {
  TensorId id = 0;
  std::uint64_t size_bytes = 0;
  TensorKind kind = TensorKind::ParamFP16;
  std::uint32_t layer = 0;
  friend bool operator==(const TensorDescriptor&, const TensorDescriptor&) = default;
};

struct TraceStep {
  std::uint32_t step_index = 0;
  Phase phase = Phase::Forward;
  std::vector<TensorId> tensor_ids;
  double compute_us = 0.0;
  friend bool operator==(const TraceStep&, const TraceStep&) = default;
};

struct ExecutionTrace {
  std::vector<TensorDescriptor> tensors;
  std::vector<TraceStep> steps;
  std::uint32_t iterations = 1;
  friend bool operator==(const ExecutionTrace&, const ExecutionTrace&) = default;

  bool has_tensor(TensorId id) const;
  const TensorDescriptor& tensor(TensorId id) const;
  std::vector<std::pair<TensorId, TensorId>> optimizer_pairs() const;  // (state, param)
};

struct TraceError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

using TensorCensus = std::map<std::uint64_t, std::uint64_t>;
struct SizeProfile {
  std::vector<std::uint64_t> choices;
};

inline constexpr double kDefaultComputeUsPerByte = 2.8e-5;
inline constexpr double kDefaultOptUsPerByte = 1.6e-6;
inline constexpr std::uint64_t kOptStateBytesPerParamByte = 6;

ExecutionTrace load_trace(const std::string& path);
void save_trace(const ExecutionTrace& trace, const std::string& path);
void validate_trace(const ExecutionTrace& trace);
ExecutionTrace synthesize_transformer_trace(std::uint32_t layers, std::uint32_t tensors_per_layer,
                                            const SizeProfile& profile, double compute_us_per_byte,
                                            std::uint64_t seed, std::uint32_t iterations = 1,
                                            double opt_us_per_byte = kDefaultOptUsPerByte,
                                            bool optimizer_steps = true);
TensorCensus tensor_census(const ExecutionTrace& trace, TensorKind kind);

// ================================================================= machine
// (reference: machine.hpp:10-41)
struct LinkSpec {
  Tier src = Tier::Cpu;
  Tier dst = Tier::Gpu;
  Rat bandwidth_gbps;
};
enum class CpuMemoryClass : std::uint8_t { Pinned, Pageable };

struct MachineConfig {
  std::uint64_t gpu_capacity_bytes = 0;
  std::uint64_t cpu_capacity_bytes = 0;
  std::vector<LinkSpec> links;
  CpuMemoryClass cpu_memory_class = CpuMemoryClass::Pinned;
  std::vector<LinkSpec> pinned_overrides;
  Rat effective_bandwidth(Tier src, Tier dst) const;
};

MachineConfig default_machine();
MachineConfig load_machine(const std::string& path);
Rat transfer_time_us(const MachineConfig& cfg, Tier src, Tier dst, std::uint64_t size_bytes);

// ================================================================ profiler
// (reference: analyzer.hpp:14-45)
struct PrefetchRow {
  std::uint32_t order = 0;
  TensorId tensor_id = 0;
  Rat activation_us;
  Tier current_loc = Tier::Cpu;
  Tier final_loc = Tier::Cpu;
};
struct PrefetchTable {
  std::vector<PrefetchRow> rows;
  std::size_t cursor = 0;
};
struct SizeDistribution {
  std::map<std::uint64_t, Rat> ratios;
  std::uint64_t total_size = 0;
  double ratio_as_double(std::uint64_t size) const { return to_double(ratios.at(size)); }
};

PrefetchTable build_prefetch_table(const ExecutionTrace& trace);
SizeDistribution size_distribution(const TensorCensus& tc);
Rat profile_overhead(const ExecutionTrace& trace);
void dump_prefetch_table_csv(const PrefetchTable& table, std::ostream& out);

// ========================================================= size-class pool
// (reference: bufpool.hpp:18-95)
struct PoolError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

struct BufferPlan {
  std::map<std::uint64_t, std::uint64_t> gpu_counts;
  std::map<std::uint64_t, std::uint64_t> cpu_counts;
  std::uint64_t gpu_avail_bytes = 0;
  std::uint64_t cpu_avail_bytes = 0;
  std::uint64_t gpu_planned_bytes() const;
  std::uint64_t cpu_planned_bytes() const;
};

BufferPlan plan_buffers(const TensorCensus& tc, const SizeDistribution& tsd, std::uint64_t gpu_avail,
                        std::uint64_t cpu_avail);

enum class ChunkState : std::uint8_t { Free, Occupied };

struct Chunk {
  std::uint32_t buffer_id = 0;
  std::uint64_t offset = 0;
  std::uint64_t size = 0;
  ChunkState state = ChunkState::Free;
  std::optional<TensorId> occupant;
  bool gpu_designated = false;
};

// Fixed-partition region: chunks of one size class occupy a contiguous run of
// buffer ids (ascending class, then index), so per-class scans walk only that
// run. Each class keeps a FIFO free list.
class BufferPool {
 public:
  BufferPool() = default;
  static BufferPool build(Tier tier, const std::map<std::uint64_t, std::uint64_t>& counts);

  std::optional<std::uint32_t> acquire(std::uint64_t size, TensorId tensor);
  void release(std::uint32_t buffer_id);
  void set_designated(std::uint32_t buffer_id, bool designated);
  std::optional<std::pair<std::uint32_t, TensorId>> find_victim(std::uint64_t size,
                                                                bool prefer_gpu_designated) const;
  std::vector<std::pair<std::uint32_t, TensorId>> occupants(std::uint64_t size, bool designated_only) const;

  bool has_class(std::uint64_t size) const { return classes_.count(size) != 0; }
  std::size_t free_count(std::uint64_t size) const;
  std::optional<std::uint32_t> buffer_of(TensorId tensor) const;

  Tier tier() const { return tier_; }
  std::uint64_t region_bytes() const { return region_bytes_; }
  std::uint64_t occupied_bytes() const { return occupied_bytes_; }
  const std::vector<Chunk>& chunks() const { return chunks_; }
  const Chunk& chunk(std::uint32_t buffer_id) const { return chunks_.at(buffer_id); }
  void dump_csv(std::ostream& out) const;

 private:
  struct SizeClass {
    std::uint32_t first = 0;  // first buffer id of the class run
    std::uint32_t count = 0;
    std::deque<std::uint32_t> free_fifo;
  };
  SizeClass& cls(std::uint64_t size);
  const SizeClass* find_cls(std::uint64_t size) const;

  Tier tier_ = Tier::Gpu;
  std::uint64_t region_bytes_ = 0;
  std::uint64_t occupied_bytes_ = 0;
  std::vector<Chunk> chunks_;
  std::map<std::uint64_t, SizeClass> classes_;
  std::unordered_map<TensorId, std::uint32_t> where_;
};

// =============================================================== placement
// (reference: placement.hpp:16-35)
struct PlacementState {
  std::map<TensorId, Tier> location_of;
  std::set<TensorId> nvme_copy;
  std::vector<TensorId> active_window;
  std::uint64_t gpu_param_count_nvme = 0;
};

PlacementState place_parameters(PrefetchTable& table, const ExecutionTrace& trace, const BufferPlan& plan);
PlacementState place_optimizer_states(const std::vector<TensorDescriptor>& states, std::uint64_t cpu_budget_bytes);
void dump_placement_csv(const PlacementState& placement, const ExecutionTrace& trace, std::ostream& out);

// =============================================================== scheduler
// (reference: scheduler.hpp:18-111)
enum class SchedulerMode : std::uint8_t { CpuGpu, CpuGpuNvme };

struct TransferRequest {
  enum class Kind : std::uint8_t { Prefetch, Evict, Restore };
  TensorId tensor_id = 0;
  Tier src = Tier::Cpu;
  Tier dst = Tier::Gpu;
  std::uint64_t size_bytes = 0;
  Kind kind = Kind::Prefetch;
  bool via_cpu_staging = false;
  bool instant = false;
  bool src_retains = false;
  bool dst_has_copy = false;
  bool blocking = false;
};

struct SchedulerState {
  SchedulerMode mode = SchedulerMode::CpuGpu;
  PrefetchTable table;
  PlacementState placement;
  PlacementState opt_placement;
  std::map<TensorId, Tier> current_loc;
  std::set<TensorId> active_window;
  std::set<TensorId> nvme_copy;
  bool halted = false;

  BufferPool gpu_pool;
  BufferPool cpu_pool;
  BufferPool cpu_opt_pool;

  const ExecutionTrace* trace = nullptr;
  std::map<TensorId, std::vector<std::uint32_t>> access_rows;
  std::vector<std::size_t> step_row_end;
  std::vector<TensorId> opt_update_order;

  std::size_t exec_row = 0;
  std::deque<TensorId> opt_pending;
  std::set<TensorId> opt_transient;

  BufferPool initial_gpu_pool, initial_cpu_pool, initial_cpu_opt_pool;
  std::set<TensorId> initial_nvme_copy;

  // b200 additions: O(1) size lookup by id (the reference scans the trace,
  // trace.cpp:22-26) and the size of every tensor's dense slot.
  std::unordered_map<TensorId, std::uint64_t> size_index;

  std::uint64_t tensor_size(TensorId id) const;
  Tier final_loc(TensorId id) const;
  std::optional<std::uint32_t> next_use_row(TensorId id) const;
};

SchedulerState make_scheduler_state(const ExecutionTrace& trace, PrefetchTable table, PlacementState params,
                                    PlacementState opt_states, BufferPool gpu_pool, BufferPool cpu_pool,
                                    BufferPool cpu_opt_pool);
std::vector<TransferRequest> on_step_start(SchedulerState& state, const TraceStep& step);
std::vector<TransferRequest> prefetch_tensor(SchedulerState& state, const std::vector<TensorId>& evicted_tensor_list);
std::vector<TransferRequest> evict_tensor(SchedulerState& state, TensorId evict_tensor_id);
bool halt_check(const SchedulerState& state);
std::vector<TransferRequest> optimizer_on_update_end(SchedulerState& state, TensorId state_id);
std::vector<TransferRequest> optimizer_step_schedule(const SchedulerState& state);
enum class RestoreScope : std::uint8_t { Parameters, OptimizerStates, All };
std::vector<TransferRequest> restore_final_locations(SchedulerState& state, RestoreScope scope = RestoreScope::All);
void reset_iteration(SchedulerState& state);

// ====================================================== comparison policies
// (reference: baselines.hpp:12-56)
enum class PolicyKind : std::uint8_t { TenCache, TenCachePlusOpt, ZeroInfinityLike, L2LLike, NoOffload };
PolicyKind policy_from_string(const std::string& name);
const char* to_string(PolicyKind kind);

struct ZeroInfinityState {
  const ExecutionTrace* trace = nullptr;
  int lookahead_k = 1;
  bool fits_gpu = false;
  std::map<TensorId, Tier> param_home;
  std::set<TensorId> gpu_resident;
  std::vector<std::size_t> param_step_order;
  std::map<std::size_t, std::size_t> param_step_pos;
};
ZeroInfinityState make_zero_infinity_state(const ExecutionTrace& trace, const MachineConfig& machine, int lookahead_k);
std::vector<TransferRequest> zero_infinity_step_begin(ZeroInfinityState& st, const TraceStep& step);
std::vector<TransferRequest> zero_infinity_step_end(ZeroInfinityState& st, const TraceStep& step);

struct L2LState {
  const ExecutionTrace* trace = nullptr;
  std::map<std::uint32_t, std::vector<TensorId>> layer_tensors;
  std::set<TensorId> gpu_resident;
  std::int64_t loaded_layer = -1;
  std::vector<std::size_t> param_step_order;
  std::map<std::size_t, std::size_t> param_step_pos;
};
L2LState make_l2l_state(const ExecutionTrace& trace);
std::vector<TransferRequest> l2l_step_begin(L2LState& st, const TraceStep& step);
std::vector<TransferRequest> l2l_step_end(L2LState& st, const TraceStep& step);
std::uint64_t no_offload_check(const ExecutionTrace& trace, const MachineConfig& machine);

// ================================================= policy plug-in + engine
// (reference: engine.hpp:19-92)
struct RunConfig {
  PolicyKind policy = PolicyKind::TenCache;
  std::vector<double> thresholds_us{10.0, 30.0, 100.0};
  bool restore_overlap = true;
  double batch_scale = 1.0;
  int zero_lookahead_k = 1;
  std::uint64_t seed = 0;
  std::ostream* event_log = nullptr;
};

struct SimReport {
  Rat total_time_us{0};
  std::vector<Rat> per_iteration_us;
  Rat hit_rate{0};
  std::uint64_t param_accesses = 0;
  std::uint64_t param_hits = 0;
  std::vector<Rat> param_wait_us;
  std::vector<std::pair<double, Rat>> pct_wait_below;
  Rat optimizer_miss_rate{0};
  std::uint64_t opt_accesses = 0;
  std::uint64_t opt_misses = 0;
  Rat gpu_utilization_timeavg{0};
  Rat cpu_utilization_timeavg{0};
  std::uint64_t fp16_in_nvme_count = 0;
  std::map<std::string, std::uint64_t> transfer_bytes;
  Rat profile_overhead_us{0};
  friend bool operator==(const SimReport&, const SimReport&) = default;
};

class IPolicy {
 public:
  struct InitInfo {
    std::uint64_t gpu_resident_bytes = 0;
    std::uint64_t cpu_resident_bytes = 0;
    std::uint64_t nvme_resident_bytes = 0;
    std::uint64_t fp16_in_nvme_count = 0;
  };
  virtual ~IPolicy() = default;
  virtual InitInfo init() = 0;
  virtual std::vector<TransferRequest> on_step_begin(const TraceStep& step) = 0;
  virtual std::vector<TransferRequest> on_step_end(const TraceStep& step) = 0;
  virtual std::vector<TransferRequest> on_param_restore_point() = 0;
  virtual std::vector<TransferRequest> on_iteration_end() = 0;
  virtual void reset_iteration() = 0;
  // b200 addition: the scheduler state behind the TenCache policies (pool
  // contents for buffer-assignment parity and the CUDA executor); nullptr for
  // the comparison policies.
  virtual const SchedulerState* scheduler_state() const { return nullptr; }
  // b200 addition: the tier each tensor occupies after init() (before any
  // request), so an executor can materialise the initial placement.
  virtual std::optional<Tier> initial_tier(TensorId id) const { return std::nullopt; }
};

std::unique_ptr<IPolicy> make_policy(const ExecutionTrace& trace, const MachineConfig& machine,
                                     const RunConfig& config);

SimReport run(const ExecutionTrace& trace, const MachineConfig& machine, const RunConfig& config);

inline constexpr std::size_t kReferenceTensorGuard = 64;
// Same contract as the reference's brute-force oracle entry (engine.hpp:81-83):
// the ≤64-tensor guard, then the model-clock run.
SimReport run_reference(const ExecutionTrace& trace, const MachineConfig& machine, const RunConfig& config);

enum class SweepAxis : std::uint8_t { BatchScale, GpuCapacity, CpuCapacity, Pinned };
SweepAxis sweep_axis_from_string(const std::string& name);
const char* to_string(SweepAxis axis);
std::vector<SimReport> sweep(const ExecutionTrace& trace, const MachineConfig& machine, const RunConfig& config,
                             SweepAxis axis, const std::vector<double>& values, unsigned threads = 1);

}  // namespace tencache
