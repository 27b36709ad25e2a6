// Alg. 3 PrefetchTensor / Alg. 4 EvictTensor, demand fetch, the halt rule,
// farthest-next-use victims, optimizer-state rotation, restore and reset
// (reference counterpart: scheduler.cpp:26-437). Every observable order of
// the reference is kept; the requests returned are the
// exact command stream the CUDA executor turns into copy-engine work.
#include <algorithm>

#include "tencache/tencache.hpp"

namespace tencache {

namespace {

struct SchedulerError : std::logic_error {
  using std::logic_error::logic_error;
};

using Req = TransferRequest;
using Kind = TransferRequest::Kind;

Req request(TensorId id, Tier src, Tier dst, std::uint64_t size, Kind kind) {
  Req r;
  r.tensor_id = id;
  r.src = src;
  r.dst = dst;
  r.size_bytes = size;
  r.kind = kind;
  return r;
}

Req staged_fetch(const SchedulerState& st, TensorId id, std::uint64_t size, Kind kind) {
  Req r = request(id, Tier::Nvme, Tier::Gpu, size, kind);
  r.via_cpu_staging = true;
  r.src_retains = st.nvme_copy.count(id) != 0;  // the NVMe replica stays
  return r;
}

template <typename Excluded>
bool excluded(const Excluded& ex, TensorId id) {
  return std::find(std::begin(ex), std::end(ex), id) != std::end(ex);
}

// Farthest next use wins; a tensor never used again this iteration beats any
// row; ties go to the lowest tensor id. Candidates arrive in buffer-id order.
template <typename Excluded>
std::optional<TensorId> farthest_next_use(const SchedulerState& st,
                                          const std::vector<std::pair<std::uint32_t, TensorId>>& cands,
                                          const Excluded& ex) {
  std::optional<TensorId> best;
  bool best_dead = false;
  std::uint32_t best_row = 0;
  for (const auto& cand : cands) {
    const TensorId t = cand.second;
    if (excluded(ex, t)) continue;
    const std::optional<std::uint32_t> next = st.next_use_row(t);
    const bool dead = !next;
    const std::uint32_t row = next.value_or(0);
    bool take;
    if (!best)
      take = true;
    else if (dead != best_dead)
      take = dead;
    else if (!dead && row != best_row)
      take = row > best_row;
    else
      take = t < *best;
    if (take) {
      best = t;
      best_dead = dead;
      best_row = row;
    }
  }
  return best;
}

const std::vector<TensorId> kNone;

std::uint32_t must(std::optional<std::uint32_t> v, const char* what) {
  if (!v) throw SchedulerError(what);
  return *v;
}

// Free one CPU parameter buffer of `size` by pushing an occupant to NVMe;
// GPU-designated occupants go first.
void spill_cpu_victim(SchedulerState& st, std::uint64_t size, std::vector<Req>& out) {
  std::optional<TensorId> victim = farthest_next_use(st, st.cpu_pool.occupants(size, true), kNone);
  if (!victim) victim = farthest_next_use(st, st.cpu_pool.occupants(size, false), kNone);
  if (!victim) throw SchedulerError("no CPU buffer of size " + std::to_string(size) + " exists");
  st.cpu_pool.release(must(st.cpu_pool.buffer_of(*victim), "victim has no CPU buffer"));
  Req r = request(*victim, Tier::Cpu, Tier::Nvme, size, Kind::Evict);
  if (!st.nvme_copy.insert(*victim).second) {  // a clean replica already exists
    r.instant = true;
    r.dst_has_copy = true;
  }
  st.current_loc[*victim] = Tier::Nvme;
  out.push_back(r);
}

template <typename Excluded>
void take_gpu_buffer(SchedulerState& st, TensorId id, std::uint64_t size, const Excluded& ex, std::vector<Req>& out) {
  if (st.gpu_pool.acquire(size, id)) return;
  const std::optional<TensorId> victim = farthest_next_use(st, st.gpu_pool.occupants(size, false), ex);
  if (!victim) throw SchedulerError("GPU class of size " + std::to_string(size) + " has no evictable buffer");
  st.active_window.erase(*victim);
  std::vector<Req> ev = evict_tensor(st, *victim);
  out.insert(out.end(), ev.begin(), ev.end());
  if (!st.gpu_pool.acquire(size, id)) throw SchedulerError("GPU buffer still unavailable after eviction");
}

// Stage `id` into its (already acquired) GPU buffer from wherever it lives.
void fetch_to_gpu(SchedulerState& st, TensorId id, Kind kind, std::vector<Req>& out) {
  const std::uint64_t size = st.tensor_size(id);
  if (st.current_loc.at(id) == Tier::Cpu) {
    st.cpu_pool.release(must(st.cpu_pool.buffer_of(id), "fetch: tensor has no CPU buffer"));
    out.push_back(request(id, Tier::Cpu, Tier::Gpu, size, kind));
  } else {
    out.push_back(staged_fetch(st, id, size, kind));
  }
  st.current_loc[id] = Tier::Gpu;
}

// An optimizer state is brought to host memory for its update: into a pooled
// slot when one is free, else through a transient buffer.
void stage_state_to_cpu(SchedulerState& st, TensorId sid, std::vector<Req>& out) {
  const std::uint64_t size = st.tensor_size(sid);
  const bool pooled = st.cpu_opt_pool.has_class(size) && st.cpu_opt_pool.acquire(size, sid).has_value();
  if (!pooled) st.opt_transient.insert(sid);
  std::erase(st.opt_pending, sid);
  out.push_back(request(sid, Tier::Nvme, Tier::Cpu, size, Kind::Prefetch));
  st.current_loc[sid] = Tier::Cpu;
}

}  // namespace

std::uint64_t SchedulerState::tensor_size(TensorId id) const {
  auto it = size_index.find(id);
  if (it != size_index.end()) return it->second;
  return trace->tensor(id).size_bytes;
}

Tier SchedulerState::final_loc(TensorId id) const {
  auto it = placement.location_of.find(id);
  return it != placement.location_of.end() ? it->second : opt_placement.location_of.at(id);
}

std::optional<std::uint32_t> SchedulerState::next_use_row(TensorId id) const {
  auto it = access_rows.find(id);
  if (it == access_rows.end()) return std::nullopt;
  auto row = std::lower_bound(it->second.begin(), it->second.end(), exec_row);
  if (row == it->second.end()) return std::nullopt;
  return *row;
}

SchedulerState make_scheduler_state(const ExecutionTrace& trace, PrefetchTable table, PlacementState params,
                                    PlacementState opt_states, BufferPool gpu_pool, BufferPool cpu_pool,
                                    BufferPool cpu_opt_pool) {
  SchedulerState st;
  st.trace = &trace;
  st.table = std::move(table);
  st.placement = std::move(params);
  st.opt_placement = std::move(opt_states);
  st.gpu_pool = std::move(gpu_pool);
  st.cpu_pool = std::move(cpu_pool);
  st.cpu_opt_pool = std::move(cpu_opt_pool);
  st.size_index.reserve(trace.tensors.size());
  for (const auto& t : trace.tensors) st.size_index.emplace(t.id, t.size_bytes);

  for (const PrefetchRow& row : st.table.rows) st.access_rows[row.tensor_id].push_back(row.order);
  st.step_row_end.assign(trace.steps.size(), 0);
  std::size_t rows = 0;
  for (std::size_t i = 0; i < trace.steps.size(); ++i) {
    if (trace.steps[i].phase != Phase::OptimizerUpdate) rows += trace.steps[i].tensor_ids.size();
    st.step_row_end[i] = rows;
  }
  for (const auto& pr : trace.optimizer_pairs()) st.opt_update_order.push_back(pr.first);

  for (const auto& [id, tier] : st.placement.location_of) st.current_loc[id] = tier;
  for (const auto& [id, tier] : st.opt_placement.location_of) st.current_loc[id] = tier;
  st.active_window.insert(st.placement.active_window.begin(), st.placement.active_window.end());
  st.nvme_copy = st.placement.nvme_copy;
  st.nvme_copy.insert(st.opt_placement.nvme_copy.begin(), st.opt_placement.nvme_copy.end());
  const bool any_nvme = std::any_of(st.current_loc.begin(), st.current_loc.end(),
                                    [](const auto& kv) { return kv.second == Tier::Nvme; });
  st.mode = any_nvme ? SchedulerMode::CpuGpuNvme : SchedulerMode::CpuGpu;

  for (TensorId id : st.placement.active_window)
    if (!st.gpu_pool.acquire(st.tensor_size(id), id)) throw SchedulerError("placement exceeds GPU pool");
  for (const auto& [id, tier] : st.placement.location_of)
    if (tier == Tier::Cpu && !st.cpu_pool.acquire(st.tensor_size(id), id))
      throw SchedulerError("placement exceeds CPU pool");
  for (TensorId sid : st.opt_update_order) {
    if (st.current_loc.at(sid) != Tier::Cpu) {
      st.opt_pending.push_back(sid);
    } else if (!st.cpu_opt_pool.acquire(st.tensor_size(sid), sid)) {
      throw SchedulerError("optimizer placement exceeds CPU pool");
    }
  }
  st.initial_gpu_pool = st.gpu_pool;
  st.initial_cpu_pool = st.cpu_pool;
  st.initial_cpu_opt_pool = st.cpu_opt_pool;
  st.initial_nvme_copy = st.nvme_copy;
  return st;
}

std::vector<TransferRequest> evict_tensor(SchedulerState& state, TensorId evict_tensor_id) {
  std::vector<Req> out;
  const TensorId id = evict_tensor_id;
  const std::uint64_t size = state.tensor_size(id);
  const std::uint32_t gpu_buf = must(state.gpu_pool.buffer_of(id), "evict_tensor: tensor not in a GPU buffer");
  const Tier home = state.final_loc(id);
  if (home == Tier::Nvme) {  // the NVMe replica is authoritative: just drop the GPU copy
    state.gpu_pool.release(gpu_buf);
    state.current_loc[id] = Tier::Nvme;
    Req r = request(id, Tier::Gpu, Tier::Nvme, size, Kind::Evict);
    r.instant = true;
    r.dst_has_copy = true;
    out.push_back(r);
    return out;
  }
  if (state.cpu_pool.free_count(size) == 0) spill_cpu_victim(state, size, out);
  const std::uint32_t cpu_buf = must(state.cpu_pool.acquire(size, id), "evict_tensor: CPU buffer unavailable after swap");
  if (home == Tier::Gpu) state.cpu_pool.set_designated(cpu_buf, true);
  out.push_back(request(id, Tier::Gpu, Tier::Cpu, size, Kind::Evict));
  state.gpu_pool.release(gpu_buf);
  state.current_loc[id] = Tier::Cpu;
  return out;
}

std::vector<TransferRequest> prefetch_tensor(SchedulerState& state, const std::vector<TensorId>& evicted_tensor_list) {
  std::vector<Req> out;
  auto& rows = state.table.rows;
  std::size_t& cur = state.table.cursor;
  for (const TensorId done : evicted_tensor_list) {
    if (cur >= rows.size() || !state.active_window.count(done)) continue;
    const std::size_t saved = cur;
    state.active_window.erase(done);
    while (cur < rows.size() && state.active_window.count(rows[cur].tensor_id)) ++cur;
    auto back_off = [&](bool halt) {
      state.active_window.insert(done);
      cur = saved;
      if (halt) state.halted = true;
    };
    // Halt: nothing left to stage, or the next needed tensor is the one that
    // just finished (evicting it would only force a reload).
    if (cur >= rows.size() || rows[cur].tensor_id == done) {
      back_off(true);
      continue;
    }
    const TensorId target = rows[cur].tensor_id;
    const std::uint64_t tsize = state.tensor_size(target);
    // Different classes: the paired eviction frees the wrong class, so a
    // same-class resident must be evictable or the prefetch is skipped.
    if (state.gpu_pool.free_count(tsize) == 0 && state.tensor_size(done) != tsize) {
      const TensorId ex[1] = {done};
      if (!farthest_next_use(state, state.gpu_pool.occupants(tsize, false), ex)) {
        back_off(false);
        continue;
      }
    }
    // Swap semantics: the target's CPU slot frees as its bytes leave for the
    // GPU, giving the eviction below a slot to land in.
    const bool from_cpu = state.current_loc.at(target) == Tier::Cpu;
    if (from_cpu) state.cpu_pool.release(must(state.cpu_pool.buffer_of(target), "prefetch: target has no CPU buffer"));
    std::vector<Req> ev = evict_tensor(state, done);
    out.insert(out.end(), ev.begin(), ev.end());
    state.active_window.insert(target);
    const TensorId ex[2] = {done, target};
    take_gpu_buffer(state, target, tsize, ex, out);
    out.push_back(from_cpu ? request(target, Tier::Cpu, Tier::Gpu, tsize, Kind::Prefetch)
                           : staged_fetch(state, target, tsize, Kind::Prefetch));
    state.current_loc[target] = Tier::Gpu;
    ++cur;
  }
  return out;
}

bool halt_check(const SchedulerState& state) {
  const auto& rows = state.table.rows;
  for (std::size_t i = state.table.cursor; i < rows.size(); ++i)
    if (!state.active_window.count(rows[i].tensor_id)) return false;
  return true;
}

std::vector<TransferRequest> on_step_start(SchedulerState& state, const TraceStep& step) {
  std::vector<Req> out;
  state.halted = false;
  state.exec_row = std::max(state.exec_row, state.step_row_end[step.step_index]);
  state.table.cursor = std::max(state.table.cursor, state.exec_row);
  if (step.phase == Phase::OptimizerUpdate) {
    const TensorId sid = step.tensor_ids.front();
    if (state.current_loc.at(sid) != Tier::Cpu) stage_state_to_cpu(state, sid, out);
    return out;
  }
  for (const TensorId id : step.tensor_ids) {
    auto loc = state.current_loc.find(id);
    if (loc == state.current_loc.end()) throw SchedulerError("access to unplaced tensor " + std::to_string(id));
    if (loc->second == Tier::Gpu) continue;
    // Demand miss: the schedule did not stage this access in time. The
    // step's own tensors are never evicted to make room.
    state.active_window.insert(id);
    take_gpu_buffer(state, id, state.tensor_size(id), step.tensor_ids, out);
    fetch_to_gpu(state, id, Kind::Prefetch, out);
  }
  return out;
}

std::vector<TransferRequest> optimizer_on_update_end(SchedulerState& state, TensorId state_id) {
  std::vector<Req> out;
  const std::uint64_t size = state.tensor_size(state_id);
  if (state.opt_transient.erase(state_id)) {  // updated outside the pool: write straight back
    out.push_back(request(state_id, Tier::Cpu, Tier::Nvme, size, Kind::Evict));
    state.current_loc[state_id] = Tier::Nvme;
    return out;
  }
  auto next = std::find_if(state.opt_pending.begin(), state.opt_pending.end(),
                           [&](TensorId id) { return state.tensor_size(id) == size; });
  const bool has_next = next != state.opt_pending.end();
  if (!has_next && state.final_loc(state_id) != Tier::Nvme) return out;  // stays resident
  state.cpu_opt_pool.release(must(state.cpu_opt_pool.buffer_of(state_id), "optimizer state has no CPU buffer"));
  out.push_back(request(state_id, Tier::Cpu, Tier::Nvme, size, Kind::Evict));
  state.current_loc[state_id] = Tier::Nvme;
  if (has_next) {
    const TensorId nid = *next;
    state.opt_pending.erase(next);
    state.cpu_opt_pool.acquire(size, nid);
    out.push_back(request(nid, Tier::Nvme, Tier::Cpu, size, Kind::Prefetch));
    state.current_loc[nid] = Tier::Cpu;
  }
  return out;
}

std::vector<TransferRequest> optimizer_step_schedule(const SchedulerState& state) {
  SchedulerState scratch = state;
  std::vector<Req> out;
  for (const TensorId sid : scratch.opt_update_order) {
    if (scratch.current_loc.at(sid) != Tier::Cpu) stage_state_to_cpu(scratch, sid, out);
    std::vector<Req> r = optimizer_on_update_end(scratch, sid);
    out.insert(out.end(), r.begin(), r.end());
  }
  return out;
}

std::vector<TransferRequest> restore_final_locations(SchedulerState& state, RestoreScope scope) {
  std::vector<Req> out;
  auto restore = [&](const std::map<TensorId, Tier>& finals) {
    for (const auto& [id, fin] : finals) {  // ascending tensor id
      const Tier cur = state.current_loc.at(id);
      if (cur == fin) continue;
      Req r = request(id, cur, fin, state.tensor_size(id), Kind::Restore);
      if (cur == Tier::Gpu && fin == Tier::Nvme && state.nvme_copy.count(id)) {
        r.instant = true;
        r.dst_has_copy = true;
      }
      if (cur == Tier::Nvme && fin == Tier::Gpu) {
        r.via_cpu_staging = true;
        r.src_retains = true;
      }
      out.push_back(r);
      state.current_loc[id] = fin;
    }
  };
  if (scope != RestoreScope::OptimizerStates) restore(state.placement.location_of);
  if (scope != RestoreScope::Parameters) restore(state.opt_placement.location_of);
  return out;
}

void reset_iteration(SchedulerState& state) {
  state.table.cursor = 0;
  state.exec_row = 0;
  state.halted = false;
  state.gpu_pool = state.initial_gpu_pool;
  state.cpu_pool = state.initial_cpu_pool;
  state.cpu_opt_pool = state.initial_cpu_opt_pool;
  state.nvme_copy = state.initial_nvme_copy;
  state.active_window = std::set<TensorId>(state.placement.active_window.begin(), state.placement.active_window.end());
  for (const auto& [id, tier] : state.placement.location_of) state.current_loc[id] = tier;
  for (const auto& [id, tier] : state.opt_placement.location_of) state.current_loc[id] = tier;
  state.opt_pending.clear();
  for (const TensorId sid : state.opt_update_order)
    if (state.current_loc.at(sid) != Tier::Cpu) state.opt_pending.push_back(sid);
  state.opt_transient.clear();
}

}  // namespace tencache
