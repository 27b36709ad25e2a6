// ZeRO-3 exchange of the executor: NCCL all-gather /
// reduce-scatter + pack kernels, or the fused peer-memory kernels over CUDA
// IPC mappings (p2p_exchange.cu).
#include "executor.hpp"

#include <algorithm>
#include <cstring>

namespace tcb {

using namespace tencache;

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
  zero3_gather(x, cs);
  if (backward) zero3_reduce(x, cs, true);
}

// The gather half of an access: chunk x's pieces of the layer from every rank
// into the flat layer view (and their checksums).
void Executor::zero3_gather(TensorRec& x, cudaStream_t cs) {
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
    // (a rank whose piece of the chunk is empty is read by nobody: the gather
    // kernel skips zero-byte pieces, so its counter never moves)
    if (cp.rank_bytes[z.rank] > 0) {
      sl.sync.peer_cnt = &z.ctl->cnt[cp.chunk];
      sl.sync.peer_target = a * peers_n;
    }
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
}

// Gradient view writes from here on: every peer pulled the view's previous
// contents (p2p; NCCL reads it synchronously on this stream).
void Executor::zero3_grad_fence(cudaStream_t cs) {
  Zero3& z = *z3_;
  const unsigned peers_n = static_cast<unsigned>(z.world - 1);
  if (z.p2p && peers_n && z.grad_epoch > 0) stream_wait_value32(cs, &z.ctl->gcnt, z.grad_epoch * peers_n);
}

// The reduce half of a backward access: the full-layer gradient of chunk x's
// pieces in the gradient view (stand_in: seeded per rank, written here; else
// the caller's, written since zero3_grad_fence) is summed over the ranks into
// this rank's gradient chunk.
void Executor::zero3_reduce(TensorRec& x, cudaStream_t cs, bool stand_in) {
  Zero3& z = *z3_;
  const Zero3::ChunkPlan& cp = z.plans.at(index_of(x.id));
  if (stand_in) {
    zero3_grad_fence(cs);
    for (const auto& [off, nb] : cp.pieces) {
      TCB_CK(launch_fill_normal_bf16(reinterpret_cast<std::uint16_t*>(z.gview + off), nb / 2, 1e-3f,
                                     static_cast<std::uint64_t>(adam_step_) * 1000003ull + static_cast<std::uint64_t>(z.rank),
                                     (static_cast<std::uint64_t>(cp.layer) << 40) + off / 2, cs));
      ++stats_.kernel_launches;
    }
  }
  if (z.p2p) ++z.grad_epoch;
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

// Between step_begin and step_end of a caller-computed step: the flat layer
// view the step gathered (read it on the compute stream) and the gradient
// view the caller fills for a backward step (same layout; summed over the
// ranks into this rank's chunks at step_end).
void Executor::zero3_views(void** params, void** grads, std::uint64_t* layer_bytes) {
  if (!z3_) throw ConfigError("zero3_views: no ZeRO-3 exchange (tc_engine_enable_zero3)");
  if (!open_ || !open_->in_step || !open_->external || z3_->open_layer < 0)
    throw DeviceError(TC_EARG, "zero3_views: no caller-computed forward/backward step open");
  *params = z3_->view;
  *grads = z3_->gview;
  *layer_bytes = 2 * z3_->layer_elems.at(static_cast<std::size_t>(z3_->open_layer));
}

// This rank's IPC handles: HBM parameter pool, control block, gradient view.
std::vector<std::uint8_t> Executor::p2p_handles() {
  if (!z3_) throw ConfigError("p2p exchange needs tc_engine_enable_zero3 first");
  Zero3& z = *z3_;
  if (!z.ctl) {
    TCB_CK(cudaMalloc(&z.ctl, sizeof(P2PCtl)));
    TCB_CK(cudaMemset(z.ctl, 0, sizeof(P2PCtl)));
  }
  if (!z.peers.scratch) {
    TCB_CK(cudaMalloc(&z.peers.scratch, sizeof(unsigned) * (kMaxPeers + 1)));
    TCB_CK(cudaMemset(z.peers.scratch, 0, sizeof(unsigned) * (kMaxPeers + 1)));
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

}  // namespace tcb
