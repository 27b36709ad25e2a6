// ZeRO-3 exchange fused into single kernels over peer memory (NVLink/NVSwitch
// P2P loads through CUDA IPC mappings) — the all-gather + unpack of a
// parameter chunk and the pack + reduce-scatter of its gradient, each one
// launch with no NCCL call and no intermediate gather buffer.
//
// Protocol (monotonic epochs, system-scope release/acquire):
//   owner  : chunk resident (copy event awaited) -> publish(off, epoch=a)
//   reader : spin ld.acquire.sys(pub_epoch[c]) >= a -> copy -> red.release.sys cnt[c] += 1
//   owner  : any later writer of the slot waits cnt[c] >= a*(N-1) (stream wait value)
// and for gradients: owner fills its view, publish_grad(g); readers pull,
// then gcnt += 1; the owner refills its view only when gcnt >= g*(N-1).
#include "dataplane.cuh"

namespace tcb {

namespace {

__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_acquire_sys64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(unsigned* p, unsigned v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void red_add_release_sys(unsigned* p, unsigned v) {
  asm volatile("red.release.sys.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__global__ void publish_kernel(P2PCtl* ctl, std::uint32_t chunk, std::uint64_t off, std::uint32_t epoch) {
  // the chunk's bytes landed before this kernel (stream order after the copy
  // event); make them and the offset visible system-wide before the epoch.
  asm volatile("fence.acq_rel.sys;" ::: "memory");
  ctl->pub_off[chunk] = off;
  asm volatile("fence.acq_rel.sys;" ::: "memory");
  st_release_sys(&ctl->pub_epoch[chunk], epoch);
}

__global__ void publish_grad_kernel(P2PCtl* ctl, std::uint32_t gepoch) {
  asm volatile("fence.acq_rel.sys;" ::: "memory");
  st_release_sys(&ctl->gpub, gepoch);
}

constexpr int kThr = 256;
constexpr std::uint64_t kTile = 64 * 1024;

struct GatherArgs {
  PeerTable t;
  std::uint32_t chunk, epoch;
  std::uint64_t bytes[kMaxPeers], view_off[kMaxPeers], tiles_before[kMaxPeers + 1];
  std::uint8_t* view;
  unsigned* done;  // per-peer tile completion counters (local scratch, zeroed)
};

// grid.x = total tiles over all peers' pieces; a CTA copies one 64 KiB tile
// of one peer's piece; the last CTA of a peer counts the read there.
__global__ void __launch_bounds__(kThr) gather_unpack_kernel(GatherArgs a) {
  int q = 0;
  while (q + 1 <= a.t.world && a.tiles_before[q + 1] <= blockIdx.x) ++q;
  const std::uint64_t tile = blockIdx.x - a.tiles_before[q];
  __shared__ unsigned long long s_off;
  if (threadIdx.x == 0) {
    const P2PCtl* c = a.t.ctl[q];
    while (ld_acquire_sys(&c->pub_epoch[a.chunk]) < a.epoch) __nanosleep(200);
    s_off = ld_acquire_sys64(&c->pub_off[a.chunk]);
  }
  __syncthreads();
  const std::uint8_t* src = a.t.pool[q] + s_off + tile * kTile;
  std::uint8_t* dst = a.view + a.view_off[q] + tile * kTile;
  const std::uint64_t len = min(kTile, a.bytes[q] - tile * kTile);
  const bool vec = ((reinterpret_cast<std::uintptr_t>(src) | reinterpret_cast<std::uintptr_t>(dst) | len) & 15) == 0;
  if (vec) {  // four 16-byte peer loads in flight per thread (NVLink latency)
    const uint4* s4 = reinterpret_cast<const uint4*>(src);
    uint4* d4 = reinterpret_cast<uint4*>(dst);
    const std::uint64_t nv = len / 16;
    std::uint64_t i = threadIdx.x;
    for (; i + 3 * kThr < nv; i += 4 * kThr) {
      const uint4 r0 = s4[i], r1 = s4[i + kThr], r2 = s4[i + 2 * kThr], r3 = s4[i + 3 * kThr];
      d4[i] = r0;
      d4[i + kThr] = r1;
      d4[i + 2 * kThr] = r2;
      d4[i + 3 * kThr] = r3;
    }
    for (; i < nv; i += kThr) d4[i] = s4[i];
  } else {
    for (std::uint64_t i = threadIdx.x; i < len; i += kThr) dst[i] = src[i];
  }
  __syncthreads();
  if (threadIdx.x == 0 && q != a.t.rank) {
    __threadfence();
    const unsigned ntiles = static_cast<unsigned>(a.tiles_before[q + 1] - a.tiles_before[q]);
    if (atomicAdd(&a.done[q], 1u) + 1 == ntiles) {
      a.done[q] = 0;  // reset the scratch for the next launch (stream-ordered)
      red_add_release_sys(&a.t.ctl[q]->cnt[a.chunk], 1u);
    }
  }
}

struct PullArgs {
  PeerTable t;
  std::uint32_t gepoch;
  std::uint64_t view_off, bytes, chunk_bytes;
  std::uint16_t* grad;
  unsigned* done;
  int vec;  // every view + view_off and grad 16-byte aligned: 16-byte loads/stores
};

__device__ __forceinline__ std::uint32_t rne_bf16(float f) {
  std::uint32_t u = __float_as_uint(f);
  if ((u & 0x7fffffffu) > 0x7f800000u) return ((u >> 16) | 0x40u) & 0xffffu;
  return (u + 0x7fffu + ((u >> 16) & 1u)) >> 16;
}

// U units of 8 elements per iteration while all U are inside the valid
// range and world <= W: U x world 16-byte loads issued before the sums.
// Advances i0 past the units it handled; same fp32 rank order as the kernel.
template <int U, int W>
__device__ __forceinline__ void pull_units(const PullArgs& a, std::uint64_t& i0, std::uint64_t stride,
                                           std::uint64_t valid) {
  if (a.t.world > W) return;
  for (; i0 + (U - 1) * stride + 8 <= valid; i0 += U * stride) {
    uint4 w[U][W];
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int q = 0; q < W; ++q)
        if (q < a.t.world) w[u][q] = *reinterpret_cast<const uint4*>(a.t.gview[q] + a.view_off + (i0 + u * stride) * 2);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      float acc[8];
      const std::uint32_t* w0 = reinterpret_cast<const std::uint32_t*>(&w[u][0]);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        acc[2 * k] = __uint_as_float(w0[k] << 16);
        acc[2 * k + 1] = __uint_as_float(w0[k] & 0xffff0000u);
      }
#pragma unroll
      for (int q = 1; q < W; ++q) {
        if (q >= a.t.world) break;
        const std::uint32_t* wq = reinterpret_cast<const std::uint32_t*>(&w[u][q]);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          acc[2 * k] += __uint_as_float(wq[k] << 16);
          acc[2 * k + 1] += __uint_as_float(wq[k] & 0xffff0000u);
        }
      }
      uint4 o;
      o.x = rne_bf16(acc[0]) | (rne_bf16(acc[1]) << 16);
      o.y = rne_bf16(acc[2]) | (rne_bf16(acc[3]) << 16);
      o.z = rne_bf16(acc[4]) | (rne_bf16(acc[5]) << 16);
      o.w = rne_bf16(acc[6]) | (rne_bf16(acc[7]) << 16);
      *reinterpret_cast<uint4*>(a.grad + i0 + u * stride) = o;
    }
  }
}

// Each thread reduces 8 bf16 values across all ranks' views (fp32, rank
// order, one rounding); padding of the chunk is written as zero.
__global__ void __launch_bounds__(kThr) pull_reduce_kernel(PullArgs a) {
  if (threadIdx.x == 0)  // every rank's gradient view of this epoch is published
    for (int q = 0; q < a.t.world; ++q)
      while (ld_acquire_sys(&a.t.ctl[q]->gpub) < a.gepoch) __nanosleep(200);
  __syncthreads();
  const std::uint64_t n = a.chunk_bytes / 2, valid = a.bytes / 2;
  const std::uint64_t stride = static_cast<std::uint64_t>(gridDim.x) * kThr * 8;
  std::uint64_t i0 = (static_cast<std::uint64_t>(blockIdx.x) * kThr + threadIdx.x) * 8;
  if (a.vec && a.t.world <= 4) {  // U units per iteration: U x world 16-byte loads in flight per thread
    pull_units<4, 2>(a, i0, stride, valid);  // world <= 2
    pull_units<2, 4>(a, i0, stride, valid);  // world <= 4 (and the rest of world <= 2)
  }
  for (std::uint64_t i = i0; i < n; i += stride) {
    if (a.vec && i + 8 <= valid) {  // 16 bytes per rank per thread, same fp32 order as below
      uint4 w[kMaxPeers];
#pragma unroll
      for (int q = 0; q < kMaxPeers; ++q)
        if (q < a.t.world) w[q] = *reinterpret_cast<const uint4*>(a.t.gview[q] + a.view_off + i * 2);
      float acc[8];
      const std::uint32_t* w0 = reinterpret_cast<const std::uint32_t*>(&w[0]);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        acc[2 * k] = __uint_as_float(w0[k] << 16);
        acc[2 * k + 1] = __uint_as_float(w0[k] & 0xffff0000u);
      }
#pragma unroll
      for (int q = 1; q < kMaxPeers; ++q) {
        if (q >= a.t.world) break;
        const std::uint32_t* wq = reinterpret_cast<const std::uint32_t*>(&w[q]);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          acc[2 * k] += __uint_as_float(wq[k] << 16);
          acc[2 * k + 1] += __uint_as_float(wq[k] & 0xffff0000u);
        }
      }
      uint4 o;
      o.x = rne_bf16(acc[0]) | (rne_bf16(acc[1]) << 16);
      o.y = rne_bf16(acc[2]) | (rne_bf16(acc[3]) << 16);
      o.z = rne_bf16(acc[4]) | (rne_bf16(acc[5]) << 16);
      o.w = rne_bf16(acc[6]) | (rne_bf16(acc[7]) << 16);
      *reinterpret_cast<uint4*>(a.grad + i) = o;
      continue;
    }
    float acc[8];
    {  // the sum starts from rank 0's value (not +0): a single rank reduces to an exact copy, -0 included
      const std::uint16_t* v = reinterpret_cast<const std::uint16_t*>(a.t.gview[0] + a.view_off);
#pragma unroll
      for (int k = 0; k < 8; ++k) acc[k] = i + k < valid ? __uint_as_float(static_cast<unsigned>(v[i + k]) << 16) : 0.0f;
    }
    for (int q = 1; q < a.t.world; ++q) {
      const std::uint16_t* v = reinterpret_cast<const std::uint16_t*>(a.t.gview[q] + a.view_off);
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (i + k < valid) acc[k] += __uint_as_float(static_cast<unsigned>(v[i + k]) << 16);
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (i + k >= n) break;
      a.grad[i + k] = static_cast<std::uint16_t>(i + k < valid ? rne_bf16(acc[k]) : 0u);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(a.done, 1u) + 1 == gridDim.x) {
      *a.done = 0;
      for (int q = 0; q < a.t.world; ++q)
        if (q != a.t.rank) red_add_release_sys(&a.t.ctl[q]->gcnt, 1u);
    }
  }
}

}  // namespace

cudaError_t launch_p2p_publish(P2PCtl* ctl, std::uint32_t chunk, std::uint64_t off, std::uint32_t epoch,
                               cudaStream_t st) {
  publish_kernel<<<1, 1, 0, st>>>(ctl, chunk, off, epoch);
  return cudaGetLastError();
}

cudaError_t launch_p2p_publish_grad(P2PCtl* ctl, std::uint32_t gepoch, cudaStream_t st) {
  publish_grad_kernel<<<1, 1, 0, st>>>(ctl, gepoch);
  return cudaGetLastError();
}

cudaError_t launch_p2p_gather_unpack(const PeerTable& t, std::uint32_t chunk, std::uint32_t epoch,
                                     const std::uint64_t* piece_bytes, const std::uint64_t* piece_view_off,
                                     std::uint8_t* view, cudaStream_t st) {
  GatherArgs a{};
  a.t = t;
  a.chunk = chunk;
  a.epoch = epoch;
  a.view = view;
  a.done = t.scratch;
  if (a.done == nullptr) return cudaErrorInvalidValue;
  a.tiles_before[0] = 0;
  for (int q = 0; q < t.world; ++q) {
    a.bytes[q] = piece_bytes[q];
    a.view_off[q] = piece_view_off[q];
    a.tiles_before[q + 1] = a.tiles_before[q] + (piece_bytes[q] + kTile - 1) / kTile;
  }
  const std::uint64_t tiles = a.tiles_before[t.world];
  if (tiles == 0) return cudaSuccess;
  gather_unpack_kernel<<<static_cast<unsigned>(tiles), kThr, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_p2p_pull_reduce(const PeerTable& t, std::uint32_t gepoch, std::uint64_t view_off,
                                   std::uint64_t bytes, std::uint64_t chunk_bytes, std::uint16_t* grad,
                                   cudaStream_t st) {
  PullArgs a{};
  a.t = t;
  a.gepoch = gepoch;
  a.view_off = view_off;
  a.bytes = bytes;
  a.chunk_bytes = chunk_bytes;
  a.grad = grad;
  if (t.scratch == nullptr) return cudaErrorInvalidValue;
  a.done = t.scratch + kMaxPeers;
  std::uintptr_t al = reinterpret_cast<std::uintptr_t>(grad) | view_off;
  for (int q = 0; q < t.world; ++q) al |= reinterpret_cast<std::uintptr_t>(t.gview[q]);
  a.vec = (al & 15) == 0 ? 1 : 0;
  const std::uint64_t units = (chunk_bytes / 2 + 8 * kThr - 1) / (8 * kThr);
  // grid-stride over <= 8 x 148 CTAs: every CTA pays a system-scope poll of
  // the peers' publish words and a completion atomic, so one unit per thread
  // (8192 CTAs per chunk) measured 2x slower than this
  const unsigned grid = static_cast<unsigned>(std::max<std::uint64_t>(1, std::min<std::uint64_t>(units, 8 * 148)));
  pull_reduce_kernel<<<grid, kThr, 0, st>>>(a);
  return cudaGetLastError();
}

}  // namespace tcb
