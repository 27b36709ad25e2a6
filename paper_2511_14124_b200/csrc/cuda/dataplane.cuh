// Device-side declarations of the data-plane kernels (sm_100a). Host
// launchers are in dataplane.cu; the C-ABI wrappers in capi/dataplane_capi.cpp.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace tcb {

struct PackSeg {  // device-side fragment with its start in the virtual stream
  std::uint64_t src_off, dst_off, bytes, vstart;
};

struct AdamScalars {
  float b1, b2, omb1, omb2, eps, step_size, inv_sqrt_bc2, decay;
};

AdamScalars adam_scalars(double lr, double b1, double b2, double eps, double wd, std::int64_t step);

// One chunk of a batched AdamW launch: n elements (a multiple of 8) at
// 16-byte aligned addresses; pout may be null.
//
// Packed split-master chunks (packed != null; n a multiple of kSplitTile):
// the state is not stored as [p32 | m | v] but in the PackedLayout below.
//  * The fp32 master's high half is the bf16 parameter at `pout` (the update's
//    own RNE output, kept in HBM) up to one rounding step: the state carries
//    the low half `lo` and one round bit rb per element: hi = B - rb for a
//    non-NaN B, hi = rb ? B & ~0x40 : B for a NaN B (the cast sets the quiet
//    bit). Exact for every fp32 value.
//  * m and v keep bits 0-23 (mantissa + the exponent's lowest bit) as they
//    are; byte 3 (sign + the exponent's top 7 bits) is coded against the
//    largest top-7 value of each 32-element group: m as a 4-bit offset (14 =
//    top bits zero, 15 = escape) with its sign, v as a 5-bit offset (30 =
//    zero, 31 = escape; v's sign is not stored). An element outside those
//    windows (or a negative v) is escaped: byte 3 of its m and v lives in
//    `ovf` (2 B/element), which the kernel reads and writes itself through a
//    device-accessible pointer (the mapped tail of the state's pinned host
//    slot), so the bytes that cross PCIe have a fixed size; one flag byte per
//    warp and tile says whether any element of its 256 used it. Bytes are
//    moved with byte permutes and SWAR arithmetic on 4 elements at a time.
// The kernel reads (lo, rb, B, planes) and writes (lo', rb', B', planes').
// p, m, v are unused for packed chunks.
struct AdamChunk {
  float* p;
  float* m;
  float* v;
  const std::uint16_t* g;
  std::uint16_t* pout;
  std::uint64_t n;
  std::uint8_t* packed = nullptr;  // PackedLayout prefix (HBM stage)
  std::uint8_t* ovf = nullptr;     // 2n bytes: raw exponents of overflow tiles (device-accessible)
};
constexpr std::uint64_t kSplitTile = 2048;  // elements per AdamW tile; packed chunks hold whole tiles

#ifdef __CUDACC__
#define TCB_HD __host__ __device__
#else
#define TCB_HD
#endif

// Byte offsets of the planes of a packed state of n parameters (n %
// kSplitTile == 0) inside its 12n-byte slot; [0, bytes) crosses PCIe
// (9.44 B/param), [ovf, ovf + 2n) is the overflow area. Per element:
// lo u16 | rb 1 bit | mlo u16 (m bits 0-15) | mb2 u8 (m bits 16-23) | vlo u16 |
// vb2 u8 | code u8 (m sign << 7 | m code << 3 | v code bits 0-2) | x2 2 bits
// (v code bits 3-4); per 32-element group: base u16 (m's largest top-7 |
// v's << 8); per tile: 8 flag bytes (one per 256 elements: an escape used the
// overflow area). The windows (m: 13
// steps of 2 binades, v: 29) cover the moments of a run whose gradient never
// changes (v ~ g^2 spans twice g's binades); an EMA over changing gradients
// is narrower.
struct PackedLayout {
  std::uint64_t n, lo, rb, mlo, mb2, vlo, vb2, code, x2, base, flags, bytes, ovf;
};
TCB_HD inline PackedLayout packed_layout(std::uint64_t n) {
  PackedLayout L{};
  L.n = n;
  L.lo = 0;
  L.rb = 2 * n;
  L.mlo = L.rb + n / 8;
  L.mb2 = L.mlo + 2 * n;
  L.vlo = L.mb2 + n;
  L.vb2 = L.vlo + 2 * n;
  L.code = L.vb2 + n;
  L.x2 = L.code + n;
  L.base = L.x2 + n / 4;
  L.flags = L.base + n / 16;
  L.bytes = (L.flags + n / 256 + 15) / 16 * 16;
  L.ovf = L.bytes;
  return L;
}
constexpr int kMaxAdamChunks = 8;
struct AdamBatch {  // kernel parameter: the chunks and their first tile in the launch's tile space
  AdamChunk chunk[kMaxAdamChunks];
  std::uint64_t tile_begin[kMaxAdamChunks + 1];
  int count;
};

// All launchers return cudaGetLastError() of the launch.
// span_min/span_max (optional): atomicMin'd with the first
// CTA's start and atomicMax'd with the last CTA's end (%globaltimer ns) — the
// kernel's resident span, free of launch and queueing gaps.
cudaError_t launch_adamw(float* p, float* m, float* v, const std::uint16_t* g, std::uint16_t* pout, std::uint64_t n,
                         const AdamScalars& s, float grad_scale, cudaStream_t st,
                         unsigned long long* span_min = nullptr, unsigned long long* span_max = nullptr);
// Up to kMaxAdamChunks chunks in one launch (same hyper-parameters and step);
// cudaErrorInvalidValue for an unaligned chunk or a count out of range.
cudaError_t launch_adamw_batch(const AdamChunk* chunks, int count, const AdamScalars& s, float grad_scale,
                               cudaStream_t st, unsigned long long* span_min = nullptr,
                               unsigned long long* span_max = nullptr);
cudaError_t launch_cast_bf16_to_f32(const std::uint16_t* in, float* out, std::uint64_t n, cudaStream_t st);
cudaError_t launch_cast_f32_to_bf16(const float* in, std::uint16_t* out, std::uint64_t n, cudaStream_t st);
// inverse = false: dst[dst_off..] <- src[src_off..]; true: dst[src_off..] <- src[dst_off..]
cudaError_t launch_pack(const PackSeg* segs, std::uint32_t n, std::uint64_t total, const void* src, void* dst,
                        bool inverse, bool aligned16, cudaStream_t st);
cudaError_t launch_checksum(const void* data, std::uint64_t bytes, unsigned long long* out, cudaStream_t st);
cudaError_t launch_spin(std::uint64_t ns, int ctas, cudaStream_t st);
// Small fills/copies of 64-bit words as kernels: never queued on a copy engine
// behind bulk DMA (dst may be mapped pinned host memory: posted PCIe writes).
cudaError_t launch_fill_u64(unsigned long long* dst, unsigned long long value, std::uint64_t n, cudaStream_t st);
cudaError_t launch_copy_u64(unsigned long long* dst, const unsigned long long* src, std::uint64_t n, cudaStream_t st);
// Diagnostic: one thread writes %globaltimer (ns) to *out when the stream reaches it.
cudaError_t launch_stamp(unsigned long long* out, cudaStream_t st);
// Deterministic N(0, sigma) bf16 fill (counter-based RNG keyed by seed, stream).
cudaError_t launch_fill_normal_bf16(std::uint16_t* out, std::uint64_t n, float sigma, std::uint64_t seed,
                                    std::uint64_t stream_id, cudaStream_t st);
// Optimizer-state init from bf16 params: p32 = float(param), m = v = 0.
cudaError_t launch_init_state(const std::uint16_t* param, float* state, std::uint64_t n, cudaStream_t st);
// Packed split-master codec (layout above), out of place, n % kSplitTile == 0;
// `packed` is a whole 12n-byte state (prefix + overflow area):
// expand: packed + bf16 params -> full [p32|m|v];
// compress: full + bf16 params -> packed; *mismatch (device word, set to
// nonzero, never cleared) when some p32 does not round to its bf16 param,
// i.e. the state is not representable split.
cudaError_t launch_state_expand(const std::uint8_t* packed, const std::uint16_t* param, float* full, std::uint64_t n,
                                cudaStream_t st);
cudaError_t launch_state_compress(const float* full, const std::uint16_t* param, std::uint8_t* packed, std::uint64_t n,
                                  unsigned* mismatch, cudaStream_t st);

int num_sms();

}  // namespace tcb

namespace tcb {

// ------------------------------------------------ ZeRO-3 exchange over peer memory
// Control block of one rank, in its HBM, mapped into every peer (CUDA IPC).
// Epochs and counters are monotonic over the run.
struct P2PCtl {
  static constexpr int kMaxChunks = 8192;
  unsigned long long pub_off[kMaxChunks];  // owner: offset of chunk c in its HBM pool
  unsigned int pub_epoch[kMaxChunks];      // owner: access count at which pub_off is valid
  unsigned int cnt[kMaxChunks];            // peers: reads of chunk c completed (N-1 per access)
  unsigned int gpub;                       // owner: backward accesses whose gradient view is ready
  unsigned int gcnt;                       // peers: gradient pulls completed (N-1 per backward access)
};

constexpr int kMaxPeers = 8;
struct PeerTable {
  int world = 1, rank = 0;
  const std::uint8_t* pool[kMaxPeers];  // peers' HBM parameter pools (self included)
  const std::uint8_t* gview[kMaxPeers]; // peers' full-layer gradient views
  P2PCtl* ctl[kMaxPeers];               // peers' control blocks
  unsigned* scratch = nullptr;          // this rank's kMaxPeers + 1 zeroed completion counters
                                        // (per engine: two engines never share them)
};

// Owner side: publish chunk c at offset `off` of the pool for access `epoch`.
cudaError_t launch_p2p_publish(P2PCtl* ctl, std::uint32_t chunk, std::uint64_t off, std::uint32_t epoch,
                               cudaStream_t st);
// Owner side: gradient view of backward access `gepoch` is ready.
cudaError_t launch_p2p_publish_grad(P2PCtl* ctl, std::uint32_t gepoch, cudaStream_t st);
// Fused all-gather + unpack: for every rank q, wait for q's publication of
// chunk c at `epoch`, copy its piece (pieces[q]: bytes, flat-layer offset)
// straight from q's pool into the local flat layer view, then count the read
// in q's control block.
cudaError_t launch_p2p_gather_unpack(const PeerTable& t, std::uint32_t chunk, std::uint32_t epoch,
                                     const std::uint64_t* piece_bytes, const std::uint64_t* piece_view_off,
                                     std::uint8_t* view, cudaStream_t st);
// Fused pack + reduce-scatter (pull): wait until every rank published its
// gradient view for backward access `gepoch`, sum (fp32, rank order) the
// pieces at [view_off, view_off+bytes) of all ranks' views, round once to
// bf16 into `grad` (S bytes; the rest zero), then count the pull in every
// peer's control block.
cudaError_t launch_p2p_pull_reduce(const PeerTable& t, std::uint32_t gepoch, std::uint64_t view_off,
                                   std::uint64_t bytes, std::uint64_t chunk_bytes, std::uint16_t* grad,
                                   cudaStream_t st);

}  // namespace tcb
