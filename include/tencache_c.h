/* b200-tencache C-ABI — the thin boundary between host code (C++ decision
 * engine, Python mirror, or any FFI) and the B200 data plane.
 *
 * The reference has no C ABI (its interface is C++: IPolicy, engine.hpp:52-74,
 * and the free functions of scheduler.hpp:73-111); SURVEY.md §8(b) fixes what
 * this layer must export. Each entry below cites the reference interface it
 * replaces or serves. All functions return 0 on success or a TC_E* code; the
 * message of the last failure on the calling thread is tc_last_error().
 * Exceptions never cross this boundary. There is no CPU fallback: a data-plane
 * call on a machine without a B200 fails with TC_ECUDA.
 */
#ifndef TENCACHE_C_H_
#define TENCACHE_C_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes: one per reference exception type ---- */
enum {
  TC_OK = 0,
  TC_EINTERNAL = 1,   /* std::logic_error incl. SchedulerError (scheduler.cpp:10-13) */
  TC_ECONFIG = 2,     /* ConfigError (types.hpp:30-33) */
  TC_EOOM = 3,        /* OomError (types.hpp:35-38) */
  TC_ETRACE = 4,      /* TraceError (trace.hpp:58-61) */
  TC_EPOOL = 5,       /* PoolError (bufpool.hpp:18-21) */
  TC_EARG = 6,        /* std::invalid_argument / domain_error / bad handle */
  TC_ECUDA = 7,       /* CUDA runtime failure (no reference counterpart) */
  TC_EIO = 8,         /* NVMe tier file I/O failure (no reference counterpart) */
  TC_ENCCL = 9,       /* NCCL failure (no reference counterpart) */
  TC_ERANGE = 10      /* output buffer too small: nothing lost, see tc_policy_call */
};

const char* tc_last_error(void);
const char* tc_version(void);

/* =================== decision engine (reference C++ API, host) ========== */
/* One TransferRequest (scheduler.hpp:20-33). flags: 1 via_cpu_staging,
 * 2 instant, 4 src_retains, 8 dst_has_copy, 16 blocking. Tiers 0 gpu 1 cpu
 * 2 nvme; kind 0 prefetch 1 evict 2 restore. */
typedef struct {
  uint32_t tensor_id;
  uint8_t src, dst, kind, flags;
  uint64_t size_bytes;
} tc_request;

typedef struct tc_policy tc_policy;

/* make_policy(trace, machine, config) + IPolicy::init (engine.hpp:62,73;
 * policies.cpp:33-93). machine_path "" = default_machine() (machine.cpp:24-40);
 * cfg_json keys: policy, thresholds_us, restore_overlap, batch_scale,
 * zero_lookahead_k, seed (engine.hpp:19-27). info = InitInfo
 * {gpu, cpu, nvme resident bytes, fp16_in_nvme_count} (engine.hpp:54-59). */
int tc_policy_create(const char* trace_path, const char* machine_path, const char* cfg_json, tc_policy** out,
                     uint64_t info[4]);
void tc_policy_destroy(tc_policy* p);

/* IPolicy hooks (engine.hpp:63-70): hook 0 on_step_begin(step), 1
 * on_step_end(step), 2 on_param_restore_point, 3 on_iteration_end,
 * 4 reset_iteration. *n = number of requests. If they do not fit (n > cap) the
 * call returns TC_ERANGE, writes none and keeps them in the handle: the policy
 * state has advanced, so fetch them with hook 5 (drain, no state change) and a
 * buffer of at least *n before any other hook. */
int tc_policy_call(tc_policy* p, int hook, uint32_t step, tc_request* out, size_t cap, size_t* n);

/* Pool views for buffer-assignment parity and the executor (bufpool.hpp:41-95):
 * which 0 gpu, 1 cpu (parameter cache), 2 cpu_opt. occupant per buffer id,
 * 0 = free, negative = GPU-designated. layout = (offset, size) per buffer id. */
int tc_policy_pool(const tc_policy* p, int which, int64_t* occupant, size_t cap, size_t* n);
int tc_policy_layout(const tc_policy* p, int which, uint64_t* offset_size, size_t cap, size_t* n);
/* Logical buffer id currently holding `tensor` in pool `which`, or -1. */
int64_t tc_policy_buffer_of(const tc_policy* p, int which, uint32_t tensor);
/* Number of steps / iterations of the trace and the index of the first
 * optimizer step (== steps when none): the engine call order of engine.cpp:363-431. */
int tc_policy_shape(const tc_policy* p, uint32_t* steps, uint32_t* iterations, uint32_t* first_opt_step);

/* run() (engine.hpp:78, engine.cpp:572-576): model-clock run; SimReport JSON
 * (exact rationals as "num/den") to report_path, event log JSONL to
 * events_path ("" = none). reference_guard != 0 applies run_reference's
 * 64-tensor guard (engine.hpp:81-83). */
int tc_run(const char* trace_path, const char* machine_path, const char* cfg_json, const char* report_path,
           const char* events_path, int reference_guard);
/* The policy call sequence of one run with pool contents after every call,
 * as JSON (same schema as the oracle's golden streams). */
int tc_decisions(const char* trace_path, const char* machine_path, const char* cfg_json, const char* out_path,
                 int with_pools);
/* sweep (engine.hpp:85-92, engine.cpp:334-384): one SimReport per value of
 * axis ("batch_scale" | "gpu_capacity" | "cpu_capacity" | "pinned"), in value
 * order, on `threads` threads; a JSON array of reports to out_path. */
int tc_sweep(const char* trace_path, const char* machine_path, const char* cfg_json, const char* axis,
             const double* values, uint32_t n, uint32_t threads, const char* out_path);
/* synthesize_transformer_trace + save_trace (trace.hpp:76-87). */
int tc_synthesize(uint32_t layers, uint32_t tensors_per_layer, const uint64_t* sizes, int nsizes,
                  double compute_us_per_byte, uint64_t seed, uint32_t iterations, double opt_us_per_byte,
                  int optimizer_steps, const char* out_path);
int tc_trace_roundtrip(const char* in_path, const char* out_path);
/* transfer_time_us (machine.cpp:101-111) as an exact "num/den" string. */
int tc_transfer_time(const char* machine_path, int src, int dst, uint64_t bytes, char* out, size_t out_len);
/* Wall-clock cost of the host decision path: init and one iteration of
 * policy calls (ns), averaged over `iterations`. */
int tc_time_decisions(const char* trace_path, const char* machine_path, const char* cfg_json, int iterations,
                      double* ns_per_iteration, double* init_ns);
int tc_time_run(const char* trace_path, const char* machine_path, const char* cfg_json, int repeats,
                double* ns_per_run);

/* ========================= data plane: sm_100a kernels ================== */
/* All pointers are device pointers unless stated; `stream` is a cudaStream_t
 * (NULL = legacy default). Kernels are asynchronous. */

/* A fragment: `bytes` at src_base+src_off <-> dst_base+dst_off. */
typedef struct {
  uint64_t src_off;
  uint64_t dst_off;
  uint64_t bytes;
} tc_segment;

/* pack / unpack of fragmented tensors into one pooled chunk.
 * A plan uploads the fragment list (host array) once to HBM with each
 * fragment's position in the concatenated stream; pack then moves every
 * fragment src_base+src_off -> dst_base+dst_off in ONE launch, and unpack is
 * the inverse (src_base+dst_off -> dst_base+src_off). Fragments must not
 * overlap at the destination. */
typedef struct tc_pack_plan tc_pack_plan;
int tc_pack_plan_create(const tc_segment* host_segs, uint32_t n, tc_pack_plan** out);
void tc_pack_plan_destroy(tc_pack_plan* plan);
uint64_t tc_pack_plan_bytes(const tc_pack_plan* plan);
int tc_pack(const tc_pack_plan* plan, const void* src_base, void* dst_base, void* stream);
int tc_unpack(const tc_pack_plan* plan, const void* src_base, void* dst_base, void* stream);

/* bf16 <-> fp32 casts (RNE, NaN -> quiet NaN; torch .to() semantics). */
int tc_cast_bf16_to_f32(const void* in, float* out, uint64_t n, void* stream);
int tc_cast_f32_to_bf16(const float* in, void* out, uint64_t n, void* stream);

/* Fused AdamW on one optimizer-state chunk (the offloaded optimizer step the
 * reference models as a timed no-op; trace.hpp:72-74 sizes it at
 * 6x the bf16 parameter bytes). state = [p32 | m | v], n elements each,
 * fp32; grad = bf16; param_out = bf16 copy of the updated p32 (may be NULL).
 * lr/b1/b2/eps/wd/step as torch.optim.AdamW; grad_scale multiplies g. */
int tc_adamw(float* state, const void* grad, void* param_out, uint64_t n, double lr, double beta1, double beta2,
             double eps, double weight_decay, int64_t step, float grad_scale, void* stream);
/* Same update with p32/m/v at independent addresses. */
int tc_adamw_split(float* p32, float* m, float* v, const void* grad, void* param_out, uint64_t n, double lr,
                   double beta1, double beta2, double eps, double weight_decay, int64_t step, float grad_scale,
                   void* stream);
/* Up to 8 chunks updated in ONE launch (same hyper-parameters and step; each
 * chunk's n a multiple of 8 with 16-byte aligned pointers, else TC_EARG):
 * what the executor uses for consecutive hoisted updates, so k chunks pay one
 * launch's front-end latency instead of k. state = [p32 | m | v] of n each. */
typedef struct {
  float* state;
  const void* grad;
  void* param_out;
  uint64_t n;
} tc_adam_chunk;
int tc_adamw_batch(const tc_adam_chunk* chunks, uint32_t count, double lr, double beta1, double beta2, double eps,
                   double weight_decay, int64_t step, float grad_scale, void* stream);
/* Packed split-master optimizer state (what the engine keeps on the host for
 * a parameter that never lives in NVMe), n % 2048 == 0, in the state's own
 * 12n-byte buffer: a prefix of tc_split_state_bytes(n) = 9.44 n bytes (what
 * crosses PCIe) and a 2n-byte overflow area behind it.
 *  - fp32 master: its low 16 bits + one round bit rb_i; the high half is the
 *    bf16 parameter B minus rb_i (for a NaN B: B with its quiet bit cleared
 *    when rb_i is set) -- exact for every fp32 value, because the update
 *    writes B = RNE(master) itself;
 *  - m, v: bytes 0-2 as stored; byte 3 (sign + top 7 exponent bits) coded
 *    against the largest top-7 value of each 32-element group (m: sign +
 *    4-bit offset, v: 5-bit offset, each with a code for zero and one for
 *    an escape); an escaped element's byte 3 lives in the overflow area.
 * Lossless for every bit pattern. tc_adamw_split_master updates such a state
 * in place, reading the current `param` (bf16, n) and writing the new one;
 * results are bit-identical to tc_adamw on the expanded state. */
uint64_t tc_split_state_bytes(uint64_t n);
int tc_adamw_split_master(void* split_state, const void* grad, void* param, uint64_t n, double lr, double beta1,
                          double beta2, double eps, double weight_decay, int64_t step, float grad_scale,
                          void* stream);
/* Codec between the packed split (12n bytes) and the full [p32|m|v] layouts
 * (device buffers, out of place). compress sets *d_mismatch (a device u32,
 * never cleared) to nonzero when some p32 does not round to its bf16 param:
 * not representable split. */
int tc_state_expand(const void* split_state, const void* param, float* full_state, uint64_t n, void* stream);
int tc_state_compress(const float* full_state, const void* param, void* split_state, uint64_t n,
                      uint32_t* d_mismatch, void* stream);
/* The 8 fp32 scalars the update uses, for parity tests. */
int tc_adamw_scalars(double lr, double beta1, double beta2, double eps, double weight_decay, int64_t step,
                     float out[8]);

/* Checksum of `bytes` (multiple of 4) at `data`: sum of u32 word * (2i+1)
 * mod 2^64, accumulated into *out (device u64). The forward/backward
 * stand-in reads every migrated byte through this. */
int tc_checksum(const void* data, uint64_t bytes, uint64_t* out, void* stream);
/* Deterministic N(0, sigma) bf16 fill (counter-based RNG keyed by seed and
 * stream_id) — the generator the engine seeds parameters and the backward
 * stand-in's gradients with; exposed so tests can regenerate them. */
int tc_fill_normal_bf16(void* out, uint64_t n, float sigma, uint64_t seed, uint64_t stream_id, void* stream);
/* Busy the compute stream for `us` microseconds on `ctas` CTAs (the layer
 * compute stand-in; trace compute_us, trace.hpp:38). */
int tc_spin(double us, int ctas, void* stream);

/* =========== executor building blocks (SURVEY.md §8(b) primitives) ====== */
/* What a host runtime with its own executor composes (the reference's
 * decisions, engine.hpp:52-71 / scheduler.hpp:20-33, turned into data
 * movement); tc_engine_* below is the same machinery driven by this repo's
 * executor. */

/* A region carved into size classes like the policy's BufferPool
 * (bufpool.cpp:47-66): classes in ascending size, chunks of a class back to
 * back. device >= 0: HBM of that device; device < 0: pinned host memory
 * (transparent huge pages + cudaHostRegister, portable). Class sizes are
 * non-zero multiples of 16 (TC_EARG). */
typedef struct tc_pool tc_pool;
int tc_pool_create(int device, const uint64_t* class_sizes, const uint32_t* counts, uint32_t n_classes,
                   tc_pool** out);
void tc_pool_destroy(tc_pool* p);
/* Address of chunk `index` of class `size` (TC_EPOOL: no such chunk, the
 * reference's PoolError UnknownSizeClass, bufpool.hpp:18-21). */
int tc_pool_chunk(tc_pool* p, uint64_t size, uint32_t index, void** out);
uint64_t tc_pool_bytes(const tc_pool* p);

/* Copy-engine copies between pinned host memory and HBM on `stream`. */
int tc_copy_h2d(void* dst, const void* src, uint64_t bytes, void* stream);
int tc_copy_d2h(void* dst, const void* src, uint64_t bytes, void* stream);

/* Events: the ordering primitive between copy streams and compute. */
typedef struct tc_event tc_event;
int tc_event_create(int timing, tc_event** out);
void tc_event_destroy(tc_event* e);
int tc_event_record(tc_event* e, void* stream);
int tc_event_wait(void* stream, tc_event* e);  /* `stream` waits for `e` */
int tc_event_query(tc_event* e, int* done);
int tc_event_synchronize(tc_event* e);
int tc_event_elapsed_ms(tc_event* start, tc_event* end, float* ms);

/* The ZeRO-3 exchange's collectives: all-gather of each
 * rank's bytes, reduce-scatter (sum) of bf16 gradients. The id comes from
 * tc_nccl_unique_id on one rank, broadcast by the caller. */
typedef struct tc_comm tc_comm;
int tc_nccl_comm_create(const uint8_t id[128], int world, int rank, int device, tc_comm** out);
void tc_nccl_comm_destroy(tc_comm* c);
int tc_nccl_allgather(tc_comm* c, const void* send, void* recv, uint64_t bytes_per_rank, void* stream);
int tc_nccl_reducescatter(tc_comm* c, const void* send, void* recv, uint64_t elems_per_rank, void* stream);

/* The NVMe tier: one logical byte range over `files` files (16 MiB stripes),
 * O_DIRECT when `direct` (offsets, sizes and buffers 4 KiB-aligned), reached
 * through pinned bounce buffers (the staging slot of engine.cpp:214-221).
 * Jobs run in submission order on a worker pool; a job may first wait for
 * `after` (e.g. the D2H copy that filled the bounce buffer). *job identifies
 * it for tc_nvme_wait (host) / tc_nvme_stream_wait (a GPU stream waits, no
 * host thread blocks). A failed job fails tc_nvme_wait with TC_EIO. */
typedef struct tc_nvme tc_nvme;
int tc_nvme_open(const char* dir, uint64_t bytes, int files, int direct, int device, tc_nvme** out);
void tc_nvme_close(tc_nvme* f);
int tc_nvme_write(tc_nvme* f, uint64_t offset, const void* pinned_src, uint64_t bytes, tc_event* after,
                  uint64_t* job);
int tc_nvme_read(tc_nvme* f, uint64_t offset, void* pinned_dst, uint64_t bytes, tc_event* after, uint64_t* job);
int tc_nvme_wait(tc_nvme* f, uint64_t job);
int tc_nvme_stream_wait(tc_nvme* f, uint64_t job, void* stream);

/* ====================== migration executor (real mode) ================= */
/* A per-GPU engine: pinned host pools and an HBM pool carved exactly like the
 * policy's BufferPools (bufpool.cpp:47-66), dedicated H2D/D2H streams,
 * per-slot events, and an NVMe tier staged through pinned bounce buffers.
 * It replays the policy's TransferRequests (scheduler.hpp:20-33) as
 * copy-engine work ordered against a compute stream. */
typedef struct tc_engine tc_engine;

typedef struct {
  int device;              /* CUDA device ordinal */
  const char* nvme_dir;    /* directory for the NVMe tier file ("" = none) */
  int gpu_spare_slots;     /* extra HBM slots per class beyond the policy tier (in-flight moves; default 16) */
  int host_spare_slots;    /* extra pinned slots per class */
  int opt_stage_slots;     /* HBM staging buffers for the optimizer pipeline; <= 0: sized from the
                              forward pass's spare H2D time (at least 12) */
  int direct_io;           /* O_DIRECT for the NVMe tier */
  uint64_t grad_bytes_per_param_byte; /* gradient bytes per bf16 param byte (1) */
  int full_master;         /* nonzero: host optimizer states keep the whole fp32 master (12 B/param each
                              way). 0 (default): a state whose parameter never leaves HBM keeps only the
                              master's low half + a round bit on the host (10.125 B/param each way): the
                              high half is the parameter's bf16 value, which the update rounds from it.
                              Lossless; states read/written through tc_engine_read/write_tensor in the
                              full [p32|m|v] layout either way. */
} tc_engine_options;

int tc_engine_create(const char* trace_path, const char* machine_path, const char* cfg_json,
                     const tc_engine_options* opts, tc_engine** out);
void tc_engine_destroy(tc_engine* e);

/* Fill every tensor's home copy with deterministic data (seeded), zero the
 * optimizer moments, and put the engine at the start of an iteration. */
int tc_engine_seed(tc_engine* e, uint64_t seed);

/* Host-side copies of a tensor, wherever it currently lives (for tests and the
 * end-to-end API): read into / write from a HOST buffer of its size. */
int tc_engine_read_tensor(tc_engine* e, uint32_t tensor, void* host_dst, uint64_t bytes);
int tc_engine_write_tensor(tc_engine* e, uint32_t tensor, const void* host_src, uint64_t bytes);
/* Host copy of a parameter's bf16 gradient (HBM). */
int tc_engine_read_grad(tc_engine* e, uint32_t tensor, void* host_dst, uint64_t bytes);
/* Device pointer of the tensor's current GPU slot (NULL if not GPU-resident).
 * Parameter bytes behind it are the high halves of split-master states
 * (tc_engine_options.full_master): write them through tc_engine_write_tensor,
 * or create the engine with full_master = 1 to write them in place. */
void* tc_engine_gpu_ptr(tc_engine* e, uint32_t tensor);
/* Gradient buffer (bf16, on GPU) of a parameter tensor. */
void* tc_engine_grad_ptr(tc_engine* e, uint32_t tensor);
/* The engine's HBM parameter pool (every GPU slot tc_engine_gpu_ptr and
 * tc_engine_step_begin return lies inside it) and its gradient region (every
 * tc_engine_grad_ptr), so a framework can alias them once as tensors and
 * slice per step instead of wrapping raw pointers every step. */
int tc_engine_regions(tc_engine* e, void** hbm_pool, uint64_t* hbm_pool_bytes, void** grads, uint64_t* grad_bytes);

typedef struct {
  double lr, beta1, beta2, eps, weight_decay;
  float grad_scale;
  int compute_mode;    /* 0: checksum only, 1: checksum + a 1-CTA spin for compute_us*batch_scale,
                          2: checksum + bf16 tensor-core GEMMs over the migrated chunk that occupy the
                             GPU for compute_us*batch_scale (cuBLAS; tc_engine_standin_info) */
  int spin_ctas;
  int flags;           /* bit 0: run optimizer updates in place (no hoisting after the last access);
                          bit 1: no pre-staging of optimizer states ahead of their updates;
                          bit 2: last iteration: no prologue of the next one (its decisions and
                                 first state loads are otherwise enqueued at the end of this call) */
} tc_step_options;

/* One training iteration: every trace step in order, policy decisions at the
 * engine's fixed call points (engine.cpp:363-431), transfers on the copy
 * streams, the fwd/bwd stand-in and the fused AdamW on the compute stream.
 * Asynchronous w.r.t. the host only where CUDA allows; returns after
 * enqueueing (call tc_engine_sync to wait). */
int tc_engine_iteration(tc_engine* e, const tc_step_options* so, void* compute_stream);
int tc_engine_sync(tc_engine* e);

/* Per-step execution driven by a training loop: the same iteration, but the
 * caller computes each forward/backward step on `compute_stream` between
 * step_begin and step_end, at the reference engine's call points
 * (engine.cpp:119-131 on_step_begin, :157-168 on_step_end, :170-187 restore
 * point / iteration end / reset; PAPER.md:599 drives them from module hooks).
 *
 *   tc_engine_iteration_begin(e, so, stream)      decisions of the iteration,
 *                                                 optimizer pre-staging
 *   for step i in trace order:
 *     tc_engine_step_begin(e, i, ptrs, cap, &n)   [restore point,] on_step_begin's
 *                                                 moves; `stream` is ordered after
 *                                                 the step tensors' arrivals;
 *                                                 ptrs[k] = HBM address of the
 *                                                 step's k-th tensor (fwd/bwd
 *                                                 steps; n = 0 for optimizer steps)
 *     ... caller's kernels on `stream` read the chunks; a backward step
 *         writes each parameter's bf16 gradient at tc_engine_grad_ptr ...
 *     tc_engine_step_end(e, i)                    the chunks are released to the
 *                                                 policy after the caller's work;
 *                                                 a backward step's gradients are
 *                                                 final: the fused AdamW of every
 *                                                 update hoisted behind it runs
 *                                                 (after the gradient lands);
 *                                                 on_step_end's moves
 *   tc_engine_iteration_end(e)                    remaining restore point,
 *                                                 on_iteration_end, reset
 *
 * Steps run exactly once each, in order (TC_EARG otherwise, nothing done).
 * so->compute_mode 0 also checksums every accessed chunk (tc_engine_step_result);
 * 3 = the caller's compute only. The engine's own stand-ins (modes 1, 2) do
 * not run. A backward step's gradient writes are ordered after the previous
 * update that read them. With a ZeRO-3 exchange every forward/backward step
 * accesses one layer's chunks: step_begin all-gathers the layer into a flat
 * view (tc_engine_zero3_views), a backward step's caller writes the
 * full-layer gradient into the gradient view, and step_end sums it over the
 * ranks into this rank's gradient chunks before their updates.
 * tc_engine_step_begin with too small a `ptrs` returns TC_ERANGE with the step
 * open (*n = its tensor count; read the addresses with tc_engine_gpu_ptr). */
int tc_engine_iteration_begin(tc_engine* e, const tc_step_options* so, void* compute_stream);
int tc_engine_step_begin(tc_engine* e, uint32_t step, void** ptrs, size_t cap, size_t* n);
int tc_engine_step_end(tc_engine* e, uint32_t step);
int tc_engine_iteration_end(tc_engine* e);
/* Give up an open iteration (the caller's step failed): the remaining moves
 * still run so placement and the next iteration's decisions stay consistent;
 * updates not yet run are skipped. No-op when no iteration is open. */
int tc_engine_iteration_abort(tc_engine* e);

/* Counters of the last iteration(s) since the previous reset_stats. */
typedef struct {
  uint64_t h2d_bytes, d2h_bytes;         /* cache-decision bytes over PCIe (category i) */
  uint64_t opt_h2d_bytes, opt_d2h_bytes; /* optimizer round trip (category ii) */
  uint64_t writeback_bytes;              /* updated-param write-back (category iii) */
  uint64_t nvme_read_bytes, nvme_write_bytes; /* category iv */
  uint64_t param_accesses, param_hits;   /* engine_internal.hpp:98-102 definition */
  uint64_t ontime_accesses;              /* prefetched accesses already landed */
  uint64_t requests, kernel_launches, copies;
  double h2d_busy_ms, d2h_busy_ms;       /* copy-engine busy time (event pairs) */
  double stall_ms;                       /* compute stream waiting on copies */
  double adam_ms;                        /* fused AdamW kernel time (CUDA events on its stream) */
  uint64_t adam_elems;
  double adam_span_ms;                   /* AdamW resident time: first CTA start to last CTA end */
  uint64_t adam_spans;                   /* launches measured in adam_span_ms */
  uint64_t adam_launches;                /* fused AdamW kernel launches (one may cover several chunks) */
  uint64_t compute_gemms;                /* stand-in GEMM launches (compute_mode 2) */
  double compute_flops;                  /* stand-in GEMM FLOPs issued */
  uint64_t split_updates;                /* updates of states held split (full_master = 0) */
  uint64_t split_elems;                  /* ... their elements (part of adam_elems) */
  uint64_t opt_logical_bytes;            /* optimizer round trip in the full 12 B/param layout, both ways */
} tc_engine_stats;

int tc_engine_stats_get(tc_engine* e, tc_engine_stats* out);
/* compute_mode 2's GEMM shape and calibrated alone-throughput, as JSON (after
 * the first iteration in that mode; "{}" before). */
int tc_engine_standin_info(tc_engine* e, char* out, size_t cap);
int tc_engine_stats_reset(tc_engine* e);
/* Compute-stream phase durations of the last iteration (ms): forward,
 * backward, optimizer (+ drain of all streams). */
int tc_engine_phase_ms(tc_engine* e, double* out, size_t cap, size_t* n);
/* checksum the fwd/bwd stand-in computed for each parameter access of the
 * last iteration (device -> host copy), in access order. */
int tc_engine_access_checksums(tc_engine* e, uint64_t* out, size_t cap, size_t* n);
/* The step's result without draining: the per-access checksums of the most
 * recently enqueued iteration, copied to pinned host memory at the end of its
 * compute stream. Waits only for that iteration's forward/backward, so its
 * optimizer write-back tail keeps overlapping the next iteration (what a
 * training loop's loss.item() waits for). out == NULL or cap == 0: only
 * sets *n (no wait). TC_EARG before any iteration. */
int tc_engine_step_result(tc_engine* e, uint64_t* out, size_t cap, size_t* n);

/* ===================== ZeRO-3 exchange ================= */
/* NCCL (libnccl.so.2 loaded at run time) unique id, to be broadcast by the
 * caller (e.g. torch.distributed) before tc_engine_enable_zero3. */
int tc_nccl_unique_id(uint8_t out[128]);
/* Switch the engine's parameter accesses to ZeRO-3: every forward/backward
 * access all-gathers the chunk from all ranks and unpacks it into the flat
 * layer view; every backward access packs the full-layer gradient and
 * reduce-scatters it (sum) into this rank's gradient chunk. layer_elems[l] =
 * flat bf16 elements of trace layer l, layer_per[l] = elements per rank
 * (ceil). Chunks of one layer are its parameter tensors in id order. */
int tc_engine_enable_zero3(tc_engine* e, int world, int rank, const uint8_t id[128], const uint64_t* layer_elems,
                           const uint64_t* layer_per, uint32_t n_layers);
/* Measured event log: for every harvested iteration, one JSONL line per copy
 * in the reference's event-log schema (engine_internal.hpp:35-47: us, kind,
 * tensor, src, dst) plus end_us, bytes and iter from CUDA events, and a
 * "stall" line (wait_us) per compute-stream wait. path "" switches it off. */
int tc_engine_event_log(tc_engine* e, const char* path);
/* Fused ZeRO-3 exchange over peer memory (no NCCL): after
 * tc_engine_enable_zero3 (an all-zero id skips the NCCL communicator), every
 * rank exports its IPC handles (HBM pool, control block, gradient view; `n`
 * bytes), the caller all-gathers them rank-major, and tc_engine_enable_p2p
 * maps the peers. Accesses then run one gather+unpack kernel and, backward,
 * one pull-reduce kernel that read the peers' HBM directly. */
int tc_engine_p2p_handles(tc_engine* e, uint8_t* out, size_t cap, size_t* n);
/* ZeRO-3 per-step execution, between tc_engine_step_begin and step_end of a
 * forward/backward step: the gathered layer (flat bf16, the layer table's
 * elements, *layer_bytes = 2 x elements; read-only) and the gradient view of
 * the same layout the caller writes in a backward step (its contents are
 * undefined at step_begin: zero it before accumulating). Both are device
 * memory, valid until step_end; write/read them on the compute stream.
 * TC_EARG outside such a step, TC_ECONFIG without a ZeRO-3 exchange. The
 * ranks run the same steps in the same order (the exchange pairs them). */
int tc_engine_zero3_views(tc_engine* e, void** params, void** grads, uint64_t* layer_bytes);
int tc_engine_enable_p2p(tc_engine* e, const uint8_t* all_blobs);
/* Bytes all-gathered + reduce-scattered (NCCL payload, all ranks' pieces) so far. */
uint64_t tc_engine_exchanged_bytes(tc_engine* e);
/* GPUDirect Storage for the NVMe tier: 1 when the
 * nvidia-fs driver is present and cuFile opened (never probed otherwise: in
 * its compatibility mode cuFile is a bounce-buffer copy, and on boxes without
 * the driver cuFileDriverOpen may not return); `why` (may be NULL) gets the
 * reason when 0. TC_GDS=0 disables it. An engine created with direct_io = 1
 * moves NVMe tier bytes file <-> HBM with it when available
 * (tc_engine_gds), else through the pinned bounce buffers. */
int tc_gds_available(char* why, size_t cap);
int tc_engine_gds(tc_engine* e);

#ifdef __cplusplus
}
#endif

#endif /* TENCACHE_C_H_ */
