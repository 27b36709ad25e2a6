// The executor's building blocks as C-ABI primitives ("What
// the C-ABI layer must export"): size-class pools in HBM or pinned host
// memory, copy-engine copies, events, the NCCL collectives of the ZeRO-3
// exchange and the NVMe tier's queued file I/O. A host runtime that makes its
// own scheduling decisions (the reference's IPolicy, engine.hpp:52-71, driven
// by its own executor) composes these; tc_engine_* is the same machinery
// driven by this repo's executor. No CPU fallback: without a device every
// call that touches one returns TC_ECUDA.
#include <cstring>
#include <memory>

#include "executor.hpp"

using namespace tcb;

struct tc_pool {
  SlotPool pool;
  bool device = false;
  int dev = 0;
};

struct tc_comm {
  ncclComm_t comm = nullptr;
  int world = 1, rank = 0, device = 0;
};

struct tc_nvme {
  std::unique_ptr<StripedFile> file;
  std::unique_ptr<NvmeQueue> queue;
  std::uint64_t last = 0;  // jobs run in submission order: each starts after the previous one
};

namespace {

cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }
cudaEvent_t as_event(tc_event* e) { return reinterpret_cast<cudaEvent_t>(e); }

}  // namespace

extern "C" {

// ---------------------------------------------------------------- pools
int tc_pool_create(int device, const uint64_t* class_sizes, const uint32_t* counts, uint32_t n_classes,
                   tc_pool** out) {
  TC_GUARD({
    if (!out || (n_classes && (!class_sizes || !counts))) return set_error(TC_EARG, "tc_pool_create: null argument");
    auto p = std::make_unique<tc_pool>();
    for (uint32_t k = 0; k < n_classes; ++k) {
      if (class_sizes[k] == 0 || class_sizes[k] % 16) return set_error(TC_EARG, "tc_pool_create: class sizes must be non-zero multiples of 16");
      p->pool.plan(class_sizes[k], counts[k]);
    }
    p->device = device >= 0;
    p->dev = device >= 0 ? device : 0;
    int cur = 0;
    TCB_CK(cudaGetDevice(&cur));
    if (p->device) TCB_CK(cudaSetDevice(device));
    p->pool.allocate(p->device, p->dev);
    if (p->device) TCB_CK(cudaSetDevice(cur));
    *out = p.release();
    return TC_OK;
  })
}

void tc_pool_destroy(tc_pool* p) {
  if (!p) return;
  p->pool.release_memory();
  delete p;
}

int tc_pool_chunk(tc_pool* p, uint64_t size, uint32_t index, void** out) {
  TC_GUARD({
    if (!p || !out) return set_error(TC_EARG, "tc_pool_chunk: null argument");
    auto& cls = p->pool.classes();
    auto it = cls.find(size);
    if (it == cls.end() || index >= it->second.slots.size())
      return set_error(TC_EPOOL, "tc_pool_chunk: no chunk " + std::to_string(index) + " of class " + std::to_string(size));
    *out = it->second.slots[index].ptr;
    return TC_OK;
  })
}

uint64_t tc_pool_bytes(const tc_pool* p) { return p ? const_cast<tc_pool*>(p)->pool.bytes() : 0; }

// ---------------------------------------------------------------- copies
int tc_copy_h2d(void* dst, const void* src, uint64_t bytes, void* stream) {
  TC_GUARD({
    if ((!dst || !src) && bytes) return set_error(TC_EARG, "tc_copy_h2d: null pointer");
    TCB_CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, as_stream(stream)));
    return TC_OK;
  })
}

int tc_copy_d2h(void* dst, const void* src, uint64_t bytes, void* stream) {
  TC_GUARD({
    if ((!dst || !src) && bytes) return set_error(TC_EARG, "tc_copy_d2h: null pointer");
    TCB_CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, as_stream(stream)));
    return TC_OK;
  })
}

// ---------------------------------------------------------------- events
int tc_event_create(int timing, tc_event** out) {
  TC_GUARD({
    if (!out) return set_error(TC_EARG, "tc_event_create: null argument");
    cudaEvent_t e = nullptr;
    TCB_CK(cudaEventCreateWithFlags(&e, timing ? cudaEventDefault : cudaEventDisableTiming));
    *out = reinterpret_cast<tc_event*>(e);
    return TC_OK;
  })
}

void tc_event_destroy(tc_event* e) {
  if (e) cudaEventDestroy(as_event(e));
}

int tc_event_record(tc_event* e, void* stream) {
  TC_GUARD({
    if (!e) return set_error(TC_EARG, "null event");
    TCB_CK(cudaEventRecord(as_event(e), as_stream(stream)));
    return TC_OK;
  })
}

int tc_event_wait(void* stream, tc_event* e) {
  TC_GUARD({
    if (!e) return set_error(TC_EARG, "null event");
    TCB_CK(cudaStreamWaitEvent(as_stream(stream), as_event(e), 0));
    return TC_OK;
  })
}

int tc_event_query(tc_event* e, int* done) {
  TC_GUARD({
    if (!e || !done) return set_error(TC_EARG, "null argument");
    const cudaError_t q = cudaEventQuery(as_event(e));
    if (q == cudaErrorNotReady) {
      *done = 0;
      return TC_OK;
    }
    TCB_CK(q);
    *done = 1;
    return TC_OK;
  })
}

int tc_event_synchronize(tc_event* e) {
  TC_GUARD({
    if (!e) return set_error(TC_EARG, "null event");
    TCB_CK(cudaEventSynchronize(as_event(e)));
    return TC_OK;
  })
}

int tc_event_elapsed_ms(tc_event* start, tc_event* end, float* ms) {
  TC_GUARD({
    if (!start || !end || !ms) return set_error(TC_EARG, "null argument");
    TCB_CK(cudaEventElapsedTime(ms, as_event(start), as_event(end)));
    return TC_OK;
  })
}

// ---------------------------------------------------------------- NCCL
int tc_nccl_comm_create(const uint8_t id[128], int world, int rank, int device, tc_comm** out) {
  TC_GUARD({
    if (!id || !out || world < 1 || rank < 0 || rank >= world) return set_error(TC_EARG, "tc_nccl_comm_create: bad arguments");
    auto c = std::make_unique<tc_comm>();
    c->world = world;
    c->rank = rank;
    c->device = device;
    ncclUniqueId uid;
    std::memcpy(uid.internal, id, sizeof(uid.internal));
    TCB_CK(cudaSetDevice(device));
    nccl_check(nccl().CommInitRank(&c->comm, world, uid, rank), "ncclCommInitRank");
    *out = c.release();
    return TC_OK;
  })
}

void tc_nccl_comm_destroy(tc_comm* c) {
  if (!c) return;
  if (c->comm) {
    try {
      nccl().CommDestroy(c->comm);
    } catch (...) {
    }
  }
  delete c;
}

int tc_nccl_allgather(tc_comm* c, const void* send, void* recv, uint64_t bytes_per_rank, void* stream) {
  TC_GUARD({
    if (!c || ((!send || !recv) && bytes_per_rank)) return set_error(TC_EARG, "tc_nccl_allgather: null argument");
    nccl_check(nccl().AllGather(send, recv, bytes_per_rank, ncclUint8, c->comm, as_stream(stream)), "ncclAllGather");
    return TC_OK;
  })
}

int tc_nccl_reducescatter(tc_comm* c, const void* send, void* recv, uint64_t elems_per_rank, void* stream) {
  TC_GUARD({
    if (!c || ((!send || !recv) && elems_per_rank)) return set_error(TC_EARG, "tc_nccl_reducescatter: null argument");
    nccl_check(nccl().ReduceScatter(send, recv, elems_per_rank, ncclBfloat16, ncclSum, c->comm, as_stream(stream)),
               "ncclReduceScatter");
    return TC_OK;
  })
}

// ---------------------------------------------------------------- NVMe tier
int tc_nvme_open(const char* dir, uint64_t bytes, int files, int direct, int device, tc_nvme** out) {
  TC_GUARD({
    if (!out || !dir) return set_error(TC_EARG, "tc_nvme_open: null argument");
    auto f = std::make_unique<tc_nvme>();
    f->file = std::make_unique<StripedFile>(dir, bytes, files > 0 ? files : 1, direct != 0);
    f->queue = std::make_unique<NvmeQueue>(device, f->file.get());
    *out = f.release();
    return TC_OK;
  })
}

void tc_nvme_close(tc_nvme* f) {
  if (!f) return;
  try {
    f->queue->wait_all();
  } catch (...) {
  }
  delete f;
}

int tc_nvme_write(tc_nvme* f, uint64_t offset, const void* pinned_src, uint64_t bytes, tc_event* after,
                  uint64_t* job) {
  TC_GUARD({
    if (!f || !pinned_src) return set_error(TC_EARG, "tc_nvme_write: null argument");
    std::vector<cudaEvent_t> w;
    if (after) w.push_back(as_event(after));
    std::vector<std::uint64_t> prev;
    if (f->last) prev.push_back(f->last);
    f->last = f->queue->submit_write(pinned_src, bytes, offset, std::move(w), std::move(prev));
    if (job) *job = f->last;
    return TC_OK;
  })
}

int tc_nvme_read(tc_nvme* f, uint64_t offset, void* pinned_dst, uint64_t bytes, tc_event* after, uint64_t* job) {
  TC_GUARD({
    if (!f || !pinned_dst) return set_error(TC_EARG, "tc_nvme_read: null argument");
    std::vector<cudaEvent_t> w;
    if (after) w.push_back(as_event(after));
    std::vector<std::uint64_t> prev;
    if (f->last) prev.push_back(f->last);
    f->last = f->queue->submit_read(pinned_dst, bytes, offset, std::move(w), std::move(prev));
    if (job) *job = f->last;
    return TC_OK;
  })
}

int tc_nvme_wait(tc_nvme* f, uint64_t job) {
  TC_GUARD({
    if (!f) return set_error(TC_EARG, "null handle");
    f->queue->wait(job);
    f->queue->check();
    return TC_OK;
  })
}

int tc_nvme_stream_wait(tc_nvme* f, uint64_t job, void* stream) {
  TC_GUARD({
    if (!f) return set_error(TC_EARG, "null handle");
    f->queue->stream_wait(as_stream(stream), job);
    return TC_OK;
  })
}

}  // extern "C"
