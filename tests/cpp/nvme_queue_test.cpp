// NVMe tier job queue (csrc/exec/nvme_io.hpp NvmeQueue) under a random
// workload shaped like the executor's: reads and writes of 24 file extents
// (some split into several 16 MiB pieces), each job ordered `after` the
// previous jobs on its extent (as executor.cpp passes r.nvme_job), a quarter
// of them also gated on a CUDA event that completes late (a host callback
// sleeps on its stream) so the dispatcher runs jobs out of submission order.
// Checks: every read returns the bytes of the last write submitted before it
// on that extent (host-side wait(), and GPU-side stream_wait() followed by an
// H2D copy on that stream), done() never decreases and never passes an
// incomplete job, wait_upto covers everything, byte counters add up.
// Prints "ok". Needs a GPU.
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstring>
#include <random>
#include <thread>
#include <vector>

#include "nvme_io.hpp"

using tcb::NvmeQueue;
using tcb::StripedFile;

#define CK(x)                                                                      \
  do {                                                                             \
    cudaError_t e_ = (x);                                                          \
    if (e_ != cudaSuccess) {                                                       \
      std::printf("cuda error %s at line %d\n", cudaGetErrorString(e_), __LINE__); \
      return 10;                                                                   \
    }                                                                              \
  } while (0)
#define REQUIRE(c)                                             \
  do {                                                         \
    if (!(c)) {                                                \
      std::printf("failed: %s (line %d)\n", #c, __LINE__); \
      return 1;                                                \
    }                                                          \
  } while (0)

static void fill(std::uint8_t* p, std::uint64_t n, std::uint32_t tag) {
  auto* w = reinterpret_cast<std::uint32_t*>(p);
  for (std::uint64_t i = 0; i < n / 4; ++i) w[i] = tag * 2654435761u + static_cast<std::uint32_t>(i);
}
static bool check(const std::uint8_t* p, std::uint64_t n, std::uint32_t tag) {
  const auto* w = reinterpret_cast<const std::uint32_t*>(p);
  for (std::uint64_t i = 0; i < n / 4; ++i)
    if (w[i] != tag * 2654435761u + static_cast<std::uint32_t>(i)) return false;
  return true;
}
static void CUDART_CB late(void* ms) {
  std::this_thread::sleep_for(std::chrono::microseconds(reinterpret_cast<std::uintptr_t>(ms)));
}

int main(int argc, char** argv) {
  const std::string dir = argc > 1 ? argv[1] : "/tmp";
  CK(cudaSetDevice(0));
  constexpr int K = 24, RING = 48, OPS = 1500;
  std::vector<std::uint64_t> ext_off(K), ext_len(K);
  std::uint64_t total = 0;
  for (int k = 0; k < K; ++k) {
    ext_len[k] = (k % 6 == 0) ? (40ull << 20) + 4096 : (1ull << 20) * (1 + k % 5);  // some span 3 pieces
    ext_off[k] = total;
    total += ext_len[k] + 12288;  // extents not stripe-aligned
  }
  const std::uint64_t maxlen = 40ull << 20 | 4096;
  StripedFile file(dir, total, 4, false);
  NvmeQueue q(0, &file);
  std::vector<std::uint8_t*> buf(RING);
  std::vector<std::uint64_t> buf_job(RING, 0);
  for (auto& b : buf) CK(cudaHostAlloc(reinterpret_cast<void**>(&b), maxlen, cudaHostAllocDefault));
  std::uint8_t* dev = nullptr;
  CK(cudaMalloc(&dev, maxlen));
  cudaStream_t s_evt, s_copy;
  CK(cudaStreamCreateWithFlags(&s_evt, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&s_copy, cudaStreamNonBlocking));

  std::vector<std::uint32_t> tag(K, 0);  // tag of the last write submitted per extent (0 = never written)
  std::vector<std::uint64_t> last_write(K, 0);
  std::vector<std::vector<std::uint64_t>> reads_since(K);
  struct PendingRead {
    std::uint64_t seq;
    int buf, k;
    std::uint32_t tag;
    bool via_stream;
  };
  std::vector<PendingRead> pending;
  std::mt19937_64 rng(11);
  std::uint64_t wbytes = 0, rbytes = 0, last_done = 0;
  std::uint32_t next_tag = 1;
  int cursor = 0, stream_checks = 0, out_of_order_seen = 0;

  auto retire = [&](const PendingRead& r) -> int {
    if (r.via_stream) {
      CK(cudaStreamSynchronize(s_copy));
      std::vector<std::uint8_t> h(ext_len[r.k]);
      CK(cudaMemcpy(h.data(), dev, ext_len[r.k], cudaMemcpyDeviceToHost));
      REQUIRE(check(h.data(), ext_len[r.k], r.tag));
    } else {
      q.wait(r.seq);
      REQUIRE(check(buf[r.buf], ext_len[r.k], r.tag));
    }
    return 0;
  };

  for (int op = 0; op < OPS; ++op) {
    const int k = static_cast<int>(rng() % K);
    const int b = cursor;
    cursor = (cursor + 1) % RING;
    if (buf_job[b]) q.wait(buf_job[b]);  // the buffer's previous job is done before it is reused
    for (auto it = pending.begin(); it != pending.end();)
      if (it->buf == b) {
        if (int rc = retire(*it)) return rc;
        it = pending.erase(it);
      } else {
        ++it;
      }
    std::vector<cudaEvent_t> waits;
    if (rng() % 4 == 0) {  // gate on an event that completes late
      cudaEvent_t e;
      CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      CK(cudaLaunchHostFunc(s_evt, late, reinterpret_cast<void*>(static_cast<std::uintptr_t>(200 + rng() % 800))));
      CK(cudaEventRecord(e, s_evt));
      waits.push_back(e);
    }
    const bool write = tag[k] == 0 || rng() % 2 == 0;
    if (write) {
      const std::uint32_t t = next_tag++;
      fill(buf[b], ext_len[k], t);
      std::vector<std::uint64_t> after = reads_since[k];
      if (last_write[k]) after.push_back(last_write[k]);
#ifdef TC_TEST_DROP_ORDER  // mutation check: without the extent ordering the test must fail
      after.clear();
#endif
      const std::uint64_t seq = q.submit_write(buf[b], ext_len[k], ext_off[k], waits, after);
      last_write[k] = seq;
      reads_since[k].clear();
      tag[k] = t;
      buf_job[b] = seq;
      wbytes += ext_len[k];
    } else {
      std::memset(buf[b], 0xee, ext_len[k]);
      std::vector<std::uint64_t> after;
      if (last_write[k]) after.push_back(last_write[k]);
#ifdef TC_TEST_DROP_ORDER
      after.clear();
#endif
      const std::uint64_t seq = q.submit_read(buf[b], ext_len[k], ext_off[k], waits, after);
      reads_since[k].push_back(seq);
      buf_job[b] = seq;
      rbytes += ext_len[k];
      const bool via_stream = stream_checks < 40 && rng() % 8 == 0 && pending.empty();
      if (via_stream) {  // GPU-side wait, then the copy that consumes the bytes
        q.stream_wait(s_copy, seq);
        CK(cudaMemcpyAsync(dev, buf[b], ext_len[k], cudaMemcpyHostToDevice, s_copy));
        ++stream_checks;
      }
      pending.push_back({seq, b, k, tag[k], via_stream});
      if (via_stream) {
        if (int rc = retire(pending.back())) return rc;
        pending.pop_back();
      }
    }
    const std::uint64_t d = q.done();
    REQUIRE(d >= last_done);  // the watermark never moves back
    last_done = d;
    for (auto it = pending.begin(); it != pending.end();)  // below the watermark = complete: bytes in place
      if (it->seq <= d) {
        REQUIRE(check(buf[it->buf], ext_len[it->k], it->tag));
        it = pending.erase(it);
      } else {
        ++it;
      }
    if (d + 1 < q.submitted()) ++out_of_order_seen;
  }
  for (const auto& r : pending)
    if (int rc = retire(r)) return rc;
  q.wait_upto(q.submitted());
  REQUIRE(q.done() == q.submitted());
  REQUIRE(q.bytes_written() == wbytes && q.bytes_read() == rbytes);
  REQUIRE(stream_checks > 0);
  for (auto* b : buf) CK(cudaFreeHost(b));
  CK(cudaFree(dev));
  std::printf("ok %d stream-checked reads, %d ops with jobs in flight\n", stream_checks, out_of_order_seen);
  return 0;
}
