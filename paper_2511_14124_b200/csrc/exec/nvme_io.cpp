#include "nvme_io.hpp"

#include <cuda.h>
#include <fcntl.h>
#include <unistd.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>

#include "capi_common.hpp"

namespace tcb {

namespace {
using WaitValue32 = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
}

void stream_wait_value32(cudaStream_t s, const unsigned* dev_addr, unsigned value) {
  static WaitValue32 fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    return reinterpret_cast<WaitValue32>(f);
  }();
  if (fn == nullptr) throw DeviceError(TC_ECUDA, "cuStreamWaitValue32 unavailable");
  if (fn(reinterpret_cast<CUstream>(s), reinterpret_cast<CUdeviceptr>(dev_addr), value, CU_STREAM_WAIT_VALUE_GEQ) !=
      CUDA_SUCCESS)
    throw DeviceError(TC_ECUDA, "cuStreamWaitValue32 failed");
}

StripedFile::StripedFile(const std::string& dir, std::uint64_t bytes, int files, bool direct) {
  files = std::max(1, files);
  const std::uint64_t stripes = (bytes + kStripe - 1) / kStripe;
  const std::uint64_t per_file = ((stripes + files - 1) / files) * kStripe;
  for (int k = 0; k < files; ++k) {
    std::string path = dir + "/tencache_nvme_XXXXXX";
    std::vector<char> tmpl(path.begin(), path.end());
    tmpl.push_back(0);
    const int fd = mkstemp(tmpl.data());
    if (fd < 0) throw DeviceError(TC_EIO, "cannot create NVMe tier file in " + dir);
    unlink(tmpl.data());
    fds_.push_back(fd);
    if (direct) fcntl(fd, F_SETFL, fcntl(fd, F_GETFL) | O_DIRECT);
    if (ftruncate(fd, static_cast<off_t>(per_file)) != 0) throw DeviceError(TC_EIO, "ftruncate NVMe tier file");
  }
}

StripedFile::~StripedFile() {
  for (int fd : fds_) close(fd);
}

bool StripedFile::io(bool write, std::uint8_t* buf, std::uint64_t bytes, std::uint64_t off) const {
  const std::uint64_t k = fds_.size();
  while (bytes) {
    const std::uint64_t stripe = off / kStripe, in = off % kStripe;
    const std::uint64_t len = std::min(bytes, kStripe - in);
    const int fd = fds_[stripe % k];
    const std::uint64_t foff = (stripe / k) * kStripe + in;
    for (std::uint64_t done = 0; done < len;) {
      const ssize_t r = write ? pwrite(fd, buf + done, len - done, static_cast<off_t>(foff + done))
                              : pread(fd, buf + done, len - done, static_cast<off_t>(foff + done));
      if (r <= 0) return false;
      done += static_cast<std::uint64_t>(r);
    }
    buf += len;
    off += len;
    bytes -= len;
  }
  return true;
}

NvmeQueue::NvmeQueue(int device, const StripedFile* file) : device_(device), file_(file) {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &fn, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess || fn == nullptr)
    throw DeviceError(TC_ECUDA, "cuStreamWaitValue32 unavailable");
  wait_fn_ = fn;
  void* h = nullptr;
  if (cudaHostAlloc(&h, 64, cudaHostAllocMapped | cudaHostAllocPortable) != cudaSuccess)
    throw DeviceError(TC_ECUDA, "cannot allocate the NVMe completion word");
  flag_ = static_cast<volatile std::uint32_t*>(h);
  *flag_ = 0;
  if (cudaHostGetDevicePointer(&flag_dev_, h, 0) != cudaSuccess)
    throw DeviceError(TC_ECUDA, "cannot map the NVMe completion word");
  // probe once: a satisfied wait must be accepted by this driver/device
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  const CUresult r = reinterpret_cast<WaitValue32>(wait_fn_)(reinterpret_cast<CUstream>(s),
                                                            reinterpret_cast<CUdeviceptr>(flag_dev_), 0,
                                                            CU_STREAM_WAIT_VALUE_GEQ);
  cudaStreamSynchronize(s);
  cudaStreamDestroy(s);
  if (r != CUDA_SUCCESS) {
    cudaFreeHost(h);
    throw DeviceError(TC_ECUDA, "stream memory operations unsupported");
  }
  dispatcher_ = std::thread([this] { dispatch(); });
  const char* env = std::getenv("TC_NVME_THREADS");
  const int nw = env ? std::max(1, std::atoi(env)) : 16;
  for (int i = 0; i < nw; ++i) workers_.emplace_back([this] { work(); });
}

NvmeQueue::~NvmeQueue() {
  {
    std::lock_guard<std::mutex> g(mu_);
    stop_ = true;
  }
  cv_.notify_all();
  piece_cv_.notify_all();
  if (dispatcher_.joinable()) dispatcher_.join();
  for (auto& w : workers_)
    if (w.joinable()) w.join();
  if (flag_) cudaFreeHost(const_cast<std::uint32_t*>(flag_));
}

static const bool kDebug = std::getenv("TC_NVME_DEBUG") != nullptr;

std::uint64_t NvmeQueue::submit(Job j) {
  std::lock_guard<std::mutex> g(mu_);
  if (!error_.empty()) throw DeviceError(TC_EIO, error_);
  j.seq = ++submitted_;
  if (kDebug)
    std::fprintf(stderr, "[nvme] submit %llu %s %llu B @%llu waits=%zu\n", static_cast<unsigned long long>(j.seq),
                 j.write ? "W" : "R", static_cast<unsigned long long>(j.bytes), static_cast<unsigned long long>(j.off),
                 j.waits.size());
  (j.write ? bytes_written_ : bytes_read_) += j.bytes;
  q_.push_back(std::move(j));
  cv_.notify_one();
  return submitted_;
}

std::uint64_t NvmeQueue::submit_read(void* dst, std::uint64_t bytes, std::uint64_t off, std::vector<cudaEvent_t> w,
                                     std::uint64_t after) {
  return submit(Job{false, dst, bytes, off, 0, std::move(w), after});
}

std::uint64_t NvmeQueue::submit_write(const void* src, std::uint64_t bytes, std::uint64_t off,
                                      std::vector<cudaEvent_t> w, std::uint64_t after) {
  return submit(Job{true, const_cast<void*>(src), bytes, off, 0, std::move(w), after});
}

void NvmeQueue::stream_wait(cudaStream_t s, std::uint64_t seq) {
  if (seq == 0 || seq <= done()) return;
  const CUresult r = reinterpret_cast<WaitValue32>(wait_fn_)(
      reinterpret_cast<CUstream>(s), reinterpret_cast<CUdeviceptr>(flag_dev_), static_cast<cuuint32_t>(seq),
      CU_STREAM_WAIT_VALUE_GEQ);
  if (r != CUDA_SUCCESS) throw DeviceError(TC_ECUDA, "cuStreamWaitValue32 failed");
}

std::string NvmeQueue::describe() {
  std::lock_guard<std::mutex> g(mu_);
  std::string s = "nvme queue: submitted " + std::to_string(submitted_) + " done " + std::to_string(done_) +
                  " flag " + std::to_string(*flag_) + " queued " + std::to_string(q_.size()) + " pieces " +
                  std::to_string(pieces_.size()) + " dispatching " + std::to_string(dispatching_) + " phase " +
                  std::to_string(dispatch_phase_) + " open:";
  int k = 0;
  for (const auto& [seq, left] : remaining_) {
    if (k++ > 8) break;
    s += " " + std::to_string(seq) + "(" + std::to_string(static_cast<int>(left)) + ")";
  }
  return s;
}

void NvmeQueue::wait(std::uint64_t seq) {
  if (kDebug) std::fprintf(stderr, "[nvme] host wait %llu\n", static_cast<unsigned long long>(seq));
  std::unique_lock<std::mutex> g(mu_);
  while (!done_cv_.wait_for(g, std::chrono::seconds(30), [&] { return done_ >= seq || !error_.empty(); })) {
    g.unlock();
    std::fprintf(stderr, "[nvme] still waiting for job %llu: %s\n", static_cast<unsigned long long>(seq),
                 describe().c_str());
    g.lock();
  }
  if (!error_.empty()) throw DeviceError(TC_EIO, error_);
}

std::uint64_t NvmeQueue::done() const {
  std::lock_guard<std::mutex> g(const_cast<std::mutex&>(mu_));
  return done_;
}

// Jobs in FIFO order: await their events, then fan out pieces of <= 16 MiB.
void NvmeQueue::dispatch() {
  cudaSetDevice(device_);
  constexpr std::uint64_t kPiece = 16ull << 20;
  for (;;) {
    Job j;
    {
      std::unique_lock<std::mutex> g(mu_);
      cv_.wait(g, [&] { return stop_ || !q_.empty(); });
      if (q_.empty()) return;
      j = std::move(q_.front());
      q_.pop_front();
      remaining_[j.seq] = ~0u;  // open (not yet split) until its pieces are queued
      dispatching_ = j.seq;
      dispatch_phase_ = 1;
    }
    bool ok = true;
    for (cudaEvent_t e : j.waits)
      if (e && cudaEventSynchronize(e) != cudaSuccess) ok = false;
    std::unique_lock<std::mutex> g(mu_);
    dispatch_phase_ = 2;
    if (j.after) done_cv_.wait(g, [&] { return done_ >= j.after || !error_.empty(); });  // same-buffer order
    dispatch_phase_ = 3;
    if (!ok) error_ = "event wait failed before NVMe I/O";
    const std::uint64_t n = std::max<std::uint64_t>(1, (j.bytes + kPiece - 1) / kPiece);
    remaining_[j.seq] = static_cast<std::uint32_t>(n);
    for (std::uint64_t k = 0; k < n; ++k) {
      const std::uint64_t o = k * kPiece;
      pieces_.push_back(Piece{j.write, static_cast<std::uint8_t*>(j.buf) + o, std::min(kPiece, j.bytes - o),
                              j.off + o, j.seq});
    }
    piece_cv_.notify_all();
  }
}

void NvmeQueue::work() {
  for (;;) {
    Piece p;
    {
      std::unique_lock<std::mutex> g(mu_);
      piece_cv_.wait(g, [&] { return stop_ || !pieces_.empty(); });
      if (pieces_.empty()) return;
      p = pieces_.front();
      pieces_.pop_front();
    }
    piece_done(p.seq, file_->io(p.write, p.buf, p.bytes, p.off));
  }
}

// A job is complete when its last piece lands; the published watermark is
// the highest seq below which every job is complete.
void NvmeQueue::piece_done(std::uint64_t seq, bool ok) {
  std::lock_guard<std::mutex> g(mu_);
  if (!ok) error_ = "NVMe tier I/O failed";
  if (--remaining_[seq] == 0) remaining_.erase(seq);
  // open = being dispatched or with pieces in flight (remaining_), or still queued (q_)
  const std::uint64_t oldest_open = remaining_.empty() ? submitted_ + 1 : remaining_.begin()->first;
  const std::uint64_t first_queued = q_.empty() ? submitted_ + 1 : q_.front().seq;
  const std::uint64_t mark = std::min(oldest_open, first_queued) - 1;
  if (kDebug)
    std::fprintf(stderr, "[nvme] piece of %llu done; mark %llu (done %llu)\n", static_cast<unsigned long long>(seq),
                 static_cast<unsigned long long>(mark), static_cast<unsigned long long>(done_));
  if (mark <= done_) return;
  done_ = mark;
  // published under the lock: two workers must never store the watermark out
  // of order (a GPU stream waiting for a value above a regressed word hangs)
  __atomic_store_n(const_cast<std::uint32_t*>(flag_), static_cast<std::uint32_t>(mark), __ATOMIC_RELEASE);
  done_cv_.notify_all();
}

}  // namespace tcb
