#include "nvme_io.hpp"

#include <cuda.h>
#include <fcntl.h>
#include <unistd.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>

#include "capi_common.hpp"
#include "dataplane.cuh"
#include "gds.hpp"

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

StripedFile::StripedFile(const std::string& dir, std::uint64_t bytes, int files, bool direct) : direct_(direct) {
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
  for (int fd : fds_) {
    Gds::release(fd);
    close(fd);
  }
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

bool StripedFile::io_device(bool write, std::uint8_t* dev, std::uint64_t bytes, std::uint64_t off) const {
  Gds& g = Gds::get();
  const std::uint64_t k = fds_.size();
  while (bytes) {
    const std::uint64_t stripe = off / kStripe, in = off % kStripe;
    const std::uint64_t len = std::min(bytes, kStripe - in);
    void* fh = g.handle(fds_[stripe % k]);
    const std::uint64_t foff = (stripe / k) * kStripe + in;
    if (!(write ? g.write(fh, dev, len, foff) : g.read(fh, dev, len, foff))) return false;
    dev += len;
    off += len;
    bytes -= len;
  }
  return true;
}

static double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
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
  void* rh = nullptr;
  if (cudaHostAlloc(&rh, sizeof(std::uint32_t) * kRing, cudaHostAllocMapped | cudaHostAllocPortable) != cudaSuccess)
    throw DeviceError(TC_ECUDA, "cannot allocate the NVMe completion ring");
  ring_ = static_cast<volatile std::uint32_t*>(rh);
  for (std::uint32_t i = 0; i < kRing; ++i) ring_[i] = 0;
  if (cudaHostGetDevicePointer(&ring_dev_, rh, 0) != cudaSuccess)
    throw DeviceError(TC_ECUDA, "cannot map the NVMe completion ring");
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
    cudaFreeHost(rh);
    throw DeviceError(TC_ECUDA, "stream memory operations unsupported");
  }
  dispatcher_ = std::thread([this] { dispatch(); });
  const char* env = std::getenv("TC_NVME_THREADS");
  const int nw = env ? std::max(1, std::atoi(env)) : 32;
  for (int i = 0; i < nw; ++i) workers_.emplace_back([this] { work(); });
}

NvmeQueue::~NvmeQueue() {
  if (std::getenv("TC_NVME_STATS"))
    std::fprintf(stderr, "[nvme] %llu reads waited %.3f s, %llu writes waited %.3f s between submit and dispatch\n",
                 static_cast<unsigned long long>(jobs_r_), wait_r_, static_cast<unsigned long long>(jobs_w_), wait_w_);
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
  if (ring_) cudaFreeHost(const_cast<std::uint32_t*>(ring_));
}

static const bool kDebug = std::getenv("TC_NVME_DEBUG") != nullptr;

std::uint64_t NvmeQueue::submit(Job j) {
  std::lock_guard<std::mutex> g(mu_);
  if (!error_.empty()) throw DeviceError(TC_EIO, error_);
  j.seq = ++submitted_;
  j.t_submit = now_s();
  std::erase(j.after, 0ull);
  if (kDebug)
    std::fprintf(stderr, "[nvme] submit %llu %s %llu B @%llu waits=%zu after=%zu\n",
                 static_cast<unsigned long long>(j.seq), j.write ? "W" : "R", static_cast<unsigned long long>(j.bytes),
                 static_cast<unsigned long long>(j.off), j.waits.size(), j.after.size());
  (j.write ? bytes_written_ : bytes_read_) += j.bytes;
  q_.push_back(std::move(j));
  cv_.notify_one();
  return submitted_;
}

std::uint64_t NvmeQueue::submit_read(void* dst, std::uint64_t bytes, std::uint64_t off, std::vector<cudaEvent_t> w,
                                     std::vector<std::uint64_t> after, std::uint64_t packed_n) {
  Job j{false, false, dst, bytes, off, 0, std::move(w), std::move(after)};
  j.packed_n = packed_n;
  return submit(std::move(j));
}

void NvmeQueue::forget_extent(std::uint64_t off) {
  std::lock_guard<std::mutex> g(mu_);
  extent_len_.erase(off);
}

// A packed state's write moves its prefix, plus the overflow area when a
// tile uses it; a read of the extent moves what its last write moved. (O_DIRECT
// files: whole 4 KiB blocks.)
std::uint64_t NvmeQueue::effective_bytes(Job& j) {
  std::uint64_t bytes = j.bytes;
  if (j.packed_n && !j.device) {
    const PackedLayout L = packed_layout(j.packed_n);
    if (j.write) {
      const std::uint8_t* fl = static_cast<const std::uint8_t*>(j.buf) + L.flags;  // a byte per 256 elements
      bool ovf = false;
      for (std::uint64_t t = 0; t < j.packed_n / 256 && !ovf; ++t) ovf = fl[t] != 0;
      bytes = ovf ? L.ovf + 2 * j.packed_n : L.bytes;
      if (file_->direct()) bytes = (bytes + 4095) / 4096 * 4096;
      bytes = std::min(bytes, j.bytes);
      extent_len_[j.off] = bytes;
    } else {
      auto e = extent_len_.find(j.off);
      if (e != extent_len_.end()) bytes = std::min(bytes, e->second);
    }
  } else if (j.write) {
    extent_len_.erase(j.off);
  }
  (j.write ? bytes_written_ : bytes_read_) -= j.bytes - bytes;
  return bytes;
}

std::uint64_t NvmeQueue::submit_read_device(void* dst, std::uint64_t bytes, std::uint64_t off,
                                            std::vector<cudaEvent_t> w, std::vector<std::uint64_t> after) {
  return submit(Job{false, true, dst, bytes, off, 0, std::move(w), std::move(after)});
}

std::uint64_t NvmeQueue::submit_write_device(const void* src, std::uint64_t bytes, std::uint64_t off,
                                             std::vector<cudaEvent_t> w, std::vector<std::uint64_t> after) {
  return submit(Job{true, true, const_cast<void*>(src), bytes, off, 0, std::move(w), std::move(after)});
}

std::uint64_t NvmeQueue::submit_write(const void* src, std::uint64_t bytes, std::uint64_t off,
                                      std::vector<cudaEvent_t> w, std::vector<std::uint64_t> after,
                                      std::uint64_t packed_n) {
  Job j{true, false, const_cast<void*>(src), bytes, off, 0, std::move(w), std::move(after)};
  j.packed_n = packed_n;
  return submit(std::move(j));
}

std::uint64_t NvmeQueue::done() const {
  std::lock_guard<std::mutex> g(mu_);
  return done_;
}

std::uint64_t NvmeQueue::submitted() const {
  std::lock_guard<std::mutex> g(mu_);
  return submitted_;
}

// A job's own completion word: a GPU stream waits for exactly the job it
// consumes, never for unrelated earlier jobs (which may be waiting on GPU work
// queued behind it).
void NvmeQueue::stream_wait(cudaStream_t s, std::uint64_t seq) {
  if (seq == 0) return;
  {
    std::lock_guard<std::mutex> g(mu_);
    if (is_done(seq)) return;
  }
  auto* word = static_cast<std::uint32_t*>(ring_dev_) + (seq % kRing);
  const CUresult r = reinterpret_cast<WaitValue32>(wait_fn_)(
      reinterpret_cast<CUstream>(s), reinterpret_cast<CUdeviceptr>(word), static_cast<cuuint32_t>(seq),
      CU_STREAM_WAIT_VALUE_GEQ);
  if (r != CUDA_SUCCESS) throw DeviceError(TC_ECUDA, "cuStreamWaitValue32 failed");
}

void NvmeQueue::stream_wait_upto(cudaStream_t s, std::uint64_t seq) {
  if (seq == 0 || seq <= done()) return;
  const CUresult r = reinterpret_cast<WaitValue32>(wait_fn_)(
      reinterpret_cast<CUstream>(s), reinterpret_cast<CUdeviceptr>(flag_dev_), static_cast<cuuint32_t>(seq),
      CU_STREAM_WAIT_VALUE_GEQ);
  if (r != CUDA_SUCCESS) throw DeviceError(TC_ECUDA, "cuStreamWaitValue32 failed");
}

std::string NvmeQueue::describe() {
  std::lock_guard<std::mutex> g(mu_);
  std::string s = "nvme queue: submitted " + std::to_string(submitted_) + " watermark " + std::to_string(done_) +
                  " flag " + std::to_string(*flag_) + " queued " + std::to_string(q_.size()) + " pieces " +
                  std::to_string(pieces_.size()) + " complete-above-watermark " + std::to_string(completed_.size()) +
                  " in flight:";
  int k = 0;
  for (const auto& [seq, left] : remaining_) {
    if (k++ > 8) break;
    s += " " + std::to_string(seq) + "(" + std::to_string(static_cast<int>(left)) + ")";
  }
  if (!q_.empty()) {
    const Job& j = q_.front();
    s += "; oldest queued " + std::to_string(j.seq) + (j.write ? " W" : " R") + " after:";
    for (std::uint64_t a : j.after) s += " " + std::to_string(a) + (is_done(a) ? "(done)" : "(open)");
  }
  return s;
}

void NvmeQueue::wait(std::uint64_t seq) {
  if (seq == 0) return;
  if (kDebug) std::fprintf(stderr, "[nvme] host wait %llu\n", static_cast<unsigned long long>(seq));
  std::unique_lock<std::mutex> g(mu_);
  while (!done_cv_.wait_for(g, std::chrono::seconds(30), [&] { return is_done(seq) || !error_.empty(); })) {
    g.unlock();
    std::fprintf(stderr, "[nvme] still waiting for job %llu: %s\n", static_cast<unsigned long long>(seq),
                 describe().c_str());
    g.lock();
  }
  if (!error_.empty()) throw DeviceError(TC_EIO, error_);
}

void NvmeQueue::wait_upto(std::uint64_t seq) {
  if (seq == 0) return;
  std::unique_lock<std::mutex> g(mu_);
  while (!done_cv_.wait_for(g, std::chrono::seconds(30), [&] { return done_ >= seq || !error_.empty(); })) {
    g.unlock();
    std::fprintf(stderr, "[nvme] still waiting for jobs up to %llu: %s\n", static_cast<unsigned long long>(seq),
                 describe().c_str());
    g.lock();
  }
  if (!error_.empty()) throw DeviceError(TC_EIO, error_);
}

int NvmeQueue::ready(const Job& j) {
  for (std::uint64_t a : j.after)
    if (!is_done(a)) return 0;
  for (cudaEvent_t e : j.waits) {
    if (!e) continue;
    const cudaError_t q = cudaEventQuery(e);
    if (q == cudaErrorNotReady) return 0;
    if (q != cudaSuccess) return -1;
  }
  return 1;
}

// Out-of-order dispatch: the first queued job whose events have completed and
// whose `after` jobs are done is split into pieces of <= 16 MiB for the pool;
// when none is ready the dispatcher re-polls (events complete without notice).
void NvmeQueue::dispatch() {
  cudaSetDevice(device_);
  constexpr std::uint64_t kPiece = 16ull << 20;
  std::unique_lock<std::mutex> g(mu_);
  for (;;) {
    if (stop_ && q_.empty()) return;
    auto it = q_.begin();
    int st = 0;
    for (; it != q_.end(); ++it) {
      if (it->seq >= done_ + kRing / 2) break;  // completion-ring window
      if ((st = ready(*it)) != 0) break;
    }
    if (it == q_.end() || st == 0) {
      cv_.wait_for(g, std::chrono::microseconds(50));
      continue;
    }
    Job j = std::move(*it);
    q_.erase(it);
    if (st < 0) {  // never touch a buffer whose producer failed; complete the job so no stream hangs,
                   // the error surfaces at the engine's next host-side check (check())
      error_ = "event wait failed before NVMe I/O (job " + std::to_string(j.seq) + ")";
      remaining_[j.seq] = 1;
      g.unlock();
      piece_done(j.seq, true);
      g.lock();
      continue;
    }
    (j.write ? wait_w_ : wait_r_) += now_s() - j.t_submit;
    ++(j.write ? jobs_w_ : jobs_r_);
    j.bytes = effective_bytes(j);
    const std::uint64_t n = std::max<std::uint64_t>(1, (j.bytes + kPiece - 1) / kPiece);
    remaining_[j.seq] = static_cast<std::uint32_t>(n);
    for (std::uint64_t k = 0; k < n; ++k) {
      const std::uint64_t o = k * kPiece;
      pieces_.push_back(Piece{j.write, j.device, static_cast<std::uint8_t*>(j.buf) + o,
                              std::min(kPiece, j.bytes - o), j.off + o, j.seq});
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
    // fault injection for tests: TC_NVME_FAIL_JOB=k fails job k's I/O
    const char* fe = std::getenv("TC_NVME_FAIL_JOB");
    const std::uint64_t fail_job = fe ? std::strtoull(fe, nullptr, 10) : 0ull;
    bool ok = p.seq != fail_job;
    if (ok) {
      try {
        ok = p.device ? file_->io_device(p.write, p.buf, p.bytes, p.off) : file_->io(p.write, p.buf, p.bytes, p.off);
      } catch (const std::exception&) {
        ok = false;  // surfaces as the queue's I/O error
      }
    }
    piece_done(p.seq, ok);
  }
}

// A job is complete when its last piece lands: its ring word is published,
// and the watermark advances over every contiguous complete job. Both are
// stored under the lock (a watermark must never regress: a GPU stream waiting
// for a value above a regressed word hangs).
void NvmeQueue::check() const {
  std::lock_guard<std::mutex> g(mu_);
  if (!error_.empty()) throw DeviceError(TC_EIO, error_);
}

void NvmeQueue::piece_done(std::uint64_t seq, bool ok) {
  std::lock_guard<std::mutex> g(mu_);
  if (!ok && error_.empty()) error_ = "NVMe tier I/O failed (job " + std::to_string(seq) + ")";
  if (--remaining_[seq] != 0) return;
  remaining_.erase(seq);
  completed_.insert(seq);
  __atomic_store_n(const_cast<std::uint32_t*>(ring_ + (seq % kRing)), static_cast<std::uint32_t>(seq),
                   __ATOMIC_RELEASE);
  while (!completed_.empty() && *completed_.begin() == done_ + 1) {
    completed_.erase(completed_.begin());
    ++done_;
  }
  __atomic_store_n(const_cast<std::uint32_t*>(flag_), static_cast<std::uint32_t>(done_), __ATOMIC_RELEASE);
  if (kDebug)
    std::fprintf(stderr, "[nvme] job %llu done; watermark %llu\n", static_cast<unsigned long long>(seq),
                 static_cast<unsigned long long>(done_));
  done_cv_.notify_all();
  cv_.notify_one();  // a queued job may have been waiting for this one
}

}  // namespace tcb
