#include "nvme_io.hpp"

#include <cuda.h>
#include <unistd.h>

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

NvmeQueue::NvmeQueue(int device, int fd) : device_(device), fd_(fd) {
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
  worker_ = std::thread([this] { run(); });
}

NvmeQueue::~NvmeQueue() {
  {
    std::lock_guard<std::mutex> g(mu_);
    stop_ = true;
  }
  cv_.notify_all();
  if (worker_.joinable()) worker_.join();
  if (flag_) cudaFreeHost(const_cast<std::uint32_t*>(flag_));
}

std::uint64_t NvmeQueue::submit(Job j) {
  std::lock_guard<std::mutex> g(mu_);
  if (!error_.empty()) throw DeviceError(TC_EIO, error_);
  j.seq = ++submitted_;
  (j.write ? bytes_written_ : bytes_read_) += j.bytes;
  q_.push_back(std::move(j));
  cv_.notify_one();
  return submitted_;
}

std::uint64_t NvmeQueue::submit_read(void* dst, std::uint64_t bytes, std::uint64_t off, std::vector<cudaEvent_t> w) {
  return submit(Job{false, dst, bytes, off, 0, std::move(w)});
}

std::uint64_t NvmeQueue::submit_write(const void* src, std::uint64_t bytes, std::uint64_t off,
                                      std::vector<cudaEvent_t> w) {
  return submit(Job{true, const_cast<void*>(src), bytes, off, 0, std::move(w)});
}

void NvmeQueue::stream_wait(cudaStream_t s, std::uint64_t seq) {
  if (seq == 0 || seq <= done()) return;
  const CUresult r = reinterpret_cast<WaitValue32>(wait_fn_)(
      reinterpret_cast<CUstream>(s), reinterpret_cast<CUdeviceptr>(flag_dev_), static_cast<cuuint32_t>(seq),
      CU_STREAM_WAIT_VALUE_GEQ);
  if (r != CUDA_SUCCESS) throw DeviceError(TC_ECUDA, "cuStreamWaitValue32 failed");
}

void NvmeQueue::wait(std::uint64_t seq) {
  std::unique_lock<std::mutex> g(mu_);
  done_cv_.wait(g, [&] { return done_ >= seq || !error_.empty(); });
  if (!error_.empty()) throw DeviceError(TC_EIO, error_);
}

std::uint64_t NvmeQueue::done() const {
  std::lock_guard<std::mutex> g(const_cast<std::mutex&>(mu_));
  return done_;
}

void NvmeQueue::run() {
  cudaSetDevice(device_);
  for (;;) {
    Job j;
    {
      std::unique_lock<std::mutex> g(mu_);
      cv_.wait(g, [&] { return stop_ || !q_.empty(); });
      if (q_.empty()) return;
      j = std::move(q_.front());
      q_.pop_front();
    }
    std::string err;
    for (cudaEvent_t e : j.waits)
      if (e && cudaEventSynchronize(e) != cudaSuccess) err = "event wait failed before NVMe I/O";
    auto* p = static_cast<std::uint8_t*>(j.buf);
    for (std::uint64_t done = 0; err.empty() && done < j.bytes;) {
      const ssize_t k = j.write ? pwrite(fd_, p + done, j.bytes - done, static_cast<off_t>(j.off + done))
                                : pread(fd_, p + done, j.bytes - done, static_cast<off_t>(j.off + done));
      if (k <= 0) err = j.write ? "NVMe tier write failed" : "NVMe tier read failed";
      else done += static_cast<std::uint64_t>(k);
    }
    {
      std::lock_guard<std::mutex> g(mu_);
      if (!err.empty()) error_ = err;
      done_ = j.seq;
    }
    __atomic_store_n(const_cast<std::uint32_t*>(flag_), static_cast<std::uint32_t>(j.seq), __ATOMIC_RELEASE);
    done_cv_.notify_all();
  }
}

}  // namespace tcb
