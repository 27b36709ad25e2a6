// Asynchronous NVMe tier I/O. A dispatcher thread takes jobs in FIFO order,
// waits for the CUDA events each depends on (the copy that filled a pinned
// buffer, or the copies that last read it) and splits it into pieces that a
// pool of worker threads pread/pwrite concurrently (queue depth for real
// NVMe, parallel copies for the page cache). Jobs complete in any order; the
// in-order completion watermark is published in a mapped host word. GPU
// streams that consume the bytes wait on that word with cuStreamWaitValue32
// (no host thread blocks in the iteration, no CUDA host callbacks); host
// code waits on a condition variable.
#pragma once

#include <condition_variable>
#include <cstdint>
#include <deque>
#include <map>
#include <string>
#include <mutex>
#include <set>
#include <thread>
#include <vector>

#include <cuda_runtime.h>

namespace tcb {

// GPU-side wait until the 32-bit word at `dev_addr` (device-accessible) is
// >= value (cuStreamWaitValue32 through the runtime's driver entry point).
void stream_wait_value32(cudaStream_t s, const unsigned* dev_addr, unsigned value);

// The NVMe tier's backing store: one logical byte range striped over K files
// in 16 MiB stripes (file = stripe % K). Buffered writes to one file
// serialise on the inode lock in the kernel; K files let the I/O pool's
// workers write in parallel.
class StripedFile {
 public:
  static constexpr std::uint64_t kStripe = 16ull << 20;
  StripedFile(const std::string& dir, std::uint64_t bytes, int files, bool direct);
  ~StripedFile();
  StripedFile(const StripedFile&) = delete;
  StripedFile& operator=(const StripedFile&) = delete;
  // Full transfer at logical offset `off`; false on an I/O error.
  bool io(bool write, std::uint8_t* buf, std::uint64_t bytes, std::uint64_t off) const;
  // The same between the file and HBM through GPUDirect Storage (gds.hpp);
  // the files must be O_DIRECT.
  bool io_device(bool write, std::uint8_t* dev, std::uint64_t bytes, std::uint64_t off) const;
  bool direct() const { return direct_; }
  int files() const { return static_cast<int>(fds_.size()); }

 private:
  std::vector<int> fds_;
  bool direct_ = false;
};

class NvmeQueue {
 public:
  // Throws DeviceError when stream memory operations are unavailable.
  NvmeQueue(int device, const StripedFile* file);
  ~NvmeQueue();

  // `after`: earlier jobs that must be complete before this one starts (the
  // buffer's previous jobs, the file extent's previous job). Jobs otherwise
  // start out of order, as soon as their events and `after` jobs are done.
  // packed_n != 0: the buffer holds a packed split-master state of packed_n
  // parameters (dataplane.cuh PackedLayout): a write moves only its prefix
  // (+ the overflow area when a tile uses it: the flags are read from the
  // buffer once its producer is done) and records that length for the
  // extent; a later read of the extent moves that many bytes.
  std::uint64_t submit_read(void* dst, std::uint64_t bytes, std::uint64_t file_off, std::vector<cudaEvent_t> waits,
                            std::vector<std::uint64_t> after = {}, std::uint64_t packed_n = 0);
  std::uint64_t submit_write(const void* src, std::uint64_t bytes, std::uint64_t file_off,
                             std::vector<cudaEvent_t> waits, std::vector<std::uint64_t> after = {},
                             std::uint64_t packed_n = 0);
  void forget_extent(std::uint64_t file_off);  // written outside the queue: whole length again
  // dst/src in HBM: the worker moves the bytes with GPUDirect Storage
  std::uint64_t submit_read_device(void* dst, std::uint64_t bytes, std::uint64_t file_off,
                                   std::vector<cudaEvent_t> waits, std::vector<std::uint64_t> after = {});
  std::uint64_t submit_write_device(const void* src, std::uint64_t bytes, std::uint64_t file_off,
                                    std::vector<cudaEvent_t> waits, std::vector<std::uint64_t> after = {});
  void stream_wait(cudaStream_t s, std::uint64_t seq);       // GPU-side wait for job `seq` alone
  void stream_wait_upto(cudaStream_t s, std::uint64_t seq);  // GPU-side wait for every job <= seq
  void wait(std::uint64_t seq);                              // host-side wait for job `seq`
  void wait_upto(std::uint64_t seq);                         // host-side wait for every job <= seq
  void wait_all() { wait_upto(submitted()); }
  std::uint64_t done() const;  // watermark: every job <= done() is complete
  // Throws DeviceError(TC_EIO) once any job failed. A failed job is still
  // published complete (a GPU stream waiting on it must not hang), so every
  // result that may have consumed its bytes is checked through this.
  void check() const;
  std::uint64_t submitted() const;
  std::uint64_t bytes_read() const { return bytes_read_; }
  std::string describe();  // state dump for hang diagnostics
  std::uint64_t bytes_written() const { return bytes_written_; }

 private:
  static constexpr std::uint32_t kRing = 1u << 16;  // per-job completion words (seq % kRing)
  struct Job {
    bool write;
    bool device = false;  // buf is HBM (GPUDirect Storage)
    void* buf;
    std::uint64_t bytes, off, seq;
    std::vector<cudaEvent_t> waits;
    std::vector<std::uint64_t> after;
    double t_submit = 0;  // steady-clock seconds (TC_NVME_STATS)
    std::uint64_t packed_n = 0;
  };
  std::uint64_t effective_bytes(Job& j);  // mu_ held, at dispatch
  std::map<std::uint64_t, std::uint64_t> extent_len_;  // file offset -> bytes the last packed write moved
  struct Piece {
    bool write;
    bool device;
    std::uint8_t* buf;
    std::uint64_t bytes, off, seq;
  };
  std::uint64_t submit(Job j);
  void dispatch();
  void work();
  void piece_done(std::uint64_t seq, bool ok);
  bool is_done(std::uint64_t seq) const { return seq <= done_ || completed_.count(seq) != 0; }  // mu_ held
  int ready(const Job& j);  // mu_ held: 1 ready, 0 not yet, -1 event failed

  int device_;
  const StripedFile* file_;
  std::deque<Piece> pieces_;
  std::map<std::uint64_t, std::uint32_t> remaining_;  // seq -> pieces left (dispatched jobs)
  std::set<std::uint64_t> completed_;                 // complete jobs above the watermark
  std::condition_variable piece_cv_;
  std::vector<std::thread> workers_;
  volatile std::uint32_t* flag_ = nullptr;  // mapped pinned word: the watermark
  void* flag_dev_ = nullptr;
  volatile std::uint32_t* ring_ = nullptr;  // mapped pinned words: ring_[seq % kRing] = seq once complete
  void* ring_dev_ = nullptr;
  void* wait_fn_ = nullptr;                 // cuStreamWaitValue32
  mutable std::mutex mu_;
  std::condition_variable cv_, done_cv_;
  std::deque<Job> q_;  // submitted, not yet dispatched (submission order)
  std::uint64_t submitted_ = 0, done_ = 0, bytes_read_ = 0, bytes_written_ = 0;
  bool stop_ = false;
  std::string error_;
  std::thread dispatcher_;
  double wait_r_ = 0, wait_w_ = 0;  // TC_NVME_STATS: submit -> dispatch time
  std::uint64_t jobs_r_ = 0, jobs_w_ = 0;
};

}  // namespace tcb
