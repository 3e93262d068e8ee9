// hostio.hpp -- host-side staging for imq_operator_apply with pageable
// buffers (the reference's callers pass std::vector memory, reference
// capi.cpp:130-138): a small persistent thread pool for parallel memcpy
// between pageable and pinned memory, and a pinned-ness probe.
#pragma once
#include <atomic>
#include <condition_variable>
#include <cstddef>
#include <memory>
#include <mutex>
#include <thread>
#include <vector>

namespace imqh {

// True when p is page-locked (cudaHostAlloc / cudaHostRegister) host memory
// the copy engines can read directly.
bool host_pinned(const void* p);

// memcpy split over a fixed set of worker threads (plus the caller).  One
// copy at a time per pool; copy() returns when every part is done.
class CopyPool {
 public:
  explicit CopyPool(int threads);
  ~CopyPool();
  CopyPool(const CopyPool&) = delete;
  CopyPool& operator=(const CopyPool&) = delete;
  void copy(void* dst, const void* src, size_t bytes);
  int threads() const { return (int)workers_.size() + 1; }

  // Streamed copy in pieces: the workers are woken ONCE and copy piece after
  // piece (each piece split over all workers, so pieces finish in order);
  // piece c is copied only after release(c + 1).  The caller overlaps its own
  // work per piece: H2D staging -- stream_begin(all released), then per piece
  // stream_wait(c) and the DMA of that piece; D2H draining -- stream_begin(none
  // released), then per piece wait for its DMA and stream_release(c + 1).
  // stream_end() returns when every piece is copied.  (A condition-variable
  // round trip per 8 MB piece cost ~1.5 ms per 134 MB vector each way.)
  void stream_begin(void* dst, const void* src, size_t bytes, size_t piece, bool all_released);
  void stream_release(size_t upto) { released_.store(upto, std::memory_order_release); }
  void stream_wait(size_t c);
  void stream_end();

 private:
  void run(int id);
  std::vector<std::thread> workers_;
  std::mutex m_;
  std::condition_variable cv_, done_cv_;
  char* dst_ = nullptr;
  const char* src_ = nullptr;
  size_t bytes_ = 0;
  unsigned long long gen_ = 0;
  int pending_ = 0;
  bool stop_ = false;
  // streamed job
  size_t piece_ = 0, n_pieces_ = 0;  // piece_ == 0: a plain copy() job
  std::atomic<size_t> released_{0};
  std::unique_ptr<std::atomic<int>[]> done_;
  size_t done_cap_ = 0;
};

}  // namespace imqh
