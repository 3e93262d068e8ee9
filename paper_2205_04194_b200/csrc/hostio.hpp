// hostio.hpp -- host-side staging for imq_operator_apply with pageable
// buffers (the reference's callers pass std::vector memory, reference
// capi.cpp:130-138): a small persistent thread pool for parallel memcpy
// between pageable and pinned memory, and a pinned-ness probe.
#pragma once
#include <condition_variable>
#include <cstddef>
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
};

}  // namespace imqh
