// hostio.cpp -- see hostio.hpp.
#include "hostio.hpp"

#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>

namespace imqh {

bool host_pinned(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

namespace {
// part `id` of `parts` of a [0, bytes) range, 4 KB aligned boundaries
void part_range(size_t bytes, int parts, int id, size_t& lo, size_t& hi) {
  const size_t per = ((bytes + (size_t)parts - 1) / (size_t)parts + 4095) & ~(size_t)4095;
  lo = std::min(bytes, per * (size_t)id);
  hi = std::min(bytes, lo + per);
}
}  // namespace

CopyPool::CopyPool(int threads) {
  for (int i = 0; i < threads - 1; ++i) workers_.emplace_back([this, i] { run(i + 1); });
}

CopyPool::~CopyPool() {
  {
    std::lock_guard<std::mutex> lk(m_);
    stop_ = true;
  }
  cv_.notify_all();
  for (auto& t : workers_) t.join();
}

void CopyPool::run(int id) {
  unsigned long long seen = 0;
  for (;;) {
    char* d;
    const char* s;
    size_t n;
    {
      std::unique_lock<std::mutex> lk(m_);
      cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
      if (stop_) return;
      seen = gen_;
      d = dst_;
      s = src_;
      n = bytes_;
    }
    size_t lo, hi;
    part_range(n, threads(), id, lo, hi);
    if (hi > lo) std::memcpy(d + lo, s + lo, hi - lo);
    {
      std::lock_guard<std::mutex> lk(m_);
      if (--pending_ == 0) done_cv_.notify_one();
    }
  }
}

void CopyPool::copy(void* dst, const void* src, size_t bytes) {
  if (workers_.empty() || bytes < (size_t)1 << 20) {
    std::memcpy(dst, src, bytes);
    return;
  }
  {
    std::lock_guard<std::mutex> lk(m_);
    dst_ = static_cast<char*>(dst);
    src_ = static_cast<const char*>(src);
    bytes_ = bytes;
    pending_ = (int)workers_.size();
    ++gen_;
  }
  cv_.notify_all();
  size_t lo, hi;
  part_range(bytes, threads(), 0, lo, hi);
  if (hi > lo) std::memcpy(static_cast<char*>(dst) + lo, static_cast<const char*>(src) + lo, hi - lo);
  std::unique_lock<std::mutex> lk(m_);
  done_cv_.wait(lk, [&] { return pending_ == 0; });
}

}  // namespace imqh
