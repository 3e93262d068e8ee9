// hostio.cpp -- see hostio.hpp.
#include "hostio.hpp"

#include <cuda_runtime.h>

#include <emmintrin.h>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <thread>

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

namespace {
// memcpy with non-temporal stores (SSE2): the staged bytes are next read by a
// DMA engine (or much later by the caller), so they should not displace the
// cache, and a streaming store skips the read-for-ownership of the
// destination line -- 2 instead of 3 bytes of DRAM traffic per byte copied.
// (glibc switches to such stores only above a per-call size far beyond a
// worker's part of an 8 MB piece.)
inline void copy_stream(char* d, const char* s, size_t n) {
  if ((reinterpret_cast<uintptr_t>(d) & 15u) != 0 || n < 256) {
    std::memcpy(d, s, n);
    return;
  }
  size_t i = 0;
  for (; i + 64 <= n; i += 64) {
    const __m128i a = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + i));
    const __m128i b = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + i + 16));
    const __m128i c = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + i + 32));
    const __m128i e = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + i + 48));
    _mm_stream_si128(reinterpret_cast<__m128i*>(d + i), a);
    _mm_stream_si128(reinterpret_cast<__m128i*>(d + i + 16), b);
    _mm_stream_si128(reinterpret_cast<__m128i*>(d + i + 32), c);
    _mm_stream_si128(reinterpret_cast<__m128i*>(d + i + 48), e);
  }
  if (i < n) std::memcpy(d + i, s + i, n - i);
  _mm_sfence();  // the stores are globally visible before the piece is reported done
}

inline void spin_pause(unsigned& n) {
  if (++n & 63u)
    __builtin_ia32_pause();
  else
    std::this_thread::yield();
}
}  // namespace

void CopyPool::run(int id) {
  unsigned long long seen = 0;
  for (;;) {
    char* d;
    const char* s;
    size_t n, piece, np;
    {
      std::unique_lock<std::mutex> lk(m_);
      cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
      if (stop_) return;
      seen = gen_;
      d = dst_;
      s = src_;
      n = bytes_;
      piece = piece_;
      np = n_pieces_;
    }
    if (piece == 0) {  // plain copy: part id of threads() (the caller takes part 0)
      size_t lo, hi;
      part_range(n, threads(), id, lo, hi);
      if (hi > lo) std::memcpy(d + lo, s + lo, hi - lo);
    } else {  // streamed: part id - 1 of the workers, piece after piece
      const int W = (int)workers_.size();
      for (size_t c = 0; c < np; ++c) {
        unsigned spins = 0;
        while (released_.load(std::memory_order_acquire) <= c) spin_pause(spins);
        const size_t off = c * piece, len = std::min(piece, n - off);
        size_t lo, hi;
        part_range(len, W, id - 1, lo, hi);
        if (hi > lo) copy_stream(d + off + lo, s + off + lo, hi - lo);
        done_[c].fetch_add(1, std::memory_order_release);
      }
    }
    {
      std::lock_guard<std::mutex> lk(m_);
      if (--pending_ == 0) done_cv_.notify_one();
    }
  }
}

void CopyPool::stream_begin(void* dst, const void* src, size_t bytes, size_t piece,
                            bool all_released) {
  const size_t np = (bytes + piece - 1) / piece;
  if (np > done_cap_) {
    done_.reset(new std::atomic<int>[np]);
    done_cap_ = np;
  }
  for (size_t c = 0; c < np; ++c) done_[c].store(0, std::memory_order_relaxed);
  released_.store(all_released ? np : 0, std::memory_order_release);
  {
    std::lock_guard<std::mutex> lk(m_);
    dst_ = static_cast<char*>(dst);
    src_ = static_cast<const char*>(src);
    bytes_ = bytes;
    piece_ = piece;
    n_pieces_ = np;
    pending_ = (int)workers_.size();
    ++gen_;
  }
  cv_.notify_all();
}

void CopyPool::stream_wait(size_t c) {
  const int W = (int)workers_.size();
  unsigned spins = 0;
  while (done_[c].load(std::memory_order_acquire) < W) spin_pause(spins);
}

void CopyPool::stream_end() {
  std::unique_lock<std::mutex> lk(m_);
  done_cv_.wait(lk, [&] { return pending_ == 0; });
  piece_ = 0;
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
    piece_ = 0;
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
