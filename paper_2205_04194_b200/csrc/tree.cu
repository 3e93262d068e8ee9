// tree.cu -- bounding square reduction, bit-exact binning, Morton sort, leaf
// offsets, and the sorted<->original gathers.
//
// Bit-exactness (reference partition.cpp:25-33): the finest-level cell index is
// floor(fl(fl(x - o) / cell_L)) with IEEE subtraction and division and no
// contraction (__dsub_rn / __ddiv_rn).  Coarser indices are i_L >> (L - l):
// cell_l = side / 2^(l+1) is an exact power-of-two rescaling of cell_L, so
// fl((x-o)/cell_l) = fl((x-o)/cell_L) * 2^-(L-l) and the floors agree; the
// per-level clamps to [0, grid_l - 1] commute with the shift.
#include <cub/device/device_radix_sort.cuh>

#include "imq_device.cuh"
#include "imq_kernels.hpp"

namespace imqk {
using namespace imqdev;

namespace {

constexpr int kThreads = 256;

// partial[b*5 + {0..4}] = minx, maxx, miny, maxy, nonfinite-count of CTA b
__global__ void __launch_bounds__(kThreads) k_minmax(const double* __restrict__ xy, long long n,
                                                     double* __restrict__ partial) {
  double mnx = INFINITY, mxx = -INFINITY, mny = INFINITY, mxy = -INFINITY, bad = 0.0;
  for (long long p = blockIdx.x * (long long)kThreads + threadIdx.x; p < n;
       p += (long long)gridDim.x * kThreads) {
    double2 v = reinterpret_cast<const double2*>(xy)[p];
    if (!isfinite(v.x) || !isfinite(v.y)) {
      bad += 1.0;
      continue;
    }
    mnx = fmin(mnx, v.x);
    mxx = fmax(mxx, v.x);
    mny = fmin(mny, v.y);
    mxy = fmax(mxy, v.y);
  }
  for (int o = 16; o > 0; o >>= 1) {
    mnx = fmin(mnx, __shfl_xor_sync(0xffffffffu, mnx, o));
    mxx = fmax(mxx, __shfl_xor_sync(0xffffffffu, mxx, o));
    mny = fmin(mny, __shfl_xor_sync(0xffffffffu, mny, o));
    mxy = fmax(mxy, __shfl_xor_sync(0xffffffffu, mxy, o));
    bad += __shfl_xor_sync(0xffffffffu, bad, o);
  }
  __shared__ double red[kThreads / 32][5];
  int w = threadIdx.x / 32, l = threadIdx.x % 32;
  if (l == 0) {
    red[w][0] = mnx; red[w][1] = mxx; red[w][2] = mny; red[w][3] = mxy; red[w][4] = bad;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < kThreads / 32; ++k) {
      mnx = fmin(mnx, red[k][0]); mxx = fmax(mxx, red[k][1]);
      mny = fmin(mny, red[k][2]); mxy = fmax(mxy, red[k][3]); bad += red[k][4];
    }
    double* o = partial + 5 * (size_t)blockIdx.x;
    o[0] = mnx; o[1] = mxx; o[2] = mny; o[3] = mxy; o[4] = bad;
  }
}

__global__ void k_minmax_final(const double* __restrict__ partial, int nparts, double* out) {
  if (threadIdx.x != 0) return;
  double mnx = INFINITY, mxx = -INFINITY, mny = INFINITY, mxy = -INFINITY, bad = 0.0;
  for (int b = 0; b < nparts; ++b) {
    const double* o = partial + 5 * (size_t)b;
    mnx = fmin(mnx, o[0]); mxx = fmax(mxx, o[1]);
    mny = fmin(mny, o[2]); mxy = fmax(mxy, o[3]); bad += o[4];
  }
  out[0] = mnx; out[1] = mxx; out[2] = mny; out[3] = mxy; out[4] = bad;
}

// partition.cpp:25-33 at the finest level; key = Morton(i, j), value = index.
__global__ void __launch_bounds__(kThreads) k_bin(const double* __restrict__ xy, long long n,
                                                  double ox, double oy, double cell, int grid,
                                                  uint32_t* __restrict__ keys,
                                                  int* __restrict__ idx) {
  long long p = blockIdx.x * (long long)kThreads + threadIdx.x;
  if (p >= n) return;
  double2 v = reinterpret_cast<const double2*>(xy)[p];
  double fi = floor(__ddiv_rn(__dsub_rn(v.x, ox), cell));
  double fj = floor(__ddiv_rn(__dsub_rn(v.y, oy), cell));
  // (int) conversion of the reference saturates only for absurd inputs; clamp
  // in double first so the integer conversion is always defined.
  fi = fmin(fmax(fi, 0.0), (double)(grid - 1));
  fj = fmin(fmax(fj, 0.0), (double)(grid - 1));
  keys[p] = morton((uint32_t)fi, (uint32_t)fj);
  idx[p] = (int)p;
}

__global__ void __launch_bounds__(kThreads) k_gather_points(const double* __restrict__ xy,
                                                            const int* __restrict__ perm,
                                                            long long n, double* __restrict__ xs,
                                                            double* __restrict__ ys) {
  long long p = blockIdx.x * (long long)kThreads + threadIdx.x;
  if (p >= n) return;
  double2 v = reinterpret_cast<const double2*>(xy)[perm[p]];
  xs[p] = v.x;
  ys[p] = v.y;
}

// leaf_start[c] = first sorted position with key >= c (lower bound).
__global__ void __launch_bounds__(kThreads) k_leaf_start(const uint32_t* __restrict__ keys,
                                                         long long n, long long n_leaves,
                                                         int* __restrict__ leaf_start) {
  long long c = blockIdx.x * (long long)kThreads + threadIdx.x;
  if (c > n_leaves) return;
  long long lo = 0, hi = n;
  while (lo < hi) {
    long long mid = (lo + hi) >> 1;
    if ((long long)keys[mid] < c) lo = mid + 1;
    else hi = mid;
  }
  leaf_start[c] = (int)lo;
}

__global__ void __launch_bounds__(kThreads) k_gather(const double* __restrict__ src,
                                                     const int* __restrict__ perm, long long n,
                                                     double* __restrict__ dst) {
  long long p = blockIdx.x * (long long)kThreads + threadIdx.x;
  if (p < n) dst[p] = src[perm[p]];
}
// Warp per listed leaf: dst[p] = src[perm[p]] for the leaf's sorted positions.
__global__ void __launch_bounds__(kThreads) k_gather_leaves(const double* __restrict__ src,
                                                            const int* __restrict__ perm,
                                                            const int* __restrict__ leaf_start,
                                                            const int* __restrict__ leaves,
                                                            int n_leaves, double* __restrict__ dst) {
  const int w = (int)((blockIdx.x * (long long)kThreads + threadIdx.x) >> 5), lane = threadIdx.x & 31;
  if (w >= n_leaves) return;
  const int q = leaves[w];
  const int e = leaf_start[q + 1];
  for (int p = leaf_start[q] + lane; p < e; p += 32) dst[p] = src[perm[p]];
}
__global__ void __launch_bounds__(kThreads) k_scatter(const double* __restrict__ src,
                                                      const int* __restrict__ perm, long long n,
                                                      double* __restrict__ dst) {
  long long p = blockIdx.x * (long long)kThreads + threadIdx.x;
  if (p < n) dst[perm[p]] = src[p];
}

inline unsigned nblk(long long n) { return (unsigned)((n + kThreads - 1) / kThreads); }

}  // namespace

int minmax_parts(long long n) {
  long long b = (n + kThreads * 8 - 1) / (kThreads * 8);
  return (int)(b < 1 ? 1 : (b > 1184 ? 1184 : b));  // 8 CTAs x 148 SMs
}
void launch_minmax(const double* xy, long long n, double* partial, int nparts, double* out5,
                   cudaStream_t s) {
  k_minmax<<<nparts, kThreads, 0, s>>>(xy, n, partial);
  k_minmax_final<<<1, 32, 0, s>>>(partial, nparts, out5);
}
void launch_bin(const double* xy, long long n, double ox, double oy, double cellL, int gridL,
                uint32_t* keys, int* idx, cudaStream_t s) {
  k_bin<<<nblk(n), kThreads, 0, s>>>(xy, n, ox, oy, cellL, gridL, keys, idx);
}
void launch_gather_points(const double* xy, const int* perm, long long n, double* xs,
                          double* ys, cudaStream_t s) {
  k_gather_points<<<nblk(n), kThreads, 0, s>>>(xy, perm, n, xs, ys);
}
void launch_leaf_start(const uint32_t* keys_sorted, long long n, long long n_leaves,
                       int* leaf_start, cudaStream_t s) {
  k_leaf_start<<<nblk(n_leaves + 1), kThreads, 0, s>>>(keys_sorted, n, n_leaves, leaf_start);
}
void launch_gather(const double* src, const int* perm, long long n, double* dst,
                   cudaStream_t s) {
  k_gather<<<nblk(n), kThreads, 0, s>>>(src, perm, n, dst);
}
void launch_gather_leaves(const double* src, const int* perm, const int* leaf_start,
                          const int* leaves, int n_leaves, double* dst, cudaStream_t s) {
  if (n_leaves > 0)
    k_gather_leaves<<<nblk(32ll * n_leaves), kThreads, 0, s>>>(src, perm, leaf_start, leaves,
                                                                 n_leaves, dst);
}
void launch_scatter(const double* src, const int* perm, long long n, double* dst,
                    cudaStream_t s) {
  k_scatter<<<nblk(n), kThreads, 0, s>>>(src, perm, n, dst);
}

size_t sort_temp_bytes(long long n, int bits) {
  size_t bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, bytes, (const uint32_t*)nullptr, (uint32_t*)nullptr,
                                  (const int*)nullptr, (int*)nullptr, (int)n, 0, bits);
  return bytes;
}
void launch_sort(void* temp, size_t temp_bytes, const uint32_t* k_in, uint32_t* k_out,
                 const int* v_in, int* v_out, long long n, int bits, cudaStream_t s) {
  cub::DeviceRadixSort::SortPairs(temp, temp_bytes, k_in, k_out, v_in, v_out, (int)n, 0, bits,
                                  s);
}

}  // namespace imqk
