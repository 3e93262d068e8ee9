// tree.cu -- bounding square reduction, bit-exact binning, stable radix sort by
// Morton key (hand-written: histogram / scan / ranked scatter), leaf offsets,
// and the sorted<->original gathers.
//
// Bit-exactness (reference partition.cpp:25-33): the finest-level cell index is
// floor(fl(fl(x - o) / cell_L)) with IEEE subtraction and division and no
// contraction (__dsub_rn / __ddiv_rn).  Coarser indices are i_L >> (L - l):
// cell_l = side / 2^(l+1) is an exact power-of-two rescaling of cell_L, so
// fl((x-o)/cell_l) = fl((x-o)/cell_L) * 2^-(L-l) and the floors agree; the
// per-level clamps to [0, grid_l - 1] commute with the shift.
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

// ---- stable LSD radix sort of (key, index) pairs, 8-bit digits ------------
// Per pass: k_sort_hist counts the digit of every 4,096-key tile
// (hist[digit][tile]), k_sort_rowscan / k_sort_digitscan turn the counts into
// the first output position of every (digit, tile), k_sort_scatter re-reads
// the tile and places each pair at that base + its rank among the tile's
// earlier pairs with the same digit.  Earlier = lower position in the input
// of the pass, so every pass is stable and a bucket's points end in ascending
// original index (partition.cpp:35-41 pushes them in index order).
namespace {
constexpr int kSortItems = 16;                                // keys per thread
constexpr int kSortTile = kThreads * kSortItems;              // 4,096 keys per CTA
constexpr int kSortWarps = kThreads / 32;
inline size_t align256(size_t b) { return (b + 255) & ~(size_t)255; }
inline long long sort_tiles(long long n) { return (n + kSortTile - 1) / kSortTile; }

__global__ void __launch_bounds__(kThreads) k_sort_hist(const uint32_t* __restrict__ keys,
                                                        long long n, int shift, long long tiles,
                                                        int* __restrict__ hist) {
  __shared__ int cnt[256];
  cnt[threadIdx.x] = 0;
  __syncthreads();
  const long long base = (long long)blockIdx.x * kSortTile;
#pragma unroll
  for (int r = 0; r < kSortItems; ++r) {
    const long long p = base + r * kThreads + threadIdx.x;
    if (p < n) atomicAdd(&cnt[(keys[p] >> shift) & 255u], 1);
  }
  __syncthreads();
  hist[(size_t)threadIdx.x * tiles + blockIdx.x] = cnt[threadIdx.x];
}

// CTA d: hist[d][.] -> its exclusive prefix sums in place, total[d] = row sum
__global__ void __launch_bounds__(kThreads) k_sort_rowscan(int* __restrict__ hist,
                                                           long long tiles,
                                                           int* __restrict__ total) {
  __shared__ int wsum[kSortWarps];
  __shared__ int carry_s;
  int* row = hist + (size_t)blockIdx.x * tiles;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (threadIdx.x == 0) carry_s = 0;
  __syncthreads();
  for (long long b0 = 0; b0 < tiles; b0 += kThreads) {
    const long long b = b0 + threadIdx.x;
    const int v = b < tiles ? row[b] : 0;
    int inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += t;
    }
    if (lane == 31) wsum[w] = inc;
    __syncthreads();
    int before = carry_s;
    for (int k = 0; k < w; ++k) before += wsum[k];
    if (b < tiles) row[b] = before + inc - v;
    __syncthreads();
    if (threadIdx.x == kThreads - 1) carry_s = before + inc;
    __syncthreads();
  }
  if (threadIdx.x == 0) total[blockIdx.x] = carry_s;
}

// total[256] -> first output position of every digit
__global__ void __launch_bounds__(kThreads) k_sort_digitscan(int* __restrict__ total) {
  __shared__ int v[256];
  v[threadIdx.x] = total[threadIdx.x];
  __syncthreads();
  if (threadIdx.x == 0) {
    int run = 0;
    for (int d = 0; d < 256; ++d) {
      const int c = v[d];
      v[d] = run;
      run += c;
    }
  }
  __syncthreads();
  total[threadIdx.x] = v[threadIdx.x];
}

// Warp w of the CTA owns positions [w * 512, (w + 1) * 512) of the tile and
// walks them 32 at a time, so (warp, round, lane) order is input order.
__global__ void __launch_bounds__(kThreads) k_sort_scatter(
    const uint32_t* __restrict__ k_in, const int* __restrict__ v_in, long long n, int shift,
    long long tiles, const int* __restrict__ hist, const int* __restrict__ digit_base,
    uint32_t* __restrict__ k_out, int* __restrict__ v_out) {
  __shared__ int cnt[kSortWarps][256];   // per-warp digit counts, then bases
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int k = 0; k < kSortWarps; ++k) cnt[k][threadIdx.x] = 0;
  __syncthreads();
  const long long base = (long long)blockIdx.x * kSortTile + (long long)w * (32 * kSortItems);
  uint32_t key[kSortItems];
  int rank[kSortItems];
#pragma unroll
  for (int r = 0; r < kSortItems; ++r) {
    const long long p = base + r * 32 + lane;
    const bool live = p < n;
    key[r] = live ? k_in[p] : 0u;
    const uint32_t d = live ? ((key[r] >> shift) & 255u) : 256u;   // 256: past the end
    const uint32_t peers = __match_any_sync(0xffffffffu, d);
    const int leader = __ffs(peers) - 1;
    int prior = 0;
    if (live && lane == leader) {
      prior = cnt[w][d];
      cnt[w][d] = prior + __popc(peers);
    }
    prior = __shfl_sync(0xffffffffu, prior, leader);
    rank[r] = prior + __popc(peers & ((1u << lane) - 1u));
    __syncwarp();
  }
  __syncthreads();
  {  // digit d = threadIdx.x: counts of the warps -> output base of each warp
    const int d = threadIdx.x;
    int run = digit_base[d] + hist[(size_t)d * tiles + blockIdx.x];
    for (int k = 0; k < kSortWarps; ++k) {
      const int c = cnt[k][d];
      cnt[k][d] = run;
      run += c;
    }
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < kSortItems; ++r) {
    const long long p = base + r * 32 + lane;
    if (p < n) {
      const int dst = cnt[w][(key[r] >> shift) & 255u] + rank[r];
      k_out[dst] = key[r];
      v_out[dst] = v_in[p];
    }
  }
}
}  // namespace

// temp: hist[256][tiles], total[256], alternate key and value buffers
size_t sort_temp_bytes(long long n, int /*bits*/) {
  return align256((size_t)256 * sort_tiles(n) * sizeof(int)) + align256(256 * sizeof(int)) +
         2 * align256((size_t)n * sizeof(uint32_t));
}
void launch_sort(void* temp, size_t /*temp_bytes*/, const uint32_t* k_in, uint32_t* k_out,
                 const int* v_in, int* v_out, long long n, int bits, cudaStream_t s) {
  if (n <= 0) return;
  const long long tiles = sort_tiles(n);
  unsigned char* t = static_cast<unsigned char*>(temp);
  int* hist = reinterpret_cast<int*>(t);
  t += align256((size_t)256 * tiles * sizeof(int));
  int* total = reinterpret_cast<int*>(t);
  t += align256(256 * sizeof(int));
  uint32_t* k_alt = reinterpret_cast<uint32_t*>(t);
  t += align256((size_t)n * sizeof(uint32_t));
  int* v_alt = reinterpret_cast<int*>(t);
  const int passes = bits <= 0 ? 1 : (bits + 7) / 8;
  const uint32_t* ks = k_in;
  const int* vs = v_in;
  for (int pass = 0; pass < passes; ++pass) {
    // the last pass writes k_out / v_out; the ones before alternate
    const bool to_out = ((passes - 1 - pass) & 1) == 0;
    uint32_t* kd = to_out ? k_out : k_alt;
    int* vd = to_out ? v_out : v_alt;
    k_sort_hist<<<(unsigned)tiles, kThreads, 0, s>>>(ks, n, 8 * pass, tiles, hist);
    k_sort_rowscan<<<256, kThreads, 0, s>>>(hist, tiles, total);
    k_sort_digitscan<<<1, kThreads, 0, s>>>(total);
    k_sort_scatter<<<(unsigned)tiles, kThreads, 0, s>>>(ks, vs, n, 8 * pass, tiles, hist, total,
                                                        kd, vd);
    ks = kd;
    vs = vd;
  }
}

}  // namespace imqk
