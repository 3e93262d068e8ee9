// expansion.cu -- far-field pipeline of the fast IMQ product on sm_100a.
//
//   P2M (leaf)   raw planar moments of every finest block from its points
//   M2M          exact binomial translation of child moments to the parent
//   transform    mu -> far-field coefficients C_{m,k} (one small linear map)
//   M2P          per (target point, source block) evaluation, the hot kernel
//
// All of it is exact in real arithmetic with respect to the reference's
// per-level moment formation (fastmv.cpp:79-100) and M2P evaluation
// (fastmv.cpp:104-138, specfun.cpp:73-91): the same bounding square, levels,
// buckets, interaction lists and truncation order.  What changes is how the
// arithmetic is organised:
//   * moments are kept as complex sums mu_{m,i} = sum u |e|^{2i} e^m, which
//     equal the reference's (w - i v)_{n,m} / P_n^m(0) with n = m + 2i; the
//     n-m odd moments of the reference are identically zero and not stored;
//   * d_{n,m} P_n^m(0) and the monomial form of P_n^m(t/rho) rho^-(n+1) are
//     folded into C_{m,k}, so a far pair is a complex Horner scheme in
//     conj(xi) = (dx, -dy)/rho^2 with real-Horner inner polynomials in
//     q = 1/rho^2: ~M^2+4M DFMA per pair instead of a Legendre recurrence
//     with one division per (n, m).
#include <cstdio>
#include <algorithm>
#include <cstdlib>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <set>
#include <tuple>

#include "imq_device.cuh"
#include "imq_kernels.hpp"

#ifndef IMQ_M2T_SMALL
#define IMQ_M2T_SMALL 1024  // parents up to which a level uses the warp-per-parent kernel (0 / 1024 / 4096 / 16384: moments 2.23 / 2.18 / 2.28 / 2.61 ms at config 4)
#endif

namespace imqk {
using namespace imqdev;

namespace {

__host__ __device__ __forceinline__ int mu_offset(int M, int m) {
  // sum_{m' < m} (floor((M - m') / 2) + 1)
  int o = 0;
  for (int mm = 0; mm < m; ++mm) o += (M - mm) / 2 + 1;
  return o;
}
__host__ __device__ __forceinline__ void mu_unindex(int M, int o, int& m, int& i) {
  m = 0;
  while (true) {
    int sz = (M - m) / 2 + 1;
    if (o < sz) break;
    o -= sz;
    ++m;
  }
  i = o;
}

// Horner layout (host_math.hpp): group m holds k = top(m)..m.
__host__ __device__ constexpr int hz_top(int M, int m) { return M - ((M - m) & 1); }
__host__ __device__ constexpr int hz_count(int M) {
  return (M + 1) * (M + 2) / 2 - (M + 1) / 2;
}

// Opt a kernel into large dynamic shared memory.  The attribute is per
// (kernel, device context) and is an upper bound, so it is raised to the
// largest size requested so far and never lowered (lowering it after a larger
// launch of another operator made that operator's next launch fail).
void ensure_smem_attr(const void* kern, size_t bytes) {
  static std::mutex mtx;
  static std::map<std::pair<const void*, int>, size_t> done;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mtx);
  size_t& cur = done[{kern, dev}];
  if (bytes > cur) {
    const cudaError_t e =
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e != cudaSuccess) {
      cudaGetLastError();
      throw std::runtime_error(std::string("cudaFuncSetAttribute (shared memory): ") +
                               cudaGetErrorString(e));
    }
    cur = bytes;
  }
}

__device__ __forceinline__ int block_count(const TreeParams& P, int level, uint32_t q) {
  int sh = 2 * (P.L - level);
  return P.leaf_start[(size_t)(q + 1) << sh] - P.leaf_start[(size_t)q << sh];
}
__device__ __forceinline__ int block_first(const TreeParams& P, int level, uint32_t q) {
  return P.leaf_start[(size_t)q << (2 * (P.L - level))];
}

// ------------------------------------------------------------------- P2M ---
// Warp per finest block; lane m accumulates mu_{m,i}, i = 0..(M-m)/2, over
// the block's points in sorted (= ascending original index) order.
template <int M>
__global__ void __launch_bounds__(128) k_p2m_leaf(const TreeParams P, const double* __restrict__ u_s,
                                                  double2* __restrict__ mu,
                                                  const int* __restrict__ leaf_list, int n_list) {
  constexpr int NI = M / 2 + 1;
  const int lane = threadIdx.x & 31;
  const long long wid = (long long)blockIdx.x * 4 + (threadIdx.x >> 5);
  const long long n_leaves = leaf_list ? n_list : 1ll << (2 * (P.L + 1));
  if (wid >= n_leaves) return;
  const long long leaf = leaf_list ? leaf_list[wid] : wid;
  const int s = P.leaf_start[leaf], e = P.leaf_start[leaf + 1];
  if (s == e) return;
  int li, lj;
  demorton((uint32_t)leaf, li, lj);
  const double zx = block_center(P.ox, li, P.cell[P.L]);
  const double zy = block_center(P.oy, lj, P.cell[P.L]);
  const int m = lane;
  double ar[NI], ai[NI];
#pragma unroll
  for (int i = 0; i < NI; ++i) ar[i] = ai[i] = 0.0;
  for (int p = s; p < e; ++p) {
    const double ex = P.xs[p] - zx, ey = P.ys[p] - zy;
    const double e2 = fma(ex, ex, ey * ey);
    // u * e^m by binary powering
    double pr = u_s[p], pi = 0.0, br = ex, bi = ey;
    int mm = m;
#pragma unroll
    for (int b = 0; b < 5; ++b) {
      if (mm & 1) {
        const double tr = pr * br - pi * bi;
        pi = pr * bi + pi * br;
        pr = tr;
      }
      const double sr = br * br - bi * bi;
      bi = 2.0 * br * bi;
      br = sr;
      mm >>= 1;
    }
    double e2p = 1.0;
#pragma unroll
    for (int i = 0; i < NI; ++i) {
      ar[i] = fma(pr, e2p, ar[i]);
      ai[i] = fma(pi, e2p, ai[i]);
      e2p *= e2;
    }
  }
  if (m <= M) {
    double2* out = mu + P.mu_off[P.L] + (size_t)leaf * P.Ke + mu_offset(M, m);
#pragma unroll
    for (int i = 0; i < NI; ++i)
      if (m + 2 * i <= M) out[i] = make_double2(ar[i], ai[i]);
  }
}

// Warp per finest block, G lanes per point (32/G points of the block per
// pass): lane g of a group accumulates the moments of m in {g, g+G, g+2G, ...}
// (m <= M).  e^g comes from binary powering of e (log2 G steps, whose last
// base is e^G), e^{g+kG} from one complex product each.  After the pass the
// 32/G groups are folded by shuffles in a fixed order (deterministic).
template <int M, int G, int WPL>
__global__ void __launch_bounds__(32 * (WPL > 4 ? WPL : 4), WPL == 1 ? 4 : 1) k_p2m_leaf_g(
    const TreeParams P, const double* __restrict__ u_s, double2* __restrict__ mu,
    const int* __restrict__ leaf_list, int n_list) {
  // WPL warps per leaf (large leaves split their points over several warps;
  // the partial sums are combined through shared memory in a fixed order)
  constexpr int NI = M / 2 + 1;
  constexpr int NM = (M + G) / G;  // m values per lane
  constexpr int LOGG = G == 8 ? 3 : (G == 16 ? 4 : 5);
  constexpr int WARPS = WPL > 4 ? WPL : 4;
  constexpr int LPC = WARPS / WPL;  // leaves per CTA
  __shared__ double2 red[WPL > 1 ? WARPS : 1][G][NM][NI];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane % G, grp = lane / G;
  const int sub = warp % WPL;
  const long long wid = (long long)blockIdx.x * LPC + warp / WPL;
  const long long n_leaves = leaf_list ? n_list : 1ll << (2 * (P.L + 1));
  const bool live = wid < n_leaves;
  const long long leaf = live ? (leaf_list ? leaf_list[wid] : wid) : 0;
  const int s = live ? P.leaf_start[leaf] : 0, e = live ? P.leaf_start[leaf + 1] : 0;
  if (WPL == 1 && s == e) return;
  int li, lj;
  demorton((uint32_t)leaf, li, lj);
  const double zx = block_center(P.ox, li, P.cell[P.L]);
  const double zy = block_center(P.oy, lj, P.cell[P.L]);
  double ar[NM][NI], ai[NM][NI];
#pragma unroll
  for (int k = 0; k < NM; ++k)
#pragma unroll
    for (int i = 0; i < NI; ++i) ar[k][i] = ai[k][i] = 0.0;
  // the next point's coordinates and weight are loaded one trip ahead (the
  // loop is otherwise bound by their load latency)
  constexpr int kStep = WPL * (32 / G);
  int p = s + grp + sub * (32 / G);
  double nx = 0.0, ny = 0.0, nu = 0.0;
  if (p < e) {
    nx = P.xs[p];
    ny = P.ys[p];
    nu = u_s[p];
  }
#pragma unroll 1
  for (; p < e; p += kStep) {
    const double ex = nx - zx, ey = ny - zy, uu = nu;
    if (p + kStep < e) {
      nx = P.xs[p + kStep];
      ny = P.ys[p + kStep];
      nu = u_s[p + kStep];
    }
    const double e2 = fma(ex, ex, ey * ey);
    double pr = uu, pi = 0.0, br = ex, bi = ey;
#pragma unroll
    for (int b = 0; b < LOGG; ++b) {
      if ((g >> b) & 1) {
        const double tr = pr * br - pi * bi;
        pi = pr * bi + pi * br;
        pr = tr;
      }
      const double sr = br * br - bi * bi;
      bi = 2.0 * br * bi;
      br = sr;
    }
    // br + i bi = e^G;  pr + i pi = u e^g
#pragma unroll
    for (int k = 0; k < NM; ++k) {
      double e2p = 1.0;
#pragma unroll
      for (int i = 0; i < NI; ++i) {
        if (k * G + 2 * i <= M) {  // compile-time bound for the largest m of slot k
          ar[k][i] = fma(pr, e2p, ar[k][i]);
          ai[k][i] = fma(pi, e2p, ai[k][i]);
        }
        e2p *= e2;
      }
      if (k + 1 < NM) {
        const double tr = pr * br - pi * bi;
        pi = pr * bi + pi * br;
        pr = tr;
      }
    }
  }
  // fold the 32/G point groups onto lanes 0..G-1
#pragma unroll
  for (int off = G; off < 32; off <<= 1)
#pragma unroll
    for (int k = 0; k < NM; ++k)
#pragma unroll
      for (int i = 0; i < NI; ++i) {
        ar[k][i] += __shfl_down_sync(0xffffffffu, ar[k][i], off);
        ai[k][i] += __shfl_down_sync(0xffffffffu, ai[k][i], off);
      }
  if constexpr (WPL > 1) {  // combine the leaf's warps in a fixed order
    if (grp == 0)
#pragma unroll
      for (int k = 0; k < NM; ++k)
#pragma unroll
        for (int i = 0; i < NI; ++i) red[warp][g][k][i] = make_double2(ar[k][i], ai[k][i]);
    __syncthreads();
    if (sub != 0 || !live || s == e) return;
    if (grp == 0)
#pragma unroll
      for (int k = 0; k < NM; ++k)
#pragma unroll
        for (int i = 0; i < NI; ++i) {
          double sr = 0.0, si = 0.0;
          for (int w = 0; w < WPL; ++w) {
            const double2 v = red[warp + w][g][k][i];
            sr += v.x;
            si += v.y;
          }
          ar[k][i] = sr;
          ai[k][i] = si;
        }
  }
  if (grp == 0) {
    double2* out = mu + P.mu_off[P.L] + (size_t)leaf * P.Ke;
#pragma unroll
    for (int k = 0; k < NM; ++k) {
      const int m = g + k * G;
      if (m > M) continue;
      const int o = mu_offset(M, m);
#pragma unroll
      for (int i = 0; i < NI; ++i)
        if (m + 2 * i <= M) out[o + i] = make_double2(ar[k][i], ai[k][i]);
    }
  }
}

// Generic order: thread per (finest block, moment index), direct powering.
__global__ void __launch_bounds__(128) k_p2m_leaf_generic(const TreeParams P,
                                                          const double* __restrict__ u_s,
                                                          double2* __restrict__ mu,
                                                          const int* __restrict__ leaf_list,
                                                          int n_list) {
  const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long n_leaves = leaf_list ? n_list : 1ll << (2 * (P.L + 1));
  const long long wid = gid / P.Ke;
  const int o = (int)(gid % P.Ke);
  if (wid >= n_leaves) return;
  const long long leaf = leaf_list ? leaf_list[wid] : wid;
  const int s = P.leaf_start[leaf], e = P.leaf_start[leaf + 1];
  if (s == e) return;
  int li, lj, m, i;
  demorton((uint32_t)leaf, li, lj);
  mu_unindex(P.M, o, m, i);
  const double zx = block_center(P.ox, li, P.cell[P.L]);
  const double zy = block_center(P.oy, lj, P.cell[P.L]);
  double ar = 0.0, ai = 0.0;
  for (int p = s; p < e; ++p) {
    const double ex = P.xs[p] - zx, ey = P.ys[p] - zy;
    const double e2 = fma(ex, ex, ey * ey);
    double pr = u_s[p], pi = 0.0, br = ex, bi = ey;
    for (int mm = m; mm; mm >>= 1) {
      if (mm & 1) {
        const double tr = pr * br - pi * bi;
        pi = pr * bi + pi * br;
        pr = tr;
      }
      const double sr = br * br - bi * bi;
      bi = 2.0 * br * bi;
      br = sr;
    }
    double e2p = 1.0, b2 = e2;
    for (int ii = i; ii; ii >>= 1) {
      if (ii & 1) e2p *= b2;
      b2 *= b2;
    }
    ar = fma(pr, e2p, ar);
    ai = fma(pi, e2p, ai);
  }
  mu[P.mu_off[P.L] + (size_t)leaf * P.Ke + o] = make_double2(ar, ai);
}

// ------------------------------------------------------------------- M2M ---
// CTA per parent block at `level`; thread per output moment (m, i), i.e.
// (a, b) = (m + i, i) of sum u e^a conj(e)^b.  With e' = e + d (d = child
// centre - parent centre):
//   mu'_{a,b} = sum_{p<=a, r<=b} C(a,p) C(b,r) d^{a-p} conj(d)^{b-r} N_{p,r},
//   N_{p,r} = mu_{p-r, r} (p >= r) or conj(mu_{r-p, p}) (p < r).
// The four children are folded into one pass: the translated sum is linear in
// N, so the CTA first forms per child the d-power tables, then every thread
// walks its (p, r) triangle once per child.  Index / binomial tables live in
// shared memory (no per-term integer search).
__global__ void k_m2m(const TreeParams P, int level, double2* __restrict__ mu,
                      const double* __restrict__ binom) {
  extern __shared__ double2 sm[];
  const int M = P.M, Ke = P.Ke;
  double2* cm = sm;                          // [4][Ke]
  double2* dp = sm + 4 * Ke;                 // [4][M+1] powers of d
  double* bn = reinterpret_cast<double*>(dp + 4 * (M + 1));  // [(M+1)^2]
  int* moff = reinterpret_cast<int*>(bn + (M + 1) * (M + 1)); // [M+1]
  const uint32_t q = blockIdx.x;
  if (block_count(P, level, q) == 0) return;
  int qi, qj;
  demorton(q, qi, qj);
  const double zx = block_center(P.ox, qi, P.cell[level]);
  const double zy = block_center(P.oy, qj, P.cell[level]);
  for (int k = threadIdx.x; k < (M + 1) * (M + 1); k += blockDim.x) bn[k] = binom[k];
  if (threadIdx.x <= M) moff[threadIdx.x] = mu_offset(M, threadIdx.x);
  int have = 0;
  for (int c = 0; c < 4; ++c) {
    const uint32_t ch = 4 * q + c;
    const bool ne = block_count(P, level + 1, ch) > 0;
    have |= (ne ? 1 : 0) << c;
    if (!ne) continue;
    const double2* src = mu + P.mu_off[level + 1] + (size_t)ch * Ke;
    for (int o = threadIdx.x; o < Ke; o += blockDim.x) cm[c * Ke + o] = src[o];
    if (threadIdx.x == 32 * (c % max(1, (int)(blockDim.x / 32)))) {
      int ci, cj;
      demorton(ch, ci, cj);
      const double dx = block_center(P.ox, ci, P.cell[level + 1]) - zx;
      const double dy = block_center(P.oy, cj, P.cell[level + 1]) - zy;
      double pr = 1.0, pi = 0.0;
      for (int k = 0; k <= M; ++k) {
        dp[c * (M + 1) + k] = make_double2(pr, pi);
        const double tr = pr * dx - pi * dy;
        pi = pr * dy + pi * dx;
        pr = tr;
      }
    }
  }
  __syncthreads();
  for (int o = threadIdx.x; o < Ke; o += blockDim.x) {
    int m = 0, oo = o;
    while (oo >= (M - m) / 2 + 1) {
      oo -= (M - m) / 2 + 1;
      ++m;
    }
    const int i = oo, a = m + i, b = i;
    double sr = 0.0, si = 0.0;
    for (int c = 0; c < 4; ++c) {
      if (!((have >> c) & 1)) continue;
      const double2* N = cm + c * Ke;
      const double2* D = dp + c * (M + 1);
      for (int p = 0; p <= a; ++p) {
        double ir = 0.0, ii = 0.0;
        for (int r = 0; r <= b; ++r) {
          double2 v;
          if (p >= r) {
            v = N[moff[p - r] + r];
          } else {
            v = N[moff[r - p] + p];
            v.y = -v.y;
          }
          const double2 d = D[b - r];  // conj(d)^{b-r} = conj(d^{b-r})
          const double cb = bn[b * (M + 1) + r];
          ir = fma(cb, fma(d.x, v.x, d.y * v.y), ir);
          ii = fma(cb, fma(d.x, v.y, -d.y * v.x), ii);
        }
        const double2 d = D[a - p];
        const double ca = bn[a * (M + 1) + p];
        sr = fma(ca, fma(d.x, ir, -d.y * ii), sr);
        si = fma(ca, fma(d.x, ii, d.y * ir), si);
      }
    }
    // m = 0 moments are real by construction (conjugate-symmetric terms);
    // keep their imaginary part exactly zero as the reference's v_{n,0} are.
    mu[P.mu_off[level] + (size_t)q * Ke + o] = make_double2(sr, m == 0 ? 0.0 : si);
  }
}

// ------------------------------------------------------------- transform ---
// CTA per kTrBlocks consecutive blocks: the sparse table is staged once in
// shared memory, then each block's K_e moments -> K coefficients.
constexpr int kTrBlocks = 8;
__global__ void k_transform(const TreeParams P, int level, const double2* __restrict__ mu,
                            double2* __restrict__ coef, const TransformTable T,
                            const int* __restrict__ block_list, int n_blocks, int nnz) {
  extern __shared__ double2 sm[];
  double2* smu = sm;                                          // [Ke]
  double* sval = reinterpret_cast<double*>(sm + P.Ke);        // [nnz]
  int* soff = reinterpret_cast<int*>(sval + nnz);             // [K + 1]
  int* sidx = soff + P.K + 1;                                 // [nnz]
  for (int e = threadIdx.x; e < nnz; e += blockDim.x) {
    sval[e] = T.val[e];
    sidx[e] = T.idx[e];
  }
  for (int o = threadIdx.x; o <= P.K; o += blockDim.x) soff[o] = T.off[o];
  for (int bb = 0; bb < kTrBlocks; ++bb) {
    const int b = blockIdx.x * kTrBlocks + bb;
    if (b >= n_blocks) break;
    const uint32_t q = block_list ? (uint32_t)block_list[b] : (uint32_t)b;
    if (block_count(P, level, q) == 0) continue;  // uniform across the CTA
    __syncthreads();
    const double2* src = mu + P.mu_off[level] + (size_t)q * P.Ke;
    for (int o = threadIdx.x; o < P.Ke; o += blockDim.x) smu[o] = src[o];
    __syncthreads();
    double2* dst = coef + P.coef_off[level] + (size_t)q * P.K;
    for (int o = threadIdx.x; o < P.K; o += blockDim.x) {
      double cr = 0.0, ci = 0.0;
      for (int e = soff[o]; e < soff[o + 1]; ++e) {
        const double2 v = smu[sidx[e]];
        cr = fma(sval[e], v.x, cr);
        ci = fma(sval[e], v.y, ci);
      }
      dst[o] = make_double2(cr, ci);
    }
  }
}

// ----------------------------------------------------- M2M + transform ---
// One warp per parent block q at `level` (kM2tWarps parents per CTA), fused:
//   1. the four children's moments N^c (level + 1, contiguous in mu) are
//      staged in shared memory;
//   2. (coef_child) their far-field coefficients C = T N^c are written -- the
//      transform of level + 1 happens here, while the moments are on chip;
//   3. the exact binomial translation (reference moments at the parent centre,
//      fastmv.cpp:79-100 formed from the children instead of the points):
//        mu'_{a,b} = sum_c sum_{p<=a} C(a,p) d_c^{a-p} Y^c_{p,b},
//        Y^c_{p,b} = sum_{r<=b} C(b,r) conj(d_c)^{b-r} N^c_{p,r},
//      (a, b) = (m + i, i), N_{p,r} = mu_{p-r,r} (p >= r) or conj(mu_{r-p,p}).
//      Separated into the r-sum and the p-sum this is ~1.3k complex MACs per
//      child at M = 16 instead of the dense [8 Ke x 2 Ke] product's 26k real
//      FMA per child; the per-level tables V_c[a][p] = C(a,p) d_c^{a-p} and
//      W_c[b][r] = C(b,r) conj(d_c)^{b-r} (d_c = +-h +- i h, exact child
//      offsets) live in shared memory;
//   4. mu' is written (and, with coef_parent, transformed too: level 1).
// The children are summed in a fixed order (c = 0..3): deterministic.
constexpr int kM2tWarps = 8;
constexpr long long kM2tSmallLevel = IMQ_M2T_SMALL;
constexpr int kM2tMaxAcc = 8;  // Ke <= 256 outputs per warp (M <= 30)
struct M2tLayout {             // dynamic shared memory layout (bytes)
  int M, H, Ke, K, nnz, ny, ysz;
  size_t v, w, tval, tidx, toff, moff, otab, ytab, yoff, warp0, per_warp, total;
  // with_v = false: the specialised kernel (no V table in shared memory)
  __host__ __device__ M2tLayout(int M_, int Ke_, int K_, int nnz_, bool with_v = true)
      : M(M_), Ke(Ke_), K(K_), nnz(nnz_) {
    H = M / 2;
    ny = 0;
    for (int b = 0; b <= H; ++b) ny += M - b + 1;
    ysz = ny > (H + 1) * (M + 1) ? ny : (H + 1) * (M + 1);
    size_t o = 0;
    auto take = [&](size_t bytes) { const size_t r = o; o += (bytes + 15) & ~(size_t)15; return r; };
    v = take(with_v ? (size_t)4 * (M + 1) * (M + 1) * 16 : 0);
    w = take((size_t)4 * (H + 1) * (H + 1) * 16);
    tval = take((size_t)nnz * 8);
    tidx = take((size_t)nnz * 4);
    toff = take((size_t)(K + 1) * 4);
    moff = take((size_t)(M + 1) * 4);
    otab = take((size_t)Ke * 4);
    ytab = take((size_t)ny * 4);
    yoff = take((size_t)(H + 1) * 4);
    warp0 = o;
    const int ytot = ysz > 4 * Ke ? ysz : 4 * Ke;  // generic: Y; specialised: partial parents
    per_warp = ((size_t)(4 * Ke + ytot + Ke) * 16 + 15) & ~(size_t)15;
    total = warp0 + kM2tWarps * per_warp;
  }
};

__global__ void __launch_bounds__(kM2tWarps * 32) k_m2m_tr(
    const TreeParams P, int level, const int* __restrict__ plist, long long p0, long long np,
    const double2* __restrict__ mu_in, double2* __restrict__ mu_out,
    double2* __restrict__ coef_child, double2* __restrict__ coef_parent,
    const double2* __restrict__ Vg, const double2* __restrict__ Wg, const TransformTable T) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int M = P.M, Ke = P.Ke, K = P.K;
  const M2tLayout lay(M, Ke, K, T.nnz);
  const int H = lay.H, ny = lay.ny, M1 = M + 1, H1 = H + 1;
  double2* V = reinterpret_cast<double2*>(smem + lay.v);
  double2* W = reinterpret_cast<double2*>(smem + lay.w);
  double* tval = reinterpret_cast<double*>(smem + lay.tval);
  int* tidx = reinterpret_cast<int*>(smem + lay.tidx);
  int* toff = reinterpret_cast<int*>(smem + lay.toff);
  int* moff = reinterpret_cast<int*>(smem + lay.moff);
  int* otab = reinterpret_cast<int*>(smem + lay.otab);  // (a << 8) | b
  int* ytab = reinterpret_cast<int*>(smem + lay.ytab);  // (p << 8) | b
  int* yoff = reinterpret_cast<int*>(smem + lay.yoff);  // Y index of (0, b)
  for (int o = threadIdx.x; o < 4 * M1 * M1; o += blockDim.x) V[o] = Vg[o];
  for (int o = threadIdx.x; o < 4 * H1 * H1; o += blockDim.x) W[o] = Wg[o];
  for (int o = threadIdx.x; o < T.nnz; o += blockDim.x) {
    tval[o] = T.val[o];
    tidx[o] = T.idx[o];
  }
  for (int o = threadIdx.x; o <= K; o += blockDim.x) toff[o] = T.off[o];
  if (threadIdx.x == 0) {
    int off = 0, o = 0, e = 0;
    for (int m = 0; m <= M; ++m) {
      moff[m] = off;
      for (int i = 0; m + 2 * i <= M; ++i) otab[o++] = ((m + i) << 8) | i;
      off += (M - m) / 2 + 1;
    }
    for (int b = 0; b <= H; ++b) {
      yoff[b] = e;
      for (int p = 0; p + b <= M; ++p) ytab[e++] = (p << 8) | b;
    }
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double2* N = reinterpret_cast<double2*>(smem + lay.warp0 + (size_t)warp * lay.per_warp);
  double2* Y = N + 4 * Ke;
  double2* MU = Y + ny;
  for (long long it = (long long)blockIdx.x * kM2tWarps + warp; it < np;
       it += (long long)gridDim.x * kM2tWarps) {
    const uint32_t q = plist ? (uint32_t)plist[it] : (uint32_t)(p0 + it);
    int have = 0;
#pragma unroll
    for (int c = 0; c < 4; ++c) have |= (block_count(P, level + 1, 4 * q + c) > 0 ? 1 : 0) << c;
    if (!have) continue;  // the parent's moments stay zero
    __syncwarp();
    const double2* src = mu_in + (size_t)(4 * q) * Ke;
    for (int o = lane; o < 4 * Ke; o += 32)
      N[o] = ((have >> (o / Ke)) & 1) ? src[o] : make_double2(0.0, 0.0);
    __syncwarp();
    if (coef_child) {  // transform of the children (level + 1)
      for (int e = lane; e < 4 * K; e += 32) {
        const int c = e / K, o = e - c * K;
        if (!((have >> c) & 1)) continue;
        double cr = 0.0, ci = 0.0;
        for (int t = toff[o]; t < toff[o + 1]; ++t) {
          const double2 x = N[c * Ke + tidx[t]];
          cr = fma(tval[t], x.x, cr);
          ci = fma(tval[t], x.y, ci);
        }
        coef_child[(size_t)(4 * q) * K + e] = make_double2(cr, ci);
      }
    }
    double ar[kM2tMaxAcc], ai[kM2tMaxAcc];
#pragma unroll
    for (int k = 0; k < kM2tMaxAcc; ++k) ar[k] = ai[k] = 0.0;
    for (int c = 0; c < 4; ++c) {
      if (!((have >> c) & 1)) continue;
      const double2* Nc = N + c * Ke;
      const double2* Wc = W + c * H1 * H1;
      const double2* Vc = V + c * M1 * M1;
      for (int e = lane; e < ny; e += 32) {  // Y[p][b] = sum_r W[b][r] N(p, r)
        const int p = ytab[e] >> 8, b = ytab[e] & 255;
        double yr = 0.0, yi = 0.0;
        for (int r = 0; r <= b; ++r) {
          double2 x;
          if (p >= r) {
            x = Nc[moff[p - r] + r];
          } else {
            x = Nc[moff[r - p] + p];
            x.y = -x.y;
          }
          const double2 w = Wc[b * H1 + r];
          yr = fma(w.x, x.x, fma(-w.y, x.y, yr));
          yi = fma(w.x, x.y, fma(w.y, x.x, yi));
        }
        Y[e] = make_double2(yr, yi);
      }
      __syncwarp();
#pragma unroll
      for (int k = 0; k < kM2tMaxAcc; ++k) {  // mu'[a][b] += sum_p V[a][p] Y[p][b]
        const int o = lane + 32 * k;
        if (o >= Ke) break;
        const int a = otab[o] >> 8, b = otab[o] & 255;
        const double2* y = Y + yoff[b];
        double sr = ar[k], si = ai[k];
        for (int p = 0; p <= a; ++p) {
          const double2 v = Vc[a * M1 + p], x = y[p];
          sr = fma(v.x, x.x, fma(-v.y, x.y, sr));
          si = fma(v.x, x.y, fma(v.y, x.x, si));
        }
        ar[k] = sr;
        ai[k] = si;
      }
      __syncwarp();
    }
    double2* dst = mu_out + (size_t)q * Ke;
#pragma unroll
    for (int k = 0; k < kM2tMaxAcc; ++k) {
      const int o = lane + 32 * k;
      if (o >= Ke) break;
      // m = 0 moments are real by construction (the reference's v_{n,0} = 0)
      const double2 r = make_double2(ar[k], (otab[o] >> 8) == (otab[o] & 255) ? 0.0 : ai[k]);
      dst[o] = r;
      MU[o] = r;
    }
    if (coef_parent) {
      __syncwarp();
      for (int o = lane; o < K; o += 32) {
        double cr = 0.0, ci = 0.0;
        for (int t = toff[o]; t < toff[o + 1]; ++t) {
          const double2 x = MU[tidx[t]];
          cr = fma(tval[t], x.x, cr);
          ci = fma(tval[t], x.y, ci);
        }
        coef_parent[(size_t)q * K + o] = make_double2(cr, ci);
      }
    }
  }
}

// Specialised orders: eight parents per warp, lane = (parent slot, child c),
// every lane running the same code on its own child (no divergence, nothing
// looked up per MAC; the generic kernel above is bound by shared-memory
// bandwidth, ~3 LDS per complex MAC):
//   transform: C = T N^c, table entries are warp-wide broadcasts;
//   translation, column by column (b = 0..M/2, compile-time):
//     Y[p] = sum_{r <= b} W_c[b][r] N(p, r),  p = 0..M-b  (W row in registers)
//     then the Taylor shift by d_c in registers (Y[p] += d_c Y[p-1], p
//     descending, repeated): Y[a] = sum_p C(a,p) d_c^{a-p} Y[p], exactly the
//     p-sum with no binomials or powers of d_c; a = b..M-b are the column's
//     outputs;
//   the four children of a parent are summed by two xor-shuffles, bitwise
//   identical on the four lanes (commutative pairs): deterministic.
constexpr int kM2sWarps = 2, kM2sSlots = 8;  // parents per warp
constexpr bool kM2sStage = true;  // stage the children in shared memory (L1-direct: 0.99 vs 0.78 ms at cfg4 level 7)
template <int M>
__host__ __device__ constexpr int mu_off_c(int m) {
  int o = 0;
  for (int mm = 0; mm < m; ++mm) o += (M - mm) / 2 + 1;
  return o;
}

// (one column per call: inlined, the compiler interleaves the columns and
// runs out of registers)
template <int M, int B>
__device__ __noinline__ void m2m_column(const double2* __restrict__ Nc, const double2* __restrict__ Wc,
                                        double dre, double dim, double2* __restrict__ dst, int c,
                                        bool write);
template <int M, int B>
__device__ __forceinline__ void m2m_columns(const double2* __restrict__ Nc,
                                            const double2* __restrict__ Wc, double dre,
                                            double dim, double2* __restrict__ dst, int c,
                                            bool write) {
  if constexpr (B <= M / 2) {
    m2m_column<M, B>(Nc, Wc, dre, dim, dst, c, write);
    m2m_columns<M, B + 1>(Nc, Wc, dre, dim, dst, c, write);
  }
}
template <int M, int B>
__device__ __noinline__ void m2m_column(const double2* __restrict__ Nc,
                                            const double2* __restrict__ Wc, double dre,
                                            double dim, double2* __restrict__ dst, int c,
                                            bool write) {
  {
    constexpr int A = M - B, H1 = M / 2 + 1;
    double yr[A + 1], yi[A + 1];
    {
      double wr[B + 1], wi[B + 1];
#pragma unroll
      for (int r = 0; r <= B; ++r) {
        const double2 w = Wc[B * H1 + r];
        wr[r] = w.x;
        wi[r] = w.y;
      }
#pragma unroll
      for (int p = 0; p <= A; ++p) {
        double sr = 0.0, si = 0.0;
#pragma unroll
        for (int r = 0; r <= B; ++r) {
          double2 x;
          if (p >= r) {
            x = Nc[mu_off_c<M>(p - r) + r];
          } else {
            x = Nc[mu_off_c<M>(r - p) + p];
            x.y = -x.y;
          }
          sr = fma(wr[r], x.x, fma(-wi[r], x.y, sr));
          si = fma(wr[r], x.y, fma(wi[r], x.x, si));
        }
        yr[p] = sr;
        yi[p] = si;
      }
    }
    // Taylor shift: after pass k, y[p] (p >= k) has absorbed d y[p-1]
#pragma unroll
    for (int k = 1; k <= A; ++k)
#pragma unroll
      for (int p = A; p >= k; --p) {
        const double tr = fma(dre, yr[p - 1], fma(-dim, yi[p - 1], yr[p]));
        const double ti = fma(dre, yi[p - 1], fma(dim, yr[p - 1], yi[p]));
        yr[p] = tr;
        yi[p] = ti;
      }
    // the parent's column: sum over the four child lanes, a fixed pairing
#pragma unroll
    for (int a = B; a <= A; ++a) {
      double vr = yr[a], vi = yi[a];
      vr += __shfl_xor_sync(0xffffffffu, vr, 1);
      vi += __shfl_xor_sync(0xffffffffu, vi, 1);
      vr += __shfl_xor_sync(0xffffffffu, vr, 2);
      vi += __shfl_xor_sync(0xffffffffu, vi, 2);
      // m = a - B = 0 moments are real by construction (reference v_{n,0} = 0)
      if (write && ((a - B) & 3) == c) dst[mu_off_c<M>(a - B) + B] = make_double2(vr, a == B ? 0.0 : vi);
    }
  }
}

template <int M>
__global__ void __launch_bounds__(kM2sWarps * 32) k_m2m_tr_s(
    const TreeParams P, int level, const int* __restrict__ plist, long long p0, long long np,
    const double2* __restrict__ mu_in, double2* __restrict__ mu_out,
    double2* __restrict__ coef_child, double2* __restrict__ coef_parent,
    const double2* __restrict__ Vg, const double2* __restrict__ Wg, const TransformTable T) {
  constexpr int H1 = M / 2 + 1, M1 = M + 1;
  constexpr int Ke = mu_off_c<M>(M + 1);
  constexpr int K = hz_count(M);
  extern __shared__ __align__(16) unsigned char smem[];
  double2* W = reinterpret_cast<double2*>(smem);                         // [4][H1][H1]
  double* tval = reinterpret_cast<double*>(W + 4 * H1 * H1);             // [nnz]
  int* tidx = reinterpret_cast<int*>(tval + T.nnz);                       // [nnz]
  int* toff = tidx + T.nnz;                                               // [K + 1]
  double2* Nall = reinterpret_cast<double2*>(
      smem + ((((size_t)4 * H1 * H1 * 16 + (size_t)T.nnz * 12 + (size_t)(K + 1) * 4) + 15) & ~(size_t)15));
  for (int o = threadIdx.x; o < 4 * H1 * H1; o += blockDim.x) W[o] = Wg[o];
  for (int o = threadIdx.x; o < T.nnz; o += blockDim.x) {
    tval[o] = T.val[o];
    tidx[o] = T.idx[o];
  }
  for (int o = threadIdx.x; o <= K; o += blockDim.x) toff[o] = T.off[o];
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int slot = lane >> 2, c = lane & 3;
  double2* N = Nall + (size_t)warp * kM2sSlots * 4 * Ke;   // [slot][child][Ke]
  const double2* Wc = W + c * H1 * H1;
  const double2 dc = Vg[c * M1 * M1 + 1 * M1 + 0];  // V_c[1][0] = C(1,0) d_c = d_c
  for (long long base = ((long long)blockIdx.x * kM2sWarps + warp) * kM2sSlots; base < np;
       base += (long long)gridDim.x * kM2sWarps * kM2sSlots) {
    const long long it = base + slot;
    const bool valid = it < np;
    const uint32_t q = valid ? (plist ? (uint32_t)plist[it] : (uint32_t)(p0 + it)) : 0u;
    const bool mine = valid && block_count(P, level + 1, 4 * q + c) > 0;
    const unsigned ballot = __ballot_sync(0xffffffffu, mine);
    const bool parent = ((ballot >> (slot * 4)) & 0xfu) != 0;
    __syncwarp();
    // stage the eight parents' children (each parent's four are contiguous)
    const double2* Nc = kM2sStage ? N + (size_t)(slot * 4 + c) * Ke : mu_in + (size_t)(4 * q + c) * Ke;
    for (int e = lane; kM2sStage && e < kM2sSlots * 4 * Ke; e += 32) {
      const int sl = e / (4 * Ke), r = e - sl * 4 * Ke;
      const long long ie = base + sl;
      double2 v = make_double2(0.0, 0.0);
      if (((ballot >> (sl * 4 + r / Ke)) & 1u) != 0) {
        const uint32_t qe = plist ? (uint32_t)plist[ie] : (uint32_t)(p0 + ie);
        v = mu_in[(size_t)(4 * qe) * Ke + r];
      }
      N[e] = v;
    }
    __syncwarp();
    if (coef_child && mine) {  // transform of this lane's child (level + 1)
      double2* cd = coef_child + (size_t)(4 * q + c) * K;
      for (int o = 0; o < K; ++o) {
        double cr = 0.0, ci = 0.0;
        for (int t = toff[o]; t < toff[o + 1]; ++t) {
          const double2 x = Nc[tidx[t]];
          cr = fma(tval[t], x.x, cr);
          ci = fma(tval[t], x.y, ci);
        }
        cd[o] = make_double2(cr, ci);
      }
    }
    double2* dst = mu_out + (size_t)q * Ke;
    m2m_columns<M, 0>(Nc, Wc, dc.x, dc.y, dst, c, parent);
    if (coef_parent && parent) {  // level 1: the parents' own coefficients
      __syncwarp();
      for (int o = c; o < K; o += 4) {
        double cr = 0.0, ci = 0.0;
        for (int t = toff[o]; t < toff[o + 1]; ++t) {
          const double2 x = dst[tidx[t]];
          cr = fma(tval[t], x.x, cr);
          ci = fma(tval[t], x.y, ci);
        }
        coef_parent[(size_t)q * K + o] = make_double2(cr, ci);
      }
    }
  }
}

// ------------------------------------------------------------------- M2P ---
constexpr int kMaxList = 384;  // 12 + 27 (L - 2) + 36 <= 372 for L <= 13
constexpr int kFarMaxR = 8;    // a far work item holds <= 32 * kFarMaxR targets

// Builds the warp's source list for a work item: every non-empty source block
// at levels 1..L-1 of the (shared) ancestor lists, then the level-L union over
// the children of the parent's 3x3 neighbourhood that some present leaf needs.
// Entries are (level << 28 | block) in the reference's list order.
// ring (levels 2..L-1): 0 = the whole list; 1 = without the "ring" of the
// level-(l-1) ancestor A (the children of A's 3x3 neighbourhood at Chebyshev
// distance >= 2 from all four children of A -- the outer ring of the 6x6
// candidate square, common to the level-l lists of all of A's descendants);
// 2 = the ring only (Chebyshev-node items of A, cheb.cu).
// lsplit (level L): 0 = the union over the item's present children; 1 = only
// its part in the outer ring of the level-(L-1) block X (needed by all of X's
// children: the fine pass); 2 = only the inner part (per-leaf items of the
// partial pass, each the leaf's own 7 of X's 12 inner-ring leaves); 4 = the
// outer ring of X for items whose targets are Chebyshev nodes of X.
__device__ int build_far_list(const TreeParams& P, uint32_t par, int s, int cnt, uint32_t* list,
                              int lane, int lmin, int lmax, int ring = 0, int lsplit = 0) {
  const int L = P.L;
  const int e = s + cnt;
  bool present = false;
  if (lane < 4) {
    const uint32_t c = 4 * par + lane;
    present = P.leaf_start[c] < e && P.leaf_start[c + 1] > s;
  }
  const uint32_t pmask = __ballot_sync(0xffffffffu, present) & 0xfu;
  int n = 0;
  for (int l = lmin; l <= lmax; ++l) {
    const int grid = 1 << (l + 1);
    int ai = 0, aj = 0, wi, wj, lo_i, lo_j;
    if (l < L) demorton(par >> (2 * (L - 1 - l)), ai, aj);
    if (l == 1) {
      lo_i = lo_j = 0;
      wi = wj = 4;
    } else {
      int pi, pj;
      if (l < L) {
        pi = ai >> 1;
        pj = aj >> 1;
      } else {
        demorton(par, pi, pj);
      }
      lo_i = max(0, 2 * pi - 2);
      lo_j = max(0, 2 * pj - 2);
      wi = min(grid - 1, 2 * pi + 3) - lo_i + 1;
      wj = min(grid - 1, 2 * pj + 3) - lo_j + 1;
    }
    const int ncand = wi * wj;
    for (int base = 0; base < ncand; base += 32) {
      const int c = base + lane;
      bool keep = false;
      uint32_t q = 0;
      if (c < ncand) {
        const int qi = lo_i + c / wj, qj = lo_j + c % wj;
        if (l < L) {
          keep = max(abs(qi - ai), abs(qj - aj)) >= 2;
          if (ring && l >= 2) {
            const int ri = qi - 2 * (ai >> 1), rj = qj - 2 * (aj >> 1);
            const bool in_ring = ri == -2 || ri == 3 || rj == -2 || rj == 3;
            keep = ring == 2 ? in_ring : (keep && !in_ring);
          }
        } else {
          int pi, pj;
          demorton(par, pi, pj);
          for (int ch = 0; ch < 4; ++ch) {
            if (!((pmask >> ch) & 1)) continue;
            const int ci = 2 * pi + (ch >> 1), cj = 2 * pj + (ch & 1);
            if (max(abs(qi - ci), abs(qj - cj)) >= 2) keep = true;
          }
          if (lsplit) {
            const int ri = qi - 2 * pi, rj = qj - 2 * pj;
            const bool outer = ri == -2 || ri == 3 || rj == -2 || rj == 3;
            // 4: the outer ring whatever the item's targets (Chebyshev nodes of X)
            keep = lsplit == 4 ? outer : (keep && (lsplit == 1 ? outer : !outer));
          }
        }
        q = morton(qi, qj);
        if (keep) keep = block_count(P, l, q) > 0;
      }
      const uint32_t bal = __ballot_sync(0xffffffffu, keep);
      if (keep) list[n + __popc(bal & ((1u << lane) - 1u))] = ((uint32_t)l << 28) | q;
      n += __popc(bal);
    }
  }
  __syncwarp();
  return n;
}

// The partial pass's per-leaf list, one leaf per half-warp (all 32 lanes
// call; lane l evaluates candidate l & 15 of its half's leaf): the level-L
// leaves of the 4x4 inner square of the leaf's level-(L-1) block at Chebyshev
// distance >= 2 from the leaf, non-empty, in the reference's row-major list
// order -- exactly build_far_list(lsplit = 2) for a one-leaf item.
__device__ int leaf_inner_list(const TreeParams& P, uint32_t leaf, bool active, int lane,
                               uint32_t* list) {
  const int L = P.L, g = 1 << (L + 1), c = lane & 15;
  int ci, cj;
  demorton(leaf, ci, cj);
  const int qi = (ci & ~1) - 1 + (c >> 2), qj = (cj & ~1) - 1 + (c & 3);
  bool keep = active && qi >= 0 && qj >= 0 && qi < g && qj < g &&
              max(abs(qi - ci), abs(qj - cj)) >= 2;
  uint32_t q = 0;
  if (keep) {
    q = morton((uint32_t)qi, (uint32_t)qj);
    keep = block_count(P, L, q) > 0;
  }
  const uint32_t bal = (__ballot_sync(0xffffffffu, keep) >> (lane & 16)) & 0xffffu;
  if (keep) list[__popc(bal & ((1u << c) - 1u))] = ((uint32_t)L << 28) | q;
  __syncwarp();
  return __popc(bal);
}

// -------------------------------------------------------- list cover check --
// imq_verify / tests: for each listed target, replays every far pass of the
// product (modes from the operator: single pass, coarse + fine + per-leaf
// partial, or Chebyshev node / ring / X-ring items) through build_far_list
// exactly as the kernels call it, with the target as a one-point item, and
// compares the (level, block) entries collected over all passes with the
// reference's interaction lists (partition.cpp:56-72; non-empty source
// blocks, fastmv.cpp:207): out = {missing, duplicated, extra, entries}.
constexpr int kCoverWarps = 4, kCoverCap = 1024;
__global__ void __launch_bounds__(kCoverWarps * 32) k_far_cover(const TreeParams P,
                                                               const int* __restrict__ targets,
                                                               int n_t, const CoverModes Mo,
                                                               const CoverGemm Gm,
                                                               int4* __restrict__ out) {
  __shared__ uint32_t lists[kCoverWarps][kMaxList];
  __shared__ uint32_t got[kCoverWarps][kCoverCap];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int it = blockIdx.x * kCoverWarps + warp;
  if (it >= n_t) return;
  const int t = targets[it], L = P.L;
  const uint32_t T = P.leaf[t], X = T >> 2;
  int ng = 0, overflow = 0;
  auto add = [&](uint32_t par, int lmin, int lmax, int ring, int lsplit) {
    const int n = build_far_list(P, par, t, 1, lists[warp], lane, lmin, lmax, ring, lsplit);
    for (int e = lane; e < n; e += 32)
      if (ng + e < kCoverCap) got[warp][ng + e] = lists[warp][e];
    if (ng + n > kCoverCap) overflow = 1;
    ng = min(kCoverCap, ng + n);
    __syncwarp();
  };
  // a pass run as a tensor-core GEMM: its offset table for the box's class
  auto add_gemm = [&](uint32_t box, int box_level, const GemmDelta* D, int nd, int nc) {
    int bi, bj;
    demorton(box, bi, bj);
    const GemmDelta* Dc = D + (size_t)(nc == 4 ? (int)(box & 3u) : 0) * nd;
    for (int d = lane; d < nd; d += 32) {
      const GemmDelta e = Dc[d];
      const int sh = e.level - box_level, g = 1 << (e.level + 1);
      const long long si = ((long long)bi << sh) + e.dx, sj = ((long long)bj << sh) + e.dy;
      bool keep = si >= 0 && sj >= 0 && si < g && sj < g;
      uint32_t q = 0;
      if (keep) {
        q = morton((uint32_t)si, (uint32_t)sj);
        keep = block_count(P, e.level, q) > 0;
      }
      const uint32_t bal = __ballot_sync(__activemask(), keep);
      if (keep) {
        const int pos = ng + __popc(bal & ((1u << lane) - 1u));
        if (pos < kCoverCap) got[warp][pos] = ((uint32_t)e.level << 28) | q;
      }
      ng = min(kCoverCap, ng + __popc(bal));
    }
    ng = __shfl_sync(0xffffffffu, ng, 0);
    __syncwarp();
  };
  // the per-leaf partial pass: its own list builder when it runs two leaves
  // per warp (both halves enumerate this target's leaf; same entries)
  auto add_part = [&]() {
    if (!Mo.leaf2) return add(X, L, L, 0, 2);
    const int n = leaf_inner_list(P, T, true, lane, lists[warp]);
    for (int e = lane; e < n; e += 32)
      if (ng + e < kCoverCap) got[warp][ng + e] = lists[warp][e];
    if (ng + n > kCoverCap) overflow = 1;
    ng = min(kCoverCap, ng + n);
    __syncwarp();
  };
  if (!Mo.split) {
    add(X, 1, L, 0, 0);
  } else if (!Mo.cheb) {
    add((X >> 2) << 2, 1, L - 2, 0, 0);
    add(X, L - 1, L, 0, Mo.lsplit ? 1 : 0);
    if (Mo.lsplit) add_part();
  } else {
    for (int l = 1; l <= Mo.lc; ++l) {
      const uint32_t q = T >> (2 * (L - l));
      if (Gm.node[l])
        add_gemm(q, l, Gm.node[l], Gm.node_nd[l], 4);
      else
        add(q << (2 * (L - 1 - l)), l, l, (Mo.ring && l >= Mo.ring_l0) ? 1 : 0, 0);
      if (Mo.ring && l + 1 >= Mo.ring_l0) {
        if (Gm.ring[l])
          add_gemm(q, l, Gm.ring[l], Gm.ring_nd[l], 1);
        else
          add((4 * q) << (2 * (L - 2 - l)), l + 1, l + 1, 2, 0);
      }
    }
    if (Mo.xring) {
      if (Gm.x)
        add_gemm(X, L - 1, Gm.x, Gm.x_nd, 4);
      else
        add(X, L - 1, L, 1, 4);
      add_part();
    } else {
      if (Mo.lsplit) add_part();
      add(X, L - 1, L, Mo.ring ? 1 : 0, Mo.lsplit ? 1 : 0);
    }
  }
  int missing = 0, dup = 0, matched = 0;
  for (int l = 1; l <= L; ++l) {
    int bi, bj;
    demorton(T >> (2 * (L - l)), bi, bj);
    const int grid = 1 << (l + 1);
    int lo_i = 0, lo_j = 0, wi = grid, wj = grid;
    if (l >= 2) {
      lo_i = max(0, 2 * (bi >> 1) - 2);
      lo_j = max(0, 2 * (bj >> 1) - 2);
      wi = min(grid - 1, 2 * (bi >> 1) + 3) - lo_i + 1;
      wj = min(grid - 1, 2 * (bj >> 1) + 3) - lo_j + 1;
    }
    for (int c = lane; c < wi * wj; c += 32) {
      const int qi = lo_i + c / wj, qj = lo_j + c % wj;
      if (max(abs(qi - bi), abs(qj - bj)) < 2) continue;
      const uint32_t q = morton(qi, qj);
      if (block_count(P, l, q) == 0) continue;
      const uint32_t key = ((uint32_t)l << 28) | q;
      int cnt = 0;
      for (int e = 0; e < ng; ++e) cnt += got[warp][e] == key;
      missing += cnt == 0;
      dup += cnt > 1;
      matched += cnt;
    }
  }
  for (int d = 16; d; d >>= 1) {
    missing += __shfl_xor_sync(0xffffffffu, missing, d);
    dup += __shfl_xor_sync(0xffffffffu, dup, d);
    matched += __shfl_xor_sync(0xffffffffu, matched, d);
  }
  if (lane == 0) out[it] = make_int4(missing, dup + overflow, ng - matched, ng);
}

// Complex Horner evaluation of one source block's expansion at R targets of
// the lane.  c: K coefficients (double2) in Horner order.  Every coefficient
// read from shared memory feeds 2R DFMAs; shared-memory -> register delivery
// (128 B/clk/SM) is the co-bottleneck with the FP64 pipe, so R >= 3 keeps the
// kernel on the DFMA roofline (profiles/).
template <int M, int R>
__device__ __forceinline__ void far_evalR(const double2* __restrict__ c, const double* dx,
                                          const double* dy, double t2, double* v) {
  double r[R], q[R];
#pragma unroll
  for (int p = 0; p < R; ++p) {
    r[p] = rsqrt_pos(fma(dx[p], dx[p], fma(dy[p], dy[p], t2)));
    q[p] = r[p] * r[p];
  }
  if constexpr (M == 0) {
#pragma unroll
    for (int p = 0; p < R; ++p) v[p] = c[0].x * r[p];
  } else {
    double xr[R], xi[R], ar[R], ai[R];
    double2 cc = c[0];  // group m = M: the single coefficient C_{M,M}
#pragma unroll
    for (int p = 0; p < R; ++p) {
      xr[p] = dx[p] * q[p];
      xi[p] = -dy[p] * q[p];
      ar[p] = cc.x;
      ai[p] = cc.y;
    }
    int o = 1;
#pragma unroll
    for (int m = M - 1; m >= 1; --m) {
      cc = c[o++];  // C_{m, top(m)}
      double gr[R], gi[R];
#pragma unroll
      for (int p = 0; p < R; ++p) {
        gr[p] = cc.x;
        gi[p] = cc.y;
      }
#pragma unroll
      for (int k = hz_top(M, m) - 1; k >= m; --k) {
        cc = c[o++];
#pragma unroll
        for (int p = 0; p < R; ++p) {
          gr[p] = fma(gr[p], q[p], cc.x);
          gi[p] = fma(gi[p], q[p], cc.y);
        }
      }
#pragma unroll
      for (int p = 0; p < R; ++p) {
        const double nr = fma(ar[p], xr[p], fma(-ai[p], xi[p], gr[p]));
        const double ni = fma(ar[p], xi[p], fma(ai[p], xr[p], gi[p]));
        ar[p] = nr;
        ai[p] = ni;
      }
    }
    // m = 0: real inner polynomial (its imaginary parts are exactly zero)
    const double* c0 = reinterpret_cast<const double*>(c + o);
    double g[R];
#pragma unroll
    for (int p = 0; p < R; ++p) g[p] = c0[0];
#pragma unroll
    for (int k = 1; k <= hz_top(M, 0); ++k) {
      const double ck = c0[2 * k];
#pragma unroll
      for (int p = 0; p < R; ++p) g[p] = fma(g[p], q[p], ck);
    }
#pragma unroll
    for (int p = 0; p < R; ++p) v[p] = fma(ar[p], xr[p], fma(-ai[p], xi[p], g[p])) * r[p];
  }
}

// Same evaluation with the Horner loops unrolled by template recursion: the
// compiler otherwise keeps the long inner loops of the low-m groups rolled
// (4 coefficients per trip, each trip stalling on its own shared loads), and
// every coefficient becomes an LDS with an immediate offset.
template <int R, int N>
__device__ __forceinline__ void horner_inner(const double2* __restrict__ c, double* gr, double* gi,
                                             const double* q) {
  if constexpr (N > 0) {
    const double2 cc = c[0];
#pragma unroll
    for (int p = 0; p < R; ++p) {
      gr[p] = fma(gr[p], q[p], cc.x);
      gi[p] = fma(gi[p], q[p], cc.y);
    }
    horner_inner<R, N - 1>(c + 1, gr, gi, q);
  }
}

template <int R, int N>
__device__ __forceinline__ void horner_real(const double2* __restrict__ c, double* g,
                                            const double* q) {
  if constexpr (N > 0) {
    const double ck = c[0].x;
#pragma unroll
    for (int p = 0; p < R; ++p) g[p] = fma(g[p], q[p], ck);
    horner_real<R, N - 1>(c + 1, g, q);
  }
}

// Groups m, m-1, ..., 1 (c points at C_{m, top(m)}); returns the offset past them.
template <int M, int R, int m>
__device__ __forceinline__ const double2* horner_groups(const double2* __restrict__ c, double* ar,
                                                        double* ai, const double* q,
                                                        const double* xr, const double* xi) {
  if constexpr (m < 1) {
    return c;
  } else {
    constexpr int n = hz_top(M, m) - m;  // coefficients after the leading one
    double gr[R], gi[R];
    const double2 cc = c[0];
#pragma unroll
    for (int p = 0; p < R; ++p) {
      gr[p] = cc.x;
      gi[p] = cc.y;
    }
    horner_inner<R, n>(c + 1, gr, gi, q);
#pragma unroll
    for (int p = 0; p < R; ++p) {
      const double nr = fma(ar[p], xr[p], fma(-ai[p], xi[p], gr[p]));
      const double ni = fma(ar[p], xi[p], fma(ai[p], xr[p], gi[p]));
      ar[p] = nr;
      ai[p] = ni;
    }
    return horner_groups<M, R, m - 1>(c + 1 + n, ar, ai, q, xr, xi);
  }
}

template <int M, int R>
__device__ __forceinline__ void far_evalT(const double2* __restrict__ c, const double* dx,
                                          const double* dy, double t2, double* v) {
  double r[R], q[R];
#pragma unroll
  for (int p = 0; p < R; ++p) {
    r[p] = rsqrt_pos(fma(dx[p], dx[p], fma(dy[p], dy[p], t2)));
    q[p] = r[p] * r[p];
  }
  if constexpr (M == 0) {
#pragma unroll
    for (int p = 0; p < R; ++p) v[p] = c[0].x * r[p];
  } else {
    double xr[R], xi[R], ar[R], ai[R];
    const double2 cc = c[0];
#pragma unroll
    for (int p = 0; p < R; ++p) {
      xr[p] = dx[p] * q[p];
      xi[p] = -dy[p] * q[p];
      ar[p] = cc.x;
      ai[p] = cc.y;
    }
    const double2* c0 = horner_groups<M, R, M - 1>(c + 1, ar, ai, q, xr, xi);
    double g[R];
#pragma unroll
    for (int p = 0; p < R; ++p) g[p] = c0[0].x;
    horner_real<R, hz_top(M, 0)>(c0 + 1, g, q);
#pragma unroll
    for (int p = 0; p < R; ++p) v[p] = fma(ar[p], xr[p], fma(-ai[p], xi[p], g[p])) * r[p];
  }
}

// Runtime-order variant (coefficients read through L1 from global memory).
__device__ __forceinline__ double far_eval_generic(const double2* __restrict__ c, int M,
                                                   double dx, double dy, double t2) {
  const double r = rsqrt_pos(fma(dx, dx, fma(dy, dy, t2)));
  const double q = r * r;
  if (M == 0) return __ldg(&c[0].x) * r;
  const double xr = dx * q, xi = -dy * q;
  double2 cc = __ldg(&c[0]);
  double ar = cc.x, ai = cc.y;
  int o = 1;
  for (int m = M - 1; m >= 1; --m) {
    cc = __ldg(&c[o++]);
    double gr = cc.x, gi = cc.y;
    for (int k = hz_top(M, m) - 1; k >= m; --k) {
      cc = __ldg(&c[o++]);
      gr = fma(gr, q, cc.x);
      gi = fma(gi, q, cc.y);
    }
    const double nr = fma(ar, xr, fma(-ai, xi, gr));
    const double ni = fma(ar, xi, fma(ai, xr, gi));
    ar = nr;
    ai = ni;
  }
  double g = __ldg(&c[o++].x);
  for (int k = hz_top(M, 0) - 1; k >= 0; --k) g = fma(g, q, __ldg(&c[o++].x));
  return fma(ar, xr, fma(-ai, xi, g)) * r;
}

// Targets of a lane: coordinates in registers; the leaf of each target is one
// of the four children of the item's level-(L-1) block, packed 2 bits each,
// with a validity bit (slots past the item's count).
template <int R>
struct Targets {
  double x[R], y[R];
  uint32_t child;  // 2 bits per slot
  uint32_t valid;  // 1 bit per slot
};

template <int R>
__device__ __forceinline__ void load_targets(const TreeParams& P, int s, int cnt, int lane,
                                             Targets<R>& T) {
  T.child = 0;
  T.valid = 0;
#pragma unroll
  for (int p = 0; p < R; ++p) {
    const bool v = lane + 32 * p < cnt;
    const int a = v ? s + lane + 32 * p : s;
    T.x[p] = P.xs[a];
    T.y[p] = P.ys[a];
    T.child |= (P.leaf[a] & 3u) << (2 * p);
    T.valid |= (v ? 1u : 0u) << p;
  }
}

// Warp per work item (<= 32 R targets of one level-(L-1) block, R per lane).
// Source coefficients are staged per warp through a STAGES-deep ring of
// shared-memory buffers filled by one-instruction TMA bulk copies
// (cp.async.bulk + mbarrier complete_tx), lane 0 producing, the warp consuming.
// Epilogue: far_s[q] = far field (near_part == nullptr), or, when the
// symmetric near field already ran, out[perm[q]] = far + sum of its 5 slots.
// Level range: items evaluate the source blocks of levels lmin..lmax; a
// fine pass (levels L-1..L) adds the coarse pass's far_add[q] first.
struct FarOut {
  double* far_s;
  const double* near_part;  // [nslots][N] or nullptr
  int nslots;
  double* out;
  const int* perm;
  const double* far_add;  // or nullptr
  int lmin, lmax;
  int ring;    // build_far_list ring mode of items without a level tag
  int lsplit;  // build_far_list level-L split of items without a level tag
};

__device__ __forceinline__ void far_store(const TreeParams& P, const FarOut& O, int q,
                                          double acc) {
  if (O.far_add) acc = O.far_add[q] + acc;
  if (!O.near_part) {
    O.far_s[q] = acc;
    return;
  }
  double nsum = 0.0;
  for (int k = 0; k < O.nslots; ++k) nsum += O.near_part[(size_t)k * P.N + q];
  O.out[O.perm ? O.perm[q] : q] = acc + nsum;
}

template <int M, int R, int WARPS, int STAGES, int MINB>
__global__ void __launch_bounds__(WARPS * 32, MINB) k_m2p_far(const TreeParams P,
                                                             const int4* __restrict__ items,
                                                             int n_items,
                                                             const double2* __restrict__ coef,
                                                             const FarOut O) {
  constexpr int K = hz_count(M);
  constexpr uint32_t kBytes = K * 16;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double2* stage = reinterpret_cast<double2*>(smem_raw) + (size_t)warp * STAGES * K;
  uint64_t* bars =
      reinterpret_cast<uint64_t*>(reinterpret_cast<double2*>(smem_raw) + WARPS * STAGES * K) +
      warp * STAGES;
  uint32_t* list = reinterpret_cast<uint32_t*>(
                       reinterpret_cast<uint64_t*>(reinterpret_cast<double2*>(smem_raw) +
                                                   WARPS * STAGES * K) +
                       WARPS * STAGES) +
                   warp * kMaxList;
  const int it = blockIdx.x * WARPS + warp;
  if (it >= n_items) return;
  if (lane == 0) {
#pragma unroll
    for (int s = 0; s < STAGES; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  __syncwarp();

  const int4 item = items[it];
  const uint32_t par = (uint32_t)item.x;
  const int s0 = item.y, cnt = item.z;
  // item.w > 0: item of level (w & 0xff) only (Chebyshev node / ring items,
  // partial-pass leaves), ring mode (w >> 8) & 15, level-L split w >> 12
  const int lev = item.w & 0xff;
  const int ring = lev > 0 ? (item.w >> 8) & 15 : O.ring;
  const int lsplit = lev > 0 ? (item.w >> 12) & 15 : O.lsplit;
  const int n = build_far_list(P, par, s0, cnt, list, lane, lev > 0 ? lev : O.lmin,
                               lev > 0 ? lev : O.lmax, ring, lsplit);
  Targets<R> T;
  load_targets<R>(P, s0, cnt, lane, T);
  const int L = P.L;
  int pi2, pj2;  // finest-level index of the item's first child
  demorton(par, pi2, pj2);
  pi2 *= 2;
  pj2 *= 2;

  auto issue = [&](int e, int slot) {
    const uint32_t ent = list[e];
    const int l = (int)(ent >> 28);
    const uint32_t q = ent & 0x0fffffffu;
    mbar_arrive_expect_tx(&bars[slot], kBytes);
    tma_load_1d(stage + (size_t)slot * K, coef + P.coef_off[l] + (size_t)q * K, kBytes,
                &bars[slot]);
  };
  if (lane == 0)
    for (int e = 0; e < STAGES && e < n; ++e) issue(e, e);

  double acc[R];
#pragma unroll
  for (int p = 0; p < R; ++p) acc[p] = 0.0;
  for (int e = 0; e < n; ++e) {
    const int slot = e % STAGES;
    const uint32_t ent = list[e];
    const int l = (int)(ent >> 28);
    int qi, qj;
    demorton(ent & 0x0fffffffu, qi, qj);
    const double zx = block_center(P.ox, qi, P.cell[l]);
    const double zy = block_center(P.oy, qj, P.cell[l]);
    // level-L sources: usable by the children of `par` at Chebyshev
    // distance >= 2 (4-bit mask over the children), others by every target
    uint32_t cmask = 0xfu;
    if (l == L) {
      cmask = 0;
#pragma unroll
      for (int ch = 0; ch < 4; ++ch)
        cmask |= (max(abs(qi - (pi2 + (ch >> 1))), abs(qj - (pj2 + (ch & 1)))) >= 2 ? 1u : 0u) << ch;
    }
    bool msk[R];
    double dx[R], dy[R], v[R];
#pragma unroll
    for (int p = 0; p < R; ++p) {
      msk[p] = ((T.valid >> p) & 1u) && ((cmask >> ((T.child >> (2 * p)) & 3u)) & 1u);
      dx[p] = T.x[p] - zx;
      dy[p] = T.y[p] - zy;
    }
    mbar_wait(&bars[slot], (uint32_t)((e / STAGES) & 1));
    far_evalT<M, R>(stage + (size_t)slot * K, dx, dy, P.t2, v);
#pragma unroll
    for (int p = 0; p < R; ++p) acc[p] += msk[p] ? v[p] : 0.0;
    __syncwarp();
    if (lane == 0 && e + STAGES < n) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(e + STAGES, slot);
    }
  }
#pragma unroll
  for (int p = 0; p < R; ++p)
    if ((T.valid >> p) & 1u) far_store(P, O, s0 + lane + 32 * p, acc[p]);
}

// Per-leaf partial pass, two leaves per warp: half-warp h (16 lanes) takes
// item 2w + h -- <= 16 R targets of ONE leaf, R per lane -- against that
// leaf's own inner-ring leaves (leaf_inner_list: the 7 of the level-(L-1)
// block's 12 inner-ring leaves at Chebyshev distance >= 2, the reference's
// level-L list minus the outer ring that the X-node pass covers).  A 64-point
// leaf runs R = 4 (8 DFMA per shared load, against 4 with 32 lanes x R = 2),
// and a 65..80-point leaf fills 80 target slots instead of 96.  Each half has
// its own TMA staging ring and producer lane (hl == 0); the two halves' lists
// may differ in length (domain edge, empty leaves): a half past its list
// waits on nothing and its (stale) evaluations are discarded.  Per target the
// sources are summed in list order with the same evaluation as k_m2p_far, so
// the result is bitwise that of the one-leaf-per-warp pass.
template <int M, int R, int WARPS, int STAGES, int MINB>
__global__ void __launch_bounds__(WARPS * 32, MINB) k_m2p_leaf2(const TreeParams P,
                                                               const int4* __restrict__ items,
                                                               int n_items,
                                                               const double2* __restrict__ coef,
                                                               const FarOut O) {
  constexpr int K = hz_count(M);
  constexpr uint32_t kBytes = K * 16;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, hl = lane & 15;
  const int hw = warp * 2 + (lane >> 4);  // half-warp index in the CTA
  double2* stage = reinterpret_cast<double2*>(smem_raw) + (size_t)hw * STAGES * K;
  uint64_t* bars =
      reinterpret_cast<uint64_t*>(reinterpret_cast<double2*>(smem_raw) + 2 * WARPS * STAGES * K) +
      hw * STAGES;
  uint32_t* list = reinterpret_cast<uint32_t*>(
                       reinterpret_cast<uint64_t*>(reinterpret_cast<double2*>(smem_raw) +
                                                   2 * WARPS * STAGES * K) +
                       2 * WARPS * STAGES) +
                   hw * 16;
  const int it0 = (blockIdx.x * WARPS + warp) * 2;
  if (it0 >= n_items) return;
  const int it = it0 + (lane >> 4);
  if (hl == 0) {
#pragma unroll
    for (int s = 0; s < STAGES; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  __syncwarp();
  const int4 item = it < n_items ? items[it] : make_int4(0, 0, 0, 0);
  const uint32_t leaf = (uint32_t)item.x;
  const int s0 = item.y, cnt = item.z;
  const int n = leaf_inner_list(P, leaf, cnt > 0, lane, list);
  const int nmax = max(n, __shfl_xor_sync(0xffffffffu, n, 16));
  double tx[R], ty[R];
  uint32_t valid = 0;
#pragma unroll
  for (int p = 0; p < R; ++p) {
    const bool v = hl + 16 * p < cnt;
    const int a = v ? s0 + hl + 16 * p : s0;
    tx[p] = P.xs[a];
    ty[p] = P.ys[a];
    valid |= (v ? 1u : 0u) << p;
  }
  const int L = P.L;
  auto issue = [&](int e, int slot) {
    const uint32_t q = list[e] & 0x0fffffffu;
    mbar_arrive_expect_tx(&bars[slot], kBytes);
    tma_load_1d(stage + (size_t)slot * K, coef + P.coef_off[L] + (size_t)q * K, kBytes,
                &bars[slot]);
  };
  if (hl == 0)
    for (int e = 0; e < STAGES && e < n; ++e) issue(e, e);
  double acc[R];
#pragma unroll
  for (int p = 0; p < R; ++p) acc[p] = 0.0;
  for (int e = 0; e < nmax; ++e) {
    const int slot = e % STAGES;
    const bool live = e < n;
    int qi = 0, qj = 0;
    if (live) demorton(list[e] & 0x0fffffffu, qi, qj);
    const double zx = block_center(P.ox, qi, P.cell[L]);
    const double zy = block_center(P.oy, qj, P.cell[L]);
    double dx[R], dy[R], v[R];
#pragma unroll
    for (int p = 0; p < R; ++p) {
      dx[p] = tx[p] - zx;
      dy[p] = ty[p] - zy;
    }
    if (live) mbar_wait(&bars[slot], (uint32_t)((e / STAGES) & 1));
    far_evalT<M, R>(stage + (size_t)slot * K, dx, dy, P.t2, v);
#pragma unroll
    for (int p = 0; p < R; ++p) acc[p] += (live && ((valid >> p) & 1u)) ? v[p] : 0.0;
    __syncwarp();
    if (hl == 0 && e + STAGES < n) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(e + STAGES, slot);
    }
  }
#pragma unroll
  for (int p = 0; p < R; ++p)
    if ((valid >> p) & 1u) far_store(P, O, s0 + hl + 16 * p, acc[p]);
}

template <int WARPS>
__global__ void __launch_bounds__(WARPS * 32) k_m2p_far_generic(const TreeParams P,
                                                               const int4* __restrict__ items,
                                                               int n_items,
                                                               const double2* __restrict__ coef,
                                                               const FarOut O) {
  __shared__ uint32_t lists[WARPS][kMaxList];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int it = blockIdx.x * WARPS + warp;
  if (it >= n_items) return;
  const int4 item = items[it];
  const uint32_t par = (uint32_t)item.x;
  const int s0 = item.y, cnt = item.z;
  uint32_t* list = lists[warp];
  const int lev = item.w & 0xff;
  const int ring = lev > 0 ? (item.w >> 8) & 15 : O.ring;
  const int lsplit = lev > 0 ? (item.w >> 12) & 15 : O.lsplit;
  const int n = build_far_list(P, par, s0, cnt, list, lane, lev > 0 ? lev : O.lmin,
                               lev > 0 ? lev : O.lmax, ring, lsplit);
  for (int p0 = lane; p0 < cnt; p0 += 32) {
    const int p = s0 + p0;
    const double x = P.xs[p], y = P.ys[p];
    int li, lj;
    demorton(P.leaf[p], li, lj);
    double acc = 0.0;
    for (int e = 0; e < n; ++e) {
      const uint32_t ent = list[e];
      const int l = (int)(ent >> 28);
      const uint32_t q = ent & 0x0fffffffu;
      int qi, qj;
      demorton(q, qi, qj);
      if (l == P.L && max(abs(qi - li), abs(qj - lj)) < 2) continue;
      const double zx = block_center(P.ox, qi, P.cell[l]);
      const double zy = block_center(P.oy, qj, P.cell[l]);
      acc += far_eval_generic(coef + P.coef_off[l] + (size_t)q * P.K, P.M, x - zx, y - zy, P.t2);
    }
    far_store(P, O, p, acc);
  }
}

// Launch configuration of the far kernel for work items of R points per lane
// (warps per CTA W, staging depth S, min CTAs per SM).  Items are grouped by
// R = ceil(count / 32) at build time, so lanes are idle only in the last
// point slot of an item.
template <int M, int R, int W, int S, int MINB>
void run_far_cfg(const TreeParams& P, const int4* items, int n_items, const double2* coef,
                 const FarOut& far_s, cudaStream_t s) {
  constexpr int K = hz_count(M);
  auto kern = k_m2p_far<M, R, W, S, MINB>;
  const size_t smem = (size_t)W * S * K * 16 + W * S * 8 + W * kMaxList * 4;
  if (smem > 48 * 1024) ensure_smem_attr((const void*)kern, smem);
  const unsigned grid = (unsigned)((n_items + W - 1) / W);
  kern<<<grid, W * 32, smem, s>>>(P, items, n_items, coef, far_s);
}

// Two leaves per warp (k_m2p_leaf2): items of <= 16 R targets, paired.
template <int M, int R, int W, int S, int MINB>
void run_leaf2_cfg(const TreeParams& P, const int4* items, int n_items, const double2* coef,
                   const FarOut& far_s, cudaStream_t s) {
  constexpr int K = hz_count(M);
  auto kern = k_m2p_leaf2<M, R, W, S, MINB>;
  const size_t smem = (size_t)2 * W * S * K * 16 + 2 * W * S * 8 + 2 * W * 16 * 4;
  if (smem > 48 * 1024) ensure_smem_attr((const void*)kern, smem);
  const unsigned grid = (unsigned)((n_items + 2 * W - 1) / (2 * W));
  kern<<<grid, W * 32, smem, s>>>(P, items, n_items, coef, far_s);
}

}  // namespace

int far_max_points_per_lane() { return kFarMaxR; }

namespace {

template <int M>
void run_far(const TreeParams& P, int R, const int4* items, int n_items, const double2* coef,
             const FarOut& far_s, cudaStream_t s) {
  switch (R) {
    case 1: return run_far_cfg<M, 1, 4, 3, 1>(P, items, n_items, coef, far_s, s);
    case 2: return run_far_cfg<M, 2, 4, 3, 1>(P, items, n_items, coef, far_s, s);
    case 3: return run_far_cfg<M, 3, 4, 3, 1>(P, items, n_items, coef, far_s, s);
    case 4: return run_far_cfg<M, 4, 4, 3, 1>(P, items, n_items, coef, far_s, s);
    case 5: return run_far_cfg<M, 5, 4, 3, 1>(P, items, n_items, coef, far_s, s);
    case 6: return run_far_cfg<M, 6, 4, 3, 1>(P, items, n_items, coef, far_s, s);
    case 7: return run_far_cfg<M, 7, 4, 3, 1>(P, items, n_items, coef, far_s, s);
    default: return run_far_cfg<M, 8, 4, 3, 1>(P, items, n_items, coef, far_s, s);
  }
}

template <int M>
void run_leaf2(const TreeParams& P, int R, const int4* items, int n_items, const double2* coef,
               const FarOut& far_s, cudaStream_t s) {
  switch (R) {
    case 1: return run_leaf2_cfg<M, 1, 4, 3, 1>(P, items, n_items, coef, far_s, s);
    case 2: return run_leaf2_cfg<M, 2, 4, 3, 1>(P, items, n_items, coef, far_s, s);
    case 3: return run_leaf2_cfg<M, 3, 4, 3, 1>(P, items, n_items, coef, far_s, s);
    case 4: return run_leaf2_cfg<M, 4, 4, 3, 1>(P, items, n_items, coef, far_s, s);
    case 5: return run_leaf2_cfg<M, 5, 4, 3, 1>(P, items, n_items, coef, far_s, s);
    case 6: return run_leaf2_cfg<M, 6, 4, 3, 1>(P, items, n_items, coef, far_s, s);
    case 7: return run_leaf2_cfg<M, 7, 4, 3, 1>(P, items, n_items, coef, far_s, s);
    default: return run_leaf2_cfg<M, 8, 4, 3, 1>(P, items, n_items, coef, far_s, s);
  }
}

template <int M, int WPL>
void run_p2m_w(const TreeParams& P, const double* u_s, double2* mu, const int* list, int n_list,
               cudaStream_t s) {
  const long long n_leaves = list ? n_list : 1ll << (2 * (P.L + 1));
  constexpr int WARPS = WPL > 4 ? WPL : 4;
  constexpr int LPC = WARPS / WPL;
  k_p2m_leaf_g<M, 8, WPL><<<(unsigned)((n_leaves + LPC - 1) / LPC), 32 * WARPS, 0, s>>>(
      P, u_s, mu, list, n_list);
}

template <int M>
void run_p2m(const TreeParams& P, const double* u_s, double2* mu, const int* list, int n_list,
             cudaStream_t s) {
  const long long n_leaves = list ? n_list : 1ll << (2 * (P.L + 1));
  // 8 lanes per point (4 points per pass) for M < 24, else the 32-lane form;
  // warps per leaf from the mean leaf occupancy (P.p2m_wpl)
  if constexpr (M < 24) {
    switch (P.p2m_wpl) {
      case 1: return run_p2m_w<M, 1>(P, u_s, mu, list, n_list, s);
      case 2: return run_p2m_w<M, 2>(P, u_s, mu, list, n_list, s);
      case 4: return run_p2m_w<M, 4>(P, u_s, mu, list, n_list, s);
      default: return run_p2m_w<M, 8>(P, u_s, mu, list, n_list, s);
    }
  } else
    k_p2m_leaf<M><<<(unsigned)((n_leaves + 3) / 4), 128, 0, s>>>(P, u_s, mu, list, n_list);
}

#define IMQ_FOR_SPECIALISED_M(X) X(0) X(1) X(2) X(4) X(6) X(8) X(10) X(12) X(14) X(16) X(18) X(20)

}  // namespace

bool m2p_specialised(int M) {
  switch (M) {
#define X(m) case m:
    IMQ_FOR_SPECIALISED_M(X)
#undef X
    return true;
    default:
      return false;
  }
}

void launch_p2m_leaf(const TreeParams& P, const double* u_s, double2* mu, const int* leaf_list,
                     int n_list, cudaStream_t s) {
  switch (P.M) {
#define X(m)                                      \
  case m:                                         \
    run_p2m<m>(P, u_s, mu, leaf_list, n_list, s); \
    return;
    IMQ_FOR_SPECIALISED_M(X)
#undef X
    default: {
      const long long n =
          (leaf_list ? (long long)n_list : (1ll << (2 * (P.L + 1)))) * (long long)P.Ke;
      k_p2m_leaf_generic<<<(unsigned)((n + 127) / 128), 128, 0, s>>>(P, u_s, mu, leaf_list,
                                                                    n_list);
    }
  }
}

void launch_m2m(const TreeParams& P, int level, double2* mu, const double* binom,
                cudaStream_t s) {
  const size_t smem = (size_t)(4 * P.Ke + 4 * (P.M + 1)) * sizeof(double2) +
                      (size_t)(P.M + 1) * (P.M + 1) * sizeof(double) + (P.M + 1) * sizeof(int);
  if (smem > 48 * 1024) ensure_smem_attr((const void*)k_m2m, smem);
  const int threads = ((P.Ke + 31) / 32) * 32 > 1024 ? 1024 : ((P.Ke + 31) / 32) * 32;
  const unsigned nb = 1u << (2 * (level + 1));
  k_m2m<<<nb, threads, smem, s>>>(P, level, mu, binom);
}

size_t m2m_tr_smem(int M, int Ke, int K, int nnz) { return M2tLayout(M, Ke, K, nnz).total; }
static bool m2m_specialised(int M) {
  switch (M) {
#define X(m) case m:
    IMQ_FOR_SPECIALISED_M(X)
#undef X
    return true;
    default:
      return false;
  }
}

void launch_m2m_tr(const TreeParams& P, int level, const int* plist, long long p0, long long np,
                   const double2* mu_in, double2* mu_out, double2* coef_child,
                   double2* coef_parent, const double2* V, const double2* W,
                   const TransformTable& T, cudaStream_t s) {
  if (np <= 0) return;
  // few parents (coarse levels): the warp-per-parent kernel spreads one
  // parent over 32 lanes (lower latency); the specialised kernel's eight
  // parents per warp pay ~70 us of per-warp latency whatever the level size
  if (m2m_specialised(P.M) && np > kM2tSmallLevel) {
    const int H1 = P.M / 2 + 1;
    const size_t ss = ((((size_t)4 * H1 * H1 * 16 + (size_t)T.nnz * 12 + (size_t)(P.K + 1) * 4) + 15) &
                       ~(size_t)15) + (kM2sStage ? (size_t)kM2sWarps * kM2sSlots * 4 * P.Ke * 16 : 0);
    const long long per = (long long)kM2sWarps * kM2sSlots;
    const unsigned grid = (unsigned)std::min<long long>((np + per - 1) / per, 148ll * 32);
    switch (P.M) {
#define X(m)                                                                                    \
  case m:                                                                                       \
    ensure_smem_attr((const void*)k_m2m_tr_s<m>, ss);                                           \
    k_m2m_tr_s<m><<<grid, kM2sWarps * 32, ss, s>>>(P, level, plist, p0, np, mu_in, mu_out,      \
                                                  coef_child, coef_parent, V, W, T);            \
    return;
      IMQ_FOR_SPECIALISED_M(X)
#undef X
      default:
        break;
    }
  }
  const size_t smem = M2tLayout(P.M, P.Ke, P.K, T.nnz).total;
  const long long want = (np + kM2tWarps - 1) / kM2tWarps;
  const unsigned grid = (unsigned)std::min<long long>(want, 148ll * 16);
  ensure_smem_attr((const void*)k_m2m_tr, smem);
  k_m2m_tr<<<grid, kM2tWarps * 32, smem, s>>>(P, level, plist, p0, np, mu_in, mu_out, coef_child,
                                             coef_parent, V, W, T);
}

void launch_transform(const TreeParams& P, const double2* mu, double2* coef,
                      const TransformTable& T, cudaStream_t s, int l_lo, int l_hi,
                      const int* block_list, int n_list) {
  const int nnz = T.nnz;
  const size_t smem = (size_t)P.Ke * sizeof(double2) + (size_t)nnz * (sizeof(double) + sizeof(int)) +
                      (size_t)(P.K + 1) * sizeof(int);
  if (smem > 48 * 1024) ensure_smem_attr((const void*)k_transform, smem);
  const int threads = ((P.K + 31) / 32) * 32 > 1024 ? 1024 : ((P.K + 31) / 32) * 32;
  if (l_lo < 1) l_lo = 1;
  if (l_hi < 1 || l_hi > P.L) l_hi = P.L;
  for (int l = l_lo; l <= l_hi; ++l) {
    const int nb = block_list ? n_list : 1 << (2 * (l + 1));
    if (nb)
      k_transform<<<(unsigned)((nb + kTrBlocks - 1) / kTrBlocks), threads, smem, s>>>(
          P, l, mu, coef, T, block_list, nb, nnz);
  }
}


void launch_m2p_far(const TreeParams& P, const int4* items, const int* group_off, int begin,
                    int end, const double2* coef, double* far_s_ptr, const cudaStream_t* streams,
                    int nstreams, const double* near_part, int nslots, double* out,
                    const int* perm, const double* far_add, int lmin, int lmax, int ring,
                    int lsplit, bool leaf2) {
  if (end <= begin) return;
  if (lmin < 1) lmin = 1;
  if (lmax < 1 || lmax > P.L) lmax = P.L;
  const FarOut far_s{far_s_ptr, near_part, nslots, out, perm, far_add, lmin, lmax, ring, lsplit};
  cudaStream_t s = streams[0];
  int launched = 0;
  if (!m2p_specialised(P.M)) {
    constexpr int W = 4;
    const int n = end - begin;
    k_m2p_far_generic<W><<<(unsigned)((n + W - 1) / W), W * 32, 0, s>>>(P, items + begin, n,
                                                                        coef, far_s);
    return;
  }
  for (int R = kFarMaxR; R >= 1; --R) {  // longest items first
    const int lo = std::max(begin, group_off[R - 1]), hi = std::min(end, group_off[R]);
    if (hi <= lo) continue;
    switch (P.M) {
#define X(m)                                                   \
  case m:                                                      \
    if (leaf2)                                                 \
      run_leaf2<m>(P, R, items + lo, hi - lo, coef, far_s,      \
                   streams[launched++ % nstreams]);           \
    else                                                       \
      run_far<m>(P, R, items + lo, hi - lo, coef, far_s,        \
                 streams[launched++ % nstreams]);             \
    break;
      IMQ_FOR_SPECIALISED_M(X)
#undef X
      default:
        break;
    }
  }
}

void launch_far_cover(const TreeParams& P, const int* targets, int n_t, const CoverModes& Mo,
                      const CoverGemm& Gm, int4* out, cudaStream_t s) {
  if (n_t > 0)
    k_far_cover<<<(unsigned)((n_t + kCoverWarps - 1) / kCoverWarps), kCoverWarps * 32, 0, s>>>(
        P, targets, n_t, Mo, Gm, out);
}

}  // namespace imqk
