// cheb.cu -- the far field of the coarse levels through Chebyshev
// interpolation on the target boxes.
//
// For a target box X at level l the reference adds, for every point of X, the
// same list of source blocks (partition.cpp:56-72; fastmv.cpp:201-212).  That
// sum F_X(x) = sum_{B in list_l(X)} F_B(x) is a smooth function on X (every
// source block sits >= 1.5 cells away), so it is evaluated with the
// reference's own M2P at n x n Chebyshev nodes of X (k_m2p_far on node
// "targets", operator.cu), turned into a tensor Chebyshev series of degree
// n-1, pushed down the levels (the restriction of a degree-(n-1) series to a
// child box is again exactly such a series), and summed at every target of
// the level-lc boxes.  With n = kChebN = 18 the interpolation error of one
// box's field is <= ~1e-13 of its maximum (tests vs the oracle).
//
// Rings: the part of a level-l list common to all four
// children of a level-(l-1) box A is evaluated once at NR x NR nodes of A and
// restricted into each child's series (k_cheb_ring_coef_mma); where t is
// large against the level-(L-1) boxes X, X's shared lists go through NX x NX
// nodes of X (k_cheb_xring_coef).  The series is evaluated at the targets on
// the FP64 tensor cores (k_cheb_eval_mma).
//
// (tables in global memory: the kernels index them per thread, which the
// constant cache would serialise)
// Layouts: per box (levels 1..lc, all boxes, level-major, Morton inside a
// level) n^2 node values / coefficients, index [box][i * n + j], i the x
// index and j the y index; x_i = c_x + (cell/2) cos(pi (i + 1/2) / n).
#include <algorithm>
#include <cstdlib>
#include <stdexcept>
#include <string>

#include "imq_device.cuh"
#include "imq_kernels.hpp"

namespace imqk {

namespace {

using namespace imqdev;
constexpr int NC = kChebN;
constexpr int NN = NC * NC;

__device__ double c_T[NN];        // T[k * NC + i] = cos(k theta_i), theta_i = pi (i + 1/2) / NC
__device__ double c_S[2][NN];     // child restriction, [half][k' * NC + k]
constexpr int NR = kChebNR;       // ring nodes per dimension (the larger variant)
constexpr int NRR = NR * NR;
static_assert(kChebNR2 <= kChebNR, "variant 1 is the smaller ring");
// per ring variant v (nr = kRingNr[v]): cos(k theta_i) at [k * nr + i], and
// ring values -> child coefficients at [half][k' * nr + i]
__device__ double c_TR[2][NRR];
__device__ double c_B[2][2][NC * NR];
constexpr int NX = kChebNX;
constexpr int NXX = NX * NX;
static_assert(NX <= NC, "the X-ring series is added into the level-(L-1) series");
__device__ double c_TX[NXX];         // cos(k theta_i), theta_i = pi (i + 1/2) / NX
constexpr int NI = kChebNI;          // own inner lists of the levels with t >= 2.5 h
static_assert(NI <= NC, "the inner-list series is added into the level series");
__device__ double c_TI[NI * NI];

__global__ void k_cheb_nodes(const TreeParams P, int l, long long box_base, double* __restrict__ nx,
                             double* __restrict__ ny) {
  const long long nb = 1ll << (2 * (l + 1));
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nb * NN) return;
  const uint32_t q = (uint32_t)(t / NN);
  const int r = (int)(t % NN), i = r / NC, j = r % NC;
  int bi, bj;
  demorton(q, bi, bj);
  const double h = 0.5 * P.cell[l];
  nx[(box_base + q) * NN + r] = block_center(P.ox, bi, P.cell[l]) + h * c_T[NC + i];
  ny[(box_base + q) * NN + r] = block_center(P.oy, bj, P.cell[l]) + h * c_T[NC + j];
}

// Ring nodes: nr x nr Chebyshev nodes of every box of level l, [box][i * nr + j].
__global__ void k_cheb_nodes_ring(const TreeParams P, int l, int v, long long node_base,
                                  double* __restrict__ nx, double* __restrict__ ny) {
  const int nr = v ? kChebNR2 : kChebNR, nrr = nr * nr;
  const long long nb = 1ll << (2 * (l + 1));
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nb * nrr) return;
  const uint32_t q = (uint32_t)(t / nrr);
  const int r = (int)(t % nrr), i = r / nr, j = r % nr;
  int bi, bj;
  demorton(q, bi, bj);
  const double h = 0.5 * P.cell[l];
  nx[node_base + t] = block_center(P.ox, bi, P.cell[l]) + h * c_TR[v][nr + i];
  ny[node_base + t] = block_center(P.oy, bj, P.cell[l]) + h * c_TR[v][nr + j];
}

// N x N Chebyshev nodes of every box of level l, [box][i * N + j], written
// from node index node_base (W = 0: X-ring nodes, NX; W = 1: inner-list
// nodes, NI).
template <int W>
__global__ void k_cheb_nodes_n(const TreeParams P, int l, long long node_base,
                               double* __restrict__ nx, double* __restrict__ ny) {
  constexpr int N = W ? NI : NX, NNn = N * N;
  const double* T = W ? c_TI : c_TX;
  const long long nb = 1ll << (2 * (l + 1));
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nb * NNn) return;
  const uint32_t q = (uint32_t)(t / NNn);
  const int r = (int)(t % NNn), i = r / N, j = r % N;
  int bi, bj;
  demorton(q, bi, bj);
  const double h = 0.5 * P.cell[l];
  nx[node_base + t] = block_center(P.ox, bi, P.cell[l]) + h * T[N + i];
  ny[node_base + t] = block_center(P.oy, bj, P.cell[l]) + h * T[N + j];
}

// Warp-per-box DCT of N x N node values, added into the box's degree-(NC-1)
// series: coef[X][k][m] += (2/N)^2 w_k w_m sum_{i,j} T_k(x_i) T_m(y_j) V[i][j]
// (W = 0: the X-ring, N = NX; W = 1: a level's own inner lists, N = NI).
constexpr int kXcWarps = 4;
template <int W>
__global__ void __launch_bounds__(kXcWarps * 32) k_cheb_dct_add(const int* __restrict__ boxes,
                                                               int n_boxes,
                                                               const double* __restrict__ vals,
                                                               double* __restrict__ coef) {
  constexpr int N = W ? NI : NX, NNn = N * N;
  __shared__ double T[NNn];
  __shared__ double V[kXcWarps][NNn], Bm[kXcWarps][NNn];
  for (int o = threadIdx.x; o < NNn; o += kXcWarps * 32) T[o] = W ? c_TI[o] : c_TX[o];
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int bx = blockIdx.x * kXcWarps + warp;
  if (bx >= n_boxes) return;
  const uint32_t x = (uint32_t)boxes[bx];
  const double* v = vals + (size_t)x * NNn;
  for (int o = lane; o < NNn; o += 32) V[warp][o] = v[o];
  __syncwarp();
  for (int o = lane; o < NNn; o += 32) {  // Bm[i][m] = sum_j V[i][j] T[m][j]
    const int i = o / N, m = o % N;
    double s = 0.0;
    for (int j = 0; j < N; ++j) s = fma(V[warp][i * N + j], T[m * N + j], s);
    Bm[warp][o] = s;
  }
  __syncwarp();
  double* c = coef + (size_t)x * NN;
  for (int o = lane; o < NNn; o += 32) {
    const int k = o / N, m = o % N;
    double s = 0.0;
    for (int i = 0; i < N; ++i) s = fma(T[k * N + i], Bm[warp][i * N + m], s);
    s *= (2.0 / N) * (2.0 / N) * (k == 0 ? 0.5 : 1.0) * (m == 0 ? 0.5 : 1.0);
    c[k * NC + m] += s;
  }
}

// One CTA per box of level l (boxes listed in `boxes`): node values ->
// Chebyshev coefficients, plus the parent's series restricted to this box;
// base_parent < 0: plus what coef already holds for the box instead (the
// parent's restricted series and ring, k_cheb_ring_coef).
__global__ void __launch_bounds__(NN) k_cheb_coef(int l, const int* __restrict__ boxes,
                                                  long long base_l, long long base_parent,
                                                  const double* __restrict__ vals,
                                                  double* __restrict__ coef) {
  // (the tables are staged in shared memory: per-thread indices differ, and
  // constant memory serialises non-uniform addresses)
  __shared__ double a[NN], b[NN], T[NN], Sx[NN], Sy[NN];
  const uint32_t q = (uint32_t)boxes[blockIdx.x];
  const int r = threadIdx.x, k = r / NC, m = r % NC;
  const double* v = vals + (base_l + q) * NN;
  a[r] = v[r];
  T[r] = c_T[r];
  const bool restrict_parent = l > 1 && base_parent >= 0;
  if (restrict_parent) {
    Sx[r] = c_S[(q >> 1) & 1][r];
    Sy[r] = c_S[q & 1][r];
  }
  __syncthreads();
  // b[i][m] = sum_j v[i][j] T[m][j]
  {
    double s = 0.0;
    for (int j = 0; j < NC; ++j) s = fma(a[k * NC + j], T[m * NC + j], s);
    b[r] = s;  // (k plays i here)
  }
  __syncthreads();
  // c[k][m] = (2/n)^2 w_k w_m sum_i T[k][i] b[i][m]
  double c = 0.0;
  for (int i = 0; i < NC; ++i) c = fma(T[k * NC + i], b[i * NC + m], c);
  c *= (2.0 / NC) * (2.0 / NC) * (k == 0 ? 0.5 : 1.0) * (m == 0 ? 0.5 : 1.0);
  if (base_parent < 0) c += coef[(base_l + q) * NN + r];
  if (restrict_parent) {
    // parent series restricted to this quadrant: S_x C_p S_y^T
    const double* cp = coef + (base_parent + (q >> 2)) * NN;
    __syncthreads();
    a[r] = cp[r];
    __syncthreads();
    {
      double s = 0.0;  // b[k][m'] = sum_j Cp[k][j] Sy[m'][j]
      for (int j = 0; j < NC; ++j) s = fma(a[k * NC + j], Sy[m * NC + j], s);
      b[r] = s;
    }
    __syncthreads();
    double s = 0.0;  // c[k'][m'] += sum_k Sx[k'][k] b[k][m']
    for (int kk = 0; kk < NC; ++kk) s = fma(Sx[k * NC + kk], b[kk * NC + m], s);
    c += s;
  }
  coef[(base_l + q) * NN + r] = c;
}


// Same evaluation on the FP64 tensor cores (mma.sync m8n8k4 f64): per group
// of 8 targets, Z = Ty C^T ([8 x m] x [m x k], m padded to 4 KS, k to 8 NT)
// with the coefficient fragments held in registers for the whole item (no
// shared-memory traffic in the loop), then out = sum_k Z[., k] T_k(x^).
// Fragments (PTX m8n8k4 .f64): A (row) lane -> [lane/4][lane%4], B (col)
// lane -> [lane%4][lane/4], C/D lane -> [lane/4][2 (lane%4) + {0,1}].
// Chebyshev values by the step identities T_{n+4} = 2 T_4 T_n - T_{n-4} and
// T_{n+8} = 2 T_8 T_n - T_{n-8}, so a lane forms only the degrees it holds.
// x-degrees k >= 8 NT (the last NC % 8) are summed with plain FMAs instead of
// a third, mostly padded DMMA tile (10 instead of 15 DMMA per 8 targets).
constexpr int kMmaKS = (NC + 3) / 4, kMmaNT = NC / 8, kMmaRem = NC % 8, kMmaWarps = 4;
static_assert(kMmaRem == 0 || kMmaNT == 2, "remainder degrees 16..NC-1");
__device__ __forceinline__ void dmma_884(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}
__global__ void __launch_bounds__(kMmaWarps * 32) k_cheb_eval_mma(
    const TreeParams P, int lc, const int4* __restrict__ items, int n_items, long long base_lc,
    const double* __restrict__ coef, double* __restrict__ out) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int it = blockIdx.x * kMmaWarps + warp;
  if (it >= n_items) return;
  const int4 item = items[it];
  const uint32_t q = (uint32_t)item.x;
  const int s0 = item.y, cnt = item.z;
  const double* c = coef + (base_lc + q) * NN;
  const int r = lane >> 2, j = lane & 3;
  double b[kMmaNT][kMmaKS];
#pragma unroll
  for (int nt = 0; nt < kMmaNT; ++nt)
#pragma unroll
    for (int s = 0; s < kMmaKS; ++s) {
      const int m = 4 * s + j, k = 8 * nt + r;
      b[nt][s] = (m < NC && k < NC) ? __ldg(&c[k * NC + m]) : 0.0;
    }
  double cr[kMmaRem > 0 ? kMmaRem : 1][kMmaKS];  // C[16 + e][4 s + j]
#pragma unroll
  for (int e = 0; e < kMmaRem; ++e)
#pragma unroll
    for (int s = 0; s < kMmaKS; ++s) {
      const int m = 4 * s + j;
      cr[e][s] = m < NC ? __ldg(&c[(8 * kMmaNT + e) * NC + m]) : 0.0;
    }
  int bi, bj;
  demorton(q, bi, bj);
  const double cx = block_center(P.ox, bi, P.cell[lc]), cy = block_center(P.oy, bj, P.cell[lc]);
  const double inv = 2.0 / P.cell[lc];
  // one group of 8 targets (lane row r): sum_{k,m} C[k][m] T_k(x^) T_m(y^)
  auto group = [&](double xh, double yh) {
    // A: T_{4s+j}(y)
    double a[kMmaKS];
    {
      const double y2 = 2.0 * yh;
      const double t2 = fma(y2, yh, -1.0), t3 = fma(y2, t2, -yh), t4 = fma(y2, t3, -t2);
      const double tj = j == 0 ? 1.0 : (j == 1 ? yh : (j == 2 ? t2 : t3));
      const double tm = j == 0 ? t4 : (j == 1 ? t3 : (j == 2 ? t2 : yh));  // T_{4-j}
      const double t4x2 = 2.0 * t4;
      a[0] = tj;
      if (kMmaKS > 1) a[1] = fma(t4x2, tj, -tm);
#pragma unroll
      for (int s = 2; s < kMmaKS; ++s) a[s] = fma(t4x2, a[s - 1], -a[s - 2]);
    }
    double d[kMmaNT][2];
#pragma unroll
    for (int nt = 0; nt < kMmaNT; ++nt) {
      d[nt][0] = d[nt][1] = 0.0;
#pragma unroll
      for (int s = 0; s < kMmaKS; ++s) dmma_884(d[nt][0], d[nt][1], a[s], b[nt][s]);
    }
    // T_{8nt + 2j + e}(x), e = 0, 1
    const double x2 = 2.0 * xh;
    double T[9];
    T[0] = 1.0;
    T[1] = xh;
#pragma unroll
    for (int k = 2; k <= 8; ++k) T[k] = fma(x2, T[k - 1], -T[k - 2]);
    const double u0 = j == 0 ? T[0] : (j == 1 ? T[2] : (j == 2 ? T[4] : T[6]));
    const double u1 = j == 0 ? T[1] : (j == 1 ? T[3] : (j == 2 ? T[5] : T[7]));
    const double w0 = j == 0 ? T[8] : (j == 1 ? T[6] : (j == 2 ? T[4] : T[2]));  // T_{8-k0}
    const double w1 = j == 0 ? T[7] : (j == 1 ? T[5] : (j == 2 ? T[3] : T[1]));  // T_{8-k1}
    const double t8x2 = 2.0 * T[8];
    double p0 = u0, p1 = u1, q0 = w0, q1 = w1;  // T_{k+8(nt-1)} roles
    double v = d[0][0] * u0 + d[0][1] * u1;
#pragma unroll
    for (int nt = 1; nt < kMmaNT; ++nt) {
      const double n0 = fma(t8x2, p0, -q0), n1 = fma(t8x2, p1, -q1);
      v = fma(d[nt][0], n0, v);
      v = fma(d[nt][1], n1, v);
      q0 = p0;
      q1 = p1;
      p0 = n0;
      p1 = n1;
    }
    // remainder degrees 16 + e: this lane's part of sum_m C[16+e][m] T_m(y),
    // times T_{16+e}(x) = 2 T_8 T_{8+e} - T_e  (summed over the row's lanes below)
#pragma unroll
    for (int e = 0; e < kMmaRem; ++e) {
      double z = 0.0;
#pragma unroll
      for (int s = 0; s < kMmaKS; ++s) z = fma(cr[e][s], a[s], z);
      const double t8e = fma(t8x2, T[e], -T[8 - e]);
      v = fma(z, fma(t8x2, t8e, -T[e]), v);
    }
    v += __shfl_xor_sync(0xffffffffu, v, 1);
    v += __shfl_xor_sync(0xffffffffu, v, 2);
    return v;
  };
  // two independent groups per trip (ILP across the DMMA chains); targets
  // past cnt repeat the last one and are not stored
  // coordinates one trip ahead
  double x0 = P.xs[s0 + min(r, cnt - 1)], y0 = P.ys[s0 + min(r, cnt - 1)];
  double x1 = P.xs[s0 + min(8 + r, cnt - 1)], y1 = P.ys[s0 + min(8 + r, cnt - 1)];
  for (int g = 0; g < cnt; g += 16) {
    const int t0 = g + r, t1 = g + 8 + r;
    const double a0 = (x0 - cx) * inv, b0 = (y0 - cy) * inv;
    const double a1 = (x1 - cx) * inv, b1 = (y1 - cy) * inv;
    if (g + 16 < cnt) {
      const int n0 = s0 + min(t0 + 16, cnt - 1), n1 = s0 + min(t1 + 16, cnt - 1);
      x0 = P.xs[n0];
      y0 = P.ys[n0];
      x1 = P.xs[n1];
      y1 = P.ys[n1];
    }
    const double v0 = group(a0, b0);
    const double v1 = group(a1, b1);
    if (j == 0 && t0 < cnt) out[s0 + t0] = v0;
    if (j == 0 && t1 < cnt) out[s0 + t1] = v1;
  }
}

// The ring coefficients on the FP64 tensor cores.  A's series is first folded
// into the ring values (exact: its degree NC-1 <= NR-1 is reproduced by the
// NR-node interpolant),  V' = V + TT C_A TT^T  (TT[i][k] = T_k(x_i)),  then
// for each child  c = B_hx V' B_hy^T.  Every product is a 24 x 24 x 20
// zero-padded GEMM of m8n8k4 DMMA tiles (fragments from shared memory); the
// zero padding of the staged matrices makes the padded outputs exactly 0.
constexpr int kRcWarps = 4, kRcP = 24;  // padded leading dimension
static_assert(NR <= 20 && NC <= 20, "k-steps of 4 up to 20");
template <bool TA, bool TB>
__device__ __forceinline__ void rc_tile(const double* A, const double* Bm, int tm, int tn,
                                        int lane, double& d0, double& d1) {
  const int r = lane >> 2, c = lane & 3;
#pragma unroll
  for (int s = 0; s < 5; ++s) {
    const int k = 4 * s + c;
    // A[m][k] (TA: stored transposed, A[k][m]);  B[k][n] (TB: stored as B[n][k])
    const double a = TA ? A[k * kRcP + tm * 8 + r] : A[(tm * 8 + r) * kRcP + k];
    const double b = TB ? Bm[(tn * 8 + r) * kRcP + k] : Bm[k * kRcP + tn * 8 + r];
    dmma_884(d0, d1, a, b);
  }
}
__global__ void __launch_bounds__(kRcWarps * 32) k_cheb_ring_coef_mma(
    int v, const int* __restrict__ boxes, int n_boxes, long long base_a,
    const double* __restrict__ coef_a, const double* __restrict__ ring_vals,
    double* __restrict__ coef_c) {
  constexpr int S = kRcP * kRcP;
  __shared__ __align__(16) double TT[S], B[2][S], Ca[S], P[S], V[S], W[2][S];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nt = kRcWarps * 32;
  const int nr = v ? kChebNR2 : kChebNR, nrr = nr * nr;  // ring variant
  for (int o = threadIdx.x; o < S; o += nt) {
    const int i = o / kRcP, k = o % kRcP;
    TT[o] = (i < nr && k < NC) ? c_TR[v][k * nr + i] : 0.0;          // [i][k]
    B[0][o] = (i < NC && k < nr) ? c_B[v][0][i * nr + k] : 0.0;      // [k'][i]
    B[1][o] = (i < NC && k < nr) ? c_B[v][1][i * nr + k] : 0.0;
    Ca[o] = P[o] = V[o] = W[0][o] = W[1][o] = 0.0;
  }
  const int r = lane >> 2, cc = lane & 3;
  for (int bx = blockIdx.x; bx < n_boxes; bx += gridDim.x) {
    const uint32_t a = (uint32_t)boxes[bx];
    __syncthreads();  // tables / previous box done
    for (int o = threadIdx.x; o < nrr; o += nt)
      V[(o / nr) * kRcP + o % nr] = ring_vals[(size_t)a * nrr + o];
    for (int o = threadIdx.x; o < NN; o += nt)
      Ca[(o / NC) * kRcP + o % NC] = coef_a[(size_t)(base_a + a) * NN + o];
    __syncthreads();
    // P[k][j] = sum_m Ca[k][m] TT[j][m]   (B operand = TT stored transposed)
    for (int t = warp; t < 9; t += kRcWarps) {
      const int tm = t / 3, tn = t % 3;
      double d0 = 0.0, d1 = 0.0;
      rc_tile<false, true>(Ca, TT, tm, tn, lane, d0, d1);
      P[(tm * 8 + r) * kRcP + tn * 8 + 2 * cc] = d0;
      P[(tm * 8 + r) * kRcP + tn * 8 + 2 * cc + 1] = d1;
    }
    __syncthreads();
    // V'[i][j] = V[i][j] + sum_k TT[i][k] P[k][j]
    for (int t = warp; t < 9; t += kRcWarps) {
      const int tm = t / 3, tn = t % 3;
      double* v = &V[(tm * 8 + r) * kRcP + tn * 8 + 2 * cc];
      double d0 = v[0], d1 = v[1];
      rc_tile<false, false>(TT, P, tm, tn, lane, d0, d1);
      __syncwarp();
      v[0] = d0;
      v[1] = d1;
    }
    __syncthreads();
    // W[h][i][m'] = sum_j V'[i][j] B[h][m'][j]
    for (int t = warp; t < 18; t += kRcWarps) {
      const int h = t / 9, tm = (t % 9) / 3, tn = t % 3;
      double d0 = 0.0, d1 = 0.0;
      rc_tile<false, true>(V, B[h], tm, tn, lane, d0, d1);
      W[h][(tm * 8 + r) * kRcP + tn * 8 + 2 * cc] = d0;
      W[h][(tm * 8 + r) * kRcP + tn * 8 + 2 * cc + 1] = d1;
    }
    __syncthreads();
    // child (hx, hy): c[k'][m'] = sum_i B[hx][k'][i] W[hy][i][m']
    for (int t = warp; t < 36; t += kRcWarps) {
      const int ch = t / 9, tm = (t % 9) / 3, tn = t % 3;
      double d0 = 0.0, d1 = 0.0;
      rc_tile<false, false>(B[ch >> 1], W[ch & 1], tm, tn, lane, d0, d1);
      const int k = tm * 8 + r, m = tn * 8 + 2 * cc;
      double* out = coef_c + (size_t)(4 * a + ch) * NN + k * NC;
      if (k < NC) {
        if (m < NC) out[m] = d0;
        if (m + 1 < NC) out[m + 1] = d1;
      }
    }
  }
}

// ------------------------------------------------------- certificate ---
// Build-time interpolation certificate (operator.cu certify()): for every
// interpolated box, the tensor Chebyshev coefficients c_{k,m} of its n x n
// node values (n <= 20) are formed, and the error of the interpolant is
// estimated from their decay (the chebfun-style tail test on the data
// itself): with B2 = max |c| over the band max(k, m) in {n-2, n-1} and B4 the
// same over {n-4, n-3}, the per-degree decay is r = sqrt(B2 / B4) (clamped to
// <= 0.9: no visible convergence), and for |c_j| ~ A r^j the neglected
// coefficients of both variables, aliased onto the interpolant, sum to about
//     est = 4 B2 r^2 / (1 - r).
// Output per listed box: {est, max |value|}.
constexpr int kTailMaxN = 20;
__global__ void __launch_bounds__(128) k_cheb_tail(const int* __restrict__ boxes, int n_boxes,
                                                   const double* __restrict__ vals, int n,
                                                   double2* __restrict__ out) {
  __shared__ double V[kTailMaxN * kTailMaxN], T[kTailMaxN * kTailMaxN],
      W[kTailMaxN * kTailMaxN];
  __shared__ double red[3][4];
  const int nn = n * n;
  for (int o = threadIdx.x; o < nn; o += blockDim.x) {
    const int k = o / n, i = o % n;  // T[k][i] = cos(pi k (i + 1/2) / n)
    T[o] = cospi((double)(k * (2 * i + 1)) / (double)(2 * n));
  }
  for (int bx = blockIdx.x; bx < n_boxes; bx += gridDim.x) {
    const int q = boxes[bx];
    const double* v = vals + (size_t)q * nn;
    __syncthreads();
    double vmax = 0.0;
    for (int o = threadIdx.x; o < nn; o += blockDim.x) {
      V[o] = v[o];
      vmax = fmax(vmax, fabs(V[o]));
    }
    __syncthreads();
    for (int o = threadIdx.x; o < nn; o += blockDim.x) {  // W[i][m] = sum_j V[i][j] T[m][j]
      const int i = o / n, m = o % n;
      double acc = 0.0;
      for (int j = 0; j < n; ++j) acc = fma(V[i * n + j], T[m * n + j], acc);
      W[o] = acc;
    }
    __syncthreads();
    double b2 = 0.0, b4 = 0.0;
    for (int o = threadIdx.x; o < nn; o += blockDim.x) {
      const int k = o / n, m = o % n, d = max(k, m);
      if (d < n - 4) continue;
      double acc = 0.0;
      for (int i = 0; i < n; ++i) acc = fma(T[k * n + i], W[i * n + m], acc);
      acc = fabs(acc * (2.0 / n) * (2.0 / n) * (k == 0 ? 0.5 : 1.0) * (m == 0 ? 0.5 : 1.0));
      if (d >= n - 2) b2 = fmax(b2, acc); else b4 = fmax(b4, acc);
    }
    for (int d = 16; d; d >>= 1) {
      b2 = fmax(b2, __shfl_xor_sync(0xffffffffu, b2, d));
      b4 = fmax(b4, __shfl_xor_sync(0xffffffffu, b4, d));
      vmax = fmax(vmax, __shfl_xor_sync(0xffffffffu, vmax, d));
    }
    if ((threadIdx.x & 31) == 0) {
      red[0][threadIdx.x >> 5] = b2;
      red[1][threadIdx.x >> 5] = b4;
      red[2][threadIdx.x >> 5] = vmax;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double a = 0.0, b = 0.0, c = 0.0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
        a = fmax(a, red[0][w]);
        b = fmax(b, red[1][w]);
        c = fmax(c, red[2][w]);
      }
      const double r = b > 0.0 ? fmin(0.9, sqrt(a / b)) : (a > 0.0 ? 0.9 : 0.0);
      out[bx] = make_double2(4.0 * a * r * r / (1.0 - r), c);
    }
  }
}

__global__ void k_absmax(const double* __restrict__ x, long long n, double* __restrict__ out) {
  double m = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    m = fmax(m, fabs(x[i]));
  for (int d = 16; d; d >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, d));
  // |x| >= 0: the bit patterns of non-negative doubles order like the values
  if ((threadIdx.x & 31) == 0)
    atomicMax(reinterpret_cast<unsigned long long*>(out), (unsigned long long)__double_as_longlong(m));
}

// Constant-table uploads are checked: a failed upload would leave stale
// interpolation tables behind every later product.
void sym_check(cudaError_t e) {
  if (e != cudaSuccess)
    throw std::runtime_error(std::string("cudaMemcpyToSymbol (Chebyshev tables): ") +
                             cudaGetErrorString(e));
}

}  // namespace

void cheb_set_tables(const double* T, const double* S_left, const double* S_right) {
  sym_check(cudaMemcpyToSymbol(c_T, T, NN * sizeof(double)));
  sym_check(cudaMemcpyToSymbol(c_S, S_left, NN * sizeof(double), 0));
  sym_check(cudaMemcpyToSymbol(c_S, S_right, NN * sizeof(double), NN * sizeof(double)));
}

void cheb_set_ring_tables(int v, const double* T_nr, const double* B_left, const double* B_right) {
  const int nr = kRingNr[v];
  sym_check(cudaMemcpyToSymbol(c_TR, T_nr, (size_t)nr * nr * sizeof(double), (size_t)v * NRR * sizeof(double)));
  const size_t bsz = (size_t)NC * NR * sizeof(double);
  sym_check(cudaMemcpyToSymbol(c_B, B_left, (size_t)NC * nr * sizeof(double), ((size_t)v * 2 + 0) * bsz));
  sym_check(cudaMemcpyToSymbol(c_B, B_right, (size_t)NC * nr * sizeof(double), ((size_t)v * 2 + 1) * bsz));
}

void cheb_set_x_tables(const double* T_nx) {
  sym_check(cudaMemcpyToSymbol(c_TX, T_nx, NXX * sizeof(double)));
}

void launch_cheb_nodes_x(const TreeParams& P, int l, double* nx, double* ny, cudaStream_t s) {
  const long long n = (1ll << (2 * (l + 1))) * NXX;
  k_cheb_nodes_n<0><<<(unsigned)((n + 255) / 256), 256, 0, s>>>(P, l, 0, nx, ny);
}

void launch_cheb_xring_coef(const int* boxes, int n_boxes, const double* vals, double* coef,
                            cudaStream_t s) {
  if (n_boxes)
    k_cheb_dct_add<0><<<(unsigned)((n_boxes + kXcWarps - 1) / kXcWarps), kXcWarps * 32, 0, s>>>(
        boxes, n_boxes, vals, coef);
}

void cheb_set_inner_tables(const double* T_ni) {
  sym_check(cudaMemcpyToSymbol(c_TI, T_ni, (size_t)NI * NI * sizeof(double)));
}

void launch_cheb_nodes_inner(const TreeParams& P, int l, long long node_base, double* nx,
                             double* ny, cudaStream_t s) {
  const long long n = (1ll << (2 * (l + 1))) * NI * NI;
  k_cheb_nodes_n<1><<<(unsigned)((n + 255) / 256), 256, 0, s>>>(P, l, node_base, nx, ny);
}

void launch_cheb_inner_coef(const int* boxes, int n_boxes, const double* vals, double* coef,
                            cudaStream_t s) {
  if (n_boxes)
    k_cheb_dct_add<1><<<(unsigned)((n_boxes + kXcWarps - 1) / kXcWarps), kXcWarps * 32, 0, s>>>(
        boxes, n_boxes, vals, coef);
}

void launch_cheb_nodes_ring(const TreeParams& P, int l, int v, long long node_base, double* nx,
                            double* ny, cudaStream_t s) {
  const long long n = (1ll << (2 * (l + 1))) * kRingNr[v] * kRingNr[v];
  k_cheb_nodes_ring<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(P, l, v, node_base, nx, ny);
}

void launch_cheb_ring_coef(int v, const int* boxes, int n_boxes, long long base_a,
                           const double* coef_a, const double* ring_vals, double* coef_c,
                           cudaStream_t s) {
  if (n_boxes) {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int grid = std::min(n_boxes, 8 * std::max(sms, 1));
    k_cheb_ring_coef_mma<<<(unsigned)grid, kRcWarps * 32, 0, s>>>(v, boxes, n_boxes, base_a, coef_a,
                                                                  ring_vals, coef_c);
  }
}

void launch_cheb_nodes(const TreeParams& P, int l, long long box_base, double* nx, double* ny,
                       cudaStream_t s) {
  const long long n = (1ll << (2 * (l + 1))) * NN;
  k_cheb_nodes<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(P, l, box_base, nx, ny);
}

void launch_cheb_coef(int l, const int* boxes, int n_boxes, long long base_l,
                      long long base_parent, const double* vals, double* coef, cudaStream_t s) {
  if (n_boxes)
    k_cheb_coef<<<(unsigned)n_boxes, NN, 0, s>>>(l, boxes, base_l, base_parent, vals, coef);
}

void launch_cheb_eval(const TreeParams& P, int lc, const int4* items, int n_items,
                      long long base_lc, const double* coef, double* out, cudaStream_t s) {
  if (n_items)
    k_cheb_eval_mma<<<(unsigned)((n_items + kMmaWarps - 1) / kMmaWarps), kMmaWarps * 32, 0, s>>>(
        P, lc, items, n_items, base_lc, coef, out);
}

int cheb_eval_points_per_item() { return 1024; }

void launch_cheb_tail(const int* boxes, int n_boxes, const double* vals, int n, double2* out,
                      cudaStream_t s) {
  if (n < 3 || n > kTailMaxN) throw std::invalid_argument("cheb tail: node count out of range");
  if (n_boxes)
    k_cheb_tail<<<(unsigned)std::min(n_boxes, 148 * 16), 128, 0, s>>>(boxes, n_boxes, vals, n, out);
}

void launch_absmax(const double* x, long long n, double* out, cudaStream_t s) {
  cudaMemsetAsync(out, 0, sizeof(double), s);
  k_absmax<<<(unsigned)std::max(1ll, std::min(148ll * 8, (n + 255) / 256)), 256, 0, s>>>(x, n, out);
}

}  // namespace imqk
