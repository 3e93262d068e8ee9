// direct.cu -- direct IMQ interactions in FP64 on sm_100a.
//
//   P2P near field (reference fastmv.cpp:161-182): b_i += sum over the 3x3
//   finest-level neighbourhood of u_j / sqrt(t^2 + |x_i - x_j|^2), i = j
//   included.  Warp per (leaf, <= 32 targets); each source leaf streams through
//   a per-warp shared-memory tile, read back as broadcasts.  The epilogue adds
//   the far field and scatters to the original point order.
//
//   Dense product / interpolant evaluation (reference.cpp:11-28,
//   solver.cpp:161-172): tiled all-pairs kernel, one target per thread, source
//   tiles staged in shared memory; every thread sums its row in ascending j.
#include <stdexcept>

#include "imq_device.cuh"
#include "imq_kernels.hpp"

namespace imqk {
using namespace imqdev;

namespace {

constexpr int kNearWarps = 4;
constexpr int kNearMaxR = 4;  // a near work item holds <= 32 * kNearMaxR targets of one leaf
constexpr int kNearSymMaxR = 8;
constexpr int kNearBlockV = 4;   // right-hand sides per block near-field launch  // symmetric items: <= 16 * kNearSymMaxR points of one leaf (half-warp)

// Warp per near work item: <= 32 R targets of one leaf, R per lane.  Every
// source point staged in the warp's shared-memory tile is read back once per
// lane and reused for its R targets (register blocking against the per-LDS
// issue cost).  item.w encodes the source subset:
//   15       all 3x3 neighbour leaves; the epilogue adds the far field, scatters;
//   16 + r   neighbour row li-1+r   -> partial sums part[r][.]      (3-way split)
//   32 + k   neighbour leaf k of 9  -> partial sums part[k][.]      (9-way split)
// Small problems split the sources for parallelism; k_near_combine adds the
// partials in a fixed order (deterministic).
template <int R>
__global__ void __launch_bounds__(kNearWarps * 32) k_p2p_near(
    const TreeParams P, const int4* __restrict__ items, int n_items,
    const double* __restrict__ u_s, const double* __restrict__ far_s, double* __restrict__ out,
    const int* __restrict__ perm, double* __restrict__ part) {
  __shared__ double2 sxy[kNearWarps][32];
  __shared__ double su[kNearWarps][32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int it = blockIdx.x * kNearWarps + warp;
  if (it >= n_items) return;
  const int4 item = items[it];
  const uint32_t leaf = (uint32_t)item.x;
  const int s0 = item.y, cnt = item.z, sel = item.w;
  double xi[R], yi[R], acc[R];
#pragma unroll
  for (int p = 0; p < R; ++p) {
    const int q = lane + 32 * p < cnt ? s0 + lane + 32 * p : s0;
    xi[p] = P.xs[q];
    yi[p] = P.ys[q];
    acc[p] = 0.0;
  }
  const double t2 = P.t2;
  const int g = 1 << (P.L + 1);
  int li, lj;
  demorton(leaf, li, lj);
  int qilo = li - 1, qihi = li + 1, qjlo = lj - 1, qjhi = lj + 1, slot = 0;
  if (sel >= 32) {
    slot = sel - 32;
    qilo = qihi = li - 1 + slot / 3;
    qjlo = qjhi = lj - 1 + slot % 3;
  } else if (sel >= 16) {
    slot = sel - 16;
    qilo = qihi = li - 1 + slot;
  }
  // the (<= 9) source leaves as one virtual range, streamed in tiles of 32
  int rs[9], rc[9], total = 0;
#pragma unroll
  for (int k = 0; k < 9; ++k) {  // static indexing keeps the ranges in registers
    const int qi = li - 1 + k / 3, qj = lj - 1 + k % 3;
    rs[k] = rc[k] = 0;
    if (qi >= max(0, qilo) && qi <= min(g - 1, qihi) && qj >= max(0, qjlo) &&
        qj <= min(g - 1, qjhi)) {
      const uint32_t q = morton(qi, qj);
      rs[k] = P.leaf_start[q];
      rc[k] = P.leaf_start[q + 1] - rs[k];
      total += rc[k];
    }
  }
  auto fetch = [&](int v, double& x, double& y, double& u) {
    // virtual index -> sorted position; padding slots carry u = 0
    int pos = -1;
#pragma unroll
    for (int k = 0; k < 9; ++k) {
      if (pos < 0 && v < rc[k]) pos = rs[k] + v;
      if (pos < 0) v -= rc[k];
    }
    if (pos < 0) {
      x = xi[0];
      y = yi[0];
      u = 0.0;
    } else {
      x = P.xs[pos];
      y = P.ys[pos];
      u = u_s[pos];
    }
  };
  double nx, ny, nu;
  fetch(lane, nx, ny, nu);
  for (int v = 0; v < total; v += 32) {
    __syncwarp();
    sxy[warp][lane] = make_double2(nx, ny);
    su[warp][lane] = nu;
    __syncwarp();
    if (v + 32 < total) fetch(v + 32 + lane, nx, ny, nu);  // in flight during the tile
#pragma unroll 8
    for (int k = 0; k < 32; ++k) {
      const double2 sp = sxy[warp][k];
      const double uk = su[warp][k];
#pragma unroll
      for (int p = 0; p < R; ++p) {
        const double dx = xi[p] - sp.x, dy = yi[p] - sp.y;
        acc[p] = fma(uk, rsqrt_pos(fma(dx, dx, fma(dy, dy, t2))), acc[p]);
      }
    }
  }
#pragma unroll
  for (int p = 0; p < R; ++p) {
    if (lane + 32 * p < cnt) {
      const int q = s0 + lane + 32 * p;
      if (sel == 15) {
        const double v = far_s[q] + acc[p];
        out[perm ? perm[q] : q] = v;
      } else {
        part[(size_t)slot * P.N + q] = acc[p];
      }
    }
  }
}

// Symmetric near field (every leaf <= 128 points), two leaves per warp: the
// half-warp h (16 lanes, shuffles and syncs on its own 16-lane mask) takes
// item 2w + h, the <= 16 R points of one leaf C, R per lane (R = ceil(count /
// 16): a 65..80-point leaf fills 80 slots instead of 96, and every staged
// source feeds 2R pair evaluations).  The item evaluates C's self tile and
// each unordered pair {C, B} with B one of its four "forward" neighbours
// (0,+1), (+1,-1), (+1,0), (+1,+1) once: forward sums sum_j u_j phi_ij
// accumulate in registers (slot 0), and the reverse sums sum_i u_i phi_ij for
// B's points are formed by a register that rotates through the half's lanes
// with one shuffle per step (lane l evaluates source (l + k) mod 16 at step
// k), ending in lane j for source j; they go to B's slot 1 + dir.  Slots are
// combined with the far field in a fixed order.  Items of one R group are
// sorted by their forward-source count, so the two halves of a warp run
// loops of (nearly) the same length.
// V right-hand sides at once (block product, V > 1): the kernel values phi
// are evaluated once and feed V forward and V reverse sums; vector v of the
// block lives at u_s + v * ustride, its partial slots at part + v * pstride.
// Every sum has the single-vector order, so a block equals V single products
// bit for bit.
template <int R, int V>
__global__ void __launch_bounds__(kNearWarps * 32) k_p2p_near_sym(
    const TreeParams P, const int4* __restrict__ items, int n_items,
    const double* __restrict__ u_s, size_t ustride, double* __restrict__ part, size_t pstride) {
  __shared__ double2 sxy[2 * kNearWarps][16];
  __shared__ double su[2 * kNearWarps][16][V];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, hl = lane & 15;
  const int hw = 2 * warp + (lane >> 4);
  const unsigned hm = 0xffffu << (lane & 16);
  const int it = (blockIdx.x * kNearWarps + warp) * 2 + (lane >> 4);
  if (it >= n_items) return;
  const int4 item = items[it];
  const uint32_t leaf = (uint32_t)item.x;
  const int s0 = item.y, cnt = item.z;
  const size_t N = (size_t)P.N;
  double xi[R], yi[R], ui[R][V], acc[R][V];
#pragma unroll
  for (int p = 0; p < R; ++p) {
    const bool v = hl + 16 * p < cnt;
    const int q = v ? s0 + hl + 16 * p : s0;
    xi[p] = P.xs[q];
    yi[p] = P.ys[q];
#pragma unroll
    for (int w = 0; w < V; ++w) {
      ui[p][w] = v ? u_s[q + w * ustride] : 0.0;  // padded targets must not feed reverse sums
      acc[p][w] = 0.0;
    }
  }
  const double t2 = P.t2;
  const int g = 1 << (P.L + 1);
  int li, lj;
  demorton(leaf, li, lj);
  // self block (the whole leaf is in this half's registers), each unordered
  // pair once: source tile pt = the targets of slot pt.  Slots p < pt take a
  // full rotation against the tile (forward into acc[p], the reverse sums
  // rotate into lane j = target j of slot pt); slot pt itself takes a half
  // rotation (k = 0: the pair (i, i), forward only; k = 1..7; k = 8 by lanes
  // 0..7 only), its reverse sums realigned by 9 lanes.
  const int ntile = (cnt + 15) / 16;
#pragma unroll
  for (int pt = 0; pt < R; ++pt) {
    if (pt >= ntile) break;
    __syncwarp(hm);
    sxy[hw][hl] = make_double2(xi[pt], yi[pt]);  // padding: a valid point, u = 0
#pragma unroll
    for (int w = 0; w < V; ++w) su[hw][hl][w] = ui[pt][w];
    __syncwarp(hm);
    if (pt > 0) {
      double racc[V];
#pragma unroll
      for (int w = 0; w < V; ++w) racc[w] = 0.0;
#pragma unroll 8
      for (int k = 0; k < 16; ++k) {
        const int jj = (hl + k) & 15;
        const double2 sp = sxy[hw][jj];
        double uk[V], r[V];
#pragma unroll
        for (int w = 0; w < V; ++w) {
          uk[w] = su[hw][jj][w];
          r[w] = 0.0;
        }
#pragma unroll
        for (int p = 0; p < R; ++p) {
          if (p < pt) {
            const double dx = xi[p] - sp.x, dy = yi[p] - sp.y;
            const double phi = rsqrt_pos(fma(dx, dx, fma(dy, dy, t2)));
#pragma unroll
            for (int w = 0; w < V; ++w) {
              acc[p][w] = fma(uk[w], phi, acc[p][w]);
              r[w] = fma(ui[p][w], phi, r[w]);
            }
          }
        }
#pragma unroll
        for (int w = 0; w < V; ++w) {
          racc[w] += r[w];
          racc[w] = __shfl_sync(hm, racc[w], (hl + 1) & 15, 16);
        }
      }
#pragma unroll
      for (int w = 0; w < V; ++w) acc[pt][w] += racc[w];
    }
    {
      const double dx0 = xi[pt] - xi[pt], dy0 = yi[pt] - yi[pt];
      const double phi0 = rsqrt_pos(fma(dx0, dx0, fma(dy0, dy0, t2)));
      double racc[V];
#pragma unroll
      for (int w = 0; w < V; ++w) {
        acc[pt][w] = fma(ui[pt][w], phi0, acc[pt][w]);  // k = 0
        racc[w] = 0.0;
      }
#pragma unroll
      for (int k = 1; k <= 8; ++k) {
        const int jj = (hl + k) & 15;
        const double2 sp = sxy[hw][jj];
        const bool on = k < 8 || hl < 8;
        const double dx = xi[pt] - sp.x, dy = yi[pt] - sp.y;
        const double phi = rsqrt_pos(fma(dx, dx, fma(dy, dy, t2)));
#pragma unroll
        for (int w = 0; w < V; ++w) {
          const double uk = on ? su[hw][jj][w] : 0.0;
          const double ul = on ? ui[pt][w] : 0.0;
          acc[pt][w] = fma(uk, phi, acc[pt][w]);
          racc[w] = fma(ul, phi, racc[w]);
          racc[w] = __shfl_sync(hm, racc[w], (hl + 1) & 15, 16);
        }
      }
#pragma unroll
      for (int w = 0; w < V; ++w) acc[pt][w] += __shfl_sync(hm, racc[w], (hl + 7) & 15, 16);
    }
  }
  // forward neighbours: forward + reverse sums over the concatenation of the
  // four neighbour ranges (tiles of 16 sources cross leaf boundaries)
  int na[4], nb[4];
#pragma unroll
  for (int dir = 0; dir < 4; ++dir) {
    const int bi = li + (dir == 0 ? 0 : 1);
    const int bj = lj + (dir == 0 ? 1 : dir - 2);
    na[dir] = nb[dir] = 0;
    if (bi > g - 1 || bj < 0 || bj > g - 1) continue;
    const uint32_t q = morton(bi, bj);
    na[dir] = P.leaf_start[q];
    nb[dir] = P.leaf_start[q + 1];
  }
  const int e1 = nb[0] - na[0], e2 = e1 + nb[1] - na[1], e3 = e2 + nb[2] - na[2];
  const int total = e3 + nb[3] - na[3];
  for (int base = 0; base < total; base += 16) {
    const int v = base + hl;
    const int dir = v < e1 ? 0 : (v < e2 ? 1 : (v < e3 ? 2 : 3));
    const int j = na[dir] + v - (dir == 0 ? 0 : (dir == 1 ? e1 : (dir == 2 ? e2 : e3)));
    __syncwarp(hm);
    if (v < total) {
      sxy[hw][hl] = make_double2(P.xs[j], P.ys[j]);
#pragma unroll
      for (int w = 0; w < V; ++w) su[hw][hl][w] = u_s[j + w * ustride];
    } else {
      sxy[hw][hl] = make_double2(xi[0], yi[0]);
#pragma unroll
      for (int w = 0; w < V; ++w) su[hw][hl][w] = 0.0;
    }
    __syncwarp(hm);
    double racc[V];
#pragma unroll
    for (int w = 0; w < V; ++w) racc[w] = 0.0;
#pragma unroll 8
    for (int k = 0; k < 16; ++k) {
      const int jj = (hl + k) & 15;
      const double2 sp = sxy[hw][jj];
      double uk[V], r[V];
#pragma unroll
      for (int w = 0; w < V; ++w) {
        uk[w] = su[hw][jj][w];
        r[w] = 0.0;
      }
#pragma unroll
      for (int p = 0; p < R; ++p) {
        const double dx = xi[p] - sp.x, dy = yi[p] - sp.y;
        const double phi = rsqrt_pos(fma(dx, dx, fma(dy, dy, t2)));
#pragma unroll
        for (int w = 0; w < V; ++w) {
          acc[p][w] = fma(uk[w], phi, acc[p][w]);
          r[w] = fma(ui[p][w], phi, r[w]);
        }
      }
#pragma unroll
      for (int w = 0; w < V; ++w) {
        racc[w] += r[w];
        racc[w] = __shfl_sync(hm, racc[w], (hl + 1) & 15, 16);
      }
    }
    if (v < total) {  // lane holds its source's reverse sums
#pragma unroll
      for (int w = 0; w < V; ++w) part[w * pstride + (size_t)(1 + dir) * N + j] = racc[w];
    }
  }
#pragma unroll
  for (int p = 0; p < R; ++p)
    if (hl + 16 * p < cnt) {
#pragma unroll
      for (int w = 0; w < V; ++w) part[w * pstride + s0 + hl + 16 * p] = acc[p][w];
    }
  // reverse slots nobody writes (no / empty backward neighbour): zero them here
#pragma unroll 1
  for (int dir = 0; dir < 4; ++dir) {
    const int ci = li - (dir == 0 ? 0 : 1);
    const int cj = lj - (dir == 0 ? 1 : dir - 2);
    bool has = ci >= 0 && cj >= 0 && cj <= g - 1;
    if (has) {
      const uint32_t q = morton(ci, cj);
      has = P.leaf_start[q + 1] > P.leaf_start[q];
    }
    if (!has)
      for (int p = hl; p < cnt; p += 16) {
#pragma unroll
        for (int w = 0; w < V; ++w) part[w * pstride + (size_t)(1 + dir) * N + s0 + p] = 0.0;
      }
  }
}

// Sharded symmetric near field: a rank evaluates the pairs {C, B} of its own
// leaves C (k_p2p_near_sym), which leaves, for an own leaf B whose backward
// neighbour C in direction d belongs to another rank, slot 1 + d unwritten.
// This kernel fills exactly those: items {b_start, b_cnt | d << 16, c_start,
// c_cnt}, part[(1 + d) N + j] = sum_{i in C} u_i phi(x_j, x_i) for j in B.
__global__ void __launch_bounds__(kNearWarps * 32) k_p2p_pull(
    const TreeParams P, const int4* __restrict__ items, int n_items,
    const double* __restrict__ u_s, double* __restrict__ part) {
  constexpr int R = kNearMaxR;
  __shared__ double2 sxy[kNearWarps][32];
  __shared__ double su[kNearWarps][32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int it = blockIdx.x * kNearWarps + warp;
  if (it >= n_items) return;
  const int4 item = items[it];
  const int b0 = item.x, nb = item.y & 0xffff, dir = item.y >> 16, c0 = item.z, nc = item.w;
  double xi[R], yi[R], acc[R];
#pragma unroll
  for (int p = 0; p < R; ++p) {
    const int q = lane + 32 * p < nb ? b0 + lane + 32 * p : b0;
    xi[p] = P.xs[q];
    yi[p] = P.ys[q];
    acc[p] = 0.0;
  }
  const double t2 = P.t2;
  for (int base = 0; base < nc; base += 32) {
    __syncwarp();
    if (base + lane < nc) {
      sxy[warp][lane] = make_double2(P.xs[c0 + base + lane], P.ys[c0 + base + lane]);
      su[warp][lane] = u_s[c0 + base + lane];
    } else {
      sxy[warp][lane] = make_double2(xi[0], yi[0]);
      su[warp][lane] = 0.0;
    }
    __syncwarp();
#pragma unroll 8
    for (int k = 0; k < 32; ++k) {
      const double2 sp = sxy[warp][k];
      const double uk = su[warp][k];
#pragma unroll
      for (int p = 0; p < R; ++p) {
        const double dx = xi[p] - sp.x, dy = yi[p] - sp.y;
        acc[p] = fma(uk, rsqrt_pos(fma(dx, dx, fma(dy, dy, t2))), acc[p]);
      }
    }
  }
#pragma unroll
  for (int p = 0; p < R; ++p)
    if (lane + 32 * p < nb) part[(size_t)(1 + dir) * P.N + b0 + lane + 32 * p] = acc[p];
}

// Symmetric near field for large leaves: items are unordered pairs of leaf
// chunks (<= 32 R points each) {A, B} -- A's chunk with itself, with the later
// chunks of its own leaf, and with every chunk of its four forward neighbour
// leaves.  Each pair's kernel values are evaluated once: forward sums for A's
// points and (pairs A != B) reverse sums for B's points, via the lane rotation
// of k_p2p_near_sym, are written to the item's two partial rows; a reduction
// kernel then adds, for every chunk, its rows in a fixed order.
template <int R>
__global__ void __launch_bounds__(kNearWarps * 32) k_p2p_pair(
    const TreeParams P, const int4* __restrict__ items, int n_items,
    const double* __restrict__ u_s, double* __restrict__ part) {
  __shared__ double2 sxy[kNearWarps][32];
  __shared__ double su[kNearWarps][32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int it = blockIdx.x * kNearWarps + warp;
  if (it >= n_items) return;
  const int4 item = items[it];
  const int a0 = item.x, na = item.y, b0 = item.z, nb = item.w;
  const bool self = a0 == b0;
  double* fwd = part + (size_t)it * (2 * kNearChunk);  // rows: forward, then reverse
  double* rev = fwd + kNearChunk;
  double xi[R], yi[R], ui[R], acc[R];
#pragma unroll
  for (int p = 0; p < R; ++p) {
    const bool v = lane + 32 * p < na;
    const int q = v ? a0 + lane + 32 * p : a0;
    xi[p] = P.xs[q];
    yi[p] = P.ys[q];
    ui[p] = v ? u_s[q] : 0.0;
    acc[p] = 0.0;
  }
  const double t2 = P.t2;
  for (int base = 0; base < nb; base += 32) {
    const int j = b0 + base + lane;
    __syncwarp();
    if (base + lane < nb) {
      sxy[warp][lane] = make_double2(P.xs[j], P.ys[j]);
      su[warp][lane] = u_s[j];
    } else {
      sxy[warp][lane] = make_double2(xi[0], yi[0]);
      su[warp][lane] = 0.0;
    }
    __syncwarp();
    if (self) {
#pragma unroll 8
      for (int k = 0; k < 32; ++k) {
        const double2 sp = sxy[warp][k];
        const double uk = su[warp][k];
#pragma unroll
        for (int p = 0; p < R; ++p) {
          const double dx = xi[p] - sp.x, dy = yi[p] - sp.y;
          acc[p] = fma(uk, rsqrt_pos(fma(dx, dx, fma(dy, dy, t2))), acc[p]);
        }
      }
    } else {
      double racc = 0.0;
#pragma unroll 8
      for (int k = 0; k < 32; ++k) {
        const int jj = (lane + k) & 31;
        const double2 sp = sxy[warp][jj];
        const double uk = su[warp][jj];
        double r = 0.0;
#pragma unroll
        for (int p = 0; p < R; ++p) {
          const double dx = xi[p] - sp.x, dy = yi[p] - sp.y;
          const double phi = rsqrt_pos(fma(dx, dx, fma(dy, dy, t2)));
          acc[p] = fma(uk, phi, acc[p]);
          r = fma(ui[p], phi, r);
        }
        racc += r;
        racc = __shfl_sync(0xffffffffu, racc, (lane + 1) & 31);
      }
      if (base + lane < nb) rev[base + lane] = racc;
    }
  }
#pragma unroll
  for (int p = 0; p < R; ++p)
    if (lane + 32 * p < na) fwd[lane + 32 * p] = acc[p];
}

// Block per chunk, thread per point: near = sum of the chunk's partial rows
// (contrib entries = row offsets into part) in their fixed list order; with
// far_s set, out[perm[q]] = far_s[q] + near (the product's final combine).
__global__ void __launch_bounds__(128) k_pair_reduce(const int2* __restrict__ chunks,
                                                     const int* __restrict__ contrib_off,
                                                     const int* __restrict__ contrib,
                                                     const double* __restrict__ part,
                                                     double* __restrict__ near_s,
                                                     const double* __restrict__ far_s,
                                                     const int* __restrict__ perm) {
  const int2 c = chunks[blockIdx.x];
  for (int k = threadIdx.x; k < c.y; k += blockDim.x) {
    double sum = 0.0;
    for (int e = contrib_off[blockIdx.x]; e < contrib_off[blockIdx.x + 1]; ++e)
      sum += part[(size_t)contrib[e] + k];
    const int q = c.x + k;
    if (far_s)
      near_s[perm ? perm[q] : q] = far_s[q] + sum;
    else
      near_s[q] = sum;
  }
}

__global__ void __launch_bounds__(256) k_near_combine(int lo, int hi, int N, int nparts,
                                                      const double* __restrict__ far_s,
                                                      const double* __restrict__ part,
                                                      double* __restrict__ out,
                                                      const int* __restrict__ perm) {
  const int q = lo + blockIdx.x * 256 + threadIdx.x;
  if (q >= hi) return;
  double nsum = 0.0;
  for (int k = 0; k < nparts; ++k) nsum += part[(size_t)k * N + q];
  out[perm ? perm[q] : q] = far_s[q] + nsum;
}

constexpr int kDirThreads = 256;
constexpr int kDirR = 4;  // targets per thread (register blocking)

// b_q = sum_j c_j / sqrt(t^2 + |x_q - y_j|^2): each thread owns kDirR targets
// and sums its rows in ascending j over source tiles staged in shared memory.
__global__ void __launch_bounds__(kDirThreads) k_direct(const double* __restrict__ txy,
                                                        long long nt,
                                                        const double* __restrict__ sxy,
                                                        const double* __restrict__ sval,
                                                        long long ns, double t2,
                                                        double* __restrict__ out) {
  __shared__ double2 sp[kDirThreads];
  __shared__ double sv[kDirThreads];
  const long long i0 = (long long)blockIdx.x * kDirThreads * kDirR + threadIdx.x;
  double xi[kDirR], yi[kDirR], acc[kDirR];
#pragma unroll
  for (int r = 0; r < kDirR; ++r) {
    const long long i = i0 + (long long)r * kDirThreads;
    double2 v = make_double2(0.0, 0.0);
    if (i < nt) v = reinterpret_cast<const double2*>(txy)[i];
    xi[r] = v.x;
    yi[r] = v.y;
    acc[r] = 0.0;
  }
  for (long long base = 0; base < ns; base += kDirThreads) {
    const long long j = base + threadIdx.x;
    __syncthreads();
    if (j < ns) {
      sp[threadIdx.x] = reinterpret_cast<const double2*>(sxy)[j];
      sv[threadIdx.x] = sval[j];
    }
    __syncthreads();
    const int nsrc = (int)min((long long)kDirThreads, ns - base);
#pragma unroll 4
    for (int k = 0; k < nsrc; ++k) {
      const double2 p = sp[k];
      const double c = sv[k];
#pragma unroll
      for (int r = 0; r < kDirR; ++r) {
        const double dx = xi[r] - p.x, dy = yi[r] - p.y;
        acc[r] = fma(c, rsqrt_pos(fma(dx, dx, fma(dy, dy, t2))), acc[r]);
      }
    }
  }
#pragma unroll
  for (int r = 0; r < kDirR; ++r) {
    const long long i = i0 + (long long)r * kDirThreads;
    if (i < nt) out[i] = acc[r];
  }
}

}  // namespace

int near_max_points_per_lane() { return kNearMaxR; }

template <int V>
static void launch_near_sym_v(const TreeParams& P, const int4* items, const int* group_off,
                              int begin, int end, const double* u_s, size_t ustride, double* part,
                              size_t pstride, cudaStream_t s) {
  for (int R = kNearSymMaxR; R >= 1; --R) {  // longest items first
    const int lo = max(begin, group_off[R - 1]), hi = min(end, group_off[R]);
    if (hi <= lo) continue;
    const unsigned grid = (unsigned)((hi - lo + 2 * kNearWarps - 1) / (2 * kNearWarps));
#define NEAR_SYM_CASE(r)                                                                        \
  case r:                                                                                       \
    k_p2p_near_sym<r, V><<<grid, kNearWarps * 32, 0, s>>>(P, items + lo, hi - lo, u_s, ustride, \
                                                          part, pstride);                       \
    break;
    switch (R) {
      NEAR_SYM_CASE(1) NEAR_SYM_CASE(2) NEAR_SYM_CASE(3) NEAR_SYM_CASE(4)
      NEAR_SYM_CASE(5) NEAR_SYM_CASE(6) NEAR_SYM_CASE(7)
      default:
        k_p2p_near_sym<8, V><<<grid, kNearWarps * 32, 0, s>>>(P, items + lo, hi - lo, u_s, ustride,
                                                              part, pstride);
        break;
    }
#undef NEAR_SYM_CASE
  }
}

void launch_p2p_near_sym(const TreeParams& P, const int4* items, const int* group_off, int begin,
                         int end, const double* u_s, double* part, cudaStream_t s) {
  launch_near_sym_v<1>(P, items, group_off, begin, end, u_s, 0, part, 0, s);
}

// Block near field: nv (2..kNearBlockV) vectors share every kernel evaluation.
int near_block_max() { return kNearBlockV; }
void launch_p2p_near_sym_block(const TreeParams& P, const int4* items, const int* group_off,
                               int begin, int end, int nv, const double* u_s, size_t ustride,
                               double* part, size_t pstride, cudaStream_t s) {
  switch (nv) {
    case 1: launch_near_sym_v<1>(P, items, group_off, begin, end, u_s, ustride, part, pstride, s); break;
    case 2: launch_near_sym_v<2>(P, items, group_off, begin, end, u_s, ustride, part, pstride, s); break;
    case 3: launch_near_sym_v<3>(P, items, group_off, begin, end, u_s, ustride, part, pstride, s); break;
    case 4: launch_near_sym_v<4>(P, items, group_off, begin, end, u_s, ustride, part, pstride, s); break;
    default: throw std::invalid_argument("near block: 1..4 vectors per launch");
  }
}

void launch_p2p_pair(const TreeParams& P, const int4* items, const int* group_off,
                     const double* u_s, double* part, cudaStream_t s) {
  for (int R = kPairR; R >= 1; --R) {
    const int lo = group_off[R - 1], n = group_off[R] - lo;
    if (n <= 0) continue;
    const unsigned grid = (unsigned)((n + kNearWarps - 1) / kNearWarps);
    double* pp = part + (size_t)lo * 2 * kNearChunk;
    switch (R) {
      case 1: k_p2p_pair<1><<<grid, kNearWarps * 32, 0, s>>>(P, items + lo, n, u_s, pp); break;
      case 2: k_p2p_pair<2><<<grid, kNearWarps * 32, 0, s>>>(P, items + lo, n, u_s, pp); break;
      case 3: k_p2p_pair<3><<<grid, kNearWarps * 32, 0, s>>>(P, items + lo, n, u_s, pp); break;
      default: k_p2p_pair<4><<<grid, kNearWarps * 32, 0, s>>>(P, items + lo, n, u_s, pp); break;
    }
  }
}

void launch_p2p_pull(const TreeParams& P, const int4* items, int n_items, const double* u_s,
                     double* part, cudaStream_t s) {
  if (n_items)
    k_p2p_pull<<<(unsigned)((n_items + kNearWarps - 1) / kNearWarps), kNearWarps * 32, 0, s>>>(
        P, items, n_items, u_s, part);
}

void launch_pair_reduce(const int2* chunks, int n_chunks, const int* contrib_off,
                        const int* contrib, const double* part, double* out,
                        const double* far_s, const int* perm, cudaStream_t s) {
  if (n_chunks)
    k_pair_reduce<<<(unsigned)n_chunks, 128, 0, s>>>(chunks, contrib_off, contrib, part, out,
                                                     far_s, perm);
}

void launch_near_combine(int lo, int hi, int N, int nparts, const double* far_s,
                         const double* part, double* out, const int* perm, cudaStream_t s) {
  if (hi <= lo) return;
  k_near_combine<<<(unsigned)((hi - lo + 255) / 256), 256, 0, s>>>(lo, hi, N, nparts, far_s,
                                                                   part, out, perm);
}

void launch_p2p_near(const TreeParams& P, const int4* items, const int* group_off, int begin,
                     int end, const double* u_s, const double* far_s, double* out,
                     const int* perm, double* part, cudaStream_t s) {
  for (int R = 1; R <= kNearMaxR; ++R) {
    const int lo = max(begin, group_off[R - 1]), hi = min(end, group_off[R]);
    if (hi <= lo) continue;
    const unsigned grid = (unsigned)((hi - lo + kNearWarps - 1) / kNearWarps);
    switch (R) {
      case 1: k_p2p_near<1><<<grid, kNearWarps * 32, 0, s>>>(P, items + lo, hi - lo, u_s, far_s, out, perm, part); break;
      case 2: k_p2p_near<2><<<grid, kNearWarps * 32, 0, s>>>(P, items + lo, hi - lo, u_s, far_s, out, perm, part); break;
      case 3: k_p2p_near<3><<<grid, kNearWarps * 32, 0, s>>>(P, items + lo, hi - lo, u_s, far_s, out, perm, part); break;
      default: k_p2p_near<4><<<grid, kNearWarps * 32, 0, s>>>(P, items + lo, hi - lo, u_s, far_s, out, perm, part); break;
    }
  }
}

void launch_direct(const double* txy, long long nt, const double* sxy, const double* sval,
                   long long ns, double t2, double* out, cudaStream_t s) {
  if (nt == 0) return;
  const long long per = (long long)kDirThreads * kDirR;
  k_direct<<<(unsigned)((nt + per - 1) / per), kDirThreads, 0, s>>>(txy, nt, sxy, sval, ns, t2,
                                                                    out);
}

}  // namespace imqk
