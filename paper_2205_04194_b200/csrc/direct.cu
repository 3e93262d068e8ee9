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
#include "imq_device.cuh"
#include "imq_kernels.hpp"

namespace imqk {
using namespace imqdev;

namespace {

constexpr int kNearWarps = 4;

__global__ void __launch_bounds__(kNearWarps * 32) k_p2p_near(
    const TreeParams P, const int4* __restrict__ items, int n_items,
    const double* __restrict__ u_s, const double* __restrict__ far_s, double* __restrict__ out,
    const int* __restrict__ perm) {
  __shared__ double sx[kNearWarps][32], sy[kNearWarps][32], su[kNearWarps][32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int it = blockIdx.x * kNearWarps + warp;
  if (it >= n_items) return;
  const int4 item = items[it];
  const uint32_t leaf = (uint32_t)item.x;
  const int s0 = item.y, cnt = item.z;
  const bool valid = lane < cnt;
  const int p = valid ? s0 + lane : s0;
  const double xi = P.xs[p], yi = P.ys[p];
  const double t2 = P.t2;
  const int g = 1 << (P.L + 1);
  int li, lj;
  demorton(leaf, li, lj);
  double acc = 0.0;
  for (int qi = max(0, li - 1); qi <= min(g - 1, li + 1); ++qi) {
    for (int qj = max(0, lj - 1); qj <= min(g - 1, lj + 1); ++qj) {
      const uint32_t q = morton(qi, qj);
      const int a = P.leaf_start[q], b = P.leaf_start[q + 1];
      for (int base = a; base < b; base += 32) {
        const int j = base + lane;
        __syncwarp();
        if (j < b) {
          sx[warp][lane] = P.xs[j];
          sy[warp][lane] = P.ys[j];
          su[warp][lane] = u_s[j];
        }
        __syncwarp();
        const int nsrc = min(32, b - base);
        int k = 0;
        for (; k + 4 <= nsrc; k += 4) {
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const double dx = xi - sx[warp][k + kk], dy = yi - sy[warp][k + kk];
            acc = fma(su[warp][k + kk], rsqrt(fma(dx, dx, fma(dy, dy, t2))), acc);
          }
        }
        for (; k < nsrc; ++k) {
          const double dx = xi - sx[warp][k], dy = yi - sy[warp][k];
          acc = fma(su[warp][k], rsqrt(fma(dx, dx, fma(dy, dy, t2))), acc);
        }
      }
    }
  }
  if (valid) {
    const double v = far_s[p] + acc;
    out[perm ? perm[p] : p] = v;
  }
}

constexpr int kDirThreads = 256;

__global__ void __launch_bounds__(kDirThreads) k_direct(const double* __restrict__ txy,
                                                        long long nt,
                                                        const double* __restrict__ sxy,
                                                        const double* __restrict__ sval,
                                                        long long ns, double t2,
                                                        double* __restrict__ out) {
  __shared__ double2 sp[kDirThreads];
  __shared__ double sv[kDirThreads];
  const long long i = (long long)blockIdx.x * kDirThreads + threadIdx.x;
  double xi = 0.0, yi = 0.0;
  if (i < nt) {
    const double2 v = reinterpret_cast<const double2*>(txy)[i];
    xi = v.x;
    yi = v.y;
  }
  double acc = 0.0;
  for (long long base = 0; base < ns; base += kDirThreads) {
    const long long j = base + threadIdx.x;
    __syncthreads();
    if (j < ns) {
      sp[threadIdx.x] = reinterpret_cast<const double2*>(sxy)[j];
      sv[threadIdx.x] = sval[j];
    }
    __syncthreads();
    const int nsrc = (int)min((long long)kDirThreads, ns - base);
    if (nsrc == kDirThreads) {
#pragma unroll 8
      for (int k = 0; k < kDirThreads; ++k) {
        const double dx = xi - sp[k].x, dy = yi - sp[k].y;
        acc = fma(sv[k], rsqrt(fma(dx, dx, fma(dy, dy, t2))), acc);
      }
    } else {
      for (int k = 0; k < nsrc; ++k) {
        const double dx = xi - sp[k].x, dy = yi - sp[k].y;
        acc = fma(sv[k], rsqrt(fma(dx, dx, fma(dy, dy, t2))), acc);
      }
    }
  }
  if (i < nt) out[i] = acc;
}

}  // namespace

void launch_p2p_near(const TreeParams& P, const int4* items, int n_items, const double* u_s,
                     const double* far_s, double* out, const int* perm, cudaStream_t s) {
  if (n_items == 0) return;
  k_p2p_near<<<(unsigned)((n_items + kNearWarps - 1) / kNearWarps), kNearWarps * 32, 0, s>>>(
      P, items, n_items, u_s, far_s, out, perm);
}

void launch_direct(const double* txy, long long nt, const double* sxy, const double* sval,
                   long long ns, double t2, double* out, cudaStream_t s) {
  if (nt == 0) return;
  k_direct<<<(unsigned)((nt + kDirThreads - 1) / kDirThreads), kDirThreads, 0, s>>>(
      txy, nt, sxy, sval, ns, t2, out);
}

}  // namespace imqk
