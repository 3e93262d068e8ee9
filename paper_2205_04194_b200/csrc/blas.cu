// blas.cu -- vector kernels of the device-resident GMRES (reference
// solver.cpp:14-28 nrm2/dot/axpy).  Reductions use a fixed grid and a fixed
// combine order, so every dot product is bitwise reproducible run to run.
// Scalars produced on the device (MGS coefficients h_ij) are consumed on the
// device, so the modified Gram-Schmidt chain needs no host round trip.
#include <cooperative_groups.h>

#include <cstdlib>

#include "imq_kernels.hpp"

namespace cg = cooperative_groups;

namespace imqk {

namespace {

constexpr int kThreads = 256;

__global__ void __launch_bounds__(kThreads) k_dot_partial(const double* __restrict__ a,
                                                          const double* __restrict__ b,
                                                          long long n,
                                                          double* __restrict__ partial) {
  double s = 0.0;
  for (long long i = blockIdx.x * (long long)kThreads + threadIdx.x; i < n;
       i += (long long)gridDim.x * kThreads)
    s = fma(a[i], b[i], s);
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  __shared__ double red[kThreads / 32];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < kThreads / 32; ++w) t += red[w];
    partial[blockIdx.x] = t;
  }
}

__global__ void __launch_bounds__(kThreads) k_dot_final(const double* __restrict__ partial,
                                                        int nparts, double* out, int take_sqrt) {
  double s = 0.0;
  for (int i = threadIdx.x; i < nparts; i += kThreads) s += partial[i];
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  __shared__ double red[kThreads / 32];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < kThreads / 32; ++w) t += red[w];
    *out = take_sqrt ? sqrt(t) : t;
  }
}

__global__ void __launch_bounds__(kThreads) k_axpy_dev(double* __restrict__ y,
                                                       const double* __restrict__ x, long long n,
                                                       const double* __restrict__ alpha,
                                                       double sign) {
  const double a = sign * *alpha;
  for (long long i = blockIdx.x * (long long)kThreads + threadIdx.x; i < n;
       i += (long long)gridDim.x * kThreads)
    y[i] = fma(a, x[i], y[i]);
}
__global__ void __launch_bounds__(kThreads) k_axpy(double* __restrict__ y,
                                                   const double* __restrict__ x, long long n,
                                                   double a) {
  for (long long i = blockIdx.x * (long long)kThreads + threadIdx.x; i < n;
       i += (long long)gridDim.x * kThreads)
    y[i] = fma(a, x[i], y[i]);
}
__global__ void __launch_bounds__(kThreads) k_div(double* __restrict__ out,
                                                  const double* __restrict__ x, long long n,
                                                  double d) {
  for (long long i = blockIdx.x * (long long)kThreads + threadIdx.x; i < n;
       i += (long long)gridDim.x * kThreads)
    out[i] = x[i] / d;
}
__global__ void __launch_bounds__(kThreads) k_sub(double* __restrict__ r,
                                                  const double* __restrict__ f,
                                                  const double* __restrict__ w, long long n) {
  for (long long i = blockIdx.x * (long long)kThreads + threadIdx.x; i < n;
       i += (long long)gridDim.x * kThreads)
    r[i] = f[i] - w[i];
}
__global__ void __launch_bounds__(kThreads) k_nonfinite(const double* __restrict__ x,
                                                        long long n, int* flag) {
  bool bad = false;
  for (long long i = blockIdx.x * (long long)kThreads + threadIdx.x; i < n;
       i += (long long)gridDim.x * kThreads)
    bad |= !isfinite(x[i]);
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
}

// FP64 pipe roofline probe: 8 independent DFMA chains per thread, no memory.
__global__ void __launch_bounds__(256) k_dfma_peak(int iters, double a, double* out) {
  double x0 = threadIdx.x * 1e-9, x1 = x0 + 1e-3, x2 = x0 + 2e-3, x3 = x0 + 3e-3;
  double x4 = x0 + 4e-3, x5 = x0 + 5e-3, x6 = x0 + 6e-3, x7 = x0 + 7e-3;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      x0 = fma(x0, a, 1e-7); x1 = fma(x1, a, 1e-7); x2 = fma(x2, a, 1e-7); x3 = fma(x3, a, 1e-7);
      x4 = fma(x4, a, 1e-7); x5 = fma(x5, a, 1e-7); x6 = fma(x6, a, 1e-7); x7 = fma(x7, a, 1e-7);
    }
  }
  const double s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  if (s == 12345.678) out[0] = s;  // keeps the chains live
}

// One Arnoldi step's modified Gram-Schmidt in a single cooperative launch:
// for i = 0..j: h_i = <w, V_i> (fixed-order grid reduction, every CTA forms
// the same total), w -= h_i V_i; then h_{j+1} = ||w||.  Each thread owns a
// fixed slice of w, so only the reductions need the grid barrier (one per
// projection, partials double-buffered).  Also flags non-finite w.
constexpr int kMgsThreads = 256;
__global__ void __launch_bounds__(kMgsThreads) k_mgs(const double* __restrict__ V, double* w,
                                                     long long n, long long ld, int j,
                                                     double* __restrict__ partial,
                                                     double* __restrict__ h, int* flag,
                                                     double* __restrict__ vnext) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double red[kMgsThreads / 32];
  __shared__ double total_sh;
  const long long stride = (long long)gridDim.x * kMgsThreads;
  const long long t0 = blockIdx.x * (long long)kMgsThreads + threadIdx.x;
  auto block_sum = [&](double v) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    double t = 0.0;
    if (threadIdx.x == 0)
      for (int k = 0; k < kMgsThreads / 32; ++k) t += red[k];
    __syncthreads();
    return t;  // valid in thread 0
  };
  auto grid_total = [&](int buf) {
    // every CTA sums the partials in the same order -> identical totals
    if (threadIdx.x == 0) {
      double t = 0.0;
      const double* pp = partial + (size_t)buf * gridDim.x;
      for (unsigned b = 0; b < gridDim.x; ++b) t += pp[b];
      total_sh = t;
    }
    __syncthreads();
    return total_sh;
  };
  bool bad = false;
  for (long long k = t0; k < n; k += stride) bad |= !isfinite(w[k]);
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
  for (int i = 0; i <= j + 1; ++i) {
    const double* Vi = V + (size_t)i * ld;
    double acc = 0.0;
    if (i <= j)
      for (long long k = t0; k < n; k += stride) acc = fma(w[k], Vi[k], acc);
    else
      for (long long k = t0; k < n; k += stride) acc = fma(w[k], w[k], acc);
    const double bs = block_sum(acc);
    if (threadIdx.x == 0) partial[(size_t)(i & 1) * gridDim.x + blockIdx.x] = bs;
    grid.sync();
    const double hi = grid_total(i & 1);
    if (i <= j) {
      if (blockIdx.x == 0 && threadIdx.x == 0) h[i] = hi;
      for (long long k = t0; k < n; k += stride) w[k] = fma(-hi, Vi[k], w[k]);
    } else {
      const double hn = sqrt(hi);
      if (blockIdx.x == 0 && threadIdx.x == 0) h[j + 1] = hn;
      if (vnext)  // next basis vector v_{j+1} = w / h_{j+1,j} (own slice)
        for (long long k = t0; k < n; k += stride) vnext[k] = w[k] / hn;
    }
  }
}

// Small vectors (N <= 8 * 1024 * 16): the same MGS in ONE thread-block
// cluster of 8 CTAs x 1024 threads.  w lives in registers (E elements per
// thread); each projection's reduction crosses the cluster through distributed
// shared memory with one cluster barrier (partials double-buffered), so a
// projection costs ~1 us instead of a grid-wide barrier.
constexpr int kClusterCtas = 8;
template <int E>
__global__ void __cluster_dims__(kClusterCtas, 1, 1) __launch_bounds__(1024)
    k_mgs_cluster(const double* __restrict__ V, double* w, int n, long long ld, int j,
                  double* __restrict__ h, int* flag, double* __restrict__ vnext) {
  cg::cluster_group cl = cg::this_cluster();
  __shared__ double red[32];
  __shared__ double slots[2][kClusterCtas];  // [buffer][source CTA]: pushed by the peers
  __shared__ double bcast;
  constexpr int T = kClusterCtas * 1024;
  const unsigned rank = cl.block_rank();
  const int tid = (int)rank * 1024 + threadIdx.x;
  double wr[E];
  bool bad = false;
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int k = tid + e * T;
    wr[e] = k < n ? w[k] : 0.0;
    bad |= k < n && !isfinite(wr[e]);
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
  cl.sync();  // every CTA of the cluster is running before the first remote store
  for (int i = 0; i <= j + 1; ++i) {
    const double* Vi = V + (size_t)i * ld;
    constexpr bool kKeep = E <= 8;  // V_i's slice stays in registers for the update (E = 16: reloaded)
    double vi[kKeep ? E : 1];
    double acc = 0.0;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int k = tid + e * T;
      const double v = (k < n && i <= j) ? Vi[k] : 0.0;
      if (kKeep) vi[e] = v;
      if (k < n) acc = fma(wr[e], i <= j ? v : wr[e], acc);
    }
    // fixed-order tree reductions (warp, CTA, cluster): every CTA forms the
    // same total.  The CTA's sum is PUSHED into every peer's slots (remote
    // stores ahead of the cluster barrier), so after the barrier each CTA
    // reads its own shared memory only.
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x < 32) {
      double t = red[threadIdx.x];
      for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
      if (threadIdx.x < kClusterCtas)
        *cl.map_shared_rank(&slots[i & 1][rank], threadIdx.x) = t;
    }
    cl.sync();
    if (threadIdx.x < 32) {
      double t = threadIdx.x < kClusterCtas ? slots[i & 1][threadIdx.x] : 0.0;
      for (int o = kClusterCtas / 2; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
      if (threadIdx.x == 0) bcast = t;
    }
    __syncthreads();
    const double tot = bcast;
    if (i <= j) {
      if (tid == 0) h[i] = tot;
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int k = tid + e * T;
        if (k < n) wr[e] = fma(-tot, kKeep ? vi[e] : Vi[k], wr[e]);
      }
    } else {
      const double hn = sqrt(tot);
      if (tid == 0) h[j + 1] = hn;
      if (vnext) {  // next basis vector v_{j+1} = w / h_{j+1,j}
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const int k = tid + e * T;
          if (k < n) wr[e] = wr[e] / hn;
        }
      }
    }
  }
  double* out = vnext ? vnext : w;
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int k = tid + e * T;
    if (k < n) out[k] = wr[e];
  }
  cl.sync();  // keep every CTA's shared memory alive until all remote stores have landed
}

inline unsigned grid_for(long long n) {
  long long b = (n + kThreads * 4 - 1) / (kThreads * 4);
  return (unsigned)(b < 1 ? 1 : (b > 1184 ? 1184 : b));
}

}  // namespace

int dot_parts(long long n) { return (int)grid_for(n); }

double measure_dfma_peak(int iters, float* ms_out) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const unsigned grid = (unsigned)sms * 8;  // 8 x 256 threads resident per SM
  double* d = nullptr;
  cudaMalloc(&d, sizeof(double));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k_dfma_peak<<<grid, 256>>>(iters / 4 + 1, 0.999999, d);  // warm-up / clocks up
  cudaEventRecord(e0);
  k_dfma_peak<<<grid, 256>>>(iters, 0.999999, d);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(d);
  if (ms_out) *ms_out = ms;
  const double flops = (double)grid * 256 * iters * 16 * 8 * 2;
  return flops / (ms * 1e-3) / 1e12;
}

// SplitMix64 counter form of random_vector (reference.cpp:94-108): the i-th
// output uses state seed + (i + 1) * gamma.
__global__ void k_random_vector(double* __restrict__ out, long long n, unsigned long long seed) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    unsigned long long z = seed + (unsigned long long)(i + 1) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    out[i] = 2.0 * ((double)(z >> 11) * 0x1.0p-53) - 1.0;
  }
}
void launch_random_vector(double* out, long long n, unsigned long long seed, cudaStream_t s) {
  k_random_vector<<<grid_for(n), kThreads, 0, s>>>(out, n, seed);
}

int mgs_grid(long long n) {
  static int max_blocks = 0;
  if (!max_blocks) {
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_mgs, kMgsThreads, 0);
    max_blocks = sms * (per_sm > 2 ? 2 : per_sm);
  }
  constexpr long long per = 4;  // elements per thread
  const long long want = (n + kMgsThreads * per - 1) / (kMgsThreads * per);
  return (int)(want < 1 ? 1 : (want > max_blocks ? max_blocks : want));
}

cudaError_t launch_mgs(const double* V, double* w, long long n, long long ld, int j,
                       double* partial, int nparts, double* h, int* flag, double* vnext,
                       cudaStream_t s) {
  constexpr long long T = kClusterCtas * 1024;
  if (n <= 16 * T) {
    const int ni = (int)n;
    const dim3 g(kClusterCtas), b(1024);
    if (n <= T) k_mgs_cluster<1><<<g, b, 0, s>>>(V, w, ni, ld, j, h, flag, vnext);
    else if (n <= 2 * T) k_mgs_cluster<2><<<g, b, 0, s>>>(V, w, ni, ld, j, h, flag, vnext);
    else if (n <= 4 * T) k_mgs_cluster<4><<<g, b, 0, s>>>(V, w, ni, ld, j, h, flag, vnext);
    else if (n <= 8 * T) k_mgs_cluster<8><<<g, b, 0, s>>>(V, w, ni, ld, j, h, flag, vnext);
    else k_mgs_cluster<16><<<g, b, 0, s>>>(V, w, ni, ld, j, h, flag, vnext);
    return cudaGetLastError();
  }
  void* args[] = {(void*)&V, (void*)&w, (void*)&n, (void*)&ld, (void*)&j,
                  (void*)&partial, (void*)&h, (void*)&flag, (void*)&vnext};
  return cudaLaunchCooperativeKernel((const void*)k_mgs, dim3(nparts), dim3(kMgsThreads), args, 0,
                                     s);
}

void launch_dot(const double* a, const double* b, long long n, double* partial, int nparts,
                double* out, int take_sqrt, cudaStream_t s) {
  k_dot_partial<<<nparts, kThreads, 0, s>>>(a, b, n, partial);
  k_dot_final<<<1, kThreads, 0, s>>>(partial, nparts, out, take_sqrt);
}
void launch_axpy_dev(double* y, const double* x, long long n, const double* alpha_dev,
                     double sign, cudaStream_t s) {
  k_axpy_dev<<<grid_for(n), kThreads, 0, s>>>(y, x, n, alpha_dev, sign);
}
void launch_axpy(double* y, const double* x, long long n, double alpha, cudaStream_t s) {
  k_axpy<<<grid_for(n), kThreads, 0, s>>>(y, x, n, alpha);
}
void launch_div(double* out, const double* x, long long n, double d, cudaStream_t s) {
  k_div<<<grid_for(n), kThreads, 0, s>>>(out, x, n, d);
}
void launch_sub(double* r, const double* f, const double* w, long long n, cudaStream_t s) {
  k_sub<<<grid_for(n), kThreads, 0, s>>>(r, f, w, n);
}
void launch_nonfinite(const double* x, long long n, int* flag, cudaStream_t s) {
  k_nonfinite<<<grid_for(n), kThreads, 0, s>>>(x, n, flag);
}

}  // namespace imqk
