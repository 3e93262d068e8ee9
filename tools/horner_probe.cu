// Microbenchmark of the far-field pair evaluation (complex Horner, M=16) with
// coefficients resident in shared memory: per-slot throughput vs points per
// lane R and unrolling of the outer m loop.  Development aid.
#include <cstdio>
#include <cuda_runtime.h>
#define M 16
__host__ __device__ constexpr int hz_top(int m) { return M - ((M - m) & 1); }
constexpr int KC = (M + 1) * (M + 2) / 2 - (M + 1) / 2;
__device__ __forceinline__ double rsq(double x) {
  double y; asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double e = fma(-x, y * y, 1.0); return fma(y * e, fma(0.375, e, 0.5), y);
}
template <int R, bool UNROLL_M>
__device__ __forceinline__ void eval(const double2* __restrict__ c, const double* dx, const double* dy, double t2, double* v) {
  double r[R], q[R], xr[R], xi[R], ar[R], ai[R];
#pragma unroll
  for (int p = 0; p < R; ++p) { r[p] = rsq(fma(dx[p], dx[p], fma(dy[p], dy[p], t2))); q[p] = r[p] * r[p];
    xr[p] = dx[p] * q[p]; xi[p] = -dy[p] * q[p]; ar[p] = c[0].x; ai[p] = c[0].y; }
  int o = 1;
  if constexpr (UNROLL_M) {
#pragma unroll
    for (int m = M - 1; m >= 1; --m) {
      double2 cc = c[o++]; double gr[R], gi[R];
#pragma unroll
      for (int p = 0; p < R; ++p) { gr[p] = cc.x; gi[p] = cc.y; }
#pragma unroll
      for (int k = hz_top(m) - 1; k >= m; --k) { cc = c[o++];
#pragma unroll
        for (int p = 0; p < R; ++p) { gr[p] = fma(gr[p], q[p], cc.x); gi[p] = fma(gi[p], q[p], cc.y); } }
#pragma unroll
      for (int p = 0; p < R; ++p) { const double nr = fma(ar[p], xr[p], fma(-ai[p], xi[p], gr[p]));
        const double ni = fma(ar[p], xi[p], fma(ai[p], xr[p], gi[p])); ar[p] = nr; ai[p] = ni; }
    }
  } else {
#pragma unroll 1
    for (int m = M - 1; m >= 1; --m) {
      double2 cc = c[o++]; double gr[R], gi[R];
#pragma unroll
      for (int p = 0; p < R; ++p) { gr[p] = cc.x; gi[p] = cc.y; }
      const int nk = hz_top(m) - m;
#pragma unroll 2
      for (int k = 0; k < nk; ++k) { cc = c[o + k];
#pragma unroll
        for (int p = 0; p < R; ++p) { gr[p] = fma(gr[p], q[p], cc.x); gi[p] = fma(gi[p], q[p], cc.y); } }
      o += nk;
#pragma unroll
      for (int p = 0; p < R; ++p) { const double nr = fma(ar[p], xr[p], fma(-ai[p], xi[p], gr[p]));
        const double ni = fma(ar[p], xi[p], fma(ai[p], xr[p], gi[p])); ar[p] = nr; ai[p] = ni; }
    }
  }
  const double* c0 = reinterpret_cast<const double*>(c + o);
  double g[R];
#pragma unroll
  for (int p = 0; p < R; ++p) g[p] = c0[0];
#pragma unroll
  for (int k = 1; k <= hz_top(0); ++k) { const double ck = c0[2 * k];
#pragma unroll
    for (int p = 0; p < R; ++p) g[p] = fma(g[p], q[p], ck); }
#pragma unroll
  for (int p = 0; p < R; ++p) v[p] = fma(ar[p], xr[p], fma(-ai[p], xi[p], g[p])) * r[p];
}
template <int R, bool U>
__global__ void __launch_bounds__(128) kern(int nsrc, double* out) {
  __shared__ double2 c[4][2][KC];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = lane; i < 2 * KC; i += 32) c[w][i / KC][i % KC] = make_double2(1e-3 * (i % 7 + 1), 2e-3 * (i % 5));
  __syncwarp();
  double x[R], y[R], acc[R];
#pragma unroll
  for (int p = 0; p < R; ++p) { x[p] = 0.3 + 1e-3 * (lane + 32 * p); y[p] = 0.2 + 1e-4 * blockIdx.x; acc[p] = 0; }
  for (int s = 0; s < nsrc; ++s) {
    const double zx = 1e-4 * s, zy = 2e-4 * s; double dx[R], dy[R], v[R];
#pragma unroll
    for (int p = 0; p < R; ++p) { dx[p] = x[p] - zx; dy[p] = y[p] - zy; }
    eval<R, U>(c[w][s & 1], dx, dy, 1e-4, v);
#pragma unroll
    for (int p = 0; p < R; ++p) acc[p] += v[p];
  }
  double t = 0;
#pragma unroll
  for (int p = 0; p < R; ++p) t += acc[p];
  if (t == 1.2345) out[0] = t;
}
template <int R, bool U>
void run(double* d) {
  const int nsrc = 200, grid = 148 * 40;
  kern<R, U><<<grid, 128>>>(nsrc, d);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0); kern<R, U><<<grid, 128>>>(nsrc, d); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  const double evals = (double)grid * 128 * R * nsrc;
  const double dfma = evals * (M * M + 4 * M);  // approx executed FP64 per eval
  cudaFuncAttributes a; cudaFuncGetAttributes(&a, kern<R, U>);
  printf("R=%d unrollM=%d regs=%3d  %.3f ms  %.2f ps/eval  ~%.0f%% of 18.4e12 DFMA/s\n", R, (int)U, a.numRegs, ms,
         ms * 1e9 / evals, 100.0 * dfma / (ms * 1e-3) / 18.39e12);
}
int main() {
  double* d; cudaMalloc(&d, 8);
  run<2, true>(d); run<4, true>(d); run<6, true>(d); run<8, true>(d);
  run<2, false>(d); run<4, false>(d); run<6, false>(d); run<8, false>(d); run<10, false>(d);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
