// Microbenchmark: DFMA throughput vs register-operand pattern on sm_100a.
// A: fma(x_i, a, imm)        (2 RF operands)
// B: fma(x_i, y_i, z)        (3 operands, z shared)
// C: fma(x_i, y_i, z_i)      (3 distinct operands)
// D: Horner from smem        g = fma(g, q, c[k]) (c via LDS.128, 2 points)
#include <cstdio>
#include <cuda_runtime.h>
#define IT 2048
__global__ void kA(double* o, double a) {
  double x[8];
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-9 + i;
  for (int it = 0; it < IT; ++it)
#pragma unroll
    for (int k = 0; k < 8; ++k)
#pragma unroll
      for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, 1e-7);
  double s = 0; for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 1.2345) o[0] = s;
}
__global__ void kB(double* o, double a) {
  double x[8], y[8];
  for (int i = 0; i < 8; ++i) { x[i] = threadIdx.x * 1e-9 + i; y[i] = a + i * 1e-12; }
  double z = a * 1e-7;
  for (int it = 0; it < IT; ++it)
#pragma unroll
    for (int k = 0; k < 8; ++k)
#pragma unroll
      for (int i = 0; i < 8; ++i) x[i] = fma(x[i], y[i], z);
  double s = 0; for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 1.2345) o[0] = s;
}
__global__ void kC(double* o, double a) {
  double x[8], y[8], z[8];
  for (int i = 0; i < 8; ++i) { x[i] = threadIdx.x * 1e-9 + i; y[i] = a + i * 1e-12; z[i] = 1e-7 * i; }
  for (int it = 0; it < IT; ++it)
#pragma unroll
    for (int k = 0; k < 8; ++k)
#pragma unroll
      for (int i = 0; i < 8; ++i) x[i] = fma(x[i], y[i], z[i]);
  double s = 0; for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 1.2345) o[0] = s;
}
__global__ void kD(double* o, double a) {
  __shared__ double2 c[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) c[i] = make_double2(1e-3 * i, 2e-3 * i);
  __syncthreads();
  double q0 = a + threadIdx.x * 1e-12, q1 = a - threadIdx.x * 1e-12;
  double g0 = 0, h0 = 0, g1 = 0, h1 = 0;
  for (int it = 0; it < IT / 4; ++it)
#pragma unroll
    for (int k = 0; k < 128; ++k) {
      double2 cc = c[(k + it) & 255];
      g0 = fma(g0, q0, cc.x); h0 = fma(h0, q0, cc.y);
      g1 = fma(g1, q1, cc.x); h1 = fma(h1, q1, cc.y);
    }
  double s = g0 + h0 + g1 + h1;
  if (s == 1.2345) o[0] = s;
}
template <int R>
__global__ void kE(double* o, double a) {  // Horner, R points, LDS.128 per 2R DFMA
  __shared__ double2 c[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) c[i] = make_double2(1e-3 * i, 2e-3 * i);
  __syncthreads();
  double q[R], g[R], h[R];
  for (int p = 0; p < R; ++p) { q[p] = a + (threadIdx.x + p) * 1e-12; g[p] = h[p] = 0; }
  for (int it = 0; it < IT / 4; ++it)
#pragma unroll
    for (int k = 0; k < 128; ++k) {
      double2 cc = c[(k + it) & 255];
#pragma unroll
      for (int p = 0; p < R; ++p) { g[p] = fma(g[p], q[p], cc.x); h[p] = fma(h[p], q[p], cc.y); }
    }
  double s = 0; for (int p = 0; p < R; ++p) s += g[p] + h[p];
  if (s == 1.2345) o[0] = s;
}
template <int R>
__global__ void kF(double* o, double a) {  // Horner, R points, coefficient from registers (no LDS)
  double q[R], g[R], h[R];
  for (int p = 0; p < R; ++p) { q[p] = a + (threadIdx.x + p) * 1e-12; g[p] = h[p] = 0; }
  double c0 = a * 1e-3, c1 = a * 2e-3;
  for (int it = 0; it < IT / 4; ++it)
#pragma unroll
    for (int k = 0; k < 128; ++k) {
#pragma unroll
      for (int p = 0; p < R; ++p) { g[p] = fma(g[p], q[p], c0); h[p] = fma(h[p], q[p], c1); }
    }
  double s = 0; for (int p = 0; p < R; ++p) s += g[p] + h[p];
  if (s == 1.2345) o[0] = s;
}
template <int R>
__global__ void kG(double* o, double a) {  // Horner, LDS.64 per R DFMA (real only)
  __shared__ double c[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) c[i] = 1e-3 * i;
  __syncthreads();
  double q[R], g[R];
  for (int p = 0; p < R; ++p) { q[p] = a + (threadIdx.x + p) * 1e-12; g[p] = 0; }
  for (int it = 0; it < IT / 4; ++it)
#pragma unroll
    for (int k = 0; k < 256; ++k) {
      double cc = c[(k + it) & 255];
#pragma unroll
      for (int p = 0; p < R; ++p) g[p] = fma(g[p], q[p], cc);
    }
  double s = 0; for (int p = 0; p < R; ++p) s += g[p];
  if (s == 1.2345) o[0] = s;
}
int main() {
  double* d; cudaMalloc(&d, 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto run = [&](const char* name, void (*k)(double*, double), double flops_per_thread) {
    k<<<sms * 8, 256>>>(d, 0.9999999);
    cudaEventRecord(e0);
    k<<<sms * 8, 256>>>(d, 0.9999999);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double tf = (double)sms * 8 * 256 * flops_per_thread / (ms * 1e-3) / 1e12;
    printf("%s %.3f ms %.2f TFLOP/s\n", name, ms, tf);
  };
  run("A fma(x,a,imm)     ", kA, IT * 64.0 * 2);
  run("B fma(x,y_i,z)     ", kB, IT * 64.0 * 2);
  run("C fma(x,y_i,z_i)   ", kC, IT * 64.0 * 2);
  run("D horner smem 2pts ", kD, (IT / 4) * 128.0 * 4 * 2);
  run("E horner lds128 R=2", kE<2>, (IT / 4) * 128.0 * 4 * 2);
  run("E horner lds128 R=3", kE<3>, (IT / 4) * 128.0 * 6 * 2);
  run("E horner lds128 R=4", kE<4>, (IT / 4) * 128.0 * 8 * 2);
  run("E horner lds128 R=6", kE<6>, (IT / 4) * 128.0 * 12 * 2);
  run("F horner regs R=1  ", kF<1>, (IT / 4) * 128.0 * 2 * 2);
  run("F horner regs R=2  ", kF<2>, (IT / 4) * 128.0 * 4 * 2);
  run("F horner regs R=4  ", kF<4>, (IT / 4) * 128.0 * 8 * 2);
  run("G horner lds64 R=2 ", kG<2>, (IT / 4) * 256.0 * 2 * 2);
  run("G horner lds64 R=4 ", kG<4>, (IT / 4) * 256.0 * 4 * 2);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
