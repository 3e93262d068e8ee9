// Microbenchmark: Horner-style DFMA streams (R points per lane, one LDS.128
// per 2R DFMA, or coefficients in registers) at controlled occupancy
// (warps per SMSP), to find the FP64-pipe ceiling of the far kernel's shape.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/occupancy_probe tools/occupancy_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
#define IT 4096
template <int R, bool LDS>
__global__ void __launch_bounds__(128) kH(double* o, double a) {
  __shared__ double2 c[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) c[i] = make_double2(1e-3 * i, 2e-3 * i);
  __syncthreads();
  double q[R], g[R], h[R];
  for (int p = 0; p < R; ++p) { q[p] = a + (threadIdx.x + p) * 1e-12; g[p] = h[p] = 0; }
  double c0 = a * 1e-3, c1 = a * 2e-3;
  for (int it = 0; it < IT / 8; ++it)
#pragma unroll
    for (int k = 0; k < 64; ++k) {
      double2 cc = LDS ? c[(k + it) & 255] : make_double2(c0 + k, c1 - k);
#pragma unroll
      for (int p = 0; p < R; ++p) { g[p] = fma(g[p], q[p], cc.x); h[p] = fma(h[p], q[p], cc.y); }
    }
  double s = 0; for (int p = 0; p < R; ++p) s += g[p] + h[p];
  if (s == 1.2345) o[0] = s;
}
int main() {
  double* d; cudaMalloc(&d, 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto run = [&](const char* name, void (*k)(double*, double), int R, int warps_per_sm) {
    const int blocks = sms * warps_per_sm / 4;  // 4-warp CTAs
    k<<<blocks, 128>>>(d, 0.9999999);
    cudaEventRecord(e0);
    k<<<blocks, 128>>>(d, 0.9999999);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double fl = (double)blocks * 128 * (IT / 8) * 64.0 * 2 * R * 2;
    printf("%-22s warps/SM %2d: %.3f ms %.2f TFLOP/s\n", name, warps_per_sm, ms, fl / (ms * 1e-3) / 1e12);
  };
  for (int w : {4, 8, 12, 16, 32}) {
    run("lds128 R=4", kH<4, true>, 4, w);
    run("lds128 R=8", kH<8, true>, 8, w);
    run("regs   R=8", kH<8, false>, 8, w);
  }
  run("lds128 R=12", kH<12, true>, 12, 8);
  run("lds128 R=16", kH<16, true>, 16, 8);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
