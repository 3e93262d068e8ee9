// FP64 tensor-core (DMMA m8n8k4) throughput vs the DFMA pipe on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void kdmma(double* o, int iters) {
  double a = threadIdx.x * 1e-9, b = 1.0 + threadIdx.x * 1e-12;
  double c[4][2] = {};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 4; ++k)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[k][0]), "+d"(c[k][1]) : "d"(a), "d"(b));
  }
  double s = 0; for (int k = 0; k < 4; ++k) s += c[k][0] + c[k][1];
  if (s == 1.2345) o[0] = s;
}
__global__ void kmix(double* o, int iters) {  // DMMA and DFMA interleaved
  double a = threadIdx.x * 1e-9, b = 1.0 + threadIdx.x * 1e-12;
  double c[2][2] = {}, x[8];
  for (int i = 0; i < 8; ++i) x[i] = i * 1e-3;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 2; ++k)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[k][0]), "+d"(c[k][1]) : "d"(a), "d"(b));
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fma(x[i], b, 1e-7);
  }
  double s = 0; for (int k = 0; k < 2; ++k) s += c[k][0] + c[k][1];
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 1.2345) o[0] = s;
}
int main() {
  double* d; cudaMalloc(&d, 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1); float ms;
  const int it = 4096, grid = sms * 8;
  kdmma<<<grid, 256>>>(d, it);
  cudaEventRecord(e0); kdmma<<<grid, 256>>>(d, it); cudaEventRecord(e1); cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  double fl = (double)grid * 8 /*warps*/ * it * 4 * 512;
  printf("DMMA m8n8k4: %.2f TFLOP/s\n", fl / (ms * 1e-3) / 1e12);
  kmix<<<grid, 256>>>(d, it);
  cudaEventRecord(e0); kmix<<<grid, 256>>>(d, it); cudaEventRecord(e1); cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  double fl2 = (double)grid * 8 * it * 2 * 512 + (double)grid * 256 * it * 8 * 2;
  printf("DMMA+DFMA mix: %.2f TFLOP/s total (%.3f ms)\n", fl2 / (ms * 1e-3) / 1e12, ms);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
