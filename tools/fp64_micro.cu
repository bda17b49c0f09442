// FP64 peak microbenchmark on B200: DMMA (mma.sync m8n8k4 f64) vs DFMA.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dmma_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[8][2];
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1},{%2},{%3},{%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0; for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.0) out[0] = s;
}
__global__ void dfma_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[16];
  for (int i = 0; i < 16; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) c[i] = fma(a, c[i], b);
  }
  double s = 0; for (int i = 0; i < 16; ++i) s += c[i];
  if (s == 12345.0) out[0] = s;
}
int main() {
  double* d; cudaMalloc(&d, 8);
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int warps = 4; warps <= 16; warps *= 2) {
    for (int bps = 1; bps <= 2; ++bps) {
      int iters = 20000;
      dim3 g(nsm * bps), b(32 * warps);
      dmma_loop<<<g, b>>>(d, 100); cudaDeviceSynchronize();
      cudaEventRecord(e0); dmma_loop<<<g, b>>>(d, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double fl = (double)g.x * warps * iters * 8 * 512;
      printf("DMMA warps/blk=%d blk/sm=%d: %.2f TFLOP/s\n", warps, bps, fl / ms / 1e9);
      dfma_loop<<<g, b>>>(d, 100); cudaDeviceSynchronize();
      cudaEventRecord(e0); dfma_loop<<<g, b>>>(d, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      fl = (double)g.x * warps * 32 * iters * 16 * 2;
      printf("DFMA warps/blk=%d blk/sm=%d: %.2f TFLOP/s\n", warps, bps, fl / ms / 1e9);
    }
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
