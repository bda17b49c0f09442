// FP64 tensor-pipe (DMMA) peak probe: the roofline denominator for the
// FP64-bound kernels (MEASURED_PEAKS.json carries only bf16 and HBM).
#include "common.cuh"
#include "sweep.cuh"

namespace vb {

__global__ void dmma_peak_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1},{%2},{%3},{%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1])
                   : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 1.2345e300) out[0] = s;
}

int probe_fp64_peak(double* tflops, cudaStream_t stream) {
  int dev = 0, nsm = 0;
  VB_CUDA(cudaGetDevice(&dev));
  VB_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  double* d = nullptr;
  VB_CUDA(cudaMalloc(&d, sizeof(double)));
  cudaEvent_t e0, e1;
  VB_CUDA(cudaEventCreate(&e0));
  VB_CUDA(cudaEventCreate(&e1));
  const int warps = 8, iters = 20000;
  dmma_peak_kernel<<<nsm * 2, 32 * warps, 0, stream>>>(d, 200);
  VB_LAUNCHED("dmma_peak_kernel");
  float best = 1e30f;
  for (int rep = 0; rep < 3; ++rep) {
    VB_CUDA(cudaEventRecord(e0, stream));
    dmma_peak_kernel<<<nsm * 2, 32 * warps, 0, stream>>>(d, iters);
    VB_LAUNCHED("dmma_peak_kernel");
    VB_CUDA(cudaEventRecord(e1, stream));
    VB_CUDA(cudaEventSynchronize(e1));
    float ms = 0;
    VB_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    if (ms < best) best = ms;
  }
  *tflops = (double)nsm * 2 * warps * iters * 8 * 512 / (best * 1e-3) / 1e12;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(d);
  return 0;
}

}  // namespace vb
