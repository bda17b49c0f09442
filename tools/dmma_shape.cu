// Ceiling of the blocked-sweep GEMM inner loop shape on B200: each warp owns a
// 16 x 16 complex sub-tile (2 x 2 DMMA fragments, re/im accumulators), reads
// 2 A + 2 B complex fragments (LDS.128) per k-step of 4 and issues 16 DMMAs
// (4 real products per complex fragment pair).  No global traffic: measures
// the smem + DMMA issue ceiling for warps/CTA x CTAs/SM.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1},{%2},{%3},{%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
template <int FM, int FN>
__global__ void shape_loop(double* out, int iters) {
  extern __shared__ double2 sm[];
  double2* As = sm;             // 64 x 16 (+pad)
  double2* Bs = sm + 64 * 20;   // 16 x 32 (+pad)
  for (int i = threadIdx.x; i < 64 * 20 + 16 * 34; i += blockDim.x) sm[i] = make_double2(i * 1e-3, 1.0);
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int wm = warp % 4, wn = (warp / 4) % 2;
  double cr[FM][FN][2] = {}, ci[FM][FN][2] = {};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      double2 a[FM], b[FN];
#pragma unroll
      for (int i = 0; i < FM; ++i) a[i] = As[(wm * 16 + i * 8 + (lane >> 2)) * 20 + kk * 4 + (lane & 3)];
#pragma unroll
      for (int j = 0; j < FN; ++j) b[j] = Bs[(kk * 4 + (lane & 3)) * 34 + wn * 16 + j * 8 + (lane >> 2)];
#pragma unroll
      for (int j = 0; j < FN; ++j)
#pragma unroll
        for (int i = 0; i < FM; ++i) {
          dmma(cr[i][j][0], cr[i][j][1], a[i].x, b[j].x);
          dmma(cr[i][j][0], cr[i][j][1], a[i].y, -b[j].y);
          dmma(ci[i][j][0], ci[i][j][1], a[i].x, b[j].y);
          dmma(ci[i][j][0], ci[i][j][1], a[i].y, b[j].x);
        }
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < FM; ++i)
#pragma unroll
    for (int j = 0; j < FN; ++j) s += cr[i][j][0] + cr[i][j][1] + ci[i][j][0] + ci[i][j][1];
  if (s == 12345.0) out[0] = s;
}
template <int FM, int FN>
void run(double* d, int nsm, int warps, int bps) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 4000;
  size_t smem = (64 * 20 + 16 * 34) * 16;
  dim3 g(nsm * bps), b(32 * warps);
  shape_loop<FM, FN><<<g, b, smem>>>(d, 10); cudaDeviceSynchronize();
  cudaEventRecord(e0); shape_loop<FM, FN><<<g, b, smem>>>(d, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double fl = (double)g.x * warps * iters * 4 * FM * FN * 4 * 512;
  printf("FM=%d FN=%d warps/blk=%2d blk/sm=%d: %.2f TFLOP/s\n", FM, FN, warps, bps, fl / ms / 1e9);
}
int main() {
  double* d; cudaMalloc(&d, 8);
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  run<2, 2>(d, nsm, 8, 1); run<2, 2>(d, nsm, 8, 2); run<2, 2>(d, nsm, 8, 3); run<2, 2>(d, nsm, 16, 1);
  run<2, 2>(d, nsm, 16, 2); run<2, 2>(d, nsm, 4, 2); run<2, 2>(d, nsm, 4, 4);
  run<1, 2>(d, nsm, 8, 2); run<2, 4>(d, nsm, 8, 2); run<4, 2>(d, nsm, 8, 2); run<2, 4>(d, nsm, 8, 1);
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
