// Shared helpers for the vibro_b200 sm_100a kernels: complex128 arithmetic on
// double2 (interleaved re/im, the numpy/torch complex128 layout), error
// plumbing for the C-ABI, and warp reductions.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <string>

namespace vb {

typedef double2 z_t;  // complex128, interleaved

__host__ __device__ __forceinline__ z_t zmake(double re, double im) { return make_double2(re, im); }
__host__ __device__ __forceinline__ z_t zadd(z_t a, z_t b) { return zmake(a.x + b.x, a.y + b.y); }
__host__ __device__ __forceinline__ z_t zsub(z_t a, z_t b) { return zmake(a.x - b.x, a.y - b.y); }
__host__ __device__ __forceinline__ z_t zmul(z_t a, z_t b) {
  return zmake(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
// a*conj(b)
__host__ __device__ __forceinline__ z_t zmulc(z_t a, z_t b) {
  return zmake(a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y);
}
// conj(a)*b
__host__ __device__ __forceinline__ z_t zcmul(z_t a, z_t b) {
  return zmake(a.x * b.x + a.y * b.y, a.x * b.y - a.y * b.x);
}
// c - a*b
__host__ __device__ __forceinline__ z_t zfms(z_t c, z_t a, z_t b) {
  return zmake(c.x - a.x * b.x + a.y * b.y, c.y - a.x * b.y - a.y * b.x);
}
// c + a*b
__host__ __device__ __forceinline__ z_t zfma(z_t c, z_t a, z_t b) {
  return zmake(c.x + a.x * b.x - a.y * b.y, c.y + a.x * b.y + a.y * b.x);
}
__host__ __device__ __forceinline__ double zabs1(z_t a) { return fabs(a.x) + fabs(a.y); }  // LAPACK dcabs1
__host__ __device__ __forceinline__ double zabs2(z_t a) { return a.x * a.x + a.y * a.y; }
// 1/a with the scaling of Smith's algorithm (robust against overflow)
__host__ __device__ __forceinline__ z_t zrecip(z_t a) {
  if (fabs(a.x) >= fabs(a.y)) {
    double t = a.y / a.x, d = a.x + a.y * t;
    return zmake(1.0 / d, -t / d);
  } else {
    double t = a.x / a.y, d = a.y + a.x * t;
    return zmake(t / d, -1.0 / d);
  }
}

// izamax-style argmax across a warp: max |re|+|im|, lowest index on ties.
__device__ __forceinline__ void warp_argmax(double& v, int& idx) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    double ov = __shfl_xor_sync(0xffffffffu, v, o);
    int oi = __shfl_xor_sync(0xffffffffu, idx, o);
    if (ov > v || (ov == v && oi < idx)) { v = ov; idx = oi; }
  }
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Device-side index checks (build variant -DVB_DEBUG_CHECKS, tools/build_variant.py):
// compute-sanitizer is unavailable on the GPU pool, so the debug build traps
// on an out-of-range pivot / column index instead of corrupting memory.
#ifdef VB_DEBUG_CHECKS
#define VB_DCHECK(cond)                                                                   \
  do {                                                                                    \
    if (!(cond)) {                                                                        \
      printf("VB_DCHECK failed: %s at %s:%d (block %d thread %d)\n", #cond, __FILE__,     \
             __LINE__, (int)blockIdx.x, (int)threadIdx.x);                                \
      __trap();                                                                           \
    }                                                                                     \
  } while (0)
#else
#define VB_DCHECK(cond) \
  do {                  \
  } while (0)
#endif

void set_error(const std::string& msg);
int check_cuda(cudaError_t e, const char* where);
int check_launch(const char* where);

}  // namespace vb

#define VB_CHECK_ARG(cond, msg)          \
  do {                                   \
    if (!(cond)) {                       \
      ::vb::set_error(std::string(msg)); \
      return 1;                          \
    }                                    \
  } while (0)

#define VB_CUDA(call)                                      \
  do {                                                     \
    int _rc = ::vb::check_cuda((call), #call);             \
    if (_rc) return _rc;                                   \
  } while (0)

#define VB_LAUNCHED(where)                   \
  do {                                       \
    int _rc = ::vb::check_launch(where);     \
    if (_rc) return _rc;                     \
  } while (0)
