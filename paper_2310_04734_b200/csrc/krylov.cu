// Batched classical Gram-Schmidt for the GPU GMRES (gmres.py), which replaces
// the reference's right-preconditioned GMRES with modified Gram-Schmidt
// (solvers.py:191-264) as the full-order solver of models without a direct
// factorisation (per-element wall impedances, general meshes).
//
// k right-hand sides run their own Arnoldi processes side by side.  Column c
// owns the basis V[:, c, 0:j] (layout: element (row, c, i) at
//   row * ldr + c * ldc + i), and one orthogonalisation pass is
//   H[c, i] = sum_row conj(V[row, c, i]) W[row, c]      (vb_batched_dots)
//   W[row, c] -= sum_i V[row, c, i] H[c, i]             (vb_batched_update)
// HBM-bound (each pass streams the k bases once): the dot kernel keeps one
// thread per (c, i) pair so a warp reads a contiguous run of a basis row, and
// reduces per-CTA partials in a fixed order in a second pass (deterministic).
#include "common.cuh"
#include "sweep.cuh"

namespace vb {

constexpr int KR_NT = 256;

// partial[cta][c * j + i] over the CTA's row range.  The k * j (column, basis
// vector) pairs are few (8 x 1..60), so the CTA's threads split into
// 256 / pairs row slots per pair: every thread streams a strided share of the
// rows (enough loads in flight to cover HBM latency), then the slots are
// summed in a fixed order in shared memory (deterministic).
__global__ void __launch_bounds__(KR_NT) batched_dots_partial(int64_t n, int k, int j, const z_t* __restrict__ V,
                                                              int64_t ldr, int64_t ldc, const z_t* __restrict__ W,
                                                              int64_t ldw, z_t* __restrict__ part, int64_t rows_per) {
  __shared__ z_t red[KR_NT];
  const int64_t r0 = (int64_t)blockIdx.x * rows_per;
  const int64_t r1 = min(n, r0 + rows_per);
  const int pairs = k * j;
  for (int pbase = 0; pbase < pairs; pbase += KR_NT) {
    const int np = min(KR_NT, pairs - pbase);
    const int nslot = KR_NT / np;           // row slots per pair
    const int p = pbase + threadIdx.x % np, slot = threadIdx.x / np;
    z_t acc = zmake(0.0, 0.0);
    if (slot < nslot) {
      const int c = p / j, i = p - c * j;
      const z_t* vp = V + c * ldc + i;
      const z_t* wp = W + c;
      for (int64_t row = r0 + slot; row < r1; row += nslot) {
        const z_t v = vp[row * ldr];
        acc = zfma(acc, zmake(v.x, -v.y), wp[row * ldw]);
      }
    }
    red[threadIdx.x] = acc;
    __syncthreads();
    if (threadIdx.x < np) {
      z_t s = zmake(0.0, 0.0);
      for (int q = 0; q < nslot; ++q) s = zadd(s, red[q * np + threadIdx.x]);  // fixed order
      part[(int64_t)blockIdx.x * pairs + pbase + threadIdx.x] = s;
    }
    __syncthreads();
  }
}

__global__ void batched_dots_reduce(int nparts, int pairs, const z_t* __restrict__ part, z_t* __restrict__ H) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= pairs) return;
  z_t acc = zmake(0.0, 0.0);
  for (int q = 0; q < nparts; ++q) acc = zadd(acc, part[(int64_t)q * pairs + p]);  // fixed order
  H[p] = acc;
}

__global__ void __launch_bounds__(KR_NT) batched_update(int64_t n, int k, int j, const z_t* __restrict__ V,
                                                        int64_t ldr, int64_t ldc, const z_t* __restrict__ H,
                                                        z_t* __restrict__ W, int64_t ldw) {
  extern __shared__ z_t hs[];  // k * j coefficients
  for (int p = threadIdx.x; p < k * j; p += KR_NT) hs[p] = H[p];
  __syncthreads();
  const int64_t total = n * k;
  for (int64_t e = (int64_t)blockIdx.x * KR_NT + threadIdx.x; e < total; e += (int64_t)gridDim.x * KR_NT) {
    const int64_t row = e / k;
    const int c = (int)(e - row * k);
    const z_t* v = V + row * ldr + c * ldc;
    z_t acc = W[row * ldw + c];
    for (int i = 0; i < j; ++i) acc = zfms(acc, v[i], hs[c * j + i]);
    W[row * ldw + c] = acc;
  }
}

static int kr_grid() {
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  return 4 * nsm;
}

size_t batched_dots_workspace_bytes(int k, int j) { return (size_t)kr_grid() * k * j * sizeof(z_t); }

int batched_dots(int64_t n, int k, int j, const z_t* V, int64_t ldr, int64_t ldc, const z_t* W, int64_t ldw, z_t* H,
                 void* work, size_t work_bytes, cudaStream_t st) {
  if (k <= 0 || j <= 0) return 0;
  VB_CHECK_ARG(work_bytes >= batched_dots_workspace_bytes(k, j), "vb_batched_dots: workspace too small");
  const int g = kr_grid();
  const int64_t rows_per = (n + g - 1) / g;
  batched_dots_partial<<<g, KR_NT, 0, st>>>(n, k, j, V, ldr, ldc, W, ldw, (z_t*)work, rows_per > 0 ? rows_per : 1);
  VB_LAUNCHED("batched_dots_partial");
  const int pairs = k * j;
  batched_dots_reduce<<<(pairs + 127) / 128, 128, 0, st>>>(g, pairs, (const z_t*)work, H);
  VB_LAUNCHED("batched_dots_reduce");
  return 0;
}

int batched_update(int64_t n, int k, int j, const z_t* V, int64_t ldr, int64_t ldc, const z_t* H, z_t* W,
                   int64_t ldw, cudaStream_t st) {
  if (k <= 0 || j <= 0 || n <= 0) return 0;
  const size_t smem = (size_t)k * j * sizeof(z_t);
  VB_CHECK_ARG(smem <= 48 * 1024, "vb_batched_update: k * j too large");
  const int64_t blocks = (n * k + KR_NT - 1) / KR_NT;
  const int g = (int)(blocks < kr_grid() ? blocks : kr_grid());
  batched_update<<<g, KR_NT, smem, st>>>(n, k, j, V, ldr, ldc, H, W, ldw);
  VB_LAUNCHED("batched_update");
  return 0;
}

}  // namespace vb
