// Fast-diagonalisation (FDM) building blocks for the full-order solver on
// structured hex27 boxes: the box operator
//   A(w) = Mz(x)My(x)Ax + Mz(x)Ay(x)Mx + Az(x)My(x)Mx + sigma Mz(x)My(x)Mx
// (A_d = K_d/rho + i w sum_walls e e^T / Z, sigma = -w^2/(rho c^2)) is a
// Kronecker sum, so with per-direction generalised eigenvectors
// V_d^T A_d V_d = Lambda_d, V_d^T M_d V_d = I:
//   A^-1 = V (Lz (+) Ly (+) Lx + sigma)^-1 V^T,   V = Vz (x) Vy (x) Vx.
// Replaces scipy splu at cfg3 size (n = 376,431), where the CPU oracle cannot
// factor at all (SURVEY §0 finding 7).
#include "common.cuh"
#include "mma.cuh"
#include "sweep.cuh"

namespace vb {

// Y = S applied along `axis` (0 = x fastest, 1 = y, 2 = z) of X with shape
// (n2, n1, n0) x nrhs (RHS fastest): Y[.., a, ..] = sum_l S[a, l] X[.., l, ..].
__global__ void axis_apply_kernel(int n2, int n1, int n0, int nrhs, int axis, const z_t* __restrict__ S,
                                  const z_t* __restrict__ X, z_t* __restrict__ Y) {
  const int64_t total = (int64_t)n2 * n1 * n0 * nrhs;
  const int nd = axis == 0 ? n0 : (axis == 1 ? n1 : n2);
  const int64_t stride = (axis == 0 ? 1 : (axis == 1 ? (int64_t)n0 : (int64_t)n0 * n1)) * nrhs;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t node = e / nrhs;
    const int q = (int)(e - node * nrhs);
    const int i = (int)(node % n0), j = (int)((node / n0) % n1), k = (int)(node / ((int64_t)n0 * n1));
    const int a = axis == 0 ? i : (axis == 1 ? j : k);
    const int64_t base = e - (int64_t)a * stride;  // element with index 0 along the axis
    const z_t* srow = S + (int64_t)a * nd;
    z_t acc = zmake(0.0, 0.0);
    for (int l = 0; l < nd; ++l) acc = zfma(acc, __ldg(srow + l), __ldg(X + base + (int64_t)l * stride));
    Y[e] = acc;
    (void)q;
  }
}

// X[k, j, i, q] /= (lz[k] + ly[j] + lx[i] + sigma)
__global__ void fdm_diag_kernel(int n2, int n1, int n0, int nrhs, const z_t* __restrict__ lz,
                                const z_t* __restrict__ ly, const z_t* __restrict__ lx, z_t sigma,
                                z_t* __restrict__ X) {
  const int64_t total = (int64_t)n2 * n1 * n0 * nrhs;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t node = e / nrhs;
    const int i = (int)(node % n0), j = (int)((node / n0) % n1), k = (int)(node / ((int64_t)n0 * n1));
    const z_t d = zadd(zadd(lz[k], ly[j]), zadd(lx[i], sigma));
    X[e] = zmul(X[e], zrecip(d));
  }
}

static unsigned grid_for(int64_t total) {
  int64_t g = (total + 255) / 256;
  return (unsigned)(g < 148 * 32 ? g : 148 * 32);
}

int axis_apply(int n2, int n1, int n0, int nrhs, int axis, const z_t* S, const z_t* X, z_t* Y, cudaStream_t st) {
  VB_CHECK_ARG(axis >= 0 && axis <= 2 && n0 > 0 && n1 > 0 && n2 > 0 && nrhs > 0, "vb_axis_apply: bad sizes");
  VB_CHECK_ARG(X != Y, "vb_axis_apply: X and Y must not alias");
  const int64_t total = (int64_t)n2 * n1 * n0 * nrhs;
  axis_apply_kernel<<<grid_for(total), 256, 0, st>>>(n2, n1, n0, nrhs, axis, S, X, Y);
  VB_LAUNCHED("axis_apply_kernel");
  return 0;
}

int fdm_diag(int n2, int n1, int n0, int nrhs, const z_t* lz, const z_t* ly, const z_t* lx, z_t sigma, z_t* X,
             cudaStream_t st) {
  const int64_t total = (int64_t)n2 * n1 * n0 * nrhs;
  fdm_diag_kernel<<<grid_for(total), 256, 0, st>>>(n2, n1, n0, nrhs, lz, ly, lx, sigma, X);
  VB_LAUNCHED("fdm_diag_kernel");
  return 0;
}

// ------------------------------------------- tensor-core FDM solve ----
// X = A^-1 B in one call.  Inside, the RHS-slowest layout (nrhs, n2, n1, n0)
// turns every direction transform into DMMA GEMMs with >= 51-wide operands:
//   x: Y (nrhs n2 n1 x n0) = X S_x^T                      one GEMM
//   y: Y_(q,k) (n1 x n0)   = S_y X_(q,k)                  nrhs n2 batched GEMMs
//   z: Y_q (n2 x n1 n0)    = S_z X_q                      nrhs batched GEMMs
// (S^T of VT_d is V_d: the eigenvectors are complex-symmetric normalised), so
// the 1-D transforms run at tensor-core rate instead of re-reading X from
// L2 once per 1-D coefficient (axis_apply_kernel).  B (n x nrhs, RHS fastest)
// is transposed in and the result transposed out through 32 x 32 tiles.
using GemmF = blk::Gemm<64, 32, 4, 2, 3, blk::EPI_SET, 16, true>;  // 3M products

__global__ void __launch_bounds__(blk::NT) fdm_gemm_kernel(int m, int n, int k, const z_t* A, int lda, int64_t sA,
                                                           const z_t* B, int ldb, int64_t sB, z_t* C, int ldc,
                                                           int64_t sC) {
  extern __shared__ double2 fdm_smem[];
  const int64_t b = blockIdx.y;
  GemmF::run(C + b * sC, ldc, A + b * sA, lda, B + b * sB, ldb, m, n, k, fdm_smem, zmake(1.0, 0.0),
             zmake(0.0, 0.0), blockIdx.x, gridDim.x);
}

// out (cols x rows, ld ldo) = in (rows x cols, ld ldi)^T
__global__ void __launch_bounds__(256) ztranspose_kernel(int rows, int cols, const z_t* __restrict__ in, int64_t ldi,
                                                         z_t* __restrict__ out, int64_t ldo) {
  __shared__ z_t t[32][33];
  const int ntr = (rows + 31) / 32;  // 1-D grid over 32 x 32 tiles
  const int64_t r0 = (int64_t)(blockIdx.x % ntr) * 32;
  const int c0 = (int)(blockIdx.x / ntr) * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  for (int y = ty; y < 32; y += 8)
    if (r0 + y < rows && c0 + tx < cols) t[y][tx] = in[(r0 + y) * ldi + c0 + tx];
  __syncthreads();
  for (int y = ty; y < 32; y += 8)
    if (c0 + y < cols && r0 + tx < rows) out[(int64_t)(c0 + y) * ldo + r0 + tx] = t[tx][y];
}

// X[q, k, j, i] /= (lz[k] + ly[j] + lx[i] + sigma)   (RHS-slowest layout)
__global__ void fdm_diag_rs_kernel(int n2, int n1, int n0, int nrhs, const z_t* __restrict__ lz,
                                   const z_t* __restrict__ ly, const z_t* __restrict__ lx, z_t sigma,
                                   z_t* __restrict__ X) {
  const int64_t nn = (int64_t)n2 * n1 * n0, total = nn * nrhs;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t node = e % nn;
    const int i = (int)(node % n0), j = (int)((node / n0) % n1), k = (int)(node / ((int64_t)n0 * n1));
    const z_t d = zadd(zadd(lz[k], ly[j]), zadd(lx[i], sigma));
    X[e] = zmul(X[e], zrecip(d));
  }
}

static int fdm_gemm(int m, int n, int k, const z_t* A, int lda, int64_t sA, const z_t* B, int ldb, int64_t sB,
                    z_t* C, int ldc, int64_t sC, int batch, cudaStream_t st) {
  const int ntiles = ((m + 63) / 64) * ((n + 31) / 32);
  int gx = ntiles;
  if (batch == 1 && gx > 2 * 148) gx = 2 * 148;  // persistent over the tiles of one big GEMM
  VB_CUDA(cudaFuncSetAttribute(fdm_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)GemmF::SMEM));
  for (int b0 = 0; b0 < batch; b0 += 65535) {  // grid.y limit
    const int nb = batch - b0 < 65535 ? batch - b0 : 65535;
    fdm_gemm_kernel<<<dim3((unsigned)gx, (unsigned)nb), blk::NT, GemmF::SMEM, st>>>(
        m, n, k, A + b0 * sA, lda, sA, B + b0 * sB, ldb, sB, C + b0 * sC, ldc, sC);
    VB_LAUNCHED("fdm_gemm_kernel");
  }
  return 0;
}

size_t fdm_solve_workspace_bytes(int n2, int n1, int n0, int nrhs) {
  return 2 * (size_t)n2 * n1 * n0 * nrhs * sizeof(z_t);
}

int fdm_solve(int n2, int n1, int n0, int nrhs, const z_t* const V[3], const z_t* const VT[3], const z_t* lx,
              const z_t* ly, const z_t* lz, z_t sigma, const z_t* B, int64_t ldb, z_t* X, int64_t ldx, void* work,
              size_t work_bytes, cudaStream_t st) {
  VB_CHECK_ARG(n0 > 0 && n1 > 0 && n2 > 0 && nrhs > 0 && B && X, "vb_fdm_solve: bad arguments");
  VB_CHECK_ARG(work && work_bytes >= fdm_solve_workspace_bytes(n2, n1, n0, nrhs), "vb_fdm_solve: workspace too small");
  const int64_t nn = (int64_t)n2 * n1 * n0;
  VB_CHECK_ARG(nn * nrhs / n0 < (int64_t)1 << 31, "vb_fdm_solve: problem too large");
  z_t* W1 = (z_t*)work;
  z_t* W2 = W1 + nn * nrhs;
  const int R = (int)(nn * nrhs / n0);
  {
    const unsigned g = (unsigned)(((nn + 31) / 32) * ((nrhs + 31) / 32));
    ztranspose_kernel<<<g, 256, 0, st>>>((int)nn, nrhs, B, ldb, W1, nn);  // W1 = B^T (nrhs x nn)
    VB_LAUNCHED("ztranspose_kernel");
  }
  const int64_t sy = (int64_t)n1 * n0, sz = nn;
  // forward: V^T along x, y, z
  if (fdm_gemm(R, n0, n0, W1, n0, 0, V[0], n0, 0, W2, n0, 0, 1, st)) return 1;                // x: W2 = W1 Vx
  if (fdm_gemm(n1, n0, n1, VT[1], n1, 0, W2, n0, sy, W1, n0, sy, nrhs * n2, st)) return 1;    // y
  if (fdm_gemm(n2, (int)sy, n2, VT[2], n2, 0, W1, (int)sy, sz, W2, (int)sy, sz, nrhs, st)) return 1;  // z
  fdm_diag_rs_kernel<<<grid_for(nn * nrhs), 256, 0, st>>>(n2, n1, n0, nrhs, lz, ly, lx, sigma, W2);
  VB_LAUNCHED("fdm_diag_rs_kernel");
  // backward: V along x, y, z
  if (fdm_gemm(R, n0, n0, W2, n0, 0, VT[0], n0, 0, W1, n0, 0, 1, st)) return 1;               // x: W1 = W2 VTx
  if (fdm_gemm(n1, n0, n1, V[1], n1, 0, W1, n0, sy, W2, n0, sy, nrhs * n2, st)) return 1;     // y
  if (fdm_gemm(n2, (int)sy, n2, V[2], n2, 0, W2, (int)sy, sz, W1, (int)sy, sz, nrhs, st)) return 1;   // z
  {
    const unsigned g = (unsigned)(((nn + 31) / 32) * ((nrhs + 31) / 32));
    ztranspose_kernel<<<g, 256, 0, st>>>(nrhs, (int)nn, W1, nn, X, ldx);  // X = W1^T (nn x nrhs)
    VB_LAUNCHED("ztranspose_kernel");
  }
  return 0;
}

}  // namespace vb
