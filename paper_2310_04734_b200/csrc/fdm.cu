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

}  // namespace vb
