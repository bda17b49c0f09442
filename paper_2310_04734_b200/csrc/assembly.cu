// FE primitives on the GPU (SURVEY §8a rows A1–A3):
//   shape.py:20-26, 56-65   quadratic Lagrange bases and Gauss rules (constant tables)
//   assembly.py:77-91       Helmholtz element integrals Kgrad_e, Mnn_e (hex27 here)
//   assembly.py:142-175     triplet stream (rows = repeat(dofs), cols = tile(dofs),
//                           elements in index order) -> canonical CSR, duplicates
//                           summed, explicit zeros kept.
//
// Pattern: a STABLE radix sort of the triplet keys row*n+col carrying the triplet
// index, so duplicates of one (row, col) stay in element order; the unique keys
// are the canonical pattern (sorted int32 column indices per row, bit-identical
// to scipy's coo -> csr -> sum_duplicates), and the sorted triplet indices are a
// gather map.  Values are then summed per CSR slot in element order by a
// gather kernel: no atomics, run-to-run bit-identical.
#include <cub/cub.cuh>

#include "common.cuh"
#include "sweep.cuh"

namespace vb {

// ---------------------------------------------------------------- tables ---
// 3-point Gauss-Legendre (shape.py:56-57 = numpy leggauss(3)), closed form.
// The element tables are indexed by lane-dependent (gauss point, node) pairs, so
// they live in global memory (L1-cached) rather than __constant__ (which
// serialises divergent addresses).
__constant__ double c_gx[3];
__constant__ double c_gw[3];
// hex27: N[g][i], dN/dxi[g][i][a]; local node i = a + 3b + 9c, Gauss point
// g = gx + 3 gy + 9 gz (x fastest, shape.py:60-65 generalised).
__device__ double c_hexN[27 * 27];
__device__ double c_hexdN[27 * 27 * 3];
__device__ double c_hexW[27];
// quad9 face (lexicographic a + 3b): N[g][i], dN/dxi[g][i][2], weights.
__device__ double c_qN[9 * 9];
__device__ double c_qdN[9 * 9 * 2];
__device__ double c_qW[9];
// quad9 at the 2x2 (reduced) rule, for the Reissner-Mindlin shear term
__device__ double c_rN[4 * 9];
__device__ double c_rdN[4 * 9 * 2];
__device__ double c_rW[4];

static void lag1d(double x, double* v) {  // shape.py:20-22
  v[0] = 0.5 * x * (x - 1.0);
  v[1] = 1.0 - x * x;
  v[2] = 0.5 * x * (x + 1.0);
}
static void dlag1d(double x, double* v) {  // shape.py:25-26
  v[0] = x - 0.5;
  v[1] = -2.0 * x;
  v[2] = x + 0.5;
}

static int init_tables() {
  static bool done = false;
  if (done) return 0;
  const double gx[3] = {-0.7745966692414834, 0.0, 0.7745966692414834};
  const double gw[3] = {0.5555555555555556, 0.8888888888888888, 0.5555555555555556};
  double hN[27 * 27], hdN[27 * 27 * 3], hW[27], qN[81], qdN[162], qW[9];
  for (int g = 0; g < 27; ++g) {
    const int g3[3] = {g % 3, (g / 3) % 3, g / 9};
    double L[3][3], D[3][3];
    for (int d = 0; d < 3; ++d) {
      lag1d(gx[g3[d]], L[d]);
      dlag1d(gx[g3[d]], D[d]);
    }
    hW[g] = gw[g3[0]] * gw[g3[1]] * gw[g3[2]];
    for (int i = 0; i < 27; ++i) {
      const int n3[3] = {i % 3, (i / 3) % 3, i / 9};
      hN[g * 27 + i] = L[0][n3[0]] * L[1][n3[1]] * L[2][n3[2]];
      for (int a = 0; a < 3; ++a) {
        double v = 1.0;
        for (int d = 0; d < 3; ++d) v *= (d == a ? D : L)[d][n3[d]];
        hdN[(g * 27 + i) * 3 + a] = v;
      }
    }
  }
  for (int g = 0; g < 9; ++g) {
    const int g2[2] = {g % 3, g / 3};
    double L[2][3], D[2][3];
    for (int d = 0; d < 2; ++d) {
      lag1d(gx[g2[d]], L[d]);
      dlag1d(gx[g2[d]], D[d]);
    }
    qW[g] = gw[g2[0]] * gw[g2[1]];
    for (int i = 0; i < 9; ++i) {
      const int n2[2] = {i % 3, i / 3};
      qN[g * 9 + i] = L[0][n2[0]] * L[1][n2[1]];
      qdN[(g * 9 + i) * 2 + 0] = D[0][n2[0]] * L[1][n2[1]];
      qdN[(g * 9 + i) * 2 + 1] = L[0][n2[0]] * D[1][n2[1]];
    }
  }
  double rN[36], rdN[72], rW[4];
  const double g2[2] = {-0.5773502691896258, 0.5773502691896258};
  for (int g = 0; g < 4; ++g) {
    double L[2][3], D[2][3];
    lag1d(g2[g % 2], L[0]);
    dlag1d(g2[g % 2], D[0]);
    lag1d(g2[g / 2], L[1]);
    dlag1d(g2[g / 2], D[1]);
    rW[g] = 1.0;
    for (int i = 0; i < 9; ++i) {
      const int n2[2] = {i % 3, i / 3};
      rN[g * 9 + i] = L[0][n2[0]] * L[1][n2[1]];
      rdN[(g * 9 + i) * 2 + 0] = D[0][n2[0]] * L[1][n2[1]];
      rdN[(g * 9 + i) * 2 + 1] = L[0][n2[0]] * D[1][n2[1]];
    }
  }
  VB_CUDA(cudaMemcpyToSymbol(c_rN, rN, sizeof(rN)));
  VB_CUDA(cudaMemcpyToSymbol(c_rdN, rdN, sizeof(rdN)));
  VB_CUDA(cudaMemcpyToSymbol(c_rW, rW, sizeof(rW)));
  VB_CUDA(cudaMemcpyToSymbol(c_gx, gx, sizeof(gx)));
  VB_CUDA(cudaMemcpyToSymbol(c_gw, gw, sizeof(gw)));
  VB_CUDA(cudaMemcpyToSymbol(c_hexN, hN, sizeof(hN)));
  VB_CUDA(cudaMemcpyToSymbol(c_hexdN, hdN, sizeof(hdN)));
  VB_CUDA(cudaMemcpyToSymbol(c_hexW, hW, sizeof(hW)));
  VB_CUDA(cudaMemcpyToSymbol(c_qN, qN, sizeof(qN)));
  VB_CUDA(cudaMemcpyToSymbol(c_qdN, qdN, sizeof(qdN)));
  VB_CUDA(cudaMemcpyToSymbol(c_qW, qW, sizeof(qW)));
  done = true;
  return 0;
}

// ------------------------------------------------------- element kernels ---
// One WARP per hex27 element (assembly.py:77-91): J = dshape^T X, detJ <= 0
// rejected, dN = dshape inv(J), then
//   Kgrad = D^T W D   with D[(g,b)][i] = dN_i/dx_b at Gauss point g (81 x 27),
//   Mnn   = N^T W N   with N[g][i]                                   (27 x 27),
// W = diag(w_g detJ_g), both as 27 x 27 (padded to 32 x 32) products on the FP64
// tensor cores: mma.sync.m8n8k4.f64, 4 x 4 fragments per warp, 21 (K) + 7 (M)
// k-steps.  The D fragments are formed on the fly from the reference-element
// gradients (shared table) and the per-point inverse Jacobians, so no element
// array of D is stored; W is applied to the A-side fragment.  The 27 x 27
// results are staged in shared memory and written with coalesced stores.
constexpr int EL_NT = 256;            // 8 warps = 8 elements in flight per CTA
constexpr int EL_WARPS = EL_NT / 32;

__device__ __forceinline__ void el_dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1},{%2},{%3},{%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

struct ElWarp {
  double X[27][3];
  double iJ[27][9];
  double wdet[28];  // [27] = 0 (padding point)
  double out[27 * 27];
};

__global__ void __launch_bounds__(EL_NT, 2) hex27_helmholtz_kernel(int n_elem, const double* __restrict__ xyz,
                                                                const int32_t* __restrict__ conn,
                                                                double* __restrict__ Ke,
                                                                double* __restrict__ Me,
                                                                int* __restrict__ bad, int chain) {
  extern __shared__ double el_smem[];
  double* sdN = el_smem;               // [27 g][27 i][3 a] reference gradients
  double* sN = sdN + 2187;             // [28 g][32 i] shape values, zero padded
  ElWarp* W = (ElWarp*)(sN + 28 * 32);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int q = tid; q < 2187; q += EL_NT) sdN[q] = c_hexdN[q];
  for (int q = tid; q < 28 * 32; q += EL_NT) {
    const int g = q >> 5, i = q & 31;
    sN[q] = (g < 27 && i < 27) ? c_hexN[g * 27 + i] : 0.0;
  }
  __syncthreads();
  ElWarp& w = W[warp];
  const int col = lane >> 2, kq = lane & 3;  // fragment column (A row / B col) and k offset
  for (int e = blockIdx.x * EL_WARPS + warp; e < n_elem; e += gridDim.x * EL_WARPS) {
    for (int q = lane; q < 81; q += 32) w.X[q / 3][q % 3] = xyz[(size_t)conn[(size_t)e * 27 + q / 3] * 3 + q % 3];
    __syncwarp();
    // J[g][a][b] = sum_i dN_i/dxi_a(g) X_i,b: 243 sums over the lanes
    double Jv[8];
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const int q = lane + 32 * t;
      double acc = 0.0;
      if (q < 243) {
        const int g = q / 9, a = (q % 9) / 3, b = q % 3;
        for (int i = 0; i < 27; ++i) acc += sdN[(g * 27 + i) * 3 + a] * w.X[i][b];
      }
      Jv[t] = acc;
    }
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const int q = lane + 32 * t;
      if (q < 243) w.iJ[q / 9][q % 9] = Jv[t];  // J first, inverted in place below
    }
    __syncwarp();
    if (lane < 27) {
      const int g = lane;
      double J[9];
#pragma unroll
      for (int t = 0; t < 9; ++t) J[t] = w.iJ[g][t];
      const double det = J[0] * (J[4] * J[8] - J[5] * J[7]) - J[1] * (J[3] * J[8] - J[5] * J[6]) +
                         J[2] * (J[3] * J[7] - J[4] * J[6]);
      if (!(det > 0.0)) atomicMin(bad, e);
      const double id = 1.0 / det;
      double* iJ = w.iJ[g];
      iJ[0] = (J[4] * J[8] - J[5] * J[7]) * id;
      iJ[1] = (J[2] * J[7] - J[1] * J[8]) * id;
      iJ[2] = (J[1] * J[5] - J[2] * J[4]) * id;
      iJ[3] = (J[5] * J[6] - J[3] * J[8]) * id;
      iJ[4] = (J[0] * J[8] - J[2] * J[6]) * id;
      iJ[5] = (J[2] * J[3] - J[0] * J[5]) * id;
      iJ[6] = (J[3] * J[7] - J[4] * J[6]) * id;
      iJ[7] = (J[1] * J[6] - J[0] * J[7]) * id;
      iJ[8] = (J[0] * J[4] - J[1] * J[3]) * id;
      if (chain) {  // chain rule dN inv(J)^T (cfg4 curved elements): store inv(J) transposed
        double tmp = iJ[1]; iJ[1] = iJ[3]; iJ[3] = tmp;
        tmp = iJ[2]; iJ[2] = iJ[6]; iJ[6] = tmp;
        tmp = iJ[5]; iJ[5] = iJ[7]; iJ[7] = tmp;
      }
      w.wdet[g] = __ldg(&c_hexW[g]) * det;
    } else if (lane == 27) {
      w.wdet[27] = 0.0;
    }
    __syncwarp();
    // ---- Kgrad = D^T W D, k = (g, b) = 0..80 padded to 84
    double acc[4][4][2];
#pragma unroll
    for (int I = 0; I < 4; ++I)
#pragma unroll
      for (int J = 0; J < 4; ++J) acc[I][J][0] = acc[I][J][1] = 0.0;
    for (int k0 = 0; k0 < 84; k0 += 4) {
      const int k = k0 + kq;
      const bool kin = k < 81;
      const int g = kin ? k / 3 : 0, b = k - 3 * (k / 3);
      const double i0 = w.iJ[g][b], i1 = w.iJ[g][3 + b], i2 = w.iJ[g][6 + b];
      const double wg = kin ? w.wdet[g] : 0.0;
      double d[4];
#pragma unroll
      for (int I = 0; I < 4; ++I) {
        const int i = 8 * I + col;
        double v = 0.0;
        if (i < 27) {
          const double* ds = sdN + (g * 27 + i) * 3;
          v = ds[0] * i0 + ds[1] * i1 + ds[2] * i2;  // dN = dshape inv(J)
        }
        d[I] = v;
      }
#pragma unroll
      for (int I = 0; I < 4; ++I) {
        const double a = wg * d[I];
#pragma unroll
        for (int J = 0; J < 4; ++J) el_dmma(acc[I][J][0], acc[I][J][1], a, d[J]);
      }
    }
#pragma unroll
    for (int I = 0; I < 4; ++I)
#pragma unroll
      for (int J = 0; J < 4; ++J)
#pragma unroll
        for (int v = 0; v < 2; ++v) {
          const int i = 8 * I + col, j = 8 * J + 2 * kq + v;
          if (i < 27 && j < 27) w.out[i * 27 + j] = acc[I][J][v];
        }
    __syncwarp();
    for (int q = lane; q < 729; q += 32) Ke[(size_t)e * 729 + q] = w.out[q];
    __syncwarp();
    // ---- Mnn = N^T W N, k = g = 0..26 padded to 28
#pragma unroll
    for (int I = 0; I < 4; ++I)
#pragma unroll
      for (int J = 0; J < 4; ++J) acc[I][J][0] = acc[I][J][1] = 0.0;
    for (int k0 = 0; k0 < 28; k0 += 4) {
      const int g = k0 + kq;
      const double wg = w.wdet[g];
      double nv[4];
#pragma unroll
      for (int I = 0; I < 4; ++I) nv[I] = sN[g * 32 + 8 * I + col];
#pragma unroll
      for (int I = 0; I < 4; ++I) {
        const double a = wg * nv[I];
#pragma unroll
        for (int J = 0; J < 4; ++J) el_dmma(acc[I][J][0], acc[I][J][1], a, nv[J]);
      }
    }
#pragma unroll
    for (int I = 0; I < 4; ++I)
#pragma unroll
      for (int J = 0; J < 4; ++J)
#pragma unroll
        for (int v = 0; v < 2; ++v) {
          const int i = 8 * I + col, j = 8 * J + 2 * kq + v;
          if (i < 27 && j < 27) w.out[i * 27 + j] = acc[I][J][v];
        }
    __syncwarp();
    for (int q = lane; q < 729; q += 32) Me[(size_t)e * 729 + q] = w.out[q];
    __syncwarp();
  }
}

constexpr size_t EL_SMEM = (2187 + 28 * 32) * sizeof(double) + EL_WARPS * sizeof(ElWarp);

// One warp per 9-node face: int_Gamma N N^T dGamma with dA = |t_xi x t_eta|.
__global__ void quad9_face_mass_kernel(int n_faces, const double* __restrict__ xyz,
                                       const int32_t* __restrict__ fconn, double* __restrict__ Fe) {
  const int lane = threadIdx.x & 31;
  const int f = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (f >= n_faces) return;
  double dA = 0.0;
  if (lane < 9) {
    const int g = lane;
    double t[2][3] = {{0, 0, 0}, {0, 0, 0}};
    for (int i = 0; i < 9; ++i) {
      const int node = fconn[(size_t)f * 9 + i];
      for (int b = 0; b < 3; ++b) {
        const double x = xyz[(size_t)node * 3 + b];
        t[0][b] += c_qdN[(g * 9 + i) * 2 + 0] * x;
        t[1][b] += c_qdN[(g * 9 + i) * 2 + 1] * x;
      }
    }
    const double cx = t[0][1] * t[1][2] - t[0][2] * t[1][1];
    const double cy = t[0][2] * t[1][0] - t[0][0] * t[1][2];
    const double cz = t[0][0] * t[1][1] - t[0][1] * t[1][0];
    dA = c_qW[g] * sqrt(cx * cx + cy * cy + cz * cz);
  }
  double w9[9];
#pragma unroll
  for (int g = 0; g < 9; ++g) w9[g] = __shfl_sync(0xffffffffu, dA, g);
  for (int q = lane; q < 81; q += 32) {
    const int i = q / 9, j = q % 9;
    double m = 0.0;
#pragma unroll
    for (int g = 0; g < 9; ++g) m += w9[g] * c_qN[g * 9 + i] * c_qN[g * 9 + j];
    Fe[(size_t)f * 81 + q] = m;
  }
}

// ------------------------------------------------ Reissner-Mindlin plate ---
// 9-node flat plate element with node DoFs (u, v, w, bx, by): membrane ("disc")
// = the reference's plane-stress element (assembly.py:31-67), bending
// kappa = [bx,x, by,y, bx,y + by,x] with D_b = E t^3/(12(1-nu^2)) (...), shear
// gamma = [w,x + bx, w,y + by] with (5/6) G t at the 2x2 rule, consistent mass
// rho t (u, v, w) and rho t^3/12 (bx, by).  One CTA per element, one thread per
// (row, col) entry of the 45 x 45 matrices.
constexpr int PL_NT = 128;

__device__ __forceinline__ void quad9_geom(const double (*X)[2], const double* dN_ref, double* dNx,
                                           double* wdet, double w, int* bad, int e) {
  double J[2][2] = {{0, 0}, {0, 0}};
  for (int i = 0; i < 9; ++i)
    for (int a = 0; a < 2; ++a)
      for (int b = 0; b < 2; ++b) J[a][b] += dN_ref[i * 2 + a] * X[i][b];
  const double det = J[0][0] * J[1][1] - J[0][1] * J[1][0];
  if (!(det > 0.0)) atomicMin(bad, e);
  const double id = 1.0 / det;
  const double iJ[2][2] = {{J[1][1] * id, -J[0][1] * id}, {-J[1][0] * id, J[0][0] * id}};
  for (int i = 0; i < 9; ++i)
    for (int b = 0; b < 2; ++b) dNx[i * 2 + b] = dN_ref[i * 2] * iJ[0][b] + dN_ref[i * 2 + 1] * iJ[1][b];
  *wdet = w * det;
}

__global__ void __launch_bounds__(PL_NT) rm_plate_kernel(int n_elem, const double* __restrict__ xyz,
                                                         const int32_t* __restrict__ conn, double E, double nu,
                                                         double rho, double t, double* __restrict__ Ke,
                                                         double* __restrict__ Me, int* __restrict__ bad) {
  __shared__ double X[9][2];
  __shared__ double dF[9][18], wF[9], NF[9][9];   // full 3x3 rule
  __shared__ double dR[4][18], wR[4], NR[4][9];   // reduced 2x2 rule
  const int tid = threadIdx.x;
  const double cm = E * t / (1.0 - nu * nu), cb = E * t * t * t / (12.0 * (1.0 - nu * nu));
  const double gs = 5.0 / 6.0 * E / (2.0 * (1.0 + nu)) * t;
  const double mt = rho * t, mr = rho * t * t * t / 12.0;
  for (int e = blockIdx.x; e < n_elem; e += gridDim.x) {
    if (tid < 18) X[tid / 2][tid % 2] = xyz[(size_t)conn[(size_t)e * 9 + tid / 2] * 3 + tid % 2];
    __syncthreads();
    if (tid < 9) {
      quad9_geom(X, &c_qdN[tid * 18], dF[tid], &wF[tid], c_qW[tid], bad, e);
      for (int i = 0; i < 9; ++i) NF[tid][i] = c_qN[tid * 9 + i];
    } else if (tid >= 32 && tid < 36) {
      const int g = tid - 32;
      quad9_geom(X, &c_rdN[g * 18], dR[g], &wR[g], c_rW[g], bad, e);
      for (int i = 0; i < 9; ++i) NR[g][i] = c_rN[g * 9 + i];
    }
    __syncthreads();
    for (int q = tid; q < 2025; q += PL_NT) {
      const int A = q / 45, B = q - A * 45;
      const int a = A / 5, pa = A - a * 5, b = B / 5, pb = B - b * 5;
      double k = 0.0, m = 0.0;
      const bool mem = pa < 2 && pb < 2, ben = pa >= 3 && pb >= 3;
      if (mem || ben) {
        // B column of (node, dof): [d/dx, 0, d/dy] for the x-type dof, [0, d/dy, d/dx] for the y-type dof
        const int ta = mem ? pa : pa - 3, tb = mem ? pb : pb - 3;
        const double c = mem ? cm : cb;
        for (int g = 0; g < 9; ++g) {
          const double ax = dF[g][a * 2], ay = dF[g][a * 2 + 1], bx = dF[g][b * 2], by = dF[g][b * 2 + 1];
          double v;
          if (ta == 0 && tb == 0) v = ax * bx + 0.5 * (1.0 - nu) * ay * by;
          else if (ta == 1 && tb == 1) v = ay * by + 0.5 * (1.0 - nu) * ax * bx;
          else if (ta == 0) v = nu * ax * by + 0.5 * (1.0 - nu) * ay * bx;
          else v = nu * ay * bx + 0.5 * (1.0 - nu) * ax * by;
          k += wF[g] * c * v;
        }
      }
      if (pa >= 2 && pb >= 2) {  // transverse shear, reduced rule
        for (int g = 0; g < 4; ++g) {
          double sa0, sa1, sb0, sb1;
          if (pa == 2) { sa0 = dR[g][a * 2]; sa1 = dR[g][a * 2 + 1]; }
          else if (pa == 3) { sa0 = NR[g][a]; sa1 = 0.0; }
          else { sa0 = 0.0; sa1 = NR[g][a]; }
          if (pb == 2) { sb0 = dR[g][b * 2]; sb1 = dR[g][b * 2 + 1]; }
          else if (pb == 3) { sb0 = NR[g][b]; sb1 = 0.0; }
          else { sb0 = 0.0; sb1 = NR[g][b]; }
          k += wR[g] * gs * (sa0 * sb0 + sa1 * sb1);
        }
      }
      if (pa == pb) {
        const double mc = pa >= 3 ? mr : mt;
        for (int g = 0; g < 9; ++g) m += wF[g] * mc * NF[g][a] * NF[g][b];
      }
      Ke[(size_t)e * 2025 + q] = k;
      Me[(size_t)e * 2025 + q] = m;
    }
    __syncthreads();
  }
}

// Device flag for the "non-positive Jacobian" check (lowest bad element id):
// one device int + one pinned host int for the whole process, reset with a
// memset (0x7f7f7f7f > any element id) — no per-call allocation.
__device__ int g_bad_elem;
static int* bad_flag_dev() {
  static int* p = nullptr;
  if (!p) cudaGetSymbolAddress((void**)&p, g_bad_elem);
  return p;
}
static int* bad_flag_host() {
  static int* h = nullptr;
  if (!h) cudaHostAlloc((void**)&h, sizeof(int), cudaHostAllocDefault);
  return h;
}
static int bad_flag_reset(cudaStream_t stream) {
  int* d = bad_flag_dev();
  if (!d || !bad_flag_host()) {
    set_error("bad-element flag allocation failed");
    return 2;
  }
  VB_CUDA(cudaMemsetAsync(d, 0x7f, sizeof(int), stream));
  return 0;
}
static int bad_flag_read(cudaStream_t stream, int32_t* out) {
  int* h = bad_flag_host();
  VB_CUDA(cudaMemcpyAsync(h, bad_flag_dev(), sizeof(int), cudaMemcpyDeviceToHost, stream));
  VB_CUDA(cudaStreamSynchronize(stream));
  *out = *h == 0x7f7f7f7f ? -1 : *h;
  return 0;
}

int rm_plate_elements(int n_elem, const double* xyz, const int32_t* conn, double E, double nu, double rho, double t,
                      double* Ke, double* Me, int32_t* bad_elem_host, cudaStream_t stream) {
  if (int rc = init_tables()) return rc;
  if (int rc = bad_flag_reset(stream)) return rc;
  if (n_elem > 0) {
    const int grid = n_elem < 148 * 16 ? n_elem : 148 * 16;
    rm_plate_kernel<<<grid, PL_NT, 0, stream>>>(n_elem, xyz, conn, E, nu, rho, t, Ke, Me, bad_flag_dev());
    VB_LAUNCHED("rm_plate_kernel");
  }
  if (int rc = bad_flag_read(stream, bad_elem_host)) return rc;
  return 0;
}

// ------------------------------------------------------ facet shells (cfg4) ---
// Flat 9-node facet shell with global node DoFs (u_x, u_y, u_z, th_x, th_y, th_z):
// the plate above in the facet frame (e1 = node 0 -> 2, e3 = corner-plane normal,
// e2 = e3 x e1; nodes projected onto that plane), with the chain rule
// dN = dshape inv(J)^T (annular frame webs have non-diagonal J), a Hughes-Brezzi
// drilling term gamma int (t3 - (v,x - u,y)/2)^2 dA (gamma = drill G t) and rotary
// inertia rho t^3/12 on t3, rotated to global per node block:
// u_loc = R u, bx = R[1].th, by = -R[0].th, t3 = R[2].th (oracle/fuselage.py).
// One CTA per element; the local 54 x 54 matrix is staged in shared memory and
// each thread forms global entries from the 3 x 3 non-zero rotation sub-blocks.
constexpr int FS_NT = 128;

__device__ __forceinline__ void quad9_geom_chain(const double (*X)[2], const double* dN_ref, double* dNx,
                                                 double* wdet, double w, int* bad, int e) {
  double J[2][2] = {{0, 0}, {0, 0}};
  for (int i = 0; i < 9; ++i)
    for (int a = 0; a < 2; ++a)
      for (int b = 0; b < 2; ++b) J[a][b] += dN_ref[i * 2 + a] * X[i][b];
  const double det = J[0][0] * J[1][1] - J[0][1] * J[1][0];
  if (!(det > 0.0)) atomicMin(bad, e);
  const double id = 1.0 / det;
  const double iJ[2][2] = {{J[1][1] * id, -J[0][1] * id}, {-J[1][0] * id, J[0][0] * id}};
  for (int i = 0; i < 9; ++i)
    for (int b = 0; b < 2; ++b) dNx[i * 2 + b] = dN_ref[i * 2] * iJ[b][0] + dN_ref[i * 2 + 1] * iJ[b][1];
  *wdet = w * det;
}

__global__ void __launch_bounds__(FS_NT) facet_shell_kernel(int n_elem, const double* __restrict__ xyz,
                                                            const int32_t* __restrict__ conn,
                                                            const int32_t* __restrict__ mat,
                                                            const double* __restrict__ props, int n_mat,
                                                            double drill, double* __restrict__ Ke,
                                                            double* __restrict__ Me, int* __restrict__ bad) {
  __shared__ double X3[9][3], X[9][2], R[3][3], T[6][6];
  __shared__ double dF[9][18], wF[9], NF[9][9];
  __shared__ double dR[4][18], wR[4], NR[4][9];
  __shared__ double Ls[54 * 54];
  const int tid = threadIdx.x;
  for (int e = blockIdx.x; e < n_elem; e += gridDim.x) {
    int m = mat[e];
    if (m < 0 || m >= n_mat) {  // reported like a degenerate element (no out-of-range read)
      if (tid == 0) atomicMin(bad, e);
      m = 0;
    }
    const double E = props[m * 4 + 0], nu = props[m * 4 + 1], rho = props[m * 4 + 2], t = props[m * 4 + 3];
    const double cm = E * t / (1.0 - nu * nu), cb = E * t * t * t / (12.0 * (1.0 - nu * nu));
    const double G = E / (2.0 * (1.0 + nu));
    const double gs = 5.0 / 6.0 * G * t, gam = drill * G * t;
    const double mt = rho * t, mr = rho * t * t * t / 12.0;
    if (tid < 27) X3[tid / 3][tid % 3] = xyz[(size_t)conn[(size_t)e * 9 + tid / 3] * 3 + tid % 3];
    __syncthreads();
    if (tid == 0) {
      double e1[3], v2[3], e3[3];
      for (int b = 0; b < 3; ++b) { e1[b] = X3[2][b] - X3[0][b]; v2[b] = X3[6][b] - X3[0][b]; }
      e3[0] = e1[1] * v2[2] - e1[2] * v2[1];
      e3[1] = e1[2] * v2[0] - e1[0] * v2[2];
      e3[2] = e1[0] * v2[1] - e1[1] * v2[0];
      const double n1 = 1.0 / sqrt(e1[0] * e1[0] + e1[1] * e1[1] + e1[2] * e1[2]);
      const double n3 = 1.0 / sqrt(e3[0] * e3[0] + e3[1] * e3[1] + e3[2] * e3[2]);
      for (int b = 0; b < 3; ++b) { R[0][b] = e1[b] * n1; R[2][b] = e3[b] * n3; }
      R[1][0] = R[2][1] * R[0][2] - R[2][2] * R[0][1];
      R[1][1] = R[2][2] * R[0][0] - R[2][0] * R[0][2];
      R[1][2] = R[2][0] * R[0][1] - R[2][1] * R[0][0];
    }
    __syncthreads();
    if (tid < 18) {
      const int i = tid / 2, a = tid % 2;
      X[i][a] = (X3[i][0] - X3[0][0]) * R[a][0] + (X3[i][1] - X3[0][1]) * R[a][1] + (X3[i][2] - X3[0][2]) * R[a][2];
    } else if (tid >= 32 && tid < 68) {
      const int q = tid - 32, p = q / 6, j = q % 6;
      double v = 0.0;
      if (p < 3 && j < 3) v = R[p][j];
      else if (p == 3 && j >= 3) v = R[1][j - 3];
      else if (p == 4 && j >= 3) v = -R[0][j - 3];
      else if (p == 5 && j >= 3) v = R[2][j - 3];
      T[p][j] = v;
    }
    __syncthreads();
    if (tid < 9) {
      quad9_geom_chain(X, &c_qdN[tid * 18], dF[tid], &wF[tid], c_qW[tid], bad, e);
      for (int i = 0; i < 9; ++i) NF[tid][i] = c_qN[tid * 9 + i];
    } else if (tid >= 32 && tid < 36) {
      const int g = tid - 32;
      quad9_geom_chain(X, &c_rdN[g * 18], dR[g], &wR[g], c_rW[g], bad, e);
      for (int i = 0; i < 9; ++i) NR[g][i] = c_rN[g * 9 + i];
    }
    __syncthreads();
    for (int pass = 0; pass < 2; ++pass) {
      // local 54 x 54 (pass 0: stiffness, pass 1: mass)
      for (int q = tid; q < 2916; q += FS_NT) {
        const int A = q / 54, B = q - A * 54;
        const int a = A / 6, pa = A - a * 6, b = B / 6, pb = B - b * 6;
        double v = 0.0;
        if (pass == 0) {
          const bool mem = pa < 2 && pb < 2, ben = (pa == 3 || pa == 4) && (pb == 3 || pb == 4);
          if (mem || ben) {
            const int ta = mem ? pa : pa - 3, tb = mem ? pb : pb - 3;
            const double c = mem ? cm : cb;
            for (int g = 0; g < 9; ++g) {
              const double ax = dF[g][a * 2], ay = dF[g][a * 2 + 1], bx = dF[g][b * 2], by = dF[g][b * 2 + 1];
              double s;
              if (ta == 0 && tb == 0) s = ax * bx + 0.5 * (1.0 - nu) * ay * by;
              else if (ta == 1 && tb == 1) s = ay * by + 0.5 * (1.0 - nu) * ax * bx;
              else if (ta == 0) s = nu * ax * by + 0.5 * (1.0 - nu) * ay * bx;
              else s = nu * ay * bx + 0.5 * (1.0 - nu) * ax * by;
              v += wF[g] * c * s;
            }
          }
          if (pa >= 2 && pa <= 4 && pb >= 2 && pb <= 4) {  // transverse shear, reduced rule
            for (int g = 0; g < 4; ++g) {
              double sa0, sa1, sb0, sb1;
              if (pa == 2) { sa0 = dR[g][a * 2]; sa1 = dR[g][a * 2 + 1]; }
              else if (pa == 3) { sa0 = NR[g][a]; sa1 = 0.0; }
              else { sa0 = 0.0; sa1 = NR[g][a]; }
              if (pb == 2) { sb0 = dR[g][b * 2]; sb1 = dR[g][b * 2 + 1]; }
              else if (pb == 3) { sb0 = NR[g][b]; sb1 = 0.0; }
              else { sb0 = 0.0; sb1 = NR[g][b]; }
              v += wR[g] * gs * (sa0 * sb0 + sa1 * sb1);
            }
          }
          const bool da = pa == 0 || pa == 1 || pa == 5, db = pb == 0 || pb == 1 || pb == 5;
          if (da && db) {  // drilling: Bd = [u: +N,y / 2, v: -N,x / 2, t3: N]
            for (int g = 0; g < 9; ++g) {
              const double sa = pa == 0 ? 0.5 * dF[g][a * 2 + 1] : (pa == 1 ? -0.5 * dF[g][a * 2] : NF[g][a]);
              const double sb = pb == 0 ? 0.5 * dF[g][b * 2 + 1] : (pb == 1 ? -0.5 * dF[g][b * 2] : NF[g][b]);
              v += wF[g] * gam * sa * sb;
            }
          }
        } else if (pa == pb) {
          const double mc = pa >= 3 ? mr : mt;
          for (int g = 0; g < 9; ++g) v += wF[g] * mc * NF[g][a] * NF[g][b];
        }
        Ls[q] = v;
      }
      __syncthreads();
      double* out = (pass == 0 ? Ke : Me) + (size_t)e * 2916;
      for (int q = tid; q < 2916; q += FS_NT) {
        const int A = q / 54, B = q - A * 54;
        const int a = A / 6, i = A - a * 6, b = B / 6, j = B - b * 6;
        const int p0 = i < 3 ? 0 : 3, q0 = j < 3 ? 0 : 3;
        double v = 0.0;
#pragma unroll
        for (int p = 0; p < 3; ++p)
#pragma unroll
          for (int r = 0; r < 3; ++r)
            v += T[p0 + p][i] * Ls[(a * 6 + p0 + p) * 54 + b * 6 + q0 + r] * T[q0 + r][j];
        out[q] = v;
      }
      __syncthreads();
    }
  }
}

int facet_shell_elements(int n_elem, const double* xyz, const int32_t* conn, const int32_t* mat,
                         const double* props, int n_mat, double drill, double* Ke, double* Me,
                         int32_t* bad_elem_host, cudaStream_t stream) {
  if (int rc = init_tables()) return rc;
  if (int rc = bad_flag_reset(stream)) return rc;
  if (n_elem > 0) {
    const int grid = n_elem < 148 * 16 ? n_elem : 148 * 16;
    facet_shell_kernel<<<grid, FS_NT, 0, stream>>>(n_elem, xyz, conn, mat, props, n_mat, drill, Ke, Me,
                                                    bad_flag_dev());
    VB_LAUNCHED("facet_shell_kernel");
  }
  if (int rc = bad_flag_read(stream, bad_elem_host)) return rc;
  return 0;
}

// ------------------------------------------------------------ pattern ---
// Triplet t = e*nr*nc + a*nc + b of element e has row rdofs[e][a] and column
// cdofs[e][b] (assembly.py:166-167: rows = repeat(dofs), cols = tile(dofs));
// a negative DoF (eliminated, e.g. a clamped plate node) drops the triplet:
// its key is the all-ones sentinel, which sorts after every real key.

__global__ void make_keys_kernel(int64_t T, int nr, int nc, int ncols, const int32_t* __restrict__ rdofs,
                                 const int32_t* __restrict__ cdofs, uint64_t KEY_DROP,
                                 uint64_t* __restrict__ keys, int32_t* __restrict__ vals) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T) return;
  const int64_t pe = (int64_t)nr * nc;
  const int64_t e = t / pe;
  const int a = (int)((t / nc) % nr), b = (int)(t % nc);
  const int row = rdofs[e * nr + a], col = cdofs[e * nc + b];
  keys[t] = (row < 0 || col < 0) ? KEY_DROP : (uint64_t)row * (uint64_t)ncols + (uint64_t)col;
  vals[t] = (int32_t)t;
}

__global__ void head_flags_kernel(int64_t T, const uint64_t* __restrict__ keys, uint64_t KEY_DROP,
                                  int32_t* __restrict__ head) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T) return;
  head[t] = (keys[t] != KEY_DROP && (t == 0 || keys[t] != keys[t - 1])) ? 1 : 0;
}

__global__ void emit_pattern_kernel(int64_t T, int ncols, const uint64_t* __restrict__ keys, uint64_t KEY_DROP,
                                    const int32_t* __restrict__ head, const int32_t* __restrict__ slot,
                                    int32_t* __restrict__ indices, int64_t* __restrict__ gptr,
                                    int32_t* __restrict__ row_count, int64_t* __restrict__ tvalid) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T) return;
  const uint64_t k = keys[t];
  if (k != KEY_DROP && (t == T - 1 || keys[t + 1] == KEY_DROP)) *tvalid = t + 1;  // valid triplet count
  if (head[t]) {
    const int s = slot[t];
    indices[s] = (int32_t)(k % (uint64_t)ncols);
    gptr[s] = t;
    atomicAdd(row_count + (int)(k / (uint64_t)ncols), 1);
  }
}

__global__ void finish_gptr_kernel(const int32_t* nnz_dev, const int64_t* tvalid, int64_t* gptr) {
  gptr[*nnz_dev] = *tvalid;
}

__global__ void nnz_kernel(int64_t T, const int32_t* head, const int32_t* slot, int32_t* nnz) {
  *nnz = slot[T - 1] + head[T - 1];
}

__global__ void csr_gather_kernel(int64_t nnz, const int64_t* __restrict__ gptr,
                                  const int32_t* __restrict__ gidx, const double* __restrict__ tv,
                                  double* __restrict__ vals) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= nnz) return;
  double acc = 0.0;
  const int64_t b = gptr[s], e = gptr[s + 1];
  for (int64_t t = b; t < e; ++t) acc += __ldg(tv + gidx[t]);
  vals[s] = acc;
}

// Two primitives sharing one pattern (Kgrad and Mnn): the gather map is read
// once for both.
__global__ void csr_gather2_kernel(int64_t nnz, const int64_t* __restrict__ gptr,
                                   const int32_t* __restrict__ gidx, const double* __restrict__ tv0,
                                   const double* __restrict__ tv1, double* __restrict__ v0,
                                   double* __restrict__ v1) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= nnz) return;
  double a0 = 0.0, a1 = 0.0;
  const int64_t b = __ldg(gptr + s), e = __ldg(gptr + s + 1);
  for (int64_t t = b; t < e; ++t) {
    const int32_t g = __ldg(gidx + t);
    a0 += __ldg(tv0 + g);
    a1 += __ldg(tv1 + g);
  }
  v0[s] = a0;
  v1[s] = a1;
}

// ------------------------------------------------------------- host side ---
struct PatternWs {
  size_t keys_a, keys_b, vals_a, head, slot, cnt, nnz, tvalid, cub;
  size_t total;
};

static size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

static int pattern_ws(int64_t T, int n, PatternWs* w) {
  size_t cub_sort = 0, cub_scan = 0;
  VB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, cub_sort, (uint64_t*)nullptr, (uint64_t*)nullptr,
                                          (int32_t*)nullptr, (int32_t*)nullptr, (int64_t)T));
  VB_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, cub_scan, (int32_t*)nullptr, (int32_t*)nullptr,
                                        (int64_t)(T > n + 1 ? T : n + 1)));
  size_t off = 0;
  w->keys_a = off; off += align256(T * 8);
  w->keys_b = off; off += align256(T * 8);
  w->vals_a = off; off += align256(T * 4);
  w->head = off; off += align256(T * 4);
  w->slot = off; off += align256(T * 4);
  w->cnt = off; off += align256((size_t)(n + 1) * 4);
  w->nnz = off; off += 256;
  w->tvalid = off; off += 256;
  w->cub = off; off += align256(cub_sort > cub_scan ? cub_sort : cub_scan);
  w->total = off;
  return 0;
}

size_t csr_pattern_workspace_bytes(int n, int64_t T) {
  PatternWs w;
  if (pattern_ws(T, n, &w)) return 0;
  return w.total;
}

static int end_bit_for(uint64_t maxkey) {
  int b = 1;
  while (b < 64 && (maxkey >> b)) ++b;
  return b;
}

int csr_pattern_from_blocks(int n_rows, int n_cols, int n_elem, int nr, int nc, const int32_t* rdofs,
                            const int32_t* cdofs, int32_t* indptr, int32_t* indices, int64_t* gptr, int32_t* gidx,
                            int64_t* nnz_host, void* work, size_t work_bytes, cudaStream_t stream) {
  const int64_t T = (int64_t)n_elem * nr * nc;
  VB_CHECK_ARG(T > 0 && T < ((int64_t)1 << 31), "vb_csr_pattern_from_blocks: triplet count out of range");
  const int nmax = n_rows > n_cols ? n_rows : n_cols;
  PatternWs w;
  if (int rc = pattern_ws(T, nmax, &w)) return rc;
  VB_CHECK_ARG(work && work_bytes >= w.total, "vb_csr_pattern_from_blocks: workspace too small");
  char* base = (char*)work;
  uint64_t* ka = (uint64_t*)(base + w.keys_a);
  uint64_t* kb = (uint64_t*)(base + w.keys_b);
  int32_t* va = (int32_t*)(base + w.vals_a);
  int32_t* head = (int32_t*)(base + w.head);
  int32_t* slot = (int32_t*)(base + w.slot);
  int32_t* cnt = (int32_t*)(base + w.cnt);
  int32_t* nnz_dev = (int32_t*)(base + w.nnz);
  int64_t* tvalid = (int64_t*)(base + w.tvalid);
  void* cubtmp = base + w.cub;
  size_t cubbytes = work_bytes - w.cub;
  const int nt = 256;
  const unsigned nb = (unsigned)((T + nt - 1) / nt);
  // keys need end_bit bits; the drop sentinel (all end_bit bits set) sorts last
  const int eb = end_bit_for((uint64_t)n_rows * (uint64_t)n_cols) + 1;
  const uint64_t drop = (eb >= 64) ? ~(uint64_t)0 : (((uint64_t)1 << eb) - 1);
  make_keys_kernel<<<nb, nt, 0, stream>>>(T, nr, nc, n_cols, rdofs, cdofs, drop, ka, va);
  VB_LAUNCHED("make_keys_kernel");
  VB_CUDA(cub::DeviceRadixSort::SortPairs(cubtmp, cubbytes, ka, kb, va, gidx, T, 0, eb, stream));
  count_launches(1);
  head_flags_kernel<<<nb, nt, 0, stream>>>(T, kb, drop, head);
  VB_LAUNCHED("head_flags_kernel");
  VB_CUDA(cub::DeviceScan::ExclusiveSum(cubtmp, cubbytes, head, slot, T, stream));
  count_launches(1);
  VB_CUDA(cudaMemsetAsync(cnt, 0, (size_t)(n_rows + 1) * 4, stream));
  VB_CUDA(cudaMemsetAsync(tvalid, 0, sizeof(int64_t), stream));
  emit_pattern_kernel<<<nb, nt, 0, stream>>>(T, n_cols, kb, drop, head, slot, indices, gptr, cnt, tvalid);
  VB_LAUNCHED("emit_pattern_kernel");
  VB_CUDA(cub::DeviceScan::ExclusiveSum(cubtmp, cubbytes, cnt, indptr, n_rows + 1, stream));
  count_launches(1);
  nnz_kernel<<<1, 1, 0, stream>>>(T, head, slot, nnz_dev);
  VB_LAUNCHED("nnz_kernel");
  finish_gptr_kernel<<<1, 1, 0, stream>>>(nnz_dev, tvalid, gptr);
  VB_LAUNCHED("finish_gptr_kernel");
  int32_t nnz = 0;
  VB_CUDA(cudaMemcpyAsync(&nnz, nnz_dev, 4, cudaMemcpyDeviceToHost, stream));
  VB_CUDA(cudaStreamSynchronize(stream));
  *nnz_host = nnz;
  return 0;
}

int csr_pattern_from_elements(int n, int n_elem, int npe, const int32_t* conn, int32_t* indptr,
                              int32_t* indices, int64_t* gptr, int32_t* gidx, int64_t* nnz_host,
                              void* work, size_t work_bytes, cudaStream_t stream) {
  return csr_pattern_from_blocks(n, n, n_elem, npe, npe, conn, conn, indptr, indices, gptr, gidx, nnz_host, work,
                                 work_bytes, stream);
}

int csr_gather2(int64_t nnz, const int64_t* gptr, const int32_t* gidx, const double* tv0, const double* tv1,
                double* v0, double* v1, cudaStream_t stream) {
  if (nnz <= 0) return 0;
  const int nt = 256;
  csr_gather2_kernel<<<(unsigned)((nnz + nt - 1) / nt), nt, 0, stream>>>(nnz, gptr, gidx, tv0, tv1, v0, v1);
  VB_LAUNCHED("csr_gather2_kernel");
  return 0;
}

int csr_gather(int64_t nnz, const int64_t* gptr, const int32_t* gidx, const double* tv, double* vals,
               cudaStream_t stream) {
  if (nnz <= 0) return 0;
  const int nt = 256;
  csr_gather_kernel<<<(unsigned)((nnz + nt - 1) / nt), nt, 0, stream>>>(nnz, gptr, gidx, tv, vals);
  VB_LAUNCHED("csr_gather_kernel");
  return 0;
}

int hex27_helmholtz(int n_elem, const double* xyz, const int32_t* conn, double* Ke, double* Me,
                    int32_t* bad_elem_host, cudaStream_t stream, int chain) {
  if (int rc = init_tables()) return rc;
  if (int rc = bad_flag_reset(stream)) return rc;
  int dev = 0, nsm = 148;
  VB_CUDA(cudaGetDevice(&dev));
  VB_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  const int need = (n_elem + EL_WARPS - 1) / EL_WARPS;
  const int grid = need < nsm * 2 ? need : nsm * 2;
  if (grid > 0) {
    VB_CUDA(cudaFuncSetAttribute(hex27_helmholtz_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)EL_SMEM));
    hex27_helmholtz_kernel<<<grid, EL_NT, EL_SMEM, stream>>>(n_elem, xyz, conn, Ke, Me, bad_flag_dev(), chain);
    VB_LAUNCHED("hex27_helmholtz_kernel");
  }
  if (int rc = bad_flag_read(stream, bad_elem_host)) return rc;
  return 0;
}

int quad9_face_mass(int n_faces, const double* xyz, const int32_t* fconn, double* Fe,
                    cudaStream_t stream) {
  if (int rc = init_tables()) return rc;
  if (n_faces <= 0) return 0;
  const int nt = 128;
  const unsigned grid = (unsigned)(((int64_t)n_faces * 32 + nt - 1) / nt);
  quad9_face_mass_kernel<<<grid, nt, 0, stream>>>(n_faces, xyz, fconn, Fe);
  VB_LAUNCHED("quad9_face_mass_kernel");
  return 0;
}

}  // namespace vb

namespace vb {

// ------------------------------------------- structured box fast path ---
// Uniform axis-aligned hex27 box.  With tensor-product bases and 3x3x3 Gauss
// the element matrices factorise, and summing them over the elements gives the
// Kronecker form of the assembled 1D matrices:
//   Kgrad = Mz (x) My (x) Kx + Mz (x) Ky (x) Mx + Kz (x) My (x) Mx,  Mnn = Mz (x) My (x) Mx
// (exact algebra; values agree with the element-order sums to rounding, the
// pattern is the same canonical CSR).  One warp per x-line of rows writes
// indices and both value arrays with consecutive lanes on consecutive slots:
// the kernel writes exactly the algorithmic bytes of the assembly.
// band tables: [d][i][o] with o = j - i + 2 in 0..4, for d = x, y, z.
__global__ void __launch_bounds__(256) hex27_box_csr_kernel(int nx, int ny, int nz, const double* __restrict__ K1,
                                                            const double* __restrict__ M1, int maxnp,
                                                            int32_t* __restrict__ indptr,
                                                            int32_t* __restrict__ indices, double* __restrict__ Kv,
                                                            double* __restrict__ Mv) {
  // Kronecker form per entry: K = kx (my mz) + mx (ky mz + kz my), M = mx (my mz).
  // The (y, z) factors P = my mz, Q = ky mz + kz my and the column bases of the
  // <= 25 neighbour lines are set up once per line task in shared memory; the x
  // factors once per row.  Each row's entries are one contiguous run of
  // cx*cy*cz slots (qz slowest, qx fastest) that the warp's lanes stride, so
  // every store instruction writes 32 consecutive entries.
  __shared__ double2 sPQ[8][25];
  __shared__ int sCol[8][25];
  __shared__ double2 sKX[8][8][5];  // (kx, mx) band rows of the task's 8 x-rows
  const int npx = 2 * nx + 1, npy = 2 * ny + 1, npz = 2 * nz + 1;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int Tx = 8 * nx + 1, Ty = 8 * ny + 1;  // nnz < 2^31 is checked by the launcher
  const int nlines = npy * npz;
  constexpr int SEG = 8;  // rows per warp task (enough tasks to fill the GPU)
  const int nseg = (npx + SEG - 1) / SEG;
  const double* Kx = K1;
  const double* Ky = K1 + (size_t)maxnp * 5;
  const double* Kz = K1 + (size_t)2 * maxnp * 5;
  const double* Mx = M1;
  const double* My = M1 + (size_t)maxnp * 5;
  const double* Mz = M1 + (size_t)2 * maxnp * 5;
  for (int task = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5); task < nlines * nseg;
       task += (int)((gridDim.x * blockDim.x) >> 5)) {
    const int line = task / nseg, seg = task - line * nseg;
    const int iy = line % npy, iz = line / npy;
    // neighbour ranges along y and z (quadratic elements: 3 or 5 nodes)
    const int ylo = (iy & 1) ? iy - 1 : max(0, iy - 2), yhi = (iy & 1) ? iy + 1 : min(npy - 1, iy + 2);
    const int zlo = (iz & 1) ? iz - 1 : max(0, iz - 2), zhi = (iz & 1) ? iz + 1 : min(npz - 1, iz + 2);
    const int cy = yhi - ylo + 1, cz = zhi - zlo + 1;
    const int py = iy < 1 ? 0 : 3 * iy + 2 * min(ny - 1, (iy - 1) >> 1);
    const int pz = iz < 1 ? 0 : 3 * iz + 2 * min(nz - 1, (iz - 1) >> 1);
    const int ix0 = seg * SEG, ix1 = min(npx, ix0 + SEG);
    const int px = ix0 < 1 ? 0 : 3 * ix0 + 2 * min(nx - 1, (ix0 - 1) >> 1);
    int start = pz * Ty * Tx + cz * (py * Tx + cy * px);
    // one round of table loads per task: (y, z) factors and the 8 rows' x bands
    __syncwarp();
    if (lane < cy * cz) {
      const int qz = lane / cy, qy = lane - qz * cy;
      const int jy = ylo + qy, jz = zlo + qz;
      const double ky = __ldg(Ky + iy * 5 + jy - iy + 2), my = __ldg(My + iy * 5 + jy - iy + 2);
      const double kz = __ldg(Kz + iz * 5 + jz - iz + 2), mz = __ldg(Mz + iz * 5 + jz - iz + 2);
      sPQ[w][lane] = make_double2(my * mz, ky * mz + kz * my);
      sCol[w][lane] = (jz * npy + jy) * npx;
    }
    for (int t = lane; t < (ix1 - ix0) * 5; t += 32) {
      const int rr = t / 5, o = t - rr * 5, ix = ix0 + rr;
      sKX[w][rr][o] = make_double2(__ldg(Kx + ix * 5 + o), __ldg(Mx + ix * 5 + o));
    }
    __syncwarp();
    for (int ix = ix0; ix < ix1; ++ix) {
      const int xlo = (ix & 1) ? ix - 1 : max(0, ix - 2), xhi = (ix & 1) ? ix + 1 : min(npx - 1, ix + 2);
      const int cx = xhi - xlo + 1, cnt = cx * cy * cz;
      if (lane == 0) indptr[(int64_t)line * npx + ix] = start;
      const double2* km_row = &sKX[w][ix - ix0][xlo - ix + 2];
      // entry e of the row: column, K and M values
      auto entry = [&](int e, int& col, double& kv, double& mv) {
        // p = e / cx (cx is 3 or 5 except on 1-element lines)
        const int p = cx == 3 ? (e * 43691) >> 17 : (cx == 5 ? (e * 52429) >> 18 : e / cx);
        const int qx = e - p * cx;
        const double2 pq = sPQ[w][p], km = km_row[qx];
        col = sCol[w][p] + xlo + qx;
        kv = km.x * pq.x + km.y * pq.y;
        mv = km.y * pq.x;
      };
      // 16-byte (value) / 8-byte (index) stores on the even-aligned body of the run
      const int head = start & 1;
      if (head && lane == 0) {
        int c; double kv, mv;
        entry(0, c, kv, mv);
        indices[start] = c; Kv[start] = kv; Mv[start] = mv;
      }
      for (int e = head + 2 * lane; e < cnt; e += 64) {
        int c0, c1 = 0; double k0, m0, k1 = 0.0, m1 = 0.0;
        entry(e, c0, k0, m0);
        const int sidx = start + e;
        if (e + 1 < cnt) {
          entry(e + 1, c1, k1, m1);
          *reinterpret_cast<int2*>(indices + sidx) = make_int2(c0, c1);
          *reinterpret_cast<double2*>(Kv + sidx) = make_double2(k0, k1);
          *reinterpret_cast<double2*>(Mv + sidx) = make_double2(m0, m1);
        } else {
          indices[sidx] = c0; Kv[sidx] = k0; Mv[sidx] = m0;
        }
      }
      start += cnt;
    }
    if (line == nlines - 1 && ix1 == npx && lane == 0) indptr[(int64_t)nlines * npx] = start;
  }
}

int64_t hex27_box_nnz(int nx, int ny, int nz) { return (8LL * nx + 1) * (8LL * ny + 1) * (8LL * nz + 1); }

int hex27_box_csr(int nx, int ny, int nz, const double* K1, const double* M1, int maxnp, int32_t* indptr,
                  int32_t* indices, double* Kv, double* Mv, cudaStream_t st) {
  VB_CHECK_ARG(nx > 0 && ny > 0 && nz > 0, "vb_hex27_box_csr: bad element counts");
  VB_CHECK_ARG(hex27_box_nnz(nx, ny, nz) < ((int64_t)1 << 31), "vb_hex27_box_csr: nnz exceeds int32");
  VB_CHECK_ARG(maxnp >= 2 * nx + 1 && maxnp >= 2 * ny + 1 && maxnp >= 2 * nz + 1, "vb_hex27_box_csr: band table too small");
  const int64_t tasks = (int64_t)(2 * ny + 1) * (2 * nz + 1) * ((2 * nx + 1 + 7) / 8);
  const int nt = 256;
  int64_t blocks = (tasks * 32 + nt - 1) / nt;
  hex27_box_csr_kernel<<<(unsigned)blocks, nt, 0, st>>>(nx, ny, nz, K1, M1, maxnp, indptr, indices, Kv, Mv);
  VB_LAUNCHED("hex27_box_csr_kernel");
  return 0;
}

}  // namespace vb
