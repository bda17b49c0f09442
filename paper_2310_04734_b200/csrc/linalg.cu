// Dense/sparse building blocks of the offline MOR phase (SURVEY §8a A7–A9):
//   CSR SpMM (real CSR x complex dense)        mor.py:81-85,117 (scipy csr_matvecs)
//   complex GEMM, op(A) in {N, C} on DMMA      mor.py:81-89,102,105 (BLAS zgemm)
//   deterministic column norms                 mor.py:127,132,157,184,188 (numpy norm)
//   dense scatter of scaled CSR primitives     mor.py:41-46 (operator at an expansion point)
#include "common.cuh"
#include "mma.cuh"
#include "sweep.cuh"

namespace vb {

// csr_spmm (CSR SpMM / SpMV) lives in spmm.cu.

// D += alpha * A (real CSR scattered into a dense complex matrix): the operator
// K - w^2 M + i w D at an expansion point (mor.py:41-46) for the dense FOM LU.
__global__ void csr_axpy_dense_kernel(int n_rows, const int32_t* __restrict__ indptr,
                                      const int32_t* __restrict__ indices,
                                      const double* __restrict__ vals, z_t alpha, z_t* __restrict__ D,
                                      int64_t ldd) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t row = warp; row < n_rows; row += nwarps) {
    const int b = indptr[row], e = indptr[row + 1];
    for (int j = b + lane; j < e; j += 32) {
      const double a = vals[j];
      z_t* d = D + row * ldd + indices[j];
      *d = zmake(d->x + alpha.x * a, d->y + alpha.y * a);
    }
  }
}

int csr_axpy_dense(int n_rows, const int32_t* indptr, const int32_t* indices, const double* vals,
                   z_t alpha, z_t* D, int64_t ldd, cudaStream_t st) {
  if (n_rows <= 0) return 0;
  const int nt = 256;
  unsigned grid = (unsigned)(((int64_t)n_rows * 32 + nt - 1) / nt);
  if (grid > 148u * 64u) grid = 148u * 64u;
  csr_axpy_dense_kernel<<<grid, nt, 0, st>>>(n_rows, indptr, indices, vals, alpha, D, ldd);
  VB_LAUNCHED("csr_axpy_dense_kernel");
  return 0;
}

// ------------------------------------------------------------------ GEMM ---
using blk::NT;
using blk::KC;

// C = alpha A B + beta C, A (m x k), B (k x n): DMMA tiles over the grid.
// n <= 16 (W -= V G in the basis orthogonalisation: V streamed once, G tiny)
// uses 128 x 16 tiles so the padded DMMA work stays below the HBM time.
using GemmNN = blk::Gemm<64, 32, 4, 2, 3, blk::EPI_AXPBY, 16, true>;     // 3M products
using GemmNN16 = blk::Gemm<128, 16, 8, 1, 3, blk::EPI_AXPBY, 16, true>;

template <class G>
__global__ void __launch_bounds__(NT) zgemm_nn_kernel(int m, int n, int k, z_t alpha, const z_t* A,
                                                      int64_t lda, const z_t* B, int64_t ldb,
                                                      z_t beta, z_t* C, int64_t ldc) {
  extern __shared__ double2 smem[];
  G::run(C, (int)ldc, A, (int)lda, B, (int)ldb, m, n, k, smem, alpha, beta, blockIdx.x, gridDim.x);
}

template <class G, int TM, int TN>
static int launch_nn(int m, int n, int k, z_t alpha, const z_t* A, int64_t lda, const z_t* B, int64_t ldb,
                     z_t beta, z_t* C, int64_t ldc, cudaStream_t st) {
  const int ntiles = ((m + TM - 1) / TM) * ((n + TN - 1) / TN);
  int dev = 0, nsm = 148, per_sm = 1;
  VB_CUDA(cudaGetDevice(&dev));
  VB_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  VB_CUDA(cudaFuncSetAttribute(zgemm_nn_kernel<G>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G::SMEM));
  VB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, zgemm_nn_kernel<G>, NT, G::SMEM));
  if (per_sm < 1) per_sm = 1;
  const int grid = ntiles < per_sm * nsm ? ntiles : per_sm * nsm;
  zgemm_nn_kernel<G><<<grid, NT, G::SMEM, st>>>(m, n, k, alpha, A, lda, B, ldb, beta, C, ldc);
  VB_LAUNCHED("zgemm_nn_kernel");
  return 0;
}

// Split-K C_part[s] = A_s^H B_s over k-chunks s (A: k x m, B: k x n, row-major):
// one (tile, chunk) per CTA, TM x TN tiles (64 x 32, or 128 x 16 when n <= 16:
// the tall-skinny V^H W of the basis orthogonalisation, where padding n = 10 to
// 32 made the kernel DMMA-bound at 3x the useful work).  Both operands stream
// through a 3-stage cp.async ring in their natural [k][.] layout (A is NOT
// transposed on the way in: the A^H fragments are read column-wise from the
// [k][i] tile, row stride == 2 (mod 8) 16-byte units so the 8 lanes of a
// quarter-warp hit 8 distinct bank groups) and conjugated in registers.
constexpr int CN_KCH = 512, CN_ST = 3;
template <int TM, int TN>
struct CnCfg {
  static constexpr int WN = TN / 16, WM = (NT / 32) / WN;  // warps, 16 x 16 each
  static_assert(WM * 16 == TM, "warp grid");
  static constexpr int LDA = TM + 2, LDB = TN + 2;
  static constexpr size_t SMEM = (size_t)CN_ST * KC * (LDA + LDB) * sizeof(z_t);
};

template <int TM, int TN>
__global__ void __launch_bounds__(NT) zgemm_cn_partial_kernel(int m, int n, int k, const z_t* __restrict__ A,
                                                              int64_t lda, const z_t* __restrict__ B,
                                                              int64_t ldb, z_t* __restrict__ part) {
  using Cfg = CnCfg<TM, TN>;
  constexpr int LDA = Cfg::LDA, LDB = Cfg::LDB;
  extern __shared__ double2 cn_smem[];
  z_t (*As)[KC * LDA] = reinterpret_cast<z_t (*)[KC * LDA]>(cn_smem);                    // [k][i]
  z_t (*Bs)[KC * LDB] = reinterpret_cast<z_t (*)[KC * LDB]>(cn_smem + CN_ST * KC * LDA);  // [k][j]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp / Cfg::WN, wn = warp % Cfg::WN;
  const int ntn = (n + TN - 1) / TN, ntm = (m + TM - 1) / TM;
  const int tile = blockIdx.x % (ntm * ntn), split = blockIdx.x / (ntm * ntn);
  const int m0 = (tile / ntn) * TM, n0 = (tile % ntn) * TN;
  const int kb = split * CN_KCH, ke = min(k, kb + CN_KCH);
  const int nch = (ke - kb + KC - 1) / KC;
  auto load = [&](int c, int st) {
    const int k0 = kb + c * KC;
#pragma unroll
    for (int q = 0; q < (KC * TM) / NT; ++q) {
      const int e = tid + q * NT, kk = e / TM, i = e - kk * TM;
      const bool ok = k0 + kk < ke && m0 + i < m;
      blk::cp_async16(&As[st][kk * LDA + i], ok ? (const void*)(A + (int64_t)(k0 + kk) * lda + m0 + i) : A, ok);
    }
#pragma unroll
    for (int q = 0; q < (KC * TN) / NT; ++q) {
      const int e = tid + q * NT, kk = e / TN, j = e - kk * TN;
      const bool ok = k0 + kk < ke && n0 + j < n;
      blk::cp_async16(&Bs[st][kk * LDB + j], ok ? (const void*)(B + (int64_t)(k0 + kk) * ldb + n0 + j) : B, ok);
    }
  };
  // 3M (Gauss) conjugate product: t1 = ar br, t2 = ai bi, t3 = (ar - ai)(br + bi);
  // Re = t1 + t2, Im = t3 - t1 + t2 (3 DMMAs per fragment pair instead of 4)
  double cr[2][2][2], ci[2][2][2], c2[2][2][2];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j)
      cr[i][j][0] = cr[i][j][1] = ci[i][j][0] = ci[i][j][1] = c2[i][j][0] = c2[i][j][1] = 0.0;
#pragma unroll
  for (int c = 0; c < CN_ST - 1; ++c) {
    if (c < nch) load(c, c);
    blk::cp_commit();
  }
  const int ar = lane >> 2, ak = lane & 3;
  for (int c = 0; c < nch; ++c) {
    blk::cp_wait<CN_ST - 2>();
    __syncthreads();
    if (c + CN_ST - 1 < nch) load(c + CN_ST - 1, (c + CN_ST - 1) % CN_ST);
    blk::cp_commit();
    const z_t* as = As[c % CN_ST];
    const z_t* bs = Bs[c % CN_ST];
#pragma unroll
    for (int kk = 0; kk < KC / 4; ++kk) {
      const int kr = kk * 4 + ak;
      z_t a[2], b[2];
#pragma unroll
      for (int i = 0; i < 2; ++i) a[i] = as[kr * LDA + wm * 16 + i * 8 + ar];  // A^H[i][k] = conj(A[k][i])
#pragma unroll
      for (int j = 0; j < 2; ++j) b[j] = bs[kr * LDB + wn * 16 + j * 8 + ar];
      double sa[2], sb[2];
#pragma unroll
      for (int i = 0; i < 2; ++i) sa[i] = a[i].x - a[i].y;
#pragma unroll
      for (int j = 0; j < 2; ++j) sb[j] = b[j].x + b[j].y;
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          blk::dmma(cr[i][j][0], cr[i][j][1], a[i].x, b[j].x);
          blk::dmma(c2[i][j][0], c2[i][j][1], a[i].y, b[j].y);
          blk::dmma(ci[i][j][0], ci[i][j][1], sa[i], sb[j]);
        }
    }
  }
  blk::cp_wait<0>();
  z_t* P = part + (int64_t)split * m * n;
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        const int row = m0 + wm * 16 + i * 8 + (lane >> 2);
        const int col = n0 + wn * 16 + j * 8 + 2 * (lane & 3) + v;
        if (row < m && col < n)
          P[(int64_t)row * n + col] = zmake(cr[i][j][v] + c2[i][j][v], ci[i][j][v] - cr[i][j][v] + c2[i][j][v]);
      }
}

template <int TM, int TN>
static int launch_cn_partial(int m, int n, int k, const z_t* A, int64_t lda, const z_t* B, int64_t ldb, z_t* work,
                             int nsplit, cudaStream_t st) {
  const int ntiles = ((m + TM - 1) / TM) * ((n + TN - 1) / TN);
  const size_t smem = CnCfg<TM, TN>::SMEM;
  VB_CUDA(cudaFuncSetAttribute(zgemm_cn_partial_kernel<TM, TN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)smem));
  zgemm_cn_partial_kernel<TM, TN><<<(unsigned)(ntiles * nsplit), NT, smem, st>>>(m, n, k, A, lda, B, ldb, work);
  VB_LAUNCHED("zgemm_cn_partial_kernel");
  return 0;
}

// C = alpha sum_s C_part[s] + beta C: a CTA owns 32 consecutive outputs (one
// per lane, coalesced split rows), its 8 warps take splits w, w + 8, ... and
// combine their partial sums in a fixed order (deterministic).
__global__ void __launch_bounds__(256) zgemm_cn_reduce_kernel(int m, int n, int nsplit,
                                                              const z_t* __restrict__ part, z_t alpha, z_t beta,
                                                              z_t* __restrict__ C, int64_t ldc) {
  __shared__ z_t red[8][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t mn = (int64_t)m * n;
  const int64_t e = (int64_t)blockIdx.x * 32 + lane;
  z_t acc = zmake(0.0, 0.0);
  if (e < mn)
    for (int s = warp; s < nsplit; s += 8) acc = zadd(acc, part[(int64_t)s * mn + e]);
  red[warp][lane] = acc;
  __syncthreads();
  if (warp == 0 && e < mn) {
#pragma unroll
    for (int w = 1; w < 8; ++w) acc = zadd(acc, red[w][lane]);
    const int64_t i = e / n, j = e - i * n;
    z_t out = zmul(alpha, acc);
    if (beta.x != 0.0 || beta.y != 0.0) out = zfma(out, beta, C[i * ldc + j]);
    C[i * ldc + j] = out;
  }
}

// ------------------------------------------------- narrow GEMV (n == 1) ---
// The in-block Gram-Schmidt of the basis orthogonalisation projects one column
// w against the j <= 64 columns already kept: y = A^H w and w -= A y.  On the
// DMMA tile kernels these are > 99 % padding; here they are HBM streams on the
// CUDA cores: a warp per row, lanes over the (<= 64) columns.  Fixed row
// partition (GV_GRID CTAs) + fixed-order reductions -> deterministic.
constexpr int GV_GRID = 4 * 148, GV_MAXM = 64;

__global__ void __launch_bounds__(256) zgemv_cn_partial_kernel(int k, int m, const z_t* __restrict__ A, int64_t lda,
                                                               const z_t* __restrict__ x, int64_t ldx,
                                                               z_t* __restrict__ part) {
  __shared__ z_t red[8][GV_MAXM];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t chunk = ((int64_t)k + gridDim.x - 1) / gridDim.x;
  const int64_t r0 = (int64_t)blockIdx.x * chunk, r1 = min((int64_t)k, r0 + chunk);
  z_t a0 = zmake(0.0, 0.0), a1 = zmake(0.0, 0.0);
  const bool c0 = lane < m, c1 = lane + 32 < m;
#pragma unroll 4
  for (int64_t r = r0 + warp; r < r1; r += 8) {
    const z_t xv = x[r * ldx];
    const z_t* Ar = A + r * lda;
    if (c0) { const z_t a = Ar[lane]; a0 = zmake(a0.x + a.x * xv.x + a.y * xv.y, a0.y + a.x * xv.y - a.y * xv.x); }
    if (c1) { const z_t a = Ar[lane + 32]; a1 = zmake(a1.x + a.x * xv.x + a.y * xv.y, a1.y + a.x * xv.y - a.y * xv.x); }
  }
  red[warp][lane] = a0;
  red[warp][lane + 32] = a1;
  __syncthreads();
  if (warp == 0) {
#pragma unroll
    for (int w = 1; w < 8; ++w) {
      a0 = zadd(a0, red[w][lane]);
      a1 = zadd(a1, red[w][lane + 32]);
    }
    if (c0) part[(int64_t)blockIdx.x * m + lane] = a0;
    if (c1) part[(int64_t)blockIdx.x * m + lane + 32] = a1;
  }
}

// y = alpha A g + beta y  (A: rows x k, k <= 64; g, y single columns): a
// thread per row (its k loads are independent and hit the same L1 lines as
// its warp neighbours'), g broadcast from shared memory.
__global__ void __launch_bounds__(256) zgemv_nn_kernel(int rows, int k, z_t alpha, const z_t* __restrict__ A,
                                                       int64_t lda, const z_t* __restrict__ g, int64_t ldg, z_t beta,
                                                       z_t* __restrict__ y, int64_t ldy) {
  __shared__ z_t gs[GV_MAXM];
  if (threadIdx.x < k) gs[threadIdx.x] = g[threadIdx.x * ldg];
  __syncthreads();
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  const z_t* Ar = A + r * lda;
  z_t acc0 = zmake(0.0, 0.0), acc1 = zmake(0.0, 0.0);
  int c = 0;
#pragma unroll 4
  for (; c + 1 < k; c += 2) {
    acc0 = zfma(acc0, Ar[c], gs[c]);
    acc1 = zfma(acc1, Ar[c + 1], gs[c + 1]);
  }
  if (c < k) acc0 = zfma(acc0, Ar[c], gs[c]);
  z_t out = zmul(alpha, zadd(acc0, acc1));
  if (beta.x != 0.0 || beta.y != 0.0) out = zfma(out, beta, y[r * ldy]);
  y[r * ldy] = out;
}

size_t zgemm_workspace_bytes(char transa, int m, int n, int k) {
  if (transa == 'N' || transa == 'n') return 0;
  if (n == 1 && m <= GV_MAXM) return (size_t)GV_GRID * m * sizeof(z_t);
  const int64_t nsplit = (k + CN_KCH - 1) / CN_KCH;
  return (size_t)nsplit * m * n * sizeof(z_t);
}

int zgemm(char transa, int m, int n, int k, z_t alpha, const z_t* A, int64_t lda, const z_t* B,
          int64_t ldb, z_t beta, z_t* C, int64_t ldc, void* work, size_t work_bytes,
          cudaStream_t st) {
  if (m <= 0 || n <= 0) return 0;
  if (transa == 'N' || transa == 'n') {
    if (k <= 0) {
      set_error("vb_zgemm: k must be positive");
      return 1;
    }
    if (n == 1 && k <= GV_MAXM) {
      zgemv_nn_kernel<<<(unsigned)((m + 255) / 256), 256, 0, st>>>(m, k, alpha, A, lda, B, ldb, beta, C, ldc);
      VB_LAUNCHED("zgemv_nn_kernel");
      return 0;
    }
    if (n <= 16) return launch_nn<GemmNN16, 128, 16>(m, n, k, alpha, A, lda, B, ldb, beta, C, ldc, st);
    return launch_nn<GemmNN, 64, 32>(m, n, k, alpha, A, lda, B, ldb, beta, C, ldc, st);
  }
  if (transa != 'C' && transa != 'c') {
    set_error("vb_zgemm: transa must be 'N' or 'C'");
    return 1;
  }
  VB_CHECK_ARG(k > 0, "vb_zgemm: k must be positive");
  VB_CHECK_ARG(work && work_bytes >= zgemm_workspace_bytes(transa, m, n, k), "vb_zgemm: workspace too small");
  if (n == 1 && m <= GV_MAXM) {
    zgemv_cn_partial_kernel<<<GV_GRID, 256, 0, st>>>(k, m, A, lda, B, ldb, (z_t*)work);
    VB_LAUNCHED("zgemv_cn_partial_kernel");
    zgemm_cn_reduce_kernel<<<(unsigned)((m + 31) / 32), 256, 0, st>>>(m, 1, GV_GRID, (const z_t*)work, alpha, beta,
                                                                      C, ldc);
    VB_LAUNCHED("zgemm_cn_reduce_kernel");
    return 0;
  }
  const int nsplit = (k + CN_KCH - 1) / CN_KCH;
  const int rc = n <= 16 ? launch_cn_partial<128, 16>(m, n, k, A, lda, B, ldb, (z_t*)work, nsplit, st)
                         : launch_cn_partial<64, 32>(m, n, k, A, lda, B, ldb, (z_t*)work, nsplit, st);
  if (rc) return rc;
  const int64_t mn = (int64_t)m * n;
  zgemm_cn_reduce_kernel<<<(unsigned)((mn + 31) / 32), 256, 0, st>>>(m, n, nsplit, (const z_t*)work,
                                                                         alpha, beta, C, ldc);
  VB_LAUNCHED("zgemm_cn_reduce_kernel");
  return 0;
}

// --------------------------------------------------------- column norms ---
// norms[j] = ||W[:, j]||_2, deterministic: fixed row blocks, fixed-order reduce.
constexpr int NRM_ROWS = 2048;

__global__ void colnorm_partial_kernel(int n, int m, const z_t* __restrict__ W, int64_t ldw,
                                       double* __restrict__ part) {
  // block = (row block, column); threads stride the rows of the block
  const int nb = (n + NRM_ROWS - 1) / NRM_ROWS;
  const int rb = blockIdx.x % nb, j = blockIdx.x / nb;
  const int r0 = rb * NRM_ROWS, r1 = min(n, r0 + NRM_ROWS);
  double s = 0.0;
  for (int i = r0 + threadIdx.x; i < r1; i += blockDim.x) s += zabs2(W[(int64_t)i * ldw + j]);
  __shared__ double red[32];
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    s = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    s = warp_sum(s);
    if (threadIdx.x == 0) part[(int64_t)j * nb + rb] = s;
  }
}

__global__ void colnorm_final_kernel(int m, int nb, const double* __restrict__ part, double* __restrict__ out) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= m) return;
  double s = 0.0;
  for (int b = 0; b < nb; ++b) s += part[(int64_t)j * nb + b];
  out[j] = sqrt(s);
}

// ------------------------------------------------------------ batched GEMV ---
// Y_b = alpha_b A_b X_b + beta_b Y_b for a batch of row-major complex matrices
// with few right-hand sides (s <= 16): the solve phase of the plane-block
// full-order solver (planes.py), a chain of HBM-bound block products.  One warp
// per row of A: 16-B coalesced loads of the row (8 in flight per lane), X from
// L1/L2, s accumulators per lane, shuffle reduction; grid.y = batch item.
constexpr int GEMV_NT = 256;

struct GemvBatch {
  vb_gemv_item it[VB_GEMV_MAX];
};

template <int S>
__device__ __forceinline__ void gemv_row(const vb_gemv_item& g, int row, int lane) {
  const z_t* __restrict__ a = (const z_t*)g.A + (int64_t)row * g.lda;
  const z_t* __restrict__ X = (const z_t*)g.X;
  const int s = S > 0 ? S : g.s;
  z_t acc[S > 0 ? S : 16];
#pragma unroll
  for (int q = 0; q < (S > 0 ? S : 16); ++q) acc[q] = zmake(0.0, 0.0);
  int c = lane;
  for (; c + 224 < g.n; c += 256) {
    z_t av[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) av[u] = __ldcs(a + c + 32 * u);
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int q = 0; q < (S > 0 ? S : 16); ++q)
        if (q < s) acc[q] = zfma(acc[q], av[u], __ldg(X + (int64_t)(c + 32 * u) * g.ldx + q));
  }
  for (; c < g.n; c += 32) {
    const z_t av = __ldcs(a + c);
#pragma unroll
    for (int q = 0; q < (S > 0 ? S : 16); ++q)
      if (q < s) acc[q] = zfma(acc[q], av, __ldg(X + (int64_t)c * g.ldx + q));
  }
#pragma unroll
  for (int q = 0; q < (S > 0 ? S : 16); ++q) {
    if (q >= s) break;
    double re = acc[q].x, im = acc[q].y;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      re += __shfl_xor_sync(0xffffffffu, re, o);
      im += __shfl_xor_sync(0xffffffffu, im, o);
    }
    if (lane == 0) {
      z_t* y = (z_t*)g.Y + (int64_t)row * g.ldy + q;
      const z_t al = zmake(g.alpha.re, g.alpha.im), be = zmake(g.beta.re, g.beta.im);
      z_t v = zmul(al, zmake(re, im));
      if (be.x != 0.0 || be.y != 0.0) v = zfma(v, be, *y);
      *y = v;
    }
  }
}

__global__ void __launch_bounds__(GEMV_NT) zgemv_batched_kernel(GemvBatch B) {
  const vb_gemv_item& g = B.it[blockIdx.y];
  const int lane = threadIdx.x & 31;
  const int row = blockIdx.x * (GEMV_NT / 32) + (threadIdx.x >> 5);
  if (row >= g.m) return;
  if (g.s == 1) gemv_row<1>(g, row, lane);
  else gemv_row<0>(g, row, lane);
}

int zgemv_batched(int n_items, const vb_gemv_item* items, cudaStream_t st) {
  for (int i0 = 0; i0 < n_items; i0 += VB_GEMV_MAX) {
    const int cnt = n_items - i0 < VB_GEMV_MAX ? n_items - i0 : VB_GEMV_MAX;
    GemvBatch B;
    int mmax = 0;
    for (int i = 0; i < cnt; ++i) {
      const vb_gemv_item& g = items[i0 + i];
      VB_CHECK_ARG(g.m >= 0 && g.n >= 0 && g.s >= 1 && g.s <= 16 && g.A && g.X && g.Y, "vb_zgemv_batched: bad item");
      B.it[i] = g;
      mmax = g.m > mmax ? g.m : mmax;
    }
    if (mmax == 0) continue;
    dim3 grid((mmax + GEMV_NT / 32 - 1) / (GEMV_NT / 32), cnt);
    zgemv_batched_kernel<<<grid, GEMV_NT, 0, st>>>(B);
    VB_LAUNCHED("zgemv_batched_kernel");
  }
  return 0;
}

size_t column_norms_workspace_bytes(int n, int m) {
  const int nb = (n + NRM_ROWS - 1) / NRM_ROWS;
  return (size_t)nb * m * sizeof(double);
}

int column_norms(int n, int m, const z_t* W, int64_t ldw, double* out, void* work, size_t wb,
                 cudaStream_t st) {
  if (m <= 0) return 0;
  VB_CHECK_ARG(n > 0, "vb_column_norms: n must be positive");
  VB_CHECK_ARG(work && wb >= column_norms_workspace_bytes(n, m), "vb_column_norms: workspace too small");
  const int nb = (n + NRM_ROWS - 1) / NRM_ROWS;
  colnorm_partial_kernel<<<(unsigned)(nb * m), 256, 0, st>>>(n, m, W, ldw, (double*)work);
  VB_LAUNCHED("colnorm_partial_kernel");
  colnorm_final_kernel<<<(m + 127) / 128, 128, 0, st>>>(m, nb, (const double*)work, out);
  VB_LAUNCHED("colnorm_final_kernel");
  return 0;
}

// W[:, j] *= scale[j] for the m columns.
__global__ void scale_columns_kernel(int n, int m, z_t* W, int64_t ldw, const double* scale) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)n * m) return;
  const int64_t i = e / m, j = e - i * m;
  const double s = scale[j];
  z_t* p = W + i * ldw + j;
  *p = zmake(p->x * s, p->y * s);
}

int scale_columns(int n, int m, z_t* W, int64_t ldw, const double* scale, cudaStream_t st) {
  const int64_t tot = (int64_t)n * m;
  if (tot <= 0) return 0;
  scale_columns_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(n, m, W, ldw, scale);
  VB_LAUNCHED("scale_columns_kernel");
  return 0;
}

}  // namespace vb
