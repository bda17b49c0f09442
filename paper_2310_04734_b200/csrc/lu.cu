// Dense complex LU of ONE large matrix across the whole GPU: the full-order
// solver at the rational expansion points and certification frequencies
// (SURVEY §8a A6).  Replaces scipy `splu(...).solve` in vibrofem/mor.py:48-49,
// 153-156 and solvers.py:62-78 for n up to ~25k (cfg1 n = 4,641).
//
// A persistent cooperative kernel (one CTA per SM, grid-wide barriers):
//   panel   : right-looking column steps over the NB = 64 panel; every CTA owns a
//             contiguous row range.  Per column: local izamax over own rows,
//             candidate rows + row j published to double-buffered scratch, ONE
//             grid barrier, then every CTA picks the same pivot (max |Re|+|Im|,
//             lowest row on ties), swaps/eliminates only its own rows.
//   swaps   : the panel's interchanges applied to all other columns (LAPACK laswp
//             on the whole row, so L stays consistent with P).
//   TRSM    : U12 = L11^-1 A12, L11^-1 by recursive doubling, DMMA strips.
//   GEMM    : A22 -= L21 U12, DMMA tiles distributed over all CTAs.
// The diagonal-block inverses L_kk^-1, U_kk^-1 and the final row permutation are
// kept for the blocked triangular solves of vb_zgetrs.
#include <cooperative_groups.h>
#include <cstdlib>

#include "common.cuh"
#include "mma.cuh"
#include "sweep.cuh"
#include "tma.cuh"
#include "tma_big.cuh"

namespace cg = cooperative_groups;

namespace vb {
namespace lu {

using blk::KC;
using blk::NB;
using blk::NT;

// Trailing update: the large-tile TMA + mbarrier DMMA GEMM (csrc/tma_big.cuh,
// 128 x 64 tiles, one CTA per SM) over a 2-D tensor map of the matrix, tiles
// spread over the CTAs.
#ifndef VB_LU_STAGES
#define VB_LU_STAGES 3
#endif
using GemmT = tma::GemmBig<VB_LU_STAGES>;

// Profiling aid (-DVB_PHASE_TIMING): CTA 0's SM cycles in panel / swaps /
// TRSM / GEMM (each phase ends at a grid barrier), vb_debug_phase_cycles 32..35.
__device__ unsigned long long g_lu_cycles[4];
#ifdef VB_PHASE_TIMING
#define LU_MARK(k)                                                              \
  do {                                                                          \
    if (blockIdx.x == 0 && threadIdx.x == 0) {                                  \
      const long long _n = clock64();                                           \
      g_lu_cycles[k] += (unsigned long long)(_n - _lt);                         \
      _lt = _n;                                                                 \
    }                                                                           \
  } while (0)
#define LU_BEGIN long long _lt = clock64()
#else
#define LU_MARK(k) \
  do {             \
  } while (0)
#define LU_BEGIN
#endif
constexpr int LDL = NB + 4;
constexpr int TRS_N = 32;
constexpr int LDS_B = TRS_N + 2;
constexpr size_t TRSM_SMEM = (size_t)(NB * LDL + NB * LDS_B) * sizeof(z_t);
constexpr size_t LU_SMEM = (GemmT::SMEM > TRSM_SMEM ? GemmT::SMEM : TRSM_SMEM) + 1024;  // + 1024-B alignment
// + the CTA's panel rows (ceil(n / grid) x (NB + 1) complex)
inline size_t lu_smem(int n, int grid) {
  const size_t rows = (size_t)((n + grid - 1) / grid) * (NB + 1) * sizeof(z_t) + 1024;
  return rows > LU_SMEM ? rows : LU_SMEM;
}

struct __align__(64) LuParams {
  tma::BigMaps maps;  // over the matrix (must stay first: 64-B aligned)
  int n;
  z_t* A;
  int64_t lda;
  int* ipiv;      // [n]   row interchanged with row j at step j
  int* perm;      // [n]   final permutation: row i of P A is row perm[i] of A
  int* info;      // [1]
  double* pval;   // [2][grid]
  int* pidx;      // [2][grid]
  z_t* prow;      // [2][grid][NB]
  z_t* rowj;      // [2][NB]
  z_t* Linv;      // [nblk][NB][NB]
  z_t* Uinv;      // [nblk][NB][NB]
  int npan;       // look-ahead kernel: CTAs [0, npan) factor the panels
  unsigned* bar;  // look-ahead kernel: the panel CTAs' barrier counter (zeroed before launch)
};

__device__ __forceinline__ void row_range(int n, int& lo, int& hi) {
  const int rpc = (n + gridDim.x - 1) / gridDim.x;
  lo = blockIdx.x * rpc;
  hi = min(n, lo + rpc);
}

// Block inverse of the 64x64 diagonal block at (k0, k0) into smem T (LDL),
// identity-padded beyond nb; LOWER uses the strictly lower part + unit diagonal.
template <bool LOWER>
__device__ void load_diag_block(const z_t* A, int64_t lda, int k0, int nb, z_t* T) {
  for (int e = threadIdx.x; e < NB * NB; e += NT) {
    const int i = e / NB, j = e - i * NB;
    z_t v = zmake(i == j ? 1.0 : 0.0, 0.0);
    if (i < nb && j < nb) {
      if (LOWER) {
        if (j < i) v = __ldcg(A + (int64_t)(k0 + i) * lda + k0 + j);
      } else {
        v = (j >= i) ? __ldcg(A + (int64_t)(k0 + i) * lda + k0 + j) : zmake(0.0, 0.0);
      }
    }
    T[i * LDL + j] = v;
  }
  __syncthreads();
  blk::tri_inv64<LOWER>(T, LDL);
}

__global__ void __launch_bounds__(NT, 1) zgetrf_kernel(const __grid_constant__ LuParams P) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(1024) char smem_raw[];
  double2* smem = (double2*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ GemmT::Bars bars;
  __shared__ z_t s_prow[NB];
  __shared__ z_t s_rowj[NB];
  __shared__ double rv[NT / 32];
  __shared__ int ri[NT / 32];
  __shared__ int s_piv, s_idx;
  __shared__ double s_val;
  const int n = P.n, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int G = gridDim.x, c = blockIdx.x;
  const int64_t lda = P.lda;
  z_t* A = P.A;
  int lo, hi;
  row_range(n, lo, hi);
  if (c == 0 && tid == 0) *P.info = 0;
  LU_BEGIN;

  for (int k0 = 0; k0 < n; k0 += NB) {
    const int nb = min(NB, n - k0), kend = k0 + nb;
    // ------------------------------------------------------------ panel
    // The CTA's own panel rows [plo, hi) live in shared memory for the 64
    // column steps (one round of loads, one write-back): only the pivot search
    // partials, the candidate rows and row j travel through global scratch.
    const int plo = max(lo, k0), pn = max(0, hi - plo);
    constexpr int LP = NB + 1;  // padded row (conflict-free row-per-thread access)
    z_t* Ps = smem;
    for (int e = tid; e < pn * nb; e += NT) {
      const int i = e / nb, t = e - i * nb;
      Ps[i * LP + t] = __ldcg(A + (int64_t)(plo + i) * lda + k0 + t);
    }
    __syncthreads();
    for (int j = k0; j < kend; ++j) {
      const int buf = j & 1, jj = j - k0;
      double v = -1.0;
      int pi = 0x7fffffff;
      for (int i = max(plo, j) + tid; i < hi; i += NT) {
        const double a = zabs1(Ps[(i - plo) * LP + jj]);
        if (a > v) { v = a; pi = i; }
      }
      warp_argmax(v, pi);
      if (lane == 0) { rv[warp] = v; ri[warp] = pi; }
      __syncthreads();
      if (warp == 0) {
        v = lane < NT / 32 ? rv[lane] : -1.0;
        pi = lane < NT / 32 ? ri[lane] : 0x7fffffff;
        warp_argmax(v, pi);
        if (lane == 0) { s_val = v; s_idx = pi; }
      }
      __syncthreads();
      if (tid == 0) {
        P.pval[buf * G + c] = s_val;
        P.pidx[buf * G + c] = s_idx;
      }
      if (s_val >= 0.0)
        for (int t = tid; t < nb; t += NT) P.prow[((int64_t)buf * G + c) * NB + t] = Ps[(s_idx - plo) * LP + t];
      if (j >= plo && j < hi)
        for (int t = tid; t < nb; t += NT) P.rowj[buf * NB + t] = Ps[(j - plo) * LP + t];
      grid.sync();
      // every CTA resolves the same pivot from the published partials
      if (warp == 0) {
        double bv = -1.0;
        int bi = 0x7fffffff, bc = 0;
        for (int q = lane; q < G; q += 32) {
          const double pv = __ldcg(P.pval + buf * G + q);
          const int px = __ldcg(P.pidx + buf * G + q);
          if (pv > bv || (pv == bv && px < bi)) { bv = pv; bi = px; bc = q; }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
          const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
          const int oc = __shfl_xor_sync(0xffffffffu, bc, o);
          if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; bc = oc; }
        }
        if (lane == 0) {
          s_val = bv;
          s_piv = bv > 0.0 ? bi : -1;
          s_idx = bc;
        }
      }
      __syncthreads();
      const int p = s_piv;
      if (p < 0) {  // exactly singular column (LAPACK: INFO = j+1, no interchange)
        if (c == 0 && tid == 0) {
          if (*P.info == 0) *P.info = j + 1;
          P.ipiv[j] = j;
        }
        __syncthreads();
        continue;
      }
      for (int t = tid; t < nb; t += NT) {
        s_prow[t] = __ldcg(P.prow + ((int64_t)buf * G + s_idx) * NB + t);
        s_rowj[t] = __ldcg(P.rowj + buf * NB + t);
      }
      VB_DCHECK(p >= j && p < n && s_idx >= 0 && s_idx < G);
      if (c == 0 && tid == 0) P.ipiv[j] = p;
      __syncthreads();
      const z_t pinv = zrecip(s_prow[jj]);
      if (p != j && j >= plo && j < hi)
        for (int t = tid; t < nb; t += NT) Ps[(j - plo) * LP + t] = s_prow[t];
      // eliminate own rows i > j; row p (if swapped) now holds the old row j
      const int r0 = max(plo, j + 1);
      const int nrows = hi - r0, ncols = nb - jj - 1;
      if (nrows > 0) {
        // multipliers first (column j), then the rank-1 update of the panel
        for (int i = r0 + tid; i < hi; i += NT) {
          const z_t aij = (i == p) ? s_rowj[jj] : Ps[(i - plo) * LP + jj];
          Ps[(i - plo) * LP + jj] = zmul(aij, pinv);
        }
        if (p != j && p >= r0 && p < hi)
          for (int t = tid; t < nb; t += NT)
            if (t != jj) Ps[(p - plo) * LP + t] = s_rowj[t];
        __syncthreads();
        if (ncols > 0)
          for (int e = tid; e < nrows * ncols; e += NT) {
            const int ii = e / ncols, t = jj + 1 + (e - ii * ncols);
            z_t* row = Ps + (r0 - plo + ii) * LP;
            row[t] = zfms(row[t], row[jj], s_prow[t]);
          }
      }
      __syncthreads();
    }
    for (int e = tid; e < pn * nb; e += NT) {
      const int i = e / nb, t = e - i * nb;
      A[(int64_t)(plo + i) * lda + k0 + t] = Ps[i * LP + t];
    }
    grid.sync();
    LU_MARK(0);
    // ------------------------------------------------------------ swaps
    {
      const int64_t ncol = (int64_t)n - nb;
      for (int64_t q = (int64_t)c * NT + tid; q < ncol; q += (int64_t)G * NT) {
        const int col = q < k0 ? (int)q : (int)(q + nb);
        for (int j = k0; j < kend; ++j) {
          const int p = __ldcg(P.ipiv + j);
          if (p != j) {
            // L2 reads (__ldcg): rows written by other CTAs earlier in this
            // kernel must never come from a stale line in this SM's L1
            const z_t t = __ldcg(A + (int64_t)j * lda + col);
            A[(int64_t)j * lda + col] = __ldcg(A + (int64_t)p * lda + col);
            A[(int64_t)p * lda + col] = t;
          }
        }
      }
    }
    grid.sync();
    LU_MARK(1);
    // ------------------------------------------------------------ TRSM
    {
      z_t* Li = smem;
      z_t* Bs = smem + NB * LDL;
      const int nblk = k0 / NB;
      const int nstrips = (n - kend + TRS_N - 1) / TRS_N;
      if (nstrips > c || c == 0) {
        load_diag_block<true>(A, lda, k0, nb, Li);
        if (c == 0)
          for (int e = tid; e < NB * NB; e += NT) P.Linv[(int64_t)nblk * NB * NB + e] = Li[(e / NB) * LDL + e % NB];
        const int wm = warp >> 1, wn = warp & 1;
        for (int st = c; st < nstrips; st += G) {
          const int cs = kend + st * TRS_N, ncol = min(TRS_N, n - cs);
          for (int e = tid; e < NB * TRS_N; e += NT) {
            const int i = e / TRS_N, jx = e - i * TRS_N;
            Bs[i * LDS_B + jx] = (i < nb && jx < ncol) ? __ldcg(A + (int64_t)(k0 + i) * lda + cs + jx) : zmake(0.0, 0.0);
          }
          __syncthreads();
          double cr[2][2][2], ci[2][2][2];
#pragma unroll
          for (int a = 0; a < 2; ++a)
#pragma unroll
            for (int b = 0; b < 2; ++b) cr[a][b][0] = cr[a][b][1] = ci[a][b][0] = ci[a][b][1] = 0.0;
          blk::warp_cmma<2, 2, false>(cr, ci, Li + (wm * 16) * LDL, LDL, Bs + wn * 16, LDS_B, (nb + 3) >> 2);
#pragma unroll
          for (int a = 0; a < 2; ++a)
#pragma unroll
            for (int b = 0; b < 2; ++b)
#pragma unroll
              for (int vv = 0; vv < 2; ++vv) {
                const int row = wm * 16 + a * 8 + (lane >> 2);
                const int col = wn * 16 + b * 8 + 2 * (lane & 3) + vv;
                if (row < nb && col < ncol) A[(int64_t)(k0 + row) * lda + cs + col] = zmake(cr[a][b][vv], ci[a][b][vv]);
              }
          __syncthreads();
        }
      }
      // U_kk^-1 for the triangular solves (U11 is final after the panel)
      if (c == (G > 1 ? 1 : 0)) {
        __syncthreads();
        load_diag_block<false>(A, lda, k0, nb, Li);
        for (int e = tid; e < NB * NB; e += NT) P.Uinv[(int64_t)nblk * NB * NB + e] = Li[(e / NB) * LDL + e % NB];
      }
    }
    grid.sync();
    LU_MARK(2);
    // ------------------------------------------------------------ GEMM
    if (kend < n) {
      GemmT::run(&P.maps, A, lda, kend, k0, k0, kend, n - kend, n - kend, nb, (char*)smem, &bars, c, G);
    }
    grid.sync();
    LU_MARK(3);
  }
  // final permutation from the interchange sequence (LAPACK ipiv semantics)
  if (c == 0) {
    for (int i = tid; i < n; i += NT) P.perm[i] = i;
    __syncthreads();
    if (tid == 0)
      for (int j = 0; j < n; ++j) {
        const int p = P.ipiv[j];
        if (p != j) {
          const int t = P.perm[j];
          P.perm[j] = P.perm[p];
          P.perm[p] = t;
        }
      }
  }
}

// ------------------------------------------------- look-ahead variant ---
// The same right-looking LU, but the next panel's factorisation (a chain of
// 64 pivot steps, latency-bound) overlaps the current trailing update
// (throughput-bound DMMA GEMM): CTAs [0, npan) are PANEL CTAs, the rest GEMM
// CTAs.  Per panel k:
//   all CTAs    : interchanges of panel k on the other columns, U12 = L11^-1 A12,
//                 then the update of panel k+1's 64 columns only (look-ahead);
//   panel CTAs  : factor panel k+1 (its rows [k0', n) re-split over the panel
//                 CTAs, held in shared memory; one barrier among the panel
//                 CTAs per column instead of a grid barrier);
//   GEMM CTAs   : meanwhile A22 -= L21 U12 on the columns right of panel k+1.
// Panel k+1 only touches its own 64 columns and the GEMM only the columns to
// their right, both reading the finished L21 / U12 of panel k; the row
// interchanges of panel k+1 reach the other columns after the grid barrier,
// as in LAPACK.  Same pivots (izamax order, lowest row on ties) and the same
// arithmetic per element as zgetrf_kernel.

// Barrier among the npan panel CTAs: monotone counter in global memory.
__device__ __forceinline__ void panel_barrier(unsigned* bar, unsigned target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(bar, 1u);
    unsigned v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
    } while ((int)(v - target) < 0);
  }
  __syncthreads();
}

// Factor panel [k0, k0 + nb) by the npan panel CTAs (pc = this CTA's index).
__device__ void la_factor_panel(const LuParams& P, int k0, int nb, int pc, unsigned& epoch, z_t* Ps, z_t* s_prow,
                                z_t* s_rowj, double* rv, int* ri, int& s_piv, int& s_idx, double& s_val) {
  const int n = P.n, np = P.npan, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t lda = P.lda;
  z_t* A = P.A;
  const int kend = k0 + nb;
  const int rpc = (n - k0 + np - 1) / np;
  const int plo = k0 + pc * rpc, phi = min(n, plo + rpc), pn = max(0, phi - plo);
  constexpr int LP = NB + 1;
  for (int e = tid; e < pn * nb; e += NT) {
    const int i = e / nb, t = e - i * nb;
    Ps[i * LP + t] = __ldcg(A + (int64_t)(plo + i) * lda + k0 + t);
  }
  __syncthreads();
  for (int j = k0; j < kend; ++j) {
    const int buf = j & 1, jj = j - k0;
    double v = -1.0;
    int pi = 0x7fffffff;
    for (int i = max(plo, j) + tid; i < phi; i += NT) {
      const double a = zabs1(Ps[(i - plo) * LP + jj]);
      if (a > v) { v = a; pi = i; }
    }
    warp_argmax(v, pi);
    if (lane == 0) { rv[warp] = v; ri[warp] = pi; }
    __syncthreads();
    if (warp == 0) {
      v = lane < NT / 32 ? rv[lane] : -1.0;
      pi = lane < NT / 32 ? ri[lane] : 0x7fffffff;
      warp_argmax(v, pi);
      if (lane == 0) { s_val = v; s_idx = pi; }
    }
    __syncthreads();
    if (tid == 0) {
      P.pval[buf * np + pc] = s_val;
      P.pidx[buf * np + pc] = s_idx;
    }
    if (s_val >= 0.0)
      for (int t = tid; t < nb; t += NT) P.prow[((int64_t)buf * np + pc) * NB + t] = Ps[(s_idx - plo) * LP + t];
    if (j >= plo && j < phi)
      for (int t = tid; t < nb; t += NT) P.rowj[buf * NB + t] = Ps[(j - plo) * LP + t];
    panel_barrier(P.bar, ++epoch * (unsigned)np);
    if (warp == 0) {
      double bv = -1.0;
      int bi = 0x7fffffff, bc = 0;
      for (int q = lane; q < np; q += 32) {
        const double pv = __ldcg(P.pval + buf * np + q);
        const int px = __ldcg(P.pidx + buf * np + q);
        if (pv > bv || (pv == bv && px < bi)) { bv = pv; bi = px; bc = q; }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        const int oc = __shfl_xor_sync(0xffffffffu, bc, o);
        if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; bc = oc; }
      }
      if (lane == 0) {
        s_val = bv;
        s_piv = bv > 0.0 ? bi : -1;
        s_idx = bc;
      }
    }
    __syncthreads();
    const int p = s_piv;
    if (p < 0) {  // exactly singular column (LAPACK: INFO = j+1, no interchange)
      if (pc == 0 && tid == 0) {
        if (*P.info == 0) *P.info = j + 1;
        P.ipiv[j] = j;
      }
      __syncthreads();
      continue;
    }
    for (int t = tid; t < nb; t += NT) {
      s_prow[t] = __ldcg(P.prow + ((int64_t)buf * np + s_idx) * NB + t);
      s_rowj[t] = __ldcg(P.rowj + buf * NB + t);
    }
    VB_DCHECK(p >= j && p < n && s_idx >= 0 && s_idx < np);
    if (pc == 0 && tid == 0) P.ipiv[j] = p;
    __syncthreads();
    const z_t pinv = zrecip(s_prow[jj]);
    if (p != j && j >= plo && j < phi)
      for (int t = tid; t < nb; t += NT) Ps[(j - plo) * LP + t] = s_prow[t];
    const int r0 = max(plo, j + 1);
    const int nrows = phi - r0, ncols = nb - jj - 1;
    if (nrows > 0) {
      for (int i = r0 + tid; i < phi; i += NT) {
        const z_t aij = (i == p) ? s_rowj[jj] : Ps[(i - plo) * LP + jj];
        Ps[(i - plo) * LP + jj] = zmul(aij, pinv);
      }
      if (p != j && p >= r0 && p < phi)
        for (int t = tid; t < nb; t += NT)
          if (t != jj) Ps[(p - plo) * LP + t] = s_rowj[t];
      __syncthreads();
      if (ncols > 0)
        for (int e = tid; e < nrows * ncols; e += NT) {
          const int ii = e / ncols, t = jj + 1 + (e - ii * ncols);
          z_t* row = Ps + (r0 - plo + ii) * LP;
          row[t] = zfms(row[t], row[jj], s_prow[t]);
        }
    }
    __syncthreads();
  }
  for (int e = tid; e < pn * nb; e += NT) {
    const int i = e / nb, t = e - i * nb;
    A[(int64_t)(plo + i) * lda + k0 + t] = Ps[i * LP + t];
  }
  __threadfence();
}

__global__ void __launch_bounds__(NT, 1) zgetrf_la_kernel(const __grid_constant__ LuParams P) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(1024) char smem_raw[];
  double2* smem = (double2*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ GemmT::Bars bars;
  __shared__ z_t s_prow[NB];
  __shared__ z_t s_rowj[NB];
  __shared__ double rv[NT / 32];
  __shared__ int ri[NT / 32];
  __shared__ int s_piv, s_idx;
  __shared__ double s_val;
  const int n = P.n, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int G = gridDim.x, c = blockIdx.x, np = P.npan;
  const bool pan = c < np;
  const int64_t lda = P.lda;
  z_t* A = P.A;
  unsigned epoch = 0;
  if (c == 0 && tid == 0) *P.info = 0;
  grid.sync();
  if (pan) la_factor_panel(P, 0, min(NB, n), c, epoch, smem, s_prow, s_rowj, rv, ri, s_piv, s_idx, s_val);
  for (int k0 = 0; k0 < n; k0 += NB) {
    const int nb = min(NB, n - k0), kend = k0 + nb;
    grid.sync();  // panel k factored and written back; the previous trailing update done
    // ------------------------------------------------ swaps + TRSM
    // each U12 strip applies panel k's interchanges to its own columns first
    // (whole column: rows j in the panel and their pivot rows below), so no
    // separate swap phase and grid barrier; the columns left of the panel
    // (finished L factors) are swapped off the critical path by the GEMM CTAs
    {
      z_t* Li = smem;
      z_t* Bs = smem + NB * LDL;
      const int nblk = k0 / NB;
      const int nstrips = (n - kend + TRS_N - 1) / TRS_N;
      if (nstrips > c || c == 0) {
        load_diag_block<true>(A, lda, k0, nb, Li);
        if (c == 0)
          for (int e = tid; e < NB * NB; e += NT) P.Linv[(int64_t)nblk * NB * NB + e] = Li[(e / NB) * LDL + e % NB];
        const int wm = warp >> 1, wn = warp & 1;
        for (int st = c; st < nstrips; st += G) {
          const int cs = kend + st * TRS_N, ncol = min(TRS_N, n - cs);
          for (int col = cs + tid; col < cs + ncol; col += NT)
            for (int j = k0; j < kend; ++j) {
              const int p = __ldcg(P.ipiv + j);
              if (p != j) {
                const z_t t = __ldcg(A + (int64_t)j * lda + col);
                A[(int64_t)j * lda + col] = __ldcg(A + (int64_t)p * lda + col);
                A[(int64_t)p * lda + col] = t;
              }
            }
          __syncthreads();
          for (int e = tid; e < NB * TRS_N; e += NT) {
            const int i = e / TRS_N, jx = e - i * TRS_N;
            Bs[i * LDS_B + jx] = (i < nb && jx < ncol) ? __ldcg(A + (int64_t)(k0 + i) * lda + cs + jx) : zmake(0.0, 0.0);
          }
          __syncthreads();
          double cr[2][2][2], ci[2][2][2];
#pragma unroll
          for (int a = 0; a < 2; ++a)
#pragma unroll
            for (int b = 0; b < 2; ++b) cr[a][b][0] = cr[a][b][1] = ci[a][b][0] = ci[a][b][1] = 0.0;
          blk::warp_cmma<2, 2, false>(cr, ci, Li + (wm * 16) * LDL, LDL, Bs + wn * 16, LDS_B, (nb + 3) >> 2);
#pragma unroll
          for (int a = 0; a < 2; ++a)
#pragma unroll
            for (int b = 0; b < 2; ++b)
#pragma unroll
              for (int vv = 0; vv < 2; ++vv) {
                const int row = wm * 16 + a * 8 + (lane >> 2);
                const int col = wn * 16 + b * 8 + 2 * (lane & 3) + vv;
                if (row < nb && col < ncol) A[(int64_t)(k0 + row) * lda + cs + col] = zmake(cr[a][b][vv], ci[a][b][vv]);
              }
          __syncthreads();
        }
      }
      if (c == (G > 1 ? 1 : 0)) {
        __syncthreads();
        load_diag_block<false>(A, lda, k0, nb, Li);
        for (int e = tid; e < NB * NB; e += NT) P.Uinv[(int64_t)nblk * NB * NB + e] = Li[(e / NB) * LDL + e % NB];
      }
    }
    grid.sync();
    if (kend >= n) {  // last panel: its interchanges on the L columns left of it, by everyone
      for (int64_t col = (int64_t)c * NT + tid; col < k0; col += (int64_t)G * NT)
        for (int j = k0; j < kend; ++j) {
          const int p = __ldcg(P.ipiv + j);
          if (p != j) {
            const z_t t = __ldcg(A + (int64_t)j * lda + col);
            A[(int64_t)j * lda + col] = __ldcg(A + (int64_t)p * lda + col);
            A[(int64_t)p * lda + col] = t;
          }
        }
      break;
    }
    // ------------------------------------------------ look-ahead update
    const int nbn = min(NB, n - kend);
    GemmT::run(&P.maps, A, lda, kend, k0, k0, kend, n - kend, nbn, nb, (char*)smem, &bars, c, G);
    grid.sync();
    // ------------------------- panel k+1 (panel CTAs) || A22 update (GEMM CTAs)
    if (pan) {
      la_factor_panel(P, kend, nbn, c, epoch, smem, s_prow, s_rowj, rv, ri, s_piv, s_idx, s_val);
    } else {
      if (kend + nbn < n)
        GemmT::run(&P.maps, A, lda, kend, k0, k0, kend + nbn, n - kend, n - kend - nbn, nb, (char*)smem, &bars,
                   c - np, G - np);
      // panel k's interchanges on the finished L columns [0, k0)
      for (int64_t col = (int64_t)(c - np) * NT + tid; col < k0; col += (int64_t)(G - np) * NT)
        for (int j = k0; j < kend; ++j) {
          const int p = __ldcg(P.ipiv + j);
          if (p != j) {
            const z_t t = __ldcg(A + (int64_t)j * lda + col);
            A[(int64_t)j * lda + col] = __ldcg(A + (int64_t)p * lda + col);
            A[(int64_t)p * lda + col] = t;
          }
        }
    }
  }
  grid.sync();
  if (c == 0) {
    for (int i = tid; i < n; i += NT) P.perm[i] = i;
    __syncthreads();
    if (tid == 0)
      for (int j = 0; j < n; ++j) {
        const int p = P.ipiv[j];
        if (p != j) {
          const int t = P.perm[j];
          P.perm[j] = P.perm[p];
          P.perm[p] = t;
        }
      }
  }
}

// ---------------------------------------------------------------- solve ---
struct SolveParams {
  int n, nrhs;
  const z_t* LU;
  int64_t lda;
  const int* perm;
  const z_t* Linv;
  const z_t* Uinv;
  const z_t* B;   // input RHS (may alias X)
  int64_t ldb;
  z_t* X;         // output / work, n x nrhs
  int64_t ldx;
  z_t* tmp;       // n x nrhs scratch for the permuted RHS when B aliases X
};

// T[i, :] -= M[i, k0 : k0+nb] yb for rows i in [i0, i0 + nrows) (T row stride
// ldt): KS threads per (row, rhs) item split k mod KS with their loads in
// flight in batches of 16, then a fixed-order shuffle reduction — instead of
// one thread per item walking a 64-long chain of dependent-latency loads.
template <int KS>
__device__ __forceinline__ void rows_update_ks(const SolveParams& S, z_t* T, int64_t ldt, int i0, int nrows, int k0,
                                               int nb, const z_t* yb) {
  const int s = S.nrhs, tid = threadIdx.x, kq = tid % KS;
  const int nitems = nrows * s;
  for (int base = 0; base < nitems; base += NT / KS) {
    const int e = base + tid / KS;
    const bool valid = e < nitems;
    const int i = i0 + (valid ? e / s : 0), r = valid ? e % s : 0;
    const z_t* Mrow = S.LU + (int64_t)i * S.lda + k0;
    constexpr int NM = 64 / KS, CH = NM < 16 ? NM : 16;
    z_t acc = zmake(0.0, 0.0);
#pragma unroll
    for (int m0 = 0; m0 < NM; m0 += CH) {
      z_t l[CH];
#pragma unroll
      for (int m = 0; m < CH; ++m) {
        const int k = kq + KS * (m0 + m);
        l[m] = (valid && k < nb) ? Mrow[k] : zmake(0.0, 0.0);
      }
#pragma unroll
      for (int m = 0; m < CH; ++m) {
        const int k = kq + KS * (m0 + m);
        if (k < nb) acc = zfma(acc, l[m], yb[k * s + r]);
      }
    }
#pragma unroll
    for (int o = 1; o < KS; o <<= 1) {
      acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
      acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
    }
    if (valid && kq == 0) {  // T rows may have been written by another CTA (X = P B): read from L2
      z_t* tp = T + (int64_t)i * ldt + r;
      *tp = zsub(__ldcg(tp), acc);
    }
  }
}

__device__ __forceinline__ void rows_update(const SolveParams& S, z_t* T, int64_t ldt, int i0, int nrows, int k0,
                                            int nb, const z_t* yb) {
  if (nrows <= 0) return;
  // the split depends on the RHS count only, so the summation order (and the
  // result) does not depend on the grid size (vb_set_lu_max_ctas)
  const int s = S.nrhs;
  if (s == 1) rows_update_ks<8>(S, T, ldt, i0, nrows, k0, nb, yb);
  else if (s == 2) rows_update_ks<4>(S, T, ldt, i0, nrows, k0, nb, yb);
  else if (s <= 4) rows_update_ks<2>(S, T, ldt, i0, nrows, k0, nb, yb);
  else
    for (int64_t e = threadIdx.x; e < (int64_t)nrows * s; e += NT) {  // many items: one thread each
      const int i = i0 + (int)(e / s), r = (int)(e % s);
      z_t acc = __ldcg(T + (int64_t)i * ldt + r);
      const z_t* Mrow = S.LU + (int64_t)i * S.lda + k0;
      for (int k = 0; k < nb; ++k) acc = zfms(acc, Mrow[k], yb[k * s + r]);
      T[(int64_t)i * ldt + r] = acc;
    }
}

// One right-hand side: y = T yb for the diagonal block with 4 lanes per row
// (k split mod 4, fixed-order shuffle reduction); true on the lane that holds
// row tid/4's value.
template <bool LOWER>
__device__ __forceinline__ bool diag_mult_s1(const z_t* Ti, const z_t* yb, int nb, z_t& out) {
  const int i = threadIdx.x >> 2, kq = threadIdx.x & 3;
  z_t acc = zmake(0.0, 0.0);
  if (i < nb) {
#pragma unroll
    for (int m = 0; m < NB / 4; ++m) {
      const int k = kq + 4 * m;
      if (k < nb && (LOWER ? k <= i : k >= i)) acc = zfma(acc, Ti[i * (NB + 1) + k], yb[k]);
    }
  }
#pragma unroll
  for (int o = 1; o < 4; o <<= 1) {
    acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
    acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
  }
  out = acc;
  return kq == 0 && i < nb;
}

constexpr int MAXRHS = 16;

__global__ void __launch_bounds__(NT, 1) zgetrs_kernel(SolveParams S) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ double2 smem_s[];
  z_t* Ti = smem_s;                 // NB x (NB+1)
  z_t* yb = smem_s + NB * (NB + 1);  // NB x MAXRHS
  const int n = S.n, s = S.nrhs, tid = threadIdx.x;
  const int G = gridDim.x, c = blockIdx.x;
  int lo, hi;
  row_range(n, lo, hi);
  // X = P B
  for (int64_t e = (int64_t)c * NT + tid; e < (int64_t)n * s; e += (int64_t)G * NT) {
    const int i = (int)(e / s), q = (int)(e - (int64_t)i * s);
    S.tmp[(int64_t)i * s + q] = S.B[(int64_t)S.perm[i] * S.ldb + q];
  }
  grid.sync();
  for (int64_t e = (int64_t)c * NT + tid; e < (int64_t)n * s; e += (int64_t)G * NT) {
    const int i = (int)(e / s), q = (int)(e - (int64_t)i * s);
    S.X[(int64_t)i * S.ldx + q] = __ldcg(S.tmp + (int64_t)i * s + q);
  }
  grid.sync();
  const int nblk = (n + NB - 1) / NB;
  // forward: L y = P b, right-looking by diagonal blocks
  for (int kb = 0; kb < nblk; ++kb) {
    const int k0 = kb * NB, nb = min(NB, n - k0), kend = k0 + nb;
    for (int e = tid; e < NB * NB; e += NT) Ti[(e / NB) * (NB + 1) + e % NB] = __ldcg(S.Linv + (int64_t)kb * NB * NB + e);
    for (int e = tid; e < nb * s; e += NT) yb[e] = __ldcg(S.X + (int64_t)(k0 + e / s) * S.ldx + e % s);
    __syncthreads();
    // y_kb = Linv * b_kb (every CTA redundantly; the owner writes it back).
    // y goes to tmp, not back into X: other CTAs may still be loading this
    // block's b from X (no barrier between their load and this store).
    if (s == 1) {
      z_t v;
      const bool mine = diag_mult_s1<true>(Ti, yb, nb, v);
      __syncthreads();
      if (mine) {
        const int i = tid >> 2;
        yb[i] = v;
        if (k0 + i >= lo && k0 + i < hi) S.tmp[k0 + i] = v;
      }
    } else {
      z_t yv[(NB * MAXRHS + NT - 1) / NT];
#pragma unroll
      for (int q = 0; q < (NB * MAXRHS + NT - 1) / NT; ++q) {
        const int e = tid + q * NT;
        yv[q] = zmake(0.0, 0.0);
        if (e < nb * s) {
          const int i = e / s, r = e - i * s;
          z_t acc = zmake(0.0, 0.0);
          for (int k = 0; k <= i; ++k) acc = zfma(acc, Ti[i * (NB + 1) + k], yb[k * s + r]);
          yv[q] = acc;
        }
      }
      __syncthreads();
#pragma unroll
      for (int q = 0; q < (NB * MAXRHS + NT - 1) / NT; ++q) {
        const int e = tid + q * NT;
        if (e < nb * s) {
          yb[e] = yv[q];
          const int i = k0 + e / s;
          if (i >= lo && i < hi) S.tmp[(int64_t)i * s + e % s] = yv[q];
        }
      }
    }
    __syncthreads();
    // own rows below the block: b_i -= L[i, k0:kend] y_kb
    rows_update(S, S.X, S.ldx, max(lo, kend), hi - max(lo, kend), k0, nb, yb);
    grid.sync();
  }
  // backward: U x = y
  for (int kb = nblk - 1; kb >= 0; --kb) {
    const int k0 = kb * NB, nb = min(NB, n - k0);
    for (int e = tid; e < NB * NB; e += NT) Ti[(e / NB) * (NB + 1) + e % NB] = __ldcg(S.Uinv + (int64_t)kb * NB * NB + e);
    for (int e = tid; e < nb * s; e += NT) yb[e] = __ldcg(S.tmp + (int64_t)(k0 + e / s) * s + e % s);
    __syncthreads();
    if (s == 1) {
      z_t v;
      const bool mine = diag_mult_s1<false>(Ti, yb, nb, v);
      __syncthreads();
      if (mine) {
        const int i = tid >> 2;
        yb[i] = v;
        if (k0 + i >= lo && k0 + i < hi) S.X[(int64_t)(k0 + i) * S.ldx] = v;
      }
    } else {
      z_t yv[(NB * MAXRHS + NT - 1) / NT];
#pragma unroll
      for (int q = 0; q < (NB * MAXRHS + NT - 1) / NT; ++q) {
        const int e = tid + q * NT;
        yv[q] = zmake(0.0, 0.0);
        if (e < nb * s) {
          const int i = e / s, r = e - i * s;
          z_t acc = zmake(0.0, 0.0);
          for (int k = i; k < nb; ++k) acc = zfma(acc, Ti[i * (NB + 1) + k], yb[k * s + r]);
          yv[q] = acc;
        }
      }
      __syncthreads();
#pragma unroll
      for (int q = 0; q < (NB * MAXRHS + NT - 1) / NT; ++q) {
        const int e = tid + q * NT;
        if (e < nb * s) {
          yb[e] = yv[q];
          const int i = k0 + e / s;
          if (i >= lo && i < hi) S.X[(int64_t)i * S.ldx + e % s] = yv[q];
        }
      }
    }
    __syncthreads();
    // own rows above the block (still y - updates, in tmp): y_i -= U[i, k0:kend] x_kb
    rows_update(S, S.tmp, s, lo, min(hi, k0) - lo, k0, nb, yb);
    grid.sync();
  }
}

constexpr size_t SOLVE_SMEM = (size_t)(NB * (NB + 1) + NB * MAXRHS) * sizeof(z_t);

// Per host thread: at most this many CTAs for the whole-GPU factor/solve
// kernels (0 = all SMs).  Independent factorisations / solves driven from
// several host threads on their own streams then share the GPU: the solves
// are latency-bound (1.26 ms at n = 3,565 on 148 CTAs, 1.29 ms on 64).
static thread_local int t_max_ctas = 0;

static int coop_grid(const void* kern, size_t smem, int* grid, int min_grid = 0) {
  int dev = 0, nsm = 0, per = 0, coop = 0;
  VB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  VB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                               (int)cudaSharedmemCarveoutMaxShared));
  VB_CUDA(cudaGetDevice(&dev));
  VB_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  VB_CUDA(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev));
  if (!coop) {
    set_error("device does not support cooperative launches");
    return 2;
  }
  VB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, NT, smem));
  if (per < 1) {
    set_error("zgetrf/zgetrs kernel does not fit on an SM");
    return 2;
  }
  *grid = nsm;  // one CTA per SM
  if (t_max_ctas > 0 && t_max_ctas < *grid) *grid = t_max_ctas;  // a share of the GPU (concurrent solves)
  if (*grid < min_grid) *grid = min_grid < nsm ? min_grid : nsm;   // ... but never fewer CTAs than n needs
  return 0;
}

}  // namespace lu

void set_lu_max_ctas(int n) { lu::t_max_ctas = n > 0 ? n : 0; }

int lu_debug_cycles(unsigned long long* out, int reset) {
  VB_CUDA(cudaMemcpyFromSymbol(out, lu::g_lu_cycles, 4 * sizeof(unsigned long long)));
  if (reset) {
    unsigned long long z[4] = {};
    VB_CUDA(cudaMemcpyToSymbol(lu::g_lu_cycles, z, sizeof(z)));
  }
  return 0;
}

size_t zgetrf_workspace_bytes(int n) {
  int grid = 148, dev = 0;  // one CTA per SM (see coop_grid; no attribute side effects here)
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&grid, cudaDevAttrMultiProcessorCount, dev);
  const int nblk = (n + lu::NB - 1) / lu::NB;
  size_t b = 0;
  b += 2 * (size_t)grid * sizeof(double);
  b += 2 * (size_t)grid * sizeof(int);
  b += 2 * (size_t)grid * lu::NB * sizeof(z_t);
  b += 2 * (size_t)lu::NB * sizeof(z_t);
  b += 2 * (size_t)nblk * lu::NB * lu::NB * sizeof(z_t);
  return b + 1024 + 256;  // + the look-ahead kernel's panel barrier counter
}

// Factor data kept for the solves: Linv/Uinv of the diagonal blocks and the
// permutation live in `factor_aux` (layout below), so a factorisation is
// (A overwritten by L\U, ipiv, aux).
size_t zgetrf_aux_bytes(int n) {
  const int nblk = (n + lu::NB - 1) / lu::NB;
  return 2 * (size_t)nblk * lu::NB * lu::NB * sizeof(z_t) + (size_t)n * sizeof(int) + 256;
}

static int zgetrf_la(int n, z_t* A, int64_t lda, int* ipiv, int* info_dev, void* aux, size_t aux_bytes, void* work,
                     size_t work_bytes, cudaStream_t st, int np) {
  const size_t prow_bytes = (size_t)((n + np - 1) / np) * (lu::NB + 1) * sizeof(z_t) + 1024;
  const size_t smem = prow_bytes > lu::LU_SMEM ? prow_bytes : lu::LU_SMEM;
  VB_CHECK_ARG(smem <= 227 * 1024, "vb_zgetrf: n too large for the look-ahead panel rows");
  int grid = 0;
  if (int rc = lu::coop_grid((const void*)lu::zgetrf_la_kernel, smem, &grid)) return rc;
  VB_CHECK_ARG(np < grid, "vb_zgetrf: too few CTAs for the look-ahead split");
  const int nblk = (n + lu::NB - 1) / lu::NB;
  VB_CHECK_ARG(work && work_bytes >= zgetrf_workspace_bytes(n), "vb_zgetrf: workspace too small");
  lu::LuParams P;
  P.n = n; P.A = A; P.lda = lda; P.ipiv = ipiv; P.info = info_dev; P.npan = np;
  char* w = (char*)work;
  P.pval = (double*)w; w += 2 * (size_t)grid * sizeof(double);
  P.pidx = (int*)w; w += 2 * (size_t)grid * sizeof(int);
  w = (char*)(((uintptr_t)w + 255) & ~(uintptr_t)255);
  P.prow = (z_t*)w; w += 2 * (size_t)grid * lu::NB * sizeof(z_t);
  P.rowj = (z_t*)w; w += 2 * (size_t)lu::NB * sizeof(z_t);
  w = (char*)(((uintptr_t)w + 255) & ~(uintptr_t)255);
  P.bar = (unsigned*)w;
  VB_CUDA(cudaMemsetAsync(P.bar, 0, sizeof(unsigned), st));
  char* x = (char*)aux;
  P.Linv = (z_t*)x; x += (size_t)nblk * lu::NB * lu::NB * sizeof(z_t);
  P.Uinv = (z_t*)x; x += (size_t)nblk * lu::NB * lu::NB * sizeof(z_t);
  P.perm = (int*)x;
  {
    const cuuint64_t dims[3] = {(cuuint64_t)2 * lda, (cuuint64_t)n, 1};
    const cuuint64_t strides[2] = {(cuuint64_t)lda * 16, (cuuint64_t)lda * 16 * n};
    const cuuint32_t box64[3] = {16, 64, 1}, box8[3] = {16, 8, 1}, es[3] = {1, 1, 1};
    if (int rc = tma_encode_map(&P.maps.a64, A, dims, strides, box64, es)) return rc;
    if (int rc = tma_encode_map(&P.maps.b8, A, dims, strides, box8, es)) return rc;
  }
  void* args[] = {&P};
  VB_CUDA(cudaLaunchCooperativeKernel((const void*)lu::zgetrf_la_kernel, grid, lu::NT, args, smem, st));
  VB_LAUNCHED("zgetrf_la_kernel");
  return 0;
}

static int g_lu_lookahead = -1;  // -1: VB_LU_LOOKAHEAD env (default on), 0 off, 1 on
void set_lu_lookahead(int on) { g_lu_lookahead = on; }

// Panel CTAs of the look-ahead kernel for order n (0: use the plain kernel):
// the panel rows [k0, n) split over them must fit shared memory, and they
// must leave most of the grid to the trailing update.
static int la_panel_ctas(int n, int grid) {
  if (g_lu_lookahead < 0) {
    const char* e = getenv("VB_LU_LOOKAHEAD");
    g_lu_lookahead = e ? atoi(e) : 1;
  }
  if (!g_lu_lookahead || grid < 48) return 0;
  // panel rows per panel CTA: 150 where that many panel CTAs still leave two
  // thirds of the grid to the trailing update (n = 3,561: 22.0 -> 20.7 ms,
  // n = 4,641: 27.9 -> 27.2 ms), else 200 (the shared-memory row limit is ~220)
  for (const int rows_max : {150, 200}) {
    int np = (n + rows_max - 1) / rows_max;
    if (np < 16) np = 16;
    if (np <= grid / 3) return np;
  }
  return 0;
}

int zgetrf(int n, z_t* A, int64_t lda, int* ipiv, int* info_dev, void* aux, size_t aux_bytes, void* work,
           size_t work_bytes, cudaStream_t st) {
  VB_CHECK_ARG(n > 0 && lda >= n, "vb_zgetrf: bad sizes");
  VB_CHECK_ARG(aux && aux_bytes >= zgetrf_aux_bytes(n), "vb_zgetrf: aux too small");
  {
    int gfull = 0;
    if (int rc = lu::coop_grid((const void*)lu::zgetrf_la_kernel, lu::LU_SMEM, &gfull)) return rc;
    const int np = la_panel_ctas(n, gfull);
    if (np > 0) return zgetrf_la(n, A, lda, ipiv, info_dev, aux, aux_bytes, work, work_bytes, st, np);
  }
  int grid = 0;
  // each CTA keeps its panel rows in shared memory: at least this many CTAs
  const int rows_max = (int)((227 * 1024 - 2048) / ((lu::NB + 1) * sizeof(z_t)));
  const int min_grid = (n + rows_max - 1) / rows_max;
  if (int rc = lu::coop_grid((const void*)lu::zgetrf_kernel, lu::LU_SMEM, &grid, min_grid)) return rc;
  const size_t smem = lu::lu_smem(n, grid);
  VB_CHECK_ARG(smem <= 227 * 1024, "vb_zgetrf: n too large for the shared-memory panel rows");
  if (int rc = lu::coop_grid((const void*)lu::zgetrf_kernel, smem, &grid, min_grid)) return rc;
  const int nblk = (n + lu::NB - 1) / lu::NB;
  VB_CHECK_ARG(work && work_bytes >= zgetrf_workspace_bytes(n), "vb_zgetrf: workspace too small");
  lu::LuParams P;
  P.n = n; P.A = A; P.lda = lda; P.ipiv = ipiv; P.info = info_dev;
  char* w = (char*)work;
  P.pval = (double*)w; w += 2 * (size_t)grid * sizeof(double);
  P.pidx = (int*)w; w += 2 * (size_t)grid * sizeof(int);
  w = (char*)(((uintptr_t)w + 255) & ~(uintptr_t)255);
  P.prow = (z_t*)w; w += 2 * (size_t)grid * lu::NB * sizeof(z_t);
  P.rowj = (z_t*)w; w += 2 * (size_t)lu::NB * sizeof(z_t);
  char* x = (char*)aux;
  P.Linv = (z_t*)x; x += (size_t)nblk * lu::NB * lu::NB * sizeof(z_t);
  P.Uinv = (z_t*)x; x += (size_t)nblk * lu::NB * lu::NB * sizeof(z_t);
  P.perm = (int*)x;
  {
    const cuuint64_t dims[3] = {(cuuint64_t)2 * lda, (cuuint64_t)n, 1};
    const cuuint64_t strides[2] = {(cuuint64_t)lda * 16, (cuuint64_t)lda * 16 * n};
    const cuuint32_t box64[3] = {16, 64, 1}, box8[3] = {16, 8, 1}, es[3] = {1, 1, 1};
    if (int rc = tma_encode_map(&P.maps.a64, A, dims, strides, box64, es)) return rc;
    if (int rc = tma_encode_map(&P.maps.b8, A, dims, strides, box8, es)) return rc;
  }
  void* args[] = {&P};
  {
    cudaError_t e = cudaLaunchCooperativeKernel((const void*)lu::zgetrf_kernel, grid, lu::NT, args, smem, st);
    if (e != cudaSuccess) {
      int per = -1;
      cudaFuncAttributes fa;
      cudaFuncGetAttributes(&fa, (const void*)lu::zgetrf_kernel);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, lu::zgetrf_kernel, lu::NT, smem);
      set_error(std::string("vb_zgetrf launch: ") + cudaGetErrorString(e) + " (grid " + std::to_string(grid) +
                ", dyn smem " + std::to_string(smem) + ", static " + std::to_string(fa.sharedSizeBytes) +
                ", max dyn " + std::to_string(fa.maxDynamicSharedSizeBytes) + ", regs " +
                std::to_string(fa.numRegs) + ", blocks/SM " + std::to_string(per) + ")");
      return 2;
    }
  }
  VB_LAUNCHED("zgetrf_kernel");
  return 0;
}

int zgetrs(int n, int nrhs, const z_t* LU, int64_t lda, const void* aux, const z_t* B, int64_t ldb,
           z_t* X, int64_t ldx, void* work, size_t work_bytes, cudaStream_t st) {
  VB_CHECK_ARG(n > 0 && nrhs >= 1 && nrhs <= lu::MAXRHS, "vb_zgetrs: 1 <= nrhs <= 16");
  VB_CHECK_ARG(work && work_bytes >= (size_t)n * nrhs * sizeof(z_t), "vb_zgetrs: workspace too small");
  int grid = 0;
  if (int rc = lu::coop_grid((const void*)lu::zgetrs_kernel, lu::SOLVE_SMEM, &grid)) return rc;
  const int nblk = (n + lu::NB - 1) / lu::NB;
  lu::SolveParams S;
  S.n = n; S.nrhs = nrhs; S.LU = LU; S.lda = lda;
  const char* x = (const char*)aux;
  S.Linv = (const z_t*)x; x += (size_t)nblk * lu::NB * lu::NB * sizeof(z_t);
  S.Uinv = (const z_t*)x; x += (size_t)nblk * lu::NB * lu::NB * sizeof(z_t);
  S.perm = (const int*)x;
  S.B = B; S.ldb = ldb; S.X = X; S.ldx = ldx; S.tmp = (z_t*)work;
  void* args[] = {&S};
  VB_CUDA(cudaLaunchCooperativeKernel((const void*)lu::zgetrs_kernel, grid, lu::NT, args, lu::SOLVE_SMEM, st));
  VB_LAUNCHED("zgetrs_kernel");
  return 0;
}

}  // namespace vb
