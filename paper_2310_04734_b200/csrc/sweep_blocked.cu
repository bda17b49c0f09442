// Reduced frequency sweep, blocked path for large reduced orders (r >~ 100:
// cfg5 r = 256/1024/2048, cfg3 r = 400).  Same contract as the shared-memory
// path (sweep_small.cu), i.e. per frequency f:
//   mor.py:73-90   A_r(f) = sum_k alpha_k(f) P_k
//   mor.py:94      numpy.linalg.solve = LAPACK zgesv (partial pivoting, izamax)
//   mor.py:96-102  y = (c_out V) x_r ;  solvers.py:334-338 mean_spl per RHS
//
// Design: a persistent kernel, ONE CTA PER FREQUENCY (grid =
// #SMs), each CTA owning a private r x (r+s) augmented matrix [A | B] in a
// global-memory workspace.  Right-looking blocked LU with outer panels of
// NB = 64 columns:
//   1. inner panels of w columns are factored in shared memory (izamax pivot
//      search as a block argmax), then fold into the rest of the outer panel
//      with a rank-w update;
//   2. the NB row interchanges are applied to the columns right of the panel;
//   3. U12 = L11^-1 A12 with L11^-1 formed explicitly in shared memory and
//      applied as a complex GEMM;
//   4. A22 -= L21 U12 — the dominant flops — as complex GEMM tiles on the FP64
//      tensor cores (mma.sync.m8n8k4.f64 = DMMA; there is no f64 tcgen05 kind),
//      4 real MMAs per complex product, operands staged through shared memory
//      with cp.async double buffering.
// B rides along as extra columns, so L is applied to it by the factorisation;
// a blocked back substitution, the output map and the SPL reduction finish
// the frequency in the same kernel.
#include "common.cuh"
#include "sweep.cuh"

namespace vb {
namespace blk {

constexpr int NT = 256;  // threads per CTA (8 warps)
constexpr int NB = 64;   // outer panel width
constexpr int KC = 16;   // complex k-chunk per shared-memory stage

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1},{%2},{%3},{%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool pred) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  int n = pred ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(n));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// Warp-level complex MMA on shared-memory operands, 8x8 fragments:
// acc (FM x FN fragments of the warp tile) += sign * A(rows) * B(cols) over
// `k4` steps of 4.  A: row-major [m][k] with leading dim lda (complex),
// B: row-major [k][n] with leading dim ldb.  Fragment layouts of
// mma.m8n8k4.row.col.f64: A[lane/4][lane%4], B[k=lane%4][n=lane/4],
// C[lane/4][2*(lane%4)+v].
template <int FM, int FN, bool NEG>
__device__ __forceinline__ void warp_cmma(double (&cr)[FM][FN][2], double (&ci)[FM][FN][2],
                                          const z_t* as, int lda, const z_t* bs, int ldb,
                                          int k4) {
  const int lane = threadIdx.x & 31;
  const int ar = lane >> 2, ak = lane & 3;
#pragma unroll 2
  for (int kk = 0; kk < k4; ++kk) {
    z_t a[FM], b[FN];
#pragma unroll
    for (int i = 0; i < FM; ++i) a[i] = as[(i * 8 + ar) * lda + kk * 4 + ak];
#pragma unroll
    for (int j = 0; j < FN; ++j) b[j] = bs[(kk * 4 + ak) * ldb + j * 8 + ar];
#pragma unroll
    for (int j = 0; j < FN; ++j) {
      // C -= A B :  Cr += ar(-br) + ai(bi) ; Ci += ar(-bi) + ai(-br)
      // C += A B :  Cr += ar(br) + ai(-bi) ; Ci += ar(bi) + ai(br)
      const double br = NEG ? -b[j].x : b[j].x;
      const double bi = NEG ? -b[j].y : b[j].y;
      const double nbi = -bi;
#pragma unroll
      for (int i = 0; i < FM; ++i) {
        dmma(cr[i][j][0], cr[i][j][1], a[i].x, br);
        dmma(cr[i][j][0], cr[i][j][1], a[i].y, nbi);
        dmma(ci[i][j][0], ci[i][j][1], a[i].x, bi);
        dmma(ci[i][j][0], ci[i][j][1], a[i].y, br);
      }
    }
  }
}

// CTA-wide C[M x N] -= A[M x K] * B[K x N] on global (workspace) operands.
// Tiles TM x TN over WM x WN warps.  One flat software pipeline runs over all
// (tile, k-chunk) iterations: A/B chunks stream through a STAGES-deep
// cp.async ring, and the C tile of the next output tile is prefetched into
// shared memory while the current tile computes, so neither the operand nor
// the C-tile latency is exposed at tile boundaries.  Accumulation starts from
// zero; the epilogue writes C_old - A*B.
template <int TM, int TN, int WM, int WN, int STAGES = 3>
struct Gemm {
  static_assert(WM * WN == NT / 32, "warp grid");
  static constexpr int FM = TM / WM / 8, FN = TN / WN / 8;
  static constexpr int LDA = KC + 4;  // == 4 (mod 8): conflict-free 128-bit fragment loads
  static constexpr int LDB = TN + 2;  // == 2 (mod 8)
  static constexpr int LDC = TN + 1;  // == 1 (mod 8): conflict-free epilogue reads
  static constexpr int A_EL = TM * LDA, B_EL = KC * LDB, C_EL = TM * LDC;
  static constexpr size_t SMEM = (size_t)(STAGES * (A_EL + B_EL) + C_EL) * sizeof(z_t);

  __device__ static void load_chunk(z_t* As, z_t* Bs, const z_t* A, int lda, const z_t* B, int ldb,
                                    int M, int N, int K, int m0, int n0, int k0) {
    const int tid = threadIdx.x;
#pragma unroll
    for (int q = 0; q < (TM * KC + NT - 1) / NT; ++q) {
      const int e = tid + q * NT;
      if ((TM * KC) % NT == 0 || e < TM * KC) {
        const int i = e / KC, k = e % KC;
        const bool p = (m0 + i < M) && (k0 + k < K);
        cp_async16(As + i * LDA + k, p ? A + (size_t)(m0 + i) * lda + k0 + k : A, p);
      }
    }
#pragma unroll
    for (int q = 0; q < (KC * TN + NT - 1) / NT; ++q) {
      const int e = tid + q * NT;
      if ((KC * TN) % NT == 0 || e < KC * TN) {
        const int k = e / TN, j = e % TN;
        const bool p = (k0 + k < K) && (n0 + j < N);
        cp_async16(Bs + k * LDB + j, p ? B + (size_t)(k0 + k) * ldb + n0 + j : B, p);
      }
    }
  }

  __device__ static void load_c(z_t* Cs, const z_t* C, int ldc, int M, int N, int m0, int n0) {
    const int tid = threadIdx.x;
#pragma unroll 4
    for (int e = tid; e < TM * TN; e += NT) {
      const int i = e / TN, j = e % TN;
      const bool p = (m0 + i < M) && (n0 + j < N);
      cp_async16(Cs + i * LDC + j, p ? C + (size_t)(m0 + i) * ldc + n0 + j : C, p);
    }
  }

  __device__ static void run(z_t* C, int ldc, const z_t* A, int lda, const z_t* B, int ldb, int M,
                             int N, int K, z_t* smem) {
    if (M <= 0 || N <= 0 || K <= 0) return;
    z_t* As = smem;
    z_t* Bs = smem + STAGES * A_EL;
    z_t* Cs = Bs + STAGES * B_EL;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int wm = warp / WN, wn = warp % WN;
    const int ntn = (N + TN - 1) / TN, nk = (K + KC - 1) / KC;
    const int T = ((M + TM - 1) / TM) * ntn * nk;
    auto issue = [&](int j) {
      if (j < T) {
        const int t = j / nk, kc = j - t * nk;
        load_chunk(As + (j % STAGES) * A_EL, Bs + (j % STAGES) * B_EL, A, lda, B, ldb, M, N, K,
                   (t / ntn) * TM, (t % ntn) * TN, kc * KC);
      }
    };
    load_c(Cs, C, ldc, M, N, 0, 0);
#pragma unroll
    for (int j = 0; j < STAGES - 1; ++j) {
      issue(j);
      cp_commit();
    }
    double cr[FM][FN][2], ci[FM][FN][2];
#pragma unroll
    for (int i = 0; i < FM; ++i)
#pragma unroll
      for (int j = 0; j < FN; ++j) cr[i][j][0] = cr[i][j][1] = ci[i][j][0] = ci[i][j][1] = 0.0;
    for (int it = 0; it < T; ++it) {
      const int t = it / nk, kc = it - t * nk;
      cp_wait<STAGES - 2>();
      __syncthreads();
      issue(it + STAGES - 1);
      if (kc == 0 && it > 0) load_c(Cs, C, ldc, M, N, (t / ntn) * TM, (t % ntn) * TN);
      cp_commit();
      const int st = it % STAGES;
      int k4 = min(KC, K - kc * KC);
      k4 = (k4 + 3) >> 2;
      warp_cmma<FM, FN, false>(cr, ci, As + st * A_EL + (wm * FM * 8) * LDA, LDA,
                               Bs + st * B_EL + wn * FN * 8, LDB, k4);
      if (kc == nk - 1) {
        if (nk < STAGES) {  // the C-tile group may still be in flight
          cp_wait<0>();
          __syncthreads();
        }
        const int m0 = (t / ntn) * TM, n0 = (t % ntn) * TN;
#pragma unroll
        for (int i = 0; i < FM; ++i)
#pragma unroll
          for (int j = 0; j < FN; ++j)
#pragma unroll
            for (int v = 0; v < 2; ++v) {
              const int lr = wm * FM * 8 + i * 8 + (lane >> 2);
              const int lc = wn * FN * 8 + j * 8 + 2 * (lane & 3) + v;
              if (m0 + lr < M && n0 + lc < N) {
                const z_t c = Cs[lr * LDC + lc];
                C[(size_t)(m0 + lr) * ldc + n0 + lc] = zmake(c.x - cr[i][j][v], c.y - ci[i][j][v]);
              }
              cr[i][j][v] = 0.0;
              ci[i][j][v] = 0.0;
            }
      }
    }
    cp_wait<0>();
  }
};

using GemmWide = Gemm<64, 64, 2, 4>;    // trailing updates
using GemmNarrow = Gemm<128, 16, 8, 1>; // back-substitution updates (N = s <= 16)

// Shared-memory layout of the TRSM stage: L11^-1 (NB x LDL) and a B strip.
constexpr int LDL = NB + 4;
constexpr int LDS_B = NB + 2;
constexpr size_t TRSM_SMEM = (size_t)(NB * LDL + NB * LDS_B) * sizeof(z_t);

struct Params {
  int r, nprim, s, n_out;
  int64_t F;
  const z_t* prims;
  const z_t* alpha;
  const z_t* b;
  int64_t b_stride_f;
  const z_t* c_r;
  z_t* y;
  double* spl;
  z_t* x;
  int* info;
  z_t* work;
  int ldw;  // leading dimension of the augmented matrix
  int w;    // inner panel width
};

__device__ __forceinline__ void block_argmax(double& v, int& idx, double* rv, int* ri) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  warp_argmax(v, idx);
  if (lane == 0) { rv[warp] = v; ri[warp] = idx; }
  __syncthreads();
  if (warp == 0) {
    v = lane < NT / 32 ? rv[lane] : -1.0;
    idx = lane < NT / 32 ? ri[lane] : 0x7fffffff;
    warp_argmax(v, idx);
  }
}

// Factor the inner panel rows [j0, r) x cols [j0, j0+wc) in shared memory.
__device__ void inner_panel(const Params& P, z_t* A, int k0, int j0, int wc, z_t* Ps, int* piv,
                            int* s_info, double* rv, int* ri, int* s_p, z_t* s_pv) {
  const int r = P.r, ldw = P.ldw, w = P.w;
  const int H = r - j0;
  const int tid = threadIdx.x;
  for (int e = tid; e < H * wc; e += NT) {
    int i = e / wc, c = e - i * wc;
    Ps[i * w + c] = A[(size_t)(j0 + i) * ldw + j0 + c];
  }
  __syncthreads();
  for (int jj = 0; jj < wc; ++jj) {
    double v = -1.0;
    int pi = 0x7fffffff;
    for (int i = jj + tid; i < H; i += NT) {
      double a = zabs1(Ps[i * w + jj]);
      if (a > v) { v = a; pi = i; }
    }
    block_argmax(v, pi, rv, ri);
    if (tid == 0) {
      if (v == 0.0) {
        if (*s_info == 0) *s_info = j0 + jj + 1;
        *s_p = -1;
      } else {
        *s_p = pi;
        *s_pv = Ps[pi * w + jj];
      }
      piv[j0 - k0 + jj] = j0 + (v == 0.0 ? jj : pi);
    }
    __syncthreads();
    const int p = *s_p;
    if (p < 0) continue;
    const z_t pv = *s_pv;
    const z_t pinv = zrecip(pv);
    for (int i = jj + 1 + tid; i < H; i += NT) {
      int src = (i == p) ? jj : i;
      Ps[i * w + jj] = zmul(Ps[src * w + jj], pinv);
    }
    if (p != jj) {
      // whole-row interchange within the inner panel (column jj is read through the swap above)
      for (int c = tid; c < wc; c += NT) {
        if (c == jj) continue;
        z_t t = Ps[jj * w + c];
        Ps[jj * w + c] = Ps[p * w + c];
        Ps[p * w + c] = t;
      }
    }
    __syncthreads();
    if (tid == 0) Ps[jj * w + jj] = pv;
    const int nc = wc - jj - 1;
    if (nc > 0) {
      for (int e = tid; e < (H - jj - 1) * nc; e += NT) {
        int ii = e / nc;
        int i = jj + 1 + ii, c = jj + 1 + (e - ii * nc);
        Ps[i * w + c] = zfms(Ps[i * w + c], Ps[i * w + jj], Ps[jj * w + c]);
      }
    }
    __syncthreads();
  }
  for (int e = tid; e < H * wc; e += NT) {
    int i = e / wc, c = e - i * wc;
    A[(size_t)(j0 + i) * ldw + j0 + c] = Ps[i * w + c];
  }
  __syncthreads();
}

// Row interchanges piv[a..b) (global row ids, relative to panel base k0) applied
// to columns [c0, c1).
__device__ void apply_swaps(z_t* A, int ldw, const int* piv, int k0, int a, int b, int c0, int c1) {
  for (int c = c0 + threadIdx.x; c < c1; c += NT) {
    for (int i = a; i < b; ++i) {
      int p = piv[i - k0];
      if (p != i) {
        z_t t = A[(size_t)i * ldw + c];
        A[(size_t)i * ldw + c] = A[(size_t)p * ldw + c];
        A[(size_t)p * ldw + c] = t;
      }
    }
  }
}

// U = L^-1 U for the wc rows of an inner panel (unit lower L = Ps[0:wc, 0:wc]),
// columns [c0, c1): one thread per column.
__device__ void inner_trsm(z_t* A, int ldw, const z_t* Ps, int w, int j0, int wc, int c0, int c1) {
  for (int c = c0 + threadIdx.x; c < c1; c += NT) {
    z_t xv[16];
#pragma unroll
    for (int i = 0; i < 16; ++i)
      if (i < wc) xv[i] = A[(size_t)(j0 + i) * ldw + c];
#pragma unroll
    for (int i = 1; i < 16; ++i) {
      if (i < wc) {
        z_t acc = xv[i];
#pragma unroll
        for (int k = 0; k < 16; ++k)
          if (k < i) acc = zfms(acc, Ps[i * w + k], xv[k]);
        xv[i] = acc;
      }
    }
#pragma unroll
    for (int i = 1; i < 16; ++i)
      if (i < wc) A[(size_t)(j0 + i) * ldw + c] = xv[i];
  }
}

// L11^-1 of the unit-lower nb x nb diagonal block at (k0, k0) into Li (NB x LDL,
// zero padded), then U12 = L11^-1 A12 in place for columns [c0, c1).
__device__ void panel_trsm(z_t* A, int ldw, int k0, int nb, int c0, int c1, z_t* smem) {
  z_t* Li = smem;             // NB x LDL
  z_t* Bs = smem + NB * LDL;  // NB x LDS_B
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // L (strictly lower part) staged in Bs, Li = I
  for (int e = tid; e < NB * NB; e += NT) {
    int i = e / NB, j = e - i * NB;
    Li[i * LDL + j] = zmake(i == j && i < nb ? 1.0 : 0.0, 0.0);
    Bs[i * LDS_B + j] = (i < nb && j < i) ? A[(size_t)(k0 + i) * ldw + k0 + j] : zmake(0.0, 0.0);
  }
  __syncthreads();
  // row i of L^-1: Li[i, j] = -sum_{k=j}^{i-1} L[i,k] Li[k,j], 4 threads per j
  {
    const int j = tid >> 2, q = tid & 3;
    for (int i = 1; i < nb; ++i) {
      z_t acc = zmake(0.0, 0.0);
      if (j < i)
        for (int k = j + q; k < i; k += 4) acc = zfma(acc, Bs[i * LDS_B + k], Li[k * LDL + j]);
      acc.x += __shfl_xor_sync(0xffffffffu, acc.x, 1);
      acc.y += __shfl_xor_sync(0xffffffffu, acc.y, 1);
      acc.x += __shfl_xor_sync(0xffffffffu, acc.x, 2);
      acc.y += __shfl_xor_sync(0xffffffffu, acc.y, 2);
      if (q == 0 && j < i) Li[i * LDL + j] = zmake(-acc.x, -acc.y);
      __syncthreads();
    }
  }
  // U12 strips of NB columns: C(nb x NB) = Li(nb x nb) * B(nb x NB)
  constexpr int FM = 4, FN = 2;  // warp grid 2 x 4 over the 64 x 64 strip
  const int wm = warp / 4, wn = warp % 4;
  const int k4 = (nb + 3) >> 2;
  for (int cs = c0; cs < c1; cs += NB) {
    const int ncol = min(NB, c1 - cs);
    for (int e = tid; e < NB * NB; e += NT) {
      int i = e / NB, j = e - i * NB;
      Bs[i * LDS_B + j] = (i < nb && j < ncol) ? A[(size_t)(k0 + i) * ldw + cs + j] : zmake(0.0, 0.0);
    }
    __syncthreads();
    double cr[FM][FN][2], ci[FM][FN][2];
#pragma unroll
    for (int i = 0; i < FM; ++i)
#pragma unroll
      for (int j = 0; j < FN; ++j) cr[i][j][0] = cr[i][j][1] = ci[i][j][0] = ci[i][j][1] = 0.0;
    warp_cmma<FM, FN, false>(cr, ci, Li + (wm * 32) * LDL, LDL, Bs + wn * 16, LDS_B, k4);
#pragma unroll
    for (int i = 0; i < FM; ++i)
#pragma unroll
      for (int j = 0; j < FN; ++j)
#pragma unroll
        for (int v = 0; v < 2; ++v) {
          int row = wm * 32 + i * 8 + (lane >> 2);
          int col = wn * 16 + j * 8 + 2 * (lane & 3) + v;
          if (row < nb && col < ncol)
            A[(size_t)(k0 + row) * ldw + cs + col] = zmake(cr[i][j][v], ci[i][j][v]);
        }
    __syncthreads();
  }
}

// Solve U[kb:kb+nb, kb:kb+nb] X = Y in place on columns [r, r+s).
__device__ void diag_backsolve(z_t* A, int ldw, int r, int s, int kb, int nb, z_t* smem) {
  z_t* Us = smem;                 // NB x (NB+1)
  z_t* Ys = smem + NB * (NB + 1); // NB x s
  const int tid = threadIdx.x;
  for (int e = tid; e < nb * nb; e += NT) {
    int i = e / nb, j = e - i * nb;
    Us[i * (NB + 1) + j] = A[(size_t)(kb + i) * ldw + kb + j];
  }
  for (int e = tid; e < nb * s; e += NT) {
    int i = e / s, c = e - i * s;
    Ys[i * s + c] = A[(size_t)(kb + i) * ldw + r + c];
  }
  __syncthreads();
  if (tid < s) {
    int k = nb - 1;
    Ys[k * s + tid] = zmul(Ys[k * s + tid], zrecip(Us[k * (NB + 1) + k]));
  }
  __syncthreads();
  for (int k = nb - 1; k > 0; --k) {
    for (int e = tid; e < k * s; e += NT) {
      int i = e / s, c = e - i * s;
      z_t v = zfms(Ys[i * s + c], Us[i * (NB + 1) + k], Ys[k * s + c]);
      if (i == k - 1) v = zmul(v, zrecip(Us[i * (NB + 1) + i]));
      Ys[i * s + c] = v;
    }
    __syncthreads();
  }
  for (int e = tid; e < nb * s; e += NT) {
    int i = e / s, c = e - i * s;
    A[(size_t)(kb + i) * ldw + r + c] = Ys[i * s + c];
  }
  __syncthreads();
}

// A = sum_k alpha_k P_k into the workspace.  Bandwidth-bound: each thread keeps
// KP x 4 independent 16-byte loads in flight (prims are shared by all CTAs and
// mostly L2-resident).
template <int KP>
__device__ __forceinline__ void form_quads(const Params& P, z_t* A, const z_t* alph) {
  const int r = P.r, ldw = P.ldw;
  const int64_t rr = (int64_t)r * r, nq = rr >> 2;
  z_t a[KP];
#pragma unroll
  for (int k = 0; k < KP; ++k) a[k] = alph[k];
  for (int64_t q = threadIdx.x; q < nq; q += NT) {
    z_t v[KP][4];
#pragma unroll
    for (int k = 0; k < KP; ++k)
#pragma unroll
      for (int e = 0; e < 4; ++e) v[k][e] = __ldg(P.prims + k * rr + 4 * q + e);
    const int64_t i = (4 * q) / r, j = 4 * q - i * r;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      z_t acc = zmul(a[0], v[0][e]);
#pragma unroll
      for (int k = 1; k < KP; ++k) acc = zfma(acc, a[k], v[k][e]);
      A[i * ldw + j + e] = acc;
    }
  }
}

__device__ void form_matrix(const Params& P, z_t* A, const z_t* alph) {
  const int r = P.r, ldw = P.ldw;
  if ((r & 3) == 0 && P.nprim <= 4) {
    switch (P.nprim) {
      case 1: form_quads<1>(P, A, alph); return;
      case 2: form_quads<2>(P, A, alph); return;
      case 3: form_quads<3>(P, A, alph); return;
      default: form_quads<4>(P, A, alph); return;
    }
  }
  const int64_t rr = (int64_t)r * r;
  for (int64_t idx = threadIdx.x; idx < rr; idx += NT) {
    z_t acc = zmake(0.0, 0.0);
    for (int k = 0; k < P.nprim; ++k) acc = zfma(acc, alph[k], __ldg(P.prims + k * rr + idx));
    const int64_t i = idx / r, j = idx - i * r;
    A[i * ldw + j] = acc;
  }
}

__global__ void __launch_bounds__(NT, 1) rom_sweep_blocked_kernel(Params P) {
  extern __shared__ double2 smem[];
  __shared__ int piv[NB];
  __shared__ double rv[NT / 32];
  __shared__ int ri[NT / 32];
  __shared__ int s_info, s_p;
  __shared__ z_t s_pv;
  __shared__ z_t alph[64];
  const int r = P.r, s = P.s, ldw = P.ldw, tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  z_t* A = P.work + (size_t)blockIdx.x * r * ldw;
  const int64_t rr = (int64_t)r * r;

  for (int64_t f = blockIdx.x; f < P.F; f += gridDim.x) {
    if (tid < P.nprim) alph[tid] = P.alpha[f * P.nprim + tid];
    if (tid == 0) s_info = 0;
    __syncthreads();
    // ---- form [A | B] ----
    form_matrix(P, A, alph);
    const z_t* bf = P.b + f * P.b_stride_f;
    for (int idx = tid; idx < r * s; idx += NT) {
      int i = idx / s, c = idx - i * s;
      A[(size_t)i * ldw + r + c] = __ldg(bf + idx);
    }
    __syncthreads();

    // ---- blocked right-looking LU on [A | B] ----
    for (int k0 = 0; k0 < r; k0 += NB) {
      const int nb = min(NB, r - k0);
      for (int j0 = k0; j0 < k0 + nb; j0 += P.w) {
        const int wc = min(P.w, k0 + nb - j0);
        inner_panel(P, A, k0, j0, wc, smem, piv, &s_info, rv, ri, &s_p, &s_pv);
        // fold the inner panel into the rest of the outer panel
        apply_swaps(A, ldw, piv, k0, j0, j0 + wc, k0, j0);
        apply_swaps(A, ldw, piv, k0, j0, j0 + wc, j0 + wc, k0 + nb);
        __syncthreads();
        if (j0 + wc < k0 + nb) {
          inner_trsm(A, ldw, smem, P.w, j0, wc, j0 + wc, k0 + nb);
          __syncthreads();
          GemmWide::run(A + (size_t)(j0 + wc) * ldw + j0 + wc, ldw, A + (size_t)(j0 + wc) * ldw + j0,
                        ldw, A + (size_t)j0 * ldw + j0 + wc, ldw, r - j0 - wc, k0 + nb - j0 - wc, wc,
                        smem);
          __syncthreads();
        }
      }
      const int c0 = k0 + nb, c1 = r + s;
      apply_swaps(A, ldw, piv, k0, k0, k0 + nb, c0, c1);
      __syncthreads();
      panel_trsm(A, ldw, k0, nb, c0, c1, smem);
      __syncthreads();
      if (c0 < r) {
        GemmWide::run(A + (size_t)c0 * ldw + c0, ldw, A + (size_t)c0 * ldw + k0, ldw,
                      A + (size_t)k0 * ldw + c0, ldw, r - c0, c1 - c0, nb, smem);
        __syncthreads();
      }
    }

    // ---- blocked back substitution on the RHS columns ----
    const int last = ((r - 1) / NB) * NB;
    for (int kb = last; kb >= 0; kb -= NB) {
      const int nb = min(NB, r - kb);
      diag_backsolve(A, ldw, r, s, kb, nb, smem);
      if (kb > 0) {
        GemmNarrow::run(A + r, ldw, A + kb, ldw, A + (size_t)kb * ldw + r, ldw, kb, s, nb, smem);
        __syncthreads();
      }
    }

    // ---- outputs ----
    if (P.x) {
      z_t* xf = P.x + f * (int64_t)r * s;
      for (int idx = tid; idx < r * s; idx += NT) {
        int i = idx / s, c = idx - i * s;
        xf[idx] = A[(size_t)i * ldw + r + c];
      }
    }
    if (P.n_out > 0 && (P.y || P.spl)) {
      double* p2 = (double*)smem;
      for (int idx = tid; idx < P.n_out * s; idx += NT) {
        int o = idx / s, c = idx - o * s;
        const z_t* cr = P.c_r + (int64_t)o * r;
        z_t acc = zmake(0.0, 0.0);
        for (int i = 0; i < r; ++i) acc = zfma(acc, __ldg(cr + i), A[(size_t)i * ldw + r + c]);
        if (P.y) P.y[(f * P.n_out + o) * s + c] = acc;
        p2[idx] = zabs2(acc);
      }
      __syncthreads();
      if (P.spl) {
        for (int c = warp; c < s; c += NT / 32) {
          double acc = 0.0;
          for (int o = lane; o < P.n_out; o += 32) acc += p2[o * s + c];
          acc = warp_sum(acc);
          if (lane == 0) {
            double prms = sqrt(acc / P.n_out / 2.0);
            P.spl[f * s + c] = 20.0 * log10(fmax(prms, 1e-300) / 20e-6);
          }
        }
      }
    }
    if (tid == 0 && P.info) P.info[f] = s_info;
    __syncthreads();
  }
}

static int ldw_of(int r, int s) { return (r + s + 3) & ~3; }

static size_t smem_bytes(int r, int s, int n_out, int w) {
  size_t m = GemmWide::SMEM;
  m = m > GemmNarrow::SMEM ? m : GemmNarrow::SMEM;
  m = m > TRSM_SMEM ? m : TRSM_SMEM;
  size_t bs = (size_t)(NB * (NB + 1) + NB * s) * sizeof(z_t);
  m = m > bs ? m : bs;
  size_t ps = (size_t)r * w * sizeof(z_t);
  m = m > ps ? m : ps;
  size_t p2 = (size_t)n_out * s * sizeof(double);
  m = m > p2 ? m : p2;
  return m;
}

static int pick_w(int r, int s, int n_out) {
  const size_t limit = 200 * 1024;
  for (int w = 16; w >= 1; w >>= 1)
    if (smem_bytes(r, s, n_out, w) <= limit && (size_t)r * w * sizeof(z_t) <= limit) return w;
  return 0;
}

}  // namespace blk

static int blocked_grid(int64_t F) {
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  return (int)(F < nsm ? F : nsm);
}

size_t sweep_blocked_workspace_bytes(int r, int s, int64_t F) {
  return (size_t)blocked_grid(F) * r * blk::ldw_of(r, s) * sizeof(z_t);
}

int sweep_blocked_supported(int r, int s, int n_out) {
  return s <= 16 && blk::pick_w(r, s, n_out) > 0;
}

int sweep_blocked_launch(int r, int nprim, int s, int n_out, int64_t F, const z_t* prims,
                         const z_t* alpha, const z_t* b, int64_t b_stride_f, const z_t* c_r, z_t* y,
                         double* spl, z_t* x, int* info, void* work, size_t work_bytes,
                         cudaStream_t stream) {
  VB_CHECK_ARG(s <= 16, "vb_rom_sweep (blocked): at most 16 RHS columns");
  VB_CHECK_ARG(nprim <= 64, "vb_rom_sweep (blocked): at most 64 primitives");
  const int w = blk::pick_w(r, s, n_out);
  VB_CHECK_ARG(w > 0, "vb_rom_sweep (blocked): reduced order too large for the inner panel");
  const size_t need = sweep_blocked_workspace_bytes(r, s, F);
  VB_CHECK_ARG(work != nullptr && work_bytes >= need, "vb_rom_sweep (blocked): workspace too small");
  blk::Params P;
  P.r = r; P.nprim = nprim; P.s = s; P.n_out = n_out; P.F = F;
  P.prims = prims; P.alpha = alpha; P.b = b; P.b_stride_f = b_stride_f; P.c_r = c_r;
  P.y = y; P.spl = spl; P.x = x; P.info = info;
  P.work = (z_t*)work; P.ldw = blk::ldw_of(r, s); P.w = w;
  const size_t smem = blk::smem_bytes(r, s, n_out, w);
  VB_CUDA(cudaFuncSetAttribute(blk::rom_sweep_blocked_kernel,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  blk::rom_sweep_blocked_kernel<<<blocked_grid(F), blk::NT, smem, stream>>>(P);
  VB_LAUNCHED("rom_sweep_blocked_kernel");
  return 0;
}

}  // namespace vb
