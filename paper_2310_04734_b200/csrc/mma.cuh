// FP64 tensor-core (DMMA, mma.sync.m8n8k4.f64) complex-MMA building blocks and
// cp.async helpers shared by the sweep, GEMM and LU kernels.
#pragma once
#include "common.cuh"

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


// warp_cmma with the 3M (Gauss) product: t1 = ar br (cr), t2 = ai bi (c2),
// t3 = (ar + ai)(br + bi) (ci); the caller forms Re = t1 - t2,
// Im = t3 - t1 - t2.  3 DMMAs per fragment pair instead of 4.
template <int FM, int FN>
__device__ __forceinline__ void warp_cmma3(double (&cr)[FM][FN][2], double (&ci)[FM][FN][2],
                                           double (&c2)[FM][FN][2], const z_t* as, int lda, const z_t* bs,
                                           int ldb, int k4) {
  const int lane = threadIdx.x & 31;
  const int ar = lane >> 2, ak = lane & 3;
#pragma unroll 2
  for (int kk = 0; kk < k4; ++kk) {
    z_t a[FM], b[FN];
    double sa[FM], sb[FN];
#pragma unroll
    for (int i = 0; i < FM; ++i) {
      a[i] = as[(i * 8 + ar) * lda + kk * 4 + ak];
      sa[i] = a[i].x + a[i].y;
    }
#pragma unroll
    for (int j = 0; j < FN; ++j) {
      b[j] = bs[(kk * 4 + ak) * ldb + j * 8 + ar];
      sb[j] = b[j].x + b[j].y;
    }
#pragma unroll
    for (int j = 0; j < FN; ++j)
#pragma unroll
      for (int i = 0; i < FM; ++i) {
        dmma(cr[i][j][0], cr[i][j][1], a[i].x, b[j].x);
        dmma(c2[i][j][0], c2[i][j][1], a[i].y, b[j].y);
        dmma(ci[i][j][0], ci[i][j][1], sa[i], sb[j]);
      }
  }
}

// CTA-wide C[M x N] -= A[M x K] * B[K x N] on global (workspace) operands.
// Tiles TM x TN over WM x WN warps.  One flat software pipeline runs over all
// (tile, k-chunk) iterations: A/B chunks stream through a STAGES-deep
// cp.async ring, and the C tile of the next output tile is prefetched into
// shared memory while the current tile computes, so neither the operand nor
// the C-tile latency is exposed at tile boundaries.  Accumulation starts from
// zero; the epilogue writes C_old - A*B (SUB) or A*B (!SUB, C not read).
// Epilogue modes: EPI_SUB  C = C_old - A*B   (LU updates)
//                 EPI_SET  C = A*B           (C not read)
//                 EPI_AXPBY C = alpha*A*B + beta*C_old
enum { EPI_SUB = 0, EPI_SET = 1, EPI_AXPBY = 2 };

template <int TM, int TN, int WM, int WN, int STAGES, int EPI, int KC = 16, bool M3 = false>
struct Gemm {
  static constexpr bool SUB = EPI != EPI_SET;  // reads C_old
  static_assert(WM * WN == NT / 32, "warp grid");
  static constexpr int FM = TM / WM / 8, FN = TN / WN / 8;
  static constexpr int LDA = KC + 4;  // == 4 (mod 8): conflict-free 128-bit fragment loads
  static constexpr int LDB = TN + 2;  // == 2 (mod 8)
  static constexpr int LDC = TN + 1;  // == 1 (mod 8): conflict-free epilogue reads
  static constexpr int A_EL = TM * LDA, B_EL = KC * LDB, C_EL = TM * LDC;
  static constexpr size_t SMEM = (size_t)(STAGES * (A_EL + B_EL) + (SUB ? C_EL : 0)) * sizeof(z_t);

  static_assert(NT % KC == 0 && NT % TN == 0, "loader mapping");
  static_assert((TM * KC) % NT == 0 && (KC * TN) % NT == 0 && (TM * TN) % NT == 0, "loader mapping");
  static constexpr int A_PER = TM * KC / NT, A_RS = NT / KC;  // rows a thread loads / row stride
  static constexpr int B_PER = KC * TN / NT, B_RS = NT / TN;
  static constexpr int C_PER = TM * TN / NT, C_RS = NT / TN;

  __device__ static __forceinline__ void cp16(unsigned s, const void* g, bool p) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(g), "r"(p ? 16 : 0));
  }

  // Per-thread loader state: the element a thread copies has a fixed column
  // (k for A, j for B/C) and rows i0 + q * RS, so only bases move per chunk.
  struct Loader {
    unsigned as0, bs0, cs0;  // shared addresses of this thread's first element
    int a_i0, a_k, b_k0, b_j;
  };

  __device__ static __forceinline__ void load_chunk(const Loader& L, int stage, const z_t* A, int lda,
                                                    const z_t* B, int ldb, int M, int N, int K, int m0,
                                                    int n0, int k0) {
    const bool kva = k0 + L.a_k < K;
    const z_t* Ab = A + (size_t)(m0 + L.a_i0) * lda + k0 + L.a_k;
    const unsigned as = L.as0 + (unsigned)(stage * A_EL * sizeof(z_t));
#pragma unroll
    for (int q = 0; q < A_PER; ++q) {
      const bool p = kva && (m0 + L.a_i0 + q * A_RS < M);
      cp16(as + (unsigned)(q * A_RS * LDA * sizeof(z_t)), p ? (const void*)(Ab + (size_t)q * A_RS * lda) : (const void*)A, p);
    }
    const bool jv = n0 + L.b_j < N;
    const z_t* Bb = B + (size_t)(k0 + L.b_k0) * ldb + n0 + L.b_j;
    const unsigned bs = L.bs0 + (unsigned)(stage * B_EL * sizeof(z_t));
#pragma unroll
    for (int q = 0; q < B_PER; ++q) {
      const bool p = jv && (k0 + L.b_k0 + q * B_RS < K);
      cp16(bs + (unsigned)(q * B_RS * LDB * sizeof(z_t)), p ? (const void*)(Bb + (size_t)q * B_RS * ldb) : (const void*)B, p);
    }
  }

  __device__ static __forceinline__ void load_c(const Loader& L, const z_t* C, int ldc, int M, int N,
                                                int m0, int n0) {
    const bool jv = n0 + L.b_j < N;
    const z_t* Cb = C + (size_t)(m0 + L.b_k0) * ldc + n0 + L.b_j;
#pragma unroll
    for (int q = 0; q < C_PER; ++q) {
      const bool p = jv && (m0 + L.b_k0 + q * C_RS < M);
      cp16(L.cs0 + (unsigned)(q * C_RS * LDC * sizeof(z_t)), p ? (const void*)(Cb + (size_t)q * C_RS * ldc) : (const void*)C, p);
    }
  }

  // Tiles t = t_first, t_first + t_step, ... of the (M/TM) x (N/TN) grid (row-major);
  // the default covers all tiles with one CTA.
  __device__ static void run(z_t* C, int ldc, const z_t* A, int lda, const z_t* B, int ldb, int M,
                             int N, int K, z_t* smem, z_t alpha = zmake(1.0, 0.0),
                             z_t beta = zmake(0.0, 0.0), int t_first = 0, int t_step = 1) {
    if (M <= 0 || N <= 0 || K <= 0) return;
    z_t* As = smem;
    z_t* Bs = smem + STAGES * A_EL;
    z_t* Cs = Bs + STAGES * B_EL;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = warp / WN, wn = warp % WN;
    const int ntn = (N + TN - 1) / TN, nk = (K + KC - 1) / KC;
    const int ntiles = ((M + TM - 1) / TM) * ntn;
    if (t_first >= ntiles) return;
    const int my_tiles = (ntiles - t_first + t_step - 1) / t_step;
    const int T = my_tiles * nk;
    Loader L;
    L.a_i0 = tid / KC;
    L.a_k = tid % KC;
    L.b_k0 = tid / TN;
    L.b_j = tid % TN;
    L.as0 = (unsigned)__cvta_generic_to_shared(As + L.a_i0 * LDA + L.a_k);
    L.bs0 = (unsigned)__cvta_generic_to_shared(Bs + L.b_k0 * LDB + L.b_j);
    L.cs0 = (unsigned)__cvta_generic_to_shared(Cs + L.b_k0 * LDC + L.b_j);
    // producer cursor (iteration p -> tile pt, chunk pk) advanced without divisions
    int pt = t_first, pk = 0, pm0 = (pt / ntn) * TM, pn0 = (pt % ntn) * TN;
    auto issue_next = [&](int p) {
      if (p < T) load_chunk(L, p % STAGES, A, lda, B, ldb, M, N, K, pm0, pn0, pk * KC);
      if (++pk == nk) {
        pk = 0;
        pt += t_step;
        pm0 = (pt / ntn) * TM;
        pn0 = (pt % ntn) * TN;
      }
    };
    if (SUB) load_c(L, C, ldc, M, N, pm0, pn0);
#pragma unroll
    for (int j = 0; j < STAGES - 1; ++j) {
      issue_next(j);
      cp_commit();
    }
    double cr[FM][FN][2], ci[FM][FN][2];
    double c2[M3 ? FM : 1][M3 ? FN : 1][2];  // 3M: sum ai bi
#pragma unroll
    for (int i = 0; i < FM; ++i)
#pragma unroll
      for (int j = 0; j < FN; ++j) cr[i][j][0] = cr[i][j][1] = ci[i][j][0] = ci[i][j][1] = 0.0;
    if (M3)
#pragma unroll
      for (int i = 0; i < (M3 ? FM : 1); ++i)
#pragma unroll
        for (int j = 0; j < (M3 ? FN : 1); ++j) c2[i][j][0] = c2[i][j][1] = 0.0;
    int t = t_first, kc = 0;
    int m0 = (t / ntn) * TM, n0 = (t % ntn) * TN;
    const z_t* as_w = As + (wm * FM * 8) * LDA;
    const z_t* bs_w = Bs + wn * FN * 8;
    for (int it = 0; it < T; ++it) {
      cp_wait<STAGES - 2>();
      __syncthreads();
      issue_next(it + STAGES - 1);
      if (SUB && kc == 0 && it > 0) load_c(L, C, ldc, M, N, m0, n0);
      cp_commit();
      const int st = it % STAGES;
      int k4 = min(KC, K - kc * KC);
      k4 = (k4 + 3) >> 2;
      if constexpr (M3)
        warp_cmma3<FM, FN>(cr, ci, c2, as_w + st * A_EL, LDA, bs_w + st * B_EL, LDB, k4);
      else
        warp_cmma<FM, FN, false>(cr, ci, as_w + st * A_EL, LDA, bs_w + st * B_EL, LDB, k4);
      if (kc == nk - 1) {
        if (SUB && nk < STAGES) {  // the C-tile group may still be in flight
          cp_wait<0>();
          __syncthreads();
        }
        const bool beta0 = beta.x == 0.0 && beta.y == 0.0;
#pragma unroll
        for (int i = 0; i < FM; ++i)
#pragma unroll
          for (int j = 0; j < FN; ++j)
#pragma unroll
            for (int v = 0; v < 2; ++v) {
              const int lr = wm * FM * 8 + i * 8 + (lane >> 2);
              const int lc = wn * FN * 8 + j * 8 + 2 * (lane & 3) + v;
              if (m0 + lr < M && n0 + lc < N) {
                z_t acc = zmake(cr[i][j][v], ci[i][j][v]);
                if constexpr (M3) {
                  const double t2 = c2[i < (M3 ? FM : 1) ? i : 0][j < (M3 ? FN : 1) ? j : 0][v];
                  acc = zmake(cr[i][j][v] - t2, ci[i][j][v] - cr[i][j][v] - t2);
                }
                z_t out;
                if (EPI == EPI_SUB) {
                  const z_t c = Cs[lr * LDC + lc];
                  out = zmake(c.x - acc.x, c.y - acc.y);
                } else if (EPI == EPI_SET || beta0) {
                  out = zmul(alpha, acc);  // C_old never contributes (may be uninitialised)
                } else {
                  out = zfma(zmul(alpha, acc), beta, Cs[lr * LDC + lc]);
                }
                C[(size_t)(m0 + lr) * ldc + n0 + lc] = out;
              }
              cr[i][j][v] = 0.0;
              ci[i][j][v] = 0.0;
              if constexpr (M3) c2[i < (M3 ? FM : 1) ? i : 0][j < (M3 ? FN : 1) ? j : 0][v] = 0.0;
            }
        kc = 0;
        t += t_step;
        m0 = (t / ntn) * TM;
        n0 = (t % ntn) * TN;
      } else {
        ++kc;
      }
    }
    cp_wait<0>();
  }
};


// In-place inverse of a 64 x 64 triangular matrix in shared memory by recursive
// doubling: 8x8 diagonal blocks per warp, then three levels of
// [A 0; C D]^-1 = [A^-1 0; -D^-1 C A^-1 D^-1]  (lower, unit diagonal) or
// [A B; 0 D]^-1 = [A^-1 -A^-1 B D^-1; 0 D^-1]  (upper, general diagonal).
// 13 barriers instead of one per row.
template <bool LOWER>
__device__ __noinline__ void tri_inv64(z_t* T, int ld) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  {
    const int o = warp * 8, j = lane;
    z_t x[8];
    if (lane < 8) {
      if (LOWER) {
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = zmake(i == j ? 1.0 : 0.0, 0.0);
#pragma unroll
        for (int i = 1; i < 8; ++i) {
          if (i > j) {
            z_t acc = zmake(0.0, 0.0);
#pragma unroll
            for (int k = 0; k < 8; ++k)
              if (k >= j && k < i) acc = zfma(acc, T[(o + i) * ld + o + k], x[k]);
            x[i] = zmake(-acc.x, -acc.y);
          }
        }
      } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = zmake(0.0, 0.0);
#pragma unroll
        for (int i = 7; i >= 0; --i) {
          if (i <= j) {
            z_t acc = zmake(i == j ? 1.0 : 0.0, 0.0);
#pragma unroll
            for (int k = 0; k < 8; ++k)
              if (k > i && k <= j) acc = zfms(acc, T[(o + i) * ld + o + k], x[k]);
            x[i] = zmul(acc, zrecip(T[(o + i) * ld + o + i]));
          }
        }
      }
    }
    __syncwarp();
    if (lane < 8) {
#pragma unroll
      for (int i = 0; i < 8; ++i)
        if (LOWER ? (i > j) : (i <= j)) T[(o + i) * ld + o + j] = x[i];
    }
  }
  __syncthreads();
  // doubling levels on the FP64 tensor cores: each h x h off-diagonal block is
  // two complex GEMMs of 8x8 fragments (warp_cmma); h/2 fragments per level,
  // at most two per warp.  Results are held in registers across the barrier
  // that separates the reads of a pass from its in-place writes.
  const int lane8 = lane >> 2, lq = lane & 3;
#pragma unroll 1
  for (int h = 8; h < 64; h *= 2) {
    const int nf = h / 8, per_blk = nf * nf, nfr = (64 / (2 * h)) * per_blk;
#pragma unroll 1
    for (int pass = 0; pass < 2; ++pass) {
      double rr[2][2], ri[2][2];
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int fr = warp + q * (NT / 32);
        rr[q][0] = rr[q][1] = ri[q][0] = ri[q][1] = 0.0;
        if (fr < nfr) {
          const int pb = fr / per_blk, fi = (fr % per_blk) / nf, fj = fr % nf, o = pb * 2 * h;
          double cr[1][1][2] = {{{0.0, 0.0}}}, ci[1][1][2] = {{{0.0, 0.0}}};
          if (pass == 0) {  // T = C A^-1 (lower) or T = B D^-1 (upper)
            if (LOWER)
              warp_cmma<1, 1, false>(cr, ci, T + (o + h + fi * 8) * ld + o, ld, T + o * ld + o + fj * 8, ld, h / 4);
            else
              warp_cmma<1, 1, false>(cr, ci, T + (o + fi * 8) * ld + o + h, ld, T + (o + h) * ld + o + h + fj * 8,
                                     ld, h / 4);
          } else {          // X = -D^-1 T (lower) or X = -A^-1 T (upper)
            if (LOWER)
              warp_cmma<1, 1, true>(cr, ci, T + (o + h + fi * 8) * ld + o + h, ld, T + (o + h) * ld + o + fj * 8,
                                    ld, h / 4);
            else
              warp_cmma<1, 1, true>(cr, ci, T + (o + fi * 8) * ld + o, ld, T + o * ld + o + h + fj * 8, ld, h / 4);
          }
          rr[q][0] = cr[0][0][0];
          rr[q][1] = cr[0][0][1];
          ri[q][0] = ci[0][0][0];
          ri[q][1] = ci[0][0][1];
        }
      }
      __syncthreads();
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int fr = warp + q * (NT / 32);
        if (fr < nfr) {
          const int pb = fr / per_blk, fi = (fr % per_blk) / nf, fj = fr % nf, o = pb * 2 * h;
          const int row = (LOWER ? o + h : o) + fi * 8 + lane8;
          const int col = (LOWER ? o : o + h) + fj * 8 + 2 * lq;
          T[row * ld + col] = zmake(rr[q][0], ri[q][0]);
          T[row * ld + col + 1] = zmake(rr[q][1], ri[q][1]);
        }
      }
      __syncthreads();
    }
  }
}

}  // namespace blk
}  // namespace vb
