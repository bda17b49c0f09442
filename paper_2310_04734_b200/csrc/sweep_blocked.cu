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
#include "mma.cuh"
#include "sweep.cuh"
#include "tma.cuh"

namespace vb {
namespace blk {


// Two CTAs per SM (<= 128 registers, <= ~110 KB shared memory each) so that one
// frequency's latency-bound phases (panel, triangular inverses) overlap the
// other's tensor-core GEMMs.
using GemmWide = Gemm<64, 32, 4, 2, 2, EPI_SUB>;   // trailing / in-panel updates
using GemmNarrow = Gemm<64, 16, 8, 1, 2, EPI_SUB>; // back-substitution updates (N = s <= 16)
using GemmOut = Gemm<64, 16, 8, 1, 2, EPI_SET>;   // y = C_R x

constexpr int LDL = NB + 4;     // == 4 (mod 8): triangular inverse used as A operand
// Workspace reads outside the TMA GEMMs: with the TMA-store epilogue (async
// proxy writes that do not update this SM's L1) they must come from L2.
#if VB_TMA_STORE_EPI
#define VB_WS_LD(p) __ldcg(p)
#else
#define VB_WS_LD(p) (*(p))
#endif

#ifndef VB_DEEP_MIN_R
#define VB_DEEP_MIN_R 384
#endif
#ifndef VB_DEEP4_MIN_R
#define VB_DEEP4_MIN_R 1536
#endif
constexpr int DEEP_MIN_R = VB_DEEP_MIN_R;    // outer steps of 2 panels (trailing K = 128) from this order on (r = 400: +3 %, tools/sweep_rates.py)
constexpr int DEEP4_MIN_R = VB_DEEP4_MIN_R;  // ... of 4 panels (K = 256)
constexpr int LDY = 16 + 2;
constexpr size_t TRSM_SMEM = (size_t)(NB * LDL) * sizeof(z_t);
constexpr size_t BACK_SMEM = (size_t)(NB * LDL + NB * LDY) * sizeof(z_t);

using GemmT = tma::GemmTma<3>;

// Optional per-phase cycle accounting (build with -DVB_PHASE_TIMING; read with
// vb_debug_phase_cycles): thread 0 of every CTA adds the clock64() span of
// each phase.  0 form, 1 leaf panel, 2 in-panel TRSM+GEMM, 3 swaps,
// 4 U12 TRSM, 5 trailing GEMM, 6 back substitution, 7 outputs.
__device__ unsigned long long g_phase_cycles[16];
#ifdef VB_PHASE_TIMING
#define PH_BEGIN long long _ph_t = clock64()
#define PH_MARK(k)                                                                     \
  do {                                                                                 \
    if (threadIdx.x == 0) {                                                            \
      const long long _n = clock64();                                                  \
      atomicAdd(&g_phase_cycles[k], (unsigned long long)(_n - _ph_t));                 \
      _ph_t = _n;                                                                      \
    }                                                                                  \
  } while (0)
#define PH_SUB(k)                                                                      \
  do {                                                                                 \
    if (threadIdx.x == 0) {                                                            \
      const long long _n = clock64();                                                  \
      atomicAdd(&g_phase_cycles[k], (unsigned long long)(_n - _sub_t));                \
      _sub_t = _n;                                                                     \
    }                                                                                  \
  } while (0)
#define PH_SUB_BEGIN long long _sub_t = clock64()
#else
#define PH_BEGIN
#define PH_SUB(k) \
  do {            \
  } while (0)
#define PH_SUB_BEGIN
#define PH_MARK(k) \
  do {             \
  } while (0)
#endif

struct __align__(64) Params {
  tma::Maps maps;  // TMA descriptors over all CTAs' workspaces (must stay first: 64-B aligned)
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
  int ldw;            // leading dimension of the augmented matrix
  int w;              // inner panel width for the full height r
  int leaf_bytes;     // shared memory available to a leaf (rows + logical ids)
  size_t cta_stride;  // workspace elements per CTA
};

// izamax candidate carried through the reductions together with its value:
// key = (logical row << 16) | physical row, so that ties resolve to the lowest
// LOGICAL row (izamax order) while the physical slot locates the row.
struct Cand {
  double v;
  int key;
  z_t val;
};

// |Re|+|Im| >= 0 (or -1 for "no candidate"): the IEEE bit patterns order like
// the values when read as signed 64-bit integers, so the comparisons run on the
// integer pipe instead of waiting for the FP64 pipe the co-resident CTA's DMMAs
// keep busy.
__device__ __forceinline__ long long vbits(double v) { return __double_as_longlong(v); }
__device__ __forceinline__ void cand_better(Cand& a, const Cand& b) {
  const long long vb = vbits(b.v), va = vbits(a.v);
  if (vb > va || (vb == va && b.key < a.key)) a = b;
}

// Block-wide izamax (max |Re|+|Im|, lowest logical row on ties): warp
// shuffles, ONE barrier, then every warp reduces the 8 partials itself.  The
// partial slots are double-buffered by the caller (column parity), so the next
// column may overwrite the other buffer without a second barrier.
__device__ __forceinline__ Cand block_argmax(Cand c, double* rv, int* ri, z_t* rz) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {  // (value, key) only: the pivot value is re-read from its row
    Cand d;
    d.v = __shfl_xor_sync(0xffffffffu, c.v, o);
    d.key = __shfl_xor_sync(0xffffffffu, c.key, o);
    d.val = zmake(0.0, 0.0);
    cand_better(c, d);
  }
  (void)rz;
  if (lane == 0) { rv[warp] = c.v; ri[warp] = c.key; }
  __syncthreads();
  Cand best{rv[0], ri[0], zmake(0.0, 0.0)};
#pragma unroll
  for (int q = 1; q < NT / 32; ++q) cand_better(best, Cand{rv[q], ri[q], zmake(0.0, 0.0)});
  return best;
}

// 1/a with one division: a is scaled by a power of two (exact) so that
// |a|^2 neither overflows nor underflows.
// 1/a: a is scaled by a power of two (exact, from the exponent bits) so that
// d = |a|^2 lies in [1, 8); 1/d by the MUFU reciprocal estimate and two
// Newton steps (a few ulp, not correctly rounded — well inside the sweep's
// tolerance) instead of a full IEEE division on the contended FP64 pipe.
__device__ __forceinline__ z_t zrecip_fast(z_t a) {
  const double m = fmax(fabs(a.x), fabs(a.y));
  // sc = 2^(1023 - eb) from the biased exponent eb of m, so m sc lies in [1, 2)
  long long eb = (__double_as_longlong(m) >> 52) & 0x7ff;
  eb = eb < 1 ? 1 : (eb > 2045 ? 2045 : eb);
  const double sc = __longlong_as_double((2046 - eb) << 52);
  const double xr = a.x * sc, xi = a.y * sc;
  const double d = xr * xr + xi * xi;
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
  double e = fma(-d, y, 1.0);
  y = fma(y, e, y);
  e = fma(-d, y, 1.0);
  y = fma(y, e, y);
  const double inv = sc * y;
  return zmake(xr * inv, -xi * inv);
}

// Factor the inner panel rows [j0, r) x cols [j0, j0+wc) in shared memory
// (zgetf2 order, LAPACK pivots).  Rows never move inside shared memory: each
// physical row carries its LOGICAL position (lg[], touched only by the thread
// owning the row), an interchange just exchanges two logical positions, and
// the pivot row — read by every thread during the rank-1 update — is never
// written in the same phase.  The update of column jj fuses the argmax of
// column jj+1, so each column costs ONE block barrier.  Rows are written back
// to global memory in logical order.
template <int W>
__device__ void inner_panel_w(const Params& P, z_t* A, int k0, int j0, int wc, z_t* Ps, int* lg, int* piv,
                              int* s_info, double* rv, int* ri, z_t* rz) {
  const int r = P.r, ldw = P.ldw, lp = W + 1;
  const int H = r - j0;
  const int tid = threadIdx.x;
  PH_SUB_BEGIN;
  for (int e = tid; e < H * wc; e += NT) {
    const int i = e / wc, c = e - i * wc;
    cp_async16(Ps + i * lp + c, A + (size_t)(j0 + i) * ldw + j0 + c, true);
  }
  cp_commit();
  for (int q = tid; q < H; q += NT) lg[q] = q;
  cp_wait<0>();
  __syncthreads();
  PH_SUB(8);
  Cand cd{-1.0, 0x7fffffff, zmake(0.0, 0.0)};
  for (int q = tid; q < H; q += NT) {
    const z_t x = Ps[q * lp];
    const double a = zabs1(x);
    if (a > cd.v) cd = Cand{a, (q << 16) | q, x};
  }
  Cand best = block_argmax(cd, rv, ri, rz);
  for (int jj = 0; jj < wc; ++jj) {
    const bool zero = !(best.v > 0.0);
    const int p = zero ? jj : (best.key >> 16);
    const int b = best.key & 0xffff;
    VB_DCHECK(zero || (p >= jj && p < H && b >= 0 && b < H));
    if (tid == 0) {
      if (zero && *s_info == 0) *s_info = j0 + jj + 1;  // LAPACK INFO: no interchange, no scaling
      piv[j0 - k0 + jj] = j0 + p;
    }
    const int nc = wc - jj - 1;
    cd = Cand{-1.0, 0x7fffffff, zmake(0.0, 0.0)};
    if (!zero) {
      const z_t pinv = zrecip_fast(Ps[b * lp + jj]);  // pivot value from its (unmoved) row
      PH_SUB(13);
      const z_t* prow = Ps + b * lp;
      for (int q = tid; q < H; q += NT) {
        int l = lg[q];
        if (l < jj) continue;                       // finished (U) row
        if (q == b) { lg[q] = jj; continue; }       // pivot row moves to logical jj
        if (l == jj) { l = p; lg[q] = p; }          // displaced row takes the pivot's slot
        z_t* row = Ps + q * lp;
        const z_t m = zmul(row[jj], pinv);
        row[jj] = m;
        // compile-time column loop: all loads of the row issue back to back
#pragma unroll
        for (int c = 1; c < W; ++c) {
          if (c > jj && c < wc) {
            const z_t nv = zfms(row[c], m, prow[c]);
            row[c] = nv;
            if (c == jj + 1) {
              const double a = zabs1(nv);
              if (a > cd.v || (a == cd.v && ((l << 16) | q) < cd.key)) cd = Cand{a, (l << 16) | q, nv};
            }
          }
        }
      }
    } else if (nc > 0) {
      for (int q = tid; q < H; q += NT) {
        const int l = lg[q];
        if (l <= jj) continue;
        const z_t x = Ps[q * lp + jj + 1];
        const double a = zabs1(x);
        if (a > cd.v || (a == cd.v && ((l << 16) | q) < cd.key)) cd = Cand{a, (l << 16) | q, x};
      }
    }
    PH_SUB(12);
    const int buf = (jj + 1) & 1;
    if (nc > 0) best = block_argmax(cd, rv + buf * (NT / 32), ri + buf * (NT / 32), rz + buf * (NT / 32));
    PH_SUB(14);
  }
  __syncthreads();
  PH_SUB(9);
  for (int e = tid; e < H * wc; e += NT) {
    const int q = e / wc, c = e - q * wc;
    A[(size_t)(j0 + lg[q]) * ldw + j0 + c] = Ps[q * lp + c];
  }
  __syncthreads();
}

__device__ void inner_panel(const Params& P, z_t* A, int k0, int j0, int wc, z_t* Ps, int* lg, int* piv,
                            int* s_info, double* rv, int* ri, z_t* rz, int pw) {
  switch (pw) {
    case 16: inner_panel_w<16>(P, A, k0, j0, wc, Ps, lg, piv, s_info, rv, ri, rz); return;
    case 8: inner_panel_w<8>(P, A, k0, j0, wc, Ps, lg, piv, s_info, rv, ri, rz); return;
    case 4: inner_panel_w<4>(P, A, k0, j0, wc, Ps, lg, piv, s_info, rv, ri, rz); return;
    case 2: inner_panel_w<2>(P, A, k0, j0, wc, Ps, lg, piv, s_info, rv, ri, rz); return;
    default: inner_panel_w<1>(P, A, k0, j0, wc, Ps, lg, piv, s_info, rv, ri, rz); return;
  }
}

// Row interchanges piv[a..b) (global row ids, relative to panel base k0) applied
// to columns [c0, c1).
__device__ void apply_swaps(z_t* A, int ldw, const int* piv, int k0, int a, int b, int c0, int c1) {
  for (int c = c0 + threadIdx.x; c < c1; c += NT) {
    for (int i = a; i < b; ++i) {
      const int p = piv[i - k0];
      if (p != i) {
        const z_t t = VB_WS_LD(A + (size_t)i * ldw + c);
        A[(size_t)i * ldw + c] = VB_WS_LD(A + (size_t)p * ldw + c);
        A[(size_t)p * ldw + c] = t;
      }
    }
  }
}

// U = L^-1 U for rows [cl, cl+n1) (unit lower L = A[cl:cl+n1, cl:cl+n1], n1 <= 32)
// on columns [c0, c1) (c1 - c0 <= 32).  Short chains (n1 < 16): L and the
// block are staged in shared memory with one round of independent loads and
// solved one thread per column; long chains: one WARP per column with the
// column's rows on the lanes (forward substitution by shuffles).
__device__ void trsm_small(z_t* A, int ldw, int cl, int n1, int c0, int c1, z_t* smem) {
  constexpr int LD = 33;
  z_t* Ls = smem;
  z_t* Xs = smem + 32 * LD;
  const int nc = c1 - c0;
  if (n1 < 16) {
    for (int e = threadIdx.x; e < n1 * n1 + n1 * nc; e += NT) {
      if (e < n1 * n1) {
        const int i = e / n1, k = e - i * n1;
        Ls[i * LD + k] = VB_WS_LD(A + (size_t)(cl + i) * ldw + cl + k);
      } else {
        const int f = e - n1 * n1, i = f / nc, c = f - i * nc;
        Xs[i * LD + c] = VB_WS_LD(A + (size_t)(cl + i) * ldw + c0 + c);
      }
    }
    __syncthreads();
    const int c = threadIdx.x;
    if (c < nc) {
      for (int i = 1; i < n1; ++i) {
        z_t x = Xs[i * LD + c];
        for (int k = 0; k < i; ++k) x = zfms(x, Ls[i * LD + k], Xs[k * LD + c]);
        Xs[i * LD + c] = x;
        A[(size_t)(cl + i) * ldw + c0 + c] = x;
      }
    }
    return;
  }
  for (int e = threadIdx.x; e < n1 * n1; e += NT) {
    const int i = e / n1, k = e - i * n1;
    Ls[i * LD + k] = VB_WS_LD(A + (size_t)(cl + i) * ldw + cl + k);
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int c = c0 + warp; c < c1; c += NT / 32) {
    z_t x = zmake(0.0, 0.0);
    if (lane < n1) x = VB_WS_LD(A + (size_t)(cl + lane) * ldw + c);
    for (int k = 0; k + 1 < n1; ++k) {
      const double xr = __shfl_sync(0xffffffffu, x.x, k), xi = __shfl_sync(0xffffffffu, x.y, k);
      if (lane > k && lane < n1) x = zfms(x, Ls[lane * LD + k], zmake(xr, xi));
    }
    if (lane >= 1 && lane < n1) A[(size_t)(cl + lane) * ldw + c] = x;
  }
}

// U12 = L11^-1 A12 in place for columns [c0, c1): L11^-1 is formed explicitly
// (identity-padded to 64) and its strictly lower part, negated, is written to
// the CTA's scratch rows [r, r+64) so that the product runs through the TMA
// GEMM as an update: U12 = A12 - N A12 with N = I - L11^-1 = -offdiag(L11^-1)
// (the unit diagonal of L11^-1 is exact, so this equals L11^-1 A12).  Each C
// tile is fully consumed as the B operand before its epilogue writes it.
__device__ void panel_trsm(const Params& P, z_t* A, int k0, int nb, int c0, int c1, z_t* smem, GemmT::Bars* bars) {
  const int ldw = P.ldw, r = P.r;
  z_t* Li = smem;  // NB x LDL
  z_t* Nsc = A + (size_t)r * ldw;
  const int tid = threadIdx.x;
  for (int e = tid; e < NB * NB; e += NT) {
    const int i = e / NB, j = e - i * NB;
    z_t v = zmake(i == j ? 1.0 : 0.0, 0.0);
    if (i < nb && j < i) v = VB_WS_LD(A + (size_t)(k0 + i) * ldw + k0 + j);
    Li[i * LDL + j] = v;
  }
  __syncthreads();
  tri_inv64<true>(Li, LDL);
  for (int e = tid; e < NB * NB; e += NT) {
    const int i = e / NB, j = e - i * NB;
    const z_t v = Li[i * LDL + j];
    Nsc[(size_t)i * ldw + j] = (j < i && i < nb) ? zmake(-v.x, -v.y) : zmake(0.0, 0.0);
  }
  __syncthreads();
  GemmT::run(&P.maps, A, ldw, r, 0, k0, c0, nb, c1 - c0, nb, (char*)smem, bars, blockIdx.x, k0, 0, 1, true);
  __syncthreads();
}

// X = U_kk^-1 Y on the diagonal block rows [kb, kb+nb) of the RHS columns.
__device__ void diag_backsolve(z_t* A, int ldw, int r, int s, int kb, int nb, z_t* smem) {
  z_t* Us = smem;              // NB x LDL
  z_t* Ys = smem + NB * LDL;   // NB x LDY
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int e = tid; e < NB * NB; e += NT) {
    const int i = e / NB, j = e - i * NB;
    z_t v = zmake(i == j ? 1.0 : 0.0, 0.0);
    if (i < nb && j < nb) v = (j >= i) ? VB_WS_LD(A + (size_t)(kb + i) * ldw + kb + j) : zmake(0.0, 0.0);
    Us[i * LDL + j] = v;
  }
  for (int e = tid; e < NB * 16; e += NT) {
    const int i = e >> 4, c = e & 15;
    Ys[i * LDY + c] = (i < nb && c < s) ? VB_WS_LD(A + (size_t)(kb + i) * ldw + r + c) : zmake(0.0, 0.0);
  }
  __syncthreads();
  tri_inv64<false>(Us, LDL);
  double cr[1][2][2], ci[1][2][2];
#pragma unroll
  for (int j = 0; j < 2; ++j) cr[0][j][0] = cr[0][j][1] = ci[0][j][0] = ci[0][j][1] = 0.0;
  warp_cmma<1, 2, false>(cr, ci, Us + (warp * 8) * LDL, LDL, Ys, LDY, (nb + 3) >> 2);
#pragma unroll
  for (int j = 0; j < 2; ++j)
#pragma unroll
    for (int v = 0; v < 2; ++v) {
      const int row = warp * 8 + (lane >> 2);
      const int col = j * 8 + 2 * (lane & 3) + v;
      if (row < nb && col < s) A[(size_t)(kb + row) * ldw + r + col] = zmake(cr[0][j][v], ci[0][j][v]);
    }
  __syncthreads();
}

// A = sum_k alpha_k P_k into the workspace.  Bandwidth-bound: each thread keeps
// KP x 4 independent 16-byte loads in flight (the primitives are shared by all
// CTAs and pinned in L2 when they fit, see sweep_blocked_launch).
// 256-bit global accesses (sm_100: LDG/STG.256): two complex per instruction
__device__ __forceinline__ void ld256(const z_t* p, z_t& a, z_t& b) {
  asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
               : "=d"(a.x), "=d"(a.y), "=d"(b.x), "=d"(b.y)
               : "l"(p));
}
__device__ __forceinline__ void st256(z_t* p, z_t a, z_t b) {
  asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(a.x), "d"(a.y), "d"(b.x), "d"(b.y)
               : "memory");
}

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
    for (int k = 0; k < KP; ++k) {  // 64 B of each primitive in two 256-bit loads
      ld256(P.prims + k * rr + 4 * q, v[k][0], v[k][1]);
      ld256(P.prims + k * rr + 4 * q + 2, v[k][2], v[k][3]);
    }
    const int64_t i = (4 * q) / r, j = 4 * q - i * r;
    z_t o[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      z_t acc = zmul(a[0], v[0][e]);
#pragma unroll
      for (int k = 1; k < KP; ++k) acc = zfma(acc, a[k], v[k][e]);
      o[e] = acc;
    }
    st256(A + i * ldw + j, o[0], o[1]);
    st256(A + i * ldw + j + 2, o[2], o[3]);
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

__global__ void __launch_bounds__(NT, 2) rom_sweep_blocked_kernel(const __grid_constant__ Params P) {
  extern __shared__ __align__(1024) char smem_raw[];
  // 1024-byte aligned base (128B-swizzled TMA boxes)
  double2* smem = (double2*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ GemmT::Bars bars;
  __shared__ int piv[4 * NB];  // the panels of an outer step (up to 4)
  __shared__ double rv[2 * (NT / 32)];
  __shared__ int ri[2 * (NT / 32)];
  __shared__ int s_info;
  __shared__ z_t rz[2 * (NT / 32)];
  __shared__ z_t alph[64];
  const int r = P.r, s = P.s, ldw = P.ldw, tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  z_t* A = P.work + (size_t)blockIdx.x * P.cta_stride;
  z_t* yscratch = A + (size_t)(r + NB) * ldw;  // rows [r, r+NB): U12 scratch

  for (int64_t f = blockIdx.x; f < P.F; f += gridDim.x) {
    if (tid < P.nprim) alph[tid] = P.alpha[f * P.nprim + tid];
    if (tid == 0) s_info = 0;
    __syncthreads();
    // ---- form [A | B] ----
    PH_BEGIN;
    form_matrix(P, A, alph);
    const z_t* bf = P.b + f * P.b_stride_f;
    for (int idx = tid; idx < r * s; idx += NT) {
      const int i = idx / s, c = idx - i * s;
      A[(size_t)i * ldw + r + c] = __ldg(bf + idx);
    }
    if (ldw > r + s) {  // padding columns are read (never used) by TMA boxes: keep them finite
      const int pw = ldw - r - s;
      for (int idx = tid; idx < r * pw; idx += NT) {
        const int i = idx / pw, c = idx - i * pw;
        A[(size_t)i * ldw + r + s + c] = zmake(0.0, 0.0);
      }
    }
    __syncthreads();

    __syncthreads();
    PH_MARK(0);
    // ---- blocked right-looking LU on [A | B] ----
    // Recursive (zgetrf2-order) panel of pnb columns from pk0: leaves of w
    // columns are factored in shared memory; after leaf l the right sibling of
    // the largest completed left subtree (2^k leaves, k = trailing ones of l) is
    // updated with one TRSM + one GEMM of depth 2^k w.  Pivots go to
    // piv[j - pbase].
    auto factor_panel = [&](int pk0, int pnb, int pbase) {
      // leaf width: the widest of 16 / 8 / P.w whose rows (r - pk0 of them)
      // fit in shared memory — lower panels get wider leaves
      const int H = r - pk0;
      int pw = P.w;
      if (pw < 16 && (size_t)H * (17 * sizeof(z_t) + sizeof(int)) <= (size_t)P.leaf_bytes) pw = 16;
      else if (pw < 8 && (size_t)H * (9 * sizeof(z_t) + sizeof(int)) <= (size_t)P.leaf_bytes) pw = 8;
      const int nleaves = (pnb + pw - 1) / pw;
      for (int l = 0; l < nleaves; ++l) {
        const int j0 = pk0 + l * pw;
        const int wc = min(pw, pk0 + pnb - j0);
        inner_panel(P, A, pbase, j0, wc, smem, (int*)(smem + (size_t)(r - j0) * (pw + 1)), piv, &s_info, rv,
                    ri, rz, pw);
        PH_MARK(1);
        PH_SUB_BEGIN;
        apply_swaps(A, ldw, piv, pbase, j0, j0 + wc, pk0, j0);
        apply_swaps(A, ldw, piv, pbase, j0, j0 + wc, j0 + wc, pk0 + pnb);
        __syncthreads();
        PH_SUB(10);
        if (l + 1 < nleaves) {
          const int kk = __ffs(~l) - 1;           // trailing ones of l
          const int n1 = (1 << kk) * pw;          // left subtree width
          const int cl = j0 + wc - n1;            // left subtree start column
          const int rc0 = j0 + wc, rc1 = min(rc0 + n1, pk0 + pnb);
          if (n1 <= 8 && rc1 - rc0 <= 8) {  // TRSM fused into the skinny update
            GemmT::run_skinny_trsm<8>(&P.maps, A, ldw, rc0, cl, cl, rc0, rc0, r - rc0, rc1 - rc0, n1, (char*)smem,
                                      &bars, blockIdx.x);
          } else if (n1 <= 16 && rc1 - rc0 <= 16) {
            GemmT::run_skinny_trsm<16>(&P.maps, A, ldw, rc0, cl, cl, rc0, rc0, r - rc0, rc1 - rc0, n1,
                                       (char*)smem, &bars, blockIdx.x);
          } else {
            trsm_small(A, ldw, cl, n1, rc0, rc1, smem);
            __syncthreads();
            PH_SUB(11);
            GemmT::run(&P.maps, A, ldw, rc0, cl, cl, rc0, r - rc0, rc1 - rc0, n1, (char*)smem, &bars,
                       blockIdx.x);
          }
          __syncthreads();
          PH_MARK(2);
        }
      }
    };
    // Outer steps of two 64-column panels with a deferred trailing update of
    // depth 128 (half the C-tile passes, twice the work per C tile): panel 2 is
    // brought up to date by panel 1 (its 64 columns only) and factored; then
    // both panels' interchanges hit the right columns, U12 is solved by block
    // forward substitution (U_a = La^-1 A_top, A_bot -= L21' U_a,
    // U_b = Lb^-1 A_bot) and A22 -= L21 U12 runs once with K = 128.  Row
    // exchanges commute with the deferred row updates because panel 2's
    // exchanges are also applied to panel 1's L columns.
    // (Small orders keep one panel per step: the extra calls of the deferred
    // scheme cost more latency than the deeper trailing GEMM saves.)
    const int mp = r >= DEEP4_MIN_R ? 4 : (r >= DEEP_MIN_R ? 2 : 1);  // panels per outer step
    for (int K0 = 0; K0 < r; K0 += mp * NB) {
      const int nbt = min(mp * NB, r - K0), npan = (nbt + NB - 1) / NB;
      // right-looking LU of the step's columns [K0, K0 + nbt), panel by panel
      for (int pj = 0; pj < npan; ++pj) {
        const int pk0 = K0 + pj * NB, pnb = min(NB, K0 + nbt - pk0), pe = pk0 + pnb;
        factor_panel(pk0, pnb, K0);
        if (pj > 0) {  // this panel's interchanges on the step's earlier L columns
          apply_swaps(A, ldw, piv, K0, pk0, pe, K0, pk0);
          __syncthreads();
        }
        if (pe < K0 + nbt) {  // bring the step's later columns up to date with this panel
          apply_swaps(A, ldw, piv, K0, pk0, pe, pe, K0 + nbt);
          __syncthreads();
          panel_trsm(P, A, pk0, pnb, pe, K0 + nbt, smem, &bars);
          GemmT::run(&P.maps, A, ldw, pe, pk0, pk0, pe, r - pe, K0 + nbt - pe, pnb, (char*)smem, &bars,
                     blockIdx.x);
          __syncthreads();
        }
      }
      const int c0 = K0 + nbt, c1 = r + s;
      apply_swaps(A, ldw, piv, K0, K0, c0, c0, c1);
      __syncthreads();
      PH_MARK(3);
      // U12 = L11^-1 A12 by block forward substitution over the step's panels
      for (int pj = 0; pj < npan; ++pj) {
        const int pk0 = K0 + pj * NB, pnb = min(NB, c0 - pk0), pe = pk0 + pnb;
        panel_trsm(P, A, pk0, pnb, c0, c1, smem, &bars);
        if (pe < c0) {
          GemmT::run(&P.maps, A, ldw, pe, pk0, pk0, c0, c0 - pe, c1 - c0, pnb, (char*)smem, &bars, blockIdx.x);
          __syncthreads();
        }
      }
      PH_MARK(4);
      if (c0 < r) {  // A22 -= L21 U12 with K = the whole step
        GemmT::run(&P.maps, A, ldw, c0, K0, K0, c0, r - c0, c1 - c0, nbt, (char*)smem, &bars, blockIdx.x);
        __syncthreads();
        PH_MARK(5);
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

    PH_MARK(6);
    // ---- outputs: x, y = C_R x (DMMA GEMM), SPL ----
    if (P.x) {
      z_t* xf = P.x + f * (int64_t)r * s;
      for (int idx = tid; idx < r * s; idx += NT) {
        const int i = idx / s, c = idx - i * s;
        xf[idx] = VB_WS_LD(A + (size_t)i * ldw + r + c);
      }
    }
    if (P.n_out > 0 && (P.y || P.spl)) {
      z_t* yt = P.y ? P.y + f * (int64_t)P.n_out * s : yscratch;
      GemmOut::run(yt, s, P.c_r, r, A + r, ldw, P.n_out, s, r, smem);
      __syncthreads();
      if (P.spl) {
        for (int c = warp; c < s; c += NT / 32) {
          double acc = 0.0;
          for (int o = lane; o < P.n_out; o += 32) acc += zabs2(yt[(size_t)o * s + c]);
          acc = warp_sum(acc);
          if (lane == 0) {
            const double prms = sqrt(acc / P.n_out / 2.0);
            P.spl[f * s + c] = 20.0 * log10(fmax(prms, 1e-300) / 20e-6);
          }
        }
      }
    }
    if (tid == 0 && P.info) P.info[f] = s_info;
    PH_MARK(7);
    __syncthreads();
  }
}

static int ldw_of(int r, int s) {
  const int l = (r + s + 3) & ~3;
  return l > NB ? l : NB;  // the U12 scratch rows hold NB columns
}

static size_t smem_bytes(int r, int w) {
  size_t m = GemmT::SMEM > GemmT::SMEM_SKINNY ? GemmT::SMEM : GemmT::SMEM_SKINNY;
  m = m > GemmNarrow::SMEM ? m : GemmNarrow::SMEM;
  m = m > GemmOut::SMEM ? m : GemmOut::SMEM;
  m = m > TRSM_SMEM ? m : TRSM_SMEM;
  m = m > BACK_SMEM ? m : BACK_SMEM;
  const size_t ps = (size_t)r * (w + 1) * sizeof(z_t) + (size_t)r * sizeof(int);  // padded rows + logical ids
  return (m > ps ? m : ps) + 1024;  // + alignment slack for the 1024-B aligned base
}

static const size_t kSmemPerCta = 111 * 1024;  // two CTAs per SM

static int pick_w(int r) {
  for (int w = 16; w >= 1; w >>= 1)
    if (smem_bytes(r, w) <= kSmemPerCta) return w;
  return 0;
}

static size_t cta_stride(int r, int s, int n_out) {
  return ((size_t)(r + NB) * ldw_of(r, s) + (size_t)n_out * s + 7) & ~(size_t)7;
}

}  // namespace blk

// Opt-in (vb_set_l2_persistence): reserving persisting L2 is device-wide state
// that outlives the call, so it is only done while the caller asked for it and
// vb_release_l2_persistence() restores the limit the process had before.
static int g_l2_persist = 0;
static size_t g_l2_prev_limit = 0;
static int g_l2_raised = 0;

void sweep_set_l2_persistence(int enable) { g_l2_persist = enable ? 1 : 0; }

int sweep_release_l2_persistence() {
  VB_CUDA(cudaFree(nullptr));  // make sure the primary context exists
  VB_CUDA(cudaCtxResetPersistingL2Cache());
  if (g_l2_raised) {
    VB_CUDA(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, g_l2_prev_limit));
    g_l2_raised = 0;
  }
  return 0;
}

static int blocked_grid(int64_t F) {
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const int64_t g = 2 * (int64_t)nsm;
  return (int)(F < g ? F : g);
}

size_t sweep_blocked_workspace_bytes(int r, int s, int n_out, int64_t F) {
  return (size_t)blocked_grid(F) * blk::cta_stride(r, s, n_out) * sizeof(z_t);
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int tma_encode_map(CUtensorMap* map, void* base, const cuuint64_t* dims, const cuuint64_t* strides,
                   const cuuint32_t* box, const cuuint32_t* es) {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    VB_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&fn, cudaEnableDefault, &q));
    if (!fn || q != cudaDriverEntryPointSuccess) {
      set_error("cuTensorMapEncodeTiled unavailable");
      return 2;
    }
  }
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, base, dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
    return 2;
  }
  return 0;
}

int sweep_debug_phase_cycles(unsigned long long* out_host, int reset) {
  VB_CUDA(cudaMemcpyFromSymbol(out_host, blk::g_phase_cycles, sizeof(unsigned long long) * 16));
  VB_CUDA(cudaMemcpyFromSymbol(out_host + 16, tma::g_gemm_cycles, sizeof(unsigned long long) * 16));
  if (int rc = lu_debug_cycles(out_host + 32, reset)) return rc;
  if (reset) {
    unsigned long long z[16] = {};
    VB_CUDA(cudaMemcpyToSymbol(blk::g_phase_cycles, z, sizeof(z)));
    VB_CUDA(cudaMemcpyToSymbol(tma::g_gemm_cycles, z, 16 * sizeof(unsigned long long)));
  }
  return 0;
}

int sweep_blocked_supported(int r, int s, int n_out) { return s <= 16 && blk::pick_w(r) > 0; }

int sweep_blocked_launch(int r, int nprim, int s, int n_out, int64_t F, const z_t* prims,
                         const z_t* alpha, const z_t* b, int64_t b_stride_f, const z_t* c_r, z_t* y,
                         double* spl, z_t* x, int* info, void* work, size_t work_bytes,
                         cudaStream_t stream) {
  VB_CHECK_ARG(s <= 16, "vb_rom_sweep (blocked): at most 16 RHS columns");
  VB_CHECK_ARG(nprim <= 64, "vb_rom_sweep (blocked): at most 64 primitives");
  const int w = blk::pick_w(r);
  VB_CHECK_ARG(w > 0, "vb_rom_sweep (blocked): reduced order too large for the inner panel");
  const size_t need = sweep_blocked_workspace_bytes(r, s, n_out, F);
  VB_CHECK_ARG(work != nullptr && work_bytes >= need, "vb_rom_sweep (blocked): workspace too small");
  blk::Params P;
  P.r = r; P.nprim = nprim; P.s = s; P.n_out = n_out; P.F = F;
  P.prims = prims; P.alpha = alpha; P.b = b; P.b_stride_f = b_stride_f; P.c_r = c_r;
  P.y = y; P.spl = spl; P.x = x; P.info = info;
  P.work = (z_t*)work; P.ldw = blk::ldw_of(r, s); P.w = w;
  P.leaf_bytes = (int)(blk::smem_bytes(r, w) - 1024);
  P.cta_stride = blk::cta_stride(r, s, n_out);
  {
    const int grid = blocked_grid(F);
    const cuuint64_t dims[3] = {(cuuint64_t)2 * P.ldw, (cuuint64_t)(r + blk::NB), (cuuint64_t)grid};
    const cuuint64_t strides[2] = {(cuuint64_t)P.ldw * 16, (cuuint64_t)P.cta_stride * 16};
    const cuuint32_t box64[3] = {16, 64, 1}, box16[3] = {16, 16, 1}, es[3] = {1, 1, 1};
    if (int rc = tma_encode_map(&P.maps.a64, work, dims, strides, box64, es)) return rc;
    if (int rc = tma_encode_map(&P.maps.b16, work, dims, strides, box16, es)) return rc;
    const cuuint32_t box8[3] = {16, 8, 1};
    if (int rc = tma_encode_map(&P.maps.b8, work, dims, strides, box8, es)) return rc;
  }
  const size_t smem = blk::smem_bytes(r, w);
  VB_CUDA(cudaFuncSetAttribute(blk::rom_sweep_blocked_kernel,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));

  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(blocked_grid(F));
  cfg.blockDim = dim3(blk::NT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  // Pin the primitives (read by every CTA for every frequency) in L2 so the
  // workspace streaming does not evict them.
  cudaLaunchAttribute attr[1];
  int dev = 0, max_persist = 0, max_window = 0;
  VB_CUDA(cudaGetDevice(&dev));
  cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, dev);
  cudaDeviceGetAttribute(&max_window, cudaDevAttrMaxAccessPolicyWindowSize, dev);
  const size_t pbytes = (size_t)nprim * r * r * sizeof(z_t);
  if (g_l2_persist && max_persist > 0 && max_window > 0) {
    const size_t win = pbytes < (size_t)max_window ? pbytes : (size_t)max_window;
    const size_t lim = win < (size_t)max_persist ? win : (size_t)max_persist;
    size_t cur = 0;
    cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize);
    if (cur < lim) {
      if (!g_l2_raised) {
        g_l2_prev_limit = cur;
        g_l2_raised = 1;
      }
      cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, lim);
    }
    attr[0].id = cudaLaunchAttributeAccessPolicyWindow;
    attr[0].val.accessPolicyWindow.base_ptr = (void*)prims;
    attr[0].val.accessPolicyWindow.num_bytes = win;
    attr[0].val.accessPolicyWindow.hitRatio = (float)((double)lim / (double)win);
    attr[0].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    attr[0].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
  }
  cudaGetLastError();  // clear any error from the optional persistence queries
  VB_CUDA(cudaLaunchKernelEx(&cfg, blk::rom_sweep_blocked_kernel, P));
  VB_LAUNCHED("rom_sweep_blocked_kernel");
  return 0;
}

}  // namespace vb
