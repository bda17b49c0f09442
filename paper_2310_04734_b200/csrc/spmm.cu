// Real-CSR x complex-dense SpMM, Y = alpha A X + beta Y (SURVEY §8a A9 first
// half; replaces scipy csr_matvecs in `K @ V`, `M @ v`, vibrofem/mor.py:81-85,
// 117, 162-179).  X, Y complex128 row-major (n x k, row stride ldx / ldy).
//
// Three kernels by column count:
//  * k <= 2   SpMV-like: 8 lanes per row, 4 loads in flight per lane, both
//             columns per lane, fixed-order shuffle reduction.
//  * (k <= 16 sub-warp CSR, used below the row-group threshold or without groups): KP = next_pow2(k) lanes per row, 32/KP rows per
//             warp; the row's (value, index) pairs are loaded KP at a time,
//             coalesced, and broadcast inside the sub-warp by shuffle.  One
//             128-B X piece per nonzero and warp instruction: no idle lanes.
//  * k > 16   row groups (`vb_csr_row_groups`): up to 8 rows whose column sets
//             are subsets of one "leader" row's set form a dense 8 x nu block
//             over the leader's columns (absent slots +0.0); the block times
//             the gathered X rows runs on the FP64 tensor cores (DMMA) with
//             the X rows staged through a cp.async ring.  Each X row is read
//             once per group instead of once per nonzero (hex27 2x2x2 node
//             blocks: 512 nonzeros over 125 columns = 4.1x less gather
//             traffic).  Column chunks are the FAST grid dimension
//             so a group tile's value rows are read from DRAM once for all chunks.
#include "common.cuh"
#include "sweep.cuh"
#include "mma.cuh"

#include <algorithm>
#include <cstdlib>
#include <vector>

namespace vb {

// ------------------------------------------------------------- k = 1, 2 ---
// SpMV-like: SW lanes per row (32/SW rows per warp), each lane strides its row
// by SW with 4 independent (value, index, x) loads in flight and keeps all KC
// columns of its nonzeros, then a fixed-order shuffle reduction.
template <int SW, int KC>
__global__ void __launch_bounds__(256) spmv_kernel(int n_rows, const int32_t* __restrict__ indptr,
                                                   const int32_t* __restrict__ indices,
                                                   const double* __restrict__ vals, const z_t* __restrict__ X,
                                                   int64_t ldx, z_t* __restrict__ Y, int64_t ldy, z_t alpha,
                                                   z_t beta) {
  constexpr int RPW = 32 / SW;
  const int lane = threadIdx.x & 31, sl = lane % SW;
  const int64_t sw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / SW;
  const int64_t nsw = ((int64_t)gridDim.x * blockDim.x) / SW;
  const bool beta0 = beta.x == 0.0 && beta.y == 0.0;
  const int64_t nr_pad = ((int64_t)n_rows + RPW - 1) / RPW * RPW;  // whole warps stay converged
  for (int64_t row = sw; row < nr_pad; row += nsw) {
    const bool rv = row < n_rows;
    const int b = rv ? __ldg(indptr + row) : 0, e = rv ? __ldg(indptr + row + 1) : 0;
    double re[KC], im[KC];
#pragma unroll
    for (int c = 0; c < KC; ++c) re[c] = im[c] = 0.0;
    int j = b + sl;
    for (; j + 3 * SW < e; j += 4 * SW) {
      double a[4];
      int ci[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        a[u] = __ldg(vals + j + u * SW);
        ci[u] = __ldg(indices + j + u * SW);
      }
      z_t x[4][KC];
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int c = 0; c < KC; ++c) x[u][c] = __ldg(X + (int64_t)ci[u] * ldx + c);
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int c = 0; c < KC; ++c) {
          re[c] = fma(a[u], x[u][c].x, re[c]);
          im[c] = fma(a[u], x[u][c].y, im[c]);
        }
    }
    for (; j < e; j += SW) {
      const double a = __ldg(vals + j);
      VB_DCHECK(__ldg(indices + j) >= 0);  // (row-compacted CSRs: columns may exceed n_rows)
      const z_t* xr = X + (int64_t)__ldg(indices + j) * ldx;
#pragma unroll
      for (int c = 0; c < KC; ++c) {
        const z_t x = __ldg(xr + c);
        re[c] = fma(a, x.x, re[c]);
        im[c] = fma(a, x.y, im[c]);
      }
    }
#pragma unroll
    for (int o = SW / 2; o > 0; o >>= 1)
#pragma unroll
      for (int c = 0; c < KC; ++c) {
        re[c] += __shfl_xor_sync(0xffffffffu, re[c], o);
        im[c] += __shfl_xor_sync(0xffffffffu, im[c], o);
      }
    if (rv && sl == 0) {
#pragma unroll
      for (int c = 0; c < KC; ++c) {
        z_t out = zmul(alpha, zmake(re[c], im[c]));
        if (!beta0) out = zfma(out, beta, Y[row * ldy + c]);
        Y[row * ldy + c] = out;
      }
    }
  }
}

// --------------------------------------------------------------- k <= 16 ---
template <int KP>
__global__ void __launch_bounds__(256) spmm_subwarp_kernel(int n_rows, const int32_t* __restrict__ indptr,
                                                           const int32_t* __restrict__ indices,
                                                           const double* __restrict__ vals, int k,
                                                           const z_t* __restrict__ X, int64_t ldx,
                                                           z_t* __restrict__ Y, int64_t ldy, z_t alpha,
                                                           z_t beta) {
  constexpr int RPW = 32 / KP;  // rows per warp
  const int lane = threadIdx.x & 31, sub = lane / KP, c = lane % KP;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const bool beta0 = beta.x == 0.0 && beta.y == 0.0;
  const bool cv = c < k;
  for (int64_t row0 = warp * RPW; row0 < n_rows; row0 += nwarps * RPW) {
    const int64_t row = row0 + sub;
    const bool rv = row < n_rows;
    const int b = rv ? __ldg(indptr + row) : 0;
    const int len = rv ? __ldg(indptr + row + 1) - b : 0;
    int mlen = len;  // trip count of the whole warp (shuffles need all lanes)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mlen = max(mlen, __shfl_xor_sync(0xffffffffu, mlen, o));
    double ar = 0.0, ai = 0.0;
    for (int j0 = 0; j0 < mlen; j0 += KP) {
      double v = 0.0;
      int col = 0;
      if (j0 + c < len) {
        v = __ldg(vals + b + j0 + c);
        col = __ldg(indices + b + j0 + c);
        VB_DCHECK(col >= 0);
      }
      const int cnt = min(KP, mlen - j0);
#pragma unroll 4
      for (int q = 0; q < cnt; ++q) {
        const double a = __shfl_sync(0xffffffffu, v, q, KP);
        const int cc = __shfl_sync(0xffffffffu, col, q, KP);
        if (cv && j0 + q < len) {
          const z_t x = __ldg(X + (int64_t)cc * ldx + c);
          ar = fma(a, x.x, ar);
          ai = fma(a, x.y, ai);
        }
      }
    }
    if (rv && cv) {
      z_t out = zmul(alpha, zmake(ar, ai));
      if (!beta0) out = zfma(out, beta, Y[row * ldy + c]);
      Y[row * ldy + c] = out;
    }
  }
}

// ------------------------------------------------------------- row groups ---
constexpr int RG = 8;  // rows per group
#ifndef VB_RG_S
#define VB_RG_S 3  // cp.async ring stages of the row-group kernels
#endif
#ifndef VB_RG_CC_MIN_K
#define VB_RG_CC_MIN_K 1000000  // set after measuring (tools/bench_offline.py, VB_RG_MODE)
#endif
constexpr int RG_CC_MIN_K = VB_RG_CC_MIN_K;

// Row-group SpMM on the FP64 tensor cores.  One warp per group: the group's
// rows x leader columns form a dense 8 x nu real block (absent slots +0.0),
// so Y[8 rows, chunk] = Vals[8, nu] . X[leader columns, chunk] is a real GEMM
// over the interleaved (re, im) columns of X: DMMA m8n8k4 with A = 8 rows x
// 4 leader columns of values, B = 4 X rows x 8 real columns, and each lane's
// (c0, c1) accumulator pair = one complex output (row = lane/4, complex
// column = 4t + lane%4).  The X rows of the leader's columns and the value
// rows stream through a per-warp cp.async ring in shared memory (S stages of
// J leader columns, zero-filled past the row end / past k): the gathers are
// in flight without holding registers and each X row is read once for all 8
// member rows.  X stage rows and value rows are padded by 32 B so that the
// fragment loads of a half-warp (4 rows x 4 consecutive doubles) fall on 4
// distinct 8-bank ranges (conflict-free).
template <int CW_, int J, int S>
struct RgCfg {
  static constexpr int CW = CW_;                             // complex columns per chunk (8..64)
  static constexpr int RS = 2 * CW + 4;                      // doubles per X stage row (padded)
  static constexpr int VR = RG + 4;                          // doubles per value row (padded)
  static constexpr int XS = J * RS;                          // doubles per X stage
  static constexpr int VS = J * VR;                          // doubles per value stage
  static constexpr int WARP_BYTES = S * (XS + VS) * 8;       // per warp
  static constexpr int NT = 2 * CW / 8;                      // 8-wide real n-tiles
};

constexpr int RG_WARPS = 4;
#ifndef VB_RG_CHUNK_FAST
#define VB_RG_CHUNK_FAST 1  // the chunks of a group tile run together: its value rows are read from DRAM once
#endif

// CC = true: the same staging, but the products on the CUDA cores without the
// padding (see rg_cc below): lane <-> complex column, the 8 member rows'
// accumulators in registers, each staged X element fused into exactly the
// rows present at that slot (its 8-bit mask, uniform over the warp).
template <int CW, int J, int S, bool CC = false>
__global__ void __launch_bounds__(32 * RG_WARPS) rg_spmm_kernel(int n_groups, const int32_t* __restrict__ g_leader,
                                                                const int32_t* __restrict__ g_rows,
                                                                const int32_t* __restrict__ g_uoff,
                                                                const int32_t* __restrict__ indptr,
                                                                const int32_t* __restrict__ indices,
                                                                const double* __restrict__ gvals, int k,
                                                                const z_t* __restrict__ X, int64_t ldx,
                                                                z_t* __restrict__ Y, int64_t ldy, z_t alpha,
                                                                z_t beta, const uint8_t* __restrict__ masks = nullptr) {
  using C = RgCfg<CW, J, S>;
  static_assert(J % 4 == 0 && 32 % J == 0, "stages of whole k4 steps inside one 32-column index block");
  static_assert((J * CW) % 32 == 0 && (J * RG / 2) % 32 == 0 || J * RG / 2 < 32, "copy rounds");
  constexpr int XP = J * CW / 32;                 // 16-B X pieces per lane per stage
  constexpr int VP = (J * RG / 2 + 31) / 32;      // 16-B value pieces per lane per stage
  extern __shared__ __align__(16) unsigned char rg_smem[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int gid = lane >> 2, tig = lane & 3;
#if VB_RG_CHUNK_FAST
  const int g = blockIdx.y * RG_WARPS + w;
#else
  const int g = blockIdx.x * RG_WARPS + w;
#endif
  if (g >= n_groups) return;
  double* xs = reinterpret_cast<double*>(rg_smem + (size_t)w * C::WARP_BYTES);
  double* vs = xs + S * C::XS;
#if VB_RG_CHUNK_FAST
  const int c0 = blockIdx.x * C::CW;  // first complex column of the chunk
#else
  const int c0 = blockIdx.y * C::CW;  // first complex column of the chunk
#endif
  const int leader = __ldg(g_leader + g);  // -1: a group of empty rows (Y = beta Y)
  const int ub = leader >= 0 ? __ldg(indptr + leader) : 0;
  const int nu = leader >= 0 ? __ldg(indptr + leader + 1) - ub : 0;
  const double* uv = gvals + (int64_t)__ldg(g_uoff + g) * RG;
  const int nst = (nu + J - 1) / J;  // stages of J leader columns
  int colv = 0;                      // leader columns of the current 32-block, lane-parallel
  auto issue = [&](int st) {
    const int slot = st % S;
    const int j0 = st * J;
    if ((j0 & 31) == 0) colv = j0 + lane < nu ? __ldg(indices + ub + j0 + lane) : 0;
    if constexpr (CW >= 32) {  // one X row per step, CW / 32 pieces per lane
#pragma unroll
      for (int jj = 0; jj < J; ++jj) {
        const int j = j0 + jj;
        const int col = __shfl_sync(0xffffffffu, colv, j & 31);
        const z_t* xr = X + (int64_t)col * ldx + c0 + lane;
#pragma unroll
        for (int t = 0; t < CW / 32; ++t) {
          const bool ok = j < nu && c0 + lane + 32 * t < k;
          blk::cp_async16(xs + slot * C::XS + jj * C::RS + 2 * (lane + 32 * t), ok ? xr + 32 * t : X, ok);
        }
      }
    } else {  // 32 / CW rows per step: piece p = lane + 32 m is row p / CW, column p % CW
#pragma unroll
      for (int m = 0; m < XP; ++m) {
        const int p = lane + 32 * m, jj = p / CW, c = p % CW, j = j0 + jj;
        const int col = __shfl_sync(0xffffffffu, colv, j & 31);
        const bool ok = j < nu && c0 + c < k;
        blk::cp_async16(xs + slot * C::XS + jj * C::RS + 2 * c, ok ? X + (int64_t)col * ldx + c0 + c : X, ok);
      }
    }
#pragma unroll
    for (int m = 0; m < VP; ++m) {  // J value rows of 8 doubles = J*4 pieces of 16 B
      const int p = lane + 32 * m, jj = p >> 2, j = j0 + jj;
      if (jj < J)
        blk::cp_async16(vs + slot * C::VS + jj * C::VR + 2 * (p & 3),
                        j < nu ? uv + (int64_t)j0 * RG + 2 * p : gvals, j < nu);
    }
    blk::cp_commit();
  };
  constexpr int NACC = CC ? 1 : C::NT;
  double acc[NACC][2];
#pragma unroll
  for (int t = 0; t < NACC; ++t) acc[t][0] = acc[t][1] = 0.0;
  constexpr int CPL = CC ? C::CW / 32 : 1;  // complex columns per lane (CUDA-core form)
  double ar[CPL][RG], ai[CPL][RG];
  if constexpr (CC) {
#pragma unroll
    for (int t = 0; t < CPL; ++t)
#pragma unroll
      for (int i = 0; i < RG; ++i) ar[t][i] = ai[t][i] = 0.0;
  }
  const uint8_t* mk = CC ? masks + __ldg(g_uoff + g) : nullptr;
#pragma unroll
  for (int st = 0; st < S - 1; ++st) {
    if (st < nst) issue(st);
    else blk::cp_commit();
  }
  for (int st = 0; st < nst; ++st) {
    blk::cp_wait<S - 2>();
    __syncwarp();
    const double* xsl = xs + (st % S) * C::XS;
    const double* vsl = vs + (st % S) * C::VS;
    if constexpr (!CC) {
#pragma unroll
      for (int q = 0; q < J / 4; ++q) {
        const double a = vsl[(4 * q + tig) * C::VR + gid];  // A[row gid][k tig]
        const double* xb = xsl + (4 * q + tig) * C::RS + gid;  // B[k tig][n gid]
#pragma unroll
        for (int t = 0; t < C::NT; ++t) blk::dmma(acc[t][0], acc[t][1], a, xb[8 * t]);
      }
    } else {
      const int jb = st * J;
#pragma unroll
      for (int q = 0; q < J; ++q) {
        const unsigned m = jb + q < nu ? __ldg(mk + jb + q) : 0u;  // uniform: one broadcast load
        const double2* vq = reinterpret_cast<const double2*>(vsl + q * C::VR);
        double2 v[RG / 2];
#pragma unroll
        for (int h = 0; h < RG / 2; ++h) v[h] = vq[h];
#pragma unroll
        for (int t = 0; t < CPL; ++t) {
          const double2 x = *reinterpret_cast<const double2*>(xsl + q * C::RS + 2 * (lane + 32 * t));
#pragma unroll
          for (int i = 0; i < RG; ++i)
            if ((m >> i) & 1u) {
              const double a = (i & 1) ? v[i >> 1].y : v[i >> 1].x;
              ar[t][i] = fma(a, x.x, ar[t][i]);
              ai[t][i] = fma(a, x.y, ai[t][i]);
            }
        }
      }
    }
    __syncwarp();
    if (st + S - 1 < nst) issue(st + S - 1);
    else blk::cp_commit();
  }
  if constexpr (CC) {
    const bool beta0 = beta.x == 0.0 && beta.y == 0.0;
#pragma unroll
    for (int i = 0; i < RG; ++i) {
      const int row = __ldg(g_rows + (int64_t)g * RG + i);
      if (row < 0) continue;
#pragma unroll
      for (int t = 0; t < CPL; ++t) {
        const int c = c0 + lane + 32 * t;
        if (c >= k) continue;
        z_t* yp = Y + (int64_t)row * ldy + c;
        z_t out = zmul(alpha, zmake(ar[t][i], ai[t][i]));
        if (!beta0) out = zfma(out, beta, *yp);
        *yp = out;
      }
    }
    return;
  }
  const int row = __ldg(g_rows + (int64_t)g * RG + gid);
  if (row < 0) return;
  const bool beta0 = beta.x == 0.0 && beta.y == 0.0;
  z_t* yr = Y + (int64_t)row * ldy + c0;
#pragma unroll
  for (int t = 0; t < C::NT; ++t) {
    const int c = 4 * t + tig;  // complex column inside the chunk
    if (c0 + c >= k) continue;
    z_t out = zmul(alpha, zmake(acc[t][0], acc[t][1]));
    if (!beta0) out = zfma(out, beta, yr[c]);
    yr[c] = out;
  }
}

// Row-group SpMM on the CUDA cores (FP64 FMA pipe), padding-free: the DMMA
// kernel above multiplies the whole dense 8 x nu block (on hex27 only 512 of
// its 1,000 slots are nonzero), so it is bound by the FP64 pipe on padding.
// Here each lane owns one complex column of a CW-wide chunk and keeps the 8
// member rows' accumulators in registers; for every union column j of the
// group the X element is loaded ONCE and fused into exactly the member rows
// present at j (the group's 8-bit mask: the same for all lanes of the
// sub-warp, so the branches do not diverge).  Per nonzero: 2 DFMA; per union
// slot: one 16-byte X load per lane plus uniform (broadcast) loads of the
// slot's column id, mask and 8 values.  G = 32 / CW groups per warp.
template <int CW>
__global__ void __launch_bounds__(256) rg_cc_kernel(int n_groups, const int32_t* __restrict__ g_leader,
                                                    const int32_t* __restrict__ g_rows,
                                                    const int32_t* __restrict__ g_uoff,
                                                    const int32_t* __restrict__ indptr,
                                                    const int32_t* __restrict__ indices,
                                                    const uint8_t* __restrict__ masks,
                                                    const double* __restrict__ gvals, int k,
                                                    const z_t* __restrict__ X, int64_t ldx, z_t* __restrict__ Y,
                                                    int64_t ldy, z_t alpha, z_t beta) {
  constexpr int G = 32 / CW;
  const int lane = threadIdx.x & 31, sub = lane / CW, c = lane % CW;
  const int64_t g = ((int64_t)blockIdx.y * (blockDim.x >> 5) + (threadIdx.x >> 5)) * G + sub;
  const int col = blockIdx.x * CW + c;
  const bool cv = col < k;
  if (g >= n_groups) return;
  const int leader = __ldg(g_leader + g);
  const int ub = leader >= 0 ? __ldg(indptr + leader) : 0;
  const int nu = leader >= 0 ? __ldg(indptr + leader + 1) - ub : 0;
  const int64_t uo = __ldg(g_uoff + g);
  const int32_t* cols = indices + ub;
  const uint8_t* mk = masks + uo;
  const double2* vv = reinterpret_cast<const double2*>(gvals + uo * RG);
  double ar[RG], ai[RG];
#pragma unroll
  for (int i = 0; i < RG; ++i) ar[i] = ai[i] = 0.0;
  const z_t* Xc = X + (cv ? col : 0);
  constexpr int U = 4;  // union slots in flight
  int j = 0;
  for (; j + U <= nu; j += U) {
    z_t x[U];
    unsigned m[U];
    double2 v[U][RG / 2];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      x[u] = cv ? __ldg(Xc + (int64_t)__ldg(cols + j + u) * ldx) : zmake(0.0, 0.0);
      m[u] = __ldg(mk + j + u);
#pragma unroll
      for (int h = 0; h < RG / 2; ++h) v[u][h] = __ldg(vv + (int64_t)(j + u) * (RG / 2) + h);
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int i = 0; i < RG; ++i)
        if ((m[u] >> i) & 1u) {
          const double a = (i & 1) ? v[u][i >> 1].y : v[u][i >> 1].x;
          ar[i] = fma(a, x[u].x, ar[i]);
          ai[i] = fma(a, x[u].y, ai[i]);
        }
  }
  for (; j < nu; ++j) {
    const z_t x = cv ? __ldg(Xc + (int64_t)__ldg(cols + j) * ldx) : zmake(0.0, 0.0);
    const unsigned m = __ldg(mk + j);
#pragma unroll
    for (int i = 0; i < RG; ++i)
      if ((m >> i) & 1u) {
        const double a = __ldg(gvals + (uo + j) * RG + i);
        ar[i] = fma(a, x.x, ar[i]);
        ai[i] = fma(a, x.y, ai[i]);
      }
  }
  if (!cv) return;
  const bool beta0 = beta.x == 0.0 && beta.y == 0.0;
#pragma unroll
  for (int i = 0; i < RG; ++i) {
    const int row = __ldg(g_rows + g * RG + i);
    if (row < 0) continue;
    z_t out = zmul(alpha, zmake(ar[i], ai[i]));
    if (!beta0) out = zfma(out, beta, Y[(int64_t)row * ldy + col]);
    Y[(int64_t)row * ldy + col] = out;
  }
}

template <int CW>
static int rg_cc_launch(int n_groups, const int32_t* g_leader, const int32_t* g_rows, const int32_t* g_uoff,
                        const int32_t* indptr, const int32_t* indices, const uint8_t* masks, const double* gvals,
                        int k, const z_t* X, int64_t ldx, z_t* Y, int64_t ldy, z_t alpha, z_t beta,
                        cudaStream_t st) {
  constexpr int G = 32 / CW, WARPS = 8;
  const int64_t warps = ((int64_t)n_groups + G - 1) / G;
  const dim3 grid((unsigned)((k + CW - 1) / CW), (unsigned)((warps + WARPS - 1) / WARPS));
  rg_cc_kernel<CW><<<grid, 32 * WARPS, 0, st>>>(n_groups, g_leader, g_rows, g_uoff, indptr, indices, masks, gvals,
                                                k, X, ldx, Y, ldy, alpha, beta);
  VB_LAUNCHED("rg_cc_kernel");
  return 0;
}

__global__ void rg_gather_values_kernel(int64_t n_slots, const int32_t* __restrict__ vmap,
                                        const double* __restrict__ vals, double* __restrict__ gvals) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_slots;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t p = vmap[i];
    gvals[i] = p >= 0 ? vals[p] : 0.0;
  }
}

// Host-side grouping of a CSR pattern (one-off per pattern, O(nnz) merges).
// Greedy in row order: an ungrouped row becomes a leader and adopts up to 7
// ungrouped rows among its own columns whose column sets are subsets of its
// set (scanned in column order).  On lexicographically numbered hex27 boxes
// this yields the 2x2x2 node blocks (vertex node as leader).
int csr_row_groups(int n, const int32_t* indptr, const int32_t* indices, int32_t* g_leader, int32_t* g_rows,
                   int32_t* g_uoff, uint8_t* masks, int32_t* vmap, int* n_groups, int64_t* n_slots) {
  std::vector<char> grouped(n, 0);
  int G = 0;
  int64_t uoff = 0;
  std::vector<int> empty;  // empty rows: packed 8 per leaderless group at the end
  for (int r = 0; r < n; ++r) {
    if (grouped[r]) continue;
    grouped[r] = 1;
    const int rb = indptr[r], re = indptr[r + 1];
    if (rb == re) {
      empty.push_back(r);
      continue;
    }
    int mem[RG];
    int nm = 0;
    mem[nm++] = r;
    for (int j = rb; j < re && nm < RG; ++j) {
      const int c = indices[j];
      if (c < 0 || c >= n || grouped[c] || indptr[c] == indptr[c + 1]) continue;  // empty rows: packed apart
      // subset test: row c's columns inside row r's columns (both sorted)
      int p = rb;
      bool sub = true;
      for (int q = indptr[c]; q < indptr[c + 1]; ++q) {
        while (p < re && indices[p] < indices[q]) ++p;
        if (p == re || indices[p] != indices[q]) { sub = false; break; }
      }
      if (!sub) continue;
      grouped[c] = 1;
      mem[nm++] = c;
    }
    if (uoff + (re - rb) > INT32_MAX) return 1;
    g_leader[G] = r;
    g_uoff[G] = (int32_t)uoff;
    for (int i = 0; i < RG; ++i) g_rows[(int64_t)G * RG + i] = i < nm ? mem[i] : -1;
    for (int j = rb; j < re; ++j) {
      masks[uoff + (j - rb)] = 0;
      for (int i = 0; i < RG; ++i) vmap[(uoff + (j - rb)) * RG + i] = -1;
    }
    for (int i = 0; i < nm; ++i) {
      const int rr = mem[i];
      int p = rb;
      for (int q = indptr[rr]; q < indptr[rr + 1]; ++q) {
        while (indices[p] < indices[q]) ++p;  // present by the subset test (leader: itself)
        masks[uoff + (p - rb)] |= (uint8_t)(1u << i);
        vmap[(uoff + (p - rb)) * RG + i] = q;
      }
    }
    uoff += re - rb;
    ++G;
  }
  for (size_t e0 = 0; e0 < empty.size(); e0 += RG) {  // Y rows only scaled by beta
    g_leader[G] = -1;
    g_uoff[G] = 0;
    for (int i = 0; i < RG; ++i) g_rows[(int64_t)G * RG + i] = e0 + i < empty.size() ? empty[e0 + i] : -1;
    ++G;
  }
  *n_groups = G;
  *n_slots = uoff;
  return 0;
}

int rg_gather_values(int64_t n_union, const int32_t* vmap, const double* vals, double* gvals, cudaStream_t st) {
  if (n_union <= 0) return 0;
  const int64_t n = n_union * RG;
  const unsigned grid = (unsigned)std::min<int64_t>((n + 255) / 256, 148 * 32);
  rg_gather_values_kernel<<<grid, 256, 0, st>>>(n, vmap, vals, gvals);
  VB_LAUNCHED("rg_gather_values_kernel");
  return 0;
}

template <int CW, int J, int S, bool CC = false>
static int rg_launch(int n_groups, const int32_t* g_leader, const int32_t* g_rows, const int32_t* g_uoff,
                     const int32_t* indptr, const int32_t* indices, const double* gvals, int k, const z_t* X,
                     int64_t ldx, z_t* Y, int64_t ldy, z_t alpha, z_t beta, cudaStream_t st,
                     const uint8_t* masks = nullptr) {
  constexpr int smem = RG_WARPS * RgCfg<CW, J, S>::WARP_BYTES;
  static bool attr = false;
  if (!attr) {
    VB_CUDA(cudaFuncSetAttribute(rg_spmm_kernel<CW, J, S, CC>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr = true;
  }
#if VB_RG_CHUNK_FAST
  const dim3 grid((unsigned)((k + CW - 1) / CW), (unsigned)((n_groups + RG_WARPS - 1) / RG_WARPS));
#else
  const dim3 grid((unsigned)((n_groups + RG_WARPS - 1) / RG_WARPS), (unsigned)((k + CW - 1) / CW));
#endif
  rg_spmm_kernel<CW, J, S, CC><<<grid, 32 * RG_WARPS, smem, st>>>(n_groups, g_leader, g_rows, g_uoff, indptr,
                                                                  indices, gvals, k, X, ldx, Y, ldy, alpha, beta,
                                                                  masks);
  VB_LAUNCHED("rg_spmm_kernel");
  return 0;
}

static int g_rg_mode = -1;  // 0 auto, 1 tensor-core (DMMA) groups, 2 CUDA-core groups

void set_rg_mode(int m) { g_rg_mode = m; }

static int rg_mode() {
  if (g_rg_mode < 0) {
    const char* e = getenv("VB_RG_MODE");
    g_rg_mode = e ? atoi(e) : 0;
  }
  return g_rg_mode;
}

int rg_spmm(int n_groups, const int32_t* g_leader, const int32_t* g_rows, const int32_t* g_uoff,
            const int32_t* indptr, const int32_t* indices, const uint8_t* masks, const double* gvals, int k,
            const z_t* X, int64_t ldx, z_t* Y, int64_t ldy, z_t alpha, z_t beta, cudaStream_t st) {
  if (n_groups <= 0 || k <= 0) return 0;
  const int mode = rg_mode();
  if (masks && k > 16 && (mode == 2 || (mode == 0 && k >= RG_CC_MIN_K))) {  // staged CUDA-core groups
    if (k <= 32) return rg_launch<32, 4, VB_RG_S, true>(n_groups, g_leader, g_rows, g_uoff, indptr, indices, gvals,
                                                        k, X, ldx, Y, ldy, alpha, beta, st, masks);
    return rg_launch<64, 4, VB_RG_S, true>(n_groups, g_leader, g_rows, g_uoff, indptr, indices, gvals, k, X, ldx,
                                           Y, ldy, alpha, beta, st, masks);
  }
  if (masks && mode == 3) {  // direct-gather CUDA-core groups (no staging)
    if (k <= 8) return rg_cc_launch<8>(n_groups, g_leader, g_rows, g_uoff, indptr, indices, masks, gvals, k, X, ldx,
                                       Y, ldy, alpha, beta, st);
    if (k <= 16) return rg_cc_launch<16>(n_groups, g_leader, g_rows, g_uoff, indptr, indices, masks, gvals, k, X,
                                         ldx, Y, ldy, alpha, beta, st);
    return rg_cc_launch<32>(n_groups, g_leader, g_rows, g_uoff, indptr, indices, masks, gvals, k, X, ldx, Y, ldy,
                            alpha, beta, st);
  }
#define VB_RG(CW, J) \
  return rg_launch<CW, J, VB_RG_S>(n_groups, g_leader, g_rows, g_uoff, indptr, indices, gvals, k, X, ldx, Y, ldy, alpha, beta, st)
#ifndef VB_RG_J8
#define VB_RG_J8 8
#endif
#ifndef VB_RG_J16
#define VB_RG_J16 4
#endif
  if (k <= 8) VB_RG(8, VB_RG_J8);
  if (k <= 16) VB_RG(16, VB_RG_J16);
  if (k <= 32) VB_RG(32, 4);
  VB_RG(64, 4);
#undef VB_RG
}

// ------------------------------------------------------------ dispatcher ---
constexpr int SPMM_CW = 64;

// k > 16 without row groups: one warp per row, lane l owns columns l, l+32 of
// a 64-column chunk (chunk = slow grid dimension, X slab L2-resident).
__global__ void spmm_chunked_kernel(int n_rows, const int32_t* __restrict__ indptr,
                                    const int32_t* __restrict__ indices, const double* __restrict__ vals,
                                    int k, const z_t* __restrict__ X, int64_t ldx, z_t* __restrict__ Y,
                                    int64_t ldy, z_t alpha, z_t beta) {
  const int lane = threadIdx.x & 31;
  const int64_t row = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (row >= n_rows) return;
  const int c0 = blockIdx.y * SPMM_CW + lane, c1 = c0 + 32;
  const bool v0 = c0 < k, v1 = c1 < k;
  const int b = __ldg(indptr + row), e = __ldg(indptr + row + 1);
  z_t a0 = zmake(0.0, 0.0), a1 = zmake(0.0, 0.0);
  for (int j0 = b; j0 < e; j0 += 32) {
    double v = 0.0;
    int col = 0;
    if (j0 + lane < e) {
      v = __ldg(vals + j0 + lane);
      col = __ldg(indices + j0 + lane);
    }
    const int cnt = min(32, e - j0);
#pragma unroll 4
    for (int q = 0; q < cnt; ++q) {
      const double a = __shfl_sync(0xffffffffu, v, q);
      const int cc = __shfl_sync(0xffffffffu, col, q);
      const z_t* xr = X + (int64_t)cc * ldx;
      if (v0) { const z_t x = __ldg(xr + c0); a0.x = fma(a, x.x, a0.x); a0.y = fma(a, x.y, a0.y); }
      if (v1) { const z_t x = __ldg(xr + c1); a1.x = fma(a, x.x, a1.x); a1.y = fma(a, x.y, a1.y); }
    }
  }
  const bool beta0 = beta.x == 0.0 && beta.y == 0.0;
  if (v0) {
    z_t out = zmul(alpha, a0);
    if (!beta0) out = zfma(out, beta, Y[row * ldy + c0]);
    Y[row * ldy + c0] = out;
  }
  if (v1) {
    z_t out = zmul(alpha, a1);
    if (!beta0) out = zfma(out, beta, Y[row * ldy + c1]);
    Y[row * ldy + c1] = out;
  }
}

int csr_spmm(int n_rows, const int32_t* indptr, const int32_t* indices, const double* vals, int k,
             const z_t* X, int64_t ldx, z_t* Y, int64_t ldy, z_t alpha, z_t beta, cudaStream_t st) {
  if (n_rows <= 0 || k <= 0) return 0;
  const int nt = 256;
  if (k > 16) {
    const dim3 grid((unsigned)(((int64_t)n_rows * 32 + nt - 1) / nt), (unsigned)((k + SPMM_CW - 1) / SPMM_CW));
    spmm_chunked_kernel<<<grid, nt, 0, st>>>(n_rows, indptr, indices, vals, k, X, ldx, Y, ldy, alpha, beta);
    VB_LAUNCHED("spmm_chunked_kernel");
    return 0;
  }
  auto grid_for = [&](int rows_per_warp) {
    int64_t warps = ((int64_t)n_rows + rows_per_warp - 1) / rows_per_warp;
    return (unsigned)std::min<int64_t>((warps * 32 + nt - 1) / nt, 148 * 64);
  };
  if (k == 1) {
    spmv_kernel<8, 1><<<grid_for(4), nt, 0, st>>>(n_rows, indptr, indices, vals, X, ldx, Y, ldy, alpha, beta);
  } else if (k == 2) {
    spmv_kernel<8, 2><<<grid_for(4), nt, 0, st>>>(n_rows, indptr, indices, vals, X, ldx, Y, ldy, alpha, beta);
  } else if (k <= 4) {
    spmm_subwarp_kernel<4><<<grid_for(8), nt, 0, st>>>(n_rows, indptr, indices, vals, k, X, ldx, Y, ldy, alpha, beta);
  } else if (k <= 8) {
    spmm_subwarp_kernel<8><<<grid_for(4), nt, 0, st>>>(n_rows, indptr, indices, vals, k, X, ldx, Y, ldy, alpha, beta);
  } else {
    spmm_subwarp_kernel<16><<<grid_for(2), nt, 0, st>>>(n_rows, indptr, indices, vals, k, X, ldx, Y, ldy, alpha, beta);
  }
  VB_LAUNCHED("spmm_kernel");
  return 0;
}

}  // namespace vb
