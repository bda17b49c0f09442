// Large-tile TMA + mbarrier complex GEMM for kernels that own a whole SM (one
// CTA per SM, up to 255 registers and ~200 KB of shared memory): the trailing
// update of the full-order LU (csrc/lu.cu).  C[M x N] -= A[M x K] B[K x N].
//
//  * 128 x 64 complex tiles, 8 warps as 4 (M) x 2 (N), 32 x 32 per warp: 4 x 4
//    DMMA fragments with separate re/im accumulators (64 doubles per lane), so
//    each A/B fragment pair loaded from shared memory feeds 8 DMMAs (twice the
//    reuse of the 64 x 32 tiles in tma.cuh).
//  * k chunks of 8 complex: A = 2 boxes of 64 rows x 8 complex, B = 8 boxes of
//    8 rows x 8 complex, 128B-swizzled, in a STAGES-deep ring (full/empty
//    mbarriers; the box issue is spread over 4 producer warps, each issuing
//    warp-collectively); the next C tile (16 boxes) is fetched by TMA while
//    the current tile computes.
//  * Tiles t_first, t_first + t_step, ... of the row-major tile grid, so all
//    CTAs of a cooperative kernel share one GEMM.
#pragma once
#include "tma.cuh"

namespace vb {
namespace tma {

struct BigMaps {
  CUtensorMap a64;  // box: 16 doubles x 64 rows x 1
  CUtensorMap b8;   // box: 16 doubles x 8 rows x 1
};

template <int STAGES>
struct GemmBig {
  static constexpr int TM = 128, TN = 64, KC = 8;
  static constexpr unsigned A_BYTES = TM * KC * 16;  // 2 boxes of 64 rows x 8 complex
  static constexpr unsigned B_BYTES = KC * TN * 16;  // 8 boxes of 8 rows x 8 complex
  static constexpr unsigned C_BYTES = TM * TN * 16;  // 16 boxes of 64 rows x 8 complex
  static constexpr size_t SMEM = (size_t)STAGES * (A_BYTES + B_BYTES) + C_BYTES;

  struct Bars {
    uint64_t full[STAGES], empty[STAGES], cfull, cempty;
  };

  // Producer work split over PW warps (warp-collective issue; warp 0 arms the
  // barrier with the whole transfer, a complete-tx may precede it).
  static constexpr int PW = 4;
  __device__ static __forceinline__ void issue_chunk(int part, const BigMaps* mp, char* As, char* Bs,
                                                     uint64_t* bar, int ar0, int ac0, int br0, int bc0, int m0,
                                                     int n0, int k0) {
    if (part == 0) {
      mbar_expect_tx_w(bar, A_BYTES + B_BYTES);
      tma_load_3d_w(As, &mp->a64, 2 * (ac0 + k0), ar0 + m0, 0, bar);
      tma_load_3d_w(As + 8192, &mp->a64, 2 * (ac0 + k0), ar0 + m0 + 64, 0, bar);
    } else {
      // warps 1..3: B boxes part-1, part+2, ... (8 boxes of 8 rows x 8 complex)
      for (int b = part - 1; b < 8; b += PW - 1)
        tma_load_3d_w(Bs + b * 1024, &mp->b8, 2 * (bc0 + n0 + 8 * b), br0 + k0, 0, bar);
    }
  }
  __device__ static __forceinline__ void issue_c(int part, const BigMaps* mp, char* Cs, uint64_t* bar, int cr0,
                                                 int cc0, int m0, int n0) {
    if (part == 0) mbar_expect_tx_w(bar, C_BYTES);
    for (int q = part; q < 16; q += PW) {  // 16 boxes of 64 rows x 8 complex
      const int h = q >> 3, b = q & 7;
      tma_load_3d_w(Cs + q * 8192, &mp->a64, 2 * (cc0 + n0 + 8 * b), cr0 + m0 + 64 * h, 0, bar);
    }
  }

  // C origin (ar0, bc0); Cg row-major with leading dimension ldc.
  __device__ static void run(const BigMaps* mp, z_t* Cg, int64_t ldc, int ar0, int ac0, int br0, int bc0, int M,
                             int N, int K, char* smem, Bars* bars, int t_first, int t_step) {
    if (M <= 0 || N <= 0 || K <= 0) return;
    const int ntn = (N + TN - 1) / TN, ntm = (M + TM - 1) / TM, nk = (K + KC - 1) / KC;
    const int ntiles_all = ntm * ntn;
    if (t_first >= ntiles_all) return;
    const int ntiles = (ntiles_all - 1 - t_first) / t_step + 1;
    const int T = ntiles * nk;
    // tile coordinates walked incrementally (one division per tile at most)
    struct Cur {
      int m, n;
    };
    auto advance = [&](Cur c) {
      c.n += t_step;
      if (c.n >= ntn) {
        c.m += c.n / ntn;
        c.n %= ntn;
      }
      return c;
    };
    const Cur c0 = {t_first / ntn, t_first % ntn};
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = warp >> 1, wn = warp & 1;
    char* As = smem;
    char* Bs = smem + STAGES * A_BYTES;
    char* Cs = Bs + STAGES * B_BYTES;
    if (tid == 0) {
#pragma unroll
      for (int s = 0; s < STAGES; ++s) {
        mbar_init(&bars->full[s], 1);
        mbar_init(&bars->empty[s], NT / 32);
      }
      mbar_init(&bars->cfull, 1);
      mbar_init(&bars->cempty, NT / 32);
      mbar_fence_init();
    }
    __syncthreads();
    int pk = 0;  // producer cursor (warps 0..PW-1, warp-collective issue)
    Cur pc = c0;
    if (warp < PW) {
      fence_proxy_async_global();  // generic writes before this GEMM -> visible to TMA
      issue_c(warp, mp, Cs, &bars->cfull, ar0, bc0, pc.m * TM, pc.n * TN);
      for (int j = 0; j < STAGES - 1 && j < T; ++j) {
        issue_chunk(warp, mp, As + j * A_BYTES, Bs + j * B_BYTES, &bars->full[j], ar0, ac0, br0, bc0, pc.m * TM,
                    pc.n * TN, pk * KC);
        if (++pk == nk) { pk = 0; pc = advance(pc); }
      }
    }
    unsigned full_ph = 0, empty_ph = 0, c_ph = 0, cempty_ph = 0;
    double cr[4][4][2], ci[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) cr[i][j][0] = cr[i][j][1] = ci[i][j][0] = ci[i][j][1] = 0.0;
#if VB_GEMM_3M
    double c2[4][4][2];  // 3M: cr = sum ar br, c2 = sum ai bi, ci = sum (ar + ai)(br + bi)
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) c2[i][j][0] = c2[i][j][1] = 0.0;
#endif
    const int ak = lane & 3, prow = perm8(lane >> 2);
    int t = 0, kc = 0;
    Cur cc = c0;  // consumer's tile
    for (int it = 0; it < T; ++it) {
      const int st = it % STAGES;
      mbar_wait(&bars->full[st], (full_ph >> st) & 1);
      full_ph ^= 1u << st;
      const char* as = As + st * A_BYTES;
      const char* bs = Bs + st * B_BYTES;
      const int kvalid = min(KC, K - kc * KC);
      const bool full = kvalid == KC;  // full chunk: no masking
#pragma unroll
      for (int kk = 0; kk < 2; ++kk) {
        const int kcol = kk * 4 + ak;
        if (full || kk * 4 < kvalid) {
          const bool kin = full || kcol < kvalid;
          z_t a[4], b[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int row = wm * 32 + i * 8 + prow;  // 0..127
            a[i] = *(const z_t*)(as + (row >> 6) * 8192 + swz(row & 63, kcol));
            if (!kin) a[i] = zmake(0.0, 0.0);
          }
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            b[j] = *(const z_t*)(bs + (wn * 4 + j) * 1024 + swz(kcol, prow));
            if (!kin) b[j] = zmake(0.0, 0.0);
          }
#if VB_GEMM_3M
          double sa[4], sb[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) sa[i] = a[i].x + a[i].y;
#pragma unroll
          for (int j = 0; j < 4; ++j) sb[j] = b[j].x + b[j].y;
#pragma unroll
          for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              blk::dmma(cr[i][j][0], cr[i][j][1], a[i].x, b[j].x);
              blk::dmma(c2[i][j][0], c2[i][j][1], a[i].y, b[j].y);
              blk::dmma(ci[i][j][0], ci[i][j][1], sa[i], sb[j]);
            }
#else
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const double br = b[j].x, bi = b[j].y, nbi = -bi;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              blk::dmma(cr[i][j][0], cr[i][j][1], a[i].x, br);
              blk::dmma(cr[i][j][0], cr[i][j][1], a[i].y, nbi);
              blk::dmma(ci[i][j][0], ci[i][j][1], a[i].x, bi);
              blk::dmma(ci[i][j][0], ci[i][j][1], a[i].y, br);
            }
          }
#endif
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars->empty[st]);
      // refill the stage consumed in the previous iteration
      if (warp < PW && it + STAGES - 1 < T) {
        const int s2 = (it + STAGES - 1) % STAGES;
        if (it >= 1) {
          mbar_wait(&bars->empty[s2], (empty_ph >> s2) & 1);
          empty_ph ^= 1u << s2;
        }
        issue_chunk(warp, mp, As + s2 * A_BYTES, Bs + s2 * B_BYTES, &bars->full[s2], ar0, ac0, br0, bc0,
                    pc.m * TM, pc.n * TN, pk * KC);
        if (++pk == nk) { pk = 0; pc = advance(pc); }
      }
      if (kc == nk - 1) {
        const int m0 = cc.m * TM, n0 = cc.n * TN;
        mbar_wait(&bars->cfull, c_ph);
        c_ph ^= 1;
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int v = 0; v < 2; ++v) {
              const int row = wm * 32 + i * 8 + prow;
              const int col = wn * 32 + j * 8 + perm8(2 * ak + v);
              if (m0 + row < M && n0 + col < N) {
                const z_t c = *(const z_t*)(Cs + ((row >> 6) * 8 + (col >> 3)) * 8192 + swz(row & 63, col & 7));
#if VB_GEMM_3M
                const double pr = cr[i][j][v] - c2[i][j][v], pi = ci[i][j][v] - cr[i][j][v] - c2[i][j][v];
                Cg[(int64_t)(ar0 + m0 + row) * ldc + bc0 + n0 + col] = zmake(c.x - pr, c.y - pi);
#else
                Cg[(int64_t)(ar0 + m0 + row) * ldc + bc0 + n0 + col] = zmake(c.x - cr[i][j][v], c.y - ci[i][j][v]);
#endif
              }
              cr[i][j][v] = 0.0;
              ci[i][j][v] = 0.0;
#if VB_GEMM_3M
              c2[i][j][v] = 0.0;
#endif
            }
        __syncwarp();
        if (lane == 0) mbar_arrive(&bars->cempty);
        if (warp < PW && t + 1 < ntiles) {
          mbar_wait(&bars->cempty, cempty_ph);
          cempty_ph ^= 1;
          const Cur nx = advance(cc);
          issue_c(warp, mp, Cs, &bars->cfull, ar0, bc0, nx.m * TM, nx.n * TN);
        }
        kc = 0;
        ++t;
        cc = advance(cc);
      } else {
        ++kc;
      }
    }
    __syncthreads();
    if (tid == 0) {
#pragma unroll
      for (int s = 0; s < STAGES; ++s) {
        mbar_inval(&bars->full[s]);
        mbar_inval(&bars->empty[s]);
      }
      mbar_inval(&bars->cfull);
      mbar_inval(&bars->cempty);
    }
  }
};

}  // namespace tma
}  // namespace vb
