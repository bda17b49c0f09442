// TMA (cp.async.bulk.tensor) + mbarrier staged complex GEMM for the blocked
// reduced-sweep kernel: C -= A * B where A, B and C are sub-blocks of the
// CTA's own workspace matrix [A_r | B] (one 3-D tensor map over all CTAs'
// workspaces: doubles x rows x CTA).
//
//  * One elected thread issues 128B-swizzled TMA boxes (8 complex x rows) into
//    a STAGES-deep shared-memory ring; completion is signalled through
//    full[] mbarriers (expect_tx), release through empty[] mbarriers (one
//    arrival per warp).  No block-wide barrier in the k-loop.
//  * The next C tile is fetched by TMA while the current tile computes.
//  * Fragment reads undo the swizzle; MMA rows/columns are permuted
//    (perm = 0,4,1,5,2,6,3,7) so that the 128-bit DMMA fragment loads of a
//    quarter-warp hit 8 distinct 16-byte bank groups.
#pragma once
#include <cuda.h>

#include "common.cuh"
#include "mma.cuh"

#ifndef VB_GEMM_3M
#define VB_GEMM_3M 1
#endif
#ifndef VB_SKINNY_3M
#define VB_SKINNY_3M 0
#endif
// GEMM epilogue variant (off by default): results written into the
// shared-memory C tile and stored by TMA (one bulk tensor store per 8-complex
// box) instead of scattered 16-byte global stores from every lane.  +2 % at
// r = 1024, but the later panel phases read the stored rows with ordinary
// (L1-cacheable) loads, and an async-proxy store does not update a line this
// SM may hold in L1; the generic stores keep L1 coherent by construction.
// With it on, sweep_blocked.cu reads its workspace from L2 (VB_WS_LD): then
// r = 1024 +0.6 %, r = 2048 -1.4 %, r = 256 -3.2 % — not worth it.
#ifndef VB_TMA_STORE_EPI
#define VB_TMA_STORE_EPI 0
#endif

namespace vb {
namespace tma {

// Profiling aid (-DVB_PHASE_TIMING): SM cycles of the general GEMM path split
// into wait-full / compute / release+produce / epilogue for warp 1 (a pure
// consumer) and thread 0 (consumer + producer); vb_debug_phase_cycles 16..23.
__device__ unsigned long long g_gemm_cycles[16];
#ifdef VB_PHASE_TIMING
#define GT_BEGIN long long _gt = clock64()
#define GT_MARK(k)                                                                  \
  do {                                                                              \
    if ((threadIdx.x & 31) == 0 && threadIdx.x < 64) {                              \
      const long long _n = clock64();                                               \
      atomicAdd(&g_gemm_cycles[(k) + (threadIdx.x ? 0 : 4)], (unsigned long long)(_n - _gt)); \
      _gt = _n;                                                                     \
    }                                                                               \
  } while (0)
#define GS_MARK(k)                                                                  \
  do {                                                                              \
    if (threadIdx.x == 32) {                                                        \
      const long long _n = clock64();                                               \
      atomicAdd(&g_gemm_cycles[8 + (k)], (unsigned long long)(_n - _gt));           \
      _gt = _n;                                                                     \
    }                                                                               \
  } while (0)
#else
#define GT_BEGIN
#define GT_MARK(k) \
  do {             \
  } while (0)
#define GS_MARK(k) \
  do {             \
  } while (0)
#endif

using blk::NT;

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_inval(uint64_t* b) {
  asm volatile("mbarrier.inval.shared::cta.b64 [%0];\n" ::"r"(smem_u32(b)));
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, unsigned bytes) {
  asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n}\n" ::"r"(smem_u32(b)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;\n" ::: "memory");
}
// 3-D tiled TMA load: coords (x = double index, y = row, z = CTA)
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int x, int y, int z,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
      : "memory");
}

// Warp-collective forms: called by ALL lanes of one warp with identical
// operands; one elected lane performs the operation.  Keeping the producer in
// warp-uniform control flow lets ptxas hold the coordinates in uniform
// registers (a single-thread `if (tid == 0)` producer compiles every UTMALDG
// into an R2UR waterfall loop, ~140 cycles per box).
__device__ __forceinline__ void mbar_expect_tx_w(uint64_t* b, unsigned bytes) {
  asm volatile(
      "{\n .reg .pred p;\n .reg .b64 st;\n elect.sync _|p, 0xffffffff;\n"
      " @p mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n}\n" ::"r"(smem_u32(b)),
      "r"(bytes)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d_w(void* dst, const CUtensorMap* map, int x, int y, int z,
                                              uint64_t* bar) {
  asm volatile(
      "{\n .reg .pred p;\n elect.sync _|p, 0xffffffff;\n"
      " @p cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n}\n" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
      : "memory");
}

// Warp-collective TMA tensor store (shared -> global) + commit of its bulk
// group; the elected lane owns the group, so completion waits are executed by
// all lanes (lanes without outstanding groups return at once).
__device__ __forceinline__ void tma_store_3d_w(const void* src, const CUtensorMap* map, int x, int y, int z) {
  asm volatile(
      "{\n .reg .pred p;\n elect.sync _|p, 0xffffffff;\n"
      " @p cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];\n"
      " @p cp.async.bulk.commit_group;\n}\n" ::"l"(map),
      "r"(x), "r"(y), "r"(z), "r"(smem_u32(src))
      : "memory");
}
__device__ __forceinline__ void bulk_wait_read_all() {
  asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_shared() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}

__device__ __forceinline__ int perm8(int x) { return (x >> 1) | ((x & 1) << 2); }

// byte offset of complex element (row, chunk) inside a 128B-swizzled box
__device__ __forceinline__ unsigned swz(int row, int chunk) {
  return (unsigned)(row * 128 + ((chunk ^ (row & 7)) << 4));
}

struct Maps {
  CUtensorMap a64;  // box: 16 doubles x 64 rows x 1 CTA
  CUtensorMap b16;  // box: 16 doubles x 16 rows x 1 CTA
  CUtensorMap b8;   // box: 16 doubles x 8 rows x 1 CTA
};

// C[M x N] -= A[M x K] B[K x N]; operand origins are (row, col) coordinates in
// the CTA's workspace matrix.  TM = 64, TN = 32, k chunks of KC_ (16 or 8)
// complex, 8 warps as 4 x 2.
template <int STAGES, int KC_ = 16>
struct GemmTma {
  static constexpr int TM = 64, TN = 32, KC = KC_;
  static_assert(KC == 16 || KC == 8, "k chunk of 8 or 16 complex");
  static constexpr unsigned A_BYTES = TM * KC * 16;   // KC/8 boxes of 64 rows x 8 complex
  static constexpr unsigned BBOX = KC * 128;          // B box: KC rows x 8 complex
  static constexpr unsigned B_BYTES = KC * TN * 16;   // 4 boxes
  static constexpr unsigned C_BYTES = TM * TN * 16;   // 4 boxes of 64 rows x 8 complex
  static constexpr size_t SMEM = (size_t)STAGES * (A_BYTES + B_BYTES) + C_BYTES;

  struct Bars {
    uint64_t full[STAGES], empty[STAGES], cfull, cempty;
    uint64_t sfull[8], sempty[8];  // skinny ring (up to 8 stages)
  };

  // issue the A and B boxes of chunk (m0, n0, k0) into stage st.  Split over
  // two producer warps: warp 0 arms the barrier with the whole stage's bytes and
  // loads A, warp 1 loads B (a complete-tx may precede the expect-tx: the phase
  // cannot complete before warp 0's arrival).
  // PW producer warps share the KC/8 + 4 boxes of a chunk (box q by warp q % PW).
  static constexpr int PW = KC / 8 + 4;
  __device__ static __forceinline__ void issue_chunk_part(int part, const Maps* mp, char* As, char* Bs,
                                                          uint64_t* bar, int cta, int ar0, int ac0, int br0, int bc0,
                                                          int m0, int n0, int k0) {
    if (part == 0) mbar_expect_tx_w(bar, A_BYTES + B_BYTES);
    if (part < KC / 8) {
      tma_load_3d_w(As + part * 8192, &mp->a64, 2 * (ac0 + k0 + 8 * part), ar0 + m0, cta, bar);
    } else {
      const int b = part - KC / 8;
      tma_load_3d_w(Bs + b * BBOX, KC == 16 ? &mp->b16 : &mp->b8, 2 * (bc0 + n0 + 8 * b), br0 + k0, cta, bar);
    }
  }
  // C tile: 4 boxes, box b by warp b (warp 0 arms the barrier)
  __device__ static __forceinline__ void issue_c(int part, const Maps* mp, char* Cs, uint64_t* bar, int cta,
                                                 int cr0, int cc0, int m0, int n0) {
    if (part == 0) mbar_expect_tx_w(bar, C_BYTES);
    if (part < 4)
      tma_load_3d_w(Cs + part * 8192, &mp->a64, 2 * (cc0 + n0 + 8 * part), cr0 + m0, cta, bar);
  }

  // Skinny in-panel updates of the recursive panel, fused with their TRSM:
  //   U = L^-1 X   (L = unit lower n1 x n1 block, X = the n1 x N block above C),
  //   C -= A U     (A: M x n1, C: M x N, n1, N <= NW = 8 or 16).
  // They are latency-bound on the C tile, so each ring stage carries a whole
  // tile — A (64 x NW) and C (64 x NW) — and all but one stage are in flight
  // while one computes (3 x 32 KB for NW = 16, 6 x 16 KB for NW = 8).  U is
  // solved in shared memory (one thread per column) while the first tiles load
  // and written back once; the tiles read it from shared memory.  8 warps x
  // (8 rows x NW columns).
  static constexpr unsigned SK_BUDGET = 3 * (2 * 8192 + 2 * 2048 + 2 * 8192);
  static constexpr int SK_LD = 17;                                  // odd stride
  static constexpr unsigned SK_TRI = 2 * 16 * SK_LD * 16;           // L and U blocks
  template <int NW>
  struct Sk {
    static constexpr int NBX = NW / 8;
    static constexpr unsigned A = NBX * 8192, C = NBX * 8192;
    static constexpr unsigned STAGE = A + C;
    static constexpr int NSTG = (int)((SK_BUDGET - SK_TRI) / STAGE) < 8 ? (int)((SK_BUDGET - SK_TRI) / STAGE) : 8;
  };
  static constexpr size_t SMEM_SKINNY = SK_BUDGET;

  template <int NW>
  __device__ static __forceinline__ void issue_tile(const Maps* mp, char* st, uint64_t* bar, int cta, int ar0,
                                                    int ac0, int bc0, int cr0, int m0) {
    using S = Sk<NW>;
    mbar_expect_tx_w(bar, S::STAGE);
#pragma unroll
    for (int h = 0; h < S::NBX; ++h) {
      tma_load_3d_w(st + h * 8192, &mp->a64, 2 * (ac0 + 8 * h), ar0 + m0, cta, bar);
      tma_load_3d_w(st + S::A + h * 8192, &mp->a64, 2 * (bc0 + 8 * h), cr0 + m0, cta, bar);
    }
  }

  // In-panel update with its TRSM: L = Ag[br0.., ac0..] (n1 x n1 unit lower),
  // X = Ag[br0.., bc0..] (n1 x N) is replaced by U = L^-1 X, then
  // C = Ag[cr0.., bc0..] -= Ag[ar0.., ac0..] U for M rows.
  template <int NW>
  __device__ static void run_skinny_trsm(const Maps* mp, z_t* Ag, int ldw, int ar0, int ac0, int br0, int bc0,
                                         int cr0, int M, int N, int K, char* smem, Bars* bars, int cta) {
    using S = Sk<NW>;
    constexpr int NST = S::NSTG;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int ntiles = (M + TM - 1) / TM;
    z_t* Ls = (z_t*)(smem + NST * S::STAGE);
    z_t* Us = Ls + 16 * SK_LD;
    GT_BEGIN;
    if (tid == 0) {
#pragma unroll
      for (int s = 0; s < NST; ++s) {
        mbar_init(&bars->sfull[s], 1);
        mbar_init(&bars->sempty[s], NT / 32);
      }
      mbar_fence_init();
    }
    __syncthreads();
    if (warp == 0) {  // warp-collective producer (see tma_load_3d_w)
      fence_proxy_async_global();
      for (int j = 0; j < NST - 1 && j < ntiles; ++j)
        issue_tile<NW>(mp, smem + j * S::STAGE, &bars->sfull[j], cta, ar0, ac0, bc0, cr0, j * TM);
    }
    // TRSM while the first tiles land: U = L^-1 X (zero-padded to NW x NW)
    for (int e = tid; e < NW * NW; e += NT) {
      const int i = e / NW, c = e % NW;
      Ls[i * SK_LD + c] = (i < K && c < i) ? Ag[(size_t)(br0 + i) * ldw + ac0 + c] : zmake(0.0, 0.0);
      Us[i * SK_LD + c] = (i < K && c < N) ? Ag[(size_t)(br0 + i) * ldw + bc0 + c] : zmake(0.0, 0.0);
    }
    __syncthreads();
    if (tid < N) {
      const int c = tid;
      for (int i = 1; i < K; ++i) {
        z_t x = Us[i * SK_LD + c];
        for (int k = 0; k < i; ++k) x = zfms(x, Ls[i * SK_LD + k], Us[k * SK_LD + c]);
        Us[i * SK_LD + c] = x;
        Ag[(size_t)(br0 + i) * ldw + bc0 + c] = x;
      }
    }
    __syncthreads();
    unsigned full_ph = 0, empty_ph = 0;
    const int ak = lane & 3, prow = perm8(lane >> 2);
    const int row = warp * 8 + prow;
    const int k4n = (K + 3) >> 2;
    GS_MARK(0);
    for (int t = 0; t < ntiles; ++t) {
      const int st = t % NST;
      mbar_wait(&bars->sfull[st], (full_ph >> st) & 1);
      full_ph ^= 1u << st;
      if (t == 0) GS_MARK(1); else GS_MARK(2);
      const char* as = smem + st * S::STAGE;
      const char* cs = as + S::A;
      double cr[S::NBX][2], ci[S::NBX][2];
#pragma unroll
      for (int j = 0; j < S::NBX; ++j) cr[j][0] = cr[j][1] = ci[j][0] = ci[j][1] = 0.0;
#if VB_SKINNY_3M
      double c2[S::NBX][2];
#pragma unroll
      for (int j = 0; j < S::NBX; ++j) c2[j][0] = c2[j][1] = 0.0;
#endif
      for (int kk = 0; kk < k4n; ++kk) {
        const int kcol = kk * 4 + ak;
        z_t a = *(const z_t*)(as + (kcol >> 3) * 8192 + swz(row, kcol & 7));
        if (kcol >= K) a = zmake(0.0, 0.0);
#if VB_SKINNY_3M
        const double sa = a.x + a.y;
#endif
#pragma unroll
        for (int j = 0; j < S::NBX; ++j) {
          const z_t b = Us[kcol * SK_LD + j * 8 + prow];  // zero rows/cols beyond K, N
#if VB_SKINNY_3M
          blk::dmma(cr[j][0], cr[j][1], a.x, b.x);
          blk::dmma(c2[j][0], c2[j][1], a.y, b.y);
          blk::dmma(ci[j][0], ci[j][1], sa, b.x + b.y);
#else
          blk::dmma(cr[j][0], cr[j][1], a.x, b.x);
          blk::dmma(cr[j][0], cr[j][1], a.y, -b.y);
          blk::dmma(ci[j][0], ci[j][1], a.x, b.y);
          blk::dmma(ci[j][0], ci[j][1], a.y, b.x);
#endif
        }
      }
#if VB_SKINNY_3M
#pragma unroll
      for (int j = 0; j < S::NBX; ++j)
#pragma unroll
        for (int v = 0; v < 2; ++v) {
          const double t1 = cr[j][v], t2 = c2[j][v];
          cr[j][v] = t1 - t2;
          ci[j][v] = ci[j][v] - t1 - t2;
        }
#endif
      const int m0 = t * TM;
#pragma unroll
      for (int j = 0; j < S::NBX; ++j)
#pragma unroll
        for (int v = 0; v < 2; ++v) {
          const int col = j * 8 + perm8(2 * ak + v);
          if (m0 + row < M && col < N) {
            const z_t c = *(const z_t*)(cs + j * 8192 + swz(row, col & 7));
            Ag[(size_t)(cr0 + m0 + row) * ldw + bc0 + col] = zmake(c.x - cr[j][v], c.y - ci[j][v]);
          }
        }
      __syncwarp();
      GS_MARK(3);
      if (lane == 0) mbar_arrive(&bars->sempty[st]);
      if (warp == 0 && t + NST - 1 < ntiles) {
        const int s2 = (t + NST - 1) % NST;
        if (t >= 1) {
          mbar_wait(&bars->sempty[s2], (empty_ph >> s2) & 1);
          empty_ph ^= 1u << s2;
        }
        issue_tile<NW>(mp, smem + s2 * S::STAGE, &bars->sfull[s2], cta, ar0, ac0, bc0, cr0, (t + NST - 1) * TM);
      }
      GS_MARK(4);
    }
    __syncthreads();
    GS_MARK(5);
    if (tid == 0) {
#pragma unroll
      for (int s = 0; s < NST; ++s) {
        mbar_inval(&bars->sfull[s]);
        mbar_inval(&bars->sempty[s]);
      }
    }
  }

  // ar0/ac0: A origin; br0/bc0: B origin; C origin (cr0, bc0) with cr0 = ar0
  // unless given; ldw for the generic-store epilogue.  smem must be 1024-byte
  // aligned.
  // t_first / t_step: this CTA computes tiles t_first, t_first + t_step, ...
  // of the row-major tile grid (several CTAs sharing one GEMM).  a_lower: A is
  // strictly lower triangular and M <= TM (the U12 product): zero k chunks are
  // skipped per warp.
  __device__ static void run(const Maps* mp, z_t* Cg, int ldw, int ar0, int ac0, int br0, int bc0, int M, int N,
                             int K, char* smem, Bars* bars, int cta, int cr0_ = -1, int t_first = 0,
                             int t_step = 1, bool a_lower = false) {
    if (M <= 0 || N <= 0 || K <= 0) return;
    const int cr0 = cr0_ < 0 ? ar0 : cr0_;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = warp >> 1, wn = warp & 1;
    const int ntn = (N + TN - 1) / TN, nk = (K + KC - 1) / KC;
    const int ntm = (M + TM - 1) / TM;
    const int ntiles_all = ntm * ntn;
    if (t_first >= ntiles_all) return;
    const int ntiles = (ntiles_all - 1 - t_first) / t_step + 1;  // this CTA's tiles
    const int T = ntiles * nk;
    // local tile l -> (m0, n0)
    // tile coordinates walked incrementally (no integer division per chunk):
    // a cursor (row tile, col tile) advanced by t_step tiles at a time
    struct Cur {
      int m, n;
    };
    auto start = [&]() { return Cur{t_first / ntn, t_first % ntn}; };
    auto advance = [&](Cur c) {
      c.n += t_step;
      if (c.n >= ntn) {
        c.m += c.n / ntn;
        c.n %= ntn;
      }
      return c;
    };
    char* As = smem;
    char* Bs = smem + STAGES * A_BYTES;
    char* Cs = Bs + STAGES * B_BYTES;
    const int cc0 = bc0;
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
    // producer cursor (warps 0..PW-1, warp-collective issue)
    int pk = 0;
    Cur pc = start();  // producer's tile
    if (warp < PW) {
      fence_proxy_async_global();  // generic writes before this GEMM -> visible to TMA
      if (warp < 4) issue_c(warp, mp, Cs, &bars->cfull, cta, cr0, cc0, pc.m * TM, pc.n * TN);
      for (int j = 0; j < STAGES - 1 && j < T; ++j) {
        issue_chunk_part(warp, mp, As + j * A_BYTES, Bs + j * B_BYTES, &bars->full[j], cta, ar0, ac0, br0, bc0,
                         pc.m * TM, pc.n * TN, pk * KC);
        if (++pk == nk) { pk = 0; pc = advance(pc); }
      }
    }
    unsigned full_ph = 0, empty_ph = 0, c_ph = 0, cempty_ph = 0;
    double cr[2][2][2], ci[2][2][2];
#if VB_GEMM_3M
    double c2[2][2][2];  // 3M: cr = sum ar br, c2 = sum ai bi, ci = sum (ar + ai)(br + bi)
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j) c2[i][j][0] = c2[i][j][1] = 0.0;
#endif
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j) cr[i][j][0] = cr[i][j][1] = ci[i][j][0] = ci[i][j][1] = 0.0;
    const int ar = lane >> 2, ak = lane & 3;
    const int prow = perm8(ar);
    int t = 0, kc = 0;
    Cur cc = start();  // consumer's tile
    GT_BEGIN;
    for (int it = 0; it < T; ++it) {
      const int st = it % STAGES;
      mbar_wait(&bars->full[st], (full_ph >> st) & 1);
      full_ph ^= 1u << st;
      GT_MARK(0);
      const char* as = As + st * A_BYTES;
      const char* bs = Bs + st * B_BYTES;
      const int kvalid = min(KC, K - kc * KC);
      // a_lower: A strictly lower triangular within a single 64-row tile, so
      // k chunk kc only reaches this warp's rows [16 wm, 16 wm + 16) if kc <= wm
      const bool skip = a_lower && kc * KC >= 16 * (wm + 1);
      // one k step of 4: fragment loads (masked past kvalid when MASK) + 16 DMMAs
      auto kstep = [&](int kk, bool mask) {
        const int kcol = kk * 4 + ak;
        const bool kin = !mask || kcol < kvalid;
        z_t a[2], b[2];
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int row = wm * 16 + i * 8 + prow;
          a[i] = *(const z_t*)(as + (kcol >> 3) * 8192 + swz(row, kcol & 7));
          if (!kin) a[i] = zmake(0.0, 0.0);
        }
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          b[j] = *(const z_t*)(bs + (wn * 2 + j) * BBOX + swz(kcol, prow));
          if (!kin) b[j] = zmake(0.0, 0.0);
        }
#if VB_GEMM_3M
        // Gauss / 3M complex product: 3 real DMMAs per fragment pair instead
        // of 4 (the operand sums cost 4 DADDs per k step, the recombination
        // is in the epilogue)
        double sa[2], sb[2];
#pragma unroll
        for (int i = 0; i < 2; ++i) sa[i] = a[i].x + a[i].y;
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
#else
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const double br = b[j].x, bi = b[j].y, nbi = -bi;
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            blk::dmma(cr[i][j][0], cr[i][j][1], a[i].x, br);
            blk::dmma(cr[i][j][0], cr[i][j][1], a[i].y, nbi);
            blk::dmma(ci[i][j][0], ci[i][j][1], a[i].x, bi);
            blk::dmma(ci[i][j][0], ci[i][j][1], a[i].y, br);
          }
        }
#endif
      };
      if (!skip) {
        if (kvalid == KC) {  // full chunk: unmasked, fully unrolled
#pragma unroll
          for (int kk = 0; kk < KC / 4; ++kk) kstep(kk, false);
        } else {
          const int k4n = (kvalid + 3) >> 2;
          for (int kk = 0; kk < k4n; ++kk) kstep(kk, true);
        }
      }
      __syncwarp();
      GT_MARK(1);
      if (lane == 0) mbar_arrive(&bars->empty[st]);
      // refill the stage consumed in the previous iteration
      if (warp < PW && it + STAGES - 1 < T) {
        const int s2 = (it + STAGES - 1) % STAGES;
        if (it >= 1) {
          mbar_wait(&bars->empty[s2], (empty_ph >> s2) & 1);
          empty_ph ^= 1u << s2;
        }
        issue_chunk_part(warp, mp, As + s2 * A_BYTES, Bs + s2 * B_BYTES, &bars->full[s2], cta, ar0, ac0, br0, bc0,
                         pc.m * TM, pc.n * TN, pk * KC);
        if (++pk == nk) { pk = 0; pc = advance(pc); }
      }
      GT_MARK(2);
      if (kc == nk - 1) {
        const int m0 = cc.m * TM, n0 = cc.n * TN;
        mbar_wait(&bars->cfull, c_ph);
        c_ph ^= 1;
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
          for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int v = 0; v < 2; ++v) {
              const int row = wm * 16 + i * 8 + prow;
              const int cfrag = 2 * ak + v;  // fragment column 0..7
              const int col = wn * 16 + j * 8 + perm8(cfrag);
              if (m0 + row < M && n0 + col < N) {
                z_t* cp = (z_t*)(Cs + (col >> 3) * 8192 + swz(row, col & 7));
                const z_t c = *cp;
#if VB_GEMM_3M
                const double pr = cr[i][j][v] - c2[i][j][v], pi = ci[i][j][v] - cr[i][j][v] - c2[i][j][v];
                const z_t o = zmake(c.x - pr, c.y - pi);
#else
                const z_t o = zmake(c.x - cr[i][j][v], c.y - ci[i][j][v]);
#endif
#if VB_TMA_STORE_EPI
                *cp = o;  // out-of-range elements keep their loaded value: the box store rewrites them unchanged
#else
                Cg[(size_t)(cr0 + m0 + row) * ldw + cc0 + n0 + col] = o;
#endif
              }
              cr[i][j][v] = 0.0;
              ci[i][j][v] = 0.0;
#if VB_GEMM_3M
              c2[i][j][v] = 0.0;
#endif
            }
#if VB_TMA_STORE_EPI
        fence_proxy_async_shared();  // this lane's results -> visible to the TMA store
#endif
        __syncwarp();
        if (lane == 0) mbar_arrive(&bars->cempty);
#if VB_TMA_STORE_EPI
        if (warp < 4) {  // box `warp` of the finished tile back to global, then the next tile's C
          mbar_wait(&bars->cempty, cempty_ph);
          cempty_ph ^= 1;
          tma_store_3d_w(Cs + warp * 8192, &mp->a64, 2 * (cc0 + n0 + 8 * warp), cr0 + m0, cta);
          if (t + 1 < ntiles) {
            bulk_wait_read_all();  // the box has left shared memory
            fence_proxy_async_global();
            const Cur nx = advance(cc);
            issue_c(warp, mp, Cs, &bars->cfull, cta, cr0, cc0, nx.m * TM, nx.n * TN);
          }
        }
#else
        if (warp < 4 && t + 1 < ntiles) {
          mbar_wait(&bars->cempty, cempty_ph);
          cempty_ph ^= 1;
          fence_proxy_async_global();
          const Cur nx = advance(cc);
          issue_c(warp, mp, Cs, &bars->cfull, cta, cr0, cc0, nx.m * TM, nx.n * TN);
        }
#endif
        GT_MARK(3);
        kc = 0;
        ++t;
        cc = advance(cc);
      } else {
        ++kc;
      }
    }
#if VB_TMA_STORE_EPI
    if (warp < 4) {  // the last tile's stores complete before anyone reads the result
      bulk_wait_all();
      fence_proxy_async_global();
    }
#endif
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
