// Matrix-free apply of the assembled uniform-box hex27 primitives (SURVEY §8a
// A9 projection / A7 Krylov operator products, fast path for cfg1 and cfg3):
//   Kgrad = Kx (x) My (x) Mz + Mx (x) Ky (x) Mz + Mx (x) My (x) Kz,
//   Mnn   = Mx (x) My (x) Mz,
// the exact Kronecker form of the element sums on a uniform box (tensor-product
// bases, 3x3x3 Gauss; the same 1D band tables as vb_hex27_box_csr, so the CSR
// that kernel writes and this operator agree to rounding).  Y = alpha Op X +
// beta Y for a complex block X (n x k, row-major), node (x, y, z) at row
// (z npy + y) npx + x.
//
// Replaces the CSR SpMM for these primitives: a CSR SpMM gathers a k-wide X
// row per nonzero (nnz k 16 B through L1, ~62 per row) and re-reads the CSR; the
// Kronecker apply streams X and Y once (plus the x-y halo) and applies three
// 5-tap 1D operators per term.  2.5-D blocking: a CTA owns a 32 x 8 (x, y) tile
// and 2 complex columns and streams z; input planes (tile + 2-node halo) land
// by cp.async 3 planes ahead, each thread keeps its halo items' 5-plane z band
// in registers, and the y and x passes (two outputs per thread) run in shared
// memory.
#include "common.cuh"
#include "mma.cuh"
#include "sweep.cuh"

namespace vb {
namespace kron {

using blk::cp_async16;
using blk::cp_commit;
using blk::cp_wait;

#ifndef VB_KRON_TX
#define VB_KRON_TX 32
#endif
#ifndef VB_KRON_TY
#define VB_KRON_TY 8
#endif
#ifndef VB_KRON_KC
#define VB_KRON_KC 2
#endif
constexpr int TX = VB_KRON_TX, TY = VB_KRON_TY, HX = TX + 4, HY = TY + 4, KC = VB_KRON_KC;
constexpr int RING = 4, AHEAD = 3;   // cp.async landing slots: newest plane + AHEAD in flight
constexpr int NTH = 256;
constexpr int PLANE = HY * HX * KC;  // complex per halo plane
constexpr int ZIT = (PLANE + NTH - 1) / NTH;  // halo items per thread (z queue in registers)
constexpr size_t SMEM = (size_t)(RING * PLANE + 2 * PLANE + 2 * TY * HX * KC) * sizeof(z_t);

struct Args {
  int npx, npy, npz, maxnp, k;
  const double* K1;  // [3][maxnp][5]: x, y, z bands, entry o couples i and i + o - 2
  const double* M1;
  const z_t* X;
  int64_t ldx;
  z_t* Y;
  int64_t ldy;
  z_t alpha, beta;
};

template <bool STIFF>
__global__ void __launch_bounds__(NTH, 2) kron3_kernel(Args a) {
  extern __shared__ double2 ksm[];
  z_t* ring = ksm;                   // [RING][HY][HX][KC] landing slots
  z_t* Tm = ring + RING * PLANE;     // [HY][HX][KC]  Mz-reduced plane
  z_t* Tk = Tm + PLANE;              // [HY][HX][KC]  Kz-reduced plane
  z_t* U = Tk + PLANE;               // [TY][HX][KC]  My Tm
  z_t* S = U + TY * HX * KC;         // [TY][HX][KC]  Ky Tm + My Tk
  const int tid = threadIdx.x;
  const int ntx = (a.npx + TX - 1) / TX;
  const int bx = blockIdx.x % ntx, by = blockIdx.x / ntx;
  const int gx0 = bx * TX - 2, gy0 = by * TY - 2;  // halo origin
  const int c0 = blockIdx.y * KC;
  const size_t mp5 = (size_t)a.maxnp * 5;
  const double *Kx = a.K1, *Ky = a.K1 + mp5, *Kz = a.K1 + 2 * mp5;
  const double *Mx = a.M1, *My = a.M1 + mp5, *Mz = a.M1 + 2 * mp5;
  const int64_t plane_rows = (int64_t)a.npx * a.npy;
  // the tile's x and y band rows (kx, mx) / (ky, my), read per item from shared
  // memory instead of through L1 (they were the kernel's long-scoreboard stalls)
  __shared__ double2 sXb[TX][5], sYb[TY][5];
  for (int e = tid; e < TX * 5; e += NTH) {
    const int tx = e / 5, o = e - tx * 5, gx = min(bx * TX + tx, a.npx - 1);
    sXb[tx][o] = make_double2(STIFF ? __ldg(Kx + gx * 5 + o) : 0.0, __ldg(Mx + gx * 5 + o));
  }
  for (int e = tid; e < TY * 5; e += NTH) {
    const int ty = e / 5, o = e - ty * 5, gy = min(by * TY + ty, a.npy - 1);
    sYb[ty][o] = make_double2(STIFF ? __ldg(Ky + gy * 5 + o) : 0.0, __ldg(My + gy * 5 + o));
  }

  auto load_plane = [&](int zp) {
    z_t* dst = ring + (zp & (RING - 1)) * PLANE;
    for (int e = tid; e < PLANE; e += NTH) {
      const int c = e % KC, hx = (e / KC) % HX, hy = e / (KC * HX);
      const int gx = gx0 + hx, gy = gy0 + hy;
      const bool ok = zp < a.npz && gx >= 0 && gx < a.npx && gy >= 0 && gy < a.npy && c0 + c < a.k;
      const z_t* src = ok ? a.X + (zp * plane_rows + (int64_t)gy * a.npx + gx) * a.ldx + c0 + c : a.X;
      cp_async16(dst + e, src, ok);
    }
  };

  // Each thread keeps the last 5 planes of its halo items in registers (the z
  // band), so a plane is read from shared memory once.  Output plane z needs
  // input planes z-2 .. z+2; the queue q[.][4] is plane z+2 after the shift.
  z_t q[ZIT][5];
#pragma unroll
  for (int i = 0; i < ZIT; ++i)
#pragma unroll
    for (int o = 0; o < 5; ++o) q[i][o] = zmake(0.0, 0.0);
  for (int zp = 0; zp < AHEAD; ++zp) {  // planes 0 .. AHEAD-1 in flight
    load_plane(zp);
    cp_commit();
  }
  // prime: planes 0, 1 into q[.][3], q[.][4] (planes -2, -1 are zero)
  for (int zp = 0; zp < 2; ++zp) {
    load_plane(zp + AHEAD);
    cp_commit();
    cp_wait<AHEAD>();
    __syncthreads();
#pragma unroll
    for (int i = 0; i < ZIT; ++i) {
      const int e = tid + i * NTH;
#pragma unroll
      for (int o = 0; o < 4; ++o) q[i][o] = q[i][o + 1];
      q[i][4] = e < PLANE ? ring[(zp & (RING - 1)) * PLANE + e] : zmake(0.0, 0.0);
    }
    __syncthreads();
  }
  for (int z = 0; z < a.npz; ++z) {
    const int zn = z + 2;  // plane entering the queue
    load_plane(zn + AHEAD);
    cp_commit();
    cp_wait<AHEAD>();      // plane zn has landed
    __syncthreads();
    // z pass from the register queue
    double mz[5], kz[5];
#pragma unroll
    for (int o = 0; o < 5; ++o) {
      mz[o] = __ldg(Mz + z * 5 + o);
      kz[o] = STIFF ? __ldg(Kz + z * 5 + o) : 0.0;
    }
#pragma unroll
    for (int i = 0; i < ZIT; ++i) {
      const int e = tid + i * NTH;
#pragma unroll
      for (int o = 0; o < 4; ++o) q[i][o] = q[i][o + 1];
      q[i][4] = e < PLANE ? ring[(zn & (RING - 1)) * PLANE + e] : zmake(0.0, 0.0);
      if (e < PLANE) {
        z_t tm = zmake(0.0, 0.0), tk = zmake(0.0, 0.0);
#pragma unroll
        for (int o = 0; o < 5; ++o) {  // band entries outside [0, npz) are zero
          tm.x += mz[o] * q[i][o].x;
          tm.y += mz[o] * q[i][o].y;
          if (STIFF) {
            tk.x += kz[o] * q[i][o].x;
            tk.y += kz[o] * q[i][o].y;
          }
        }
        Tm[e] = tm;
        if (STIFF) Tk[e] = tk;
      }
    }
    __syncthreads();
    // y pass on the (TY x HX) strip, two output rows per thread
    for (int e = tid; e < (TY / 2) * HX * KC; e += NTH) {
      const int c = e % KC, hx = (e / KC) % HX, ty = 2 * (e / (KC * HX));
      z_t tm[6], tk[6];
#pragma unroll
      for (int j = 0; j < 6; ++j) {
        const int qi = ((ty + j) * HX + hx) * KC + c;
        tm[j] = Tm[qi];
        if (STIFF) tk[j] = Tk[qi];
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int gy = by * TY + ty + h;
        z_t u = zmake(0.0, 0.0), sv = zmake(0.0, 0.0);
        if (gy < a.npy) {
#pragma unroll
          for (int o = 0; o < 5; ++o) {
            const double2 yb = sYb[ty + h][o];
            const double m = yb.y;
            u.x += m * tm[h + o].x;
            u.y += m * tm[h + o].y;
            if (STIFF) {
              const double ky = yb.x;
              sv.x += ky * tm[h + o].x + m * tk[h + o].x;
              sv.y += ky * tm[h + o].y + m * tk[h + o].y;
            }
          }
        }
        const int qo = ((ty + h) * HX + hx) * KC + c;
        U[qo] = u;
        if (STIFF) S[qo] = sv;
      }
    }
    __syncthreads();
    // x pass + output, two output columns per thread
    for (int e = tid; e < TY * (TX / 2) * KC; e += NTH) {
      const int c = e % KC, tx = 2 * ((e / KC) % (TX / 2)), ty = e / (KC * (TX / 2));
      const int gy = by * TY + ty;
      if (gy >= a.npy || c0 + c >= a.k) continue;
      z_t u[6], sv[6];
#pragma unroll
      for (int j = 0; j < 6; ++j) {
        const int qi = (ty * HX + tx + j) * KC + c;
        u[j] = U[qi];
        if (STIFF) sv[j] = S[qi];
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int gx = bx * TX + tx + h;
        if (gx >= a.npx) continue;
        z_t out = zmake(0.0, 0.0);
#pragma unroll
        for (int o = 0; o < 5; ++o) {
          const double2 xb = sXb[tx + h][o];
          const double m = xb.y;
          if (STIFF) {
            const double kx = xb.x;
            out.x += kx * u[h + o].x + m * sv[h + o].x;
            out.y += kx * u[h + o].y + m * sv[h + o].y;
          } else {
            out.x += m * u[h + o].x;
            out.y += m * u[h + o].y;
          }
        }
        z_t* yp = a.Y + (z * plane_rows + (int64_t)gy * a.npx + gx) * a.ldy + c0 + c;
        z_t r = zmul(a.alpha, out);
        if (a.beta.x != 0.0 || a.beta.y != 0.0) r = zfma(r, a.beta, *yp);
        *yp = r;
      }
    }
    // Tm/Tk/U/S are rewritten only after the next plane's barriers; the landing
    // slot refilled next was consumed before this plane's first barrier
  }
  cp_wait<0>();
}

}  // namespace kron

int kron3_apply(int npx, int npy, int npz, const double* K1, const double* M1, int maxnp, int stiff, int k,
                z_t alpha, const z_t* X, int64_t ldx, z_t beta, z_t* Y, int64_t ldy, cudaStream_t st) {
  VB_CHECK_ARG(npx > 0 && npy > 0 && npz > 0 && k >= 0, "vb_kron3_apply: bad sizes");
  VB_CHECK_ARG(maxnp >= npx && maxnp >= npy && maxnp >= npz, "vb_kron3_apply: band table too small");
  VB_CHECK_ARG(ldx >= k && ldy >= k, "vb_kron3_apply: bad leading dimension");
  if (k == 0) return 0;
  kron::Args a{npx, npy, npz, maxnp, k, K1, M1, X, ldx, Y, ldy, alpha, beta};
  const dim3 grid((unsigned)(((npx + kron::TX - 1) / kron::TX) * ((npy + kron::TY - 1) / kron::TY)),
                  (unsigned)((k + kron::KC - 1) / kron::KC));
  if (stiff) {
    VB_CUDA(cudaFuncSetAttribute(kron::kron3_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)kron::SMEM));
    kron::kron3_kernel<true><<<grid, kron::NTH, kron::SMEM, st>>>(a);
  } else {
    VB_CUDA(cudaFuncSetAttribute(kron::kron3_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)kron::SMEM));
    kron::kron3_kernel<false><<<grid, kron::NTH, kron::SMEM, st>>>(a);
  }
  VB_LAUNCHED("kron3_kernel");
  return 0;
}

}  // namespace vb
