// Fused in-block Gram-Schmidt of the basis build: the
// column loop of _orthonormalise (vibrofem/mor.py:122-135: every column of a
// new block, after the block has been projected on V, is orthogonalised
// against the block's kept columns — twice — and kept iff
// ||w|| > ORTH_DROP_TOL * ||w_raw||) as ONE persistent cooperative kernel per
// block instead of ~8 launches and a host round trip per column.
//
// Rows are split into one contiguous range per CTA.  Every reduction (the
// nk projections Q^H w, ||w||^2) is a per-CTA partial -> grid barrier -> every
// CTA sums all partials in the same fixed order (deterministic, identical
// decisions on every CTA).  Partials are double-buffered across rounds.
//   pass: h = Q^H w ; w -= Q h          (two passes = CGS2)
//   keep: ref > 0 && ||w|| > tol*ref     (the reference drop rule)
//   DGKS: a kept column with ||w|| < reorth*ref gets a third pass
//   Q[:, nk] = w / ||w||
// no_drop = 1 is the re-orthonormalisation of already kept columns (pass 2 of
// the block CGS2, in place: Q == W).
#include <cooperative_groups.h>
#include <cstdlib>

#include "common.cuh"
#include "sweep.cuh"

namespace vb {
namespace bgs {

namespace cg = cooperative_groups;

constexpr int NT = 256;
constexpr int KMAX = 16;  // block width handled by the fused kernel
constexpr int L = 2 * KMAX;

struct Args {
  int n, kb;
  z_t* W;
  int64_t ldw;
  const double* refs;
  double tol, reorth;
  int no_drop;
  z_t* Q;
  int64_t ldq;
  int32_t* kept;
  int32_t* nk_out;
  double* part;  // [2][grid][L]
};

// Sum v[0..len) over the CTA (fixed order); result in out[0..len) (shared).
__device__ __forceinline__ void cta_reduce(double (&v)[L], int len, double (*red)[L], double* out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int l = 0; l < L; ++l) {
    if (l < len) {
      double s = v[l];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) red[warp][l] = s;
    }
  }
  __syncthreads();
  if (threadIdx.x < len) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < NT / 32; ++w) s += red[w][threadIdx.x];
    out[threadIdx.x] = s;
  }
  __syncthreads();
}

// Grid-wide sum of this CTA's partial v[0..len) into out[0..len) (shared).
__device__ void grid_reduce(cg::grid_group& grid, const Args& a, int& rnd, double (&v)[L], int len,
                            double (*red)[L], double* cta_sum, double* out) {
  cta_reduce(v, len, red, cta_sum);
  double* buf = a.part + (size_t)(rnd & 1) * gridDim.x * L;
  if (threadIdx.x < len) buf[(size_t)blockIdx.x * L + threadIdx.x] = cta_sum[threadIdx.x];
  ++rnd;
  grid.sync();
  double t[L];
#pragma unroll
  for (int l = 0; l < L; ++l) t[l] = 0.0;
  for (int c = threadIdx.x; c < (int)gridDim.x; c += NT) {
#pragma unroll
    for (int l = 0; l < L; ++l)
      if (l < len) t[l] += __ldcg(buf + (size_t)c * L + l);
  }
  cta_reduce(t, len, red, out);
}

__global__ void __launch_bounds__(NT) block_gs_kernel(Args a) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double red[NT / 32][L];
  __shared__ double cta_sum[L];
  __shared__ double h[L];
  const int chunk = (a.n + gridDim.x - 1) / gridDim.x;
  const int r0 = blockIdx.x * chunk, r1 = min(a.n, r0 + chunk);
  int nk = 0, rnd = 0;
  double v[L];

  // w -= Q[:, :nk] (Q[:, :nk]^H w) on this CTA's rows (after a grid reduction)
  auto project = [&](int j) {
#pragma unroll
    for (int l = 0; l < L; ++l) v[l] = 0.0;
    for (int i = r0 + threadIdx.x; i < r1; i += NT) {
      const z_t w = a.W[(int64_t)i * a.ldw + j];
      const z_t* q = a.Q + (int64_t)i * a.ldq;
#pragma unroll
      for (int c = 0; c < KMAX; ++c)
        if (c < nk) {
          const z_t qc = q[c];  // conj(q) w
          v[2 * c] += qc.x * w.x + qc.y * w.y;
          v[2 * c + 1] += qc.x * w.y - qc.y * w.x;
        }
    }
    grid_reduce(grid, a, rnd, v, 2 * nk, red, cta_sum, h);
    for (int i = r0 + threadIdx.x; i < r1; i += NT) {
      z_t* wp = a.W + (int64_t)i * a.ldw + j;
      z_t w = *wp;
      const z_t* q = a.Q + (int64_t)i * a.ldq;
#pragma unroll
      for (int c = 0; c < KMAX; ++c)
        if (c < nk) w = zfms(w, q[c], zmake(h[2 * c], h[2 * c + 1]));
      *wp = w;
    }
  };
  // Second CGS pass fused with the norm (one grid reduction instead of two):
  // h2 = Q^H w' and ||w'||^2 from the same partials, w'' = w' - Q h2 and
  // ||w''||^2 = ||w'||^2 - ||h2||^2.  After a first pass h2 is a rounding-level
  // correction (~eps ||w_raw||), so the subtraction loses nothing at the drop
  // threshold (||w''|| ~ 1e-10 ||w_raw||): (eps / 1e-10)^2 relative.
  auto project_norm = [&](int j) -> double {
#pragma unroll
    for (int l = 0; l < L; ++l) v[l] = 0.0;
    for (int i = r0 + threadIdx.x; i < r1; i += NT) {
      const z_t w = a.W[(int64_t)i * a.ldw + j];
      const z_t* q = a.Q + (int64_t)i * a.ldq;
#pragma unroll
      for (int c = 0; c < KMAX; ++c)
        if (c < nk) {
          const z_t qc = q[c];
          v[2 * c] += qc.x * w.x + qc.y * w.y;
          v[2 * c + 1] += qc.x * w.y - qc.y * w.x;
        }
#pragma unroll
      for (int l = 0; l < L; ++l)
        if (l == 2 * nk) v[l] += zabs2(w);
    }
    grid_reduce(grid, a, rnd, v, 2 * nk + 1, red, cta_sum, h);
    double hh = 0.0;
    for (int i = r0 + threadIdx.x; i < r1; i += NT) {
      z_t* wp = a.W + (int64_t)i * a.ldw + j;
      z_t w = *wp;
      const z_t* q = a.Q + (int64_t)i * a.ldq;
#pragma unroll
      for (int c = 0; c < KMAX; ++c)
        if (c < nk) w = zfms(w, q[c], zmake(h[2 * c], h[2 * c + 1]));
      *wp = w;
    }
    for (int c = 0; c < nk; ++c) hh += h[2 * c] * h[2 * c] + h[2 * c + 1] * h[2 * c + 1];
    return sqrt(fmax(h[2 * nk] - hh, 0.0));
  };
  auto norm = [&](int j) -> double {
#pragma unroll
    for (int l = 0; l < L; ++l) v[l] = 0.0;
    for (int i = r0 + threadIdx.x; i < r1; i += NT) v[0] += zabs2(a.W[(int64_t)i * a.ldw + j]);
    grid_reduce(grid, a, rnd, v, 1, red, cta_sum, h);
    return sqrt(h[0]);
  };

  for (int j = 0; j < a.kb; ++j) {
    double nw;
    if (nk) {
      project(j);            // CGS pass 1
      nw = project_norm(j);  // CGS pass 2 + ||w||, one reduction
    } else {
      nw = norm(j);
    }
    const double ref = a.no_drop ? 0.0 : a.refs[j];
    const bool keep = a.no_drop || (ref > 0.0 && nw > a.tol * ref);
    if (keep) {
      if (!a.no_drop && nk && nw < a.reorth * ref) {  // DGKS third pass (mor.py _polish)
        project(j);
        nw = norm(j);
      }
      const double inv = 1.0 / nw;
      for (int i = r0 + threadIdx.x; i < r1; i += NT) {
        const z_t w = a.W[(int64_t)i * a.ldw + j];
        a.Q[(int64_t)i * a.ldq + nk] = zmake(w.x * inv, w.y * inv);
      }
      // the next column's projections read Q[:, nk] on the same rows only
      __syncthreads();
      ++nk;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) a.kept[j] = keep ? 1 : 0;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *a.nk_out = nk;
}

static int grid_size() {
  static int g = 0;
  if (!g) {
    int dev = 0, sms = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, block_gs_kernel, NT, 0);
    int want = 2;  // CTAs per SM (VB_BGS_PER_SM: fewer CTAs = cheaper grid reductions, less row parallelism)
    if (const char* e = getenv("VB_BGS_PER_SM")) want = atoi(e) > 0 ? atoi(e) : want;
    g = sms * (per < want ? per : want);
  }
  return g;
}

}  // namespace bgs

size_t block_gs_workspace_bytes() {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return (size_t)2 * (2 * (size_t)sms) * bgs::L * sizeof(double);
}

int block_gs(int n, int kb, z_t* W, int64_t ldw, const double* refs, double tol, double reorth, int no_drop,
             z_t* Q, int64_t ldq, int32_t* kept, int32_t* nk, void* work, size_t wb, cudaStream_t st) {
  VB_CHECK_ARG(n > 0 && kb >= 0 && kb <= bgs::KMAX, "vb_block_gs: need n > 0 and 0 <= kb <= 16");
  VB_CHECK_ARG(ldq >= kb && ldw >= kb, "vb_block_gs: leading dimensions too small");
  if (kb == 0) return 0;
  const int g = bgs::grid_size();
  VB_CHECK_ARG(g > 0, "vb_block_gs: kernel does not fit on an SM");
  VB_CHECK_ARG(work && wb >= (size_t)2 * g * bgs::L * sizeof(double), "vb_block_gs: workspace too small");
  bgs::Args a{n, kb, W, ldw, refs, tol, reorth, no_drop, Q, ldq, kept, nk, (double*)work};
  void* args[] = {&a};
  VB_CUDA(cudaLaunchCooperativeKernel((const void*)bgs::block_gs_kernel, dim3(g), dim3(bgs::NT), args, 0, st));
  VB_LAUNCHED("block_gs_kernel");
  return 0;
}

}  // namespace vb
