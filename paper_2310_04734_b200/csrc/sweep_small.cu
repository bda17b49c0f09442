// Reduced frequency sweep, shared-memory-resident path (r*(r+s) complex128 fits
// one CTA's shared memory, i.e. r <~ 100).  Replaces, per frequency f:
//   mor.py:73-90   A_r(f) = sum_k alpha_k(f) P_k  (affine form of V^H A(f) V)
//   mor.py:94      numpy.linalg.solve = LAPACK zgesv (partial pivoting, izamax)
//   mor.py:96-102  y = (c_out V) x_r
//   solvers.py:334-338 mean_spl over the output rows, per RHS column
//
// One CTA owns one frequency at a time (grid-stride over F).  The augmented
// matrix [A | B] lives in shared memory; the elimination applies L^-1 P to B
// as it goes, so only the back substitution remains.  Pivot search is a warp
// argmax with LAPACK izamax semantics (max |Re|+|Im|, lowest row on ties).
#include "common.cuh"

namespace vb {

template <int NT>
__global__ void __launch_bounds__(NT) rom_sweep_small_kernel(
    int r, int nprim, int s, int n_out, int64_t F, const z_t* __restrict__ prims,
    const z_t* __restrict__ alpha, const z_t* __restrict__ b, int64_t b_stride_f,
    const z_t* __restrict__ c_r, z_t* __restrict__ y, double* __restrict__ spl,
    z_t* __restrict__ x, int* __restrict__ info) {
  extern __shared__ double2 smem[];
  const int ld = r + s;
  z_t* As = smem;                       // r x ld
  z_t* lvec = As + (size_t)r * ld;      // r
  z_t* alph = lvec + r;                 // nprim
  double* p2 = (double*)(alph + nprim); // n_out * s  (|y|^2 scratch)
  __shared__ int s_piv;
  __shared__ int s_info;
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int64_t rr = (int64_t)r * r;

  for (int64_t f = blockIdx.x; f < F; f += gridDim.x) {
    if (tid < nprim) alph[tid] = alpha[f * nprim + tid];
    if (tid == 0) s_info = 0;
    __syncthreads();
    // ---- form A_r(f) = sum_k alpha_k P_k and load B ----
    for (int idx = tid; idx < r * r; idx += NT) {
      z_t acc = zmake(0.0, 0.0);
      for (int k = 0; k < nprim; ++k) acc = zfma(acc, alph[k], __ldg(prims + k * rr + idx));
      int i = idx / r, j = idx - i * r;
      As[i * ld + j] = acc;
    }
    const z_t* bf = b + f * b_stride_f;
    for (int idx = tid; idx < r * s; idx += NT) {
      int i = idx / s, c = idx - i * s;
      As[i * ld + r + c] = __ldg(bf + idx);
    }
    __syncthreads();

    // ---- right-looking LU with partial pivoting on [A | B] ----
    for (int k = 0; k < r; ++k) {
      if (warp == 0) {
        double v = -1.0;
        int pi = 0x7fffffff;
        for (int i = k + lane; i < r; i += 32) {
          double a = zabs1(As[i * ld + k]);
          if (a > v) { v = a; pi = i; }
        }
        warp_argmax(v, pi);
        if (lane == 0) {
          if (!(v > 0.0)) {  // zero (or NaN) pivot column: LAPACK sets info and skips
            if (s_info == 0) s_info = k + 1;
            s_piv = -1;
          } else {
            s_piv = pi;
          }
        }
      }
      __syncthreads();
      const int p = s_piv;
      if (p < 0) {  // uniform across the block; the barrier keeps warp 0 from
        __syncthreads();  // publishing step k+1's pivot before every warp read p
        continue;
      }
      VB_DCHECK(p >= k && p < r);
      const z_t pv = As[p * ld + k];
      const z_t pinv = zrecip(pv);
      // phase A: multipliers (read column k through the swap) and swap cols > k
      for (int i = k + 1 + tid; i < r; i += NT) {
        int src = (i == p) ? k : i;
        lvec[i] = zmul(As[src * ld + k], pinv);
      }
      if (p != k) {
        for (int j = k + 1 + tid; j < ld; j += NT) {
          z_t t = As[k * ld + j];
          As[k * ld + j] = As[p * ld + j];
          As[p * ld + j] = t;
        }
      }
      __syncthreads();
      // phase B: rank-1 update of the trailing block (incl. the RHS columns)
      if (tid == 0) As[k * ld + k] = pv;
      const int m = r - k - 1, n = ld - k - 1;
      for (int idx = tid; idx < m * n; idx += NT) {
        int ii = idx / n;
        int i = k + 1 + ii, j = k + 1 + (idx - ii * n);
        As[i * ld + j] = zfms(As[i * ld + j], lvec[i], As[k * ld + j]);
      }
      __syncthreads();
    }

    // ---- back substitution U X = Y (Y in columns r..r+s-1) ----
    if (tid < s) {
      int k = r - 1;
      As[k * ld + r + tid] = zmul(As[k * ld + r + tid], zrecip(As[k * ld + k]));
    }
    __syncthreads();
    for (int k = r - 1; k > 0; --k) {
      for (int idx = tid; idx < k * s; idx += NT) {
        int i = idx / s, c = idx - i * s;
        z_t v = zfms(As[i * ld + r + c], As[i * ld + k], As[k * ld + r + c]);
        if (i == k - 1) v = zmul(v, zrecip(As[i * ld + i]));
        As[i * ld + r + c] = v;
      }
      __syncthreads();
    }

    // ---- outputs ----
    if (x) {
      z_t* xf = x + f * (int64_t)r * s;
      for (int idx = tid; idx < r * s; idx += NT) {
        int i = idx / s, c = idx - i * s;
        xf[idx] = As[i * ld + r + c];
      }
    }
    if (n_out > 0 && (y || spl)) {
      for (int idx = tid; idx < n_out * s; idx += NT) {
        int o = idx / s, c = idx - o * s;
        const z_t* cr = c_r + (int64_t)o * r;
        z_t acc = zmake(0.0, 0.0);
        for (int i = 0; i < r; ++i) acc = zfma(acc, __ldg(cr + i), As[i * ld + r + c]);
        if (y) y[(f * n_out + o) * s + c] = acc;
        p2[idx] = zabs2(acc);
      }
      __syncthreads();
      if (spl) {
        // warp w reduces RHS columns w, w+nwarps, ... in a fixed order (deterministic)
        for (int c = warp; c < s; c += NT / 32) {
          double acc = 0.0;
          for (int o = lane; o < n_out; o += 32) acc += p2[o * s + c];
          acc = warp_sum(acc);
          if (lane == 0) {
            double prms = sqrt(acc / n_out / 2.0);
            spl[f * s + c] = 20.0 * log10(fmax(prms, 1e-300) / 20e-6);
          }
        }
      }
    }
    if (tid == 0 && info) info[f] = s_info;
    __syncthreads();
  }
}

size_t sweep_small_smem_bytes(int r, int nprim, int s, int n_out) {
  return sizeof(z_t) * ((size_t)r * (r + s) + r + nprim) + sizeof(double) * (size_t)n_out * s;
}

int sweep_small_launch(int r, int nprim, int s, int n_out, int64_t F, const z_t* prims,
                       const z_t* alpha, const z_t* b, int64_t b_stride_f, const z_t* c_r, z_t* y,
                       double* spl, z_t* x, int* info, cudaStream_t stream) {
  constexpr int NT = 256;
  size_t smem = sweep_small_smem_bytes(r, nprim, s, n_out);
  auto kern = rom_sweep_small_kernel<NT>;
  VB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int dev = 0, nsm = 0, per_sm = 0;
  VB_CUDA(cudaGetDevice(&dev));
  VB_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  VB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NT, smem));
  if (per_sm < 1) per_sm = 1;
  int64_t grid = (int64_t)nsm * per_sm;
  if (grid > F) grid = F;
  if (grid < 1) return 0;
  kern<<<(unsigned)grid, NT, smem, stream>>>(r, nprim, s, n_out, F, prims, alpha, b, b_stride_f, c_r,
                                              y, spl, x, info);
  VB_LAUNCHED("rom_sweep_small_kernel");
  return 0;
}

}  // namespace vb
