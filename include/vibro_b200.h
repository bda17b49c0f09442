/*
 * vibro_b200 — C ABI of the B200-native MOR frequency-sweep path.
 *
 * Drop-in boundary.  The reference (`vibrofem`, pure Python)
 * has no FFI; its boundary is the duck-typed provider API of
 * vibrofem/mor.py and vibrofem/assembly.py.  Each entry point below replaces
 * the compiled third-party routine that reference call site binds (scipy
 * SuperLU / sparsetools, LAPACK zgesv, BLAS zgemm), with the reference call
 * site cited.  The Python host (paper_2310_04734_b200/) mirrors the
 * reference classes and binds these symbols with ctypes.
 *
 * Conventions
 *  - All array pointers are DEVICE pointers (cudaMalloc / torch CUDA tensors)
 *    unless the parameter name ends in `_host`.
 *  - complex128 is interleaved (re, im) doubles: the numpy / torch layout.
 *  - Dense matrices are row-major (C order) with the stated leading dimension.
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *    Every call is stream-ordered and asynchronous unless documented otherwise.
 *  - Return value: 0 on success, 1 invalid argument, 2 CUDA error,
 *    3 unsupported shape.  vb_last_error() returns the message of the last
 *    failure on the calling host thread.
 */
#ifndef VIBRO_B200_H
#define VIBRO_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  double re, im;
} vb_complex;

/* Library version string, e.g. "vibro_b200 0.1.0 sm_100a". */
const char* vb_version(void);

/* Message of the last failing call on this host thread ("" if none). */
const char* vb_last_error(void);

/*
 * Reduced frequency sweep over an affine reduced operator.
 *
 * Replaces, for every frequency f_i (i < F):
 *   vibrofem/mor.py:73-90   ReducedModel.reduced_system:  A_r = V^H K V - w^2 V^H M V (+ i w V^H D V)
 *                            written as A_r(f_i) = sum_k alpha[i,k] * prims[k]
 *   vibrofem/mor.py:92-94   ReducedModel.solve: numpy.linalg.solve(A_r, b_r) (LAPACK zgesv)
 *   vibrofem/mor.py:96-102  ReducedModel.output: y = (c_out V) x_r
 *   vibrofem/solvers.py:334-338 mean_spl(y[:, c]) for each RHS column c
 *
 *  r, nprim, s, n_out, F : reduced order, number of primitives, RHS columns,
 *                          output rows, frequencies
 *  prims  [nprim][r][r]  complex128   projected primitives V^H P_k V
 *  alpha  [F][nprim]     complex128   per-frequency coefficients
 *  b      [r][s] (b_stride_f = 0) or [F][r][s] (b_stride_f = r*s)  complex128
 *  c_r    [n_out][r]     complex128   reduced output map c_out V
 *  y      [F][n_out][s]  complex128   out, may be NULL
 *  spl    [F][s]         float64      out (dB re 20 uPa), may be NULL
 *  x      [F][r][s]      complex128   out reduced solutions, may be NULL
 *  info   [F]            int32        out, 0 or k+1 for the first exactly-zero
 *                                     pivot (LAPACK zgetrf INFO), may be NULL
 *  work / work_bytes     device scratch of at least
 *                        vb_rom_sweep_workspace_bytes(r, nprim, s, n_out, F)
 */
size_t vb_rom_sweep_workspace_bytes(int r, int nprim, int s, int n_out, int64_t F);
int vb_rom_sweep(int r, int nprim, int s, int n_out, int64_t F, const vb_complex* prims,
                 const vb_complex* alpha, const vb_complex* b, int64_t b_stride_f,
                 const vb_complex* c_r, vb_complex* y, double* spl, vb_complex* x, int32_t* info,
                 void* work, size_t work_bytes, void* stream);

/* Which algorithm vb_rom_sweep uses for (r, s, n_out): 0 = shared-memory
 * resident (one CTA per frequency), 1 = blocked (global-memory batched LU). */
int vb_rom_sweep_path(int r, int nprim, int s, int n_out);

/* Testing hook: force the sweep algorithm (0 shared-memory, 1 blocked) for
 * every later call in this process; -1 restores the automatic choice.  A
 * forced shared-memory path still fails with rc=3 when it does not fit. */
void vb_set_sweep_path_override(int path);

/* Measured FP64 tensor-pipe (DMMA, mma.sync.m8n8k4.f64) throughput of this
 * device in TFLOP/s, written to *tflops_host; synchronous (~10 ms).  Used as
 * the FP64 roofline denominator (MEASURED_PEAKS.json has no FP64 entry). */
int vb_probe_fp64_peak(double* tflops_host, void* stream);

/* Number of this library's kernel launches since load (process-wide counter,
 * incremented on every successful launch). */
int64_t vb_launch_count(void);

#ifdef __cplusplus
}
#endif

#endif /* VIBRO_B200_H */
