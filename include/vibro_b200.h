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

/* ------------------------------------------------------------------------
 * FE primitives
 * ---------------------------------------------------------------------- */

/*
 * Canonical CSR pattern of an element triplet stream.  Replaces
 * vibrofem/assembly.py:160-175 (rows = repeat(dofs, e), cols = tile(dofs, e)
 * per element in index order; scipy coo_matrix.tocsr() + sum_duplicates()):
 * indptr/indices are bit-identical to scipy's (sorted int32 column indices,
 * explicit zeros kept because the pattern is structural).
 *  conn        [n_elem][npe] int32 global dof ids
 *  indptr      [n+1]  out
 *  indices     [n_elem*npe*npe] out (first *nnz_host used)
 *  gather_ptr  [n_elem*npe*npe + 1] out: slot s sums triplets
 *              gather_idx[gather_ptr[s] .. gather_ptr[s+1]) in element order
 *  gather_idx  [n_elem*npe*npe] out
 *  nnz_host    out (HOST pointer); the call synchronises the stream.
 */
size_t vb_csr_pattern_workspace_bytes(int n, int n_elem, int npe);
int vb_csr_pattern_from_elements(int n, int n_elem, int npe, const int32_t* conn, int32_t* indptr,
                                 int32_t* indices, int64_t* gather_ptr, int32_t* gather_idx,
                                 int64_t* nnz_host, void* work, size_t work_bytes, void* stream);

/* Rectangular / constrained generalisation: triplet t = e*nr*nc + a*nc + b has
 * row row_dofs[e][a] and column col_dofs[e][b] (n_rows x n_cols matrix); a
 * negative DoF (eliminated, e.g. clamped) drops the triplet.  Same outputs and
 * gather semantics as vb_csr_pattern_from_elements (gather lists index the
 * full triplet stream, so dropped triplets are simply never referenced). */
size_t vb_csr_pattern_blocks_workspace_bytes(int n_rows, int n_cols, int n_elem, int nr, int nc);
int vb_csr_pattern_from_blocks(int n_rows, int n_cols, int n_elem, int nr, int nc, const int32_t* row_dofs,
                               const int32_t* col_dofs, int32_t* indptr, int32_t* indices, int64_t* gather_ptr,
                               int32_t* gather_idx, int64_t* nnz_host, void* work, size_t work_bytes, void* stream);

/* 9-node Reissner-Mindlin + membrane plate element matrices (cfg2 plate; no
 * reference counterpart — restated with the conventions of
 * vibrofem/assembly.py:31-67): node DoFs (u, v, w, bx, by), local nodes a + 3b,
 * xyz [n_nodes][3] (plate in the x-y plane), conn [n_elem][9],
 * Ke, Me [n_elem][45][45] out (undamped; the loss factor is applied as a
 * complex scalar (1 + i eta(f)) on the assembled stiffness). */
int vb_rm_plate_elements(int n_elem, const double* xyz, const int32_t* conn, double E, double nu, double rho,
                         double t, double* Ke, double* Me, int32_t* bad_elem_host, void* stream);

/* CSR values from triplet values: vals[s] = sum of triplet_vals over the
 * slot's gather list, in element order (deterministic; assembly.py:172-173). */
int vb_csr_gather(int64_t nnz, const int64_t* gather_ptr, const int32_t* gather_idx,
                  const double* triplet_vals, double* vals, void* stream);

/* The same for two primitives sharing the pattern (Kgrad, Mnn): one pass over
 * the gather map. */
int vb_csr_gather2(int64_t nnz, const int64_t* gather_ptr, const int32_t* gather_idx, const double* tv0,
                   const double* tv1, double* vals0, double* vals1, void* stream);

/* Unscaled Helmholtz integrals of 27-node hexahedra (vibrofem/assembly.py:77-91
 * generalised to 3D: J = dshape^T X, dN = dshape inv(J), 3x3x3 Gauss):
 *  xyz [n_nodes][3], conn [n_elem][27] (local node a + 3b + 9c),
 *  Ke, Me [n_elem][27][27] out (row-major; the triplet value order of
 *  assembly.py:166-170).  *bad_elem_host = first element with detJ <= 0, or -1
 *  (the reference raises ValueError); synchronises the stream. */
int vb_hex27_helmholtz_elements(int n_elem, const double* xyz, const int32_t* conn, double* Ke,
                                double* Me, int32_t* bad_elem_host, void* stream);

/* Structured fast path (uniform axis-aligned hex27 box of nx x ny x nz equal
 * elements, BASELINE cfg1/cfg3): writes indptr [n+1], indices / Kvals / Mvals
 * [vb_hex27_box_nnz] directly — the same canonical pattern as
 * vb_csr_pattern_from_elements, values from the Kronecker form of the assembled
 * 1D quadratic matrices (the element sums of assembly.py:142-175 factorise):
 *  K1, M1 [3][maxnp][5] (device): band entries (offset j - i + 2) of the 1D
 *  stiffness / mass along x, y, z. */
int64_t vb_hex27_box_nnz(int nx, int ny, int nz);
int vb_hex27_box_csr(int nx, int ny, int nz, const double* K1, const double* M1, int maxnp, int32_t* indptr,
                     int32_t* indices, double* Kvals, double* Mvals, void* stream);

/* Impedance-wall primitive: int_Gamma N N^T dGamma on 9-node faces
 * (face_conn [n_faces][9], lexicographic), Fe [n_faces][9][9] out. */
int vb_quad9_face_mass(int n_faces, const double* xyz, const int32_t* face_conn, double* Fe,
                       void* stream);

/* cfg4 synthetic fuselage (BASELINE configs[3]; no reference element, SURVEY
 * §8c tier 2 — checked against oracle/fuselage.py):
 * the Helmholtz integrals of vb_hex27_helmholtz_elements with the chain rule
 * dN = dshape inv(J)^T instead of the reference's dshape inv(J)
 * (vibrofem/assembly.py:88; equal for diagonal J, the fuselage's mapped
 * cylindrical elements have non-diagonal J). */
int vb_hex27_helmholtz_elements_chain(int n_elem, const double* xyz, const int32_t* conn, double* Ke,
                                      double* Me, int32_t* bad_elem_host, void* stream);

/* Flat 9-node facet shells (skin, lining, floor, frame webs, stringers) in
 * global node DoFs (u_x, u_y, u_z, th_x, th_y, th_z): membrane = the
 * reference's plane-stress element (vibrofem/assembly.py:31-67), Reissner-
 * Mindlin bending + 2x2 shear, Hughes-Brezzi drilling term (drill * G t),
 * rotated from the facet frame.  mat [n_elem] indexes props [n_mat][4] =
 * (E, nu, rho, t) (device); Ke, Me [n_elem][54][54] out.  *bad_elem_host =
 * first element with detJ <= 0 or a material index outside [0, n_mat), or -1. */
int vb_facet_shell_elements(int n_elem, const double* xyz, const int32_t* conn, const int32_t* mat,
                            const double* props, int n_mat, double drill, double* Ke, double* Me,
                            int32_t* bad_elem_host, void* stream);

/* ------------------------------------------------------------------------
 * Offline-phase linear algebra
 * ---------------------------------------------------------------------- */

/* Y = alpha * A X + beta * Y with A a real CSR (float64 values, int32 indices)
 * and X (n_cols x k), Y (n_rows x k) complex row-major.  Replaces scipy
 * csr_matvecs in `K @ V`, `M @ v` (vibrofem/mor.py:81-85, 117, 162-179). */
int vb_csr_spmm(int n_rows, const int32_t* indptr, const int32_t* indices, const double* vals, int k,
                const vb_complex* X, int64_t ldx, vb_complex* Y, int64_t ldy, vb_complex alpha,
                vb_complex beta, void* stream);

/* Row-group form of a CSR pattern for the many-column SpMM (HOST pointers,
 * one-off per pattern; same call sites as vb_csr_spmm).  Greedy in row order:
 * an ungrouped row becomes a group leader and adopts up to 7 ungrouped rows
 * among its columns whose column sets are subsets of its own.  Outputs (sized
 * by the caller for the worst case: n_rows groups, nnz union slots):
 *   g_leader[G] (-1: a group of up to 8 EMPTY rows, listed after all others),
 *   g_rows[G][8] (member rows, -1 padded), g_uoff[G] (offset of
 *   the group's union = the leader's CSR row in the union space),
 *   masks[U] (bit i: member i has that column), vmap[U][8] (CSR position of
 *   (member i, union column j), -1 absent); *n_groups = G, *n_union = U. */
int vb_csr_row_groups(int n_rows, const int32_t* indptr_host, const int32_t* indices_host, int32_t* g_leader_host,
                      int32_t* g_rows_host, int32_t* g_uoff_host, uint8_t* masks_host, int32_t* vmap_host,
                      int* n_groups_host, int64_t* n_union_host);

/* gvals[U][8] = vmap >= 0 ? vals[vmap] : 0 (device): the values of one
 * primitive on its pattern's row groups. */
int vb_rg_gather_values(int64_t n_union, const int32_t* vmap, const double* vals, double* gvals, void* stream);

/* Y = alpha * A X + beta * Y through the row groups of A (device pointers;
 * indptr/indices are A's CSR arrays, which hold each group's union).  Equal
 * to vb_csr_spmm to rounding (dense 8-row blocks on the FP64 tensor cores). */
int vb_rg_spmm(int n_groups, const int32_t* g_leader, const int32_t* g_rows, const int32_t* g_uoff,
               const int32_t* indptr, const int32_t* indices, const uint8_t* masks, const double* gvals, int k,
               const vb_complex* X, int64_t ldx, vb_complex* Y, int64_t ldy, vb_complex alpha, vb_complex beta,
               void* stream);

/* Row-group SpMM kernel choice (default 0 = by column count): 1 forces the
 * FP64-tensor-core (DMMA) form over the padded dense 8-row blocks, 2 the
 * padding-free CUDA-core form (per-slot 8-bit membership masks).  Process-
 * wide; also read from the VB_RG_MODE environment variable at first use. */
void vb_set_rg_spmm_mode(int mode);

/* In-block Gram-Schmidt of a new basis block (vibrofem/mor.py:122-135, the
 * column loop of _orthonormalise after the block is projected on V), fused
 * into one cooperative kernel: for each column j of W (n x kb, kb <= 16),
 * two CGS passes against the kept columns Q[:, :nk], keep iff
 * refs[j] > 0 and ||w|| > drop_tol * refs[j] (a kept column with
 * ||w|| < reorth_ratio * refs[j] gets a third pass), Q[:, nk++] = w / ||w||.
 * W is overwritten with the orthogonalised columns.  kept[kb] (0/1) and
 * *nk (device) out.  no_drop = 1: keep every column (refs unused); Q may
 * equal W (in place).  Deterministic fixed-order reductions. */
size_t vb_block_gs_workspace_bytes(void);
int vb_block_gs(int n, int kb, vb_complex* W, int64_t ldw, const double* refs, double drop_tol, double reorth_ratio,
                int no_drop, vb_complex* Q, int64_t ldq, int32_t* kept, int32_t* nk, void* work, size_t work_bytes,
                void* stream);

/* Y = alpha * Op X + beta * Y for the assembled primitives of a uniform hex27
 * box WITHOUT the CSR: Op = Kx(x)My(x)Mz + Mx(x)Ky(x)Mz + Mx(x)My(x)Kz
 * (stiff = 1, Kgrad) or Mx(x)My(x)Mz (stiff = 0, Mnn), the exact Kronecker
 * form of the element sums; K1/M1 are the [3][maxnp][5] band tables of the 1D
 * assembled matrices (x, y, z; entry o couples nodes i and i+o-2), the same
 * tables vb_hex27_box_csr takes, so Op equals that CSR to rounding.  Grid of
 * npx x npy x npz nodes, row (z npy + y) npx + x; X, Y complex n x k row-major.
 * Replaces `P @ V` (mor.py:81-85, 117) for box primitives. */
int vb_kron3_apply(int npx, int npy, int npz, const double* K1, const double* M1, int maxnp, int stiff, int k,
                   vb_complex alpha, const vb_complex* X, int64_t ldx, vb_complex beta, vb_complex* Y,
                   int64_t ldy, void* stream);

/* D += alpha * A: scatter a scaled real CSR primitive into a dense complex
 * matrix (row-major, ldd) — assembles K - w^2 M + i w D at an expansion point
 * (vibrofem/mor.py:41-46) for the dense full-order LU. */
int vb_csr_axpy_dense(int n_rows, const int32_t* indptr, const int32_t* indices, const double* vals,
                      vb_complex alpha, vb_complex* D, int64_t ldd, void* stream);

/* Complex GEMM on the FP64 tensor cores (DMMA).  Replaces numpy/BLAS zgemm in
 * vibrofem/mor.py:81-89, 102, 105, 117-118, 129-131.
 *  transa = 'N': C (m x n) = alpha A B + beta C,    A m x k, B k x n
 *  transa = 'C': C (m x n) = alpha A^H B + beta C,  A k x m, B k x n
 *                (split-K over k with a fixed-order reduction: deterministic)
 * All row-major with the given leading dimensions. */
size_t vb_zgemm_workspace_bytes(char transa, int m, int n, int k);
int vb_zgemm(char transa, int m, int n, int k, vb_complex alpha, const vb_complex* A, int64_t lda,
             const vb_complex* B, int64_t ldb, vb_complex beta, vb_complex* C, int64_t ldc, void* work,
             size_t work_bytes, void* stream);

/*
 * Dense complex LU with partial pivoting of ONE n x n matrix (row-major, lda),
 * in place, on the whole GPU (persistent cooperative kernel).  The full-order
 * solver at expansion / certification frequencies: replaces scipy
 * splu(csc(A(f))) in vibrofem/mor.py:48-49, 153-156 (and the residual
 * contract of solvers.py:62-78) for n up to ~25k.  Pivoting follows LAPACK
 * zgetf2 (izamax: max |Re|+|Im|, lowest row on ties).
 *  ipiv [n] out (0-based row interchanged with row j at step j)
 *  info [1] out (device): 0, or k+1 for the first exactly-zero pivot
 *  aux  out: diagonal-block inverses + permutation used by vb_zgetrs
 *  (vb_zgetrf_aux_bytes(n)); keep it with the factors.
 */
/* Batched complex GEMV with few right-hand sides:
 *   Y_b (m x s) = alpha_b A_b (m x n) X_b (n x s) + beta_b Y_b,  1 <= s <= 16,
 * all row-major device arrays; items is a HOST array.  The solve phase of the
 * plane-block full-order solver (cfg4: replaces the triangular solves of
 * scipy splu's `lu.solve`, vibrofem/mor.py:49, 156, 166, 175). */
#define VB_GEMV_MAX 32
typedef struct {
  int32_t m, n, s, pad;
  const vb_complex* A;
  int64_t lda;
  const vb_complex* X;
  int64_t ldx;
  vb_complex* Y;
  int64_t ldy;
  vb_complex alpha, beta;
} vb_gemv_item;
int vb_zgemv_batched(int n_items, const vb_gemv_item* items, void* stream);

size_t vb_zgetrf_workspace_bytes(int n);
size_t vb_zgetrf_aux_bytes(int n);
int vb_zgetrf(int n, vb_complex* A, int64_t lda, int32_t* ipiv, int32_t* info, void* aux,
              size_t aux_bytes, void* work, size_t work_bytes, void* stream);

/* Calling host thread only: launch vb_zgetrf / vb_zgetrs on at most n CTAs
 * (0 = one per SM, the default), so that independent factorisations and
 * solves issued from several host threads on their own streams run
 * concurrently (e.g. the expansion points of one Krylov basis). */
void vb_set_lu_max_ctas(int n);

/* Whole-GPU LU variant (default 1, also env VB_LU_LOOKAHEAD at first use):
 * 1 = look-ahead kernel (a group of panel CTAs factors panel k+1 while the
 * other CTAs run the trailing update of panel k) where the order and grid
 * allow it, 0 = one grid barrier per panel column for all CTAs.  Same pivots
 * and results either way. */
void vb_set_lu_lookahead(int on);

/* X = A^-1 B from vb_zgetrf factors (1 <= nrhs <= 16; B may alias X).
 * Replaces SuperLU `lu.solve` (vibrofem/mor.py:49, 156, 166, 175). */
size_t vb_zgetrs_workspace_bytes(int n, int nrhs);
int vb_zgetrs(int n, int nrhs, const vb_complex* LU, int64_t lda, const void* aux, const vb_complex* B,
              int64_t ldb, vb_complex* X, int64_t ldx, void* work, size_t work_bytes, void* stream);

/*
 * Fast-diagonalisation full-order solver on structured hex27 boxes (cfg3,
 * n = 376k, where scipy splu — vibrofem/mor.py:48-49, 153-156 — is
 * impractical).  The box operator is a Kronecker sum; the host computes the
 * per-direction generalised eigenpairs, the device applies
 *   x = V (Lz (+) Ly (+) Lx + sigma)^-1 V^T b,  V = Vz (x) Vy (x) Vx.
 * Arrays are (n2, n1, n0) nodes x nrhs, RHS fastest (node id k n1 n0 + j n0 + i).
 *  vb_axis_apply: Y = S applied along axis (0 = x, 1 = y, 2 = z); S is
 *                 n_axis x n_axis row-major; X and Y must not alias.
 *  vb_fdm_diag:   X /= (lz[k] + ly[j] + lx[i] + sigma).
 */
int vb_axis_apply(int n2, int n1, int n0, int nrhs, int axis, const vb_complex* S, const vb_complex* X,
                  vb_complex* Y, void* stream);
int vb_fdm_diag(int n2, int n1, int n0, int nrhs, const vb_complex* lz, const vb_complex* ly,
                const vb_complex* lx, vb_complex sigma, vb_complex* X, void* stream);
/*  vb_fdm_solve: X = A^-1 B in one call on the FP64 tensor cores (the three
 *  1-D transforms each way as DMMA GEMMs in an internal RHS-slowest layout,
 *  transposed in and out).  V_d / VT_d: n_d x n_d row-major eigenvectors and
 *  their transposes; B, X: n x nrhs row-major with leading dimensions;
 *  work >= vb_fdm_solve_workspace_bytes (2 n nrhs complex).  Replaces the
 *  per-column scipy splu solve (vibrofem/mor.py:48-49, 153-156) on boxes. */
size_t vb_fdm_solve_workspace_bytes(int n2, int n1, int n0, int nrhs);
int vb_fdm_solve(int n2, int n1, int n0, int nrhs, const vb_complex* Vx, const vb_complex* Vy, const vb_complex* Vz,
                 const vb_complex* VTx, const vb_complex* VTy, const vb_complex* VTz, const vb_complex* lx,
                 const vb_complex* ly, const vb_complex* lz, vb_complex sigma, const vb_complex* B, int64_t ldb,
                 vb_complex* X, int64_t ldx, void* work, size_t work_bytes, void* stream);

/* norms[j] = ||W[:, j]||_2 for an n x m complex row-major W (deterministic). */
size_t vb_column_norms_workspace_bytes(int n, int m);
int vb_column_norms(int n, int m, const vb_complex* W, int64_t ldw, double* norms, void* work,
                    size_t work_bytes, void* stream);

/* W[:, j] *= scale[j] (scale: device float64[m]). */
int vb_scale_columns(int n, int m, vb_complex* W, int64_t ldw, const double* scale, void* stream);

/* Batched classical Gram-Schmidt pass of k side-by-side Arnoldi processes
 * (GPU GMRES, gmres.py; replaces the MGS loop of solvers.py:236-239 in the
 * reference's gmres, solvers.py:191-264).  Column c's basis is V[:, c, 0:j]
 * with element (row, c, i) at V[row * ldr + c * ldc + i]; W is n x k
 * row-major (ldw).  vb_batched_dots: H[c * j + i] = sum_row conj(V[row,c,i])
 * W[row,c] (per-CTA partials reduced in a fixed order: deterministic);
 * vb_batched_update: W[row,c] -= sum_i V[row,c,i] H[c * j + i]. */
size_t vb_batched_dots_workspace_bytes(int k, int j);
int vb_batched_dots(int64_t n, int k, int j, const vb_complex* V, int64_t ldr, int64_t ldc, const vb_complex* W,
                    int64_t ldw, vb_complex* H, void* work, size_t work_bytes, void* stream);
int vb_batched_update(int64_t n, int k, int j, const vb_complex* V, int64_t ldr, int64_t ldc, const vb_complex* H,
                      vb_complex* W, int64_t ldw, void* stream);

/* Measured FP64 tensor-pipe (DMMA, mma.sync.m8n8k4.f64) throughput of this
 * device in TFLOP/s, written to *tflops_host; synchronous (~10 ms).  Used as
 * the FP64 roofline denominator (MEASURED_PEAKS.json has no FP64 entry). */
int vb_probe_fp64_peak(double* tflops_host, void* stream);

/* Profiling aid: per-phase SM-cycle totals of the blocked sweep kernel (36
 * counters; non-zero only in a library built with -DVB_PHASE_TIMING).  Phases:
 * form, leaf panel, in-panel TRSM+GEMM, interchanges, U12 TRSM, trailing GEMM,
 * back substitution, outputs; 8..15 leaf sub-phases; 16..23 the TMA GEMM's
 * wait/compute/epilogue split for a consumer warp and for the producer thread;
 * 24..29 the skinny (in-panel) GEMM split; 32..35 vb_zgetrf's panel / swaps /
 * TRSM / GEMM phases (CTA 0). */
int vb_debug_phase_cycles(unsigned long long* cycles_host, int reset);

/* Opt-in L2 persistence for the blocked reduced sweep (default off): while
 * enabled, each vb_rom_sweep launch on the blocked path raises the device's
 * persisting-L2 limit to the primitives' size and marks them persisting
 * (access-policy window), so the per-frequency workspace streaming does not
 * evict them.  Device-wide state: pair with vb_release_l2_persistence. */
void vb_set_l2_persistence(int enable);

/* Give back the L2 set-aside reserved while persistence was enabled: resets
 * persisting lines and restores the persisting-L2 limit the device had
 * before the first raise. */
int vb_release_l2_persistence(void);

/* Number of this library's kernel launches since load (process-wide counter,
 * incremented on every successful launch). */
int64_t vb_launch_count(void);

#ifdef __cplusplus
}
#endif

#endif /* VIBRO_B200_H */
