// extern "C" entry points of libvibro_b200.so (declared in include/vibro_b200.h).
#include <atomic>
#include <string>

#include "../../include/vibro_b200.h"
#include "common.cuh"
#include "sweep.cuh"

namespace vb {

static thread_local std::string g_last_error;
static std::atomic<int64_t> g_launches{0};

void set_error(const std::string& msg) { g_last_error = msg; }

int check_cuda(cudaError_t e, const char* where) {
  if (e == cudaSuccess) return 0;
  set_error(std::string(where) + ": " + cudaGetErrorString(e));
  return 2;
}

int check_launch(const char* where) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return check_cuda(e, where);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return 0;
}

void count_launches(int64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

}  // namespace vb

using vb::z_t;

extern "C" {

const char* vb_version(void) { return "vibro_b200 0.1.0 sm_100a"; }

const char* vb_last_error(void) { return vb::g_last_error.c_str(); }

int64_t vb_launch_count(void) { return vb::g_launches.load(); }

int vb_release_l2_persistence(void) { return vb::sweep_release_l2_persistence(); }

void vb_set_l2_persistence(int enable) { vb::sweep_set_l2_persistence(enable); }

int vb_rom_sweep_path(int r, int nprim, int s, int n_out) { return vb::sweep_path(r, nprim, s, n_out); }

void vb_set_sweep_path_override(int path) { vb::sweep_set_override(path); }

void vb_set_rg_spmm_mode(int mode) { vb::set_rg_mode(mode); }

int vb_probe_fp64_peak(double* tflops_host, void* stream) {
  VB_CHECK_ARG(tflops_host != nullptr, "vb_probe_fp64_peak: null output");
  return vb::probe_fp64_peak(tflops_host, (cudaStream_t)stream);
}

size_t vb_rom_sweep_workspace_bytes(int r, int nprim, int s, int n_out, int64_t F) {
  return vb::sweep_workspace_bytes(r, nprim, s, n_out, F);
}

int vb_rom_sweep(int r, int nprim, int s, int n_out, int64_t F, const vb_complex* prims,
                 const vb_complex* alpha, const vb_complex* b, int64_t b_stride_f,
                 const vb_complex* c_r, vb_complex* y, double* spl, vb_complex* x, int32_t* info,
                 void* work, size_t work_bytes, void* stream) {
  VB_CHECK_ARG(r >= 1 && nprim >= 1 && nprim <= 64 && s >= 1 && n_out >= 0 && F >= 0,
               "vb_rom_sweep: bad sizes");
  if (F == 0) return 0;  // nothing to sweep (alpha / outputs may be empty, i.e. NULL)
  VB_CHECK_ARG(prims && alpha && b, "vb_rom_sweep: null input");
  VB_CHECK_ARG(n_out == 0 || c_r, "vb_rom_sweep: c_r is NULL with n_out > 0");
  VB_CHECK_ARG(b_stride_f == 0 || b_stride_f >= (int64_t)r * s, "vb_rom_sweep: bad b_stride_f");
  if (F == 0) return 0;
  return vb::sweep_run(r, nprim, s, n_out, F, (const z_t*)prims, (const z_t*)alpha, (const z_t*)b,
                       b_stride_f, (const z_t*)c_r, (z_t*)y, spl, (z_t*)x, info, work, work_bytes,
                       (cudaStream_t)stream);
}

size_t vb_csr_pattern_workspace_bytes(int n, int n_elem, int npe) {
  return vb::csr_pattern_workspace_bytes(n, (int64_t)n_elem * npe * npe);
}

int vb_csr_pattern_from_elements(int n, int n_elem, int npe, const int32_t* conn, int32_t* indptr,
                                 int32_t* indices, int64_t* gather_ptr, int32_t* gather_idx,
                                 int64_t* nnz_host, void* work, size_t work_bytes, void* stream) {
  VB_CHECK_ARG(n > 0 && n_elem > 0 && npe > 0, "vb_csr_pattern_from_elements: bad sizes");
  VB_CHECK_ARG(conn && indptr && indices && gather_ptr && gather_idx && nnz_host,
               "vb_csr_pattern_from_elements: null pointer");
  return vb::csr_pattern_from_elements(n, n_elem, npe, conn, indptr, indices, gather_ptr, gather_idx,
                                       nnz_host, work, work_bytes, (cudaStream_t)stream);
}

size_t vb_csr_pattern_blocks_workspace_bytes(int n_rows, int n_cols, int n_elem, int nr, int nc) {
  return vb::csr_pattern_workspace_bytes(n_rows > n_cols ? n_rows : n_cols, (int64_t)n_elem * nr * nc);
}

int vb_csr_pattern_from_blocks(int n_rows, int n_cols, int n_elem, int nr, int nc, const int32_t* row_dofs,
                               const int32_t* col_dofs, int32_t* indptr, int32_t* indices, int64_t* gather_ptr,
                               int32_t* gather_idx, int64_t* nnz_host, void* work, size_t work_bytes, void* stream) {
  VB_CHECK_ARG(n_rows > 0 && n_cols > 0 && n_elem > 0 && nr > 0 && nc > 0, "vb_csr_pattern_from_blocks: bad sizes");
  VB_CHECK_ARG(row_dofs && col_dofs && indptr && indices && gather_ptr && gather_idx && nnz_host,
               "vb_csr_pattern_from_blocks: null pointer");
  return vb::csr_pattern_from_blocks(n_rows, n_cols, n_elem, nr, nc, row_dofs, col_dofs, indptr, indices, gather_ptr,
                                     gather_idx, nnz_host, work, work_bytes, (cudaStream_t)stream);
}

int vb_rm_plate_elements(int n_elem, const double* xyz, const int32_t* conn, double E, double nu, double rho,
                         double t, double* Ke, double* Me, int32_t* bad_elem_host, void* stream) {
  VB_CHECK_ARG(n_elem >= 0 && xyz && conn && Ke && Me && bad_elem_host && t > 0,
               "vb_rm_plate_elements: bad arguments");
  return vb::rm_plate_elements(n_elem, xyz, conn, E, nu, rho, t, Ke, Me, bad_elem_host, (cudaStream_t)stream);
}

int vb_csr_gather2(int64_t nnz, const int64_t* gather_ptr, const int32_t* gather_idx, const double* tv0,
                   const double* tv1, double* vals0, double* vals1, void* stream) {
  VB_CHECK_ARG(nnz >= 0, "vb_csr_gather2: bad nnz");
  return vb::csr_gather2(nnz, gather_ptr, gather_idx, tv0, tv1, vals0, vals1, (cudaStream_t)stream);
}

int vb_csr_gather(int64_t nnz, const int64_t* gather_ptr, const int32_t* gather_idx,
                  const double* triplet_vals, double* vals, void* stream) {
  VB_CHECK_ARG(nnz >= 0, "vb_csr_gather: bad nnz");
  return vb::csr_gather(nnz, gather_ptr, gather_idx, triplet_vals, vals, (cudaStream_t)stream);
}

int vb_hex27_helmholtz_elements(int n_elem, const double* xyz, const int32_t* conn, double* Ke,
                                double* Me, int32_t* bad_elem_host, void* stream) {
  VB_CHECK_ARG(n_elem >= 0 && xyz && conn && Ke && Me && bad_elem_host,
               "vb_hex27_helmholtz_elements: bad arguments");
  return vb::hex27_helmholtz(n_elem, xyz, conn, Ke, Me, bad_elem_host, (cudaStream_t)stream);
}

int vb_hex27_helmholtz_elements_chain(int n_elem, const double* xyz, const int32_t* conn, double* Ke,
                                      double* Me, int32_t* bad_elem_host, void* stream) {
  VB_CHECK_ARG(n_elem >= 0 && xyz && conn && Ke && Me && bad_elem_host,
               "vb_hex27_helmholtz_elements_chain: bad arguments");
  return vb::hex27_helmholtz(n_elem, xyz, conn, Ke, Me, bad_elem_host, (cudaStream_t)stream, 1);
}

int vb_facet_shell_elements(int n_elem, const double* xyz, const int32_t* conn, const int32_t* mat,
                            const double* props, int n_mat, double drill, double* Ke, double* Me,
                            int32_t* bad_elem_host, void* stream) {
  VB_CHECK_ARG(n_elem >= 0 && n_mat > 0 && xyz && conn && mat && props && Ke && Me && bad_elem_host &&
                   drill >= 0.0,
               "vb_facet_shell_elements: bad arguments");
  return vb::facet_shell_elements(n_elem, xyz, conn, mat, props, n_mat, drill, Ke, Me, bad_elem_host,
                                  (cudaStream_t)stream);
}

int vb_quad9_face_mass(int n_faces, const double* xyz, const int32_t* face_conn, double* Fe,
                       void* stream) {
  VB_CHECK_ARG(n_faces >= 0 && xyz && face_conn && Fe, "vb_quad9_face_mass: bad arguments");
  return vb::quad9_face_mass(n_faces, xyz, face_conn, Fe, (cudaStream_t)stream);
}

static inline z_t zc(vb_complex a) { return vb::zmake(a.re, a.im); }

int vb_csr_spmm(int n_rows, const int32_t* indptr, const int32_t* indices, const double* vals, int k,
                const vb_complex* X, int64_t ldx, vb_complex* Y, int64_t ldy, vb_complex alpha,
                vb_complex beta, void* stream) {
  VB_CHECK_ARG(n_rows >= 0 && k >= 0, "vb_csr_spmm: bad sizes");
  return vb::csr_spmm(n_rows, indptr, indices, vals, k, (const z_t*)X, ldx, (z_t*)Y, ldy, zc(alpha),
                      zc(beta), (cudaStream_t)stream);
}

int vb_csr_row_groups(int n_rows, const int32_t* indptr, const int32_t* indices, int32_t* g_leader,
                      int32_t* g_rows, int32_t* g_uoff, uint8_t* masks, int32_t* vmap, int* n_groups,
                      int64_t* n_union) {
  VB_CHECK_ARG(n_rows >= 0 && indptr && indices && g_leader && g_rows && g_uoff && masks && vmap && n_groups &&
                   n_union,
               "vb_csr_row_groups: bad arguments");
  VB_CHECK_ARG(vb::csr_row_groups(n_rows, indptr, indices, g_leader, g_rows, g_uoff, masks, vmap, n_groups,
                                  n_union) == 0,
               "vb_csr_row_groups: union space exceeds int32");
  return 0;
}

int vb_rg_gather_values(int64_t n_union, const int32_t* vmap, const double* vals, double* gvals, void* stream) {
  VB_CHECK_ARG(n_union >= 0, "vb_rg_gather_values: bad sizes");
  return vb::rg_gather_values(n_union, vmap, vals, gvals, (cudaStream_t)stream);
}

int vb_rg_spmm(int n_groups, const int32_t* g_leader, const int32_t* g_rows, const int32_t* g_uoff,
               const int32_t* indptr, const int32_t* indices, const uint8_t* masks, const double* gvals, int k,
               const vb_complex* X, int64_t ldx, vb_complex* Y, int64_t ldy, vb_complex alpha, vb_complex beta,
               void* stream) {
  VB_CHECK_ARG(n_groups >= 0 && k >= 0, "vb_rg_spmm: bad sizes");
  return vb::rg_spmm(n_groups, g_leader, g_rows, g_uoff, indptr, indices, masks, gvals, k, (const z_t*)X, ldx,
                     (z_t*)Y, ldy, zc(alpha), zc(beta), (cudaStream_t)stream);
}

size_t vb_block_gs_workspace_bytes(void) { return vb::block_gs_workspace_bytes(); }

int vb_block_gs(int n, int kb, vb_complex* W, int64_t ldw, const double* refs, double drop_tol, double reorth_ratio,
                int no_drop, vb_complex* Q, int64_t ldq, int32_t* kept, int32_t* nk, void* work, size_t work_bytes,
                void* stream) {
  VB_CHECK_ARG(W && Q && kept && nk && (no_drop || refs), "vb_block_gs: null pointer");
  return vb::block_gs(n, kb, (z_t*)W, ldw, refs, drop_tol, reorth_ratio, no_drop, (z_t*)Q, ldq, kept, nk, work,
                      work_bytes, (cudaStream_t)stream);
}

int vb_csr_axpy_dense(int n_rows, const int32_t* indptr, const int32_t* indices, const double* vals,
                      vb_complex alpha, vb_complex* D, int64_t ldd, void* stream) {
  VB_CHECK_ARG(n_rows >= 0 && D, "vb_csr_axpy_dense: bad arguments");
  return vb::csr_axpy_dense(n_rows, indptr, indices, vals, zc(alpha), (z_t*)D, ldd, (cudaStream_t)stream);
}

size_t vb_zgemm_workspace_bytes(char transa, int m, int n, int k) {
  return vb::zgemm_workspace_bytes(transa, m, n, k);
}

int vb_zgemm(char transa, int m, int n, int k, vb_complex alpha, const vb_complex* A, int64_t lda,
             const vb_complex* B, int64_t ldb, vb_complex beta, vb_complex* C, int64_t ldc, void* work,
             size_t work_bytes, void* stream) {
  VB_CHECK_ARG(m >= 0 && n >= 0 && k >= 0, "vb_zgemm: bad sizes");
  return vb::zgemm(transa, m, n, k, zc(alpha), (const z_t*)A, lda, (const z_t*)B, ldb, zc(beta),
                   (z_t*)C, ldc, work, work_bytes, (cudaStream_t)stream);
}

size_t vb_column_norms_workspace_bytes(int n, int m) { return vb::column_norms_workspace_bytes(n, m); }

int vb_column_norms(int n, int m, const vb_complex* W, int64_t ldw, double* norms, void* work,
                    size_t work_bytes, void* stream) {
  return vb::column_norms(n, m, (const z_t*)W, ldw, norms, work, work_bytes, (cudaStream_t)stream);
}

int vb_scale_columns(int n, int m, vb_complex* W, int64_t ldw, const double* scale, void* stream) {
  VB_CHECK_ARG(n >= 0 && m >= 0, "vb_scale_columns: bad sizes");
  return vb::scale_columns(n, m, (z_t*)W, ldw, scale, (cudaStream_t)stream);
}

size_t vb_batched_dots_workspace_bytes(int k, int j) { return vb::batched_dots_workspace_bytes(k, j); }

int vb_batched_dots(int64_t n, int k, int j, const vb_complex* V, int64_t ldr, int64_t ldc, const vb_complex* W,
                    int64_t ldw, vb_complex* H, void* work, size_t work_bytes, void* stream) {
  VB_CHECK_ARG(n >= 0 && k >= 0 && j >= 0 && (k * j == 0 || (V && W && H)), "vb_batched_dots: bad arguments");
  return vb::batched_dots(n, k, j, (const z_t*)V, ldr, ldc, (const z_t*)W, ldw, (z_t*)H, work, work_bytes,
                          (cudaStream_t)stream);
}

int vb_batched_update(int64_t n, int k, int j, const vb_complex* V, int64_t ldr, int64_t ldc, const vb_complex* H,
                      vb_complex* W, int64_t ldw, void* stream) {
  VB_CHECK_ARG(n >= 0 && k >= 0 && j >= 0 && (k * j == 0 || (V && W && H)), "vb_batched_update: bad arguments");
  return vb::batched_update(n, k, j, (const z_t*)V, ldr, ldc, (const z_t*)H, (z_t*)W, ldw, (cudaStream_t)stream);
}

size_t vb_zgetrf_workspace_bytes(int n) { return vb::zgetrf_workspace_bytes(n); }
size_t vb_zgetrf_aux_bytes(int n) { return vb::zgetrf_aux_bytes(n); }

int vb_zgetrf(int n, vb_complex* A, int64_t lda, int32_t* ipiv, int32_t* info, void* aux,
              size_t aux_bytes, void* work, size_t work_bytes, void* stream) {
  VB_CHECK_ARG(A && ipiv && info, "vb_zgetrf: null pointer");
  return vb::zgetrf(n, (z_t*)A, lda, ipiv, info, aux, aux_bytes, work, work_bytes, (cudaStream_t)stream);
}

void vb_set_lu_max_ctas(int n) { vb::set_lu_max_ctas(n); }

void vb_set_lu_lookahead(int on) { vb::set_lu_lookahead(on); }

int vb_zgemv_batched(int n_items, const vb_gemv_item* items, void* stream) {
  VB_CHECK_ARG(n_items >= 0 && (n_items == 0 || items), "vb_zgemv_batched: bad arguments");
  return vb::zgemv_batched(n_items, items, (cudaStream_t)stream);
}

size_t vb_zgetrs_workspace_bytes(int n, int nrhs) { return (size_t)n * nrhs * sizeof(vb_complex); }

int vb_zgetrs(int n, int nrhs, const vb_complex* LU, int64_t lda, const void* aux, const vb_complex* B,
              int64_t ldb, vb_complex* X, int64_t ldx, void* work, size_t work_bytes, void* stream) {
  VB_CHECK_ARG(LU && aux && B && X, "vb_zgetrs: null pointer");
  return vb::zgetrs(n, nrhs, (const z_t*)LU, lda, aux, (const z_t*)B, ldb, (z_t*)X, ldx, work, work_bytes,
                    (cudaStream_t)stream);
}

int vb_axis_apply(int n2, int n1, int n0, int nrhs, int axis, const vb_complex* S, const vb_complex* X,
                  vb_complex* Y, void* stream) {
  return vb::axis_apply(n2, n1, n0, nrhs, axis, (const z_t*)S, (const z_t*)X, (z_t*)Y, (cudaStream_t)stream);
}

int vb_fdm_diag(int n2, int n1, int n0, int nrhs, const vb_complex* lz, const vb_complex* ly,
                const vb_complex* lx, vb_complex sigma, vb_complex* X, void* stream) {
  VB_CHECK_ARG(n0 > 0 && n1 > 0 && n2 > 0 && nrhs > 0 && lz && ly && lx && X, "vb_fdm_diag: bad arguments");
  return vb::fdm_diag(n2, n1, n0, nrhs, (const z_t*)lz, (const z_t*)ly, (const z_t*)lx, zc(sigma), (z_t*)X,
                      (cudaStream_t)stream);
}

size_t vb_fdm_solve_workspace_bytes(int n2, int n1, int n0, int nrhs) {
  return vb::fdm_solve_workspace_bytes(n2, n1, n0, nrhs);
}

int vb_fdm_solve(int n2, int n1, int n0, int nrhs, const vb_complex* Vx, const vb_complex* Vy, const vb_complex* Vz,
                 const vb_complex* VTx, const vb_complex* VTy, const vb_complex* VTz, const vb_complex* lx,
                 const vb_complex* ly, const vb_complex* lz, vb_complex sigma, const vb_complex* B, int64_t ldb,
                 vb_complex* X, int64_t ldx, void* work, size_t work_bytes, void* stream) {
  VB_CHECK_ARG(Vx && Vy && Vz && VTx && VTy && VTz && lx && ly && lz, "vb_fdm_solve: null factor pointer");
  VB_CHECK_ARG(ldb >= nrhs && ldx >= nrhs, "vb_fdm_solve: leading dimension smaller than nrhs");
  const z_t* V[3] = {(const z_t*)Vx, (const z_t*)Vy, (const z_t*)Vz};
  const z_t* VT[3] = {(const z_t*)VTx, (const z_t*)VTy, (const z_t*)VTz};
  return vb::fdm_solve(n2, n1, n0, nrhs, V, VT, (const z_t*)lx, (const z_t*)ly, (const z_t*)lz, zc(sigma),
                       (const z_t*)B, ldb, (z_t*)X, ldx, work, work_bytes, (cudaStream_t)stream);
}

int64_t vb_hex27_box_nnz(int nx, int ny, int nz) { return vb::hex27_box_nnz(nx, ny, nz); }

int vb_hex27_box_csr(int nx, int ny, int nz, const double* K1, const double* M1, int maxnp, int32_t* indptr,
                     int32_t* indices, double* Kvals, double* Mvals, void* stream) {
  VB_CHECK_ARG(K1 && M1 && indptr && indices && Kvals && Mvals, "vb_hex27_box_csr: null pointer");
  return vb::hex27_box_csr(nx, ny, nz, K1, M1, maxnp, indptr, indices, Kvals, Mvals, (cudaStream_t)stream);
}

int vb_kron3_apply(int npx, int npy, int npz, const double* K1, const double* M1, int maxnp, int stiff, int k,
                   vb_complex alpha, const vb_complex* X, int64_t ldx, vb_complex beta, vb_complex* Y,
                   int64_t ldy, void* stream) {
  VB_CHECK_ARG(K1 && M1 && X && Y, "vb_kron3_apply: null pointer");
  return vb::kron3_apply(npx, npy, npz, K1, M1, maxnp, stiff, k, zc(alpha), (const z_t*)X, ldx, zc(beta),
                         (z_t*)Y, ldy, (cudaStream_t)stream);
}

int vb_debug_phase_cycles(unsigned long long* cycles_host, int reset) {
  VB_CHECK_ARG(cycles_host != nullptr, "vb_debug_phase_cycles: null output");
  return vb::sweep_debug_phase_cycles(cycles_host, reset);
}

}  // extern "C"
