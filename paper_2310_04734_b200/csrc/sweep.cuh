// Internal interface of the reduced-sweep kernels (dispatch in sweep.cu).
#pragma once
#include <cuda.h>

#include "common.cuh"
#include "../../include/vibro_b200.h"

namespace vb {

// 3-D FP64 tensor map (doubles x rows x slabs, 128B swizzle) for the TMA GEMMs.
int tma_encode_map(CUtensorMap* map, void* base, const cuuint64_t* dims, const cuuint64_t* strides,
                   const cuuint32_t* box, const cuuint32_t* es);

size_t sweep_small_smem_bytes(int r, int nprim, int s, int n_out);
int sweep_small_launch(int r, int nprim, int s, int n_out, int64_t F, const z_t* prims,
                       const z_t* alpha, const z_t* b, int64_t b_stride_f, const z_t* c_r, z_t* y,
                       double* spl, z_t* x, int* info, cudaStream_t stream);

int sweep_path(int r, int nprim, int s, int n_out);
void sweep_set_override(int path);
void set_rg_mode(int mode);
void sweep_set_l2_persistence(int enable);
int sweep_release_l2_persistence();
size_t sweep_workspace_bytes(int r, int nprim, int s, int n_out, int64_t F);
int sweep_run(int r, int nprim, int s, int n_out, int64_t F, const z_t* prims, const z_t* alpha,
              const z_t* b, int64_t b_stride_f, const z_t* c_r, z_t* y, double* spl, z_t* x,
              int* info, void* work, size_t work_bytes, cudaStream_t stream);
void count_launches(int64_t n);
int probe_fp64_peak(double* tflops, cudaStream_t stream);

size_t sweep_blocked_workspace_bytes(int r, int s, int n_out, int64_t F);
int sweep_blocked_supported(int r, int s, int n_out);
int sweep_debug_phase_cycles(unsigned long long* out_host, int reset);
int lu_debug_cycles(unsigned long long* out, int reset);
int kron3_apply(int npx, int npy, int npz, const double* K1, const double* M1, int maxnp, int stiff, int k,
                z_t alpha, const z_t* X, int64_t ldx, z_t beta, z_t* Y, int64_t ldy, cudaStream_t st);
int sweep_blocked_launch(int r, int nprim, int s, int n_out, int64_t F, const z_t* prims,
                         const z_t* alpha, const z_t* b, int64_t b_stride_f, const z_t* c_r, z_t* y,
                         double* spl, z_t* x, int* info, void* work, size_t work_bytes,
                         cudaStream_t stream);


// assembly.cu
size_t csr_pattern_workspace_bytes(int n, int64_t T);
int csr_pattern_from_elements(int n, int n_elem, int npe, const int32_t* conn, int32_t* indptr,
                              int32_t* indices, int64_t* gptr, int32_t* gidx, int64_t* nnz_host,
                              void* work, size_t work_bytes, cudaStream_t stream);
int csr_pattern_from_blocks(int n_rows, int n_cols, int n_elem, int nr, int nc, const int32_t* rdofs,
                            const int32_t* cdofs, int32_t* indptr, int32_t* indices, int64_t* gptr, int32_t* gidx,
                            int64_t* nnz_host, void* work, size_t work_bytes, cudaStream_t stream);
int rm_plate_elements(int n_elem, const double* xyz, const int32_t* conn, double E, double nu, double rho, double t,
                      double* Ke, double* Me, int32_t* bad_elem_host, cudaStream_t stream);
int csr_gather2(int64_t nnz, const int64_t* gptr, const int32_t* gidx, const double* tv0, const double* tv1,
                double* v0, double* v1, cudaStream_t stream);
int csr_gather(int64_t nnz, const int64_t* gptr, const int32_t* gidx, const double* tv, double* vals,
               cudaStream_t stream);
int hex27_helmholtz(int n_elem, const double* xyz, const int32_t* conn, double* Ke, double* Me,
                    int32_t* bad_elem_host, cudaStream_t stream, int chain = 0);
int facet_shell_elements(int n_elem, const double* xyz, const int32_t* conn, const int32_t* mat,
                         const double* props, int n_mat, double drill, double* Ke, double* Me,
                         int32_t* bad_elem_host, cudaStream_t stream);
int quad9_face_mass(int n_faces, const double* xyz, const int32_t* fconn, double* Fe,
                    cudaStream_t stream);


int64_t hex27_box_nnz(int nx, int ny, int nz);
int hex27_box_csr(int nx, int ny, int nz, const double* K1, const double* M1, int maxnp, int32_t* indptr,
                  int32_t* indices, double* Kv, double* Mv, cudaStream_t st);

// spmm.cu
int csr_row_groups(int n, const int32_t* indptr, const int32_t* indices, int32_t* g_leader, int32_t* g_rows,
                   int32_t* g_uoff, uint8_t* masks, int32_t* vmap, int* n_groups, int64_t* n_slots);
int rg_gather_values(int64_t n_union, const int32_t* vmap, const double* vals, double* gvals, cudaStream_t st);
int rg_spmm(int n_groups, const int32_t* g_leader, const int32_t* g_rows, const int32_t* g_uoff,
            const int32_t* indptr, const int32_t* indices, const uint8_t* masks, const double* gvals, int k,
            const z_t* X, int64_t ldx, z_t* Y, int64_t ldy, z_t alpha, z_t beta, cudaStream_t st);
int csr_spmm(int n_rows, const int32_t* indptr, const int32_t* indices, const double* vals, int k,
             const z_t* X, int64_t ldx, z_t* Y, int64_t ldy, z_t alpha, z_t beta, cudaStream_t st);
// blockgs.cu
size_t block_gs_workspace_bytes();
int block_gs(int n, int kb, z_t* W, int64_t ldw, const double* refs, double tol, double reorth, int no_drop,
             z_t* Q, int64_t ldq, int32_t* kept, int32_t* nk, void* work, size_t wb, cudaStream_t st);
// linalg.cu
int csr_axpy_dense(int n_rows, const int32_t* indptr, const int32_t* indices, const double* vals,
                   z_t alpha, z_t* D, int64_t ldd, cudaStream_t st);
size_t zgemm_workspace_bytes(char transa, int m, int n, int k);
int zgemm(char transa, int m, int n, int k, z_t alpha, const z_t* A, int64_t lda, const z_t* B,
          int64_t ldb, z_t beta, z_t* C, int64_t ldc, void* work, size_t work_bytes, cudaStream_t st);
size_t batched_dots_workspace_bytes(int k, int j);
int batched_dots(int64_t n, int k, int j, const z_t* V, int64_t ldr, int64_t ldc, const z_t* W, int64_t ldw, z_t* H,
                 void* work, size_t work_bytes, cudaStream_t st);
int batched_update(int64_t n, int k, int j, const z_t* V, int64_t ldr, int64_t ldc, const z_t* H, z_t* W,
                   int64_t ldw, cudaStream_t st);
int zgemv_batched(int n_items, const vb_gemv_item* items, cudaStream_t st);
size_t column_norms_workspace_bytes(int n, int m);
int column_norms(int n, int m, const z_t* W, int64_t ldw, double* out, void* work, size_t wb,
                 cudaStream_t st);
int scale_columns(int n, int m, z_t* W, int64_t ldw, const double* scale, cudaStream_t st);


// lu.cu
size_t zgetrf_workspace_bytes(int n);
size_t zgetrf_aux_bytes(int n);
int zgetrf(int n, z_t* A, int64_t lda, int* ipiv, int* info_dev, void* aux, size_t aux_bytes, void* work,
           size_t work_bytes, cudaStream_t st);
void set_lu_max_ctas(int n);
void set_lu_lookahead(int on);
int zgetrs(int n, int nrhs, const z_t* LU, int64_t lda, const void* aux, const z_t* B, int64_t ldb,
           z_t* X, int64_t ldx, void* work, size_t work_bytes, cudaStream_t st);


// fdm.cu
int axis_apply(int n2, int n1, int n0, int nrhs, int axis, const z_t* S, const z_t* X, z_t* Y, cudaStream_t st);
size_t fdm_solve_workspace_bytes(int n2, int n1, int n0, int nrhs);
int fdm_solve(int n2, int n1, int n0, int nrhs, const z_t* const V[3], const z_t* const VT[3], const z_t* lx,
              const z_t* ly, const z_t* lz, z_t sigma, const z_t* B, int64_t ldb, z_t* X, int64_t ldx, void* work,
              size_t work_bytes, cudaStream_t st);
int fdm_diag(int n2, int n1, int n0, int nrhs, const z_t* lz, const z_t* ly, const z_t* lx, z_t sigma, z_t* X,
             cudaStream_t st);

}  // namespace vb
