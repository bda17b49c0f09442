// Internal interface of the reduced-sweep kernels (dispatch in sweep.cu).
#pragma once
#include "common.cuh"

namespace vb {

size_t sweep_small_smem_bytes(int r, int nprim, int s, int n_out);
int sweep_small_launch(int r, int nprim, int s, int n_out, int64_t F, const z_t* prims,
                       const z_t* alpha, const z_t* b, int64_t b_stride_f, const z_t* c_r, z_t* y,
                       double* spl, z_t* x, int* info, cudaStream_t stream);

int sweep_path(int r, int nprim, int s, int n_out);
void sweep_set_override(int path);
size_t sweep_workspace_bytes(int r, int nprim, int s, int n_out, int64_t F);
int sweep_run(int r, int nprim, int s, int n_out, int64_t F, const z_t* prims, const z_t* alpha,
              const z_t* b, int64_t b_stride_f, const z_t* c_r, z_t* y, double* spl, z_t* x,
              int* info, void* work, size_t work_bytes, cudaStream_t stream);
void count_launches(int64_t n);
int probe_fp64_peak(double* tflops, cudaStream_t stream);

size_t sweep_blocked_workspace_bytes(int r, int s, int n_out, int64_t F);
int sweep_blocked_supported(int r, int s, int n_out);
int sweep_blocked_launch(int r, int nprim, int s, int n_out, int64_t F, const z_t* prims,
                         const z_t* alpha, const z_t* b, int64_t b_stride_f, const z_t* c_r, z_t* y,
                         double* spl, z_t* x, int* info, void* work, size_t work_bytes,
                         cudaStream_t stream);

}  // namespace vb
