// Reduced-sweep dispatcher: shared-memory path for small r, blocked batched
// LU (sweep_blocked.cu) otherwise.
#include "sweep.cuh"

namespace vb {

static const size_t kSmallSmemLimit = 200 * 1024;

int sweep_path(int r, int nprim, int s, int n_out) {
  return sweep_small_smem_bytes(r, nprim, s, n_out) <= kSmallSmemLimit ? 0 : 1;
}

size_t sweep_workspace_bytes(int r, int nprim, int s, int n_out, int64_t F) {
  if (sweep_path(r, nprim, s, n_out) == 0) return 0;
  return 0;
}

int sweep_run(int r, int nprim, int s, int n_out, int64_t F, const z_t* prims, const z_t* alpha,
              const z_t* b, int64_t b_stride_f, const z_t* c_r, z_t* y, double* spl, z_t* x,
              int* info, void* work, size_t work_bytes, cudaStream_t stream) {
  if (sweep_path(r, nprim, s, n_out) == 0)
    return sweep_small_launch(r, nprim, s, n_out, F, prims, alpha, b, b_stride_f, c_r, y, spl, x,
                              info, stream);
  set_error("vb_rom_sweep: blocked path not built yet");
  return 3;
}

}  // namespace vb
