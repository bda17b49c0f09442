// Reduced-sweep dispatcher: shared-memory path for small r, blocked batched
// LU (sweep_blocked.cu) otherwise.
#include "sweep.cuh"

namespace vb {

static const size_t kSmallSmemLimit = 200 * 1024;
static int g_override = -1;

void sweep_set_override(int path) { g_override = path; }

int sweep_path(int r, int nprim, int s, int n_out) {
  if (g_override == 0 || g_override == 1) return g_override;
  return sweep_small_smem_bytes(r, nprim, s, n_out) <= kSmallSmemLimit ? 0 : 1;
}

size_t sweep_workspace_bytes(int r, int nprim, int s, int n_out, int64_t F) {
  if (sweep_path(r, nprim, s, n_out) == 0) return 0;
  return sweep_blocked_workspace_bytes(r, s, n_out, F);
}

int sweep_run(int r, int nprim, int s, int n_out, int64_t F, const z_t* prims, const z_t* alpha,
              const z_t* b, int64_t b_stride_f, const z_t* c_r, z_t* y, double* spl, z_t* x,
              int* info, void* work, size_t work_bytes, cudaStream_t stream) {
  if (sweep_path(r, nprim, s, n_out) == 0) {
    if (sweep_small_smem_bytes(r, nprim, s, n_out) > kSmallSmemLimit) {
      set_error("vb_rom_sweep: shared-memory path forced but r*(r+s) does not fit");
      return 3;
    }
    return sweep_small_launch(r, nprim, s, n_out, F, prims, alpha, b, b_stride_f, c_r, y, spl, x,
                              info, stream);
  }
  if (!sweep_blocked_supported(r, s, n_out)) {
    set_error("vb_rom_sweep: shape not supported by the blocked path (s <= 16, r*w panel in smem)");
    return 3;
  }
  return sweep_blocked_launch(r, nprim, s, n_out, F, prims, alpha, b, b_stride_f, c_r, y, spl, x,
                              info, work, work_bytes, stream);
}

}  // namespace vb
