"""ctypes binding of libvibro_b200.so (the C ABI declared in include/vibro_b200.h).

The library is built in-tree by `paper_2310_04734_b200.build.build_library()`
(nvcc, sm_100a).  There is no CPU fallback: if the library is missing or a
call fails, a RuntimeError is raised (the reference CLI maps RuntimeError to
exit code 3, vibrofem/cli.py:465-474).
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import torch

PKG_DIR = Path(__file__).resolve().parent
# VB_LIB_PATH: an alternative build of the same library (tools/build_variant.py
# experiments); the product path is the in-tree build
LIB_PATH = Path(os.environ["VB_LIB_PATH"]).resolve() if os.environ.get("VB_LIB_PATH") else PKG_DIR / "libvibro_b200.so"

_z = C.c_void_p  # vb_complex* (device)


class VbComplex(C.Structure):
    _fields_ = [("re", C.c_double), ("im", C.c_double)]


class VbGemvItem(C.Structure):
    _fields_ = [("m", C.c_int32), ("n", C.c_int32), ("s", C.c_int32), ("pad", C.c_int32),
                ("A", C.c_void_p), ("lda", C.c_int64), ("X", C.c_void_p), ("ldx", C.c_int64),
                ("Y", C.c_void_p), ("ldy", C.c_int64), ("alpha", VbComplex), ("beta", VbComplex)]


def zc(v) -> VbComplex:
    v = complex(v)
    return VbComplex(v.real, v.imag)
_SIGS = {
    "vb_version": (C.c_char_p, []),
    "vb_last_error": (C.c_char_p, []),
    "vb_launch_count": (C.c_int64, []),
    "vb_release_l2_persistence": (C.c_int, []),
    "vb_set_l2_persistence": (None, [C.c_int]),
    "vb_debug_phase_cycles": (C.c_int, [C.POINTER(C.c_uint64), C.c_int]),
    "vb_rom_sweep_path": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int]),
    "vb_set_sweep_path_override": (None, [C.c_int]),
    "vb_set_rg_spmm_mode": (None, [C.c_int]),
    "vb_probe_fp64_peak": (C.c_int, [C.POINTER(C.c_double), C.c_void_p]),
    "vb_rom_sweep_workspace_bytes": (C.c_size_t, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int64]),
    "vb_csr_pattern_workspace_bytes": (C.c_size_t, [C.c_int, C.c_int, C.c_int]),
    "vb_csr_pattern_from_elements": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p,
                                               C.c_void_p, C.c_void_p, C.c_void_p,
                                               C.POINTER(C.c_int64), C.c_void_p, C.c_size_t,
                                               C.c_void_p]),
    "vb_csr_pattern_blocks_workspace_bytes": (C.c_size_t, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int]),
    "vb_csr_pattern_from_blocks": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p,
                                             C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                             C.POINTER(C.c_int64), C.c_void_p, C.c_size_t, C.c_void_p]),
    "vb_rm_plate_elements": (C.c_int, [C.c_int, C.c_void_p, C.c_void_p, C.c_double, C.c_double, C.c_double,
                                       C.c_double, C.c_void_p, C.c_void_p, C.POINTER(C.c_int32), C.c_void_p]),
    "vb_csr_gather": (C.c_int, [C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "vb_csr_gather2": (C.c_int, [C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                 C.c_void_p, C.c_void_p]),
    "vb_hex27_helmholtz_elements": (C.c_int, [C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                              C.POINTER(C.c_int32), C.c_void_p]),
    "vb_hex27_box_nnz": (C.c_int64, [C.c_int, C.c_int, C.c_int]),
    "vb_hex27_box_csr": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p,
                                   C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "vb_quad9_face_mass": (C.c_int, [C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "vb_zgemv_batched": (C.c_int, [C.c_int, C.c_void_p, C.c_void_p]),
    "vb_hex27_helmholtz_elements_chain": (C.c_int, [C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                                    C.POINTER(C.c_int32), C.c_void_p]),
    "vb_facet_shell_elements": (C.c_int, [C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int,
                                          C.c_double, C.c_void_p, C.c_void_p, C.POINTER(C.c_int32), C.c_void_p]),
    "vb_csr_spmm": (C.c_int, [C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, _z, C.c_int64, _z,
                              C.c_int64, VbComplex, VbComplex, C.c_void_p]),
    "vb_csr_row_groups": (C.c_int, [C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                    C.c_void_p, C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_int64)]),
    "vb_rg_gather_values": (C.c_int, [C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "vb_rg_spmm": (C.c_int, [C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                             C.c_void_p, C.c_int, _z, C.c_int64, _z, C.c_int64, VbComplex, VbComplex,
                             C.c_void_p]),
    "vb_block_gs_workspace_bytes": (C.c_size_t, []),
    "vb_block_gs": (C.c_int, [C.c_int, C.c_int, _z, C.c_int64, C.c_void_p, C.c_double, C.c_double, C.c_int, _z,
                              C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p]),
    "vb_kron3_apply": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int,
                                 VbComplex, _z, C.c_int64, VbComplex, _z, C.c_int64, C.c_void_p]),
    "vb_csr_axpy_dense": (C.c_int, [C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, VbComplex, _z, C.c_int64,
                                    C.c_void_p]),
    "vb_zgemm_workspace_bytes": (C.c_size_t, [C.c_char, C.c_int, C.c_int, C.c_int]),
    "vb_zgemm": (C.c_int, [C.c_char, C.c_int, C.c_int, C.c_int, VbComplex, _z, C.c_int64, _z, C.c_int64,
                           VbComplex, _z, C.c_int64, C.c_void_p, C.c_size_t, C.c_void_p]),
    "vb_column_norms_workspace_bytes": (C.c_size_t, [C.c_int, C.c_int]),
    "vb_column_norms": (C.c_int, [C.c_int, C.c_int, _z, C.c_int64, C.c_void_p, C.c_void_p, C.c_size_t,
                                  C.c_void_p]),
    "vb_batched_dots_workspace_bytes": (C.c_size_t, [C.c_int, C.c_int]),
    "vb_batched_dots": (C.c_int, [C.c_int64, C.c_int, C.c_int, _z, C.c_int64, C.c_int64, _z, C.c_int64, _z,
                                  C.c_void_p, C.c_size_t, C.c_void_p]),
    "vb_batched_update": (C.c_int, [C.c_int64, C.c_int, C.c_int, _z, C.c_int64, C.c_int64, _z, _z, C.c_int64,
                                    C.c_void_p]),
    "vb_scale_columns": (C.c_int, [C.c_int, C.c_int, _z, C.c_int64, C.c_void_p, C.c_void_p]),
    "vb_zgetrf_workspace_bytes": (C.c_size_t, [C.c_int]),
    "vb_zgetrf_aux_bytes": (C.c_size_t, [C.c_int]),
    "vb_zgetrf": (C.c_int, [C.c_int, _z, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t,
                            C.c_void_p, C.c_size_t, C.c_void_p]),
    "vb_set_lu_max_ctas": (None, [C.c_int]),
    "vb_set_lu_lookahead": (None, [C.c_int]),
    "vb_zgetrs_workspace_bytes": (C.c_size_t, [C.c_int, C.c_int]),
    "vb_zgetrs": (C.c_int, [C.c_int, C.c_int, _z, C.c_int64, C.c_void_p, _z, C.c_int64, _z, C.c_int64,
                            C.c_void_p, C.c_size_t, C.c_void_p]),
    "vb_axis_apply": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _z, _z, _z, C.c_void_p]),
    "vb_fdm_diag": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, _z, _z, _z, VbComplex, _z, C.c_void_p]),
    "vb_fdm_solve_workspace_bytes": (C.c_size_t, [C.c_int, C.c_int, C.c_int, C.c_int]),
    "vb_fdm_solve": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, _z, _z, _z, _z, _z, _z, _z, _z, _z, VbComplex,
                               _z, C.c_int64, _z, C.c_int64, C.c_void_p, C.c_size_t, C.c_void_p]),
    "vb_rom_sweep": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int64, _z, _z, _z, C.c_int64,
                               _z, _z, C.c_void_p, _z, C.c_void_p, C.c_void_p, C.c_size_t,
                               C.c_void_p]),
}

_lib = None


def exported_symbols() -> list[str]:
    return list(_SIGS)


def load():
    """Load (once) and return the ctypes handle; raises if the build is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise RuntimeError(f"vibro_b200 native library not built: {LIB_PATH} missing "
                           "(run __graft_entry__.build()); there is no CPU fallback")
    lib = C.CDLL(str(LIB_PATH))
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(rc: int, what: str):
    if rc != 0:
        msg = load().vb_last_error().decode()
        raise RuntimeError(f"{what} failed (rc={rc}): {msg}")


def ptr(t) -> C.c_void_p | None:
    """Device pointer of a CUDA tensor (None for None)."""
    if t is None:
        return None
    if not t.is_cuda:
        raise RuntimeError("vibro_b200: expected a CUDA tensor")
    if not t.is_contiguous():
        raise RuntimeError("vibro_b200: expected a contiguous tensor")
    return C.c_void_p(t.data_ptr())


def stream_handle(stream=None) -> C.c_void_p:
    """cudaStream_t of `stream` (default: torch's current stream on the current
    device, read without building a torch.cuda.Stream object: ~1 us instead of
    ~14 us per call on the many-small-launch offline paths)."""
    if stream is not None:
        return C.c_void_p(stream.cuda_stream)
    return C.c_void_p(torch._C._cuda_getCurrentRawStream(torch._C._cuda_getDevice()))


def launch_count() -> int:
    return int(load().vb_launch_count())


def require_cuda():
    if not torch.cuda.is_available():
        raise RuntimeError("vibro_b200 needs a CUDA device (B200, sm_100a); no CPU fallback")
    if os.environ.get("VB_ALLOW_NON_SM100") != "1":
        major, minor = torch.cuda.get_device_capability()
        if (major, minor) != (10, 0):
            raise RuntimeError(f"vibro_b200 is built for sm_100a; found sm_{major}{minor}")


def probe_fp64_peak() -> float:
    v = C.c_double(0.0)
    check(load().vb_probe_fp64_peak(C.byref(v), stream_handle()), "vb_probe_fp64_peak")
    return float(v.value)
