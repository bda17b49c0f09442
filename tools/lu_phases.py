"""Phase split of vb_zgetrf (panel / swaps / TRSM / GEMM, CTA 0's SM cycles) from a
-DVB_PHASE_TIMING build of the library (built into /tmp, loaded instead of the
production .so)."""
import ctypes as C
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2310_04734_b200 import _lib, build  # noqa: E402

out = Path("/tmp/libvibro_b200_phase.so")
objs = []
for src in build.sources():
    o = Path("/tmp") / (src.stem + "_ph.o")
    subprocess.run([build.nvcc()] + [f for f in build.NVCC_FLAGS if f != "-shared"] +
                   ["-DVB_PHASE_TIMING", "-c", str(src), "-o", str(o)], check=True)
    objs.append(str(o))
subprocess.run([build.nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", str(out)] + objs,
               check=True)
_lib.LIB_PATH = out
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_2310_04734_b200 import solvers  # noqa: E402

lib = _lib.load()
for n in [int(x) for x in sys.argv[1:]] or [4641, 20890]:
    A = torch.randn(n, n, dtype=torch.complex128, device="cuda")
    A.diagonal().add_(n ** 0.5)
    solvers.DenseLU(A, copy=True)
    torch.cuda.synchronize()
    buf = (C.c_uint64 * 36)()
    lib.vb_debug_phase_cycles(buf, 1)
    solvers.DenseLU(A, copy=True)
    torch.cuda.synchronize()
    lib.vb_debug_phase_cycles(buf, 1)
    v = np.array(list(buf)[32:36], dtype=float)
    print(f"n={n}: total {v.sum() / 1.9e6:.1f} ms @1.9GHz; " +
          ", ".join(f"{k} {100 * x / v.sum():.1f}%" for k, x in zip(["panel", "swaps", "trsm", "gemm"], v)))
