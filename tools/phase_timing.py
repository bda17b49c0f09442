"""Per-phase cycle split of the blocked sweep (builds a VB_PHASE_TIMING copy of
the library into /tmp and loads it instead of the production .so)."""
import ctypes as C
import os
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
from paper_2310_04734_b200 import sweep, workloads  # noqa: E402

names = ["form", "leaf panel", "in-panel trsm+gemm", "interchanges", "U12 trsm", "trailing gemm", "back subst", "outputs"]
lib = _lib.load()
nf = int(os.environ.get("NF", "296"))
for r in [int(x) for x in sys.argv[1:]] or [1024]:
    w = workloads.cfg5(r=r)
    rs = sweep.ReducedSweep(w.prims, w.b, w.c_r, kinds=w.kinds)
    f = torch.from_numpy(w.freqs[:nf]).cuda()
    rs.sweep_device(f)
    torch.cuda.synchronize()
    buf = (C.c_uint64 * 36)()
    lib.vb_debug_phase_cycles(buf, 1)
    rs.sweep_device(f)
    torch.cuda.synchronize()
    lib.vb_debug_phase_cycles(buf, 1)
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record()
    rs.sweep_device(f)
    t1.record()
    torch.cuda.synchronize()
    print(f"r={r} F={nf}: {t0.elapsed_time(t1):.2f} ms per launch")
    v = np.array(list(buf), dtype=float)
    print("total Mcycles per CTA-freq", v[:8].sum() / nf / 1e6)
    sub = v[8:16]
    gm = v[16:24]
    sk = v[24:32]
    skn = ["setup", "first tile wait", "tile waits", "compute+epilogue", "release/produce", "final barrier"]
    print(f"r={r}: skinny warp1 " + ", ".join(f"{n} {100 * x / v[:8].sum():.1f}%" for n, x in zip(skn, sk)))
    v = v[:8]
    gn = ["wait full", "compute", "release/produce", "epilogue"]
    print(f"r={r}: gemm warp1 " + ", ".join(f"{n} {100 * x / v.sum():.1f}%" for n, x in zip(gn, gm[:4])))
    print(f"r={r}: gemm thr0  " + ", ".join(f"{n} {100 * x / v.sum():.1f}%" for n, x in zip(gn, gm[4:])))
    subn = ["leaf load", "leaf factor", "leaf swaps", "leaf trsm_small", "col update", "col pivot-recip", "col argmax"]
    print(f"r={r}: sub-phases " + ", ".join(f"{n} {100 * x / v.sum():.1f}%" for n, x in zip(subn, sub)))
    print(f"r={r}: " + ", ".join(f"{n} {100 * x / v.sum():.1f}%" for n, x in zip(names, v)))
