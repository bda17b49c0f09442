"""In-tree build of libvibro_b200.so with nvcc for sm_100a (no JIT cache: the
.so travels to the GPU box with the repo snapshot)."""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG_DIR = Path(__file__).resolve().parent
CSRC = PKG_DIR / "csrc"
OUT = PKG_DIR / "libvibro_b200.so"
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-O3", "-std=c++17",
              "-Xcompiler", "-fPIC", "-shared", "--expt-relaxed-constexpr"]


def nvcc() -> str:
    cand = [os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"]
    for c in cand:
        if c and (Path(c).exists() or c == "nvcc"):
            return c
    raise RuntimeError("nvcc not found")


def sources() -> list[Path]:
    return sorted(CSRC.glob("*.cu"))


def up_to_date() -> bool:
    if not OUT.exists():
        return False
    t = OUT.stat().st_mtime
    deps = list(CSRC.glob("*.cu")) + list(CSRC.glob("*.cuh")) + [PKG_DIR.parent / "include" / "vibro_b200.h"]
    return all(p.stat().st_mtime <= t for p in deps)


def build_library(force: bool = False, verbose: bool = False) -> Path:
    if not force and up_to_date():
        return OUT
    objs = []
    tmpdir = PKG_DIR / "build_obj"
    tmpdir.mkdir(exist_ok=True)
    procs = []
    for src in sources():
        obj = tmpdir / (src.stem + ".o")
        objs.append(obj)
        if not force and obj.exists() and obj.stat().st_mtime >= max(
                [src.stat().st_mtime] + [h.stat().st_mtime for h in CSRC.glob("*.cuh")]
                + [(PKG_DIR.parent / "include" / "vibro_b200.h").stat().st_mtime]):
            continue
        cmd = [nvcc()] + [f for f in NVCC_FLAGS if f != "-shared"] + os.environ.get("VB_NVCC_EXTRA", "").split() \
            + ["-c", str(src), "-o", str(obj)]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
    failed = []
    for src, p in procs:
        out, _ = p.communicate()
        if verbose or p.returncode:
            sys.stderr.write(out.decode())
        if p.returncode:
            failed.append(src.name)
    if failed:
        raise RuntimeError(f"nvcc failed for {failed}")
    cmd = [nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-Xcompiler", "-fPIC",
           "-o", str(OUT)] + [str(o) for o in objs]
    subprocess.run(cmd, check=True)
    return OUT


if __name__ == "__main__":
    build_library(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(OUT)
