"""Build a copy of libvibro_b200.so with extra -D flags into tools/variants/NAME.so
(cross-compiled here, shipped to the GPU box with the repo snapshot):
    python tools/build_variant.py NAME -DVB_KRON_TX=16 -DVB_KRON_KC=4
Load it in a fresh process with VB_LIB_PATH=tools/variants/NAME.so."""
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2310_04734_b200 import build  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
out_dir = ROOT / "tools" / "variants"
tmp = Path("/tmp") / f"vb_variant_{name}"
out_dir.mkdir(exist_ok=True)
tmp.mkdir(exist_ok=True)


def comp(src):
    o = tmp / (src.stem + ".o")
    subprocess.run([build.nvcc()] + [f for f in build.NVCC_FLAGS if f != "-shared"] + defs +
                   ["-c", str(src), "-o", str(o)], check=True)
    return str(o)


with ThreadPoolExecutor(8) as ex:
    objs = list(ex.map(comp, build.sources()))
subprocess.run([build.nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o",
                str(out_dir / f"{name}.so")] + objs, check=True)
print(out_dir / f"{name}.so")
