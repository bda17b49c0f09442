"""The C-ABI library loads without a GPU and exports exactly what
include/vibro_b200.h declares (CPU-only; no compute calls)."""

import ctypes
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "vibro_b200.h"


def declared():
    txt = HEADER.read_text()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(vb_[a-z0-9_]+)\s*\(", txt)))


def test_library_builds_and_exports_every_declared_symbol():
    from paper_2310_04734_b200 import _lib, build
    build.build_library()
    lib = ctypes.CDLL(str(_lib.LIB_PATH))
    names = declared()
    assert names, "header declares no entry points"
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    # the Python binding covers the whole header, with no stale names
    assert sorted(_lib.exported_symbols()) == names


def test_version_and_error_plumbing_without_gpu():
    from paper_2310_04734_b200 import _lib
    lib = _lib.load()
    assert lib.vb_version().decode().startswith("vibro_b200")
    assert lib.vb_last_error() is not None
    # argument validation fails loudly before touching the device
    rc = lib.vb_rom_sweep(0, 1, 1, 1, 1, None, None, None, 0, None, None, None, None, None, None, 0, None)
    assert rc == 1
    assert "bad sizes" in lib.vb_last_error().decode()


def test_no_cpu_fallback_without_cuda(monkeypatch):
    import torch
    from paper_2310_04734_b200 import _lib
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError):
        _lib.require_cuda()
