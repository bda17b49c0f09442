"""Run-to-run determinism of the offline path on the reference benchmark
(tests/golden/fuselage_slice.npz through the drop-in): FOM solve, Krylov
block, orthonormalisation, and one greedy iteration, each twice."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np
import torch

from paper_2310_04734_b200 import mor
from paper_2310_04734_b200.model_operator import load_operator_npz


def main():
    root = Path(__file__).resolve().parents[1]
    fom, grid, _ = load_operator_npz(root / "tests" / "golden" / "fuselage_slice.npz")
    f = grid[100]
    x1 = fom.solve(f)
    x2 = fom.solve(f)
    print("FOM solve identical:", np.array_equal(x1, x2), float(np.abs(x1 - x2).max()))
    lu = fom.factor(f)
    b = fom.load_dev(f)
    y1, y2 = lu.solve(b), lu.solve(b)
    print("LU solve identical (same factor):", torch.equal(y1, y2))
    lu2 = fom.factor(f)
    print("two factorisations identical:", torch.equal(lu.lu.A, lu2.lu.A) if hasattr(lu, "lu") else "n/a")
    Q1, _ = mor.krylov_block_dev(fom, f, 4)
    Q2, _ = mor.krylov_block_dev(fom, f, 4)
    print("krylov block identical:", torch.equal(Q1, Q2), float((Q1 - Q2).abs().max()))
    V1 = mor._orthonormalise(None, Q1)
    V2 = mor._orthonormalise(None, Q1.clone())
    print("orthonormalise identical:", torch.equal(V1, V2))
    rom = mor.ReducedModel(fom=fom, V=V1, window=(grid[0], grid[-1]))
    o1 = rom.outputs(grid[::4])
    o2 = rom.outputs(grid[::4])
    print("rom outputs identical:", np.array_equal(np.array(o1), np.array(o2)))


if __name__ == "__main__":
    main()
