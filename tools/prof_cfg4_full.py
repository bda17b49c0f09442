"""cfg4 at the full BASELINE resolution (n = 2,408,303): generator + GPU
element kernels + CSR assembly, for ncu captures of the assembly kernels."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2310_04734_b200 import fuselage as fz

fom, info = fz.fuselage_model(fz.cfg4_spec_full(), solver=False)
torch.cuda.synchronize()
print("n", fom.n, "nnz", sum(t.P.nnz for t in fom.affine.K + fom.affine.M))
