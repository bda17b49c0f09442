"""One cfg3-size structured box assembly (vb_hex27_box_csr) for ncu."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2310_04734_b200 import assembly, workloads

for _ in range(2):
    K, M = assembly.assemble_helmholtz_box(workloads.CFG3_BOX, workloads.CFG3_NE)
torch.cuda.synchronize()
print("ok", K.nnz)
