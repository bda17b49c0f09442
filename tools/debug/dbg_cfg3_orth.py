import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2310_04734_b200 import workloads, mor, linalg
fom, lay = workloads.cfg3_model()
V = None
info = []
for f0 in lay["points"][:2]:
    blocks = mor.krylov_blocks_mimo_dev(fom, f0, lay["moments"], second_order=True)
    for j, (Q, br) in enumerate(blocks):
        G = Q.conj().T @ Q
        e = torch.abs(G - torch.eye(Q.shape[1], dtype=G.dtype, device=G.device)).max().item()
        info.append((f0, j, Q.shape[1], br, e))
        r0 = 0 if V is None else V.shape[1]
        V = mor._orthonormalise(V, Q)
        G = V.conj().T @ V
        eV = torch.abs(G - torch.eye(V.shape[1], dtype=G.dtype, device=G.device)).max().item()
        print(f0, j, "block cols", Q.shape[1], "breakdown", br, "block orth", e, "V", r0, "->", V.shape[1], "V orth", eV, flush=True)
