import sys, time, torch
sys.path.insert(0, ".")
from paper_2310_04734_b200 import mor, workloads
def T(): torch.cuda.synchronize(); return time.perf_counter()
t0 = T(); fom, lay = workloads.cfg3_model(); t1 = T(); print("model (assembly)", round(t1 - t0, 3))
V = None; tk = 0.0; to = 0.0
for f0 in lay["points"]:
    a = T(); blocks = list(mor.krylov_blocks_mimo_dev(fom, f0, lay["moments"], second_order=True)); b = T(); tk += b - a
    for Q, _ in blocks:
        V = mor._orthonormalise(V, Q)
    c = T(); to += c - b
print("krylov", round(tk, 3), "orthonormalise", round(to, 3), "r", V.shape[1])
a = T(); rom = mor.ReducedModel(fom=fom, V=V, window=(20.0, 300.0)); P = rom._projected(); b = T(); print("projection", round(b - a, 3))
a = T(); res = mor.rom_sweep([rom], list(lay["freqs"])); b = T(); print("sweep", round(b - a, 3))
