import sys, time, torch
sys.path.insert(0, ".")
from paper_2310_04734_b200 import mor, workloads
def T(): torch.cuda.synchronize(); return time.perf_counter()
for rep in range(3):
    t0 = T(); fom, lay = workloads.cfg3_model(); t1 = T()
    V = None; tk = 0.0; to = 0.0
    for f0 in lay["points"]:
        a = T(); blocks = list(mor.krylov_blocks_mimo_dev(fom, f0, lay["moments"], second_order=True)); b = T(); tk += b - a
        for Q, _ in blocks:
            V = mor._orthonormalise(V, Q)
        c = T(); to += c - b
    a = T(); rom = mor.ReducedModel(fom=fom, V=V, window=(20.0, 300.0)); P = rom._projected(); b = T(); tp = b - a
    a = T(); res = mor.rom_sweep([rom], list(lay["freqs"])); b = T(); ts = b - a
    print(f"rep {rep}: assembly {t1 - t0:.3f} krylov {tk:.3f} orthonormalise {to:.3f} projection {tp:.3f} "
          f"sweep {ts:.3f} total {b - t0:.3f} r {V.shape[1]}")
    del fom, V, rom, P, res
