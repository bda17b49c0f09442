import sys, time, torch
sys.path.insert(0, ".")
from paper_2310_04734_b200 import mor, workloads
def T(): torch.cuda.synchronize(); return time.perf_counter()
fom, lay = workloads.cfg3_model()
allq = []
for f0 in lay["points"]:
    allq += [Q for Q, _ in mor.krylov_blocks_mimo_dev(fom, f0, lay["moments"], second_order=True)]
for rep in range(3):
    V = None; ts = []
    for Q in allq:
        a = T(); V = mor._orthonormalise(V, Q); ts.append(T() - a)
    print("rep", rep, "total", round(sum(ts), 3), "r", V.shape[1], " ".join(f"{t*1e3:.1f}" for t in ts))
from torch.profiler import profile, ProfilerActivity
V = None
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    for Q in allq:
        V = mor._orthonormalise(V, Q)
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="self_cuda_time_total", row_limit=14))
print(prof.key_averages().table(sort_by="self_cpu_time_total", row_limit=8))
