import sys, time, torch
sys.path.insert(0, ".")
from paper_2310_04734_b200 import mor, workloads
def T(): torch.cuda.synchronize(); return time.perf_counter()
fom, lay = workloads.cfg3_model()
for rep in range(2):
    a = T()
    for f0 in lay["points"]:
        list(mor.krylov_blocks_mimo_dev(fom, f0, lay["moments"], second_order=True))
    print("rep", rep, "krylov", round(T() - a, 3))
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    for f0 in lay["points"]:
        list(mor.krylov_blocks_mimo_dev(fom, f0, lay["moments"], second_order=True))
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="self_cuda_time_total", row_limit=16))
print(prof.key_averages().table(sort_by="self_cpu_time_total", row_limit=6))
a = T()
for f0 in lay["points"]:
    fom.factor(f0)
print("factor x5", round(T() - a, 3))
a = T()
for f0 in lay["points"]:
    lu = fom.factor(f0); B = fom.load_dev(f0, "cuda"); lu.solve(B)
print("factor+solve x5", round(T() - a, 3))
