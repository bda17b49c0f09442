import sys, time, torch
sys.path.insert(0, ".")
from paper_2310_04734_b200 import mor, workloads
def T(): torch.cuda.synchronize(); return time.perf_counter()
fom, lay = workloads.cfg3_model()
V = torch.linalg.qr(torch.randn(fom.n, 400, dtype=torch.complex128, device="cuda"))[0].contiguous()
for t in fom.affine.D:
    P = t.P
    lens = P.indptr[1:] - P.indptr[:-1]
    print("D term rows nonempty", int((lens > 0).sum()), "of", P.n, "nnz", P.nnz, "support", mor._row_support(P) is not None)
for rep in range(2):
    a = T(); rom = mor.ReducedModel(fom=fom, V=V, window=(20.0, 300.0)); rom._projected(); print("projection", round(T() - a, 4))
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    rom = mor.ReducedModel(fom=fom, V=V, window=(20.0, 300.0)); rom._projected(); torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="self_cuda_time_total", row_limit=10))
