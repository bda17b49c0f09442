import sys, time, torch
sys.path.insert(0, ".")
from paper_2310_04734_b200 import mor
n = 376431
g = torch.Generator(device="cuda").manual_seed(0)
V = torch.linalg.qr(torch.randn(n, 300, dtype=torch.complex128, device="cuda", generator=g))[0].contiguous()
B = torch.randn(n, 10, dtype=torch.complex128, device="cuda", generator=g)
for _ in range(2):
    mor._orthonormalise(V, B)
torch.cuda.synchronize()
t = time.perf_counter(); W = mor._orthonormalise(V, B); torch.cuda.synchronize(); print("one call", time.perf_counter() - t)
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    mor._orthonormalise(V, B); torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="self_cuda_time_total", row_limit=14))
from paper_2310_04734_b200 import linalg
def tm(fn, it=10):
    fn(); torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(it): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / it
for nc in (10, 16, 32):
    X = torch.randn(n, nc, dtype=torch.complex128, device="cuda", generator=g)
    G = linalg.zgemm("C", V, X)
    tc = tm(lambda: linalg.zgemm("C", V, X)); tn = tm(lambda: linalg.zgemm("N", V, G, -1.0, 1.0, X))
    gb = V.numel() * 16 / 1e9
    print(f"nc={nc}: CN {tc:.3f} ms ({gb/tc:.0f} TB/s eq)  NN {tn:.3f} ms ({gb/tn:.0f} TB/s eq)")
    ref = V.conj().T @ X
    print("  CN err", float((linalg.zgemm("C", V, X) - ref).abs().max() / ref.abs().max()))
    Y = X.clone(); linalg.zgemm("N", V, G, -1.0, 1.0, Y)
    print("  NN err", float((Y - (X - V @ G)).abs().max() / X.abs().max()))
