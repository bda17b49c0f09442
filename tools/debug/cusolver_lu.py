import torch
for n in (4641, 10000, 20890):
    A = torch.randn(n, n, dtype=torch.complex128, device="cuda")
    torch.linalg.lu_factor(A); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); torch.linalg.lu_factor(A); b.record(); b.synchronize()
    ms = a.elapsed_time(b)
    print(f"cusolver n={n}: {ms:.1f} ms {8/3*n**3/ms/1e9:.2f} TF/s")
