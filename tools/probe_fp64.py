"""Probe FP64 / complex128 GEMM throughput and a few device properties on the box."""
import json, os, time, torch
d = torch.device("cuda:0")
p = torch.cuda.get_device_properties(0)
out = {"name": p.name, "sms": p.multi_processor_count, "smem_optin": getattr(p, "shared_memory_per_block_optin", None),
       "l2": getattr(p, "L2_cache_size", None), "cpu_count": os.cpu_count()}
def tgemm(dtype, n, it=10):
    a = torch.randn(n, n, dtype=dtype, device=d); b = torch.randn(n, n, dtype=dtype, device=d)
    for _ in range(3): c = a @ b
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(it): c = a @ b
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / it
    fl = (8 if dtype.is_complex else 2) * n ** 3
    return fl / ms / 1e9
for n in (2048, 4096, 8192):
    out[f"dgemm_{n}_tflops"] = tgemm(torch.float64, n)
    out[f"zgemm_{n}_tflops"] = tgemm(torch.complex128, n)
# batched small LU via torch (cusolver/magma) for comparison
for r in (32, 256, 1024):
    B = {32: 4096, 256: 512, 1024: 32}[r]
    A = torch.randn(B, r, r, dtype=torch.complex128, device=d)
    for _ in range(2): torch.linalg.lu_factor(A)
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(3): torch.linalg.lu_factor(A)
    torch.cuda.synchronize(); dt = (time.perf_counter() - t) / 3
    out[f"torch_lu_factor_r{r}_per_s"] = B / dt
print(json.dumps(out, indent=1))
json.dump(out, open("gpurun_out/probe_fp64.json", "w"), indent=1)
