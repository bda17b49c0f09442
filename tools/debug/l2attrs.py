import ctypes, torch
torch.cuda.init()
lib = ctypes.CDLL("libcudart.so.12") if False else None
try:
    from cuda.bindings import runtime as rt
except Exception:
    from cuda import cudart as rt
for name in ("cudaDevAttrMaxPersistingL2CacheSize", "cudaDevAttrMaxAccessPolicyWindowSize", "cudaDevAttrL2CacheSize"):
    attr = getattr(rt.cudaDeviceAttr, name)
    err, v = rt.cudaDeviceGetAttribute(attr, 0)
    print(name, v / 2**20, "MiB")
