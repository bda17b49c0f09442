import torch
def t(fn, reps=5):
    fn(); torch.cuda.synchronize(); best = 1e9
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); b.synchronize(); best = min(best, a.elapsed_time(b))
    return best
for mb in (466, 2000):
    n = mb * 2**20 // 8
    x = torch.empty(n, dtype=torch.float64, device="cuda")
    y = torch.empty_like(x)
    ms = t(lambda: x.fill_(1.0))
    print(f"fill {mb} MB: {ms:.3f} ms {mb*2**20/ms/1e6:.0f} GB/s")
    ms = t(lambda: y.copy_(x))
    print(f"copy {mb} MB: {ms:.3f} ms {2*mb*2**20/ms/1e6:.0f} GB/s (r+w)")
