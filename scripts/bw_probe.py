"""HBM bandwidth probe (diagnostics): write-only fill vs copy on this B200."""
import torch

def t(fn, n=20):
    for _ in range(3): fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); s.record()
    for _ in range(n): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / n * 1e-3

for mb in (64, 256, 1024):
    n = mb * (1 << 20) // 2
    a = torch.empty(n, dtype=torch.bfloat16, device="cuda"); b = torch.empty_like(a)
    w = t(lambda: a.fill_(float("-inf")))
    c = t(lambda: b.copy_(a))
    print(f"{mb:5d} MB: fill {2*n/w/1e9:7.0f} GB/s ({w*1e6:.1f} us)  copy {4*n/c/1e9:7.0f} GB/s ({c*1e6:.1f} us)")
