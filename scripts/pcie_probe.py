"""PCIe D2H probe (diagnostics): back-to-back device->pinned copies of the
config-2 bitmask size (4.1 MB) and larger, one and two streams."""
import torch

for mb in (1, 4.1, 16, 64):
    n = int(mb * (1 << 20))
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    h = [torch.empty(n, dtype=torch.uint8, pin_memory=True) for _ in range(2)]
    s = torch.cuda.Stream()
    for _ in range(3):
        h[0].copy_(d, non_blocking=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        e0.record(s)
        for i in range(40):
            h[i & 1].copy_(d, non_blocking=True)
        e1.record(s)
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 40 * 1e-3
    print(f"D2H {mb:5.1f} MB: {n / t / 1e9:6.1f} GB/s ({t * 1e6:.0f} us per copy)")
