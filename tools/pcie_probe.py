"""Raw pinned H2D / D2H bandwidth on this box (the e2e ceiling)."""
import time

import torch

n = 2304 * 1000 * 1000
d = torch.empty(n, dtype=torch.uint8, device="cuda")
h = torch.empty(n, dtype=torch.uint8).pin_memory()
for name, src, dst in (("D2H", d, h), ("H2D", h, d)):
    dst.copy_(src, non_blocking=True)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(3):
        dst.copy_(src, non_blocking=True)
    torch.cuda.synchronize()
    print(name, round(3 * n / (time.perf_counter() - t) / 1e9, 1), "GB/s")
