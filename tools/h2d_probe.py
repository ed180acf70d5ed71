"""Host->device copy bandwidth from pinned memory (the e2e path's H2D), alone and beside a
running training step."""
import sys
import time

import torch

for mb in (1, 10, 40):
    n = mb * (1 << 20)
    h = torch.empty(n, dtype=torch.uint8).pin_memory()
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    s = torch.cuda.Stream()
    for _ in range(3):
        d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        e0.record()
        for _ in range(20):
            d.copy_(h, non_blocking=True)
        e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    print(f"H2D {mb:3d} MB: {ms * 1e3:7.1f} us  {n / ms / 1e6:6.1f} GB/s")
    dh = torch.empty(n, dtype=torch.uint8).pin_memory()
    e0.record()
    for _ in range(20):
        dh.copy_(d, non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    print(f"D2H {mb:3d} MB: {ms * 1e3:7.1f} us  {n / ms / 1e6:6.1f} GB/s")
