"""Pinned host<->device copy throughput on the box (the e2e path's floor)."""
import time
import torch

for mb in (8, 67, 134):
    n = mb * 1024 * 1024 // 8
    h = torch.empty(n, dtype=torch.float64).pin_memory()
    d = torch.empty(n, dtype=torch.float64, device="cuda")
    for name, f in (("H2D", lambda: d.copy_(h, non_blocking=True)), ("D2H", lambda: h.copy_(d, non_blocking=True))):
        f(); torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(5):
            f()
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t) / 5
        print(f"{name} {mb} MB: {dt * 1e3:.2f} ms  {n * 8 / dt / 1e9:.1f} GB/s", flush=True)
