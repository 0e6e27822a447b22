"""Breakdown of the host-buffer solve (lr_solve) against the device solve."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1609_09068_b200 as lr  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
g = lr.config_graph(cfg, 0)
eng = lr.Engine(g, 100, device=0)
n = g.n
p = lr.SolverParams(0.85, 1e-12)
wd = torch.full((n,), 1.0 / n, dtype=torch.float64, device="cuda")
r3d = torch.empty_like(wd)
r1d = torch.empty_like(wd)
wh = torch.full((n,), 1.0 / n, dtype=torch.float64).pin_memory()
r3h = torch.empty(n, dtype=torch.float64).pin_memory()
r1h = torch.empty(n, dtype=torch.float64).pin_memory()


def wall(f, reps=5):
    f()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t = time.perf_counter()
        f()
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t) * 1e3)
    return np.median(ts)


print("device solve (wall)", wall(lambda: eng.solve_ptr(wd.data_ptr(), r3d.data_ptr(), r1d.data_ptr(), False, p)))
print("host solve r3+r1 (wall)", wall(lambda: eng.solve_ptr(wh.data_ptr(), r3h.data_ptr(), r1h.data_ptr(), True, p)))
print("host solve device_ms", eng.solve_ptr(wh.data_ptr(), r3h.data_ptr(), r1h.data_ptr(), True, p)["device_ms"])
print("host solve r3 only (wall)", wall(lambda: eng.solve_ptr(wh.data_ptr(), r3h.data_ptr(), 0, True, p)))
print("H2D w", wall(lambda: wd.copy_(wh, non_blocking=True)))
print("D2H r3", wall(lambda: r3h.copy_(r3d, non_blocking=True)))
info = eng.solve_ptr(wd.data_ptr(), r3d.data_ptr(), r1d.data_ptr(), False, p)
print("info", info)
# pageable host buffers (what a std::vector or numpy caller passes): staged through
# pinned buffers by lr_solve (LR_LIB pointing at an older build shows the plain path)
wp = np.full(n, 1.0 / n)
r3p = np.empty(n)
print("host solve r3 only, pinned (wall)", wall(lambda: eng.solve_ptr(wh.data_ptr(), r3h.data_ptr(), 0, True, p)))
print("host solve r3 only, pageable (wall)", wall(lambda: eng.solve_ptr(wp.ctypes.data, r3p.ctypes.data, 0, True, p)))
