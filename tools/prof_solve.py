"""Profiling driver: build a config graph, then run N device solves (for ncu)."""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1609_09068_b200 as lr  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--shrink", type=int, default=0)
ap.add_argument("--solves", type=int, default=2)
a = ap.parse_args()
g = lr.config_graph(a.config, a.shrink)
eng = lr.Engine(g)
w = np.full(g.n, 1.0 / g.n)
for _ in range(a.solves):
    r3, r1, info, it = eng.solve(w, lr.SolverParams(0.85, 1e-12))
print({k: info[k] for k in ("device_ms", "spmv_active_ms", "spmv_active_launches", "spmv_bytes", "kernel_launches")})
print("spmv GB/s", info["spmv_bytes"] / (info["spmv_active_ms"] / 1e3) / 1e9 if info["spmv_active_ms"] else None)
