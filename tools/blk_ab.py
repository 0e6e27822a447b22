"""K5 vs K4c A/B on one graph and plan: the same Engine re-uploaded under
several LR_BLK* settings (read at upload; LR_BLK_L1 per launch), a few solves
each; prints the SpMV's algorithmic GB/s (12 B/edge + 32 B/row per active
launch), the device time, and the largest relative R3 difference from K4c
with iteration totals."""
import argparse
import ctypes as C
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1609_09068_b200 as lr  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=5)
ap.add_argument("--shrink", type=int, default=0)
ap.add_argument("--solves", type=int, default=3)
ap.add_argument("--baseline", action="store_true")
ap.add_argument("variants", nargs="*", default=["LR_BLK=0", "LR_BLK=1"],
                help="space-separated VAR=v[,VAR=v] settings, one upload each")
a = ap.parse_args()
t = time.time()
g = lr.config_graph(a.config, a.shrink)
os.environ["LR_BLK"] = "0"
eng = lr.Engine(g, baseline=a.baseline)
print(f"config {a.config} shrink {a.shrink}: n={g.n} m={g.m}, setup {time.time() - t:.0f}s", flush=True)
w = np.full(g.n, 1.0 / g.n)
ref = None
for v in a.variants:
    for k in [k for k in os.environ if k.startswith("LR_BLK")]:
        del os.environ[k]
    for kv in v.split(","):
        k, x = kv.split("=", 1)
        os.environ[k] = x
    t = time.time()
    lr._check(lr.lib().lr_ctx_upload(eng._h, C.byref(eng._layout)))
    up = time.time() - t
    rates, dev = [], []
    for _ in range(a.solves):
        r3, _, info, it = eng.solve(w, lr.SolverParams(0.85, 1e-12))
        rates.append(info["spmv_bytes"] / (info["spmv_active_ms"] / 1e3) / 1e9)
        dev.append(info["device_ms"])
    if ref is None:
        ref = (r3.copy(), info["total_iterations"], it.copy())
        diff = 0.0
    else:
        diff = float(np.max(np.abs(r3 - ref[0]) / ref[0]))
    same_it = info["total_iterations"] == ref[1] and np.array_equal(it, ref[2])
    print(f"{v:40s} blk_units {eng.blk_units()} upload {up:.1f}s  SpMV {np.median(rates):.0f} GB/s "
          f"(runs {', '.join(f'{r:.0f}' for r in rates)})  device {np.median(dev):.1f} ms  "
          f"max rel diff vs first {diff:.2e}  iterations {info['total_iterations']} same {same_it}", flush=True)
