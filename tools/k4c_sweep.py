"""K4c A/B driver: one graph and plan, then device solves under several
LR_SPMV_HEAD values (read at every launch); prints K4c's algorithmic GB/s
(12 B/edge + 32 B/row per launch over the CUDA-event time of the active
launches).  Run once per library build (LR_LIB selects a variant)."""
import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1609_09068_b200 as lr  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=5)
ap.add_argument("--shrink", type=int, default=0)
ap.add_argument("--heads", default="8192")
ap.add_argument("--solves", type=int, default=3)
ap.add_argument("--hot", default="", help="LR_L2_HOT_FRAC values (re-upload per value)")
ap.add_argument("--keep", default="", help="LR_SPMV_KEEP values (re-upload per value)")
ap.add_argument("--env", action="append", default=[],
                help="VAR=v1,v2,...: per-launch knobs (no re-upload), swept at the first --heads value")
a = ap.parse_args()
t = time.time()
g = lr.config_graph(a.config, a.shrink)
eng = lr.Engine(g)
print(f"lib {lr.library_path()} setup {time.time() - t:.0f}s", flush=True)
w = np.full(g.n, 1.0 / g.n)


def reupload():
    import ctypes as C
    lr._check(lr.lib().lr_ctx_upload(eng._h, C.byref(eng._layout)))


for var, vals in (("LR_L2_HOT_FRAC", a.hot), ("LR_SPMV_KEEP", a.keep)):
    for v in [x for x in vals.split(",") if x]:
        os.environ[var] = v
        reupload()
        rates = []
        for _ in range(a.solves):
            _, _, info, _ = eng.solve(w, lr.SolverParams(0.85, 1e-12))
            rates.append(info["spmv_bytes"] / (info["spmv_active_ms"] / 1e3) / 1e9)
        print(f"{var}={v}: K4c {np.median(rates):.0f} GB/s (runs {', '.join(f'{r:.0f}' for r in rates)})", flush=True)
        del os.environ[var]
    if vals:
        reupload()
for spec in a.env:
    var, vals = spec.split("=", 1)
    os.environ["LR_SPMV_HEAD"] = a.heads.split(",")[0]
    for v in vals.split(","):
        os.environ[var] = v
        rates = []
        for _ in range(a.solves):
            _, _, info, _ = eng.solve(w, lr.SolverParams(0.85, 1e-12))
            rates.append(info["spmv_bytes"] / (info["spmv_active_ms"] / 1e3) / 1e9)
        print(f"{var}={v}: K4c {np.median(rates):.0f} GB/s (runs {', '.join(f'{r:.0f}' for r in rates)}), "
              f"device {info['device_ms']:.1f} ms", flush=True)
    del os.environ[var]
for h in a.heads.split(","):
    os.environ["LR_SPMV_HEAD"] = h
    rates = []
    for _ in range(a.solves):
        _, _, info, _ = eng.solve(w, lr.SolverParams(0.85, 1e-12))
        rates.append(info["spmv_bytes"] / (info["spmv_active_ms"] / 1e3) / 1e9)
    print(f"head {h}: K4c {np.median(rates):.0f} GB/s (runs {', '.join(f'{r:.0f}' for r in rates)}), "
          f"device {info['device_ms']:.1f} ms", flush=True)
