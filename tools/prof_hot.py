"""A/B the L2 hot-head fraction of K4b (env LR_L2_HOT_FRAC, read at upload)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1609_09068_b200 as lr  # noqa: E402

cfg = int(sys.argv[1])
fracs = sys.argv[2].split(",")
g = lr.config_graph(cfg, int(sys.argv[3]) if len(sys.argv) > 3 else 0)
w = np.full(g.n, 1.0 / g.n)
for f in fracs:
    os.environ["LR_L2_HOT_FRAC"] = f
    eng = lr.Engine(g)
    best = None
    for _ in range(3):
        _, _, info, _ = eng.solve(w, lr.SolverParams(0.85, 1e-12))
        ms = info["spmv_active_ms"] / max(info["spmv_active_launches"], 1)
        best = ms if best is None else min(best, ms)
    print(f"config {cfg} hot frac {f}: {best:.3f} ms/iter  "
          f"{info['spmv_bytes'] / info['spmv_active_launches'] / best / 1e6:.0f} GB/s", flush=True)
    del eng
