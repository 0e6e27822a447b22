"""A/B the shared-memory head size of K4b on one graph (env LR_SPMV_HEAD is read at upload)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1609_09068_b200 as lr  # noqa: E402

cfg = int(sys.argv[1])
heads = [int(x) for x in sys.argv[2].split(",")]
g = lr.config_graph(cfg, int(sys.argv[3]) if len(sys.argv) > 3 else 0)
plan = None
w = np.full(g.n, 1.0 / g.n)
for h in heads:
    os.environ["LR_SPMV_HEAD"] = str(h)
    eng = lr.Engine(g)
    best = None
    for _ in range(3):
        _, _, info, _ = eng.solve(w, lr.SolverParams(0.85, 1e-12))
        ms = info["spmv_active_ms"] / max(info["spmv_active_launches"], 1)
        best = ms if best is None else min(best, ms)
    print(f"config {cfg} head {h:6d}: {best:.3f} ms/iter  {info['spmv_bytes'] / info['spmv_active_launches'] / best / 1e6:.0f} GB/s",
          flush=True)
    del eng
