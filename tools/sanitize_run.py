"""Small solves that reach every device code path, for compute-sanitizer
(memcheck / racecheck / synccheck, one tool per run): config 1 at 1/8 size
(singletons, CACs, small SCCs, CTA power series), config 2 at 1/64 (the grid
SpMV K4c with segmented heavy rows), config 3 at 1/512 (dangling-heavy CACs),
config 4 at 1/32 (deep level chain, large CACs on the side stream), plus the
whole-graph baseline and a row-sharded one-rank solve with chunked exchange."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1609_09068_b200 as lr  # noqa: E402

for cfg, shrink in ((1, 3), (2, 6), (3, 9), (4, 5)):
    g = lr.config_graph(cfg, shrink)
    w = np.full(g.n, 1.0 / g.n)
    res = lr.compute_pagerank(g, w, lr.SolverParams(0.85, 1e-12))
    print(f"config {cfg} shrink {shrink}: n={g.n} units={len(res.unit_iters)} iters={int(res.unit_iters.max())}",
          flush=True)
g = lr.config_graph(2, 6)
w = np.full(g.n, 1.0 / g.n)
print("baseline iterations", int(lr.compute_baseline(g, w, lr.SolverParams(0.85, 1e-12)).report["total_iterations"]))
if os.environ.get("LR_SANITIZE_SHARDED", "1") == "1":
    os.environ["LR_XCHG_CHUNKS"] = "3"
    eng = lr.Engine(g, rank=0, world=1, nccl_id=lr.nccl_unique_id())
    print("sharded one-rank iterations", int(eng.solve(w, lr.SolverParams(0.85, 1e-12))[3].max()))
print("done")
