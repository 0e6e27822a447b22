import os, sys, numpy as np
sys.path.insert(0, '/root/repo')
import paper_1609_09068_b200 as lr
g = lr.config_graph(int(sys.argv[1]))
eng = lr.Engine(g)
w = np.full(g.n, 1.0 / g.n)
for h in sys.argv[2:]:
    os.environ["LR_SPMV_HEAD"] = h
    for _ in range(2):
        r3, r1, info, it = eng.solve(w, lr.SolverParams(0.85, 1e-12))
    print("head", h, {k: round(info[k], 3) for k in ("device_ms", "spmv_active_ms")}, flush=True)
