"""One-rank sharded solve (NCCL communicator of size 1, chunked exchange) against the plain solve:
what the row-sharded code path costs on one GPU."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1609_09068_b200 as lr  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
g = lr.config_graph(cfg, 0)
w = np.full(g.n, 1.0 / g.n)
p = lr.SolverParams(0.85, 1e-12)
plain = lr.Engine(g)
for _ in range(2):
    r3a, _, ia, ita = plain.solve(w, p)
print(f"plain: device {ia['device_ms']:.1f} ms, blk units {plain.blk_units()}", flush=True)
del plain
for chunks in (1, 4):
    os.environ["LR_XCHG_CHUNKS"] = str(chunks)
    eng = lr.Engine(g, rank=0, world=1, nccl_id=lr.nccl_unique_id())
    for _ in range(2):
        r3b, _, ib, itb = eng.solve(w, p)
    print(f"sharded, 1 rank, {chunks} chunks: device {ib['device_ms']:.1f} ms, blk units {eng.blk_units()}, "
          f"iterations equal {np.array_equal(ita, itb)}, max rel diff {np.max(np.abs(r3a - r3b) / r3a):.2e}", flush=True)
    del eng
