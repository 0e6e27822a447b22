"""Generates tests/golden/*.npz from the reference itself (oracle/_ref, the
levelrank sources compiled unmodified).  Run here, where /root/reference
exists:  python tests/golden/make_golden.py
The fixtures pin both the oracle restatement (CPU tests) and the GPU path
(-m gpu tests) on boxes where the reference is not available."""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, ROOT)
from oracle_py import Ref  # noqa: E402


def random_corpus(ref, seed=424242, trials=40):
    rng = np.random.default_rng(seed)
    out = {}
    for t in range(trials):
        n = int(rng.integers(2, 64))
        p = float(rng.uniform(0.02, 0.2))
        A = rng.random((n, n)) < p
        keep = t % 4 == 0
        if t % 2:
            np.fill_diagonal(A, False)
        s, d = (x.astype(np.int32) for x in np.nonzero(A))
        w = rng.uniform(0.05, 5.0, n)
        th = [1, 2, 100][t % 3]
        c = [0.5, 0.85, 0.95][(t // 3) % 3]
        g = ref.graph(n, s, d, keep)
        res = g.compute_pagerank(w, c, 1e-12, th)
        part = g.partition()
        pre = f"g{t}_"
        out.update({pre + "n": np.int64(n), pre + "src": s, pre + "dst": d, pre + "keep": np.int64(keep),
                    pre + "w": w, pre + "c": np.float64(c), pre + "th": np.int64(th), pre + "ranks": res.ranks,
                    pre + "unit_iters": res.unit_iters, pre + "comp_of": part.comp_of, pre + "kinds": part.kinds,
                    pre + "levels": part.levels, pre + "total_edge_work": np.int64(res.report["total_edge_work"])})
    out["trials"] = np.int64(trials)
    return out


def config_cases(ref):
    import paper_1609_09068_b200 as lr
    out = {}
    for cfg, shrink in [(1, 3), (2, 8), (3, 10), (4, 6)]:
        g = lr.config_graph(cfg, shrink)
        off, tgt, _, _ = g.csr()
        src = np.repeat(np.arange(g.n, dtype=np.int32), np.diff(off))
        rg = ref.graph(g.n, src, tgt)
        w = np.full(g.n, 1.0 / g.n)
        res = rg.compute_pagerank(w, 0.85, 1e-12, 100)
        pre = f"cfg{cfg}_"
        out.update({pre + "shrink": np.int64(shrink), pre + "n": np.int64(g.n), pre + "m": np.int64(g.m),
                    pre + "edge_checksum": np.int64((tgt.astype(np.int64) * 2654435761 % 1000003).sum()),
                    pre + "ranks": res.ranks, pre + "unit_iters": res.unit_iters,
                    pre + "total_edge_work": np.int64(res.report["total_edge_work"])})
    return out


if __name__ == "__main__":
    ref = Ref()
    np.savez_compressed(os.path.join(HERE, "random_corpus.npz"), **random_corpus(ref))
    np.savez_compressed(os.path.join(HERE, "config_cases.npz"), **config_cases(ref))
    print("wrote", os.listdir(HERE))
