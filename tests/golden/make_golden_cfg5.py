"""Generates tests/golden/config5.npz: the reference's own result on the
north-star graph (BASELINE config 5, R-MAT scale 26, edge factor 16), run
through oracle/_ref (the levelrank sources compiled unmodified, -O3 -DNDEBUG).

Run here, where /root/reference exists (about 30 min and 30 GB RSS, one core
for the solve):   python tests/golden/make_golden_cfg5.py

The graph comes from the product generator (lr.config_graph(5)); the fixture
pins the graph by n, m and an edge checksum, so the GPU test regenerates the
same graph on the box.  Stored:
  * the reference partition, per vertex (levels and kinds, bit-exact) as
    SHA-256 digests, plus its PartitionStats;
  * every unit's iteration count in schedule order and the SolveReport counters;
  * R3 at a seeded uniform sample of 2^20 vertices (indices regenerated from
    SAMPLE_SEED) and at the giant SCC's 16384 highest-out-degree rows (the
    columns K4c keeps in shared memory) and 16384 highest-in-degree rows (the
    segmented rows whose sums are combined across CTAs);
  * sum(R3) (R1 = R3 / sum).
"""
import hashlib
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, ROOT)

SAMPLE_SEED = 20261020
SAMPLE = 1 << 20
HEAD = 16384


def edge_checksum(tgt):
    s = 0
    for i in range(0, len(tgt), 1 << 26):
        s += int((tgt[i:i + (1 << 26)].astype(np.int64) * 2654435761 % 1000003).sum())
    return s


def sample_indices(n):
    return np.sort(np.random.default_rng(SAMPLE_SEED).choice(n, SAMPLE, replace=False)).astype(np.int64)


def vertex_digests(comp_of, kinds, levels):
    lv = levels[comp_of].astype(np.int32)
    kd = kinds[comp_of].astype(np.uint8)
    return (hashlib.sha256(comp_of.astype(np.int32).tobytes()).hexdigest(),
            hashlib.sha256(lv.tobytes()).hexdigest(), hashlib.sha256(kd.tobytes()).hexdigest())


def main():
    import paper_1609_09068_b200 as lr
    from oracle_py import Ref

    t = time.time()
    g = lr.config_graph(5)
    off, tgt, _, deg = g.csr()
    n, m = g.n, g.m
    print(f"generated n={n} m={m} in {time.time() - t:.0f}s", flush=True)
    cks = edge_checksum(tgt)
    src = np.repeat(np.arange(n, dtype=np.int32), np.diff(off))
    indeg = np.bincount(tgt, minlength=n)
    del g, off
    ref = Ref()
    t = time.time()
    rg = ref.graph(n, src, tgt)
    del src, tgt
    assert rg.m == m
    print(f"reference graph in {time.time() - t:.0f}s", flush=True)

    t = time.time()
    part = rg.partition(0)
    print(f"reference partition in {time.time() - t:.0f}s: k={len(part.kinds)}", flush=True)
    d_comp, d_lv, d_kd = vertex_digests(part.comp_of, part.kinds, part.levels)
    scc = np.flatnonzero(part.kinds == 0)
    giant = scc[np.argmax(part.sizes[scc])]
    members = np.flatnonzero(part.comp_of == giant)
    head_out = members[np.lexsort((members, -deg[members]))[:HEAD]]
    head_in = members[np.lexsort((members, -indeg[members]))[:HEAD]]
    stats = np.array(part.stats, np.int64)
    max_level = part.max_level
    del part

    w = np.full(n, 1.0 / n)
    t = time.time()
    res = rg.compute_pagerank(w, 0.85, 1e-12, 100)
    print(f"reference compute_pagerank in {time.time() - t:.0f}s: units={len(res.unit_iters)} "
          f"giant iters={res.unit_iters.max()}", flush=True)
    r3 = res.ranks
    total = float(np.add.reduce(r3, dtype=np.float64))  # pairwise; a 1e-15 cross-check of sum(R1) only
    idx = sample_indices(n)
    out = {
        "n": np.int64(n), "m": np.int64(m), "edge_checksum": np.int64(cks),
        "digest_comp_of": np.array(d_comp), "digest_levels": np.array(d_lv), "digest_kinds": np.array(d_kd),
        "partition_stats": stats, "max_level": np.int64(max_level),
        "unit_iters": res.unit_iters.astype(np.int64), "unit_kinds": res.unit_kinds.astype(np.int8),
        "sample_seed": np.int64(SAMPLE_SEED), "sample_r3": r3[idx],
        "head_out": head_out.astype(np.int32), "head_out_r3": r3[head_out],
        "head_in": head_in.astype(np.int32), "head_in_r3": r3[head_in],
        "r3_sum": np.float64(total),
    }
    for k, v in res.report.items():
        out["report_" + k] = np.array(v)
    np.savez_compressed(os.path.join(HERE, "config5.npz"), **out)
    print("wrote config5.npz", {k: (v.shape if hasattr(v, "shape") else v) for k, v in out.items()}, flush=True)


if __name__ == "__main__":
    main()
