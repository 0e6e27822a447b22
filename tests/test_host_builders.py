"""Host builders at sizes that cross the bucketed transpose's 2^16-row buckets
(parallel.hpp bucket_csr): Graph::from_edges (proj/src/graph.cpp:14-36
semantics: sorted, deduplicated rows, loop flags) and the whole-graph baseline
layout, checked against numpy restatements."""
import numpy as np
import pytest


@pytest.mark.parametrize("n,m,seed", [(40000, 250000, 1), (140001, 900000, 2), (65536, 300000, 3)])
def test_from_edges_csr_matches_numpy(lr, n, m, seed):
    rng = np.random.default_rng(seed)
    src = rng.integers(0, n, m, dtype=np.int64).astype(np.int32)
    dst = rng.integers(0, n, m, dtype=np.int64).astype(np.int32)
    g = lr.Graph.from_edges(n, src=src, dst=dst)
    off, tgt, loops, _ = g.csr()
    key = np.unique(src.astype(np.int64) * n + dst)  # dedup, sorted by (src, dst)
    s2, d2 = key // n, key % n
    np.testing.assert_array_equal(tgt, d2.astype(np.int32))
    np.testing.assert_array_equal(off, np.concatenate([[0], np.cumsum(np.bincount(s2, minlength=n))]))
    np.testing.assert_array_equal(loops.astype(bool), np.isin(np.arange(n), s2[s2 == d2]))


@pytest.mark.parametrize("keep", [False, True])
def test_baseline_layout_large(lr, keep):
    rng = np.random.default_rng(11 + keep)
    n, m = 150000, 600000
    src = rng.integers(0, n, m).astype(np.int32)
    dst = (src + rng.integers(0, 3000, m)).astype(np.int64) % n  # some locality, some self-loops
    g = lr.Graph.from_edges(n, src=src, dst=dst.astype(np.int32), loop_policy=int(keep))
    off, tgt, _, _ = g.csr()
    L = lr.Plan(g, baseline=True).layout()
    vo, iptr, isrc = L["vertex_of"], L["iptr"], L["isrc"]
    s_all = np.repeat(np.arange(n), np.diff(off))
    sel = keep | (s_all != tgt)
    s_e, d_e = s_all[sel], tgt[sel]
    order = np.lexsort((s_e, d_e))  # by destination, then source ascending
    indeg = np.bincount(d_e, minlength=n)
    np.testing.assert_array_equal(np.diff(iptr), indeg[vo])
    # every row: its in-neighbours (as vertices), source ascending, equal to the numpy in-lists
    got = vo[isrc]
    want_start = np.concatenate([[0], np.cumsum(indeg)])
    want = s_e[order]
    for r in range(n):
        v = vo[r]
        np.testing.assert_array_equal(got[iptr[r]:iptr[r + 1]], want[want_start[v]:want_start[v + 1]])


def test_concurrent_plan_builds_agree(lr):
    """Two host threads building plans at once (the C-ABI releases the GIL):
    one gets the persistent worker pool, the other falls back to its own
    threads; both layouts equal a plan built alone."""
    import threading
    g = lr.config_graph(2, 2)
    want = lr.Plan(g).layout()
    out = [None, None]

    def build(i):
        out[i] = lr.Plan(g).layout()

    ts = [threading.Thread(target=build, args=(i,)) for i in range(2)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for got in out:
        for k in ("vertex_of", "iptr", "isrc", "xptr", "xsrc", "unit_kind", "unit_row_begin"):
            assert np.array_equal(got[k], want[k]), k
