"""Host C++ (partition, schedule, layout, generators) against the oracle, CPU only."""
import os
import tempfile

import numpy as np
import pytest

from conftest import FIXTURE8, random_graph
from layout_emu import emulate

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def both(lr, oracle, n, s, d, keep=False):
    return lr.Graph.from_edges(n, src=s, dst=d, loop_policy=int(keep)), oracle.graph(n, s, d, keep)


def assert_same_partition(a, b):
    assert np.array_equal(a.comp_of, b.comp_of)
    assert np.array_equal(a.kinds, b.kinds)
    assert np.array_equal(a.levels, b.levels)
    assert np.array_equal(a.sizes, b.sizes)
    assert a.max_level == b.max_level
    assert tuple(a.stats) == tuple(b.stats)


def test_graph_from_edges_semantics(lr):
    g = lr.Graph.from_edges(4, [(0, 1), (0, 1), (2, 2), (3, 0), (0, 3)])
    off, tgt, loop, deg = g.csr()
    assert list(off) == [0, 2, 2, 3, 4] and list(tgt) == [1, 3, 2, 0]
    assert list(loop) == [0, 0, 1, 0] and list(deg) == [2, 0, 0, 1]
    gk = lr.Graph.from_edges(4, [(2, 2), (2, 1)], loop_policy=lr.LoopPolicy.Keep)
    assert list(gk.csr()[3]) == [0, 0, 2, 0]
    with pytest.raises(ValueError):
        lr.Graph.from_edges(3, [(0, 3)])
    with pytest.raises(ValueError):
        lr.Graph.from_csr(2, [0, 2, 2], [1, 1])


def test_edge_list_io(lr):
    with tempfile.TemporaryDirectory() as d:
        p = os.path.join(d, "g.tsv")
        with open(p, "w") as f:
            f.write("# comment\n0\t1\r\n1\t0\n\n5\t1\n")
        g = lr.Graph.load_edge_list(p, dense_ids=True)
        assert (g.n, g.m) == (6, 3)
        g2 = lr.Graph.load_edge_list(p, dense_ids=False)
        assert (g2.n, g2.m) == (3, 3)
        with open(p, "w") as f:
            f.write("0 1\n")
        with pytest.raises(OSError):
            lr.Graph.load_edge_list(p)
        with pytest.raises(OSError):
            lr.Graph.load_edge_list(os.path.join(d, "missing.tsv"))


def test_partition_random_corpora(lr, oracle):
    rng = np.random.default_rng(1001)
    for t in range(400):
        n = int(rng.integers(1, 40))
        s, d = random_graph(rng, n, float(rng.uniform(0.0, 0.3)), loops=t % 2 == 0)
        g, go = both(lr, oracle, n, s, d)
        assert_same_partition(lr.find_components(g), go.partition())
        a, b = lr.find_components_scc_only(g), go.partition(merge=False)
        assert np.array_equal(a.comp_of, b.comp_of) and np.array_equal(a.levels, b.levels)


@pytest.mark.parametrize("edges,n,want", [
    ([(0, 1), (1, 2), (2, 3)], 4, [[0, 1, 2, 3]]),                   # chain -> one CAC
    ([(0, 1), (0, 2), (0, 3)], 4, [[0, 1, 2, 3]]),                   # star
    ([(0, 1), (1, 2), (0, 2)], 3, [[0, 1, 2]]),                      # transitive absorption
    ([(0, 1), (1, 2), (2, 3), (3, 2), (0, 4)], 5, [[0, 1], [2, 3], [4]]),  # next-level-only absorption
    ([(0, 1), (0, 2), (2, 3), (3, 2)], 4, [[0], [1], [2, 3]]),      # SCC veto
    ([(0, 0), (1, 1), (0, 1)], 2, [[0, 1]]),                         # self-loops ignored
])
def test_partition_corner_cases(lr, edges, n, want):
    # proj/tests/test_partition.cpp:56-129
    p = lr.find_components(lr.Graph.from_edges(n, edges))
    comps = sorted(sorted(np.nonzero(p.comp_of == c)[0].tolist()) for c in range(p.component_count()))
    assert comps == want


def test_long_chain_iterative(lr):
    # proj/tests/test_partition.cpp:225-238
    n = 200_000
    g = lr.Graph.from_edges(n, src=np.arange(n - 1), dst=np.arange(1, n))
    p = lr.find_components(g)
    assert p.component_count() == 1 and p.kinds[0] == 1 and p.levels[0] == 0 and p.sizes[0] == n
    assert p.stats[0] == n - 1 and p.stats[1] == n - 1


def test_schedule_parity(lr, oracle):
    rng = np.random.default_rng(910)
    for t in range(150):
        n = int(rng.integers(1, 40))
        keep = t % 4 == 0
        s, d = random_graph(rng, n, float(rng.uniform(0.0, 0.25)), loops=True)
        g, go = both(lr, oracle, n, s, d, keep)
        for th in (1, 2, 100):
            a, b = lr.build_schedule(g, th), go.schedule(th)
            for k in ("level_values", "level_unit_begin", "level_cross_begin", "unit_kind", "unit_level",
                      "unit_size", "unit_ids_begin", "unit_edges_begin", "ids", "edge_src", "edge_dst",
                      "cross_src", "cross_dst", "cross_deg", "permutation"):
                assert np.array_equal(getattr(a, k), getattr(b, k)), (t, th, k)
            assert (a.intra, a.cross, a.dropped) == (b.intra, b.cross, b.dropped)
    with pytest.raises(ValueError):
        lr.build_schedule(lr.Graph.from_edges(8, FIXTURE8), 0)


def test_layout_invariants(lr):
    g = lr.config_graph(1, shrink=2)
    L = lr.Plan(g, 100).layout()
    n = L["n"]
    assert np.array_equal(L["row_of"][L["vertex_of"]], np.arange(n))
    assert L["level_row_begin"][0] == 0 and L["level_row_begin"][-1] == n
    assert np.all(np.diff(L["level_row_begin"]) > 0) and np.all(np.diff(L["unit_row_begin"]) > 0)
    # pull sources always come from finished rows: cross from earlier levels, CAC from earlier depth slices
    lvl = np.repeat(np.arange(L["n_levels"]), np.diff(L["level_row_begin"]))
    rows = np.repeat(np.arange(n), np.diff(L["xptr"]))
    assert np.all(lvl[L["xsrc"]] < lvl[rows])
    for u in np.nonzero(L["unit_kind"] == 1)[0]:
        a, b = L["unit_row_begin"][u], L["unit_row_begin"][u + 1]
        dp = L["depth_ptr"][L["cac_depth_begin"][u]:]
        k = int(np.searchsorted(dp, b)) + 1
        depth = np.repeat(np.arange(k - 1), np.diff(dp[:k]))
        for r in range(a, b):
            src = L["isrc"][L["iptr"][r]:L["iptr"][r + 1]]
            assert np.all((src >= a) & (src < b)) and np.all(depth[src - a] < depth[r - a])


def test_layout_emulation_bit_exact(lr, oracle):
    """The device algorithm, executed literally on the host, reproduces the
    oracle bit for bit except through dense SccSmall solves."""
    rng = np.random.default_rng(7)
    for t in range(150):
        n = int(rng.integers(1, 45))
        keep = t % 3 == 0
        s, d = random_graph(rng, n, float(rng.uniform(0.0, 0.2)), loops=t % 2 == 0)
        g, go = both(lr, oracle, n, s, d, keep)
        w = rng.uniform(0.05, 5, n)
        th, c = [1, 2, 100][t % 3], [0.5, 0.85, 0.95][t % 3]
        ref = go.compute_pagerank(w, c, 1e-12, th)
        L = lr.Plan(g, th).layout()
        r3, it = emulate(L, w, c, 1e-12, oracle.iteration_cap(c, 1e-12))
        assert np.array_equal(it, ref.unit_iters)
        if (L["unit_kind"] == 2).any():
            np.testing.assert_allclose(r3, ref.ranks, rtol=1e-12)
        else:
            assert np.array_equal(r3, ref.ranks), t


@pytest.mark.parametrize("cfg,shrink", [(1, 2), (2, 6), (3, 8), (4, 5), (1, 0), (2, 2), (3, 5), (4, 2), (5, 8)])
def test_config_partition_parity(lr, oracle, cfg, shrink):
    g = lr.config_graph(cfg, shrink)
    off, tgt, _, _ = g.csr()
    go = oracle.graph_from_csr(g.n, off, tgt)
    assert_same_partition(lr.find_components(g), go.partition())
    a, b = lr.Plan(g, 100).schedule(), go.schedule(100)
    for k in ("unit_kind", "ids", "permutation", "cross_src", "edge_src", "edge_dst"):
        assert np.array_equal(getattr(a, k), getattr(b, k)), k


def test_partition_medium_random_structures(lr, oracle):
    """Graphs big enough for every stage of the parallel partition: trimming
    rounds, a giant SCC found by forward/backward reachability (above the
    16k-member parallel threshold), small SCCs left to Tarjan, long chains of
    single-vertex components absorbing CACs, kept and ignored self-loops."""
    rng = np.random.default_rng(77)
    for t in range(12):
        n = int(rng.integers(20_000, 60_000))
        m = int(n * rng.uniform(0.8, 3.0))
        src = rng.integers(0, n, m)
        dst = np.where(rng.random(m) < 0.7, np.minimum(src + rng.integers(1, 6, m), n - 1), rng.integers(0, n, m))
        if t % 3 == 0:  # a dense core: one giant SCC
            core = rng.integers(0, n // 2, 4 * n)
            src = np.concatenate([src, core])
            dst = np.concatenate([dst, rng.integers(0, n // 2, 4 * n)])
        if t % 2:
            loops = rng.integers(0, n, n // 50)
            src, dst = np.concatenate([src, loops]), np.concatenate([dst, loops])
        keep = t % 4 == 1
        g = lr.Graph.from_edges(n, src=src.astype(np.int32), dst=dst.astype(np.int32), loop_policy=int(keep))
        off, tgt, _, _ = g.csr()
        go = oracle.graph_from_csr(n, off, tgt, keep)
        assert_same_partition(lr.find_components(g), go.partition())
        a, b = lr.find_components_scc_only(g), go.partition(merge=False)
        assert np.array_equal(a.comp_of, b.comp_of) and np.array_equal(a.levels, b.levels), t


def test_generators_deterministic(lr):
    a, b = lr.rmat(12, 8, seed=3), lr.rmat(12, 8, seed=3)
    assert np.array_equal(a.csr()[1], b.csr()[1])
    assert not np.array_equal(a.csr()[1], lr.rmat(12, 8, seed=4).csr()[1])
    off, tgt, loop, _ = a.csr()
    assert not loop.any()  # R-MAT self-loops removed
    d = lr.dangle(a, 0.3, 2)
    dd = np.diff(d.csr()[0])
    assert 0.2 < np.mean(dd == 0) < 0.6
    z = np.load(os.path.join(GOLDEN, "config_cases.npz"))
    for cfg in (1, 2, 3, 4):
        g = lr.config_graph(cfg, int(z[f"cfg{cfg}_shrink"]))
        tgt = g.csr()[1]
        assert (g.n, g.m) == (int(z[f"cfg{cfg}_n"]), int(z[f"cfg{cfg}_m"]))
        assert int((tgt.astype(np.int64) * 2654435761 % 1000003).sum()) == int(z[f"cfg{cfg}_edge_checksum"])


def test_oracle_on_config_golden(lr, oracle):
    z = np.load(os.path.join(GOLDEN, "config_cases.npz"))
    for cfg in (1, 2, 3, 4):
        g = lr.config_graph(cfg, int(z[f"cfg{cfg}_shrink"]))
        off, tgt, _, _ = g.csr()
        res = oracle.graph_from_csr(g.n, off, tgt).compute_pagerank(np.full(g.n, 1.0 / g.n), 0.85, 1e-12, 100)
        assert np.array_equal(res.unit_iters, z[f"cfg{cfg}_unit_iters"])
        np.testing.assert_allclose(res.ranks, z[f"cfg{cfg}_ranks"], rtol=1e-13)


def test_layout_shared_in_edges_equals_plain_path(lr, monkeypatch):
    """The plan's fast path (the partition's in-edge lists and cross-edge bits
    shared with the layout, giant-SCC shortcuts) against the public two-call
    path (find_components + build_layout: own transpose, every edge's
    components looked up) on graphs with a giant SCC, kept and ignored
    self-loops, trees and chains around it: every layout array equal."""
    rng = np.random.default_rng(2024)
    for t in range(8):
        n = int(rng.integers(30_000, 80_000))
        m = int(n * rng.uniform(1.0, 3.0))
        src = rng.integers(0, n, m)
        dst = np.where(rng.random(m) < 0.6, np.minimum(src + rng.integers(1, 8, m), n - 1), rng.integers(0, n, m))
        if t % 4 != 3:  # a dense core: one giant SCC with edges in and out of it
            k = n // (2 + t % 3)
            src = np.concatenate([src, rng.integers(0, k, 5 * n)])
            dst = np.concatenate([dst, rng.integers(0, k, 5 * n)])
            # a hub, so the partition takes its reachability route for the giant SCC
            hub = rng.integers(0, k, 600)
            src = np.concatenate([src, np.zeros(300, np.int64), hub[300:]])
            dst = np.concatenate([dst, hub[:300], np.zeros(300, np.int64)])
        if t % 2 == 0:
            loops = rng.integers(0, n, n // 20)
            src, dst = np.concatenate([src, loops]), np.concatenate([dst, loops])
        keep = t % 4 in (0, 1)
        g = lr.Graph.from_edges(n, src=src.astype(np.int32), dst=dst.astype(np.int32), loop_policy=int(keep))
        th = [100, 2, 100_000][t % 3]
        monkeypatch.delenv("LR_PLAN_PLAIN", raising=False)
        fast = lr.Plan(g, th).layout()
        monkeypatch.setenv("LR_PLAN_PLAIN", "1")
        plain = lr.Plan(g, th).layout()
        monkeypatch.delenv("LR_PLAN_PLAIN", raising=False)
        assert fast.keys() == plain.keys()
        for k in fast:
            a, b = fast[k], plain[k]
            if isinstance(a, np.ndarray):
                assert np.array_equal(a, b), (t, k)
            else:
                assert a == b, (t, k)
        if t % 4 != 3:
            assert (fast["unit_kind"] == 3).any() or th == 100_000
