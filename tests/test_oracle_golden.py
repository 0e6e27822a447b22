"""The CPU oracle (oracle/lr_oracle.c) pinned against the reference's own
known-answer tests (proj/tests/*.cpp), against the reference
compiled from its own sources (oracle/_ref) and against golden fixtures the
reference produced (tests/golden/make_golden.py)."""
import os

import numpy as np
import pytest

from conftest import FIXTURE8, random_graph

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def g_from(oracle, n, edges, keep=False):
    e = np.asarray(edges, np.int32).reshape(-1, 2)
    return oracle.graph(n, e[:, 0], e[:, 1], keep)


def test_fixture8_ranks_and_report(oracle):
    # proj/tests/test_engine.cpp:23-75
    g = g_from(oracle, 8, FIXTURE8)
    res = g.compute_pagerank(np.ones(8), 0.85, 1e-9, 100)
    want = [1.0, 2.99670691547750, 1.425, 1.84906695938529, 1.605625, 3.81947320938530, 9.72636742121042,
            9.26741230802886]
    np.testing.assert_allclose(res.ranks, want, rtol=1e-10)
    assert res.ranks[0] == 1.0 and abs(res.ranks[2] - 1.425) < 1e-12 and abs(res.ranks[4] - 1.605625) < 1e-12
    r = res.report
    assert (r["vertices"], r["edges"], r["components"], r["scc_components"], r["cac_components"],
            r["singleton_cacs"], r["largest_component"], r["largest_is_scc"], r["max_level"],
            r["level_count"]) == (8, 11, 4, 2, 2, 1, 3, 0, 2, 3)
    assert (r["large_scc_vertices"], r["eps_tot"], r["total_iterations"], r["iterative_edge_work"],
            r["single_pass_edge_work"], r["cross_edge_count"], r["total_edge_work"]) == (0, 0.0, 0, 0, 11, 4, 11)
    assert list(res.unit_kinds) == [0, 2, 1, 2]


def test_fixture8_partition(oracle):
    # proj/tests/test_partition.cpp:24-54,131-138
    g = g_from(oracle, 8, FIXTURE8)
    p = g.partition()
    assert list(p.comp_of) == [0, 1, 2, 1, 2, 2, 3, 3]
    assert list(p.kinds) == [1, 0, 1, 0]
    assert list(p.levels) == [2, 1, 0, 0]
    assert list(p.sizes) == [1, 2, 3, 2]
    assert p.max_level == 2
    assert tuple(int(x) for x in p.stats) == (11, 4, 8)
    plain = g.partition(merge=False)
    assert plain.max_level == 3
    assert [int(plain.levels[plain.comp_of[v]]) for v in range(8)] == [3, 1, 2, 1, 1, 0, 0, 0]


def test_fixture8_schedule(oracle):
    # proj/tests/test_schedule.cpp:27-72
    s = g_from(oracle, 8, FIXTURE8).schedule(100)
    assert list(s.level_values) == [2, 1, 0]
    assert list(s.unit_kind) == [0, 2, 1, 2]
    assert list(s.ids) == [0, 1, 3, 2, 4, 5, 6, 7]
    assert list(zip(s.edge_src[s.unit_edges_begin[1]:s.unit_edges_begin[2]],
                    s.edge_dst[s.unit_edges_begin[1]:s.unit_edges_begin[2]])) == [(0, 1), (1, 0)]
    assert list(zip(s.edge_src[s.unit_edges_begin[2]:s.unit_edges_begin[3]],
                    s.edge_dst[s.unit_edges_begin[2]:s.unit_edges_begin[3]])) == [(0, 1), (0, 2), (1, 2)]
    assert list(zip(s.cross_src, s.cross_dst, s.cross_deg)) == [(0, 1, 2), (0, 2, 2), (1, 5, 3), (1, 6, 3)]
    assert list(s.level_cross_begin) == [0, 2, 4, 4]
    assert list(s.permutation) == [0, 1, 3, 2, 4, 5, 6, 7]
    assert (s.intra, s.cross, s.dropped) == (7, 4, 0)
    # small_threshold splits SCCs by size (test_schedule.cpp:74-79)
    g = g_from(oracle, 8, FIXTURE8)
    assert g.schedule(3).unit_kind[1] == 2 and g.schedule(2).unit_kind[1] == 3 and g.schedule(1).unit_kind[1] == 3
    with pytest.raises(ValueError):
        g.schedule(0)


def test_iteration_counts(oracle):
    # proj/tests/test_solvers.cpp:176-205, acceptance.cpp:195-218
    two = g_from(oracle, 2, [(0, 1), (1, 0)])
    res = two.compute_pagerank(np.ones(2), 0.85, 1e-9, 1)
    assert list(res.unit_iters) == [128]
    np.testing.assert_allclose(res.ranks, [1 / 0.15] * 2, rtol=1e-8)
    res = two.compute_pagerank(np.array([0.5, 0.5]), 0.85, 1.0, 1)
    assert list(res.unit_iters) == [1]
    np.testing.assert_allclose(res.ranks, [0.925, 0.925], rtol=1e-15)
    leaky = g_from(oracle, 3, [(0, 1), (1, 0), (0, 2), (1, 2)])
    res = leaky.compute_pagerank(np.ones(3), 0.85, 1e-9, 1)
    assert res.unit_iters[res.unit_kinds == 3][0] == 25
    cyc = [(v, (v + 1) % 64) for v in range(64)]
    r64 = g_from(oracle, 64, cyc).compute_pagerank(np.ones(64), 0.85, 1e-9, 1)
    assert r64.unit_iters[0] == 128
    lk = g_from(oracle, 65, cyc + [(v, 64) for v in range(64)]).compute_pagerank(np.ones(65), 0.85, 1e-9, 1)
    assert lk.unit_iters[lk.unit_kinds == 3][0] < 128


def test_cap_and_bound(oracle):
    # proj/tests/test_solvers.cpp:52-56, test_engine.cpp:181-189
    assert oracle.iteration_cap(0.85, 1e-9) == 1280
    assert oracle.iteration_cap(0.85, 0.9) == 16
    assert oracle.iteration_cap(0.5, 1e-9) == 300
    assert oracle.iteration_cap(0.85, 1e-12) == 1710
    assert oracle.error_bound(0, 100, 0.85, 1e-9) == (0.0, 0.0)
    tot, avg = oracle.error_bound(1000, 10000, 0.85, 1e-9)
    assert abs(tot - 1000 * 1e-9 * 0.85 / 0.15) <= 1e-12 * tot and abs(avg - tot / 1e4) <= 1e-12 * avg


def test_cac_closed_forms(oracle):
    # proj/tests/test_solvers.cpp:88-121 (whole graph is one CAC)
    r = g_from(oracle, 2, [(0, 1)]).compute_pagerank(np.ones(2), 0.85, 1e-9).ranks
    assert r[0] == 1.0 and abs(r[1] - 1.85) < 1e-15
    r = g_from(oracle, 3, [(0, 1), (1, 2)]).compute_pagerank(np.ones(3), 0.85, 1e-9).ranks
    np.testing.assert_allclose(r, [1, 1.85, 2.5725], rtol=1e-15)
    r = g_from(oracle, 4, [(0, 1), (0, 2), (1, 3), (2, 3)]).compute_pagerank(np.ones(4), 0.85, 1e-9).ranks
    assert abs(r[1] - 1.425) < 1e-15 and abs(r[3] - 3.4225) < 1e-15


def test_keep_loops_singletons(oracle):
    # proj/tests/test_solvers.cpp:58-86
    r = g_from(oracle, 1, [(0, 0)], keep=True).compute_pagerank(np.ones(1), 0.85, 1e-9).ranks
    assert abs(r[0] - 1 / 0.15) < 1e-12
    r = g_from(oracle, 2, [(0, 0), (0, 1)], keep=True).compute_pagerank(np.ones(2), 0.85, 1e-9).ranks
    assert abs(r[0] - 40 / 23) < 1e-12
    r = g_from(oracle, 1, [(0, 0)], keep=False).compute_pagerank(np.ones(1), 0.85, 1e-9).ranks
    assert r[0] == 1.0


def test_degenerate_inputs(oracle):
    # proj/tests/test_engine.cpp:191-223
    empty = oracle.graph(0, [], [])
    assert len(empty.compute_pagerank(np.zeros(0), 0.85, 1e-9).ranks) == 0
    g = g_from(oracle, 8, FIXTURE8)
    z = g.compute_pagerank(np.zeros(8), 0.85, 1e-9)
    assert z.report["all_weights_zero"] == 1 and not z.ranks.any()
    with pytest.raises(ValueError):
        g.compute_pagerank(np.ones(7), 0.85, 1e-9)
    w = np.ones(8)
    w[3] = -0.25
    with pytest.raises(ValueError):
        g.compute_pagerank(w, 0.85, 1e-9)
    with pytest.raises(ValueError):
        g.compute_pagerank(np.ones(8), 1.0, 1e-9)
    iso = oracle.graph(5, [], [])
    w = np.array([1.0, 0.5, 0.0, 2.0, 0.25])
    assert np.array_equal(iso.compute_pagerank(w, 0.85, 1e-9).ranks, w)


def test_small_and_large_agree(oracle):
    # proj/tests/test_solvers.cpp:227-241
    rng = np.random.default_rng(112358)
    for _ in range(40):
        n = int(rng.integers(2, 50))
        s = list(range(n))
        d = [(v + 1) % n for v in range(n)]
        A = rng.random((n, n)) < 0.08
        np.fill_diagonal(A, False)
        xs, xd = np.nonzero(A)
        g = oracle.graph(n, np.r_[s, xs], np.r_[d, xd])
        w = 0.1 + rng.integers(0, 50, n) / 10.0
        direct = g.compute_pagerank(w, 0.85, 1e-9, 100).ranks
        series = g.compute_pagerank(w, 0.85, 1e-14, 1).ranks
        assert np.abs(direct - series).max() <= 1e-10


def test_partitioned_vs_dense_and_baseline(oracle):
    # proj/tests/test_engine.cpp:95-112
    rng = np.random.default_rng(8086)
    for trial in range(30):
        n = int(rng.integers(2, 40))
        s, d = random_graph(rng, n, 0.12, loops=True)
        g = oracle.graph(n, s, d)
        w = 0.05 + rng.integers(0, 200, n) / 40.0
        c = [0.5, 0.85, 0.95][trial % 3]
        M = np.eye(n)
        off, tgt, loop, deg = g.csr()
        for u in range(n):
            for v in tgt[off[u]:off[u + 1]]:
                if v != u:
                    M[v, u] -= c / deg[u]
        exact = np.linalg.solve(M, w)
        part = g.compute_pagerank(w, c, 1e-12, 2).ranks
        base, rep = g.compute_baseline(w, c, 1e-12)
        assert np.abs(part - exact).max() <= 1e-9
        assert np.abs(base - exact).max() <= 1e-9
        assert rep["iterative_edge_work"] == rep["total_iterations"] * rep["iterative_edges"]


def test_r1_normalisation_matches_bridge(oracle, ref):
    # R1 = R3/||R3||_1 equals the eigenvector oracle of solvers.cpp:200-244
    rng = np.random.default_rng(6174)
    for _ in range(20):
        n = int(rng.integers(2, 16))
        s, d = random_graph(rng, n, 0.2)
        w = 0.2 + rng.integers(0, 40, n) / 20.0
        r3 = oracle.graph(n, s, d).compute_pagerank(w, 0.85, 1e-13, 2).ranks
        r1_bridge, _, _ = ref.graph(n, s, d).oracle_bridge(w, 0.85)
        np.testing.assert_allclose(oracle.normalize_r1(r3), r1_bridge, rtol=1e-9, atol=1e-13)


def test_oracle_equals_reference_bitwise(oracle, ref):
    rng = np.random.default_rng(20261020)
    for t in range(150):
        n = int(rng.integers(1, 60))
        s, d = random_graph(rng, n, float(rng.uniform(0.0, 0.25)), loops=t % 2 == 0)
        keep = t % 3 == 0
        go, gr = oracle.graph(n, s, d, keep), ref.graph(n, s, d, keep)
        a, b = go.partition(), gr.partition()
        assert np.array_equal(a.comp_of, b.comp_of) and np.array_equal(a.kinds, b.kinds)
        assert np.array_equal(a.levels, b.levels) and a.stats == b.stats
        w = rng.uniform(0.05, 5, n)
        th = [1, 2, 100][t % 3]
        x, y = go.compute_pagerank(w, 0.85, 1e-12, th), gr.compute_pagerank(w, 0.85, 1e-12, th)
        assert np.array_equal(x.unit_iters, y.unit_iters)
        assert np.array_equal(x.ranks, y.ranks), t
        sa, sb = go.schedule(th), gr.schedule(th)
        for k in ("unit_kind", "ids", "edge_src", "edge_dst", "cross_src", "cross_dst", "cross_deg", "permutation"):
            assert np.array_equal(getattr(sa, k), getattr(sb, k)), k


def test_reference_acceptance_suite():
    # the reference's own acceptance binary, built from its sources against the shim
    exe = os.path.join(os.path.dirname(os.path.dirname(__file__)), "oracle", "_ref", "acceptance")
    if not os.path.exists(exe):
        pytest.skip("oracle/_ref not built")
    import subprocess
    out = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout
    assert out.stdout.count("PASS") == 10 and "SKIP 10" in out.stdout


def test_oracle_vs_golden(oracle):
    z = np.load(os.path.join(GOLDEN, "random_corpus.npz"))
    for t in range(int(z["trials"])):
        p = f"g{t}_"
        g = oracle.graph(int(z[p + "n"]), z[p + "src"], z[p + "dst"], bool(z[p + "keep"]))
        res = g.compute_pagerank(z[p + "w"], float(z[p + "c"]), 1e-12, int(z[p + "th"]))
        assert np.array_equal(res.unit_iters, z[p + "unit_iters"])
        np.testing.assert_allclose(res.ranks, z[p + "ranks"], rtol=1e-13)
        part = g.partition()
        assert np.array_equal(part.comp_of, z[p + "comp_of"]) and np.array_equal(part.levels, z[p + "levels"])
        assert res.report["total_edge_work"] == int(z[p + "total_edge_work"])
