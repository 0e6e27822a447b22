"""The whole-graph power series (compute_baseline, proj/src/engine.cpp:184-218;
solve_baseline, proj/src/solvers.cpp:164-198) on the GPU: host layout checks
(CPU) and parity with the oracle's compute_baseline (GPU)."""
import numpy as np
import pytest

from conftest import FIXTURE8, random_graph


def _walk_degree(off, tgt, n, keep):
    deg = np.diff(off).astype(np.int64)
    if not keep:
        for u in range(n):
            deg[u] -= int(np.any(tgt[off[u]:off[u + 1]] == u))
    return deg


@pytest.mark.parametrize("keep", [False, True])
def test_baseline_layout(lr, keep):
    rng = np.random.default_rng(7 + keep)
    n = 300
    s, d = random_graph(rng, n, 0.03, loops=True)
    g = lr.Graph.from_edges(n, src=s, dst=d, loop_policy=int(keep))
    L = lr.Plan(g, baseline=True).layout()
    off, tgt, _, _ = g.csr()
    wd = _walk_degree(off, tgt, n, keep)
    assert L["n_levels"] == 1 and L["n_units"] == 1 and L["unit_kind"][0] == 3
    assert L["unit_edges"][0] == wd.sum()
    vo = L["vertex_of"]
    assert sorted(vo) == list(range(n))
    np.testing.assert_array_equal(L["row_of"][vo], np.arange(n))
    indeg = np.diff(L["iptr"])
    empty = indeg == 0
    assert not np.any(np.diff(empty.astype(int)) < 0)  # rows without in-edges last
    for cls in (~empty, empty):  # each class by descending walk degree
        assert np.all(np.diff(wd[vo][cls]) <= 0)
    np.testing.assert_array_equal(L["deg"], wd[vo])
    assert len(L["xsrc"]) == 0
    # in-edges of every row: its in-neighbours (ignored loops dropped), source ascending
    ins = [[] for _ in range(n)]
    for u in range(n):
        for v in tgt[off[u]:off[u + 1]]:
            if v != u or keep:
                ins[v].append(u)
    iptr, isrc = L["iptr"], L["isrc"]
    for r in range(n):
        got = vo[isrc[iptr[r]:iptr[r + 1]]]
        np.testing.assert_array_equal(got, ins[vo[r]])


def test_baseline_plan_has_no_schedule(lr):
    g = lr.Graph.from_edges(8, FIXTURE8)
    p = lr.Plan(g, baseline=True)
    with pytest.raises(ValueError):
        p.schedule()
    with pytest.raises(ValueError):
        p.census()


@pytest.mark.gpu
def test_baseline_fixture8(lr, oracle):
    g = lr.Graph.from_edges(8, FIXTURE8)
    go = oracle.graph(8, np.array([a for a, _ in FIXTURE8], np.int32), np.array([b for _, b in FIXTURE8], np.int32))
    ref, rrep = go.compute_baseline(np.ones(8), 0.85, 1e-9)
    res = lr.compute_baseline(g, np.ones(8), lr.SolverParams(0.85, 1e-9))
    np.testing.assert_allclose(res.ranks, ref, rtol=1e-10)
    for k in ("total_iterations", "iterative_edge_work", "total_edge_work"):
        assert res.report[k] == rrep[k], k


@pytest.mark.gpu
def test_baseline_random_graphs(lr, oracle):
    rng = np.random.default_rng(2024)
    for trial in range(60):
        n = int(rng.integers(2, 80))
        keep = trial % 3 == 0
        s, d = random_graph(rng, n, float(rng.uniform(0.02, 0.25)), loops=trial % 2 == 0)
        g = lr.Graph.from_edges(n, src=s, dst=d, loop_policy=int(keep))
        go = oracle.graph(n, s, d, keep)
        w = rng.uniform(0.0, 3.0, n)
        c = [0.5, 0.85, 0.99][trial % 3]
        ref, rrep = go.compute_baseline(w, c, 1e-12)
        res = lr.compute_baseline(g, w, lr.SolverParams(c, 1e-12))
        assert res.report["total_iterations"] == rrep["total_iterations"], trial
        assert res.report["iterative_edge_work"] == rrep["iterative_edge_work"], trial
        rel = np.abs(res.ranks - ref) / np.maximum(np.abs(ref), 1e-300)
        assert rel.max() <= 1e-10, (trial, rel.max())


@pytest.mark.gpu
@pytest.mark.parametrize("cfg,shrink", [(1, 1), (2, 4), (3, 6)])
def test_baseline_config_recipes(lr, oracle, cfg, shrink):
    """Grid-sized whole graphs (K4c over every vertex, dangling rows included)."""
    g = lr.config_graph(cfg, shrink)
    off, tgt, _, _ = g.csr()
    go = oracle.graph_from_csr(g.n, off, tgt)
    w = np.full(g.n, 1.0 / g.n)
    ref, rrep = go.compute_baseline(w, 0.85, 1e-12)
    res = lr.compute_baseline(g, w, lr.SolverParams(0.85, 1e-12))
    assert res.report["total_iterations"] == rrep["total_iterations"]
    assert res.report["total_edge_work"] == rrep["total_edge_work"]
    rel = np.abs(res.ranks - ref) / np.abs(ref)
    assert rel.max() <= 1e-10, rel.max()
    np.testing.assert_allclose(res.r1, oracle.normalize_r1(ref), rtol=1e-10)


@pytest.mark.gpu
def test_baseline_agrees_with_partitioned_solve(lr):
    """Same fixed point: partitioned and baseline differ only by the series
    truncation, far below 1e-6 relative at tol 1e-12."""
    g = lr.config_graph(2, 5)
    w = np.full(g.n, 1.0 / g.n)
    a = lr.compute_pagerank(g, w, lr.SolverParams(0.85, 1e-12))
    b = lr.compute_baseline(g, w, lr.SolverParams(0.85, 1e-12))
    assert np.max(np.abs(a.ranks - b.ranks) / a.ranks) < 1e-6


@pytest.mark.gpu
def test_baseline_degenerate_inputs(lr):
    g0 = lr.Graph.from_edges(0, [])
    assert len(lr.compute_baseline(g0, np.zeros(0)).ranks) == 0
    g = lr.Graph.from_edges(8, FIXTURE8)
    z = lr.compute_baseline(g, np.zeros(8))
    assert z.report["all_weights_zero"] and not z.ranks.any()
    with pytest.raises(ValueError):
        lr.compute_baseline(g, -np.ones(8))
    with pytest.raises(ValueError):
        lr.compute_baseline(g, np.ones(7))
