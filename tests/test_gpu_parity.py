"""GPU parity: the CUDA path through the C-ABI against the CPU oracle."""
import numpy as np
import pytest

from conftest import FIXTURE8, random_graph

pytestmark = pytest.mark.gpu

FIX8_RANKS = [1.0, 2.99670691547750, 1.425, 1.84906695938529, 1.605625, 3.81947320938530,
              9.72636742121042, 9.26741230802886]  # proj/tests/test_engine.cpp:23-34


def oracle_graph(oracle, g):
    off, tgt, _, _ = g.csr()
    return oracle.graph_from_csr(g.n, off, tgt)


def test_fixture8_ranks(lr):
    g = lr.Graph.from_edges(8, FIXTURE8)
    res = lr.compute_pagerank(g, np.ones(8), lr.SolverParams(0.85, 1e-9))
    np.testing.assert_allclose(res.ranks, FIX8_RANKS, rtol=1e-12)
    assert res.report["components"] == 4 and res.report["level_count"] == 3
    assert res.report["total_edge_work"] == 11 and res.report["cross_edge_count"] == 4


def test_random_graphs_all_kinds(lr, oracle):
    rng = np.random.default_rng(1003)
    for trial in range(120):
        n = int(rng.integers(2, 60))
        keep = trial % 4 == 0
        s, d = random_graph(rng, n, float(rng.uniform(0.02, 0.2)), loops=trial % 2 == 0)
        g = lr.Graph.from_edges(n, src=s, dst=d, loop_policy=int(keep))
        go = oracle.graph(n, s, d, keep)
        w = rng.uniform(0.05, 5.0, n)
        th = [1, 2, 100][trial % 3]
        c = [0.5, 0.85, 0.99][(trial // 3) % 3]
        ref = go.compute_pagerank(w, c, 1e-12, th)
        res = lr.compute_pagerank(g, w, lr.SolverParams(c, 1e-12), small_threshold=th)
        assert np.array_equal(res.unit_iters, ref.unit_iters), trial
        rel = np.abs(res.ranks - ref.ranks) / np.maximum(np.abs(ref.ranks), 1e-300)
        assert rel.max() <= 1e-10, (trial, rel.max())
        for k in ("total_edge_work", "iterative_edge_work", "single_pass_edge_work", "large_scc_vertices",
                  "components", "max_level", "total_iterations"):
            assert res.report[k] == ref.report[k], (trial, k)


@pytest.mark.parametrize("cfg,shrink", [(1, 1), (2, 4), (3, 6), (4, 5)])
def test_config_recipes(lr, oracle, cfg, shrink):
    g = lr.config_graph(cfg, shrink)
    go = oracle_graph(oracle, g)
    w = np.full(g.n, 1.0 / g.n)
    ref = go.compute_pagerank(w, 0.85, 1e-12, 100)
    res = lr.compute_pagerank(g, w, lr.SolverParams(0.85, 1e-12))
    assert np.array_equal(res.unit_iters, ref.unit_iters)
    rel = np.abs(res.ranks - ref.ranks) / np.abs(ref.ranks)
    assert rel.max() <= 1e-10, rel.max()
    np.testing.assert_allclose(res.r1, oracle.normalize_r1(ref.ranks), rtol=1e-10)
    assert res.report["total_edge_work"] == ref.report["total_edge_work"]


@pytest.mark.parametrize("shrink,chunks", [(6, 1), (6, 4), (3, 4), (3, 7)])
def test_sharded_path_single_rank(lr, monkeypatch, shrink, chunks):
    """The multi-GPU code path (row shards, the s' exchange cut into chunks
    that overlap the next chunk's SpMV on a second stream, deferred stop
    decision) on a one-rank communicator reproduces the unsharded solve bit
    for bit."""
    monkeypatch.setenv("LR_XCHG_CHUNKS", str(chunks))
    g = lr.config_graph(2, shrink)
    w = np.full(g.n, 1.0 / g.n)
    r3a, r1a, _, ita = lr.Engine(g).solve(w, lr.SolverParams(0.85, 1e-12))
    eng = lr.Engine(g, rank=0, world=1, nccl_id=lr.nccl_unique_id())
    r3b, r1b, _, itb = eng.solve(w, lr.SolverParams(0.85, 1e-12))
    assert np.array_equal(ita, itb)
    if chunks == 1:
        assert np.array_equal(r3a, r3b) and np.array_equal(r1a, r1b)
    else:
        # chunk cuts move K4c's tile boundaries, so rows spanning lanes are
        # summed in a different tree (as in any row-sharded run): last-bit
        # differences only, iteration counts identical
        assert np.max(np.abs(r3a - r3b) / r3a) <= 1e-14
        assert np.max(np.abs(r1a - r1b) / r1a) <= 1e-14


def test_engine_reuse_and_zero_weights(lr):
    g = lr.config_graph(2, 8)
    eng = lr.Engine(g)
    r3a, r1a, _, _ = eng.solve(np.full(g.n, 1.0 / g.n), lr.SolverParams(0.85, 1e-12))
    r3b, r1b, _, _ = eng.solve(np.full(g.n, 1.0 / g.n), lr.SolverParams(0.85, 1e-12))
    assert np.array_equal(r3a, r3b) and np.array_equal(r1a, r1b)
    z3, z1, info, _ = eng.solve(np.zeros(g.n), lr.SolverParams(0.85, 1e-9))
    assert info["all_weights_zero"] == 1 and not z3.any() and not z1.any()
    with pytest.raises(ValueError):
        w = np.ones(g.n)
        w[3] = -1
        eng.solve(w, lr.SolverParams(0.85, 1e-9))


def test_graph_replay_with_new_weights_and_params(lr, oracle):
    """Runs of static levels are CUDA-graph replays (ctx.cu segments): each solve
    must see its own weights and parameters, through host and device buffers,
    and agree bit for bit with the directly enqueued level loop (LR_GRAPHS=0)."""
    import os
    import torch
    g = lr.config_graph(4, 6)  # deep DAG: every level static
    off, tgt, _, _ = g.csr()
    go = oracle.graph_from_csr(g.n, off, tgt)
    eng = lr.Engine(g)
    rng = np.random.default_rng(5)
    for trial, c in enumerate((0.85, 0.5, 0.85)):
        w = rng.uniform(0.1, 2.0, g.n)
        ref = go.compute_pagerank(w, c, 1e-12, 100)
        r3, r1, _, it = eng.solve(w, lr.SolverParams(c, 1e-12))
        assert np.array_equal(it, ref.unit_iters), trial
        assert np.max(np.abs(r3 - ref.ranks) / ref.ranks) <= 1e-10, trial
        # device buffers (copied into the context's weight buffer for the replay)
        wd = torch.tensor(w, dtype=torch.float64, device="cuda")
        r3d = torch.empty_like(wd)
        r1d = torch.empty_like(wd)
        eng.solve_ptr(wd.data_ptr(), r3d.data_ptr(), r1d.data_ptr(), host=False, params=lr.SolverParams(c, 1e-12))
        assert np.array_equal(r3d.cpu().numpy(), r3), trial
        os.environ["LR_GRAPHS"] = "0"
        try:
            r3n, r1n, _, _ = eng.solve(w, lr.SolverParams(c, 1e-12))
        finally:
            os.environ.pop("LR_GRAPHS", None)
        assert np.array_equal(r3n, r3) and np.array_equal(r1n, r1), trial


@pytest.mark.parametrize("cfg,shrink", [(3, 6), (1, 2), (4, 5)])
def test_split_levels_single_rank(lr, monkeypatch, cfg, shrink):
    """Levels whose CTA-solved units are split over the ranks (every level here:
    LR_DIST_MIN_ROWS=0), on a one-rank communicator: the owner-only task lists,
    the per-level range broadcasts and the reduced iteration counts reproduce
    the replicated solve bit for bit."""
    monkeypatch.setenv("LR_XCHG_CHUNKS", "1")
    monkeypatch.setenv("LR_DIST_MIN_ROWS", "0")
    g = lr.config_graph(cfg, shrink)
    w = np.full(g.n, 1.0 / g.n)
    r3a, r1a, ia, ita = lr.Engine(g).solve(w, lr.SolverParams(0.85, 1e-12))
    eng = lr.Engine(g, rank=0, world=1, nccl_id=lr.nccl_unique_id())
    r3b, r1b, ib, itb = eng.solve(w, lr.SolverParams(0.85, 1e-12))
    assert np.array_equal(ita, itb)
    assert np.array_equal(r3a, r3b) and np.array_equal(r1a, r1b)
    assert ia["total_iterations"] == ib["total_iterations"]
    assert ia["iterative_edge_work"] == ib["iterative_edge_work"]


def test_unit_times(lr, monkeypatch):
    """UnitRecord::wall_ms on the GPU (LR_UNIT_TIMES=1): the units of a
    config-1 graph (all four kinds) get positive device spans; the giant
    unit's includes its grid SpMV time; results are unchanged."""
    g = lr.config_graph(1, 2)
    w = np.full(g.n, 1.0 / g.n)
    r3a = lr.Engine(g).solve(w, lr.SolverParams(0.85, 1e-12))[0]
    monkeypatch.setenv("LR_UNIT_TIMES", "1")
    eng = lr.Engine(g)
    r3b, _, info, it = eng.solve(w, lr.SolverParams(0.85, 1e-12))
    assert np.array_equal(r3a, r3b)
    ms = eng.unit_times()
    # (units in the global-scratch small-SCC kernel or CAC slices are not timed: 0)
    assert len(ms) == eng.n_units and (ms > 0).mean() > 0.9 and ms.max() < info["device_ms"] + 1e-9
    g2 = lr.config_graph(2, 6)
    e2 = lr.Engine(g2)
    _, _, info2, it2 = e2.solve(np.full(g2.n, 1.0 / g2.n), lr.SolverParams(0.85, 1e-12))
    L = e2.plan.layout()
    big = int(np.argmax(np.where(L["unit_kind"] == 3, L["unit_edges"], -1)))
    assert e2.unit_times()[big] >= 0.5 * info2["spmv_ms"]
