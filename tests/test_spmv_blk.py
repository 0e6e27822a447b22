"""K5 (k_spmv_blk, spmv.cu): the dest-blocked, source-sorted power-series SpMV
of large grid units, forced onto small graphs (LR_BLK_MIN_ROWS=0) with small
blocks and parts so every path runs: many blocks, blocks split over several
parts (partial rows through yacc, last part finishes), padding dummies, rows
without in-edges (the whole-graph baseline layout), kept self-loops.  Against
the CPU oracle: per-unit iteration counts equal, R3 within 1e-10 relative
(the shared-memory accumulation order is not the reference's push order)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CASES = [  # (block rows, entries per part)
    (16384, 0),   # defaults: one block at these sizes
    (512, 0),     # many blocks, about eight parts per SM
    (256, 256),   # every block split into 256-entry parts
    (4000, 1024), # block rows not a power of two
]


def _force(monkeypatch, br, part):
    monkeypatch.setenv("LR_BLK", "1")
    monkeypatch.setenv("LR_BLK_MIN_ROWS", "0")
    monkeypatch.setenv("LR_BLK_MIN_DEG", "0")
    monkeypatch.setenv("LR_BLK_ROWS", str(br))
    if part:
        monkeypatch.setenv("LR_BLK_PART", str(part))
    else:
        monkeypatch.delenv("LR_BLK_PART", raising=False)


def _check(res, ref):
    assert np.array_equal(res.unit_iters, ref.unit_iters)
    rel = np.abs(res.ranks - ref.ranks) / np.maximum(np.abs(ref.ranks), 1e-300)
    assert rel.max() <= 1e-10, rel.max()
    assert res.report["total_edge_work"] == ref.report["total_edge_work"]
    assert res.report["total_iterations"] == ref.report["total_iterations"]


@pytest.mark.parametrize("br,part", CASES)
@pytest.mark.parametrize("cfg,shrink", [(2, 4), (3, 5)])
def test_blk_configs(lr, oracle, monkeypatch, cfg, shrink, br, part):
    _force(monkeypatch, br, part)
    g = lr.config_graph(cfg, shrink)
    off, tgt, _, _ = g.csr()
    w = np.full(g.n, 1.0 / g.n)
    ref = oracle.graph_from_csr(g.n, off, tgt).compute_pagerank(w, 0.85, 1e-12, 100)
    eng = lr.Engine(g)
    assert eng.blk_units() >= 1
    r3, r1, info, it = eng.solve(w, lr.SolverParams(0.85, 1e-12))
    res = lr.EngineResult(r3, r1, {"total_edge_work": ref.report["total_edge_work"],
                                    "total_iterations": info["total_iterations"]}, it)
    _check(res, ref)
    assert abs(r1.sum() - 1.0) < 1e-12


@pytest.mark.parametrize("br,part", CASES[1:3])
def test_blk_random_kept_loops(lr, oracle, monkeypatch, br, part):
    _force(monkeypatch, br, part)
    rng = np.random.default_rng(7)
    for t in range(3):
        n = int(rng.integers(6000, 9000))  # giant SCC past the CTA power series: a grid unit
        m = 8 * n
        e = np.unique(rng.integers(0, n, m) * n + rng.integers(0, n, m))
        s, d = (e // n).astype(np.int32), (e % n).astype(np.int32)
        keep = t % 2
        g = lr.Graph.from_edges(n, src=s, dst=d, loop_policy=keep)
        w = rng.random(n)
        eng = lr.Engine(g)
        assert eng.blk_units() == 1
        ref = oracle.graph(n, s, d, keep).compute_pagerank(w, 0.85, 1e-12, 100)
        res = lr.compute_pagerank(g, w, lr.SolverParams(0.85, 1e-12))
        _check(res, ref)


@pytest.mark.parametrize("br,part", CASES[1:3])
def test_blk_baseline(lr, oracle, monkeypatch, br, part):
    """The whole-graph power series (compute_baseline) through K5: rows without
    in-edges get y = 0."""
    _force(monkeypatch, br, part)
    g = lr.config_graph(3, 6)
    off, tgt, _, _ = g.csr()
    w = np.full(g.n, 1.0 / g.n)
    ref, rrep = oracle.graph_from_csr(g.n, off, tgt).compute_baseline(w, 0.85, 1e-12)
    assert lr.Engine(g, baseline=True).blk_units() == 1
    res = lr.compute_baseline(g, w, lr.SolverParams(0.85, 1e-12))
    assert res.report["total_iterations"] == rrep["total_iterations"]
    rel = np.abs(res.ranks - ref) / np.maximum(np.abs(ref), 1e-300)
    assert rel.max() <= 1e-10, rel.max()


@pytest.mark.gpu
@pytest.mark.parametrize("br,chunks", [(512, 1), (512, 4), (4000, 3), (256, 7)])
def test_blk_sharded_single_rank(lr, monkeypatch, br, chunks):
    """K5 in the row-sharded (multi-GPU) path: one layout per exchange chunk of
    the rank's shard, maxima held until the last chunk and published for the
    all-reduce -- on a one-rank communicator, against the unsharded K4c solve."""
    g = lr.config_graph(2, 4)
    w = np.full(g.n, 1.0 / g.n)
    monkeypatch.setenv("LR_BLK", "0")
    r3a, r1a, _, ita = lr.Engine(g).solve(w, lr.SolverParams(0.85, 1e-12))
    _force(monkeypatch, br, 0)
    monkeypatch.setenv("LR_XCHG_CHUNKS", str(chunks))
    eng = lr.Engine(g, rank=0, world=1, nccl_id=lr.nccl_unique_id())
    assert eng.blk_units() == chunks
    r3b, r1b, info, itb = eng.solve(w, lr.SolverParams(0.85, 1e-12))
    assert np.array_equal(ita, itb)
    assert np.max(np.abs(r3a - r3b) / r3a) <= 1e-13
    assert np.max(np.abs(r1a - r1b) / r1a) <= 1e-13
    r3c, _, _, itc = eng.solve(w, lr.SolverParams(0.85, 1e-12))  # a second solve on the same context
    assert np.array_equal(itb, itc) and np.max(np.abs(r3c - r3b) / r3b) <= 1e-13
