"""GPU parity on the reference's edge cases and on every device code path.

Each graph is shaped to force one path of the CUDA solve (heavy cross rows,
segmented SpMV rows, CAC slices, the three SccSmall solvers, deep level
chains) and is checked against the oracle restatement: ranks to 1e-10
relative, per-unit iteration counts and report counters exactly.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def check(lr, oracle, n, src, dst, w=None, c=0.85, tol=1e-12, th=100, keep=False):
    src = np.asarray(src, dtype=np.int32)
    dst = np.asarray(dst, dtype=np.int32)
    w = np.full(n, 1.0 / max(n, 1)) if w is None else np.asarray(w, dtype=np.float64)
    g = lr.Graph.from_edges(n, src=src, dst=dst, loop_policy=int(keep))
    ref = oracle.graph(n, src, dst, keep).compute_pagerank(w, c, tol, th)
    res = lr.compute_pagerank(g, w, lr.SolverParams(c, tol), small_threshold=th)
    assert np.array_equal(res.unit_iters, ref.unit_iters)
    if n:
        rel = np.abs(res.ranks - ref.ranks) / np.maximum(np.abs(ref.ranks), 1e-300)
        assert rel.max() <= 1e-10, rel.max()
    for k in ("total_edge_work", "iterative_edge_work", "components", "level_count", "total_iterations"):
        assert res.report[k] == ref.report[k], k
    return res


# proj/tests/test_engine.cpp:191-223
def test_degenerate_inputs(lr):
    empty = lr.Graph.from_edges(0, src=np.zeros(0, np.int32), dst=np.zeros(0, np.int32))
    assert len(lr.compute_pagerank(empty, np.zeros(0), lr.SolverParams(0.85, 1e-9)).ranks) == 0
    from conftest import FIXTURE8
    g = lr.Graph.from_edges(8, FIXTURE8)
    z = lr.compute_pagerank(g, np.zeros(8), lr.SolverParams(0.85, 1e-9))
    assert z.report["all_weights_zero"] == 1 and not z.ranks.any()
    with pytest.raises(ValueError):
        lr.compute_pagerank(g, np.ones(7), lr.SolverParams(0.85, 1e-9))
    w = np.ones(8)
    w[3] = -0.25
    with pytest.raises(ValueError):
        lr.compute_pagerank(g, w, lr.SolverParams(0.85, 1e-9))
    with pytest.raises(ValueError):
        lr.compute_pagerank(g, np.ones(8), lr.SolverParams(1.0, 1e-9))
    iso = lr.Graph.from_edges(5, src=np.zeros(0, np.int32), dst=np.zeros(0, np.int32))
    w = np.array([1.0, 0.5, 0.0, 2.0, 0.25])
    assert np.array_equal(lr.compute_pagerank(iso, w, lr.SolverParams(0.85, 1e-9)).ranks, w)


# proj/tests/test_solvers.cpp (kept self-loops: closed forms)
def test_kept_self_loops(lr, oracle):
    r = check(lr, oracle, 1, [0], [0], w=[1.0], keep=True, tol=1e-9).ranks
    assert abs(r[0] - 1 / 0.15) < 1e-12
    r = check(lr, oracle, 2, [0, 0], [0, 1], w=[1.0, 1.0], keep=True, tol=1e-9).ranks
    assert abs(r[0] - 40 / 23) < 1e-12


def test_heavy_cross_rows(lr, oracle):
    # one sink with 20,000 cross in-edges (> kCrossSplit: split over warps) and
    # one with 3,000 (> kCrossLight: warp butterfly)
    n = 20_003
    src = np.r_[np.arange(3, n), np.arange(3, 3003)]
    dst = np.r_[np.zeros(n - 3, np.int32), np.ones(3000, np.int32)]
    check(lr, oracle, n, src, dst)


def test_segmented_spmv_rows(lr, oracle):
    # a 6,000-vertex SCC (grid SpMV) whose vertex 0 has 5,999 intra in-edges
    # (segments of kSegNnz) and vertex 1 has 600 (long row)
    m = 6000
    ring_s = np.arange(m)
    ring_d = (ring_s + 1) % m
    src = np.r_[ring_s, np.arange(1, m), np.arange(2, 602)]
    dst = np.r_[ring_d, np.zeros(m - 1, np.int32), np.ones(600, np.int32)]
    res = check(lr, oracle, m, src, dst)
    assert res.report["large_scc_vertices"] == m


def test_big_cac_slices_and_depth(lr, oracle):
    # a 40,000-vertex out-tree (one CAC > kCacBlockMaxRows: grid-wide depth
    # slices) and a 20,000-vertex path (one CAC, 20,000 depth slices)
    rng = np.random.default_rng(7)
    n1 = 40_000
    parent = np.array([rng.integers(0, v) for v in range(1, n1)], dtype=np.int32)
    n2 = 20_000
    src = np.r_[parent, n1 + np.arange(n2 - 1)]
    dst = np.r_[np.arange(1, n1), n1 + np.arange(1, n2)]
    check(lr, oracle, n1 + n2, src, dst)


def test_cac_heavy_parent_rows(lr, oracle):
    # DAG: 300 sources all feeding one vertex (a CAC row with > kCrossLight parents), then a chain
    src = np.r_[np.arange(300), 300 + np.arange(50)]
    dst = np.r_[np.full(300, 300), 301 + np.arange(50)]
    check(lr, oracle, 351, src, dst)


def _scc(rng, base, m, deg=4):
    s = np.arange(m)
    extra_s = rng.integers(0, m, m * deg)
    extra_d = rng.integers(0, m, m * deg)
    keep = extra_s != extra_d
    return base + np.r_[s, extra_s[keep]], base + np.r_[(s + 1) % m, extra_d[keep]]


@pytest.mark.parametrize("m,th,c", [
    (2, 100, 0.85),      # tensor-core block Gauss-Jordan: one partial 8 x 8 block
    (8, 100, 0.85),      # one full block
    (9, 100, 0.85),      # a full block, then a one-row block
    (33, 100, 0.5),      # five blocks, the last partial
    (64, 100, 0.85),     # eight blocks, the largest tensor-core system
    (65, 100, 0.85),     # tensor cores, system in shared memory (above kSmallMmaMaxM), one-row last block
    (127, 200, 0.85),    # tensor cores, shared memory, partial last block
    (128, 200, 0.99),    # tensor cores, shared memory, largest (kSmallMmaSmemMaxM)
    (120, 200, 0.85),    # tensor cores, shared memory, row stride 8 mod 16 with a 16-row pad
    (150, 200, 0.85),    # normalised shared-memory Gauss-Jordan (m > kSmallTileMaxM)
    (220, 300, 0.85),    # global-scratch path (m > kSmallSmemMaxM)
    (100, 200, 0.9999),  # c near 1 (the fraction-free tile would underflow): tensor cores, shared memory
])
def test_small_scc_paths(lr, oracle, m, th, c):
    rng = np.random.default_rng(m)
    s1, d1 = _scc(rng, 0, m)
    s2, d2 = _scc(rng, m, 7)
    src = np.r_[s1, s2, [m + 1]]
    dst = np.r_[d1, d2, [3]]
    check(lr, oracle, m + 7, src, dst, th=th, c=c)


def test_cta_and_grid_power_series(lr, oracle):
    # SccLarge units on both sides of the CTA limit (kCtaLargeMaxRows rows) in one level
    rng = np.random.default_rng(11)
    s1, d1 = _scc(rng, 0, 3000, 3)
    s2, d2 = _scc(rng, 3000, 5000, 3)
    res = check(lr, oracle, 8000, np.r_[s1, s2], np.r_[d1, d2], c=0.9)
    assert (res.unit_iters > 0).sum() == 2


def test_ragged_weights(lr, oracle):
    # zeros, tiny and huge weights on a random graph with every unit kind
    rng = np.random.default_rng(5)
    n = 3000
    src = rng.integers(0, n, 9000)
    dst = rng.integers(0, n, 9000)
    w = rng.uniform(0, 1, n) * (rng.random(n) < 0.5)
    w[:10] = 1e-280
    w[10:20] = 1e120
    check(lr, oracle, n, src, dst, w=w, th=50)


def test_grid_units_converging_apart(lr, oracle):
    """Three grid-sized SccLarge units in one level whose weights differ by
    orders of magnitude: they stop at different iterations, and K4c's launches
    skip the finished units' tasks (unit done flags) while the others go on."""
    rng = np.random.default_rng(17)
    parts, base = [], 0
    for m in (6000, 5000, 4500):
        s, d = _scc(rng, base, m, deg=5)
        parts.append((s, d))
        base += m
    n = base
    src = np.concatenate([p[0] for p in parts])
    dst = np.concatenate([p[1] for p in parts])
    w = np.concatenate([np.full(6000, 1.0), np.full(5000, 1e-4), np.full(4500, 1e-8)])
    check(lr, oracle, n, src, dst, w=w)


def test_big_cac_structure_staged(lr, oracle):
    # a 20,000-row CAC (random out-tree plus forward chords, kept self-loops):
    # too large to stage whole, so k_cac_big stages only its structure and the
    # rows publish their pushed terms (cac_sweep_compact); plus a leaf with 100
    # parents (warp path).  Every row but that leaf is summed in the
    # reference's order: bit-exact.
    rng = np.random.default_rng(11)
    n = 20_000
    v = np.arange(1, n - 1)
    parent = (rng.random(n - 2) * v).astype(np.int32)
    cu = rng.integers(0, n - 2, 3000)
    cv = rng.integers(0, n - 2, 3000)
    keep = cu != cv
    cu, cv = np.minimum(cu, cv)[keep], np.maximum(cu, cv)[keep]
    loops = np.arange(0, n - 1, 97)
    heavy = rng.choice(n - 1, 100, replace=False)
    src = np.r_[parent, cu, loops, heavy]
    dst = np.r_[v, cv, loops, np.full(100, n - 1)]
    w = rng.random(n) + 0.5
    res = check(lr, oracle, n, src, dst, w=w, keep=True)
    ref = oracle.graph(n, np.asarray(src, np.int32), np.asarray(dst, np.int32), True).compute_pagerank(
        w, 0.85, 1e-12, 100)
    assert np.array_equal(res.ranks[: n - 1], ref.ranks[: n - 1])


def test_small_sccs_every_size_with_loops(lr, oracle):
    # one level of SccSmall units of every size 2..64 (the tensor-core path),
    # kept self-loops on some rows (diagonal entries other than 1), fed by one
    # upstream vertex
    rng = np.random.default_rng(5)
    src, dst, base = [], [], 1
    for m in range(2, 65):
        s1, d1 = _scc(rng, base, m, deg=3)
        loops = base + np.arange(0, m, 5)
        src += [s1, loops, [0]]
        dst += [d1, loops, [base]]
        base += m
    w = rng.random(base) + 0.1
    check(lr, oracle, base, np.concatenate(src), np.concatenate(dst), w=w, keep=True)


@pytest.mark.parametrize("m,th,keep", [(99, 100, True), (128, 200, False), (150, 200, True), (64, 100, True)])
def test_dense_small_scc_shared_memory_cap(lr, oracle, m, th, keep):
    """Complete SCCs below small_threshold whose in-edge stash outgrows
    k_level's 227 KB of shared memory (99 rows with kept loops: 232 KB) run
    in the global-scratch solve instead of failing the launch."""
    s, d = np.meshgrid(np.arange(m), np.arange(m), indexing="ij")
    s, d = s.ravel(), d.ravel()
    if not keep:
        s, d = s[s != d], d[s != d]
    # a second, sparse SCC on the same level keeps the k_level path busy too
    ring = np.arange(m, m + 40)
    s = np.concatenate([s, ring, [0]])
    d = np.concatenate([d, np.roll(ring, -1), [m]])
    w = np.random.default_rng(m).uniform(0.1, 2.0, m + 40)
    check(lr, oracle, m + 40, s, d, w=w, th=th, keep=keep)


@pytest.mark.parametrize("cfg,shrink", [(4, 3), (1, 1)])
def test_split_start_weights_bit_identical(lr, monkeypatch, cfg, shrink):
    """Large CACs' start weights summed in two halves across consecutive
    levels (kTaskRowsPart one level early, kTaskRowsFin at the row's level)
    give exactly the one-pass gather's ranks: the split is a prefix of each
    row's ordered cross list, so the additions and their order are unchanged."""
    g = lr.config_graph(cfg, shrink)
    w = np.full(g.n, 1.0 / g.n)
    monkeypatch.setenv("LR_XSPLIT", "0")
    a = lr.Engine(g).solve(w, lr.SolverParams(0.85, 1e-12))
    monkeypatch.setenv("LR_XSPLIT", "1")
    b = lr.Engine(g).solve(w, lr.SolverParams(0.85, 1e-12))
    assert np.array_equal(a[3], b[3])
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_cta_series_source_order_iteration_counts(lr, oracle, monkeypatch):
    """The CTA power series sums each row's first twelve in-edges pairwise and,
    by default, reorders in-edges for shared-memory banks; with the layout's
    source order (LR_BANK_ORDER=0) and by default, per-unit iteration counts
    equal the reference's and ranks agree to 1e-10."""
    g = lr.config_graph(1, 2)
    off, tgt, _, _ = g.csr()
    w = np.full(g.n, 1.0 / g.n)
    ref = oracle.graph_from_csr(g.n, off, tgt).compute_pagerank(w, 0.85, 1e-12, 100)
    for order in ("0", "1"):
        monkeypatch.setenv("LR_BANK_ORDER", order)
        res = lr.compute_pagerank(g, w, lr.SolverParams(0.85, 1e-12))
        assert np.array_equal(res.unit_iters, ref.unit_iters), order
        assert (np.abs(res.ranks - ref.ranks) / ref.ranks).max() <= 1e-10, order
