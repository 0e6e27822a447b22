"""The unit solvers of the reference's library API (solvers.hpp:31-54) on
the GPU (csrc/host/unit_solve.cpp through lr_solve_unit) against the
reference's own solve_singletons / solve_cac / solve_small_scc /
solve_large_scc (oracle/_ref), unit by unit, on the units of the reference's
own schedules: singletons and CACs bit for bit, dense SCC solves to 1e-12,
power series to 1e-10 with identical iteration counts; a cyclic 'CAC' raises
the reference's logic error."""
import numpy as np
import pytest

from conftest import FIXTURE8, random_graph

pytestmark = pytest.mark.gpu


def _units(sched):
    for u in range(len(sched.unit_kind)):
        i0, i1 = sched.unit_ids_begin[u], sched.unit_ids_begin[u + 1]
        e0, e1 = sched.unit_edges_begin[u], sched.unit_edges_begin[u + 1]
        yield (int(sched.unit_kind[u]), sched.ids[i0:i1], sched.edge_src[e0:e1], sched.edge_dst[e0:e1])


def test_unit_solvers_match_reference(lr, ref):
    rng = np.random.default_rng(31)
    graphs = [(8, *map(np.array, zip(*FIXTURE8)), False)]
    for t in range(14):
        n = int(rng.integers(5, 160))
        s, d = random_graph(rng, n, float(rng.uniform(0.01, 0.12)), loops=t % 2 == 0)
        graphs.append((n, np.asarray(s), np.asarray(d), t % 3 == 0))
    seen = set()
    for n, s, d, keep in graphs:
        g = lr.Graph.from_edges(n, src=s.astype(np.int32), dst=d.astype(np.int32), loop_policy=int(keep))
        rg = ref.graph(n, s, d, keep)
        for th in (100, 3):
            for kind, ids, es, ed in _units(rg.schedule(th)):
                w = rng.uniform(0.1, 2.0, len(ids))
                for c, tol in ((0.85, 1e-12), (0.5, 1e-9)):
                    want, wit, wvis = rg.solve_unit(kind, ids, es, ed, w, c, tol)
                    got, it, vis = lr.solve_unit(g, kind, ids, es, ed, w, lr.SolverParams(c, tol))
                    seen.add(kind)
                    if kind in (0, 1):
                        assert np.array_equal(got, want), (kind, got, want)
                        assert vis == wvis or kind == 0
                    elif kind == 2:
                        np.testing.assert_allclose(got, want, rtol=1e-12)
                    else:
                        assert it == wit
                        np.testing.assert_allclose(got, want, rtol=1e-10)
    assert seen == {0, 1, 2, 3}


def test_cac_solver_rejects_a_cycle(lr):
    g = lr.Graph.from_edges(3, [(0, 1), (1, 2), (2, 0)])
    with pytest.raises(lr.CycleError):
        lr.solve_unit(g, "cac", [0, 1, 2], [0, 1, 2], [1, 2, 0], np.ones(3), lr.SolverParams(0.85, 1e-9))


def test_power_series_stats_match_reference(lr, ref):
    """solve_large_scc with PowerSeriesStats: iteration count exact, ranks
    bit-exact (rows pulled in source order), the increments' L1 norms and the
    smallest increment entry equal to the reference's up to summation order."""
    rng = np.random.default_rng(5)
    done = 0
    for t in range(12):
        n = int(rng.integers(20, 300))
        s, d = random_graph(rng, n, float(rng.uniform(0.02, 0.08)), loops=t % 2 == 0)
        keep = t % 3 == 0
        g = lr.Graph.from_edges(n, src=s, dst=d, loop_policy=int(keep))
        rg = ref.graph(n, s, d, keep)
        for kind, ids, es, ed in _units(rg.schedule(1)):
            if kind != 3:
                continue
            w = rng.uniform(0.1, 2.0, len(ids))
            want, wit, wl1, wmin = rg.large_scc_stats(ids, es, ed, w, 0.85, 1e-12)
            got, it, l1, mn = lr.solve_large_scc_stats(g, ids, es, ed, w, lr.SolverParams(0.85, 1e-12))
            assert it == wit and len(l1) == len(wl1) == it
            assert np.array_equal(got, want)
            np.testing.assert_allclose(l1, wl1, rtol=1e-13)
            assert mn == wmin
            done += 1
    assert done > 5
