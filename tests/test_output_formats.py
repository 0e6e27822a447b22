"""Output formats: the product's writers (csrc/host/report.cpp
through lr_report_format / lr_ranks_format) are byte-equal to the
reference's -- SolveReport::write_text / write_json from proj/src/report.cpp
compiled unmodified into oracle/_ref, and the CLI's ranks TSV / bench CSV row
(proj/src/cli.cpp:80-83, :271-275).  CPU tests format the reference's own
reports and random field values; the GPU test formats our solve's report
against the reference's report of the same run (wall times zeroed)."""
import numpy as np
import pytest

from conftest import FIXTURE8


def _units(sched, iters, wall=None):
    size = np.diff(sched.unit_ids_begin)
    edges = np.diff(sched.unit_edges_begin)
    wall = np.zeros(len(size)) if wall is None else wall
    return [(int(k), int(lv), int(s), int(e), int(it), float(w))
            for k, lv, s, e, it, w in zip(sched.unit_kind, sched.unit_level, size, edges, iters, wall)]


def _ref_run(ref, n, src, dst, w, c, tol, th=100, parallel=False):
    g = ref.graph(n, np.asarray(src, np.int32), np.asarray(dst, np.int32))
    res = g.compute_pagerank(w, c, tol, th, parallel=parallel, threads=4 if parallel else 0)
    rep = dict(res.report)
    rep.update(method="partitioned", mode="parallel" if parallel else "sequential", c=c, tol=tol,
               small_threshold=th, keep_loops=0, largest_component_kind="scc" if rep["largest_is_scc"] else "cac")
    return res, rep, _units(g.schedule(th), res.unit_iters)


@pytest.mark.parametrize("fmt", ["text", "json", "csv_row"])
def test_reference_reports_byte_equal(lr, ref, fmt):
    s, d = zip(*FIXTURE8)
    cases = [(8, s, d, np.ones(8), 0.85, 1e-9, 100, False), (8, s, d, np.ones(8), 0.85, 1e-12, 1, True)]
    g1 = lr.config_graph(1, 4)
    off, tgt, _, _ = g1.csr()
    src = np.repeat(np.arange(g1.n, dtype=np.int32), np.diff(off))
    cases.append((g1.n, src, tgt, np.full(g1.n, 1.0 / g1.n), 0.85, 1e-12, 100, False))
    for n, src, dst, w, c, tol, th, par in cases:
        _, rep, units = _ref_run(ref, n, src, dst, w, c, tol, th, par)
        wall = np.random.default_rng(n).uniform(0, 50, len(units))
        units = [u[:5] + (float(x),) for u, x in zip(units, wall)]
        ours = lr.format_report(rep, units, fmt)
        theirs = ref.format_report(rep, units, fmt)
        assert ours == theirs, (fmt, ours[:400], theirs[:400])
    head = lr.format_report({}, (), "csv_header")
    assert head == "method,c,tol,total_iterations,iter_edge_work,wall_ms\n"


def test_random_report_values_byte_equal(lr, ref):
    rng = np.random.default_rng(5)
    ints = ["vertices", "edges", "components", "scc_components", "cac_components", "singleton_cacs",
            "largest_component", "max_level", "level_count", "large_scc_vertices", "total_iterations",
            "iterative_edge_work", "iterative_edges", "single_pass_edge_work", "cross_edge_count", "total_edge_work"]

    def rnd_double():
        k = rng.integers(0, 6)
        return [0.0, float(rng.integers(0, 10**6)), float(rng.uniform(0, 1)), float(rng.uniform(0, 1)) * 10.0 ** rng.integers(-300, 300),
                float(np.float64(rng.integers(1, 2**53)) / 2.0 ** int(rng.integers(0, 80))), 1e-12][k]

    for t in range(300):
        rep = {k: int(rng.integers(-1, 2**40)) if k not in ("largest_component", "max_level", "level_count")
               else int(rng.integers(-1, 2**31 - 1)) for k in ints}
        for k in ("eps_tot", "eps_avg", "mean_iterations_per_edge", "wall_ms", "c", "tol"):
            rep[k] = rnd_double()
        rep.update(method=["partitioned", "baseline"][t % 2], mode=["sequential", "parallel"][t % 3 == 0],
                   keep_loops=t % 5 == 0, small_threshold=int(rng.integers(1, 1000)), threads=int(rng.integers(1, 64)),
                   all_weights_zero=t % 7 == 0, largest_component_kind=["scc", "cac"][t % 2])
        units = [(int(rng.integers(0, 4)), int(rng.integers(0, 100)), int(rng.integers(1, 10**6)),
                  int(rng.integers(0, 10**9)), int(rng.integers(0, 2000)), rnd_double()) for _ in range(t % 4)]
        for fmt in ("text", "json", "csv_row"):
            assert lr.format_report(rep, units, fmt) == ref.format_report(rep, units, fmt), (t, fmt)


def test_ranks_tsv_byte_equal(lr, ref, tmp_path):
    rng = np.random.default_rng(9)
    r = np.concatenate([rng.uniform(0, 1, 500), rng.uniform(0, 1, 500) * 10.0 ** rng.integers(-320, 300, 500),
                        [0.0, 1.0, 1e-300, 5e-324, 1.7976931348623157e308, 123456789012.5, 0.1 + 0.2]])
    ours = lr.format_ranks(r)
    assert ours == ref.format_ranks(r)
    p = tmp_path / "ranks.tsv"
    lr.write_ranks(r, p)
    assert p.read_text() == ours
    assert lr.format_ranks(np.zeros(0)) == ""


@pytest.mark.gpu
def test_gpu_solve_report_matches_reference_output(lr, ref):
    """Our GPU run's report, written by our writer, equals the reference's
    report of its own CPU run written by the reference's writer (wall times
    zeroed in both): every counter, bound and unit record, byte for byte."""
    s, d = zip(*FIXTURE8)
    for tol, th in ((1e-9, 100), (1e-12, 1)):
        _, rep_ref, units_ref = _ref_run(ref, 8, s, d, np.ones(8), 0.85, tol, th)
        g = lr.Graph.from_edges(8, FIXTURE8)
        res = lr.compute_pagerank(g, np.ones(8), lr.SolverParams(0.85, tol), small_threshold=th)
        rep = dict(res.report)
        rep["wall_ms"] = rep_ref["wall_ms"] = 0.0
        units = lr.report_units(lr.Plan(g, th), res.unit_iters)
        for fmt in ("text", "json", "csv_row"):
            assert lr.format_report(rep, units, fmt) == ref.format_report(rep_ref, units_ref, fmt), fmt
        assert lr.format_ranks(res.ranks).splitlines()[0].startswith("0\t1")
