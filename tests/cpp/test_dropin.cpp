// C++ drop-in check: a reference-style caller compiled against
// include/levelrank/*.hpp (with an Eigen on the include path, so the Eigen
// overloads are the ones instantiated) and linked to liblevelrank_b200.so.
// The cases restate the reference's engine known answers
// (proj/tests/test_engine.cpp: fixture ranks and report :23-93, forced power
// series :95-115, weight propagation :169-179, error bound :181-189,
// degenerate inputs :191-223, baseline report :225-235) plus the graph and
// partition entry points.  Test infrastructure: built by tests/cpp/Makefile,
// run by tests/test_cpp_dropin.py on a GPU box.  Prints one line per failed
// check and exits with the failure count.
#include <cmath>
#include <cstdio>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "levelrank/engine.hpp"

#ifndef LEVELRANK_B200_HAVE_EIGEN
#error "this test instantiates the Eigen overloads: put an Eigen/Dense on the include path"
#endif

using namespace levelrank;

static int failures = 0;
#define CHECK(cond)                                                      \
  do {                                                                   \
    if (!(cond)) {                                                       \
      ++failures;                                                        \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);        \
    }                                                                    \
  } while (0)
#define CHECK_THROWS(expr, type)                                         \
  do {                                                                   \
    bool got = false;                                                    \
    try {                                                                \
      (void)(expr);                                                      \
    } catch (const type&) {                                              \
      got = true;                                                        \
    } catch (...) {                                                      \
    }                                                                    \
    if (!got) {                                                          \
      ++failures;                                                        \
      std::printf("FAIL %s:%d: %s throws %s\n", __FILE__, __LINE__, #expr, #type); \
    }                                                                    \
  } while (0)

static bool close_rel(double a, double b, double eps) { return std::fabs(a - b) <= eps * std::max(std::fabs(b), 1.0); }

// the paper's 8-vertex example (proj/tests/test_support.cpp:14-21)
static Graph fixture8() {
  return Graph::from_edges(8, {{0, 1}, {0, 2}, {1, 3}, {2, 4}, {2, 5}, {1, 5}, {4, 5}, {6, 7}, {3, 1}, {7, 6}, {1, 6}});
}

int main() {
  const Graph g = fixture8();
  {  // closed-form ranks, the reference caller's spelling
    const auto res = compute_pagerank(g, Eigen::VectorXd::Ones(8), {0.85, 1e-9});
    const double want[8] = {1.0, 2.99670691547750, 1.425, 1.84906695938529,
                            1.605625, 3.81947320938530, 9.72636742121042, 9.26741230802886};
    for (int v = 0; v < 8; ++v) CHECK(close_rel(res.ranks(v), want[v], 1e-10));
    double s = 0;
    for (int v = 0; v < 8; ++v) s += res.ranks(v);
    CHECK(close_rel(res.r1.sum(), 1.0, 1e-12) && close_rel(res.r1(6), want[6] / s, 1e-12));
    const SolveReport& rep = res.report;
    CHECK(rep.method == "partitioned" && rep.mode == "sequential" && rep.threads == 1);
    CHECK(rep.vertices == 8 && rep.edges == 11 && rep.components == 4);
    CHECK(rep.scc_components == 2 && rep.cac_components == 2 && rep.singleton_cacs == 1);
    CHECK(rep.largest_component == 3 && rep.largest_component_kind == "cac");
    CHECK(rep.max_level == 2 && rep.level_count == 3);
    CHECK(rep.large_scc_vertices == 0 && rep.eps_tot == 0.0 && rep.total_iterations == 0);
    CHECK(rep.single_pass_edge_work == 11 && rep.cross_edge_count == 4 && rep.total_edge_work == 11);
    CHECK(!rep.all_weights_zero);
    CHECK(rep.units.size() == 4);
    if (rep.units.size() == 4) {
      CHECK(rep.units[0].kind == UnitKind::SingletonGroup && rep.units[0].level == 2);
      CHECK(rep.units[1].kind == UnitKind::SccSmall && rep.units[1].size == 2);
      CHECK(rep.units[2].kind == UnitKind::Cac && rep.units[2].edges == 3);
      CHECK(rep.units[3].kind == UnitKind::SccSmall && rep.units[3].level == 0);
    }
    std::ostringstream text, json;
    rep.write_text(text);
    rep.write_json(json);
    CHECK(text.str().rfind("method: partitioned\n", 0) == 0);
    CHECK(json.str().find("\"total_edge_work\": 11") != std::string::npos);
  }
  {  // small_threshold 1 forces the power series on both SCCs
    const auto res = compute_pagerank(g, Eigen::VectorXd::Ones(8), {0.85, 1e-12}, ExecutionMode::Sequential, 1);
    CHECK(res.report.large_scc_vertices == 4);
    CHECK(close_rel(res.report.eps_tot, 4 * 1e-12 * 0.85 / 0.15, 1e-12));
    CHECK(close_rel(res.report.eps_avg, res.report.eps_tot / 8.0, 1e-12));
    CHECK(res.report.total_iterations > 0 && res.report.iterative_edges == 4);
    CHECK(res.report.iterative_edge_work == res.report.total_edge_work - res.report.single_pass_edge_work);
    const auto exact = compute_pagerank(g, Eigen::VectorXd::Ones(8), {0.85, 1e-12});
    CHECK((res.ranks - exact.ranks).cwiseAbs().maxCoeff() <= 1e-9);
    const auto par = compute_pagerank(g, Eigen::VectorXd::Ones(8), {0.85, 1e-12}, ExecutionMode::Parallel, 1, 4);
    CHECK(par.ranks == res.ranks && par.report.mode == "parallel" && par.report.threads == 4);
  }
  {  // weight propagation along cross edges
    Eigen::VectorXd ranks(2);
    ranks << 1.0, 3.0;
    Eigen::VectorXd weights = Eigen::VectorXd::Zero(4);
    weights(3) = 0.5;
    const std::vector<CrossEdge> cross{{0, 2, 2}, {0, 3, 2}, {1, 3, 3}};
    propagate_weights(cross, ranks, 0.85, weights);
    CHECK(close_rel(weights(2), 0.425, 1e-15));
    CHECK(close_rel(weights(3), 0.5 + 0.425 + 0.85, 1e-15));
    CHECK(weights(0) == 0.0);
  }
  {  // error bound
    const ErrorBound zero = error_bound(0, 100, {0.85, 1e-9});
    CHECK(zero.eps_tot == 0.0 && zero.eps_avg == 0.0);
    const ErrorBound b = error_bound(1000, 10000, {0.85, 1e-9});
    CHECK(close_rel(b.eps_tot, 1000 * 1e-9 * 0.85 / 0.15, 1e-12));
    CHECK(close_rel(b.eps_avg, b.eps_tot / 10000.0, 1e-12));
  }
  {  // degenerate inputs
    const Graph empty = Graph::from_edges(0, {});
    const auto res = compute_pagerank(empty, Eigen::VectorXd(), {0.85, 1e-9});
    CHECK(res.ranks.size() == 0 && res.report.components == 0);
    const auto zero = compute_pagerank(g, Eigen::VectorXd::Zero(8), {0.85, 1e-9});
    CHECK(zero.report.all_weights_zero && zero.ranks.cwiseAbs().maxCoeff() == 0.0);
    const auto bzero = compute_baseline(g, Eigen::VectorXd::Zero(8), {0.85, 1e-9});
    CHECK(bzero.report.all_weights_zero);
    CHECK_THROWS(compute_pagerank(g, Eigen::VectorXd::Ones(7), {0.85, 1e-9}), std::invalid_argument);
    CHECK_THROWS(compute_baseline(g, Eigen::VectorXd::Ones(9), {0.85, 1e-9}), std::invalid_argument);
    Eigen::VectorXd w = Eigen::VectorXd::Ones(8);
    w(3) = -0.25;
    CHECK_THROWS(compute_pagerank(g, w, {0.85, 1e-9}), std::invalid_argument);
    CHECK_THROWS(compute_baseline(g, w, {0.85, 1e-9}), std::invalid_argument);
    CHECK_THROWS(compute_pagerank(g, Eigen::VectorXd::Ones(8), {1.0, 1e-9}), std::invalid_argument);
    CHECK_THROWS(compute_pagerank(g, Eigen::VectorXd::Ones(8), {0.85, 0.0}), std::invalid_argument);
    const Graph iso = Graph::from_edges(5, {});
    Eigen::VectorXd wi(5);
    wi << 1.0, 0.5, 0.0, 2.0, 0.25;
    const auto ri = compute_pagerank(iso, wi, {0.85, 1e-9});
    CHECK(ri.ranks == wi && ri.report.level_count == 1 && ri.report.units.size() == 1);
  }
  {  // baseline report shape, and the whole-graph series agrees with the partitioned solve
    const auto res = compute_baseline(g, Eigen::VectorXd::Ones(8), {0.85, 1e-12});
    CHECK(res.report.method == "baseline" && res.report.vertices == 8);
    CHECK(res.report.total_iterations > 0 && res.report.iterative_edges == 11);
    CHECK(res.report.iterative_edge_work == res.report.total_iterations * 11);
    const auto part = compute_pagerank(g, Eigen::VectorXd::Ones(8), {0.85, 1e-12});
    CHECK((res.ranks - part.ranks).cwiseAbs().maxCoeff() <= 1e-9);
  }
  {  // graph / partition / schedule entry points
    std::istringstream in("# fixture\n0\t1\r\n1\t0\n1\t2\n");
    const Graph p = parse_edge_list(in, true);
    CHECK(p.vertex_count() == 3 && p.edge_count() == 3);
    CHECK_THROWS(load_edge_list("/nonexistent/edges.tsv", true), IoError);
    std::istringstream bad("0 1\n");
    CHECK_THROWS(parse_edge_list(bad, true), ParseError);
    PartitionStats st;
    const Partition part = find_components(g, &st);
    CHECK(part.component_count() == 4 && part.max_level == 2 && st.finish_calls > 0);
    const Schedule s = build_schedule(g, part, 100);
    CHECK(s.levels.size() == 3 && s.cross_edge_count == 4 && s.intra_edge_count == 7);
    CHECK_THROWS(build_schedule(g, part, 0), std::invalid_argument);
  }
  {  // the span API and output writers
    std::vector<double> w(8, 1.0);
    const EngineResult r = compute_pagerank(g, std::span<const double>(w), SolverParams{0.85, 1e-9});
    std::ostringstream ranks, csv;
    write_ranks(ranks, r.ranks);
    CHECK(ranks.str().rfind("0\t1\n1\t2.99670691548\n", 0) == 0);
    write_bench_header(csv);
    write_bench_row(csv, r.report);
    CHECK(csv.str() == "method,c,tol,total_iterations,iter_edge_work,wall_ms\npartitioned,0.85,1e-09,0,0," +
                           [&] {
                             char b[64];
                             std::snprintf(b, sizeof b, "%.15g", r.report.wall_ms);
                             return std::string(b);
                           }() + "\n");
  }
  std::printf("%s: %d failure(s)\n", failures ? "FAILED" : "ok", failures);
  return failures;
}
