// Output formats of the hot path's callers, byte-compatible
// with the reference:
//   * SolveReport::write_text  -- "key: value" lines, doubles at 15 significant
//     digits, then one "unit: ..." line per unit   (proj/src/report.cpp:24-60)
//   * SolveReport::write_json  -- nlohmann::json dump(2): sections parameters /
//     census / bound / work, keys in std::map order  (proj/src/report.cpp:62-113)
//   * write_ranks              -- "v<TAB>rank" at 12 significant digits
//                                                     (proj/src/cli.cpp:80-83)
//   * bench CSV                -- method,c,tol,total_iterations,iter_edge_work,
//                                 wall_ms             (proj/src/cli.cpp:262-281)
// Every field is listed once in kFields, in text order with its JSON section;
// both writers walk that table.  The JSON number formatting (Grisu2 digits,
// ".0" on integral doubles) is nlohmann's own: the same single-header library
// the reference links, here from the copy that ships with this image.
#include <charconv>
#include <cstdio>
#include <ostream>
#include <string>
#include <variant>

#include <nlohmann/json.hpp>

#include "levelrank/engine.hpp"

namespace levelrank {
inline namespace b200 {
namespace {

using Value = std::variant<std::string, bool, std::int64_t, double>;

struct Field {
  const char* section;  // JSON object holding it ("" = top level)
  const char* key;      // text and JSON key
  Value (*get)(const SolveReport&);
};

#define LR_FIELD(sec, key, expr) \
  Field { sec, key, [](const SolveReport& r) -> Value { return expr; } }

const Field kFields[] = {
    LR_FIELD("parameters", "method", r.method),
    LR_FIELD("parameters", "mode", r.mode),
    LR_FIELD("parameters", "c", r.c),
    LR_FIELD("parameters", "tol", r.tol),
    LR_FIELD("parameters", "keep_loops", r.keep_loops),
    LR_FIELD("parameters", "small_threshold", std::int64_t{r.small_threshold}),
    LR_FIELD("parameters", "threads", std::int64_t{r.threads}),
    LR_FIELD("census", "vertices", r.vertices),
    LR_FIELD("census", "edges", r.edges),
    LR_FIELD("census", "components", r.components),
    LR_FIELD("census", "scc_components", r.scc_components),
    LR_FIELD("census", "cac_components", r.cac_components),
    LR_FIELD("census", "singleton_cacs", r.singleton_cacs),
    LR_FIELD("census", "largest_component", std::int64_t{r.largest_component}),
    LR_FIELD("census", "largest_component_kind", r.largest_component_kind),
    LR_FIELD("census", "max_level", std::int64_t{r.max_level}),
    LR_FIELD("census", "level_count", std::int64_t{r.level_count}),
    LR_FIELD("bound", "large_scc_vertices", r.large_scc_vertices),
    LR_FIELD("bound", "eps_tot", r.eps_tot),
    LR_FIELD("bound", "eps_avg", r.eps_avg),
    LR_FIELD("work", "total_iterations", r.total_iterations),
    LR_FIELD("work", "iterative_edge_work", r.iterative_edge_work),
    LR_FIELD("work", "iterative_edges", r.iterative_edges),
    LR_FIELD("work", "single_pass_edge_work", r.single_pass_edge_work),
    LR_FIELD("work", "cross_edges", r.cross_edge_count),
    LR_FIELD("work", "total_edge_work", r.total_edge_work),
    LR_FIELD("work", "mean_iterations_per_edge", r.mean_iterations_per_edge),
    LR_FIELD("", "all_weights_zero", r.all_weights_zero),
    LR_FIELD("", "wall_ms", r.wall_ms),
};
#undef LR_FIELD

const char* unit_kind_name(UnitKind k) {
  static const char* const names[] = {"singleton_group", "cac", "scc_small", "scc_large"};
  const auto i = static_cast<unsigned>(k);
  return i < 4 ? names[i] : "unknown";
}

// std::ostream << double under setprecision(p) with the default float field
// is printf's %.{p}g.
void put_g(std::ostream& out, double x, int prec) {
  char buf[64];
  std::snprintf(buf, sizeof buf, "%.*g", prec, x);
  out << buf;
}

void put_text(std::ostream& out, const Value& v) {
  std::visit(
      [&](const auto& x) {
        using T = std::decay_t<decltype(x)>;
        if constexpr (std::is_same_v<T, bool>) out << (x ? "true" : "false");
        else if constexpr (std::is_same_v<T, double>) put_g(out, x, 15);
        else out << x;
      },
      v);
}

nlohmann::json to_json(const Value& v) {
  return std::visit([](const auto& x) { return nlohmann::json(x); }, v);
}

}  // namespace

void SolveReport::write_text(std::ostream& out) const {
  for (const Field& f : kFields) {
    out << f.key << ": ";
    put_text(out, f.get(*this));
    out << '\n';
  }
  for (const UnitRecord& u : units) {
    out << "unit: kind=" << unit_kind_name(u.kind) << " level=" << u.level << " size=" << u.size
        << " edges=" << u.edges << " iterations=" << u.iterations << " wall_ms=";
    put_g(out, u.wall_ms, 15);
    out << '\n';
  }
}

void SolveReport::write_json(std::ostream& out) const {
  nlohmann::json doc = nlohmann::json::object();
  for (const Field& f : kFields) {
    nlohmann::json& slot = *f.section ? doc[f.section][f.key] : doc[f.key];
    slot = to_json(f.get(*this));
  }
  nlohmann::json list = nlohmann::json::array();
  for (const UnitRecord& u : units)
    list.push_back(nlohmann::json{{"kind", unit_kind_name(u.kind)},
                                  {"level", u.level},
                                  {"size", u.size},
                                  {"edges", u.edges},
                                  {"iterations", u.iterations},
                                  {"wall_ms", u.wall_ms}});
  doc["units"] = std::move(list);
  out << doc.dump(2) << '\n';
}

void write_ranks(std::ostream& out, std::span<const double> ranks) {
  std::string line;
  char num[40];
  for (std::size_t v = 0; v < ranks.size(); ++v) {
    const auto r = std::to_chars(num, num + sizeof num, static_cast<long long>(v));
    line.assign(num, r.ptr);
    line += '\t';
    std::snprintf(num, sizeof num, "%.12g", ranks[v]);
    line += num;
    line += '\n';
    out << line;
  }
}

void write_bench_header(std::ostream& out) { out << "method,c,tol,total_iterations,iter_edge_work,wall_ms\n"; }

void write_bench_row(std::ostream& out, const SolveReport& r) {
  out << r.method << (r.mode == "parallel" ? "_parallel" : "") << ',';
  put_g(out, r.c, 15);
  out << ',';
  put_g(out, r.tol, 15);
  out << ',' << r.total_iterations << ',' << r.iterative_edge_work << ',';
  put_g(out, r.wall_ms, 15);
  out << '\n';
}

}  // namespace b200
}  // namespace levelrank
