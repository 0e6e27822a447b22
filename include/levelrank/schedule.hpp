// levelrank-b200 host API: level-major schedule and the device Layout.
//
// build_schedule is the drop-in for proj/src/schedule.cpp:32-137 (same unit
// list, kinds, order, singleton-group slotting, local ids, cross buckets and
// permutation).  build_layout is what the GPU path consumes instead: the same
// units, laid out level-major in HBM with *pull* (in-edge) CSRs whose per-row
// source order reproduces the reference's summation order, so every term and
// every accumulation order of the singleton, CAC, propagation and power-series
// paths matches the reference.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <iosfwd>
#include <utility>
#include <vector>

#include "levelrank/graph.hpp"
#include "levelrank/partition.hpp"

namespace levelrank {
inline namespace b200 {

enum class UnitKind : std::uint8_t { SingletonGroup, Cac, SccSmall, SccLarge };

/// solvers.cpp:84-85 throws std::logic_error when a CAC never drains; this
/// subtype lets the C-ABI tell it apart from other logic errors.
class CycleError : public std::logic_error {
 public:
  using std::logic_error::logic_error;
};

struct SolveUnit {
  UnitKind kind = UnitKind::SingletonGroup;
  std::int32_t level = 0;
  std::vector<VertexId> global_ids;
  std::vector<std::pair<VertexId, VertexId>> edges;
  [[nodiscard]] VertexId size() const noexcept { return static_cast<VertexId>(global_ids.size()); }
};

struct CrossEdge {
  VertexId src = 0;
  VertexId dst = 0;
  VertexId src_out_degree = 0;
};

struct ScheduleLevel {
  std::int32_t level = 0;
  std::vector<SolveUnit> units;
  std::vector<CrossEdge> cross_edges;
};

struct Schedule {
  std::vector<ScheduleLevel> levels;
  std::vector<VertexId> permutation;
  EdgeId intra_edge_count = 0;
  EdgeId cross_edge_count = 0;
  EdgeId dropped_loop_count = 0;
};

/// schedule.cpp:32-137 (std::invalid_argument if small_threshold < 1).
Schedule build_schedule(const Graph& g, const Partition& p, VertexId small_threshold);

/// Device layout of one graph (host copy; uploaded by lr_ctx_upload).
/// Rows are vertices in level-major order: levels descending, then units in
/// schedule order, then within a unit:
///   SingletonGroup / SccSmall: ascending vertex id
///     (= the reference's local ids, schedule.cpp:101-109)
///   SccLarge: descending in-unit out-degree, then vertex id (gather
///     locality; each row's in-edge list keeps the reference's order)
///   Cac: ascending (intra-CAC depth, vertex id); depth = longest path from
///     the CAC's in-degree-0 vertices, so each depth slice depends only on
///     earlier slices.
struct Layout {
  VertexId n = 0;
  std::int32_t max_level = -1;
  bool keep_loops = false;
  std::vector<std::int32_t> level_row_begin;   // n_levels + 1, level index 0 = max_level
  std::vector<std::int32_t> level_unit_begin;  // n_levels + 1
  uvector<VertexId> vertex_of;             // row -> vertex
  uvector<VertexId> row_of;                // vertex -> row
  uvector<VertexId> deg;                   // walk out-degree per row
  std::vector<std::uint8_t> loop;              // per row: keep && self-loop (singleton/CAC factor)
  // cross in-edges (pull) per row; sources as rows, ordered (source level
  // descending, source vertex ascending) = propagate_weights order.
  uvector<EdgeId> xptr;
  uvector<VertexId> xsrc;
  // intra-unit in-edges (pull) per row; sources as rows.  SCC rows: source
  // vertex ascending (the reference's push order over unit.edges); CAC rows:
  // source Kahn dequeue position (solve_cac's push order).  Self-loops appear
  // only in SCC rows under LoopPolicy::Keep.
  uvector<EdgeId> iptr;
  uvector<VertexId> isrc;
  // units in schedule order
  std::vector<std::uint8_t> unit_kind;      // UnitKind
  std::vector<std::int32_t> unit_level;     // partition level
  std::vector<std::int32_t> unit_row_begin; // n_units + 1
  std::vector<EdgeId> unit_edges;           // reference unit.edges.size()
  // CAC depth slices: for CAC unit u, rows [depth_ptr[cac_depth_begin[u]+d],
  // depth_ptr[cac_depth_begin[u]+d+1]) have depth d.  -1 for other kinds.
  std::vector<std::int64_t> cac_depth_begin;
  std::vector<std::int32_t> depth_ptr;
  // totals (schedule.hpp:45-50)
  EdgeId intra_edge_count = 0;
  EdgeId cross_edge_count = 0;
  EdgeId dropped_loop_count = 0;
  [[nodiscard]] std::int32_t level_count() const noexcept { return max_level + 1; }
  [[nodiscard]] std::int64_t unit_count() const noexcept {
    return static_cast<std::int64_t>(unit_kind.size());
  }
};

/// The reference's schedule permutation (vertex -> row of schedule.cpp:49-52,
/// order: level desc, component size desc, component id, vertex id).
std::vector<VertexId> schedule_permutation(const Partition& p);

/// Multi-threaded layout build (std::invalid_argument if small_threshold < 1).
Layout build_layout(const Graph& g, const Partition& p, VertexId small_threshold);

/// The whole graph as ONE power-series unit (kind SccLarge, one level, no
/// cross edges): the device layout of compute_baseline / solve_baseline
/// (proj/src/engine.cpp:184-218, proj/src/solvers.cpp:164-198), the
/// partition-free "basic method".  Rows by descending walk out-degree (ties by
/// vertex id), vertices without in-edges last; every row's in-edges by source vertex ascending (the
/// reference's push order); ignored self-loops dropped, kept ones included;
/// unit_edges = walk_edge_count (proj/src/engine.cpp:20-24).
Layout build_baseline_layout(const Graph& g);

}  // namespace b200
}  // namespace levelrank
