// Plan-build internals shared by the partition and the layout: the graph's
// in-edge lists are built once (by the partition, which needs them for its
// backward reachability and wavefront release) and reused by the layout for
// its per-row pull lists, instead of a second transpose of every edge.
#pragma once

#include <cstdint>
#include <vector>

#include "levelrank/partition.hpp"
#include "levelrank/schedule.hpp"

namespace levelrank {
inline namespace b200 {
namespace detail {

struct InEdges {
  uvector<EdgeId> off;    // n + 1
  uvector<VertexId> src;  // per target vertex: sources ascending, self-loops left out
};

Partition find_components_with_in_edges(const Graph& g, PartitionStats* stats, InEdges& in);
Layout build_layout_from(const Graph& g, const Partition& p, VertexId small_threshold, const InEdges& in);

}  // namespace detail
}  // namespace b200
}  // namespace levelrank
