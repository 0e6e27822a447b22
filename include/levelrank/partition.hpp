// levelrank-b200 host API: SCC/CAC partition with longest-path levels.
//
// Drop-in for proj/include/levelrank/partition.hpp:1-82.  find_components is
// an independent iterative Tarjan + CAC absorption (the one-pass rule of
// proj/src/partition.cpp:52-145).  Theorem 1 of the paper makes the partition
// unique, and component ids are dense by first appearance in vertex order, so
// comp_of / kinds / levels / sizes are bit-exact with the reference (tested in
// tests/test_partition.py against oracle/ and oracle/_ref).
#pragma once

#include <compare>
#include <cstdint>
#include <utility>
#include <vector>

#include "levelrank/graph.hpp"

namespace levelrank {
inline namespace b200 {

enum class ComponentKind : std::uint8_t { Scc, Cac };

struct Partition {
  std::vector<VertexId> comp_of;
  std::vector<ComponentKind> kinds;
  std::vector<std::int32_t> levels;
  std::vector<VertexId> sizes;
  std::int32_t max_level = -1;
  [[nodiscard]] std::size_t component_count() const noexcept { return kinds.size(); }
};

struct PartitionStats {
  EdgeId explore_edge_visits = 0;
  EdgeId merge_scan_edge_visits = 0;
  VertexId finish_calls = 0;
};

Partition find_components(const Graph& g, PartitionStats* stats = nullptr);
Partition find_components_scc_only(const Graph& g);

struct CanonicalComponent {
  std::vector<VertexId> members;
  ComponentKind kind = ComponentKind::Cac;
  std::int32_t level = 0;
  auto operator<=>(const CanonicalComponent&) const = default;
};
std::vector<CanonicalComponent> canonical_components(const Partition& p);
std::vector<std::uint8_t> big_scc_flags(const Partition& p);

struct PartitionCensus {
  std::int64_t components = 0;
  std::int64_t scc_components = 0;
  std::int64_t cac_components = 0;
  std::int64_t singleton_cacs = 0;
  VertexId largest_component = 0;
  ComponentKind largest_kind = ComponentKind::Cac;
  std::int32_t max_level = -1;
  std::int32_t level_count = 0;
  std::vector<std::int64_t> components_per_level;
  std::vector<std::pair<VertexId, std::int64_t>> size_histogram;
};
/// partition.cpp:353-382.
PartitionCensus census(const Partition& p);

}  // namespace b200
}  // namespace levelrank
