// Drop-in for parsim/collectives.hpp: allreduce_mean on the GPU, folding the
// P buffers in the configured reference order (naive / ring /
// hierarchical; pipelined_ring folds as ring) with the mean as sum * (1/P),
// bit-identical to the reference's dense folds.  Topology, WorkerGroup, the
// alpha-beta cost model (comm_cost, ...) stay the reference's own.  See
// numerics.hpp for usage.
//
//   allreduce_mean(group, algo, topo)   collectives.hpp:135-148
//   allreduce_mean(group, algo)         collectives.hpp:150-154 (flat, dpn = P)
#pragma once

#include "parsim/numerics.hpp"

#define allreduce_mean parsim_reference_allreduce_mean
#include_next "parsim/collectives.hpp"
#undef allreduce_mean

namespace parsim {

namespace dropin_detail {
inline parsim_b200::CollectiveAlgorithm algo_of(CollectiveAlgorithm a) {
  switch (a) {
    case CollectiveAlgorithm::naive: return parsim_b200::CollectiveAlgorithm::naive;
    case CollectiveAlgorithm::ring: return parsim_b200::CollectiveAlgorithm::ring;
    case CollectiveAlgorithm::hierarchical: return parsim_b200::CollectiveAlgorithm::hierarchical;
    case CollectiveAlgorithm::pipelined_ring: return parsim_b200::CollectiveAlgorithm::pipelined_ring;
  }
  detail::fail("allreduce_mean: unknown algorithm");
}
inline parsim_b200::Topology topo_of(const Topology& t) {
  parsim_b200::Topology o;
  o.racks = t.racks;
  o.nodes_per_rack = t.nodes_per_rack;
  o.devices_per_node = t.devices_per_node;
  return o;
}
}  // namespace dropin_detail

inline DenseVector allreduce_mean(const WorkerGroup& group, CollectiveAlgorithm algo, const Topology& topo) {
  const std::size_t dim = group.checked_dim();
  const auto a = dropin_detail::algo_of(algo);
  if (dim == 0) return DenseVector{};
  const parsim_b200::Topology t = dropin_detail::topo_of(topo);
  std::lock_guard<std::mutex> lk(parsim_dropin::lock());
  return parsim_dropin::device().allreduce_mean(group.buffers, a, &t);
}

inline DenseVector allreduce_mean(const WorkerGroup& group, CollectiveAlgorithm algo) {
  Topology flat;
  flat.devices_per_node = std::max<std::size_t>(group.size(), 1);
  return allreduce_mean(group, algo, flat);
}

}  // namespace parsim
