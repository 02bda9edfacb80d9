// Drop-in for parsim/strategies.hpp: the data-parallel steps on the GPU.
// sync_data_parallel_step runs every worker's error-feedback compression
// (top-k: fused K1; 1-bit), the rank-ordered fold of the decompressed
// messages in the configured order and the SGD update as psb_sync_step --
// decompressed messages are never materialised.  async_step is the Eq. 12
// update.  StrategyConfig, HyperParams, StalenessTracker and the
// TP / PP / MoE parts stay the reference's own.  See numerics.hpp for usage.
//
//   sync_data_parallel_step(workers, params, h, cfg, topo, ef*)  strategies.hpp:86-113
//   sync_data_parallel_step(workers, params, h, cfg, ef*)        strategies.hpp:115-121
//   async_step(params, g, tau, eta)                              strategies.hpp:125-129
#pragma once

#include "parsim/collectives.hpp"
#include "parsim/compression.hpp"
#include "parsim/numerics.hpp"

#define sync_data_parallel_step parsim_reference_sync_data_parallel_step
#define async_step parsim_reference_async_step
#include_next "parsim/strategies.hpp"
#undef sync_data_parallel_step
#undef async_step

namespace parsim {

inline DenseVector sync_data_parallel_step(const WorkerGroup& workers, const DenseVector& params,
                                           const HyperParams& h, const StrategyConfig& cfg,
                                           const Topology& topo,
                                           std::vector<ErrorFeedbackState>* ef_states = nullptr) {
  const std::size_t dim = workers.checked_dim();
  detail::require(dim == params.size(), "sync_data_parallel_step: worker/param dim mismatch");
  if (cfg.compressor.kind != CompressorKind::none && ef_states != nullptr)
    detail::require(ef_states->size() == workers.size(),
                    "sync_data_parallel_step: one error-feedback state per worker required");
  if (dim == 0) return params;
  const auto kind = cfg.compressor.kind == CompressorKind::topk
                        ? parsim_b200::CompressorKind::topk
                        : (cfg.compressor.kind == CompressorKind::onebit ? parsim_b200::CompressorKind::onebit
                                                                         : parsim_b200::CompressorKind::none);
  const parsim_b200::Topology t = dropin_detail::topo_of(topo);
  std::lock_guard<std::mutex> lk(parsim_dropin::lock());
  std::vector<parsim_b200::ErrorFeedbackState> st;
  const bool ef = kind != parsim_b200::CompressorKind::none && ef_states != nullptr;
  if (ef)
    for (const auto& s : *ef_states) st.push_back({s.residual});
  DenseVector out = parsim_dropin::device().sync_data_parallel_step(
      workers.buffers, params, h.learning_rate, kind, cfg.compressor.top_k,
      dropin_detail::algo_of(cfg.collective), ef ? &st : nullptr, &t);
  if (ef)
    for (std::size_t p = 0; p < st.size(); ++p) (*ef_states)[p].residual = std::move(st[p].residual);
  return out;
}

inline DenseVector sync_data_parallel_step(const WorkerGroup& workers, const DenseVector& params,
                                           const HyperParams& h, const StrategyConfig& cfg,
                                           std::vector<ErrorFeedbackState>* ef_states = nullptr) {
  Topology flat;
  flat.devices_per_node = std::max<std::size_t>(workers.size(), 1);
  return sync_data_parallel_step(workers, params, h, cfg, flat, ef_states);
}

inline DenseVector async_step(const DenseVector& params, const DenseVector& g_p, std::size_t tau, double eta) {
  const double scale = eta / (1.0 + static_cast<double>(tau));
  return vec_axpy(-scale, g_p, params);
}

}  // namespace parsim
