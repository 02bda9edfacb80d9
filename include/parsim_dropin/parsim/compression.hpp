// Drop-in for parsim/compression.hpp: the compressors, decompress and the
// error-feedback step on the GPU (f64 instantiations of the sm_100a kernels),
// with the reference's types (CompressedGradient and its payloads,
// ErrorFeedbackState, CompressorConfig) and error behaviour.  Wire codec and
// compression ratios stay the reference's own.  See numerics.hpp for usage.
//
//   compress_onebit   compression.hpp:67-77    sign bits exact; scale within
//                                              1e-12 rel (fixed-shape sum)
//   compress_topk     compression.hpp:81-99    bit-exact (radix select, ties
//                                              to the lower index)
//   compress          compression.hpp:101-111
//   decompress        compression.hpp:113-142  device scatter + validation
//   ef_compress_step  compression.hpp:146-157  fused K1 (top-k) / 1-bit EF
#pragma once

#include "parsim/numerics.hpp"

#define compress_onebit parsim_reference_compress_onebit
#define compress_topk parsim_reference_compress_topk
#define compress parsim_reference_compress
#define decompress parsim_reference_decompress
#define ef_compress_step parsim_reference_ef_compress_step
#include_next "parsim/compression.hpp"
#undef compress_onebit
#undef compress_topk
#undef compress
#undef decompress
#undef ef_compress_step

namespace parsim {

namespace dropin_detail {
inline CompressedGradient from_topk(parsim_b200::TopKMessage&& m) {
  TopKPayload p;
  p.dim = m.dim;
  p.indices = std::move(m.indices);
  p.values = std::move(m.values);
  return {p};
}
inline CompressedGradient from_signbit(parsim_b200::SignBitMessage&& m) {
  SignBitPayload p;
  p.dim = m.dim;
  p.scale = m.scale;
  p.sign_bytes = std::move(m.sign_bytes);
  return {p};
}
}  // namespace dropin_detail

inline CompressedGradient compress_onebit(const DenseVector& g) {
  detail::require(!g.empty(), "compress_onebit: empty vector");
  std::lock_guard<std::mutex> lk(parsim_dropin::lock());
  return dropin_detail::from_signbit(parsim_dropin::device().compress_onebit(g));
}

inline CompressedGradient compress_topk(const DenseVector& g, std::size_t k) {
  detail::require(k >= 1 && k <= g.size(), "compress_topk: k out of range (k=" + std::to_string(k) +
                                               ", dim=" + std::to_string(g.size()) + ")");
  std::lock_guard<std::mutex> lk(parsim_dropin::lock());
  return dropin_detail::from_topk(parsim_dropin::device().compress_topk(g, k));
}

inline CompressedGradient compress(const DenseVector& g, const CompressorConfig& cfg) {
  switch (cfg.kind) {
    case CompressorKind::none:
      return {DensePayload{g}};
    case CompressorKind::onebit:
      return compress_onebit(g);
    case CompressorKind::topk:
      return compress_topk(g, cfg.top_k);
  }
  detail::fail("compress: unknown compressor kind");
}

inline DenseVector decompress(const CompressedGradient& c) {
  if (const auto* d = std::get_if<DensePayload>(&c.payload)) return d->values;
  std::lock_guard<std::mutex> lk(parsim_dropin::lock());
  if (const auto* s = std::get_if<SignBitPayload>(&c.payload))
    return parsim_dropin::device().decompress_signbit(s->dim, s->scale, s->sign_bytes);
  const auto& t = std::get<TopKPayload>(c.payload);
  return parsim_dropin::device().decompress_topk(t.dim, t.indices, t.values);
}

inline CompressedGradient ef_compress_step(ErrorFeedbackState& state, const DenseVector& g,
                                           const CompressorConfig& cfg) {
  detail::require(state.residual.size() == g.size(), "ef_compress_step: residual/gradient dimension mismatch");
  switch (cfg.kind) {
    case CompressorKind::topk: {
      detail::require(cfg.top_k >= 1 && cfg.top_k <= g.size(),
                      "compress_topk: k out of range (k=" + std::to_string(cfg.top_k) + ", dim=" +
                          std::to_string(g.size()) + ")");
      std::lock_guard<std::mutex> lk(parsim_dropin::lock());
      parsim_b200::ErrorFeedbackState st{state.residual};
      auto m = parsim_dropin::device().ef_compress_step_topk(st, g, cfg.top_k);
      state.residual = std::move(st.residual);
      return dropin_detail::from_topk(std::move(m));
    }
    case CompressorKind::onebit: {
      detail::require(!g.empty(), "compress_onebit: empty vector");
      std::lock_guard<std::mutex> lk(parsim_dropin::lock());
      parsim_b200::ErrorFeedbackState st{state.residual};
      auto m = parsim_dropin::device().ef_compress_step_onebit(st, g);
      state.residual = std::move(st.residual);
      return dropin_detail::from_signbit(std::move(m));
    }
    case CompressorKind::none: {
      // p = r + g is the message; r' = p - p (+0, NaN for a non-finite p),
      // both as one-worker axpy passes on the device
      if (g.empty()) return {DensePayload{DenseVector{}}};
      DenseVector p = vec_axpy(1.0, g, state.residual);
      state.residual = vec_axpy(-1.0, p, p);  // the device pass raises on a non-finite entry
      return {DensePayload{std::move(p)}};
    }
  }
  detail::fail("compress: unknown compressor kind");
}

}  // namespace parsim
