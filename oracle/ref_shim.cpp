// ref_shim.cpp -- extern "C" entry points into the UNMODIFIED reference headers.
//
// TEST INFRASTRUCTURE ONLY (see oracle/psb_oracle.c header).  This file holds
// no reference source: it #includes the reference's own headers from the path
// given on the command line (oracle/Makefile, REF_INCLUDE, default
// /root/reference/proj/include) and exposes the hot-path functions over plain
// pointers so tests/ and bench.py (reference arm, cpu_baseline) can call the
// reference implementation itself.  Output: oracle/_ref/libparsim_ref.so.
//
// Functions wrapped (all in namespace parsim):
//   compress_topk        parsim/compression.hpp:81-99
//   compress_onebit      parsim/compression.hpp:67-77
//   ef_compress_step     parsim/compression.hpp:146-157
//   decompress           parsim/compression.hpp:113-142
//   allreduce_mean       parsim/collectives.hpp:135-154
//   sync_data_parallel_step  parsim/strategies.hpp:86-113
//   async_step           parsim/strategies.hpp:125-129
//   vec_axpy             parsim/numerics.hpp:70-78
//   SeededRng            parsim/numerics.hpp:152-178
//   wire_encode / wire_decode  parsim/compression.hpp:188-239
//   bpr_batch_gradient / bpr_batch_loss  parsim/trainer.hpp:98-138

#include <cstring>
#include <exception>
#include <thread>
#include <vector>

#include "parsim/collectives.hpp"
#include "parsim/compression.hpp"
#include "parsim/numerics.hpp"
#include "parsim/strategies.hpp"
#include "parsim/trainer.hpp"

using namespace parsim;

namespace {
thread_local char g_err[512];

int fail_with(const std::exception& e) {
  std::strncpy(g_err, e.what(), sizeof(g_err) - 1);
  g_err[sizeof(g_err) - 1] = 0;
  return 1;
}

CompressorConfig make_cfg(int kind, std::size_t k) {
  CompressorConfig c;
  c.kind = kind == 0 ? CompressorKind::none : (kind == 1 ? CompressorKind::onebit : CompressorKind::topk);
  c.top_k = k;
  return c;
}

CollectiveAlgorithm make_algo(int a) {
  switch (a) {
    case 0: return CollectiveAlgorithm::naive;
    case 1: return CollectiveAlgorithm::ring;
    case 2: return CollectiveAlgorithm::hierarchical;
    default: return CollectiveAlgorithm::pipelined_ring;
  }
}

Topology make_topo(std::size_t racks, std::size_t npr, std::size_t dpn) {
  Topology t;
  t.racks = racks;
  t.nodes_per_rack = npr;
  t.devices_per_node = dpn;
  return t;
}

// Message -> flat outputs.  For top-k: idx/val arrays of length k.  For
// onebit: sign bytes + scale.  For none: dense values in val.
void export_msg(const CompressedGradient& m, std::uint64_t* idx, double* val, std::uint8_t* sign_bytes,
                double* scale, std::size_t* count) {
  if (auto* t = std::get_if<TopKPayload>(&m.payload)) {
    for (std::size_t j = 0; j < t->indices.size(); ++j) {
      if (idx) idx[j] = t->indices[j];
      if (val) val[j] = t->values[j];
    }
    if (count) *count = t->indices.size();
  } else if (auto* s = std::get_if<SignBitPayload>(&m.payload)) {
    if (sign_bytes) std::memcpy(sign_bytes, s->sign_bytes.data(), s->sign_bytes.size());
    if (scale) *scale = s->scale;
    if (count) *count = s->sign_bytes.size();
  } else {
    auto& d = std::get<DensePayload>(m.payload);
    if (val) std::memcpy(val, d.values.data(), d.values.size() * sizeof(double));
    if (count) *count = d.values.size();
  }
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err; }

int ref_splitmix_stream(std::uint64_t seed, std::size_t n, std::uint64_t* out) {
  SeededRng r(seed);
  for (std::size_t i = 0; i < n; ++i) out[i] = r.next_u64();
  return 0;
}

// SeededRng::uniform(lo, hi) stream, used to regenerate the reference tests'
// own inputs (e.g. acceptance.cpp:133-170, test_compression.cpp:118-135).
int ref_uniform_stream(std::uint64_t seed, std::size_t n, double lo, double hi, double* out) {
  SeededRng r(seed);
  for (std::size_t i = 0; i < n; ++i) out[i] = r.uniform(lo, hi);
  return 0;
}

int ref_compress_topk(const double* g, std::size_t n, std::size_t k, std::uint64_t* idx, double* val) {
  try {
    DenseVector v(g, g + n);
    export_msg(compress_topk(v, k), idx, val, nullptr, nullptr, nullptr);
    return 0;
  } catch (const std::exception& e) {
    return fail_with(e);
  }
}

int ref_compress_onebit(const double* g, std::size_t n, std::uint8_t* sign_bytes, double* scale) {
  try {
    DenseVector v(g, g + n);
    export_msg(compress_onebit(v), nullptr, nullptr, sign_bytes, scale, nullptr);
    return 0;
  } catch (const std::exception& e) {
    return fail_with(e);
  }
}

// One ef_compress_step; residual is in/out.  kind: 0 none, 1 onebit, 2 topk.
// Outputs: topk -> idx/val (k entries); onebit -> sign_bytes/scale; none -> val (n).
int ref_ef_compress_step(int kind, std::size_t k, double* residual, const double* g, std::size_t n,
                         std::uint64_t* idx, double* val, std::uint8_t* sign_bytes, double* scale) {
  try {
    ErrorFeedbackState st{DenseVector(residual, residual + n)};
    DenseVector v(g, g + n);
    auto msg = ef_compress_step(st, v, make_cfg(kind, k));
    std::memcpy(residual, st.residual.data(), n * sizeof(double));
    export_msg(msg, idx, val, sign_bytes, scale, nullptr);
    return 0;
  } catch (const std::exception& e) {
    return fail_with(e);
  }
}

// bufs: P rows of n.  algo: 0 naive 1 ring 2 hierarchical 3 pipelined_ring.
int ref_allreduce_mean(int algo, std::size_t P, const double* bufs, std::size_t n, std::size_t racks,
                       std::size_t npr, std::size_t dpn, double* out) {
  try {
    WorkerGroup wg;
    for (std::size_t p = 0; p < P; ++p) wg.buffers.emplace_back(bufs + p * n, bufs + (p + 1) * n);
    DenseVector m = dpn == 0 ? allreduce_mean(wg, make_algo(algo))
                             : allreduce_mean(wg, make_algo(algo), make_topo(racks, npr, dpn));
    std::memcpy(out, m.data(), n * sizeof(double));
    return 0;
  } catch (const std::exception& e) {
    return fail_with(e);
  }
}

// sync_data_parallel_step.  params in/out.  residuals: P rows of n (in/out),
// or nullptr for "no error-feedback state" (strategies.hpp:97-102).
// dpn == 0 selects the no-topology overload (strategies.hpp:115-121).
// threads > 1 runs the per-worker ef_compress_step calls of the step on
// worker threads (SPEC.md:238 allows it; the fold stays serial), used only by
// bench.py's reference arm as the "P cores" variant.
int ref_sync_step(int kind, std::size_t k, int algo, std::size_t P, const double* grads, double* params,
                  std::size_t n, double lr, double* residuals, std::size_t racks, std::size_t npr,
                  std::size_t dpn) {
  try {
    WorkerGroup wg;
    for (std::size_t p = 0; p < P; ++p) wg.buffers.emplace_back(grads + p * n, grads + (p + 1) * n);
    DenseVector theta(params, params + n);
    HyperParams h;
    h.learning_rate = lr;
    StrategyConfig cfg;
    cfg.data_degree = P;
    cfg.collective = make_algo(algo);
    cfg.compressor = make_cfg(kind, k);
    std::vector<ErrorFeedbackState> ef;
    if (residuals) {
      for (std::size_t p = 0; p < P; ++p)
        ef.push_back(ErrorFeedbackState{DenseVector(residuals + p * n, residuals + (p + 1) * n)});
    }
    DenseVector out = dpn == 0
                          ? sync_data_parallel_step(wg, theta, h, cfg, residuals ? &ef : nullptr)
                          : sync_data_parallel_step(wg, theta, h, cfg, make_topo(racks, npr, dpn),
                                                    residuals ? &ef : nullptr);
    std::memcpy(params, out.data(), n * sizeof(double));
    if (residuals) {
      for (std::size_t p = 0; p < P; ++p)
        std::memcpy(residuals + p * n, ef[p].residual.data(), n * sizeof(double));
    }
    return 0;
  } catch (const std::exception& e) {
    return fail_with(e);
  }
}

// Same step with the P ef_compress_step calls spread over `threads` host
// threads, then the reference's own decompress + allreduce_mean + vec_axpy,
// serially, in the reference order (strategies.hpp:105-112).  Reference
// functions only; this is the "all host threads" reference arm.
int ref_sync_step_threaded(int kind, std::size_t k, int algo, std::size_t P, const double* grads,
                           double* params, std::size_t n, double lr, double* residuals, int threads) {
  try {
    std::vector<ErrorFeedbackState> ef(P);
    std::vector<CompressedGradient> msgs(P);
    for (std::size_t p = 0; p < P; ++p)
      ef[p].residual.assign(residuals + p * n, residuals + (p + 1) * n);
    CompressorConfig cc = make_cfg(kind, k);
    std::vector<std::thread> pool;
    std::vector<std::string> errs(P);
    int T = threads < 1 ? 1 : threads;
    for (int t = 0; t < T; ++t) {
      pool.emplace_back([&, t]() {
        for (std::size_t p = (std::size_t)t; p < P; p += (std::size_t)T) {
          try {
            DenseVector g(grads + p * n, grads + (p + 1) * n);
            msgs[p] = ef_compress_step(ef[p], g, cc);
          } catch (const std::exception& e) {
            errs[p] = e.what();
          }
        }
      });
    }
    for (auto& th : pool) th.join();
    for (auto& e : errs)
      if (!e.empty()) throw std::invalid_argument(e);
    WorkerGroup dec;
    for (std::size_t p = 0; p < P; ++p) dec.buffers.push_back(decompress(msgs[p]));
    DenseVector mean = allreduce_mean(dec, make_algo(algo));
    DenseVector theta(params, params + n);
    DenseVector out = vec_axpy(-lr, mean, theta);
    std::memcpy(params, out.data(), n * sizeof(double));
    for (std::size_t p = 0; p < P; ++p)
      std::memcpy(residuals + p * n, ef[p].residual.data(), n * sizeof(double));
    return 0;
  } catch (const std::exception& e) {
    return fail_with(e);
  }
}

int ref_async_step(const double* params, const double* g, std::size_t n, std::size_t tau, double eta,
                   double* out) {
  try {
    DenseVector t(params, params + n), gg(g, g + n);
    DenseVector o = async_step(t, gg, tau, eta);
    std::memcpy(out, o.data(), n * sizeof(double));
    return 0;
  } catch (const std::exception& e) {
    return fail_with(e);
  }
}

int ref_vec_axpy(double a, const double* x, const double* y, std::size_t n, double* out) {
  try {
    DenseVector xx(x, x + n), yy(y, y + n);
    DenseVector o = vec_axpy(a, xx, yy);
    std::memcpy(out, o.data(), n * sizeof(double));
    return 0;
  } catch (const std::exception& e) {
    return fail_with(e);
  }
}

// decompress of a top-k payload (compression.hpp:113-142), including its
// validation (out-of-range / unsorted indices -> invalid_argument).
int ref_decompress_topk(std::size_t dim, const std::uint64_t* idx, const double* val, std::size_t k,
                        double* out) {
  try {
    TopKPayload t;
    t.dim = dim;
    t.indices.assign(idx, idx + k);
    t.values.assign(val, val + k);
    DenseVector o = decompress(CompressedGradient{t});
    std::memcpy(out, o.data(), dim * sizeof(double));
    return 0;
  } catch (const std::exception& e) {
    return fail_with(e);
  }
}

}  // extern "C"

// wire_encode of a TopKPayload{dim, idx, val} (parsim/compression.hpp:188-209);
// returns the byte count (out may be null to query it).
extern "C" size_t ref_wire_encode_topk(uint64_t dim, const uint64_t* idx, const double* val, size_t k, uint8_t* out) {
  TopKPayload t;
  t.dim = dim;
  t.indices.assign(idx, idx + k);
  t.values.assign(val, val + k);
  const std::vector<std::uint8_t> w = wire_encode(CompressedGradient{t});
  if (out) std::memcpy(out, w.data(), w.size());
  return w.size();
}

// wire_decode(topk) (parsim/compression.hpp:213-239): count, or -1 with the
// reference's message in ref_last_error() on truncated input.
extern "C" long long ref_wire_decode_topk(const uint8_t* in, size_t nbytes, uint64_t* dim, uint64_t* idx,
                                          double* val) {
  try {
    const std::vector<std::uint8_t> w(in, in + nbytes);
    const CompressedGradient c = wire_decode(WireKind::topk, w);
    const auto& t = std::get<TopKPayload>(c.payload);
    *dim = t.dim;
    if (idx && val)
      for (std::size_t j = 0; j < t.indices.size(); ++j) {
        idx[j] = t.indices[j];
        val[j] = t.values[j];
      }
    return (long long)t.indices.size();
  } catch (const std::exception& e) {
    fail_with(e);
    return -1;
  }
}

// wire_encode of a SignBitPayload built by compress_onebit(g) (compression.hpp:67-77).
extern "C" size_t ref_wire_encode_onebit(const double* g, size_t n, uint8_t* out) {
  const DenseVector x(g, g + n);
  const std::vector<std::uint8_t> w = wire_encode(compress_onebit(x));
  if (out) std::memcpy(out, w.data(), w.size());
  return w.size();
}

// bpr_batch_gradient + bpr_batch_loss on flat f64 theta (trainer.hpp:98-138).
extern "C" int ref_bpr_batch_gradient(const double* theta, size_t users, size_t items, size_t dim,
                                      const uint32_t* u, const uint32_t* p, const uint32_t* q, size_t B,
                                      double* grad_out, double* loss_out) {
  try {
    const DenseVector th(theta, theta + (users + items) * dim);
    std::vector<BprTriple> batch(B);
    for (size_t t = 0; t < B; ++t) batch[t] = {u[t], p[t], q[t]};
    const DenseVector g = bpr_batch_gradient(th, users, items, dim, batch);
    std::memcpy(grad_out, g.data(), g.size() * sizeof(double));
    if (loss_out) *loss_out = bpr_batch_loss(th, users, items, dim, batch);
    return 0;
  } catch (const std::exception& e) {
    return fail_with(e);
  }
}

// The reference's data-parallel trainer (trainer.hpp:197-261) on a given
// train split: RecModel::init(users, items, dim, seed), then `steps` steps of
// `mode` (0 sync, 1 async); returns the final flat theta and the loss curve
// (step, loss) every 100 steps (curve_out: 2 doubles per point, up to cap).
extern "C" int ref_train(size_t users, size_t items, size_t dim, const uint64_t* tu, const uint64_t* ti, size_t ntrain,
                         size_t P, int mode, size_t steps, size_t batch, double lr, int kind, size_t k, int algo,
                         uint64_t seed, uint64_t init_seed, double* theta_out, double* curve_out, size_t curve_cap,
                         size_t* curve_n) {
  try {
    ChronoSplit split;
    for (size_t i = 0; i < ntrain; ++i) split.train.push_back({tu[i], ti[i], (std::int64_t)i});
    StrategyConfig cfg;
    cfg.data_degree = P;
    cfg.mode = mode ? ExecutionMode::async : ExecutionMode::sync;
    cfg.collective = make_algo(algo);
    cfg.compressor = make_cfg(kind, k);
    HyperParams h;
    h.learning_rate = lr;
    h.batch_size = batch;
    h.steps = steps;
    TrainResult r = train(RecModel::init(users, items, dim, init_seed), split, cfg, h, seed);
    const DenseVector th = flatten_params(r.model);
    std::memcpy(theta_out, th.data(), th.size() * sizeof(double));
    size_t m = 0;
    for (const auto& pt : r.loss_curve) {
      if (m >= curve_cap) break;
      curve_out[2 * m] = (double)pt.first;
      curve_out[2 * m + 1] = pt.second;
      ++m;
    }
    *curve_n = m;
    return 0;
  } catch (const std::exception& e) {
    return fail_with(e);
  }
}

// evaluate_topk (trainer.hpp:269-324) of a flat theta on given splits.
extern "C" int ref_evaluate_topk(size_t users, size_t items, size_t dim, const double* theta, const uint64_t* tu,
                                 const uint64_t* ti, size_t ntrain, const uint64_t* vu, const uint64_t* vi, size_t nval,
                                 const uint64_t* su, const uint64_t* si, size_t ntest, size_t K, size_t negatives,
                                 uint64_t seed, double* out4) {
  try {
    RecModel m = RecModel::init(users, items, dim, 1);
    unflatten_params(DenseVector(theta, theta + (users + items) * dim), m);
    ChronoSplit split;
    for (size_t i = 0; i < ntrain; ++i) split.train.push_back({tu[i], ti[i], (std::int64_t)i});
    for (size_t i = 0; i < nval; ++i) split.validation.push_back({vu[i], vi[i], (std::int64_t)i});
    for (size_t i = 0; i < ntest; ++i) split.test.push_back({su[i], si[i], (std::int64_t)i});
    const EvalResult r = evaluate_topk(m, split, K, negatives, seed);
    out4[0] = r.hr_at_10;
    out4[1] = r.ndcg_at_10;
    out4[2] = (double)r.num_eval_users;
    out4[3] = (double)r.skipped;
    return 0;
  } catch (const std::exception& e) {
    return fail_with(e);
  }
}

// generate_synthetic + chrono_split (dataset.hpp:115-176): the split's
// (user, item) columns; sizes in n3[3] (train, validation, test).
extern "C" int ref_synthetic_split(size_t users, size_t items, size_t interactions, uint64_t seed, uint64_t* tu,
                                   uint64_t* ti, uint64_t* vu, uint64_t* vi, uint64_t* su, uint64_t* si, size_t* n3) {
  try {
    const ChronoSplit sp = chrono_split(generate_synthetic(users, items, interactions, seed));
    auto put = [](const std::vector<Interaction>& v, uint64_t* u, uint64_t* i) {
      for (size_t j = 0; j < v.size(); ++j) {
        u[j] = v[j].user;
        i[j] = v[j].item;
      }
    };
    put(sp.train, tu, ti);
    put(sp.validation, vu, vi);
    put(sp.test, su, si);
    n3[0] = sp.train.size();
    n3[1] = sp.validation.size();
    n3[2] = sp.test.size();
    return 0;
  } catch (const std::exception& e) {
    return fail_with(e);
  }
}

// load_model (trainer.hpp:351-378) of a file: dims into dims3, flat theta out.
extern "C" int ref_load_model(const char* path, size_t* dims3, double* theta_out, size_t cap) {
  try {
    const RecModel m = load_model(path);
    dims3[0] = m.num_users();
    dims3[1] = m.num_items();
    dims3[2] = m.embedding_dim();
    const DenseVector th = flatten_params(m);
    if (th.size() > cap) return fail_with(std::invalid_argument("ref_load_model: capacity"));
    std::memcpy(theta_out, th.data(), th.size() * sizeof(double));
    return 0;
  } catch (const std::exception& e) {
    return fail_with(e);
  }
}

// comm_cost (collectives.hpp:184-215) on a topology given as 3 counts + 6
// link figures {intra_bw, inter_bw, rack_bw, intra_lat, inter_lat, rack_lat}.
extern "C" int ref_comm_cost(int algo, double msg_bytes, size_t P, const size_t* counts3, const double* links6,
                             size_t span_devices, double* out) {
  try {
    Topology t = make_topo(counts3[0], counts3[1], counts3[2]);
    t.intra_node_bw = links6[0];
    t.inter_node_bw = links6[1];
    t.inter_rack_bw = links6[2];
    t.intra_node_lat = links6[3];
    t.inter_node_lat = links6[4];
    t.inter_rack_lat = links6[5];
    *out = comm_cost(static_cast<CollectiveAlgorithm>(algo), msg_bytes, P, t, span_devices);
    return 0;
  } catch (const std::exception& e) {
    return fail_with(e);
  }
}
