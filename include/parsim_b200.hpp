// parsim_b200.hpp -- C++ drop-in facade for the reference's data-parallel
// gradient path, over the C ABI in psb.h.
//
// The reference (/root/reference/proj/include/parsim) is header-only C++ with
// host std::vector<double> in and out.  This header keeps those shapes and
// semantics for the hot-path functions and runs them on the GPU through
// libpsb.so in f64 -- bit-identical to the reference except the 1-bit scale
// (sign bits exact; scale = sum|g|/n as a fixed-shape device sum, within 1e-12
// relative of the reference's sequential fold, and the 1-bit residual with it;
// tests/test_facade_gpu.py).  The reference's own signatures, types and tests
// are served by the drop-in headers in include/parsim_dropin/ (built on this
// class):
//
//   compress_topk            parsim/compression.hpp:81-99
//   ef_compress_step (topk)  parsim/compression.hpp:146-157
//   compress_onebit, ef_compress_step (1-bit) parsim/compression.hpp:67-77, 146-157
//   decompress               parsim/compression.hpp:113-142
//   allreduce_mean           parsim/collectives.hpp:135-154
//   sync_data_parallel_step  parsim/strategies.hpp:86-121 (top-k / 1-bit / none)
//   async_step               parsim/strategies.hpp:125-129
//   vec_axpy                 parsim/numerics.hpp:70-78
//
// Precondition failures and non-finite results throw std::invalid_argument
// (as the reference's detail::require / check_finite); CUDA/NCCL failures
// throw std::runtime_error.  Link: -lpsb -lcudart.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "psb.h"

namespace parsim_b200 {

using DenseVector = std::vector<double>;

enum class CollectiveAlgorithm { naive, ring, hierarchical, pipelined_ring };
enum class CompressorKind { none, onebit, topk };

struct Topology {  // parsim/collectives.hpp:18-39 (grouping fields)
  std::size_t racks = 1, nodes_per_rack = 1, devices_per_node = 1;
};

struct TopKMessage {  // parsim/compression.hpp:42-46
  std::size_t dim = 0;
  std::vector<std::size_t> indices;
  DenseVector values;
};

struct SignBitMessage {  // parsim/compression.hpp:31-40
  std::size_t dim = 0;
  double scale = 0.0;
  std::vector<std::uint8_t> sign_bytes;
  bool positive_at(std::size_t i) const { return (sign_bytes[i / 8] >> (i % 8)) & 1u; }
};

struct ErrorFeedbackState {  // parsim/compression.hpp:58-62
  DenseVector residual;
  static ErrorFeedbackState zeros(std::size_t dim) { return {DenseVector(dim, 0.0)}; }
};

inline psb_order to_order(CollectiveAlgorithm a) {
  switch (a) {
    case CollectiveAlgorithm::naive: return PSB_ORDER_NAIVE;
    case CollectiveAlgorithm::hierarchical: return PSB_ORDER_HIER;
    default: return PSB_ORDER_RING;  // ring, pipelined_ring (collectives.hpp:142-143)
  }
}

// One device context: a psb_ctx, a stream and grow-only device buffers.
class Device {
 public:
  explicit Device(int device = 0, std::size_t max_n = 1 << 20, std::size_t max_k = 1 << 16,
                  int max_workers = 16)
      : dev_(device), max_n_(max_n), max_k_(max_k), max_w_(max_workers) {
    ck_cuda(cudaSetDevice(device), "cudaSetDevice");
    ck_cuda(cudaStreamCreate(&st_), "cudaStreamCreate");
    ck(psb_ctx_create(&ctx_, device, max_n, max_k, max_workers), "psb_ctx_create");
  }
  ~Device() {
    for (void* p : bufs_) cudaFree(p);
    if (ctx_) psb_ctx_destroy(ctx_);
    if (st_) cudaStreamDestroy(st_);
  }
  Device(const Device&) = delete;
  Device& operator=(const Device&) = delete;

  // compress_topk(g, k): k largest |g|, ties -> lower index, indices ascending.
  TopKMessage compress_topk(const DenseVector& g, std::size_t k) {
    require(k >= 1 && k <= g.size(), "compress_topk: k out of range (k=" + std::to_string(k) +
                                         ", dim=" + std::to_string(g.size()) + ")");
    fit(g.size(), k, 1);
    double* dg = upload(0, g);
    TopKMessage m = run_topk(dg, nullptr, g.size(), k);
    return m;
  }

  // ef_compress_step(state, g, {topk, k}).
  TopKMessage ef_compress_step_topk(ErrorFeedbackState& st, const DenseVector& g, std::size_t k) {
    require(st.residual.size() == g.size(), "ef_compress_step: residual/gradient dimension mismatch");
    require(k >= 1 && k <= g.size(), "compress_topk: k out of range (k=" + std::to_string(k) +
                                         ", dim=" + std::to_string(g.size()) + ")");
    fit(g.size(), k, 1);
    double* dg = upload(0, g);
    double* dr = upload(1, st.residual);
    TopKMessage m = run_topk(dg, dr, g.size(), k);
    download(dr, st.residual);
    return m;
  }

  // compress_onebit(g): sign bits (sign(0) = +1) and scale = sum|g| / n.
  SignBitMessage compress_onebit(const DenseVector& g) {
    require(!g.empty(), "compress_onebit: empty vector");
    fit(g.size(), 1, 1);
    double* dg = upload(0, g);
    return run_onebit(dg, nullptr, g.size());
  }

  // decompress(TopKPayload) on the device: zeros + scatter, with the
  // reference's index validation (compression.hpp:127-140) raised from the
  // device as std::invalid_argument.
  DenseVector decompress_topk(std::size_t dim, const std::vector<std::size_t>& indices, const DenseVector& values) {
    require(indices.size() == values.size(), "decompress: index/value count mismatch");
    for (std::size_t j = 0; j < indices.size(); ++j)  // beyond the device's u32 indices: out of range anyway
      require(indices[j] < dim && indices[j] <= 0xffffffffull,
              "decompress: index " + std::to_string(indices[j]) + " out of range for dim " + std::to_string(dim));
    DenseVector out(dim, 0.0);
    if (dim == 0 || indices.empty()) return out;
    fit(dim, indices.size(), 1);
    std::vector<uint32_t> i32(indices.begin(), indices.end());
    uint32_t* di = static_cast<uint32_t*>(buf(4, i32.size() * 4));
    ck_cuda(cudaMemcpy(di, i32.data(), i32.size() * 4, cudaMemcpyHostToDevice), "cudaMemcpy");
    double* dv = upload(5, values);
    double* dout = static_cast<double*>(buf(1, dim * sizeof(double)));
    ck_cuda(cudaMemsetAsync(dout, 0, dim * sizeof(double), st_), "cudaMemsetAsync");
    ck(psb_decompress_topk(ctx_, PSB_F64, di, dv, i32.size(), dim, dout, st_), "decompress");
    check();
    download(dout, out);
    return out;
  }

  // decompress(SignBitPayload): +-scale per sign bit, through the 1-bit mean
  // kernel with one worker (mean = value * (1/1)).
  DenseVector decompress_signbit(std::size_t dim, double scale, const std::vector<std::uint8_t>& sign_bytes) {
    require(sign_bytes.size() == (dim + 7) / 8, "decompress: sign byte count does not match dim");
    DenseVector out(dim);
    if (dim == 0) return out;
    fit(dim, 1, 1);
    const std::size_t nw = (dim + 31) / 32;
    std::vector<uint32_t> words(nw, 0u);
    std::memcpy(words.data(), sign_bytes.data(), sign_bytes.size());
    uint32_t* dw = static_cast<uint32_t*>(buf(2, nw * 4));
    ck_cuda(cudaMemcpy(dw, words.data(), nw * 4, cudaMemcpyHostToDevice), "cudaMemcpy");
    double* ds = static_cast<double*>(buf(3, sizeof(double)));
    ck_cuda(cudaMemcpy(ds, &scale, sizeof(double), cudaMemcpyHostToDevice), "cudaMemcpy");
    double* dout = static_cast<double*>(buf(1, dim * sizeof(double)));
    psb_topology t{0, 0, 0};
    ck(psb_onebit_mean_sgd(ctx_, PSB_F64, 1, dw, ds, PSB_ORDER_NAIVE, &t, 0.0, nullptr, dim, dout, st_),
       "decompress");
    check();
    download(dout, out);
    return out;
  }

  // ef_compress_step(state, g, {onebit}).
  SignBitMessage ef_compress_step_onebit(ErrorFeedbackState& st, const DenseVector& g) {
    require(!g.empty(), "compress_onebit: empty vector");
    require(st.residual.size() == g.size(), "ef_compress_step: residual/gradient dimension mismatch");
    fit(g.size(), 1, 1);
    double* dg = upload(0, g);
    double* dr = upload(1, st.residual);
    SignBitMessage m = run_onebit(dg, dr, g.size());
    download(dr, st.residual);
    return m;
  }

  // allreduce_mean(group, algo[, topo]).
  DenseVector allreduce_mean(const std::vector<DenseVector>& group, CollectiveAlgorithm algo,
                             const Topology* topo = nullptr) {
    require(!group.empty(), "WorkerGroup: no workers");
    const std::size_t n = group[0].size();
    for (const auto& b : group) require(b.size() == n, "WorkerGroup: dim mismatch across workers");
    fit(n, 1, (int)group.size());
    double* bufs = upload_rows(0, group);
    double* mean = static_cast<double*>(buf(1, n * sizeof(double)));
    psb_topology t = topo_of(topo, group.size());
    ck(psb_dense_mean_sgd(ctx_, PSB_F64, (int)group.size(), bufs, to_order(algo), &t, 1.0, nullptr, n,
                          mean, st_),
       "allreduce_mean");
    check();
    DenseVector out(n);
    download(mean, out);
    return out;
  }

  // sync_data_parallel_step(workers, params, h, cfg[, topo], ef_states).
  // residuals == nullptr: transient zero residuals (strategies.hpp:97-102).
  DenseVector sync_data_parallel_step(const std::vector<DenseVector>& workers, const DenseVector& params,
                                      double lr, CompressorKind kind, std::size_t top_k,
                                      CollectiveAlgorithm algo, std::vector<ErrorFeedbackState>* residuals,
                                      const Topology* topo = nullptr) {
    require(!workers.empty(), "WorkerGroup: no workers");
    const std::size_t n = workers[0].size(), P = workers.size();
    for (const auto& b : workers) require(b.size() == n, "WorkerGroup: dim mismatch across workers");
    require(n == params.size(), "sync_data_parallel_step: worker/param dim mismatch");
    if (kind != CompressorKind::none && residuals)
      require(residuals->size() == P, "sync_data_parallel_step: one error-feedback state per worker required");
    fit(n, kind == CompressorKind::topk ? top_k : 1, (int)P);
    double* dg = upload_rows(0, workers);
    double* dth = upload(1, params);
    double* dr = nullptr;
    if (kind != CompressorKind::none) {
      std::vector<DenseVector> rows;
      if (residuals)
        for (auto& s : *residuals) rows.push_back(s.residual);
      else
        rows.assign(P, DenseVector(n, 0.0));
      dr = upload_rows(2, rows);
    }
    psb_step_desc d{};
    d.compressor = kind == CompressorKind::topk ? PSB_COMP_TOPK
                                                 : (kind == CompressorKind::onebit ? PSB_COMP_ONEBIT : PSB_COMP_NONE);
    d.dtype = PSB_F64;
    d.n = n;
    d.k = top_k;
    d.workers = (int)P;
    d.g = dg;
    d.r = dr;
    d.theta = dth;
    d.lr = lr;
    d.order = to_order(algo);
    d.topo = topo_of(topo, P);
    ck(psb_sync_step(ctx_, &d, st_), "sync_data_parallel_step");
    check();
    DenseVector out(n);
    download(dth, out);
    if (residuals && dr) {
      for (std::size_t p = 0; p < P; ++p)
        ck_cuda(cudaMemcpy((*residuals)[p].residual.data(), dr + p * n, n * sizeof(double),
                           cudaMemcpyDeviceToHost),
                "cudaMemcpy");
    }
    return out;
  }

  // vec_axpy(a, x, y) = a*x + y with a separate multiply and add.
  DenseVector vec_axpy(double a, const DenseVector& x, const DenseVector& y) {
    require(x.size() == y.size(), "vec_axpy: dimension mismatch (" + std::to_string(x.size()) + " vs " +
                                      std::to_string(y.size()) + ")");
    fit(x.size(), 1, 1);
    double* dx = upload(0, x);
    double* dy = upload(1, y);
    psb_topology t{0, 0, 0};
    ck(psb_dense_mean_sgd(ctx_, PSB_F64, 1, dx, PSB_ORDER_NAIVE, &t, -a, dy, x.size(), nullptr, st_),
       "vec_axpy");
    check("vec_axpy: non-finite entry");
    DenseVector out(x.size());
    download(dy, out);
    return out;
  }

  // async_step(params, g, tau, eta) = vec_axpy(-eta/(1+tau), g, params).
  DenseVector async_step(const DenseVector& params, const DenseVector& g, std::size_t tau, double eta) {
    const double scale = eta / (1.0 + static_cast<double>(tau));
    return vec_axpy(-scale, g, params);
  }

  psb_ctx* ctx() { return ctx_; }

 private:
  static void require(bool ok, const std::string& msg) {
    if (!ok) throw std::invalid_argument(msg);
  }
  void ck(psb_status s, const char* where) {
    if (s == PSB_OK) return;
    const std::string msg = std::string(where) + ": " + (ctx_ ? psb_last_error(ctx_) : psb_status_string(s));
    if (s == PSB_EINVAL || s == PSB_ENONFINITE) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
  }
  static void ck_cuda(cudaError_t e, const char* where) {
    if (e != cudaSuccess) throw std::runtime_error(std::string(where) + ": " + cudaGetErrorString(e));
  }
  void check(const char* nonfinite_msg = nullptr) {
    psb_status s = psb_check(ctx_, st_);
    if (s == PSB_ENONFINITE && nonfinite_msg) throw std::invalid_argument(nonfinite_msg);
    ck(s, "psb_check");
  }
  void fit(std::size_t n, std::size_t k, int w) {
    if (n <= max_n_ && k <= max_k_ && w <= max_w_) return;
    psb_ctx_destroy(ctx_);
    ctx_ = nullptr;
    max_n_ = std::max(n, max_n_);
    max_k_ = std::max(k, max_k_);
    max_w_ = std::max(w, max_w_);
    ck(psb_ctx_create(&ctx_, dev_, max_n_, max_k_, max_w_), "psb_ctx_create");
  }
  void* buf(int slot, std::size_t bytes) {
    if ((int)bufs_.size() <= slot) {
      bufs_.resize(slot + 1, nullptr);
      caps_.resize(slot + 1, 0);
    }
    if (caps_[slot] < bytes) {
      if (bufs_[slot]) cudaFree(bufs_[slot]);
      ck_cuda(cudaMalloc(&bufs_[slot], bytes), "cudaMalloc");
      caps_[slot] = bytes;
    }
    return bufs_[slot];
  }
  double* upload(int slot, const DenseVector& v) {
    double* d = static_cast<double*>(buf(slot, std::max<std::size_t>(1, v.size()) * sizeof(double)));
    ck_cuda(cudaMemcpy(d, v.data(), v.size() * sizeof(double), cudaMemcpyHostToDevice), "cudaMemcpy");
    return d;
  }
  double* upload_rows(int slot, const std::vector<DenseVector>& rows) {
    const std::size_t n = rows.empty() ? 0 : rows[0].size();
    double* d = static_cast<double*>(buf(slot, std::max<std::size_t>(1, rows.size() * n) * sizeof(double)));
    for (std::size_t p = 0; p < rows.size(); ++p)
      ck_cuda(cudaMemcpy(d + p * n, rows[p].data(), n * sizeof(double), cudaMemcpyHostToDevice), "cudaMemcpy");
    return d;
  }
  void download(const double* d, DenseVector& v) {
    ck_cuda(cudaMemcpy(v.data(), d, v.size() * sizeof(double), cudaMemcpyDeviceToHost), "cudaMemcpy");
  }
  static psb_topology topo_of(const Topology* t, std::size_t P) {
    if (!t) return psb_topology{0, 0, 0};  // flat: devices_per_node = P (collectives.hpp:150-154)
    (void)P;
    return psb_topology{(uint32_t)t->racks, (uint32_t)t->nodes_per_rack, (uint32_t)t->devices_per_node};
  }
  SignBitMessage run_onebit(double* dg, double* dr, std::size_t n) {
    const std::size_t nw = (n + 31) / 32;
    uint32_t* words = static_cast<uint32_t*>(buf(2, nw * 4));
    double* scale = static_cast<double*>(buf(3, sizeof(double)));
    ck(psb_ef_onebit(ctx_, PSB_F64, dg, dr, n, words, scale, st_), "ef_compress_step");
    check();
    SignBitMessage m;
    m.dim = n;
    std::vector<uint32_t> hw(nw);
    ck_cuda(cudaMemcpy(hw.data(), words, nw * 4, cudaMemcpyDeviceToHost), "cudaMemcpy");
    m.sign_bytes.resize((n + 7) / 8);
    std::memcpy(m.sign_bytes.data(), hw.data(), m.sign_bytes.size());
    ck_cuda(cudaMemcpy(&m.scale, scale, sizeof(double), cudaMemcpyDeviceToHost), "cudaMemcpy");
    return m;
  }
  TopKMessage run_topk(double* dg, double* dr, std::size_t n, std::size_t k) {
    uint32_t* idx = static_cast<uint32_t*>(buf(4, k * 4));
    double* val = static_cast<double*>(buf(5, k * sizeof(double)));
    ck(psb_ef_topk(ctx_, PSB_F64, 0, dg, dr, n, k, idx, val, st_), "ef_compress_step");
    check();
    TopKMessage m;
    m.dim = n;
    std::vector<uint32_t> hi(k);
    m.values.resize(k);
    ck_cuda(cudaMemcpy(hi.data(), idx, k * 4, cudaMemcpyDeviceToHost), "cudaMemcpy");
    ck_cuda(cudaMemcpy(m.values.data(), val, k * sizeof(double), cudaMemcpyDeviceToHost), "cudaMemcpy");
    m.indices.assign(hi.begin(), hi.end());
    return m;
  }

  int dev_;
  std::size_t max_n_, max_k_;
  int max_w_;
  cudaStream_t st_ = nullptr;
  psb_ctx* ctx_ = nullptr;
  std::vector<void*> bufs_;
  std::vector<std::size_t> caps_;
};

}  // namespace parsim_b200
