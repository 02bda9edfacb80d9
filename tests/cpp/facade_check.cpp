// facade_check.cpp -- drives include/parsim_b200.hpp (the C++ drop-in facade)
// on inputs written by tests/test_facade_gpu.py and writes the results back,
// so the test can compare them with the f64 oracle (pinned to the reference).
//
// usage: facade_check <dir>
//   in:  <dir>/g.bin (P x n f64), <dir>/meta.txt ("P n k steps lr")
//   out: <dir>/topk_idx.bin, topk_val.bin, ef_res.bin, mean_<algo>.bin,
//        sync_theta.bin, sync_res.bin, onebit.bin, async.bin, errors.txt
#include <cstdio>
#include <fstream>
#include <string>
#include <vector>

#include "parsim_b200.hpp"

using namespace parsim_b200;

static std::vector<double> read_f64(const std::string& f, std::size_t count) {
  std::vector<double> v(count);
  std::ifstream in(f, std::ios::binary);
  in.read(reinterpret_cast<char*>(v.data()), count * sizeof(double));
  return v;
}
template <class T>
static void write_bin(const std::string& f, const std::vector<T>& v) {
  std::ofstream out(f, std::ios::binary);
  out.write(reinterpret_cast<const char*>(v.data()), v.size() * sizeof(T));
}

int main(int argc, char** argv) {
  if (argc < 2) return 2;
  const std::string dir = argv[1];
  std::size_t P, n, k, steps;
  double lr;
  {
    std::ifstream m(dir + "/meta.txt");
    m >> P >> n >> k >> steps >> lr;
  }
  std::vector<double> all = read_f64(dir + "/g.bin", P * n * steps);
  auto grad = [&](std::size_t s, std::size_t p) {
    return DenseVector(all.begin() + (s * P + p) * n, all.begin() + (s * P + p + 1) * n);
  };
  Device dev(0, n, k, (int)P);

  // compress_topk on worker 0, step 0
  TopKMessage t = dev.compress_topk(grad(0, 0), k);
  write_bin(dir + "/topk_idx.bin", std::vector<unsigned long long>(t.indices.begin(), t.indices.end()));
  write_bin(dir + "/topk_val.bin", t.values);

  // ef_compress_step (topk) over all steps on worker 1
  ErrorFeedbackState st = ErrorFeedbackState::zeros(n);
  std::vector<double> idx_trace;
  for (std::size_t s = 0; s < steps; ++s) {
    TopKMessage m = dev.ef_compress_step_topk(st, grad(s, 1 % P), k);
    for (auto i : m.indices) idx_trace.push_back((double)i);
    idx_trace.insert(idx_trace.end(), m.values.begin(), m.values.end());
  }
  idx_trace.insert(idx_trace.end(), st.residual.begin(), st.residual.end());
  write_bin(dir + "/ef_res.bin", idx_trace);

  // allreduce_mean, every algorithm, step-0 gradients
  std::vector<DenseVector> group;
  for (std::size_t p = 0; p < P; ++p) group.push_back(grad(0, p));
  const char* names[] = {"naive", "ring", "hierarchical", "pipelined_ring"};
  const CollectiveAlgorithm algos[] = {CollectiveAlgorithm::naive, CollectiveAlgorithm::ring,
                                       CollectiveAlgorithm::hierarchical, CollectiveAlgorithm::pipelined_ring};
  for (int a = 0; a < 4; ++a) write_bin(dir + "/mean_" + names[a] + ".bin", dev.allreduce_mean(group, algos[a]));

  // sync_data_parallel_step with top-k + EF, ring, all steps
  DenseVector theta(n, 0.0);
  std::vector<ErrorFeedbackState> ef(P, ErrorFeedbackState::zeros(n));
  for (std::size_t s = 0; s < steps; ++s) {
    std::vector<DenseVector> ws;
    for (std::size_t p = 0; p < P; ++p) ws.push_back(grad(s, p));
    theta = dev.sync_data_parallel_step(ws, theta, lr, CompressorKind::topk, k, CollectiveAlgorithm::ring, &ef);
  }
  write_bin(dir + "/sync_theta.bin", theta);
  std::vector<double> rr;
  for (auto& e : ef) rr.insert(rr.end(), e.residual.begin(), e.residual.end());
  write_bin(dir + "/sync_res.bin", rr);

  // onebit EF step: [scale, residual...] and the sign bytes
  ErrorFeedbackState so = ErrorFeedbackState::zeros(n);
  SignBitMessage sb = dev.ef_compress_step_onebit(so, grad(0, 0));
  std::vector<double> ob{sb.scale};
  ob.insert(ob.end(), so.residual.begin(), so.residual.end());
  write_bin(dir + "/onebit.bin", ob);
  write_bin(dir + "/onebit_bytes.bin", sb.sign_bytes);

  // async_step with tau = 3
  write_bin(dir + "/async.bin", dev.async_step(grad(0, 0), grad(0, 1 % P), 3, 0.1));

  // error behaviour: std::invalid_argument with the reference's messages
  std::ofstream err(dir + "/errors.txt");
  try {
    dev.compress_topk(DenseVector{1, 2}, 0);
  } catch (const std::invalid_argument& e) {
    err << "invalid_argument: " << e.what() << "\n";
  }
  try {
    ErrorFeedbackState bad = ErrorFeedbackState::zeros(3);
    dev.ef_compress_step_topk(bad, DenseVector{1, 2}, 1);
  } catch (const std::invalid_argument& e) {
    err << "invalid_argument: " << e.what() << "\n";
  }
  std::printf("facade_check ok\n");
  return 0;
}
