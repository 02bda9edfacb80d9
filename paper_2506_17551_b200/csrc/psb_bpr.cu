// psb_bpr.cu -- the gradient producer that feeds the path:
// BPR (pairwise logistic) loss and its analytic gradient for the reference's
// matrix-factorisation recommender, on the device.
//
// Replaces bpr_batch_loss / bpr_batch_gradient (parsim/trainer.hpp:98-138).
// Flat layout (trainer.hpp:86-91): user rows [0, users), item rows
// [users, users + items), dim columns each.  Per triple t (batch order):
//   x_t   = sum_k u[k] * (p[k] - n[k])        (sequential in k, :103/:124)
//   c_t   = -sigmoid(-x_t) * (1/B)            (:127, sigmoid = 1/(1+exp(x)))
//   g_u  += c_t * (p - n);  g_p += c_t * u;  g_n -= c_t * u      (:131-135)
// The reference accumulates every row's contributions in batch order (user,
// then positive, then negative within a triple).  Here the 3B contributions
// are stably sorted by row (CUB radix sort keeps the batch order of equal
// rows), and one warp per touched row folds them in that order with
// separate RN multiply and add -- the same operations in the same order.
// The only deviation is exp(): the device's double exp is within 1 ulp of
// glibc's, so c_t (and hence the gradient) carries a relative tolerance of a
// few ulp (tests: 1e-14); all zero/non-zero structure is exact.
#include <cub/device/device_radix_sort.cuh>

#include "psb_internal.cuh"

namespace {

template <class T>
__global__ void k_bpr_coeff(const T* __restrict__ theta, uint32_t users, uint32_t dim, const uint32_t* __restrict__ u,
                            const uint32_t* __restrict__ p, const uint32_t* __restrict__ q, uint32_t B,
                            double* __restrict__ coeff, double* __restrict__ lossv, uint32_t* __restrict__ rows,
                            uint32_t* __restrict__ seq) {
  const double inv = 1.0 / (double)B;
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < B; t += gridDim.x * blockDim.x) {
    const T* ur = theta + (size_t)u[t] * dim;
    const T* pr = theta + ((size_t)users + p[t]) * dim;
    const T* nr = theta + ((size_t)users + q[t]) * dim;
    double x = 0.0;
    for (uint32_t k = 0; k < dim; ++k)
      x = __dadd_rn(x, __dmul_rn((double)ur[k], __dsub_rn((double)pr[k], (double)nr[k])));
    const double s = 1.0 / (1.0 + exp(x));  // sigmoid(-x)
    coeff[t] = __dmul_rn(-s, inv);
    // softplus_neg(x) = log(1 + exp(-x)) without overflow (trainer.hpp:80-83)
    lossv[t] = x > 0 ? log1p(exp(-x)) : -x + log1p(exp(x));
    rows[3 * t + 0] = u[t];
    rows[3 * t + 1] = users + p[t];
    rows[3 * t + 2] = users + q[t];
    seq[3 * t + 0] = 3 * t + 0;
    seq[3 * t + 1] = 3 * t + 1;
    seq[3 * t + 2] = 3 * t + 2;
  }
}

// One warp per run of equal rows in the sorted contribution list.
template <class T>
__global__ void k_bpr_rows(const T* __restrict__ theta, uint32_t users, uint32_t dim, const uint32_t* __restrict__ u,
                           const uint32_t* __restrict__ p, const uint32_t* __restrict__ q,
                           const double* __restrict__ coeff, const uint32_t* __restrict__ rows_sorted,
                           const uint32_t* __restrict__ seq_sorted, uint32_t ncontrib, T* __restrict__ grad) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t j = warp; j < ncontrib; j += nwarps) {
    const uint32_t row = rows_sorted[j];
    if (j > 0 && rows_sorted[j - 1] == row) continue;  // not the start of a run
    uint32_t end = j + 1;
    while (end < ncontrib && rows_sorted[end] == row) ++end;
    for (uint32_t k = lane; k < dim; k += 32) {
      T acc = T(0);
      for (uint32_t e = j; e < end; ++e) {
        const uint32_t s = seq_sorted[e];
        const uint32_t t = s / 3, role = s - 3 * t;
        const T c = (T)coeff[t];
        const T* ur = theta + (size_t)u[t] * dim;
        if (role == 0) {
          const T* pr = theta + ((size_t)users + p[t]) * dim;
          const T* nr = theta + ((size_t)users + q[t]) * dim;
          acc = add_rn(acc, mul_rn(c, sub_rn(pr[k], nr[k])));
        } else if (role == 1) {
          acc = add_rn(acc, mul_rn(c, ur[k]));
        } else {
          acc = sub_rn(acc, mul_rn(c, ur[k]));
        }
      }
      grad[(size_t)row * dim + k] = acc;
    }
  }
}

// Mean loss: the batch's softplus values summed in batch order (trainer.hpp:107).
__global__ void k_bpr_loss(const double* __restrict__ lossv, uint32_t B, double* __restrict__ out) {
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    double acc = 0.0;
    for (uint32_t t = 0; t < B; ++t) acc = __dadd_rn(acc, lossv[t]);
    *out = acc / (double)B;
  }
}

__global__ void k_bpr_check(const uint32_t* __restrict__ u, const uint32_t* __restrict__ p,
                            const uint32_t* __restrict__ q, uint32_t B, uint32_t users, uint32_t items,
                            uint32_t* flags) {
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < B; t += gridDim.x * blockDim.x)
    if (u[t] >= users || p[t] >= items || q[t] >= items) atomicOr(flags, 128u);
}

}  // namespace

extern "C" psb_status psb_bpr_gradient(psb_ctx* c, psb_dtype dt, const void* theta, uint32_t users, uint32_t items,
                                       uint32_t dim, const uint32_t* user, const uint32_t* pos, const uint32_t* neg,
                                       uint32_t B, void* grad, double* loss_out, psb_stream_t stream) {
  PSB_REQUIRE(c, c != nullptr, "null ctx");
  PSB_REQUIRE(c, dt == PSB_F32 || dt == PSB_F64, "bpr_batch_gradient: bad dtype");
  PSB_REQUIRE(c, B >= 1, "bpr_batch_gradient: empty batch");
  PSB_REQUIRE(c, users >= 1 && items >= 1 && dim >= 1, "RecModel: sizes must be >= 1");
  PSB_REQUIRE(c, theta && user && pos && neg && grad, "bpr_batch_gradient: null buffer");
  PSB_REQUIRE(c, (uint64_t)B * 3 < (1ull << 31), "bpr_batch_gradient: batch too large");
  cudaStream_t st = (cudaStream_t)stream;
  const size_t es = dt == PSB_F64 ? 8 : 4;
  const size_t n = ((size_t)users + items) * dim;
  const uint32_t nc = 3 * B;
  // workspace: coeff[B] f64 | loss[B] f64 | rows[3B] | seq[3B] | rows_s[3B] | seq_s[3B] | loss scalar | cub temp
  size_t cub_bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, cub_bytes, (const uint32_t*)nullptr, (uint32_t*)nullptr,
                                  (const uint32_t*)nullptr, (uint32_t*)nullptr, (int)nc, 0, 32, st);
  auto al = [](size_t b) { return (b + 255) & ~(size_t)255; };
  const size_t o_loss = al(8 * (size_t)B), o_rows = o_loss + al(8 * (size_t)B), o_seq = o_rows + al(4 * (size_t)nc),
               o_rs = o_seq + al(4 * (size_t)nc), o_ss = o_rs + al(4 * (size_t)nc), o_l = o_ss + al(4 * (size_t)nc),
               o_cub = o_l + 256, total = o_cub + al(cub_bytes);
  if (c->work_bytes < total) {
    if (c->d_work) cudaFree(c->d_work);
    c->d_work = nullptr;
    c->work_bytes = 0;
    if (cudaMalloc(&c->d_work, total) != cudaSuccess) return psb_set_err(c, PSB_ENOMEM, "bpr workspace: out of memory");
    c->work_bytes = total;
  }
  uint8_t* w = reinterpret_cast<uint8_t*>(c->d_work);
  double* coeff = reinterpret_cast<double*>(w);
  double* lossv = reinterpret_cast<double*>(w + o_loss);
  uint32_t* rows = reinterpret_cast<uint32_t*>(w + o_rows);
  uint32_t* seq = reinterpret_cast<uint32_t*>(w + o_seq);
  uint32_t* rows_s = reinterpret_cast<uint32_t*>(w + o_rs);
  uint32_t* seq_s = reinterpret_cast<uint32_t*>(w + o_ss);
  double* lsum = reinterpret_cast<double*>(w + o_l);
  const unsigned gb = (unsigned)std::max<uint32_t>(1, std::min<uint32_t>((B + 255) / 256, c->num_sms * 8));
  k_bpr_check<<<gb, 256, 0, st>>>(user, pos, neg, B, users, items, c->d_flags);
  CUDA_TRY(c, cudaMemsetAsync(grad, 0, es * n, st), "bpr_batch_gradient");
  if (dt == PSB_F64)
    k_bpr_coeff<double><<<gb, 256, 0, st>>>((const double*)theta, users, dim, user, pos, neg, B, coeff, lossv, rows, seq);
  else
    k_bpr_coeff<float><<<gb, 256, 0, st>>>((const float*)theta, users, dim, user, pos, neg, B, coeff, lossv, rows, seq);
  int bits = 1;
  while (bits < 32 && ((uint64_t)users + items) >> bits) ++bits;
  cudaError_t e = cub::DeviceRadixSort::SortPairs(w + o_cub, cub_bytes, rows, rows_s, seq, seq_s, (int)nc, 0, bits, st);
  if (e != cudaSuccess) return psb_cuda_err(c, e, "bpr_batch_gradient (sort)");
  const unsigned gr = (unsigned)std::max<uint32_t>(1, std::min<uint32_t>((nc + 7) / 8, c->num_sms * 16));
  if (dt == PSB_F64)
    k_bpr_rows<double><<<gr, 256, 0, st>>>((const double*)theta, users, dim, user, pos, neg, coeff, rows_s, seq_s, nc,
                                           (double*)grad);
  else
    k_bpr_rows<float><<<gr, 256, 0, st>>>((const float*)theta, users, dim, user, pos, neg, coeff, rows_s, seq_s, nc,
                                          (float*)grad);
  if (loss_out) {
    k_bpr_loss<<<1, 32, 0, st>>>(lossv, B, lsum);
    CUDA_TRY(c, cudaMemcpyAsync(loss_out, lsum, sizeof(double), cudaMemcpyDeviceToDevice, st), "bpr loss");
  }
  c->launches += loss_out ? 5 : 4;
  PSB_LAUNCH_CHECK(c, "psb_bpr_gradient");
  return PSB_OK;
}

// ------------------------------------------------- sampled ranking (HR/NDCG)
namespace {
// One warp per test record: rank = 1 + #{candidates c : s(c) > s(true) or
// (s(c) == s(true) and c < true item)} (trainer.hpp:307-312); scores are the
// reference's sequential f64 dot products (RecModel::score, :40-47).
template <class T>
__global__ void k_rank_candidates(const T* __restrict__ theta, uint32_t users, uint32_t dim, uint32_t R,
                                  const uint32_t* __restrict__ ru, const uint32_t* __restrict__ ri,
                                  const uint32_t* __restrict__ cands, uint32_t ncand, uint32_t* __restrict__ rank) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  auto score = [&](uint32_t u, uint32_t item) {
    const T* ur = theta + (size_t)u * dim;
    const T* ir = theta + ((size_t)users + item) * dim;
    double s = 0.0;
    for (uint32_t k = 0; k < dim; ++k) s = __dadd_rn(s, __dmul_rn((double)ur[k], (double)ir[k]));
    return s;
  };
  for (uint32_t r = warp; r < R; r += nwarps) {
    const uint32_t u = ru[r], it = ri[r];
    const double ts = score(u, it);
    uint32_t cnt = 0;
    for (uint32_t j = lane; j < ncand; j += 32) {
      const uint32_t c = cands[(size_t)r * ncand + j];
      if (c == 0xffffffffu) continue;  // padding
      const double s = score(u, c);
      cnt += (s > ts || (s == ts && c < it)) ? 1u : 0u;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    if (lane == 0) rank[r] = 1 + cnt;
  }
}
}  // namespace

extern "C" psb_status psb_rank_candidates(psb_ctx* c, psb_dtype dt, const void* theta, uint32_t users, uint32_t dim,
                                          uint32_t R, const uint32_t* rec_user, const uint32_t* rec_item,
                                          const uint32_t* cands, uint32_t ncand, uint32_t* rank_out,
                                          psb_stream_t stream) {
  PSB_REQUIRE(c, c != nullptr, "null ctx");
  PSB_REQUIRE(c, dt == PSB_F32 || dt == PSB_F64, "evaluate_topk: bad dtype");
  PSB_REQUIRE(c, R >= 1, "evaluate_topk: empty test split");
  PSB_REQUIRE(c, theta && rec_user && rec_item && rank_out && (ncand == 0 || cands), "evaluate_topk: null buffer");
  cudaStream_t st = (cudaStream_t)stream;
  const unsigned grid = (unsigned)std::max<uint32_t>(1, std::min<uint32_t>((R + 7) / 8, c->num_sms * 16));
  if (dt == PSB_F64)
    k_rank_candidates<double><<<grid, 256, 0, st>>>((const double*)theta, users, dim, R, rec_user, rec_item, cands,
                                                    ncand, rank_out);
  else
    k_rank_candidates<float><<<grid, 256, 0, st>>>((const float*)theta, users, dim, R, rec_user, rec_item, cands,
                                                   ncand, rank_out);
  c->launches += 1;
  PSB_LAUNCH_CHECK(c, "psb_rank_candidates");
  return PSB_OK;
}
