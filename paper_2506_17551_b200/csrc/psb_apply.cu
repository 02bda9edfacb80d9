// psb_apply.cu -- aggregate + apply without dense messages.
//
// Replaces, for P workers' messages, the reference sequence
//   decompress(msg_p)                      parsim/strategies.hpp:108, compression.hpp:113-142
//   allreduce_mean(decompressed, algo)     strategies.hpp:110, collectives.hpp:135-148
//   vec_axpy(-lr, mean, params)            strategies.hpp:112, numerics.hpp:70-78
// and the async per-worker update async_step (strategies.hpp:125-129) applied
// in worker order (trainer.hpp:245-254).
//
// Sparse layout: P payload blocks (psb_payload_bytes), each with k indices
// ascending.  The index space is cut into segments of S = 2^seg_shift
// entries; k_seg_offsets finds each worker's sub-range per segment, and
// k_sparse_apply gives one CTA per segment: workers' values are scattered
// into shared memory slots vals[q][i] with a presence mask, then the lowest
// worker touching an index folds the P dense values (+0 where absent) in the
// configured reference order and updates theta once: (-lr)*(sum*(1/P)) +
// theta with separate RN multiply and add (no FMA).  HBM traffic: read the
// P*k pairs once, read+write theta at the touched indices only.
#include "psb_fold.cuh"

namespace {

struct WorkerCoefs {
  double v[PSB_MAX_P];  // eta/(1+tau_p) per worker (async), by value in the launch
};

struct PayloadView {
  const uint8_t* base;
  size_t block_bytes;
  size_t val_off;    // byte offset of values (or int8 codes) inside a block
  size_t scale_off;  // TOPK_Q8: byte offset of the f32 scales
  int q8;
};

__device__ __forceinline__ const uint32_t* pl_idx(const PayloadView& v, int q) {
  return reinterpret_cast<const uint32_t*>(v.base + (size_t)q * v.block_bytes);
}

template <class T>
__device__ __forceinline__ T pl_val(const PayloadView& v, int q, size_t j) {
  const uint8_t* b = v.base + (size_t)q * v.block_bytes;
  if (v.q8) {
    const int8_t code = reinterpret_cast<const int8_t*>(b + v.val_off)[j];
    const float sc = reinterpret_cast<const float*>(b + v.scale_off)[j >> 7];
    return (T)__fmul_rn((float)code, sc);
  }
  return reinterpret_cast<const T*>(b + v.val_off)[j];
}

__global__ void k_seg_offsets(PayloadView v, int P, size_t k, uint32_t nseg, int seg_shift,
                              uint32_t* __restrict__ seg_off) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  const size_t work1 = (size_t)P * k;
  const size_t work2 = (size_t)P * (nseg + 1);
  const size_t work = work1 > work2 ? work1 : work2;
  for (size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x; t < work; t += stride) {
    if (t < work1) {
      const int q = (int)(t / k);
      const size_t j = t - (size_t)q * k;
      const uint32_t* idx = pl_idx(v, q);
      const long long sj = (long long)(idx[j] >> seg_shift);
      const long long sp = j ? (long long)(idx[j - 1] >> seg_shift) : -1ll;
      uint32_t* row = seg_off + (size_t)q * (nseg + 1);
      for (long long s = sp + 1; s <= sj && s <= (long long)nseg; ++s) row[s] = (uint32_t)j;
    }
    if (t < work2) {
      const int q = (int)(t / (nseg + 1));
      const uint32_t s = (uint32_t)(t - (size_t)q * (nseg + 1));
      const uint32_t last = pl_idx(v, q)[k - 1] >> seg_shift;
      if (s > last) seg_off[(size_t)q * (nseg + 1) + s] = (uint32_t)k;
    }
  }
}

template <class T, bool ASYNC>
__global__ void __launch_bounds__(256) k_sparse_apply(PayloadView v, int P, uint32_t nseg,
                                                      int seg_shift,
                                                      const uint32_t* __restrict__ seg_off,
                                                      int order, uint32_t dpn, uint32_t npr,
                                                      T coef, WorkerCoefs wscale,
                                                      T* __restrict__ theta, size_t n,
                                                      T* __restrict__ mean_out, uint32_t* flags) {
  extern __shared__ __align__(16) unsigned char smem[];
  const uint32_t S = 1u << seg_shift;
  uint32_t* mask = reinterpret_cast<uint32_t*>(smem);
  T* vals = reinterpret_cast<T*>(smem + (size_t)S * 4);
  __shared__ uint32_t lo[PSB_MAX_P], hi[PSB_MAX_P];
  __shared__ uint32_t sh_any, sh_bad;
  __shared__ T coefs[PSB_MAX_P];
  if (threadIdx.x == 0) sh_bad = 0;
  if (ASYNC && threadIdx.x < (unsigned)P) coefs[threadIdx.x] = (T)(-wscale.v[threadIdx.x]);
  const T inv = (T)(1.0 / (double)P);
  bool bad = false;

  for (uint32_t seg = blockIdx.x; seg < nseg; seg += gridDim.x) {
    __syncthreads();
    if (threadIdx.x == 0) sh_any = 0;
    __syncthreads();
    if (threadIdx.x < (unsigned)P) {
      const uint32_t* row = seg_off + (size_t)threadIdx.x * (nseg + 1);
      lo[threadIdx.x] = row[seg];
      hi[threadIdx.x] = row[seg + 1];
      if (hi[threadIdx.x] > lo[threadIdx.x]) atomicOr(&sh_any, 1u);
    }
    __syncthreads();
    if (!sh_any) continue;
    for (uint32_t i = threadIdx.x; i < S; i += blockDim.x) mask[i] = 0;
    __syncthreads();
    const size_t seg_base = (size_t)seg << seg_shift;
    for (int q = 0; q < P; ++q) {
      const uint32_t* idx = pl_idx(v, q);
      for (uint32_t j = lo[q] + threadIdx.x; j < hi[q]; j += blockDim.x) {
        const uint32_t il = (uint32_t)(idx[j] - seg_base);
        vals[(size_t)q * S + il] = pl_val<T>(v, q, j);
        atomicOr(&mask[il], 1u << q);
      }
    }
    __syncthreads();
    for (int q = 0; q < P; ++q) {
      const uint32_t* idx = pl_idx(v, q);
      for (uint32_t j = lo[q] + threadIdx.x; j < hi[q]; j += blockDim.x) {
        const size_t i = idx[j];
        const uint32_t il = (uint32_t)(i - seg_base);
        const uint32_t m = mask[il];
        if (__ffs(m) - 1 != q) continue;  // the lowest touching worker owns index i
        T th = theta ? theta[i] : T(0);
        if (ASYNC) {
          uint32_t mm = m;
          while (mm) {
            const int w = __ffs(mm) - 1;
            mm &= mm - 1;
            th = add_rn(mul_rn(coefs[w], vals[(size_t)w * S + il]), th);
          }
        } else {
          auto get = [&](int w) -> T { return ((m >> w) & 1u) ? vals[(size_t)w * S + il] : T(0); };
          const T mean = mul_rn(fold_sum<T>(get, P, order, i, n, dpn, npr), inv);
          th = add_rn(mul_rn(coef, mean), th);
          if (mean_out) mean_out[i] = mean;
        }
        if (theta) {
          theta[i] = th;
          bad |= !is_finite(th);
        }
      }
    }
  }
  if (bad) sh_bad = 1;
  __syncthreads();
  if (threadIdx.x == 0 && sh_bad) atomicOr(flags, 1u);
}

// P == 1: one payload, every touched index owned by worker 0.
template <class T, bool ASYNC>
__global__ void k_sparse_apply1(PayloadView v, size_t k, T coef, T* __restrict__ theta,
                                T* __restrict__ mean_out, uint32_t* flags) {
  const uint32_t* idx = pl_idx(v, 0);
  bool bad = false;
  for (size_t j = (size_t)blockIdx.x * blockDim.x + threadIdx.x; j < k;
       j += (size_t)gridDim.x * blockDim.x) {
    const uint32_t i = idx[j];
    const T val = pl_val<T>(v, 0, j);
    const T mean = ASYNC ? val : mul_rn(val, T(1));
    if (!ASYNC && mean_out) mean_out[i] = mean;
    if (theta) {
      const T th = add_rn(mul_rn(coef, mean), theta[i]);
      theta[i] = th;
      bad |= !is_finite(th);
    }
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flags, 1u);
}

// Dense fold (compressor none) or 1-bit fold over P workers, + SGD.
template <class T, bool ONEBIT>
__global__ void __launch_bounds__(256) k_dense_apply(const T* __restrict__ bufs,
                                                     const uint32_t* __restrict__ words,
                                                     const double* __restrict__ scales, int P,
                                                     int order, uint32_t dpn, uint32_t npr, T coef,
                                                     T* __restrict__ theta, size_t n,
                                                     T* __restrict__ mean_out, uint32_t* flags) {
  __shared__ T sc[PSB_MAX_P];
  if (ONEBIT && threadIdx.x < (unsigned)P) sc[threadIdx.x] = (T)scales[threadIdx.x];
  __syncthreads();
  const size_t nw = (n + 31) / 32;
  const T inv = (T)(1.0 / (double)P);
  bool bad = false;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x) {
    auto get = [&](int q) -> T {
      if (ONEBIT) {
        const uint32_t w = words[(size_t)q * nw + (i >> 5)];
        return ((w >> (i & 31)) & 1u) ? sc[q] : -sc[q];
      }
      return bufs[(size_t)q * n + i];
    };
    const T mean = mul_rn(fold_sum<T>(get, P, order, i, n, dpn, npr), inv);
    if (mean_out) mean_out[i] = mean;
    if (theta) {
      const T th = add_rn(mul_rn(coef, mean), theta[i]);
      theta[i] = th;
      bad |= !is_finite(th);
    }
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flags, 1u);
}

template <class T>
__global__ void k_decompress_topk(const uint32_t* __restrict__ idx, const T* __restrict__ val,
                                  size_t k, size_t n, T* __restrict__ out, uint32_t* flags) {
  uint32_t f = 0;
  for (size_t j = (size_t)blockIdx.x * blockDim.x + threadIdx.x; j < k;
       j += (size_t)gridDim.x * blockDim.x) {
    const uint32_t i = idx[j];
    if (i >= n) {
      f |= 2u;
      continue;
    }
    if (j > 0 && idx[j - 1] >= i) f |= 4u;
    out[i] = val[j];
  }
  if (f) atomicOr(flags, f);
}

PayloadView make_view(psb_compressor c, psb_dtype dt, const void* payloads, size_t k) {
  PayloadView v;
  v.base = reinterpret_cast<const uint8_t*>(payloads);
  v.block_bytes = psb_payload_bytes(c, dt, k);
  v.val_off = psb_align16(k * 4);
  v.q8 = c == PSB_COMP_TOPK_Q8;
  v.scale_off = v.val_off + psb_align16(k);
  return v;
}

void topo_fields(const psb_topology* topo, int P, uint32_t* dpn, uint32_t* npr) {
  if (!topo || topo->devices_per_node == 0) {
    *dpn = (uint32_t)P;  // flat topology: devices_per_node = P (collectives.hpp:150-154)
    *npr = 1;
  } else {
    *dpn = topo->devices_per_node;
    *npr = topo->nodes_per_rack ? topo->nodes_per_rack : 1;
  }
}

template <class T>
psb_status sparse_impl(psb_ctx* c, psb_compressor comp, int P, const void* payloads, size_t k,
                       psb_order order, const psb_topology* topo, double lr,
                       const double* wscale_host, bool async_mode, T* theta, size_t n, T* mean_out,
                       cudaStream_t st) {
  PayloadView v = make_view(comp, sizeof(T) == 8 ? PSB_F64 : PSB_F32, payloads, k);
  uint32_t dpn, npr;
  topo_fields(topo, P, &dpn, &npr);
  const T coef = (T)(-lr);
  if (P == 1) {
    const unsigned grid = (unsigned)std::min<size_t>((k + 255) / 256, (size_t)c->num_sms * 32);
    if (async_mode)
      k_sparse_apply1<T, true><<<grid, 256, 0, st>>>(v, k, (T)(-wscale_host[0]), theta, nullptr,
                                                     c->d_flags);
    else
      k_sparse_apply1<T, false><<<grid, 256, 0, st>>>(v, k, coef, theta, mean_out, c->d_flags);
    c->launches += 1;
    PSB_LAUNCH_CHECK(c, "psb_sparse_mean_sgd");
    return PSB_OK;
  }
  // segment size: P*S*sizeof(T) + 4*S <= 96 KB, S <= 4096
  int seg_shift = 12;
  while (seg_shift > 6 && ((size_t)P * sizeof(T) + 4) << seg_shift > 96 * 1024) --seg_shift;
  const uint32_t nseg = (uint32_t)((n + ((size_t)1 << seg_shift) - 1) >> seg_shift);
  PSB_REQUIRE(c, (size_t)P * (nseg + 1) <= c->seg_cap, "sparse apply: segment table exceeds ctx capacity");
  const size_t work = std::max((size_t)P * k, (size_t)P * (nseg + 1));
  const unsigned g1 = (unsigned)std::min<size_t>((work + 255) / 256, (size_t)c->num_sms * 16);
  k_seg_offsets<<<g1, 256, 0, st>>>(v, P, k, nseg, seg_shift, c->d_seg_off);
  const size_t smem = (((size_t)P * sizeof(T) + 4) << seg_shift);
  WorkerCoefs ws{};
  if (async_mode)
    for (int q = 0; q < P; ++q) ws.v[q] = wscale_host[q];
  const unsigned grid = nseg;
  if (async_mode) {
    auto kern = k_sparse_apply<T, true>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kern<<<grid, 256, smem, st>>>(v, P, nseg, seg_shift, c->d_seg_off, (int)order, dpn, npr, coef,
                                  ws, theta, n, nullptr, c->d_flags);
  } else {
    auto kern = k_sparse_apply<T, false>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kern<<<grid, 256, smem, st>>>(v, P, nseg, seg_shift, c->d_seg_off, (int)order, dpn, npr, coef,
                                  ws, theta, n, mean_out, c->d_flags);
  }
  c->launches += 2;
  PSB_LAUNCH_CHECK(c, "psb_sparse_mean_sgd");
  return PSB_OK;
}

template <class T, bool ONEBIT>
psb_status dense_impl(psb_ctx* c, int P, const void* bufs, const uint32_t* words,
                      const double* scales, psb_order order, const psb_topology* topo, double lr,
                      T* theta, size_t n, T* mean_out, cudaStream_t st) {
  uint32_t dpn, npr;
  topo_fields(topo, P, &dpn, &npr);
  const unsigned grid = (unsigned)std::min<size_t>((n + 255) / 256, (size_t)c->num_sms * 16);
  k_dense_apply<T, ONEBIT><<<grid, 256, 0, st>>>((const T*)bufs, words, scales, P, (int)order, dpn,
                                                 npr, (T)(-lr), theta, n, mean_out, c->d_flags);
  c->launches += 1;
  PSB_LAUNCH_CHECK(c, "dense apply");
  return PSB_OK;
}

}  // namespace

static psb_status check_common(psb_ctx* c, int P, size_t n, psb_order order, const psb_topology* topo) {
  PSB_REQUIRE(c, c != nullptr, "null ctx");
  PSB_REQUIRE(c, P >= 1 && P <= PSB_MAX_P, "WorkerGroup: no workers");
  PSB_REQUIRE(c, P <= c->max_workers, "apply: P exceeds ctx max_workers");
  PSB_REQUIRE(c, n >= 1 && n <= c->max_n, "apply: n out of range for ctx");
  PSB_REQUIRE(c, order == PSB_ORDER_NAIVE || order == PSB_ORDER_RING || order == PSB_ORDER_HIER,
              "allreduce_mean: unknown algorithm");
  if (topo && topo->devices_per_node)
    PSB_REQUIRE(c, topo->racks >= 1 && topo->nodes_per_rack >= 1, "Topology: counts must be >= 1");
  return PSB_OK;
}

extern "C" psb_status psb_sparse_mean_sgd(psb_ctx* c, psb_compressor comp, psb_dtype dt, int P,
                                          const void* payloads, size_t k, psb_order order,
                                          const psb_topology* topo, double lr, void* theta,
                                          size_t n, void* mean_out, psb_stream_t stream) {
  psb_status s = check_common(c, P, n, order, topo);
  if (s) return s;
  PSB_REQUIRE(c, comp == PSB_COMP_TOPK || (comp == PSB_COMP_TOPK_Q8 && dt == PSB_F32),
              "psb_sparse_mean_sgd: payload kind must be TOPK (or TOPK_Q8 with f32)");
  PSB_REQUIRE(c, k >= 1 && k <= n, "compress_topk: k out of range");
  cudaStream_t st = (cudaStream_t)stream;
  if (dt == PSB_F32)
    return sparse_impl<float>(c, comp, P, payloads, k, order, topo, lr, nullptr, false,
                              (float*)theta, n, (float*)mean_out, st);
  return sparse_impl<double>(c, comp, P, payloads, k, order, topo, lr, nullptr, false,
                             (double*)theta, n, (double*)mean_out, st);
}

extern "C" psb_status psb_sparse_async_apply(psb_ctx* c, psb_compressor comp, psb_dtype dt, int P,
                                             const void* payloads, size_t k,
                                             const double* scale_per_worker, void* theta, size_t n,
                                             psb_stream_t stream) {
  psb_status s = check_common(c, P, n, PSB_ORDER_NAIVE, nullptr);
  if (s) return s;
  PSB_REQUIRE(c, comp == PSB_COMP_TOPK || (comp == PSB_COMP_TOPK_Q8 && dt == PSB_F32),
              "psb_sparse_async_apply: payload kind must be TOPK (or TOPK_Q8 with f32)");
  PSB_REQUIRE(c, k >= 1 && k <= n, "compress_topk: k out of range");
  PSB_REQUIRE(c, scale_per_worker != nullptr, "psb_sparse_async_apply: null scales");
  cudaStream_t st = (cudaStream_t)stream;
  if (dt == PSB_F32)
    return sparse_impl<float>(c, comp, P, payloads, k, PSB_ORDER_NAIVE, nullptr, 0.0,
                              scale_per_worker, true, (float*)theta, n, nullptr, st);
  return sparse_impl<double>(c, comp, P, payloads, k, PSB_ORDER_NAIVE, nullptr, 0.0,
                             scale_per_worker, true, (double*)theta, n, nullptr, st);
}

extern "C" psb_status psb_dense_mean_sgd(psb_ctx* c, psb_dtype dt, int P, const void* bufs,
                                         psb_order order, const psb_topology* topo, double lr,
                                         void* theta, size_t n, void* mean_out,
                                         psb_stream_t stream) {
  psb_status s = check_common(c, P, n, order, topo);
  if (s) return s;
  cudaStream_t st = (cudaStream_t)stream;
  if (dt == PSB_F32)
    return dense_impl<float, false>(c, P, bufs, nullptr, nullptr, order, topo, lr, (float*)theta,
                                    n, (float*)mean_out, st);
  return dense_impl<double, false>(c, P, bufs, nullptr, nullptr, order, topo, lr, (double*)theta,
                                   n, (double*)mean_out, st);
}

extern "C" psb_status psb_onebit_mean_sgd(psb_ctx* c, psb_dtype dt, int P, const uint32_t* words,
                                          const double* scales, psb_order order,
                                          const psb_topology* topo, double lr, void* theta,
                                          size_t n, void* mean_out, psb_stream_t stream) {
  psb_status s = check_common(c, P, n, order, topo);
  if (s) return s;
  cudaStream_t st = (cudaStream_t)stream;
  if (dt == PSB_F32)
    return dense_impl<float, true>(c, P, nullptr, words, scales, order, topo, lr, (float*)theta, n,
                                   (float*)mean_out, st);
  return dense_impl<double, true>(c, P, nullptr, words, scales, order, topo, lr, (double*)theta, n,
                                  (double*)mean_out, st);
}

extern "C" psb_status psb_decompress_topk(psb_ctx* c, psb_dtype dt, const uint32_t* idx,
                                          const void* val, size_t k, size_t n, void* out,
                                          psb_stream_t stream) {
  PSB_REQUIRE(c, c != nullptr, "null ctx");
  PSB_REQUIRE(c, out != nullptr && (k == 0 || (idx && val)), "psb_decompress_topk: null pointer");
  if (k == 0) return PSB_OK;
  const unsigned grid = (unsigned)std::min<size_t>((k + 255) / 256, (size_t)c->num_sms * 8);
  if (dt == PSB_F32)
    k_decompress_topk<float><<<grid, 256, 0, (cudaStream_t)stream>>>(idx, (const float*)val, k, n,
                                                                      (float*)out, c->d_flags);
  else
    k_decompress_topk<double><<<grid, 256, 0, (cudaStream_t)stream>>>(idx, (const double*)val, k, n,
                                                                       (double*)out, c->d_flags);
  c->launches += 1;
  PSB_LAUNCH_CHECK(c, "psb_decompress_topk");
  return PSB_OK;
}
