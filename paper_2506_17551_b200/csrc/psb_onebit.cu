// psb_onebit.cu -- 1-bit sign compressor with error feedback.
//
// Replaces ef_compress_step(state, g, {onebit}) (parsim/compression.hpp:146-157)
// with compress_onebit (:67-77):
//   p = r + g;  scale = l1_norm(p) / dim  (numerics.hpp:96-101, f64)
//   sign bit i = (p_i >= 0)  (sign(0) = +1, :74)
//   r' = p - (+-scale)       (decompress :113-120, residual :153-154)
// Pass 1 (k_onebit_pass1) streams g and r once: writes p into r, the sign
// words (warp-shuffle OR of per-lane nibbles; little-endian u32 words are
// byte-identical to the reference's sign_bytes) and one f64 partial |p| sum
// per CTA over a fixed element range.  The last CTA sums the partials in a
// fixed order (deterministic; differs from the reference's sequential fold
// only in rounding, see DESIGN.md tolerance).  Pass 2 rewrites r = p -+ scale.
#include "psb_internal.cuh"

namespace {

template <class T>
struct V16;
template <>
struct V16<float> {
  static constexpr int W = 4;
};
template <>
struct V16<double> {
  static constexpr int W = 2;
};

template <class T>
__global__ void __launch_bounds__(256) k_onebit_pass1(const T* __restrict__ g, T* __restrict__ r,
                                                      size_t n, size_t chunk_vecs,
                                                      uint32_t* __restrict__ words,
                                                      double* __restrict__ partials,
                                                      double* __restrict__ scale_out,
                                                      uint32_t* done, uint32_t* flags) {
  constexpr int W = V16<T>::W;
  constexpr int LPW = 32 / W;  // lanes per 32-bit word
  __shared__ double sh[8];
  __shared__ int am_last;
  const size_t nvec = (n + W - 1) / W;  // vector slots (last may be partial)
  const size_t v0 = (size_t)blockIdx.x * chunk_vecs;
  const size_t v1 = min(nvec, v0 + chunk_vecs);
  const int lane = threadIdx.x & 31;
  const bool vec_ok = ((((uintptr_t)g) | ((uintptr_t)r)) & 15) == 0;
  double acc = 0.0;
  bool bad = false;
  // chunk_vecs is a multiple of 256 (CTA) so warps stay aligned to 32-vector
  // groups: a warp covers W*32 consecutive elements = W words.
  for (size_t vb = v0; vb < v1; vb += blockDim.x) {
    const size_t v = vb + threadIdx.x;
    uint32_t nib = 0;
    if (v < v1) {
      const size_t e0 = v * W;
      T x[W];
      if (vec_ok && e0 + W <= n) {
        if (W == 4) {
          float4 gv = *reinterpret_cast<const float4*>(g + e0);
          float4 rv = r ? *reinterpret_cast<const float4*>(r + e0) : make_float4(0, 0, 0, 0);
          const float* gp = &gv.x;
          const float* rp = &rv.x;
          for (int c = 0; c < W; ++c) x[c] = r ? (T)add_rn(rp[c], gp[c]) : (T)gp[c];
          if (r) *reinterpret_cast<float4*>(r + e0) = make_float4(x[0], x[1], x[2], x[3]);
        } else {
          double2 gv = *reinterpret_cast<const double2*>(g + e0);
          double2 rv = r ? *reinterpret_cast<const double2*>(r + e0) : make_double2(0, 0);
          const double* gp = &gv.x;
          const double* rp = &rv.x;
          for (int c = 0; c < W; ++c) x[c] = r ? (T)add_rn(rp[c], gp[c]) : (T)gp[c];
          if (r) *reinterpret_cast<double2*>(r + e0) = make_double2(x[0], x[1]);
        }
#pragma unroll
        for (int c = 0; c < W; ++c) {
          acc += fabs((double)x[c]);
          nib |= (x[c] >= T(0) ? 1u : 0u) << c;
          bad |= !is_finite(x[c]);
        }
      } else {
        for (int c = 0; c < W; ++c) {
          const size_t e = e0 + c;
          if (e < n) {
            T p = r ? add_rn(r[e], g[e]) : g[e];
            if (r) r[e] = p;
            acc += fabs((double)p);
            nib |= (p >= T(0) ? 1u : 0u) << c;
            bad |= !is_finite(p);
          }
        }
      }
    }
    uint32_t wbits = nib << (W * (lane % LPW));
#pragma unroll
    for (int o = 1; o < LPW; o <<= 1) wbits |= __shfl_xor_sync(0xffffffffu, wbits, o);
    const size_t word = (vb + (threadIdx.x & ~31)) * W / 32 + lane / LPW;
    if ((lane % LPW) == 0 && (vb + (threadIdx.x & ~31) + (size_t)(lane / LPW) * LPW) < v1)
      words[word] = wbits;
  }
  // fixed-shape block reduction of the f64 partial
#pragma unroll
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) sh[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += sh[w];
    partials[blockIdx.x] = s;
  }
  if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(flags, 1u);
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) am_last = atomicAdd(done, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!am_last) return;
  __threadfence();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (unsigned b = 0; b < gridDim.x; ++b) s += __ldcg(partials + b);
    scale_out[0] = s / (double)n;
    *done = 0;
  }
}

template <class T>
__global__ void k_onebit_pass2(T* __restrict__ r, size_t n, const double* __restrict__ scale,
                               uint32_t* flags) {
  const T s = (T)scale[0];
  bool bad = false;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x) {
    const T p = r[i];
    const T res = sub_rn(p, p >= T(0) ? s : -s);
    r[i] = res;
    bad |= !is_finite(res);
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flags, 1u);
}

template <class T>
psb_status onebit_impl(psb_ctx* c, const T* g, T* r, size_t n, uint32_t* words, double* scale_out,
                       cudaStream_t st) {
  constexpr int W = V16<T>::W;
  const size_t nvec = (n + W - 1) / W;
  size_t grid = std::min<size_t>((size_t)c->num_sms * 4, (nvec + 255) / 256);
  if (grid < 1) grid = 1;
  size_t chunk = (nvec + grid - 1) / grid;
  chunk = (chunk + 255) / 256 * 256;
  grid = (nvec + chunk - 1) / chunk;
  PSB_REQUIRE(c, grid <= c->partials_cap, "onebit: partials capacity");
  uint32_t* done = reinterpret_cast<uint32_t*>(c->d_partials + c->partials_cap);
  k_onebit_pass1<T><<<(unsigned)grid, 256, 0, st>>>(g, r, n, chunk, words, c->d_partials, scale_out,
                                                    done, c->d_flags);
  c->launches += 1;
  if (r) {
    const unsigned g2 = (unsigned)std::min<size_t>((n + 255) / 256, (size_t)c->num_sms * 16);
    k_onebit_pass2<T><<<g2, 256, 0, st>>>(r, n, scale_out, c->d_flags);
    c->launches += 1;
  }
  PSB_LAUNCH_CHECK(c, "psb_ef_onebit");
  return PSB_OK;
}

}  // namespace

extern "C" psb_status psb_ef_onebit(psb_ctx* c, psb_dtype dt, const void* g, void* r, size_t n,
                                    uint32_t* words_out, double* scale_out, psb_stream_t stream) {
  PSB_REQUIRE(c, c != nullptr, "null ctx");
  PSB_REQUIRE(c, n >= 1, "compress_onebit: empty vector");
  PSB_REQUIRE(c, n <= c->max_n, "ef_compress_step: n exceeds ctx max_n");
  PSB_REQUIRE(c, g && words_out && scale_out, "psb_ef_onebit: null pointer");
  cudaStream_t st = (cudaStream_t)stream;
  if (dt == PSB_F32) return onebit_impl<float>(c, (const float*)g, (float*)r, n, words_out, scale_out, st);
  return onebit_impl<double>(c, (const double*)g, (double*)r, n, words_out, scale_out, st);
}
