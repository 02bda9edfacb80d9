// psb_gen.cu -- counter-based synthetic gradients (input generation only).
//
// Same integer + fp32 recipe as oracle/psb_oracle.c:orc_generate, built on
// mix64 (parsim/numerics.hpp:181-186), so host and device produce identical
// bits (SURVEY.md 8d "Synthetic inputs").  All fp32 ops are RN without
// contraction (__fadd_rn/__fmul_rn) to match the host build (-ffp-contract=off).
#include "psb_internal.cuh"

namespace {

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

__device__ __forceinline__ float u24(uint64_t h) {
  return __fmul_rn((float)(uint32_t)(h >> 40), 5.9604644775390625e-08f /* 2^-24 */);
}

__device__ __forceinline__ float gen_one(int dist, uint64_t base, uint64_t base_row, size_t n_emb,
                                         size_t i) {
  if (dist == PSB_DIST_UNIFORM) return __fsub_rn(__fmul_rn(2.0f, u24(mix64(base + i))), 1.0f);
  if (dist == PSB_DIST_TIES) {
    const uint64_t v = mix64(base + i) >> 40;
    const int bucket = (int)((v * 5) >> 24);
    return __fmul_rn((float)(bucket - 2), 0.25f);
  }
  const float a = u24(mix64(base + 4 * i + 0));
  const float b = u24(mix64(base + 4 * i + 1));
  const float c = u24(mix64(base + 4 * i + 2));
  const float d = u24(mix64(base + 4 * i + 3));
  const float z = __fmul_rn(__fsub_rn(__fadd_rn(__fadd_rn(a, b), __fadd_rn(c, d)), 2.0f), 1.7320508e-3f);
  if (i < n_emb) {
    const uint64_t row = i >> 6;
    const uint64_t zr = mix64(base_row + 2 * row) >> 40;
    if (((zr * 20) >> 24) < 19) return 0.0f;
    const uint32_t e = (uint32_t)(((mix64(base_row + 2 * row + 1) >> 40) * 7) >> 24);
    return __fmul_rn(z, __uint_as_float((127u - e) << 23));
  }
  return z;
}

__global__ void k_generate(int dist, uint64_t base, uint64_t base_row, size_t n, size_t n_emb,
                           float* __restrict__ out) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  const size_t nv = n / 4;
  float4* o4 = reinterpret_cast<float4*>(out);
  const bool aligned = ((uintptr_t)out & 15) == 0;
  if (aligned) {
    for (size_t v = (size_t)blockIdx.x * blockDim.x + threadIdx.x; v < nv; v += stride) {
      const size_t i = v * 4;
      o4[v] = make_float4(gen_one(dist, base, base_row, n_emb, i),
                          gen_one(dist, base, base_row, n_emb, i + 1),
                          gen_one(dist, base, base_row, n_emb, i + 2),
                          gen_one(dist, base, base_row, n_emb, i + 3));
    }
    for (size_t i = nv * 4 + (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
      out[i] = gen_one(dist, base, base_row, n_emb, i);
  } else {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
      out[i] = gen_one(dist, base, base_row, n_emb, i);
  }
}

uint64_t host_mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

}  // namespace

extern "C" psb_status psb_generate(psb_dist dist, uint64_t seed, uint32_t rank, uint32_t step,
                                   size_t n, float* out, psb_stream_t stream) {
  if (n == 0) return PSB_OK;
  if (!out || (int)dist < 0 || (int)dist > 2) return PSB_EINVAL;
  const uint64_t base = host_mix64(seed ^ (((uint64_t)rank << 32) | (uint64_t)step));
  const uint64_t base_row = host_mix64(base ^ 0x5851F42D4C957F2DULL);
  const size_t n_emb = (n * 3 / 5) & ~(size_t)63;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const unsigned grid = (unsigned)std::min<size_t>((n / 4 + 255) / 256 + 1, (size_t)sms * 16);
  k_generate<<<grid, 256, 0, (cudaStream_t)stream>>>((int)dist, base, base_row, n, n_emb, out);
  return cudaGetLastError() == cudaSuccess ? PSB_OK : PSB_ECUDA;
}
