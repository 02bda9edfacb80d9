// psb_wire.cu -- the reference's wire encoding of compressed messages, on
// the device.
//
// Replaces wire_encode / wire_decode (parsim/compression.hpp:159-239),
// little-endian throughout:
//   Dense:   u64 dim | dim x f64
//   SignBit: u64 dim | f64 scale | ceil(dim/8) sign bytes (bit i%8 of byte i/8)
//   TopK:    u64 dim | u64 count | count x (u64 index, f64 value)
// Values travel as f64 (the reference's DenseVector): f32 payloads widen
// exactly on encode; decoding into f32 rounds to nearest (exact for messages
// that came from f32).  The sign words of psb_ef_onebit are byte-identical to
// the reference's sign bytes, so that body is a straight copy.
// Every record is one 16-byte store: the encoders run at copy bandwidth.
#include "psb_internal.cuh"

namespace {

template <class T>
__global__ void k_wire_encode_topk(uint64_t dim, const uint32_t* __restrict__ idx, const T* __restrict__ val,
                                   size_t k, uint8_t* __restrict__ out) {
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    reinterpret_cast<unsigned long long*>(out)[0] = dim;
    reinterpret_cast<unsigned long long*>(out)[1] = k;
  }
  ulonglong2* rec = reinterpret_cast<ulonglong2*>(out + 16);
  for (size_t j = (size_t)blockIdx.x * blockDim.x + threadIdx.x; j < k; j += (size_t)gridDim.x * blockDim.x)
    rec[j] = make_ulonglong2((unsigned long long)idx[j],
                             (unsigned long long)__double_as_longlong((double)val[j]));
}

// hdr[0] = dim, hdr[1] = count are read back by the host wrapper; flags: 16 =
// truncated, 32 = count over the caller's capacity, 64 = index >= 2^32
template <class T>
__global__ void k_wire_decode_topk(const uint8_t* __restrict__ in, size_t nbytes, size_t k_cap,
                                   uint32_t* __restrict__ idx, T* __restrict__ val,
                                   unsigned long long* __restrict__ hdr, uint32_t* flags) {
  if (nbytes < 16) {
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicOr(flags, 16u);
    return;
  }
  const unsigned long long dim = reinterpret_cast<const unsigned long long*>(in)[0];
  const unsigned long long count = reinterpret_cast<const unsigned long long*>(in)[1];
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    hdr[0] = dim;
    hdr[1] = count;
  }
  if (count > (nbytes - 16) / 16) {
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicOr(flags, 16u);
    return;
  }
  if (count > k_cap) {
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicOr(flags, 32u);
    return;
  }
  const ulonglong2* rec = reinterpret_cast<const ulonglong2*>(in + 16);
  uint32_t f = 0;
  for (size_t j = (size_t)blockIdx.x * blockDim.x + threadIdx.x; j < count; j += (size_t)gridDim.x * blockDim.x) {
    const ulonglong2 r = rec[j];
    if (r.x >> 32) f |= 64u;
    idx[j] = (uint32_t)r.x;
    val[j] = (T)__longlong_as_double((long long)r.y);
  }
  if (f) atomicOr(flags, f);
}

__global__ void k_wire_encode_signbit(uint64_t dim, const uint32_t* __restrict__ words,
                                      const double* __restrict__ scale, uint8_t* __restrict__ out) {
  const size_t nb = (size_t)((dim + 7) / 8);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    reinterpret_cast<unsigned long long*>(out)[0] = dim;
    reinterpret_cast<double*>(out)[1] = *scale;
  }
  const uint8_t* src = reinterpret_cast<const uint8_t*>(words);
  for (size_t b = (size_t)blockIdx.x * blockDim.x + threadIdx.x; b < nb; b += (size_t)gridDim.x * blockDim.x)
    out[16 + b] = src[b];
}

template <class T>
__global__ void k_wire_encode_dense(uint64_t dim, const T* __restrict__ x, uint8_t* __restrict__ out) {
  if (blockIdx.x == 0 && threadIdx.x == 0) reinterpret_cast<unsigned long long*>(out)[0] = dim;
  double* v = reinterpret_cast<double*>(out + 8);
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < dim; i += (size_t)gridDim.x * blockDim.x)
    v[i] = (double)x[i];
}

unsigned grid_for(const psb_ctx* c, size_t work) {
  return (unsigned)std::max<size_t>(1, std::min<size_t>((work + 255) / 256, (size_t)c->num_sms * 8));
}

}  // namespace

extern "C" size_t psb_wire_bytes(psb_wire_kind kind, uint64_t dim, size_t k) {
  switch (kind) {
    case PSB_WIRE_DENSE: return 8 + 8 * (size_t)dim;
    case PSB_WIRE_SIGNBIT: return 16 + (size_t)((dim + 7) / 8);
    case PSB_WIRE_TOPK: return 16 + 16 * k;
  }
  return 0;
}

extern "C" psb_status psb_wire_encode_topk(psb_ctx* c, psb_dtype dt, uint64_t dim, const uint32_t* idx,
                                           const void* val, size_t k, void* out, psb_stream_t stream) {
  PSB_REQUIRE(c, c != nullptr, "null ctx");
  PSB_REQUIRE(c, dt == PSB_F32 || dt == PSB_F64, "wire_encode: bad dtype");
  PSB_REQUIRE(c, out != nullptr && (k == 0 || (idx && val)), "wire_encode: null pointer");
  PSB_REQUIRE(c, ((uintptr_t)out & 15) == 0, "wire_encode: output must be 16-byte aligned");
  cudaStream_t st = (cudaStream_t)stream;
  uint8_t* o = reinterpret_cast<uint8_t*>(out);
  if (dt == PSB_F32) k_wire_encode_topk<float><<<grid_for(c, k), 256, 0, st>>>(dim, idx, (const float*)val, k, o);
  else k_wire_encode_topk<double><<<grid_for(c, k), 256, 0, st>>>(dim, idx, (const double*)val, k, o);
  c->launches += 1;
  PSB_LAUNCH_CHECK(c, "psb_wire_encode_topk");
  return PSB_OK;
}

extern "C" psb_status psb_wire_decode_topk(psb_ctx* c, psb_dtype dt, const void* in, size_t nbytes, size_t k_cap,
                                           uint32_t* idx, void* val, uint64_t* dim_out, size_t* count_out,
                                           psb_stream_t stream) {
  PSB_REQUIRE(c, c != nullptr, "null ctx");
  PSB_REQUIRE(c, dt == PSB_F32 || dt == PSB_F64, "wire_decode: bad dtype");
  PSB_REQUIRE(c, in != nullptr && idx && val && dim_out && count_out, "wire_decode: null pointer");
  PSB_REQUIRE(c, ((uintptr_t)in & 15) == 0, "wire_decode: input must be 16-byte aligned");
  cudaStream_t st = (cudaStream_t)stream;
  unsigned long long* hdr = reinterpret_cast<unsigned long long*>(c->d_flags + 8);  // 2 x u64 scratch
  const uint8_t* i8 = reinterpret_cast<const uint8_t*>(in);
  const size_t work = nbytes >= 16 ? (nbytes - 16) / 16 : 1;
  // the decoder reports through its own flag word (d_flags[4]), so the
  // sticky step flags (d_flags[0]: non-finite, peer timeout) stay untouched
  // for the caller's next psb_check
  uint32_t* dflag = c->d_flags + 4;
  CUDA_TRY(c, cudaMemsetAsync(dflag, 0, sizeof(uint32_t), st), "psb_wire_decode_topk");
  if (dt == PSB_F32)
    k_wire_decode_topk<float><<<grid_for(c, work), 256, 0, st>>>(i8, nbytes, k_cap, idx, (float*)val, hdr, dflag);
  else
    k_wire_decode_topk<double><<<grid_for(c, work), 256, 0, st>>>(i8, nbytes, k_cap, idx, (double*)val, hdr,
                                                                   dflag);
  c->launches += 1;
  PSB_LAUNCH_CHECK(c, "psb_wire_decode_topk");
  unsigned long long h[2] = {0, 0};
  uint32_t f = 0;
  CUDA_TRY(c, cudaMemcpyAsync(h, hdr, sizeof(h), cudaMemcpyDeviceToHost, st), "psb_wire_decode_topk");
  CUDA_TRY(c, cudaMemcpyAsync(&f, dflag, sizeof(f), cudaMemcpyDeviceToHost, st), "psb_wire_decode_topk");
  CUDA_TRY(c, cudaStreamSynchronize(st), "psb_wire_decode_topk");
  if (f & 16u) return psb_set_err(c, PSB_EINVAL, "wire_decode: truncated input");
  if (f & 32u) return psb_set_err(c, PSB_EINVAL, "wire_decode: message exceeds the output capacity");
  if (f & 64u) return psb_set_err(c, PSB_EINVAL, "wire_decode: index exceeds the 32-bit range");
  *dim_out = h[0];
  *count_out = (size_t)h[1];
  return PSB_OK;
}

extern "C" psb_status psb_wire_encode_signbit(psb_ctx* c, uint64_t dim, const uint32_t* words,
                                              const double* scale, void* out, psb_stream_t stream) {
  PSB_REQUIRE(c, c != nullptr, "null ctx");
  PSB_REQUIRE(c, words && scale && out, "wire_encode: null pointer");
  cudaStream_t st = (cudaStream_t)stream;
  k_wire_encode_signbit<<<grid_for(c, (dim + 7) / 8), 256, 0, st>>>(dim, words, scale, (uint8_t*)out);
  c->launches += 1;
  PSB_LAUNCH_CHECK(c, "psb_wire_encode_signbit");
  return PSB_OK;
}

extern "C" psb_status psb_wire_encode_dense(psb_ctx* c, psb_dtype dt, const void* x, uint64_t dim, void* out,
                                            psb_stream_t stream) {
  PSB_REQUIRE(c, c != nullptr, "null ctx");
  PSB_REQUIRE(c, dt == PSB_F32 || dt == PSB_F64, "wire_encode: bad dtype");
  PSB_REQUIRE(c, x && out, "wire_encode: null pointer");
  PSB_REQUIRE(c, ((uintptr_t)out & 7) == 0, "wire_encode: output must be 8-byte aligned");
  cudaStream_t st = (cudaStream_t)stream;
  if (dt == PSB_F32) k_wire_encode_dense<float><<<grid_for(c, dim), 256, 0, st>>>(dim, (const float*)x, (uint8_t*)out);
  else k_wire_encode_dense<double><<<grid_for(c, dim), 256, 0, st>>>(dim, (const double*)x, (uint8_t*)out);
  c->launches += 1;
  PSB_LAUNCH_CHECK(c, "psb_wire_encode_dense");
  return PSB_OK;
}
