// psb_q8.cu -- 8-bit per-block quantizer and the dense 8-bit all-reduce.
//
// NO REFERENCE CODE: multi-bit quantization is a non-goal of the reference
// (SPEC.md:182); the rule implemented here is specified, and restated on the
// CPU, in oracle/psb_oracle.c:orc_q8_quant:
//   per block of B consecutive elements: scale = absmax / 127  (IEEE f32 div)
//   code = clamp(rint(p / scale), -127, 127)  (IEEE div, round-half-even), 0 if scale == 0
//   xhat = code * scale;  error feedback r' = p - xhat (compression.hpp:153-154 shape)
// One warp per block; each lane owns 4 consecutive elements per 128-element
// row (float4 / char4 accesses); the next block's loads are issued before the
// current block is processed (register double buffer) to keep HBM busy.
//
// Dense 8-bit "hierarchical" all-reduce (cfg3), P = W local workers x R ranks:
//   1. quantize each local worker's p = r + g          (k_q8_quant)
//   2. all-to-all of int8 shards + scales (NCCL grouped send/recv): rank q
//      receives block-shard q of every worker
//   3. k_q8_reduce: fold the P dequantized values in the configured
//      reference order (collectives.hpp:68-128), * (1/P), requantize the mean
//      per block; with R == 1 also apply SGD in the same pass
//   4. NCCL allgather of the requantized shards
//   5. k_q8_apply: theta = (-lr) * (code*scale) + theta (no FMA)
#include "psb_fold.cuh"

namespace {

// code = clamp(rint(RN(p / scale)), -127, 127), bit-identical to the IEEE
// division of the spec, but computed from y = p * inv (inv = RN(1/scale), one
// division per block): |y - RN(p/scale)| <= 3 ulp, so rint(y) == rint(RN(p/scale))
// unless y lies within 3 ulp (< 6.1e-5 for |y| < 128) of a half-integer; those
// rare lanes, and a non-finite inv, take the exact division.
__device__ __forceinline__ int q8_code(float p, float scale, float inv) {
  if (!(scale > 0.f)) return 0;
  const float y = __fmul_rn(p, inv);
  const float fr = fabsf(y - rintf(y));
  int q;
  if (is_finite(inv) && fabsf(fr - 0.5f) > 6.1e-5f) q = __float2int_rn(y);
  else q = __float2int_rn(__fdiv_rn(p, scale));
  return q > 127 ? 127 : (q < -127 ? -127 : q);
}

// Loads one block's p = r + x for this lane: VPL rows of 4 elements.
template <int VPL>
__device__ __forceinline__ void q8_load(const float* __restrict__ x, const float* __restrict__ r, size_t n,
                                        size_t lo, bool full, int lane, float (&p)[VPL][4]) {
#pragma unroll
  for (int it = 0; it < VPL; ++it) {
    const size_t e = lo + (size_t)it * 128 + lane * 4;
    if (full) {
      const float4 xv = __ldcs(reinterpret_cast<const float4*>(x + e));
      if (r) {
        const float4 rv = __ldcs(reinterpret_cast<const float4*>(r + e));
        p[it][0] = __fadd_rn(rv.x, xv.x);
        p[it][1] = __fadd_rn(rv.y, xv.y);
        p[it][2] = __fadd_rn(rv.z, xv.z);
        p[it][3] = __fadd_rn(rv.w, xv.w);
      } else {
        p[it][0] = xv.x; p[it][1] = xv.y; p[it][2] = xv.z; p[it][3] = xv.w;
      }
    } else {
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const size_t ei = e + c;
        p[it][c] = ei < n ? (r ? __fadd_rn(r[ei], x[ei]) : x[ei]) : 0.f;
      }
    }
  }
}

template <int VPL>
__global__ void __launch_bounds__(256) k_q8_quant(const float* __restrict__ x, float* __restrict__ r,
                                                  size_t n, int8_t* __restrict__ codes,
                                                  float* __restrict__ scales, uint32_t* flags) {
  constexpr int B = VPL * 128;
  const int lane = threadIdx.x & 31;
  const size_t nb = (n + B - 1) / B;
  const size_t warp = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const size_t nwarps = ((size_t)gridDim.x * blockDim.x) >> 5;
  const bool vec_ok = ((((uintptr_t)x) | ((uintptr_t)r) | ((uintptr_t)codes)) & 15) == 0;
  bool bad = false;
  float p[VPL][4];
  size_t blk = warp;
  if (blk < nb) q8_load<VPL>(x, r, n, blk * B, vec_ok && blk * B + B <= n, lane, p);
  for (; blk < nb; blk += nwarps) {
    const size_t lo = blk * B;
    const bool full = vec_ok && lo + B <= n;
    // prefetch the next block of this warp before working on this one
    float pn[VPL][4];
    const size_t nxt = blk + nwarps;
    if (nxt < nb) q8_load<VPL>(x, r, n, nxt * B, vec_ok && nxt * B + B <= n, lane, pn);
    float amax = 0.f;
#pragma unroll
    for (int it = 0; it < VPL; ++it)
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        amax = fmaxf(amax, fabsf(p[it][c]));
        bad |= !is_finite(p[it][c]);
      }
#pragma unroll
    for (int o = 16; o; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    const float scale = __fdiv_rn(amax, 127.0f);
    const float inv = __frcp_rn(scale);
    if (lane == 0) scales[blk] = scale;
#pragma unroll
    for (int it = 0; it < VPL; ++it) {
      const size_t e = lo + (size_t)it * 128 + lane * 4;
      int q[4];
      float res[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        q[c] = q8_code(p[it][c], scale, inv);
        res[c] = __fsub_rn(p[it][c], __fmul_rn((float)q[c], scale));
      }
      if (full) {
        *reinterpret_cast<char4*>(codes + e) =
            make_char4((signed char)q[0], (signed char)q[1], (signed char)q[2], (signed char)q[3]);
        if (r) __stcs(reinterpret_cast<float4*>(r + e), make_float4(res[0], res[1], res[2], res[3]));
      } else {
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          if (e + c < n) {
            codes[e + c] = (int8_t)q[c];
            if (r) r[e + c] = res[c];
          }
        }
      }
    }
#pragma unroll
    for (int it = 0; it < VPL; ++it)
#pragma unroll
      for (int c = 0; c < 4; ++c) p[it][c] = pn[it][c];
  }
  if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(flags, 1u);
}

__global__ void k_q8_dequant(const int8_t* __restrict__ codes, const float* __restrict__ scales,
                             size_t n, uint32_t B, float* __restrict__ out) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x)
    out[i] = __fmul_rn((float)codes[i], scales[i / B]);
}

__device__ __forceinline__ float4 add4(float4 a, float4 b) {
  return make_float4(__fadd_rn(a.x, b.x), __fadd_rn(a.y, b.y), __fadd_rn(a.z, b.z), __fadd_rn(a.w, b.w));
}

// The reference fold orders (psb_fold.cuh) on 4 consecutive elements at once;
// ring_start is the rotated first worker of their (common) ring chunk.
template <class Get4>
__device__ __forceinline__ float4 fold_sum4(const Get4& get4, int P, int order, int ring_start,
                                            uint32_t dpn, uint32_t npr) {
  float4 acc;
  if (order == PSB_ORDER_RING) {
    acc = get4(ring_start);
    for (int s = 1; s < P; ++s) {
      int q = ring_start + s;
      if (q >= P) q -= P;
      acc = add4(acc, get4(q));
    }
  } else if (order == PSB_ORDER_HIER && dpn < (uint32_t)P) {
    const uint32_t nodes = ((uint32_t)P + dpn - 1) / dpn;
    float4 total = make_float4(0.f, 0.f, 0.f, 0.f);
    bool have_total = false;
    for (uint32_t nb = 0; nb < nodes; nb += npr) {
      float4 rack = make_float4(0.f, 0.f, 0.f, 0.f);
      bool have_rack = false;
      for (uint32_t nd = nb; nd < nodes && nd < nb + npr; ++nd) {
        const uint32_t base = nd * dpn;
        float4 node = get4((int)base);
        for (uint32_t p = base + 1; p < base + dpn && p < (uint32_t)P; ++p) node = add4(node, get4((int)p));
        rack = have_rack ? add4(rack, node) : node;
        have_rack = true;
      }
      total = have_total ? add4(total, rack) : rack;
      have_total = true;
    }
    acc = total;
  } else {
    acc = get4(0);
    for (int q = 1; q < P; ++q) acc = add4(acc, get4(q));
  }
  return acc;
}

__device__ __forceinline__ uint32_t ring_chunk(size_t i, size_t n, int P) {
  uint32_t j = (uint32_t)((i * (size_t)P) / n);
  while (j + 1 < (uint32_t)P && ((size_t)(j + 1) * n) / (size_t)P <= i) ++j;
  while (j > 0 && ((size_t)j * n) / (size_t)P > i) --j;
  return j;
}

// Fold P workers' dequantized values over blocks [blk_lo, blk_hi) (global block
// ids), requantize the mean per block into (mcodes, mscales) at global offsets,
// and, when theta != nullptr, apply SGD directly (single-rank path).
// Worker q's codes for global element e live at wcodes + q*wstride + (e - e_base),
// scales at wscales + q*sstride + (blk - blk_lo).
template <int VPL>
__global__ void __launch_bounds__(256) k_q8_reduce(
    Q8Workers wv, int P, size_t blk_lo, size_t blk_hi, size_t n, int order, uint32_t dpn,
    uint32_t npr, int8_t* __restrict__ mcodes, float* __restrict__ mscales, float coef,
    float* __restrict__ theta, float* __restrict__ mean_out, uint32_t* flags) {
  constexpr int B = VPL * 128;
  const int lane = threadIdx.x & 31;
  const size_t warp = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const size_t nwarps = ((size_t)gridDim.x * blockDim.x) >> 5;
  const size_t e_base = blk_lo * B;
  const float inv = (float)(1.0 / (double)P);
  uintptr_t al = ((uintptr_t)mcodes) | ((uintptr_t)theta);
  for (int q = 0; q < P; ++q) al |= (uintptr_t)wv.codes[q];
  const bool vec_ok = (al & 15) == 0 && !mean_out;
  bool bad = false;
  RingChunk rc;
  for (size_t blk = blk_lo + warp; blk < blk_hi; blk += nwarps) {
    float m[VPL][4];
    float amax = 0.f;
    // issue the theta loads first: independent of the fold, overlaps its latency
    float4 thv[VPL];
    if (theta && vec_ok) {
#pragma unroll
      for (int it = 0; it < VPL; ++it) {
        const size_t e0 = blk * B + (size_t)it * 128 + lane * 4;
        if (e0 + 4 <= n) thv[it] = __ldcs(reinterpret_cast<const float4*>(theta + e0));
      }
    }
#pragma unroll
    for (int it = 0; it < VPL; ++it) {
      const size_t e0 = blk * B + (size_t)it * 128 + lane * 4;
      const bool full = vec_ok && e0 + 4 <= n;
      int rs0 = 0;
      bool same_chunk = true;
      if (order == PSB_ORDER_RING) {  // cached: divisions only when the chunk changes
        rs0 = rc.start_for(e0, n, P);
        same_chunk = e0 + 3 < rc.hi;
      }
      if (full && same_chunk) {
        auto get4 = [&](int q) -> float4 {
          const char4 cv = *reinterpret_cast<const char4*>(wv.codes[q] + (e0 - e_base));
          const float sc = wv.scales[q][blk - blk_lo];
          return make_float4(__fmul_rn((float)cv.x, sc), __fmul_rn((float)cv.y, sc),
                             __fmul_rn((float)cv.z, sc), __fmul_rn((float)cv.w, sc));
        };
        const float4 s = fold_sum4(get4, P, order, rs0, dpn, npr);
        m[it][0] = __fmul_rn(s.x, inv);
        m[it][1] = __fmul_rn(s.y, inv);
        m[it][2] = __fmul_rn(s.z, inv);
        m[it][3] = __fmul_rn(s.w, inv);
      } else {
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const size_t e = e0 + c;
          float mean = 0.f;
          if (e < n) {
            auto get = [&](int q) -> float {
              const int8_t code = wv.codes[q][e - e_base];
              const float sc = wv.scales[q][blk - blk_lo];
              return __fmul_rn((float)code, sc);
            };
            mean = __fmul_rn(fold_sum<float>(get, P, order, e, n, dpn, npr), inv);
          }
          m[it][c] = mean;
        }
      }
#pragma unroll
      for (int c = 0; c < 4; ++c) amax = fmaxf(amax, fabsf(m[it][c]));
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    const float scale = __fdiv_rn(amax, 127.0f);
    const float inv = __frcp_rn(scale);
    if (lane == 0) mscales[blk] = scale;
#pragma unroll
    for (int it = 0; it < VPL; ++it) {
      const size_t e0 = blk * B + (size_t)it * 128 + lane * 4;
      int q[4];
      float mh[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        q[c] = q8_code(m[it][c], scale, inv);
        mh[c] = __fmul_rn((float)q[c], scale);
      }
      if (vec_ok && e0 + 4 <= n) {
        *reinterpret_cast<char4*>(mcodes + e0) =
            make_char4((signed char)q[0], (signed char)q[1], (signed char)q[2], (signed char)q[3]);
        if (theta) {
          float4 th = thv[it];
          th.x = __fadd_rn(__fmul_rn(coef, mh[0]), th.x);
          th.y = __fadd_rn(__fmul_rn(coef, mh[1]), th.y);
          th.z = __fadd_rn(__fmul_rn(coef, mh[2]), th.z);
          th.w = __fadd_rn(__fmul_rn(coef, mh[3]), th.w);
          __stcs(reinterpret_cast<float4*>(theta + e0), th);
          bad |= !is_finite(th.x) || !is_finite(th.y) || !is_finite(th.z) || !is_finite(th.w);
        }
      } else {
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const size_t e = e0 + c;
          if (e >= n) continue;
          mcodes[e] = (int8_t)q[c];
          if (theta) {
            const float th = __fadd_rn(__fmul_rn(coef, mh[c]), theta[e]);
            theta[e] = th;
            if (mean_out) mean_out[e] = mh[c];
            bad |= !is_finite(th);
          }
        }
      }
    }
  }
  if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(flags, 1u);
}

// k_q8_reduce for the multi-rank path's common case (compile-time P, the
// plain worker-order fold -- naive, or hierarchical within one node -- full
// blocks, no theta): each warp holds the codes and scales of its NEXT block in
// registers while it folds the current one, so a block's loads overlap the
// previous block's fold / requantize instead of exposing DRAM latency per
// block.  Same per-element operations as k_q8_reduce.
template <int VPL, int PT>
__global__ void __launch_bounds__(256) k_q8_reduce_pipe(Q8Workers wv, size_t blk_lo, size_t blk_hi,
                                                        int8_t* __restrict__ mcodes, float* __restrict__ mscales) {
  constexpr int B = VPL * 128;
  const int lane = threadIdx.x & 31;
  const size_t warp = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const size_t nwarps = ((size_t)gridDim.x * blockDim.x) >> 5;
  const size_t e_base = blk_lo * B;
  const float inv = (float)(1.0 / (double)PT);
  char4 cc[PT][VPL], cn[PT][VPL];
  float sc[PT], sn[PT];
  auto load = [&](size_t blk, char4 (&c)[PT][VPL], float (&sv)[PT]) {
#pragma unroll
    for (int q = 0; q < PT; ++q) {
#pragma unroll
      for (int it = 0; it < VPL; ++it)
        c[q][it] = *reinterpret_cast<const char4*>(wv.codes[q] + (blk * B - e_base) + (size_t)it * 128 + lane * 4);
      sv[q] = wv.scales[q][blk - blk_lo];
    }
  };
  size_t blk = blk_lo + warp;
  if (blk < blk_hi) load(blk, cc, sc);
  for (; blk < blk_hi; blk += nwarps) {
    const size_t nxt = blk + nwarps;
    if (nxt < blk_hi) load(nxt, cn, sn);
    float m[VPL][4];
    float amax = 0.f;
#pragma unroll
    for (int it = 0; it < VPL; ++it) {
      float4 acc = make_float4(__fmul_rn((float)cc[0][it].x, sc[0]), __fmul_rn((float)cc[0][it].y, sc[0]),
                               __fmul_rn((float)cc[0][it].z, sc[0]), __fmul_rn((float)cc[0][it].w, sc[0]));
#pragma unroll
      for (int q = 1; q < PT; ++q) {
        acc.x = __fadd_rn(acc.x, __fmul_rn((float)cc[q][it].x, sc[q]));
        acc.y = __fadd_rn(acc.y, __fmul_rn((float)cc[q][it].y, sc[q]));
        acc.z = __fadd_rn(acc.z, __fmul_rn((float)cc[q][it].z, sc[q]));
        acc.w = __fadd_rn(acc.w, __fmul_rn((float)cc[q][it].w, sc[q]));
      }
      m[it][0] = __fmul_rn(acc.x, inv);
      m[it][1] = __fmul_rn(acc.y, inv);
      m[it][2] = __fmul_rn(acc.z, inv);
      m[it][3] = __fmul_rn(acc.w, inv);
#pragma unroll
      for (int c = 0; c < 4; ++c) amax = fmaxf(amax, fabsf(m[it][c]));
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    const float scale = __fdiv_rn(amax, 127.0f);
    const float rinv = __frcp_rn(scale);
    if (lane == 0) mscales[blk] = scale;
#pragma unroll
    for (int it = 0; it < VPL; ++it) {
      const size_t e0 = blk * B + (size_t)it * 128 + lane * 4;
      *reinterpret_cast<char4*>(mcodes + e0) =
          make_char4((signed char)q8_code(m[it][0], scale, rinv), (signed char)q8_code(m[it][1], scale, rinv),
                     (signed char)q8_code(m[it][2], scale, rinv), (signed char)q8_code(m[it][3], scale, rinv));
    }
#pragma unroll
    for (int q = 0; q < PT; ++q) {
      sc[q] = sn[q];
#pragma unroll
      for (int it = 0; it < VPL; ++it) cc[q][it] = cn[q][it];
    }
  }
}

constexpr int kQ8Stages = 4;  // TMA ring depth of the q8 kernels

// The multi-rank reduce reading every worker's codes and scales of this
// rank's shard in place (local arena or the peers' NVLink-mapped arenas) with
// 1-D TMA bulk copies into a kQ8Stages ring of 8-block tiles, instead of a
// pull into local memory followed by k_q8_reduce_pipe.  Same per-element
// operations (compile-time P, plain worker-order fold).  Full tiles only; the
// host reduces a ragged tail with k_q8_reduce*.
template <int VPL, int PT>
__global__ void __launch_bounds__(256) k_q8_reduce_tma(Q8Workers wv, size_t blk_lo, size_t ntiles,
                                                       int8_t* __restrict__ mcodes, float* __restrict__ mscales) {
  constexpr int B = VPL * 128;
  constexpr uint32_t CB = 8 * B;        // code bytes per worker per tile
  constexpr uint32_t SB = 8 * 4;        // scale bytes per worker per tile
  constexpr uint32_t STG = PT * (CB + SB);
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t full[kQ8Stages];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const size_t my_tiles = ntiles > blockIdx.x ? (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kQ8Stages; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](size_t i) {
    const int s = (int)(i % kQ8Stages);
    const size_t t = blockIdx.x + i * gridDim.x;  // tile within the shard
    unsigned char* st = smem + (size_t)s * STG;
    mbar_expect_tx(&full[s], STG);
#pragma unroll
    for (int q = 0; q < PT; ++q) {
      tma_load_1d(st + (size_t)q * CB, wv.codes[q] + t * CB, CB, &full[s]);
      tma_load_1d(st + (size_t)PT * CB + (size_t)q * SB, wv.scales[q] + t * 8, SB, &full[s]);
    }
  };
  if (threadIdx.x == 0)
    for (size_t i = 0; i < my_tiles && i < (size_t)kQ8Stages; ++i) issue(i);
  const float inv = (float)(1.0 / (double)PT);
  for (size_t i = 0; i < my_tiles; ++i) {
    const int s = (int)(i % kQ8Stages);
    mbar_wait(&full[s], (uint32_t)((i / kQ8Stages) & 1));
    const unsigned char* st = smem + (size_t)s * STG;
    const size_t blk = blk_lo + (blockIdx.x + i * gridDim.x) * 8 + wid;
    float sc[PT];
#pragma unroll
    for (int q = 0; q < PT; ++q) sc[q] = reinterpret_cast<const float*>(st + (size_t)PT * CB + (size_t)q * SB)[wid];
    float m[VPL][4];
    float amax = 0.f;
#pragma unroll
    for (int it = 0; it < VPL; ++it) {
      const int o = wid * B + it * 128 + lane * 4;
      char4 cv = *reinterpret_cast<const char4*>(st + o);
      float4 acc = make_float4(__fmul_rn((float)cv.x, sc[0]), __fmul_rn((float)cv.y, sc[0]),
                               __fmul_rn((float)cv.z, sc[0]), __fmul_rn((float)cv.w, sc[0]));
#pragma unroll
      for (int q = 1; q < PT; ++q) {
        cv = *reinterpret_cast<const char4*>(st + (size_t)q * CB + o);
        acc.x = __fadd_rn(acc.x, __fmul_rn((float)cv.x, sc[q]));
        acc.y = __fadd_rn(acc.y, __fmul_rn((float)cv.y, sc[q]));
        acc.z = __fadd_rn(acc.z, __fmul_rn((float)cv.z, sc[q]));
        acc.w = __fadd_rn(acc.w, __fmul_rn((float)cv.w, sc[q]));
      }
      m[it][0] = __fmul_rn(acc.x, inv);
      m[it][1] = __fmul_rn(acc.y, inv);
      m[it][2] = __fmul_rn(acc.z, inv);
      m[it][3] = __fmul_rn(acc.w, inv);
#pragma unroll
      for (int c = 0; c < 4; ++c) amax = fmaxf(amax, fabsf(m[it][c]));
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    const float scale = __fdiv_rn(amax, 127.0f);
    const float rinv = __frcp_rn(scale);
    if (lane == 0) mscales[blk] = scale;
#pragma unroll
    for (int it = 0; it < VPL; ++it) {
      const size_t e0 = blk * B + (size_t)it * 128 + lane * 4;
      *reinterpret_cast<char4*>(mcodes + e0) =
          make_char4((signed char)q8_code(m[it][0], scale, rinv), (signed char)q8_code(m[it][1], scale, rinv),
                     (signed char)q8_code(m[it][2], scale, rinv), (signed char)q8_code(m[it][3], scale, rinv));
    }
    __syncthreads();  // every warp is done with stage s
    if (threadIdx.x == 0 && i + kQ8Stages < my_tiles) issue(i + kQ8Stages);
  }
}

// Single-rank fused step (R == 1): per block of B elements, each local worker
// q's p = r + g is quantized (codes stay in registers), r' = p - xhat written,
// and xhat = code*scale folded in the reference order; the mean is requantized
// per block and applied to theta.  Bitwise the same as k_q8_quant followed by
// k_q8_reduce (same per-element operations in the same order), without the
// int8 round trip through HBM: 12 B/element per worker + 8 B theta.
// Fold orders handled sequentially: naive, hierarchical (node/rack/total
// accumulators), and ring when P == 1; the host uses the unfused path for a
// ring fold over several local workers (its start worker varies per chunk).
// The warp walks (block, worker) items; the next item's loads are issued
// before the current one is processed (register double buffer).
template <int VPL, bool HIER>
__global__ void __launch_bounds__(256) k_q8_step1(const float* __restrict__ g, size_t gstride,
                                                  float* __restrict__ r, size_t rstride, int P, size_t n,
                                                  int order, uint32_t dpn, uint32_t npr, float coef,
                                                  float* __restrict__ theta, float* __restrict__ mean_out,
                                                  uint32_t* flags) {
  constexpr int B = VPL * 128;
  const int lane = threadIdx.x & 31;
  const size_t nb = (n + B - 1) / B;
  const size_t warp = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const size_t nwarps = ((size_t)gridDim.x * blockDim.x) >> 5;
  const bool vec_ok = ((((uintptr_t)g) | ((uintptr_t)r) | ((uintptr_t)theta) | ((uintptr_t)mean_out) |
                        (gstride * 4) | (rstride * 4)) & 15) == 0;
  const float inv_p = (float)(1.0 / (double)P);
  bool bad = false;
  auto load = [&](size_t blk, int q, float (&p)[VPL][4]) {
    const size_t lo = blk * B;
    q8_load<VPL>(g + (size_t)q * gstride, r ? r + (size_t)q * rstride : nullptr, n, lo, vec_ok && lo + B <= n,
                 lane, p);
  };
  float p[VPL][4];
  size_t blk = warp;
  int q = 0;
  if (blk < nb) load(blk, 0, p);
  float acc[VPL][4], node[HIER ? VPL : 1][4], rack[HIER ? VPL : 1][4];
  float4 thv[VPL];
  while (blk < nb) {
    const size_t lo = blk * B;
    const bool full = vec_ok && lo + B <= n;
    if (q == 0 && full) {
#pragma unroll
      for (int it = 0; it < VPL; ++it)
        thv[it] = __ldcs(reinterpret_cast<const float4*>(theta + lo + (size_t)it * 128 + lane * 4));
    }
    // next item's loads first
    float pn[VPL][4];
    size_t nblk = blk;
    int nq = q + 1;
    if (nq == P) {
      nq = 0;
      nblk = blk + nwarps;
    }
    if (nblk < nb) load(nblk, nq, pn);
    // quantize worker q's block; EF residual; dequantized value x
    float amax = 0.f;
#pragma unroll
    for (int it = 0; it < VPL; ++it)
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        amax = fmaxf(amax, fabsf(p[it][c]));
        bad |= !is_finite(p[it][c]);
      }
#pragma unroll
    for (int o = 16; o; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    const float scale = __fdiv_rn(amax, 127.0f);
    const float inv = __frcp_rn(scale);
    float* rq = r ? r + (size_t)q * rstride : nullptr;
#pragma unroll
    for (int it = 0; it < VPL; ++it) {
      const size_t e = lo + (size_t)it * 128 + lane * 4;
      float x[4], res[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        x[c] = __fmul_rn((float)q8_code(p[it][c], scale, inv), scale);
        res[c] = __fsub_rn(p[it][c], x[c]);
      }
      if (rq) {
        if (full) {
          __stcs(reinterpret_cast<float4*>(rq + e), make_float4(res[0], res[1], res[2], res[3]));
        } else {
#pragma unroll
          for (int c = 0; c < 4; ++c)
            if (e + c < n) rq[e + c] = res[c];
        }
      }
      // fold (collectives.hpp:68-128 orders, sequential form)
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        if constexpr (!HIER) {
          acc[it][c] = q == 0 ? x[c] : __fadd_rn(acc[it][c], x[c]);
        } else {
          const uint32_t uq = (uint32_t)q, nd = uq / dpn;
          node[it][c] = uq % dpn == 0 ? x[c] : __fadd_rn(node[it][c], x[c]);
          if (uq % dpn == dpn - 1 || q == P - 1) {
            rack[it][c] = nd % npr == 0 ? node[it][c] : __fadd_rn(rack[it][c], node[it][c]);
            if (nd % npr == npr - 1 || q == P - 1)
              acc[it][c] = nd < npr ? rack[it][c] : __fadd_rn(acc[it][c], rack[it][c]);
          }
        }
      }
    }
    if (q == P - 1) {
      // mean, per-block requantization, SGD
      float m[VPL][4];
      float mmax = 0.f;
#pragma unroll
      for (int it = 0; it < VPL; ++it)
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          m[it][c] = __fmul_rn(acc[it][c], inv_p);
          mmax = fmaxf(mmax, fabsf(m[it][c]));
        }
#pragma unroll
      for (int o = 16; o; o >>= 1) mmax = fmaxf(mmax, __shfl_xor_sync(0xffffffffu, mmax, o));
      const float ms = __fdiv_rn(mmax, 127.0f);
      const float minv = __frcp_rn(ms);
#pragma unroll
      for (int it = 0; it < VPL; ++it) {
        const size_t e = lo + (size_t)it * 128 + lane * 4;
        float mh[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) mh[c] = __fmul_rn((float)q8_code(m[it][c], ms, minv), ms);
        if (full) {
          float4 th = thv[it];
          th.x = __fadd_rn(__fmul_rn(coef, mh[0]), th.x);
          th.y = __fadd_rn(__fmul_rn(coef, mh[1]), th.y);
          th.z = __fadd_rn(__fmul_rn(coef, mh[2]), th.z);
          th.w = __fadd_rn(__fmul_rn(coef, mh[3]), th.w);
          __stcs(reinterpret_cast<float4*>(theta + e), th);
          if (mean_out) *reinterpret_cast<float4*>(mean_out + e) = make_float4(mh[0], mh[1], mh[2], mh[3]);
          bad |= !is_finite(th.x) || !is_finite(th.y) || !is_finite(th.z) || !is_finite(th.w);
        } else {
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            if (e + c >= n) continue;
            const float th = __fadd_rn(__fmul_rn(coef, mh[c]), theta[e + c]);
            theta[e + c] = th;
            if (mean_out) mean_out[e + c] = mh[c];
            bad |= !is_finite(th);
          }
        }
      }
    }
#pragma unroll
    for (int it = 0; it < VPL; ++it)
#pragma unroll
      for (int c = 0; c < 4; ++c) p[it][c] = pn[it][c];
    blk = nblk;
    q = nq;
  }
  if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(flags, 1u);
}

// ---- TMA-pipelined single-worker step (W = P = 1, the cfg3 bench shape) ----
// The register double buffer of k_q8_step1 keeps ~64 B per lane in flight and
// three CTAs per SM resident (72 registers), which leaves HBM at ~70 % of its
// measured peak.  Here one elected thread streams tiles of 8 blocks (g, r and
// theta: 3 x 8*B*4 bytes) into a ring of kQ8Stages shared-memory stages with
// 1-D bulk copies (cp.async.bulk, mbarrier complete_tx), so the bytes in
// flight no longer depend on registers; each warp then quantizes one block
// of the stage exactly as k_q8_step1 does (same per-element operations, same
// order) and stores r' and theta' straight to global memory.

template <int VPL>
__global__ void __launch_bounds__(256) k_q8_step1_tma(const float* __restrict__ g, float* __restrict__ r, size_t n,
                                                      float coef, float* __restrict__ theta,
                                                      float* __restrict__ mean_out, uint32_t* flags) {
  constexpr int B = VPL * 128;
  constexpr int TE = 8 * B;                    // elements per tile (one block per warp)
  constexpr uint32_t kArr = TE * 4;            // bytes per array per stage
  extern __shared__ __align__(128) unsigned char smem[];
  float* sg = reinterpret_cast<float*>(smem);                    // [stage][TE]
  float* sr = sg + (size_t)kQ8Stages * TE;
  float* sth = sr + (size_t)kQ8Stages * TE;
  __shared__ __align__(8) uint64_t full[kQ8Stages];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const size_t ntiles_full = n / TE;  // TMA streams full tiles; a ragged tail is read directly
  const size_t my_tiles = ntiles_full > blockIdx.x ? (ntiles_full - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kQ8Stages; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](size_t i) {  // local tile i -> stage i % kQ8Stages
    const int s = (int)(i % kQ8Stages);
    const size_t base = (blockIdx.x + i * gridDim.x) * (size_t)TE;
    mbar_expect_tx(&full[s], 3 * kArr);
    tma_load_1d(sg + (size_t)s * TE, g + base, kArr, &full[s]);
    tma_load_1d(sr + (size_t)s * TE, r + base, kArr, &full[s]);
    tma_load_1d(sth + (size_t)s * TE, theta + base, kArr, &full[s]);
  };
  if (threadIdx.x == 0)
    for (size_t i = 0; i < my_tiles && i < (size_t)kQ8Stages; ++i) issue(i);
  bool bad = false;
  auto process = [&](const float* pg, const float* pr, const float* pth, size_t lo, bool from_smem) {
    // one block of B elements at global offset lo; pg/pr/pth point at its first element
    float p[VPL][4];
#pragma unroll
    for (int it = 0; it < VPL; ++it) {
      const int o = it * 128 + lane * 4;
      float4 gv, rv;
      if (from_smem) {
        gv = *reinterpret_cast<const float4*>(pg + o);
        rv = *reinterpret_cast<const float4*>(pr + o);
      } else {
        gv = make_float4(0.f, 0.f, 0.f, 0.f);
        rv = gv;
        float* gp = &gv.x;
        float* rp = &rv.x;
        for (int c = 0; c < 4; ++c)
          if (lo + o + c < n) {
            gp[c] = pg[o + c];
            rp[c] = pr[o + c];
          }
      }
      p[it][0] = __fadd_rn(rv.x, gv.x);
      p[it][1] = __fadd_rn(rv.y, gv.y);
      p[it][2] = __fadd_rn(rv.z, gv.z);
      p[it][3] = __fadd_rn(rv.w, gv.w);
    }
    float amax = 0.f;
#pragma unroll
    for (int it = 0; it < VPL; ++it)
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        amax = fmaxf(amax, fabsf(p[it][c]));
        bad |= !is_finite(p[it][c]);
      }
#pragma unroll
    for (int o = 16; o; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    const float scale = __fdiv_rn(amax, 127.0f);
    const float inv = __frcp_rn(scale);
    float m[VPL][4];
    float mmax = 0.f;
#pragma unroll
    for (int it = 0; it < VPL; ++it) {
      const size_t e = lo + (size_t)it * 128 + lane * 4;
      float res[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const float x = __fmul_rn((float)q8_code(p[it][c], scale, inv), scale);
        res[c] = __fsub_rn(p[it][c], x);
        m[it][c] = __fmul_rn(x, 1.0f);  // mean over P = 1: x * (1/1)
        mmax = fmaxf(mmax, fabsf(m[it][c]));
      }
      if (from_smem) {
        __stcs(reinterpret_cast<float4*>(r + e), make_float4(res[0], res[1], res[2], res[3]));
      } else {
        for (int c = 0; c < 4; ++c)
          if (e + c < n) r[e + c] = res[c];
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) mmax = fmaxf(mmax, __shfl_xor_sync(0xffffffffu, mmax, o));
    const float ms = __fdiv_rn(mmax, 127.0f);
    const float minv = __frcp_rn(ms);
#pragma unroll
    for (int it = 0; it < VPL; ++it) {
      const int o = it * 128 + lane * 4;
      const size_t e = lo + o;
      float mh[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) mh[c] = __fmul_rn((float)q8_code(m[it][c], ms, minv), ms);
      if (from_smem) {
        float4 th = *reinterpret_cast<const float4*>(pth + o);
        th.x = __fadd_rn(__fmul_rn(coef, mh[0]), th.x);
        th.y = __fadd_rn(__fmul_rn(coef, mh[1]), th.y);
        th.z = __fadd_rn(__fmul_rn(coef, mh[2]), th.z);
        th.w = __fadd_rn(__fmul_rn(coef, mh[3]), th.w);
        __stcs(reinterpret_cast<float4*>(theta + e), th);
        if (mean_out) *reinterpret_cast<float4*>(mean_out + e) = make_float4(mh[0], mh[1], mh[2], mh[3]);
        bad |= !is_finite(th.x) || !is_finite(th.y) || !is_finite(th.z) || !is_finite(th.w);
      } else {
        for (int c = 0; c < 4; ++c) {
          if (e + c >= n) continue;
          const float t2 = __fadd_rn(__fmul_rn(coef, mh[c]), pth[o + c]);
          theta[e + c] = t2;
          if (mean_out) mean_out[e + c] = mh[c];
          bad |= !is_finite(t2);
        }
      }
    }
  };
  for (size_t i = 0; i < my_tiles; ++i) {
    const int s = (int)(i % kQ8Stages);
    mbar_wait(&full[s], (uint32_t)((i / kQ8Stages) & 1));
    const size_t base = (blockIdx.x + i * gridDim.x) * (size_t)TE;
    const size_t off = (size_t)s * TE + (size_t)wid * B;
    process(sg + off, sr + off, sth + off, base + (size_t)wid * B, true);
    __syncthreads();  // every warp is done with stage s
    if (threadIdx.x == 0 && i + kQ8Stages < my_tiles) issue(i + kQ8Stages);
  }
  // ragged tail (blocks past the last full tile): CTA 0, one block per warp
  if (blockIdx.x == 0) {
    for (size_t lo = ntiles_full * TE + (size_t)wid * B; lo < n; lo += 8 * (size_t)B)
      process(g + lo, r + lo, theta + lo, lo, false);
  }
  if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(flags, 1u);
}

// The quantizer of the multi-rank path (EF on: x and r streamed) with the
// same TMA ring as k_q8_step1_tma: one elected thread streams tiles of 8
// blocks of x and r into kQ8Stages shared-memory stages; each warp quantizes
// one block (same per-element operations as k_q8_quant) and stores its codes,
// scale and residual.
template <int VPL>
__global__ void __launch_bounds__(256) k_q8_quant_tma(const float* __restrict__ x, float* __restrict__ r, size_t n,
                                                      int8_t* __restrict__ codes, float* __restrict__ scales,
                                                      uint32_t* flags) {
  constexpr int B = VPL * 128;
  constexpr int TE = 8 * B;
  constexpr uint32_t kArr = TE * 4;
  extern __shared__ __align__(128) unsigned char smem[];
  float* sx = reinterpret_cast<float*>(smem);  // [stage][TE]
  float* sr = sx + (size_t)kQ8Stages * TE;
  __shared__ __align__(8) uint64_t full[kQ8Stages];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const size_t ntiles_full = n / TE;
  const size_t my_tiles = ntiles_full > blockIdx.x ? (ntiles_full - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kQ8Stages; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](size_t i) {
    const int s = (int)(i % kQ8Stages);
    const size_t base = (blockIdx.x + i * gridDim.x) * (size_t)TE;
    mbar_expect_tx(&full[s], 2 * kArr);
    tma_load_1d(sx + (size_t)s * TE, x + base, kArr, &full[s]);
    tma_load_1d(sr + (size_t)s * TE, r + base, kArr, &full[s]);
  };
  if (threadIdx.x == 0)
    for (size_t i = 0; i < my_tiles && i < (size_t)kQ8Stages; ++i) issue(i);
  bool bad = false;
  auto process = [&](const float* px, const float* pr, size_t lo, bool from_smem) {
    float p[VPL][4];
#pragma unroll
    for (int it = 0; it < VPL; ++it) {
      const int o = it * 128 + lane * 4;
      float4 xv, rv;
      if (from_smem) {
        xv = *reinterpret_cast<const float4*>(px + o);
        rv = *reinterpret_cast<const float4*>(pr + o);
      } else {
        xv = make_float4(0.f, 0.f, 0.f, 0.f);
        rv = xv;
        float* xp = &xv.x;
        float* rp = &rv.x;
        for (int c = 0; c < 4; ++c)
          if (lo + o + c < n) {
            xp[c] = px[o + c];
            rp[c] = pr[o + c];
          }
      }
      p[it][0] = __fadd_rn(rv.x, xv.x);
      p[it][1] = __fadd_rn(rv.y, xv.y);
      p[it][2] = __fadd_rn(rv.z, xv.z);
      p[it][3] = __fadd_rn(rv.w, xv.w);
    }
    float amax = 0.f;
#pragma unroll
    for (int it = 0; it < VPL; ++it)
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        amax = fmaxf(amax, fabsf(p[it][c]));
        bad |= !is_finite(p[it][c]);
      }
#pragma unroll
    for (int o = 16; o; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    const float scale = __fdiv_rn(amax, 127.0f);
    const float inv = __frcp_rn(scale);
    if (lane == 0) scales[lo / B] = scale;
#pragma unroll
    for (int it = 0; it < VPL; ++it) {
      const size_t e = lo + (size_t)it * 128 + lane * 4;
      int q[4];
      float res[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        q[c] = q8_code(p[it][c], scale, inv);
        res[c] = __fsub_rn(p[it][c], __fmul_rn((float)q[c], scale));
      }
      if (from_smem) {
        *reinterpret_cast<char4*>(codes + e) =
            make_char4((signed char)q[0], (signed char)q[1], (signed char)q[2], (signed char)q[3]);
        __stcs(reinterpret_cast<float4*>(r + e), make_float4(res[0], res[1], res[2], res[3]));
      } else {
        for (int c = 0; c < 4; ++c)
          if (e + c < n) {
            codes[e + c] = (int8_t)q[c];
            r[e + c] = res[c];
          }
      }
    }
  };
  for (size_t i = 0; i < my_tiles; ++i) {
    const int s = (int)(i % kQ8Stages);
    mbar_wait(&full[s], (uint32_t)((i / kQ8Stages) & 1));
    const size_t base = (blockIdx.x + i * gridDim.x) * (size_t)TE;
    const size_t off = (size_t)s * TE + (size_t)wid * B;
    process(sx + off, sr + off, base + (size_t)wid * B, true);
    __syncthreads();  // every warp is done with stage s
    if (threadIdx.x == 0 && i + kQ8Stages < my_tiles) issue(i + kQ8Stages);
  }
  if (blockIdx.x == 0) {  // ragged tail: CTA 0, one block per warp
    for (size_t lo = ntiles_full * TE + (size_t)wid * B; lo < n; lo += 8 * (size_t)B)
      process(x + lo, r + lo, lo, false);
  }
  if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(flags, 1u);
}

// theta += (-lr) * mean, the mean read shard by shard from the rank that
// reduced it (Q8Shards: local buffer, or the peers' NVLink-mapped arenas).
__global__ void __launch_bounds__(256) k_q8_apply(Q8Shards ms, int R, size_t n,
                                                  uint32_t B, float coef, float* __restrict__ theta,
                                                  float* __restrict__ mean_out, uint32_t* flags) {
  bool bad = false;
  const size_t nv = n / 4;
  uintptr_t al = (uintptr_t)theta;
  for (int q = 0; q < R; ++q) al |= (uintptr_t)ms.codes[q];
  const bool vec_ok = (al & 15) == 0 && !mean_out;
  const int lb = 31 - __clz((int)B);  // B is a power of two (128..1024): no 64-bit divisions
  const uint32_t nbs32 = (uint32_t)(ms.nbs < 0xffffffffu ? ms.nbs : 0xffffffffu);
  auto owner = [&](size_t e) { return R == 1 ? 0 : (int)((uint32_t)(e >> lb) / nbs32); };
  auto code_at = [&](size_t e) { return ms.codes[owner(e)][e]; };
  auto scale_at = [&](size_t e) { return ms.scales[owner(e)][e >> lb]; };
  if (vec_ok) {
    // U float4 groups per thread per iteration, every load issued before any
    // use (U x 20 B in flight per thread; coalesced: group u of the warp is
    // 32 consecutive float4)
    constexpr int U = 4;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (size_t v0 = (size_t)blockIdx.x * blockDim.x + threadIdx.x; v0 < nv; v0 += U * stride) {
      char4 cv[U];
      float sc[U];
      float4 th[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const size_t v = v0 + u * stride;
        if (v < nv) {
          const size_t e = v * 4;
          const int o = owner(e);
          cv[u] = *reinterpret_cast<const char4*>(ms.codes[o] + e);
          sc[u] = ms.scales[o][e >> lb];
          th[u] = __ldcs(reinterpret_cast<const float4*>(theta + e));
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const size_t v = v0 + u * stride;
        if (v >= nv) continue;
        float4 t = th[u];
        t.x = __fadd_rn(__fmul_rn(coef, __fmul_rn((float)cv[u].x, sc[u])), t.x);
        t.y = __fadd_rn(__fmul_rn(coef, __fmul_rn((float)cv[u].y, sc[u])), t.y);
        t.z = __fadd_rn(__fmul_rn(coef, __fmul_rn((float)cv[u].z, sc[u])), t.z);
        t.w = __fadd_rn(__fmul_rn(coef, __fmul_rn((float)cv[u].w, sc[u])), t.w);
        __stcs(reinterpret_cast<float4*>(theta + v * 4), t);
        bad |= !is_finite(t.x) || !is_finite(t.y) || !is_finite(t.z) || !is_finite(t.w);
      }
    }
    for (size_t e = nv * 4 + (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
         e += (size_t)gridDim.x * blockDim.x) {
      const float th = __fadd_rn(__fmul_rn(coef, __fmul_rn((float)code_at(e), scale_at(e))), theta[e]);
      theta[e] = th;
      bad |= !is_finite(th);
    }
  } else {
    for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
         e += (size_t)gridDim.x * blockDim.x) {
      const float mhat = __fmul_rn((float)code_at(e), scale_at(e));
      const float th = __fadd_rn(__fmul_rn(coef, mhat), theta[e]);
      theta[e] = th;
      if (mean_out) mean_out[e] = mhat;
      bad |= !is_finite(th);
    }
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flags, 1u);
}

// theta += (-lr) * mean over TMA-staged tiles: one elected thread streams
// tiles of 8 blocks of theta (local) and of the requantized mean codes --
// read in place from the rank that reduced each block's shard, over NVLink
// for the other ranks (1-D bulk copies from the mapped arenas, split at shard
// boundaries) -- into a ring of kQ8Stages stages; each warp applies one block.
// The scales are local (gathered beforehand, 4 B per block).  Replaces the
// pull of the mean shards + k_q8_apply: the remote code reads overlap the
// theta stream.
template <int VPL>
__global__ void __launch_bounds__(256) k_q8_apply_tma(Q8Shards ms, const float* __restrict__ scales, size_t n,
                                                      float coef, float* __restrict__ theta, uint32_t* flags) {
  constexpr int B = VPL * 128;
  constexpr int TE = 8 * B;
  extern __shared__ __align__(128) unsigned char smem[];
  float* sth = reinterpret_cast<float*>(smem);                                        // [stage][TE]
  int8_t* scd = reinterpret_cast<int8_t*>(smem + (size_t)kQ8Stages * TE * sizeof(float));  // [stage][TE]
  __shared__ __align__(8) uint64_t full[kQ8Stages];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const size_t ntiles_full = n / TE;
  const size_t my_tiles = ntiles_full > blockIdx.x ? (ntiles_full - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  const size_t nbs = ms.nbs;
  // a peer timed out in the exchange (flag 8): its shard may be stale, theta
  // is left untouched and psb_check reports PSB_ESTATE
  if (flags != nullptr && (__ldcg(flags) & 8u)) return;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kQ8Stages; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](size_t i) {
    const int s = (int)(i % kQ8Stages);
    const size_t base = (blockIdx.x + i * gridDim.x) * (size_t)TE;
    mbar_expect_tx(&full[s], TE * 4 + TE);
    tma_load_1d(sth + (size_t)s * TE, theta + base, TE * 4, &full[s]);
    size_t cur = base / B;
    const size_t end = cur + 8;
    while (cur < end) {  // the tile's codes, one bulk copy per owning rank
      const size_t o = cur / nbs;
      const size_t stop = min(end, (o + 1) * nbs);
      tma_load_1d(scd + (size_t)s * TE + (cur * B - base), ms.codes[o] + cur * B, (uint32_t)((stop - cur) * B),
                  &full[s]);
      cur = stop;
    }
  };
  if (threadIdx.x == 0)
    for (size_t i = 0; i < my_tiles && i < (size_t)kQ8Stages; ++i) issue(i);
  bool bad = false;
  for (size_t i = 0; i < my_tiles; ++i) {
    const int s = (int)(i % kQ8Stages);
    const size_t base = (blockIdx.x + i * gridDim.x) * (size_t)TE;
    const size_t blk = base / B + wid;
    const float sc = scales ? scales[blk] : ms.scales[blk / nbs][blk];  // issued before the wait
    mbar_wait(&full[s], (uint32_t)((i / kQ8Stages) & 1));
#pragma unroll
    for (int it = 0; it < VPL; ++it) {
      const int o = wid * B + it * 128 + lane * 4;
      const char4 cv = *reinterpret_cast<const char4*>(scd + (size_t)s * TE + o);
      float4 th = *reinterpret_cast<const float4*>(sth + (size_t)s * TE + o);
      th.x = __fadd_rn(__fmul_rn(coef, __fmul_rn((float)cv.x, sc)), th.x);
      th.y = __fadd_rn(__fmul_rn(coef, __fmul_rn((float)cv.y, sc)), th.y);
      th.z = __fadd_rn(__fmul_rn(coef, __fmul_rn((float)cv.z, sc)), th.z);
      th.w = __fadd_rn(__fmul_rn(coef, __fmul_rn((float)cv.w, sc)), th.w);
      __stcs(reinterpret_cast<float4*>(theta + base + o), th);
      bad |= !is_finite(th.x) || !is_finite(th.y) || !is_finite(th.z) || !is_finite(th.w);
    }
    __syncthreads();  // every warp is done with stage s
    if (threadIdx.x == 0 && i + kQ8Stages < my_tiles) issue(i + kQ8Stages);
  }
  if (blockIdx.x == 0) {  // ragged tail (elements past the last full tile): CTA 0, direct loads
    for (size_t e = ntiles_full * TE + threadIdx.x; e < n; e += blockDim.x) {
      const size_t blk = e / B;
      const float sb = scales ? scales[blk] : ms.scales[blk / nbs][blk];
      const float th = __fadd_rn(__fmul_rn(coef, __fmul_rn((float)ms.codes[blk / nbs][e], sb)), theta[e]);
      theta[e] = th;
      bad |= !is_finite(th);
    }
  }
  if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(flags, 1u);
}

}  // namespace

psb_status psb_q8_quant_launch(psb_ctx* c, const float* x, float* r, size_t n, uint32_t B,
                               int8_t* codes, float* scales, cudaStream_t st) {
  const size_t nb = (n + B - 1) / B;
  if (r != nullptr && !c->q8_no_tma && ((((uintptr_t)x) | ((uintptr_t)r) | ((uintptr_t)codes)) & 15) == 0 &&
      (B == 128 || B == 256 || B == 512)) {  // B = 1024: the register-pipelined kernel below
    const size_t smem = (size_t)kQ8Stages * 2 * 8 * B * sizeof(float);
    const unsigned tgrid = (unsigned)std::max<size_t>(1, std::min<size_t>((n / (8 * B)) + 1, (size_t)c->num_sms * 2));
#define PSB_QT(V)                                                                                           \
  do {                                                                                                      \
    cudaFuncSetAttribute(k_q8_quant_tma<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);        \
    k_q8_quant_tma<V><<<tgrid, 256, smem, st>>>(x, r, n, codes, scales, c->d_flags);                        \
  } while (0)
    switch (B) {
      case 128: PSB_QT(1); break;
      case 256: PSB_QT(2); break;
      default: PSB_QT(4); break;
    }
#undef PSB_QT
    c->launches += 1;
    PSB_LAUNCH_CHECK(c, "psb_q8_quantize");
    return PSB_OK;
  }
  const unsigned grid = (unsigned)std::max<size_t>(1, std::min<size_t>((nb + 7) / 8, (size_t)c->num_sms * 8));
  switch (B) {
    case 128: k_q8_quant<1><<<grid, 256, 0, st>>>(x, r, n, codes, scales, c->d_flags); break;
    case 256: k_q8_quant<2><<<grid, 256, 0, st>>>(x, r, n, codes, scales, c->d_flags); break;
    case 512: k_q8_quant<4><<<grid, 256, 0, st>>>(x, r, n, codes, scales, c->d_flags); break;
    case 1024: k_q8_quant<8><<<grid, 256, 0, st>>>(x, r, n, codes, scales, c->d_flags); break;
    default: return psb_set_err(c, PSB_EINVAL, "q8: block must be 128, 256, 512 or 1024");
  }
  c->launches += 1;
  PSB_LAUNCH_CHECK(c, "psb_q8_quantize");
  return PSB_OK;
}

psb_status psb_q8_reduce_launch(psb_ctx* c, const Q8Workers& wv, int P, size_t blk_lo,
                                size_t blk_hi, size_t n, uint32_t B, psb_order order, uint32_t dpn,
                                uint32_t npr, int8_t* mcodes, float* mscales, double lr,
                                float* theta, float* mean_out, cudaStream_t st) {
  if (blk_hi <= blk_lo) return PSB_OK;
  // common multi-rank case: the pipelined kernel over the full blocks, the
  // generic one for a ragged last block
  uintptr_t al = (uintptr_t)mcodes;
  for (int q = 0; q < P; ++q) al |= (uintptr_t)wv.codes[q];
  const bool plain = order == PSB_ORDER_NAIVE || (order == PSB_ORDER_HIER && dpn >= (uint32_t)P);
  if (!c->q8_no_pipe && plain && !theta && !mean_out && (al & 15) == 0 && (P == 2 || P == 4 || P == 8)) {
    const size_t full_hi = std::min(blk_hi, n / B);
    if (full_hi > blk_lo) {
      const size_t nbf = full_hi - blk_lo;
      const unsigned g2 = (unsigned)std::max<size_t>(1, std::min<size_t>((nbf + 7) / 8, (size_t)c->num_sms * 8));
      // register budget: the double buffer holds P * B / 128 char4 per lane
      const int vpl = (int)(B / 128);
#define PSB_REDP(V, PP) k_q8_reduce_pipe<V, PP><<<g2, 256, 0, st>>>(wv, blk_lo, full_hi, mcodes, mscales)
      if (P == 2 && vpl == 1) PSB_REDP(1, 2);
      else if (P == 2 && vpl == 2) PSB_REDP(2, 2);
      else if (P == 2 && vpl == 4) PSB_REDP(4, 2);
      else if (P == 4 && vpl == 1) PSB_REDP(1, 4);
      else if (P == 4 && vpl == 2) PSB_REDP(2, 4);
      else if (P == 8 && vpl == 1) PSB_REDP(1, 8);
      else goto generic;
#undef PSB_REDP
      c->launches += 1;
      PSB_LAUNCH_CHECK(c, "q8 reduce");
      if (full_hi == blk_hi) return PSB_OK;
      // the ragged last block: the workers' pointers rebased to it
      Q8Workers wt = wv;
      for (int q = 0; q < P; ++q) {
        wt.codes[q] += (full_hi - blk_lo) * B;
        wt.scales[q] += full_hi - blk_lo;
      }
      return psb_q8_reduce_launch(c, wt, P, full_hi, blk_hi, n, B, order, dpn, npr, mcodes, mscales, lr, theta,
                                  mean_out, st);
    }
  }
generic:
  const size_t nb = blk_hi - blk_lo;
  const unsigned grid = (unsigned)std::max<size_t>(1, std::min<size_t>((nb + 7) / 8, (size_t)c->num_sms * 8));
  const float coef = (float)(-lr);
#define PSB_RED(V)                                                                                \
  k_q8_reduce<V><<<grid, 256, 0, st>>>(wv, P, blk_lo, blk_hi, n,                                    \
                                       (int)order, dpn, npr, mcodes, mscales, coef, theta, mean_out, \
                                       c->d_flags)
  switch (B) {
    case 128: PSB_RED(1); break;
    case 256: PSB_RED(2); break;
    case 512: PSB_RED(4); break;
    case 1024: PSB_RED(8); break;
    default: return psb_set_err(c, PSB_EINVAL, "q8: block must be 128, 256, 512 or 1024");
  }
#undef PSB_RED
  c->launches += 1;
  PSB_LAUNCH_CHECK(c, "q8 reduce");
  return PSB_OK;
}

psb_status psb_q8_step1_launch(psb_ctx* c, const float* g, size_t gstride, float* r, size_t rstride,
                               int P, size_t n, uint32_t B, psb_order order, uint32_t dpn, uint32_t npr,
                               double lr, float* theta, float* mean_out, cudaStream_t st) {
  const size_t nb = (n + B - 1) / B;
  const unsigned grid = (unsigned)std::max<size_t>(1, std::min<size_t>((nb + 7) / 8, (size_t)c->num_sms * 8));
  const float coef = (float)(-lr);
  if (c->prof) cudaEventRecord(psb_prof_event(c), st);
  const bool hier = order == PSB_ORDER_HIER && dpn < (uint32_t)P;
  const bool tma = P == 1 && r != nullptr && !c->q8_no_tma && B <= 512 &&  // B = 1024 tiles exceed smem
                   ((((uintptr_t)g) | ((uintptr_t)r) | ((uintptr_t)theta) | ((uintptr_t)mean_out)) & 15) == 0;
  if (tma) {
    const size_t smem = (size_t)kQ8Stages * 3 * 8 * B * sizeof(float);
    const unsigned tgrid = (unsigned)std::max<size_t>(1, std::min<size_t>((n / (8 * B)) + 1, (size_t)c->num_sms * 2));
#define PSB_T1(V)                                                                                         \
  do {                                                                                                    \
    cudaFuncSetAttribute(k_q8_step1_tma<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);      \
    k_q8_step1_tma<V><<<tgrid, 256, smem, st>>>(g, r, n, coef, theta, mean_out, c->d_flags);              \
  } while (0)
    switch (B) {
      case 128: PSB_T1(1); break;
      case 256: PSB_T1(2); break;
      case 512: PSB_T1(4); break;
      default: return psb_set_err(c, PSB_EINVAL, "q8: block must be 128, 256 or 512 here");
    }
#undef PSB_T1
    if (c->prof) cudaEventRecord(psb_prof_event(c), st);
    c->launches += 1;
    PSB_LAUNCH_CHECK(c, "q8 fused step (TMA)");
    return PSB_OK;
  }
#define PSB_S1(V)                                                                                          \
  (hier ? k_q8_step1<V, true><<<grid, 256, 0, st>>>(g, gstride, r, rstride, P, n, (int)order, dpn, npr, coef, \
                                                     theta, mean_out, c->d_flags)                            \
        : k_q8_step1<V, false><<<grid, 256, 0, st>>>(g, gstride, r, rstride, P, n, (int)order, dpn, npr,      \
                                                      coef, theta, mean_out, c->d_flags))
  switch (B) {
    case 128: PSB_S1(1); break;
    case 256: PSB_S1(2); break;
    case 512: PSB_S1(4); break;
    case 1024: PSB_S1(8); break;
    default: return psb_set_err(c, PSB_EINVAL, "q8: block must be 128, 256, 512 or 1024");
  }
#undef PSB_S1
  if (c->prof) cudaEventRecord(psb_prof_event(c), st);
  c->launches += 1;
  PSB_LAUNCH_CHECK(c, "q8 fused step");
  return PSB_OK;
}

// Returns the number of full 8-block tiles reduced (the caller reduces the
// rest), or -1 when the TMA reduce does not apply (P / B combination).
long long psb_q8_reduce_tma_launch(psb_ctx* c, const Q8Workers& wv, int P, size_t blk_lo, size_t blk_hi, uint32_t B,
                                   int8_t* mcodes, float* mscales, cudaStream_t st) {
  const size_t ntiles = (blk_hi - blk_lo) / 8;
  if (ntiles == 0) return 0;
  const unsigned grid = (unsigned)std::min<size_t>(ntiles, (size_t)c->num_sms * 2);
#define PSB_RT(V, PP)                                                                                       \
  do {                                                                                                      \
    const size_t smem = (size_t)kQ8Stages * PP * (8 * V * 128 + 32);                                        \
    cudaFuncSetAttribute(k_q8_reduce_tma<V, PP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);    \
    k_q8_reduce_tma<V, PP><<<grid, 256, smem, st>>>(wv, blk_lo, ntiles, mcodes, mscales);                  \
  } while (0)
  const int vpl = (int)(B / 128);
  if (P == 2 && vpl == 1) PSB_RT(1, 2);
  else if (P == 2 && vpl == 2) PSB_RT(2, 2);
  else if (P == 2 && vpl == 4) PSB_RT(4, 2);
  else if (P == 4 && vpl == 1) PSB_RT(1, 4);
  else if (P == 4 && vpl == 2) PSB_RT(2, 4);
  else if (P == 8 && vpl == 1) PSB_RT(1, 8);
  else if (P == 8 && vpl == 2) PSB_RT(2, 8);
  else return -1;
#undef PSB_RT
  c->launches += 1;
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return -2;
  return (long long)ntiles;
}

psb_status psb_q8_apply_tma_launch(psb_ctx* c, const Q8Shards& ms, const float* scales, size_t n, uint32_t B,
                                   double lr, float* theta, cudaStream_t st) {
  const size_t smem = (size_t)kQ8Stages * 8 * B * 5;
  const unsigned tgrid = (unsigned)std::max<size_t>(1, std::min<size_t>((n / (8 * B)) + 1, (size_t)c->num_sms * 4));
#define PSB_QA(V)                                                                                           \
  do {                                                                                                      \
    cudaFuncSetAttribute(k_q8_apply_tma<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);        \
    k_q8_apply_tma<V><<<tgrid, 256, smem, st>>>(ms, scales, n, (float)(-lr), theta, c->d_flags);            \
  } while (0)
  switch (B) {
    case 128: PSB_QA(1); break;
    case 256: PSB_QA(2); break;
    case 512: PSB_QA(4); break;
    default: return psb_set_err(c, PSB_EINVAL, "q8 TMA apply: block must be 128, 256 or 512");
  }
#undef PSB_QA
  c->launches += 1;
  PSB_LAUNCH_CHECK(c, "q8 apply");
  return PSB_OK;
}

psb_status psb_q8_apply_launch(psb_ctx* c, const Q8Shards& ms, int R, size_t n,
                               uint32_t B, double lr, float* theta, float* mean_out,
                               cudaStream_t st) {
  const unsigned grid = (unsigned)std::min<size_t>((n / 4 + 255) / 256 + 1, (size_t)c->num_sms * 8);
  k_q8_apply<<<grid, 256, 0, st>>>(ms, R, n, B, (float)(-lr), theta, mean_out, c->d_flags);
  c->launches += 1;
  PSB_LAUNCH_CHECK(c, "q8 apply");
  return PSB_OK;
}

extern "C" psb_status psb_q8_quantize(psb_ctx* c, const float* x, float* r, size_t n,
                                      uint32_t block, int8_t* codes, float* scales,
                                      psb_stream_t stream) {
  PSB_REQUIRE(c, c != nullptr, "null ctx");
  PSB_REQUIRE(c, n >= 1 && x && codes && scales, "psb_q8_quantize: bad arguments");
  return psb_q8_quant_launch(c, x, r, n, block, codes, scales, (cudaStream_t)stream);
}

extern "C" psb_status psb_q8_dequantize(psb_ctx* c, const int8_t* codes, const float* scales,
                                        size_t n, uint32_t block, float* out, psb_stream_t stream) {
  PSB_REQUIRE(c, c != nullptr, "null ctx");
  PSB_REQUIRE(c, n >= 1 && block >= 1 && codes && scales && out, "psb_q8_dequantize: bad arguments");
  const unsigned grid = (unsigned)std::min<size_t>((n + 255) / 256, (size_t)c->num_sms * 16);
  k_q8_dequant<<<grid, 256, 0, (cudaStream_t)stream>>>(codes, scales, n, block, out);
  c->launches += 1;
  PSB_LAUNCH_CHECK(c, "psb_q8_dequantize");
  return PSB_OK;
}
