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
#include "psb_debug.h"

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
  int idx16;  // indices stored as u16 offsets inside their apply segment (wire16 payloads)
  // direct multi-rank mode (wpr > 0): worker q's block lives in rank q / wpr's
  // NVLink-mapped arena at rank_base[q / wpr] + q * block_bytes, its segment
  // offset rows at rank_base[q / wpr] + tab_off + q * (nseg + 1) words
  int wpr;
  size_t tab_off;
  const uint8_t* rank_base[PSB_MAX_P];
};

__device__ __forceinline__ const uint8_t* pl_block(const PayloadView& v, int q) {
  return (v.wpr ? v.rank_base[q / v.wpr] : v.base) + (size_t)q * v.block_bytes;
}

__device__ __forceinline__ const uint32_t* pl_idx(const PayloadView& v, int q) {
  return reinterpret_cast<const uint32_t*>(pl_block(v, q));
}

template <class T>
__device__ __forceinline__ T pl_val(const PayloadView& v, int q, size_t j) {
  const uint8_t* b = pl_block(v, q);
  if (v.q8) {
    const int8_t code = reinterpret_cast<const int8_t*>(b + v.val_off)[j];
    const float sc = reinterpret_cast<const float*>(b + v.scale_off)[j >> 7];
    return (T)__fmul_rn((float)code, sc);
  }
  return reinterpret_cast<const T*>(b + v.val_off)[j];
}

// Per-worker segment offsets: seg_off[q][s] = first payload position of worker
// q whose index is >= s*S (k past the end).  Grid (x, P); 32-bit positions.
#ifdef PSB_APPLY_TRACE
__device__ unsigned long long g_apply_trace[8];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define APPLY_MARK(slot)                                             \
  do {                                                               \
    __syncthreads();                                                 \
    if (threadIdx.x == 0) {                                          \
      const unsigned long long t_ = gtimer();                        \
      atomicAdd(&g_apply_trace[slot], t_ - t_prev);                  \
      t_prev = t_;                                                   \
    }                                                                \
  } while (0)
#else
#define APPLY_MARK(slot) \
  do {                   \
  } while (0)
#endif

constexpr int kSegU = 8;  // entries per thread in k_seg_offsets

// With out16 != nullptr it also writes worker q's wire16 payload (u16
// in-segment offset | value, psb_wire16_bytes layout) at out16 + q * out_stride
// in the same pass (vbytes: 4 or 8).
__global__ void __launch_bounds__(256) k_seg_offsets(PayloadView v, int P, uint32_t k, uint32_t nseg,
                                                     int seg_shift, uint32_t* __restrict__ seg_off,
                                                     uint8_t* __restrict__ out16, size_t out_stride, int vbytes) {
  const int q = blockIdx.y;
  const uint32_t* idx = pl_idx(v, q);
  uint32_t* row = seg_off + (size_t)q * (nseg + 1);
  const uint32_t base = blockIdx.x * (blockDim.x * kSegU) + threadIdx.x;
  uint32_t cur[kSegU], prv[kSegU];
#pragma unroll
  for (int u = 0; u < kSegU; ++u) {
    const uint32_t j = base + u * blockDim.x;
    cur[u] = j < k ? idx[j] : 0u;
    prv[u] = (j && j < k) ? idx[j - 1] : 0u;
  }
  if (out16) {
    const uint32_t mask = (1u << seg_shift) - 1u;
    uint8_t* o = out16 + (size_t)q * out_stride;
    uint16_t* lo16 = reinterpret_cast<uint16_t*>(o);
    const uint8_t* vsrc = pl_block(v, q) + v.val_off;
    uint8_t* vdst = o + ((2 * (size_t)k + 15) & ~(size_t)15);
#pragma unroll
    for (int u = 0; u < kSegU; ++u) {
      const uint32_t j = base + u * blockDim.x;
      if (j >= k) continue;
      lo16[j] = (uint16_t)(cur[u] & mask);
      if (vbytes == 8)
        reinterpret_cast<uint64_t*>(vdst)[j] = reinterpret_cast<const uint64_t*>(vsrc)[j];
      else
        reinterpret_cast<uint32_t*>(vdst)[j] = reinterpret_cast<const uint32_t*>(vsrc)[j];
    }
  }
#pragma unroll
  for (int u = 0; u < kSegU; ++u) {
    const uint32_t j = base + u * blockDim.x;
    if (j >= k) continue;
    const uint32_t s0 = j ? (prv[u] >> seg_shift) + 1 : 0;
    for (uint32_t s = s0; s <= (cur[u] >> seg_shift); ++s) row[s] = j;
  }
  const uint32_t last = idx[k - 1] >> seg_shift;
  for (uint32_t s = last + 1 + blockIdx.x * blockDim.x + threadIdx.x; s <= nseg; s += gridDim.x * blockDim.x)
    row[s] = k;
}

// Bitmap-rank apply (P >= 2), one segment of S = 2^seg_shift indices at a
// time.  The segment's entries of all P workers form one flat range
// e in [0, tot) (worker q owns [vb[q], vb[q+1])).  Each worker's touched
// indices become a presence bitmap; the first entry of a worker in each
// bitmap word records that entry's position in the value stage there, so the
// value of index i in worker q2's list sits at pre[q2][w] + popc(word &
// below) (only words holding a set bit are ever queried, so no scan is
// needed).  The lowest worker touching i owns it: it folds the P dense values
// (+0 where absent) in the configured reference order and updates theta once
// (async: applies the present workers in order).  PT > 0 fixes P at compile
// time (worker lookup in registers); PT == 0 is the generic kernel.
//
// TMA (the default for gathered f32/f64 top-k and wire16 payloads):
// persistent CTAs, and each segment's entries (index and value ranges of the
// P workers, widened to 16-byte boundaries) arrive in shared memory by 1-D
// bulk copies on an mbarrier, double-buffered: warp 0 issues the copies of
// the CTA's next segment between the two phases of the current one, so the
// entry loads overlap the current fold and the dependent global round trips
// left per segment are the theta loads.  A segment too large for the stage
// reads its entries from global memory (the non-TMA path).
// Without TMA (q8 values, direct / sharded multi-rank views): one CTA per
// segment, entries loaded by the threads in batches and staged when tot <=
// vcap.
#ifndef PSB_APPLY_U
#define PSB_APPLY_U 2
#endif
#ifndef PSB_APPLY_U1
#define PSB_APPLY_U1 2
#endif
// CTA shapes (measured on B200): non-TMA 256 threads x 4 CTAs/SM, and
// 128 x 6 for P = 8 (more segments in flight; P = 8 324 -> 269 us); TMA
// 256 x 4 with a 1792-entry stage (P = 8 186 -> 170 us vs 3 CTAs/SM).
// bitmap words per worker of psb_apply_seg_shift(P) (psb_internal.cuh)
__host__ __device__ constexpr int apply_nw(int P) {
  int sh = 15;
  while (sh > 10 && ((long)P * 8) << (sh - 5) > PSB_APPLY_BM_BYTES) --sh;
  return (1 << sh) >> 5;
}
#ifndef PSB_APPLY_TMA_MINB
#define PSB_APPLY_TMA_MINB 4
#endif
__host__ __device__ constexpr int apply_threads(int PT, bool TMA) { return TMA ? 256 : PT == 8 ? 128 : 256; }
__host__ __device__ constexpr int apply_minb(int PT, bool TMA) { return TMA ? PSB_APPLY_TMA_MINB : PT == 8 ? 6 : 4; }

template <class T, bool ASYNC, int PT, bool TMA>
__global__ void __launch_bounds__(apply_threads(PT, TMA), apply_minb(PT, TMA))
    k_sparse_apply_bm(PayloadView v, int P_rt, uint32_t nseg, uint32_t seg_lo, const uint32_t* __restrict__ range,
                      int seg_shift, uint32_t vcap, uint32_t ci_bytes, uint32_t cv_bytes, uint32_t light_max,
                      const uint32_t* __restrict__ seg_off, int order, uint32_t dpn, uint32_t npr, T coef,
                      WorkerCoefs wscale, T* __restrict__ theta, size_t n, T* __restrict__ mean_out,
                      uint32_t* __restrict__ list_idx, T* __restrict__ list_val, uint32_t* list_cnt,
                      uint32_t* flags) {
  constexpr int U = PSB_APPLY_U;    // touched indices per thread per batch (fold)
  constexpr int U1 = PSB_APPLY_U1;  // entries per thread per batch (global entry loads)
  const int P = PT > 0 ? PT : P_rt;
  extern __shared__ __align__(16) unsigned char smem[];
  // bitmap words per worker (a compile-time constant for PT > 0, so every
  // shared-memory lookup below has an immediate per-worker offset)
  const uint32_t NW = PT > 0 ? (uint32_t)apply_nw(PT) : (1u << seg_shift) >> 5;
  uint32_t* bm = reinterpret_cast<uint32_t*>(smem);  // [P][NW] presence bits
  uint32_t* pre = bm + (size_t)P * NW;                 // [P][NW] stage position of a word's first entry
  unsigned char* stage0 = reinterpret_cast<unsigned char*>(pre + (size_t)P * NW);
  // segment descriptors, double-buffered under TMA: first payload position,
  // flat entry bases, stage positions of each worker's first index / value
  __shared__ uint32_t lo_s[2][PSB_MAX_P], vb_s[2][PSB_MAX_P + 1], bi_s[2][PSB_MAX_P], bv_s[2][PSB_MAX_P];
  __shared__ uint32_t stg_s[2], rot_s[2];
  __shared__ __align__(8) uint64_t mbar[2];
  __shared__ T coefs[PSB_MAX_P];
  __shared__ uint16_t wlist[apply_threads(PT, TMA) / 32][1024];  // per-warp touched-index list
  if (ASYNC && threadIdx.x < (unsigned)P) coefs[threadIdx.x] = (T)(-wscale.v[threadIdx.x]);
  const T inv = (T)(1.0 / (double)P);
  bool bad = false;
  RingChunk rc;
  const uint32_t lane = threadIdx.x & 31;
  const bool warp0 = threadIdx.x < 32;
  const uint32_t ib = v.idx16 ? 2u : 4u;  // bytes per stored index

#ifdef PSB_APPLY_TRACE
  unsigned long long t_prev = gtimer();
#endif
  // a peer timed out in the exchange (flag 8, psb_peer.cu): its payload slot
  // may hold the previous step's data, so theta is left untouched and the
  // step reports PSB_ESTATE at the caller's psb_check (checked once the
  // first segment's offsets are in, so the two loads overlap; no copy is
  // issued when it is set)
  const uint32_t flag0 = flags != nullptr ? __ldcg(flags) : 0u;
  if (range) {  // segment range decided on the device (sharded multi-rank apply)
    seg_lo = range[0];
    nseg = range[1] - range[0];
  }
  // warp 0, lanes < P: worker lane's payload positions [l, l + cnt) in segment seg
  auto fetch = [&](uint32_t seg, uint32_t& l, uint32_t& cnt) {
    l = 0;
    cnt = 0;
    if (lane < (uint32_t)P) {
      const uint32_t* row = v.wpr ? reinterpret_cast<const uint32_t*>(v.rank_base[lane / v.wpr] + v.tab_off) +
                                        (size_t)lane * (nseg + 1)
                                  : seg_off + (size_t)lane * (nseg + 1);
      l = row[seg];
      cnt = row[seg + 1] - l;
    }
  };
  auto warp_incl = [&](uint32_t x) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= (uint32_t)o) x += t;
    }
    return x;
  };
  // warp 0: descriptor of a segment into buffer b; under TMA also issue its
  // bulk copies when the widened ranges fit the stage
  auto describe = [&](int b, uint32_t seg, uint32_t l, uint32_t cnt) {
    uint32_t incl = warp_incl(cnt);
    // a segment of at most light_max entries is k_sparse_apply_light's:
    // described as empty here
    if (TMA && __shfl_sync(0xffffffffu, incl, 31) <= light_max) {
      cnt = 0;
      incl = 0;
    }
    const uint32_t tot = __shfl_sync(0xffffffffu, incl, 31);
    uint32_t bi = incl - cnt, bv = incl - cnt;  // non-TMA / unstaged: the flat entry index
    bool fits = false;
    uint32_t ai = 0, li = 0, av = 0, lv = 0, oi = 0, ov = 0, si = 0, sv = 0;
    if (TMA && tot) {
      const uint32_t EI = 16u / ib, EV = 16u / (uint32_t)sizeof(T);
      ai = l & ~(EI - 1);
      li = cnt ? ((l + cnt + EI - 1) & ~(EI - 1)) - ai : 0;
      av = l & ~(EV - 1);
      lv = cnt ? ((l + cnt + EV - 1) & ~(EV - 1)) - av : 0;
      const uint32_t ii = warp_incl(li), iv = warp_incl(lv);
      oi = ii - li;
      ov = iv - lv;
      si = __shfl_sync(0xffffffffu, ii, 31) * ib;
      sv = __shfl_sync(0xffffffffu, iv, 31) * (uint32_t)sizeof(T);
      fits = si <= ci_bytes && sv <= cv_bytes;
      if (fits) {
        bi = oi + (l - ai);
        bv = ov + (l - av);
      }
    } else if (!TMA) {
      fits = tot <= vcap;
    }
    if (lane < (uint32_t)P) {
      lo_s[b][lane] = l;
      vb_s[b][lane + 1] = incl;
      bi_s[b][lane] = bi;
      bv_s[b][lane] = bv;
    }
    if (lane == 0) {
      vb_s[b][0] = 0;
      stg_s[b] = fits ? 1u : 0u;
      // bitmap slot rotation (phase 2): one ring chunk for the whole segment?
      uint32_t rs = 0;
      if (!ASYNC && order == PSB_ORDER_RING) {
        const size_t b0 = (size_t)(seg_lo + seg) << seg_shift;
        const size_t last = min(b0 + ((size_t)1 << seg_shift), n) - 1;
        const int r0 = rc.start_for(b0, n, P);
        rs = (rc.lo <= b0 && last < rc.hi) ? (uint32_t)r0 : 0x80000000u;  // high bit: per-index order
      }
      rot_s[b] = rs;
    }
    if (TMA && fits) {
      if (lane == 0) mbar_expect_tx(&mbar[b], si + sv);
      __syncwarp();
      if (cnt) {
        const uint8_t* blk = pl_block(v, (int)lane);
        tma_load_1d(stage0 + (size_t)oi * ib, blk + (size_t)ai * ib, li * ib, &mbar[b]);
        tma_load_1d(stage0 + ci_bytes + (size_t)b * cv_bytes + (size_t)ov * sizeof(T), blk + v.val_off + (size_t)av * sizeof(T),
                    lv * (uint32_t)sizeof(T), &mbar[b]);
      }
    }
  };

  uint32_t par = 0;        // TMA: mbarrier phase parity per buffer
  uint32_t nl = 0, nc = 0;  // TMA, warp 0: offsets of the CTA's next segment
  if (TMA) {
    if (threadIdx.x == 0) {
      mbar_init(&mbar[0], 1);
      mbar_init(&mbar[1], 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    if (warp0 && blockIdx.x < nseg) {
      uint32_t l, cnt;
      fetch(blockIdx.x, l, cnt);
      if (!(flag0 & 8u)) describe(0, blockIdx.x, l, cnt);
      if (blockIdx.x + gridDim.x < nseg) fetch(blockIdx.x + gridDim.x, nl, nc);
    }
  }
  {
    uint4* b4 = reinterpret_cast<uint4*>(bm);
    for (uint32_t w = threadIdx.x; w < ((uint32_t)P * NW) >> 2; w += blockDim.x) b4[w] = make_uint4(0, 0, 0, 0);
  }
  int b = 0;
  for (uint32_t seg = blockIdx.x; seg < nseg; seg += gridDim.x, b = TMA ? b ^ 1 : 0) {
    if (!TMA) {
      __syncthreads();  // the previous segment is done with the descriptor
      if (warp0) {
        uint32_t l, cnt;
        fetch(seg, l, cnt);
        describe(0, seg, l, cnt);
      }
    }
    // the bitmaps are all-zero here: cleared before the loop, and phase 2
    // re-zeroes the words it consumed
    __syncthreads();
    APPLY_MARK(0);
    if (flag0 & 8u) return;  // uniform across the CTA
    const uint32_t* lo = lo_s[b];
    const uint32_t* vb = vb_s[b];
    const uint32_t tot = vb[P];
    const bool staged = stg_s[b] != 0;
    const size_t seg_base = (size_t)(seg_lo + seg) << seg_shift;
    // bitmap slot of worker q: (q - rot) mod P, so a fold over slots 0..P-1
    // is the reference order when it is one rotation of the workers for the
    // whole segment (naive: rot 0; ring: the segment lies in one ring chunk,
    // rot = its start); otherwise (ring across a chunk boundary,
    // multi-node hierarchical) slot = worker and the per-index order below
    const uint32_t rsv = rot_s[b];
    const int rot = (int)(rsv & 0x7fffffffu);
    const bool plain = ASYNC || order == PSB_ORDER_NAIVE || (order == PSB_ORDER_HIER && dpn >= (uint32_t)P) ||
                       (order == PSB_ORDER_RING && !(rsv >> 31));
    auto slot_of = [&](int q) { return q - rot + (q < rot ? P : 0); };
    auto worker_at = [&](int sl) { return sl + rot - (sl + rot >= P ? P : 0); };
    // TMA: one index stage (read by phase 1 only, so the next segment's
    // copies may overwrite it once phase 1 is done) and two value stages
    unsigned char* st = stage0;
    const T* sval = reinterpret_cast<const T*>(st + (TMA ? ci_bytes + (size_t)b * cv_bytes : 0));
    const uint32_t scap = TMA ? cv_bytes / (uint32_t)sizeof(T) : vcap;  // value slots of the stage
    if (tot) {
      uint32_t vbr[PT > 0 ? PT : 1];
      if constexpr (PT > 0) {
#pragma unroll
        for (int p = 0; p < PT; ++p) vbr[p] = vb[p];
      }
      // worker owning flat entry e, and the flat index of that worker's first entry
      auto worker_of = [&](uint32_t e, uint32_t& base) {
        int q = 0;
        base = 0;
        if constexpr (PT > 0) {
#pragma unroll
          for (int p = 1; p < PT; ++p)
            if (e >= vbr[p]) {
              q = p;
              base = vbr[p];
            }
        } else {
          for (int p = 1; p < P; ++p) q += e >= vb[p];
          base = vb[q];
        }
        return q;
      };
      auto mark = [&](int q, uint32_t il, uint32_t ilp, uint32_t r) {
        const uint32_t w = il >> 5;
        const int sl = slot_of(q);
        atomicOr(&bm[(size_t)sl * NW + w], 1u << (il & 31));
        if (ilp == 0xffffffffu || (ilp >> 5) != w) pre[(size_t)sl * NW + w] = bv_s[b][q] + r;
        // warm L2 with theta at this index: phase 2 reads it after the barrier
#ifndef PSB_APPLY_NO_PF
        if (theta) asm volatile("prefetch.global.L2 [%0];" ::"l"(theta + seg_base + il));
#endif
      };
      // 1. presence bitmaps and word positions
      if (TMA && staged) {
        mbar_wait(&mbar[b], (par >> b) & 1u);
        par ^= 1u << b;
        auto staged_entry = [&](int q, uint32_t r) {
          const uint32_t pos = bi_s[b][q] + r;
          uint32_t il, ilp = 0xffffffffu;
          if (v.idx16) {
            const uint16_t* s16 = reinterpret_cast<const uint16_t*>(st);
            il = s16[pos];
            if (r) ilp = s16[pos - 1];
          } else {
            const uint32_t* s32 = reinterpret_cast<const uint32_t*>(st);
            il = s32[pos] - (uint32_t)seg_base;
            if (r) ilp = s32[pos - 1] - (uint32_t)seg_base;
          }
          mark(q, il, ilp, r);
        };
        if constexpr (PT > 0 && (apply_threads(PT, TMA) / 32) % (PT > 0 ? PT : 1) == 0) {
          // warps own workers: warp w takes worker w % P, part w / P of its entries
          const int wid = threadIdx.x >> 5, q = wid % PT, nparts = (int)(blockDim.x >> 5) / PT;
          const uint32_t cq = vb[q + 1] - vb[q];
          for (uint32_t r = (uint32_t)(wid / PT) * 32 + lane; r < cq; r += (uint32_t)nparts * 32) staged_entry(q, r);
        } else {
          for (uint32_t e = threadIdx.x; e < tot; e += blockDim.x) {
            uint32_t base;
            const int q = worker_of(e, base);
            staged_entry(q, e - base);
          }
        }
      } else {
        // entries from global memory; a batch issues all its loads first
        T* sv_w = reinterpret_cast<T*>(st);
        for (uint32_t e0 = threadIdx.x; e0 < tot; e0 += U1 * blockDim.x) {
          uint32_t il[U1], ilp[U1], rr[U1];
          T val[U1];
          int qq[U1];
#pragma unroll
          for (int u = 0; u < U1; ++u) {
            const uint32_t e = e0 + u * blockDim.x;
            qq[u] = -1;
            if (e < tot) {
              uint32_t base;
              const int q = worker_of(e, base);
              const uint32_t rq = e - base;
              const uint32_t j = lo[q] + rq;
              qq[u] = q;
              rr[u] = rq;
              if (v.idx16) {  // wire16: the in-segment offset is stored directly
                const uint16_t* lo16 = reinterpret_cast<const uint16_t*>(pl_block(v, q));
                il[u] = lo16[j];
                ilp[u] = rq ? (uint32_t)lo16[j - 1] : 0xffffffffu;
              } else {
                const uint32_t* idx = pl_idx(v, q);
                il[u] = (uint32_t)(idx[j] - seg_base);
                ilp[u] = rq ? (uint32_t)(idx[j - 1] - seg_base) : 0xffffffffu;
              }
              if (!TMA && staged) val[u] = pl_val<T>(v, q, j);
            }
          }
#pragma unroll
          for (int u = 0; u < U1; ++u) {
            if (qq[u] < 0) continue;
            mark(qq[u], il[u], ilp[u], rr[u]);
            if (!TMA && staged) sv_w[e0 + u * blockDim.x] = val[u];
          }
        }
      }
    }
    APPLY_MARK(1);
    __syncthreads();
    // the CTA's next segment: descriptor and bulk copies into the other buffer
    // (its previous user finished before this iteration's first barrier)
    if (TMA && warp0 && seg + gridDim.x < nseg) {
      describe(b ^ 1, seg + gridDim.x, nl, nc);
      if (seg + 2 * gridDim.x < nseg) fetch(seg + 2 * gridDim.x, nl, nc);
    }
    if (!tot) continue;  // uniform across the CTA
    // 2. fold and update.  Each warp compacts the touched indices of 32
    //    bitmap words at a time into its shared list (word, bit order), then
    //    folds them lane-parallel: the lanes' work no longer follows the
    //    words' popcounts, and neighbouring lanes read neighbouring theta
    //    sectors.  theta loads of up to U indices are issued together; the
    //    consumed bitmap words are re-zeroed for the next segment.
    for (uint32_t w0 = (threadIdx.x >> 5) << 5; w0 < NW; w0 += blockDim.x) {
      const uint32_t w = w0 + lane;  // NW is a multiple of 32 (S >= 2^10)
      uint32_t uni = 0;
      for (int q = 0; q < P; ++q) uni |= bm[(size_t)q * NW + w];
      const uint32_t c = __popc(uni);
      const uint32_t incl = warp_incl(c);
      const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
      if (!total) continue;  // uniform across the warp (and the words are zero)
      uint16_t* wl = wlist[threadIdx.x >> 5];
      for (uint32_t off = incl - c; uni; uni &= uni - 1) wl[off++] = (uint16_t)((w << 5) | (__ffs(uni) - 1));
      uint32_t lbase = 0;
      if (list_idx) {  // list mode (sharded multi-rank apply): one slot per touched index
        if (lane == 0) lbase = atomicAdd(list_cnt, total);
        lbase = __shfl_sync(0xffffffffu, lbase, 0);
      }
      __syncwarp();
      for (uint32_t t0 = lane; t0 < total; t0 += 32 * U) {
        uint32_t li[U];
        T th[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint32_t t = t0 + 32 * u;
          li[u] = 0xffffffffu;
          if (t < total) {
            li[u] = wl[t];
            th[u] = theta ? theta[seg_base + li[u]] : T(0);
          }
        }
        auto finish = [&](auto get) {
#pragma unroll
          for (int u = 0; u < U; ++u) {
            if (li[u] == 0xffffffffu) continue;
            const uint32_t ww = li[u] >> 5;
            const uint32_t bit = 1u << (li[u] & 31), below = bit - 1u;
            const size_t i = seg_base + li[u];
            auto g = [&](int q2) { return get(q2, ww, bit, below); };
            T t = th[u];
            if (ASYNC) {  // slot = worker
              auto step = [&](int q2) {
                const T x = add_rn(mul_rn(coefs[q2], g(q2)), t);
                t = (bm[(size_t)q2 * NW + ww] & bit) ? x : t;
              };
              if constexpr (PT > 0) {
#pragma unroll
                for (int q2 = 0; q2 < PT; ++q2) step(q2);
              } else {
                for (int q2 = 0; q2 < P; ++q2) step(q2);
              }
            } else {
              T sum;
              if (plain) {  // the reference order is the slot order
                sum = g(0);
                if constexpr (PT > 0) {
#pragma unroll
                  for (int s2 = 1; s2 < PT; ++s2) sum = add_rn(sum, g(s2));
                } else {
                  for (int s2 = 1; s2 < P; ++s2) sum = add_rn(sum, g(s2));
                }
              } else {
                const int rs = order == PSB_ORDER_RING ? rc.start_for(i, n, P) : 0;
                sum = fold_sum_start<T>(g, P, order, rs, dpn, npr);
              }
              const T mean = mul_rn(sum, inv);
              t = add_rn(mul_rn(coef, mean), t);
              if (mean_out) mean_out[i] = mean;
            }
            if (theta) {
              theta[i] = t;
              bad |= !is_finite(t);
            }
            if (list_idx) {
              const uint32_t lp = lbase + t0 + 32 * u;
              list_idx[lp] = (uint32_t)i;
              list_val[lp] = t;
            }
          }
        };
        if (staged) {
          // branch-free: every worker's lookup is issued; absent ones read a
          // clamped (unused) slot and contribute +0
          finish([&](int q2, uint32_t ww, uint32_t bit, uint32_t below) -> T {
            const uint32_t word = bm[(size_t)q2 * NW + ww];
            const uint32_t at = min(pre[(size_t)q2 * NW + ww] + __popc(word & below), scap - 1);
            const T x = sval[at];
            return (word & bit) ? x : T(0);
          });
        } else {
          finish([&](int q2, uint32_t ww, uint32_t bit, uint32_t below) -> T {  // q2: slot
            const uint32_t word = bm[(size_t)q2 * NW + ww];
            if (!(word & bit)) return T(0);
            const int q = worker_at(q2);
            return pl_val<T>(v, q, lo[q] - vb[q] + pre[(size_t)q2 * NW + ww] + __popc(word & below));
          });
        }
      }
      __syncwarp();  // the list is rewritten by the warp's next chunk
      for (int q = 0; q < P; ++q) bm[(size_t)q * NW + w] = 0u;
    }
    APPLY_MARK(2);
  }
  if (bad) atomicOr(flags, 1u);
}

// Segments of at most 32 entries (most of the index space of a skewed
// gradient: 60 % of cfg2's segments hold ~17), one warp each: a lane per
// entry, the lanes holding the same index found with __match_any_sync; the
// lowest one (the lowest worker) folds the P values (+0 where absent) in the
// reference order and updates theta once -- no bitmaps, no CTA barriers.
// Bitwise the same arithmetic as k_sparse_apply_bm.
template <class T, bool ASYNC>
__global__ void __launch_bounds__(256) k_sparse_apply_light(PayloadView v, int P, uint32_t nseg, int seg_shift,
                                                            uint32_t light_max, const uint32_t* __restrict__ seg_off,
                                                            int order, uint32_t dpn, uint32_t npr, T coef,
                                                            WorkerCoefs wscale, T* __restrict__ theta, size_t n,
                                                            T* __restrict__ mean_out, uint32_t* flags) {
  __shared__ int sq[8][32];
  __shared__ T sv[8][32];
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (flags != nullptr && (__ldcg(flags) & 8u)) return;  // a peer timed out: theta untouched
  const T inv = (T)(1.0 / (double)P);
  bool bad = false;
  RingChunk rc;
  const uint32_t warp = blockIdx.x * (blockDim.x >> 5) + wid, nwarps = gridDim.x * (blockDim.x >> 5);
  for (uint32_t seg = warp; seg < nseg; seg += nwarps) {
    uint32_t l = 0, cnt = 0;
    if (lane < (uint32_t)P) {
      const uint32_t* row = v.wpr ? reinterpret_cast<const uint32_t*>(v.rank_base[lane / v.wpr] + v.tab_off) +
                                        (size_t)lane * (nseg + 1)
                                  : seg_off + (size_t)lane * (nseg + 1);
      l = row[seg];
      cnt = row[seg + 1] - l;
    }
    uint32_t incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= (uint32_t)o) incl += t;
    }
    const uint32_t tot = __shfl_sync(0xffffffffu, incl, 31);
    if (tot == 0 || tot > light_max) continue;  // uniform; heavy segments are the TMA kernel's
    // worker of entry `lane`: the lowest p with lane < incl_p
    int q = -1;
    uint32_t base = 0, lq = 0;
    for (int p = P - 1; p >= 0; --p) {
      const uint32_t ip = __shfl_sync(0xffffffffu, incl, p), cp = __shfl_sync(0xffffffffu, cnt, p);
      const uint32_t pl = __shfl_sync(0xffffffffu, l, p);
      if (lane < ip && lane >= ip - cp) {
        q = p;
        base = ip - cp;
        lq = pl;
      }
    }
    const size_t seg_base = (size_t)seg << seg_shift;
    uint32_t i32 = 0xffffffffu;
    T x = T(0);
    if (lane < tot) {
      const uint32_t j = lq + (lane - base);
      if (v.idx16)
        i32 = (uint32_t)seg_base + reinterpret_cast<const uint16_t*>(pl_block(v, q))[j];
      else
        i32 = pl_idx(v, q)[j];
      x = pl_val<T>(v, q, j);
    }
    sq[wid][lane] = q;
    sv[wid][lane] = x;
    const unsigned act = __ballot_sync(0xffffffffu, lane < tot);
    const unsigned grp = __match_any_sync(0xffffffffu, i32);
    __syncwarp();
    if (lane < tot && (__ffs(grp) - 1) == (int)lane) {  // the group's owner: its lowest worker
      const size_t i = i32;
      const unsigned mem = grp & act;
      auto g = [&](int qq) -> T {
        for (unsigned m = mem; m; m &= m - 1) {
          const int ml = __ffs(m) - 1;
          if (sq[wid][ml] == qq) return sv[wid][ml];
        }
        return T(0);
      };
      T t = theta ? theta[i] : T(0);
      if (ASYNC) {
        for (unsigned m = mem; m; m &= m - 1) {  // present workers in worker order
          const int ml = __ffs(m) - 1;
          t = add_rn(mul_rn((T)(-wscale.v[sq[wid][ml]]), sv[wid][ml]), t);
        }
      } else {
        const int rs = order == PSB_ORDER_RING ? rc.start_for(i, n, P) : 0;
        const T mean = mul_rn(fold_sum_start<T>(g, P, order, rs, dpn, npr), inv);
        t = add_rn(mul_rn(coef, mean), t);
        if (mean_out) mean_out[i] = mean;
      }
      if (theta) {
        theta[i] = t;
        bad |= !is_finite(t);
      }
    }
    __syncwarp();
  }
  if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(flags, 1u);
}

// Dense payloads (P*k a large fraction of n): fold by streaming.  One CTA per
// segment (S <= 32 KB of accumulator) folds the workers in the reference
// order, one pass per worker: pass s adds the s-th worker's values at its
// indices (the first present value initialises the element).  Skipping the
// absent workers' +0 terms only changes the sign of a zero sum, and the
// reference's result is recovered exactly by one final RN(acc + (+0)) where
// any worker was absent (a -0 partial sum becomes +0 at the first absent
// worker and stays +0; any other value is unchanged by +0).  theta then
// streams through once: theta = RN(RN(-lr * RN(acc * (1/P))) + theta) (acc =
// +0 where no worker is present: theta + (-0) leaves theta bitwise
// unchanged, so the host requires lr >= 0).  A segment crossing a ring chunk
// boundary is two ranges with their own rotation.  Plain orders only (naive,
// ring, hierarchical within one node).
constexpr int kDenseTile = 8192;

template <class T>
__global__ void __launch_bounds__(256) k_dense_fold_apply(PayloadView v, int P, uint32_t nseg, int seg_shift,
                                                          const uint32_t* __restrict__ seg_off, int ring, T coef,
                                                          T* __restrict__ theta, size_t n, uint32_t* flags) {
  constexpr uint32_t TT = kDenseTile * 4 / sizeof(T);  // 32 KB of accumulator
  __shared__ __align__(16) T acc[TT];
  __shared__ uint8_t cnt[TT];
  __shared__ uint32_t lo_s[PSB_MAX_P], cnt_s[PSB_MAX_P];
  const T inv = (T)(1.0 / (double)P);
  const uint32_t S = 1u << seg_shift;  // <= TT (host)
  bool bad = false;
  if (flags != nullptr && (__ldcg(flags) & 8u)) return;
  RingChunk rc;
  for (uint32_t seg = blockIdx.x; seg < nseg; seg += gridDim.x) {
    const size_t tlo = (size_t)seg << seg_shift;
    const size_t thi = min(tlo + S, n);
    __syncthreads();  // the previous segment is done with shared memory
    if (threadIdx.x < (unsigned)P) {
      const uint32_t* row = seg_off + (size_t)threadIdx.x * (nseg + 1);
      lo_s[threadIdx.x] = row[seg];
      cnt_s[threadIdx.x] = row[seg + 1] - row[seg];
    }
    for (uint32_t e = threadIdx.x; e < S / 4; e += blockDim.x) reinterpret_cast<uint32_t*>(cnt)[e] = 0u;
    size_t b = thi;  // first index of the second range (ring chunk boundary)
    int rotA = 0, rotB = 0;
    if (ring) {
      rotA = rc.start_for(tlo, n, P);
      if (rc.hi < thi) {
        b = rc.hi;
        rotB = rc.start_for(b, n, P);
      }
    }
    __syncthreads();
    for (int s = 0; s < P; ++s) {
      for (int r = 0; r < 2; ++r) {
        const size_t rlo = r ? b : tlo, rhi = r ? thi : b;
        if (rlo >= rhi) continue;
        int q = (r ? rotB : rotA) + s;
        if (q >= P) q -= P;
        const uint32_t l = lo_s[q], c = cnt_s[q];
        const uint8_t* blk = pl_block(v, q);
        for (uint32_t j = threadIdx.x; j < c; j += blockDim.x) {
          const uint32_t jj = l + j;
          const size_t i = v.idx16 ? (tlo + reinterpret_cast<const uint16_t*>(blk)[jj])
                                   : (size_t)reinterpret_cast<const uint32_t*>(blk)[jj];
          if (i < rlo || i >= rhi) continue;
          const uint32_t e = (uint32_t)(i - tlo);
          const T x = pl_val<T>(v, q, jj);
          acc[e] = cnt[e] ? add_rn(acc[e], x) : x;
          cnt[e] += 1;
        }
      }
      __syncthreads();  // worker s's additions precede worker s+1's
    }
    const uint32_t m = (uint32_t)(thi - tlo);
    auto fin = [&](uint32_t e) -> T {  // the reference's sum: +0 where any worker is absent
      const T a = cnt[e] ? acc[e] : T(0);
      return cnt[e] < (uint32_t)P ? add_rn(a, T(0)) : a;
    };
    if (sizeof(T) == 4 && (m & 3) == 0 && ((((uintptr_t)theta) + tlo * 4) & 15) == 0) {
      const float cf = (float)coef, iv = (float)inv;
      for (uint32_t e4 = threadIdx.x; e4 < m / 4; e4 += blockDim.x) {
        float4 th = __ldcs(reinterpret_cast<const float4*>(theta + tlo) + e4);
        const uint32_t e = e4 * 4;
        th.x = __fadd_rn(__fmul_rn(cf, __fmul_rn((float)fin(e), iv)), th.x);
        th.y = __fadd_rn(__fmul_rn(cf, __fmul_rn((float)fin(e + 1), iv)), th.y);
        th.z = __fadd_rn(__fmul_rn(cf, __fmul_rn((float)fin(e + 2), iv)), th.z);
        th.w = __fadd_rn(__fmul_rn(cf, __fmul_rn((float)fin(e + 3), iv)), th.w);
        __stcs(reinterpret_cast<float4*>(theta + tlo) + e4, th);
        bad |= !is_finite(th.x) || !is_finite(th.y) || !is_finite(th.z) || !is_finite(th.w);
      }
    } else {
      for (uint32_t e = threadIdx.x; e < m; e += blockDim.x) {
        const T th = add_rn(mul_rn(coef, mul_rn(fin(e), inv)), theta[tlo + e]);
        theta[tlo + e] = th;
        bad |= !is_finite(th);
      }
    }
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flags, 1u);
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
  RingChunk rc;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x) {
    auto get = [&](int q) -> T {
      if (ONEBIT) {
        const uint32_t w = words[(size_t)q * nw + (i >> 5)];
        return ((w >> (i & 31)) & 1u) ? sc[q] : -sc[q];
      }
      return bufs[(size_t)q * n + i];
    };
    const int rs = order == PSB_ORDER_RING ? rc.start_for(i, n, P) : 0;
    const T mean = mul_rn(fold_sum_start<T>(get, P, order, rs, dpn, npr), inv);
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
  PayloadView v{};
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
                       cudaStream_t st, const uint32_t* tab = nullptr, const PayloadView* vdirect = nullptr) {
  PayloadView v = vdirect ? *vdirect : make_view(comp, sizeof(T) == 8 ? PSB_F64 : PSB_F32, payloads, k);
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
  // bitmap segments: P * (S/32) * 8 B <= 16 KB (2^10 <= S <= 2^15), plus a
  // stage of vcap (value, local index) pairs; a segment with more entries
  // reads them from L2 instead
  const int seg_shift = psb_apply_seg_shift(P);
  const uint32_t nseg = (uint32_t)((n + ((size_t)1 << seg_shift) - 1) >> seg_shift);
  PSB_REQUIRE(c, k <= 0xffffffffu, "sparse apply: k exceeds 32-bit positions");
  // dense payloads: the streaming fold (plain orders, no mean_out / async,
  // lr >= 0, gathered or wire16 views), over segments of at most 32 KB of
  // accumulator (its own offset table when the apply computes the table)
  const bool plain_order = order == PSB_ORDER_NAIVE || order == PSB_ORDER_RING ||
                           (order == PSB_ORDER_HIER && dpn >= (uint32_t)P);
  const int dshift = sizeof(T) == 4 ? 13 : 12;
  // (P = 2 measured slower dense: rho 10 % 376 -> 425 us)
  if (c->dense_fold_pct && P >= 4 && !async_mode && !mean_out && theta && plain_order && !v.q8 && !v.wpr &&
      !(coef > T(0)) &&
      (!tab || seg_shift <= dshift) && (double)P * (double)k * 100.0 >= (double)c->dense_fold_pct * (double)n) {
    int sh = seg_shift;
    uint32_t ns = nseg;
    if (!tab) {
      sh = std::min(seg_shift, dshift);
      ns = (uint32_t)((n + ((size_t)1 << sh) - 1) >> sh);
      PSB_REQUIRE(c, (size_t)P * (ns + 1) <= c->seg_cap, "dense fold: segment table exceeds ctx capacity");
      const unsigned gx = (unsigned)((k + 256 * kSegU - 1) / (256 * kSegU));
      k_seg_offsets<<<dim3(gx, (unsigned)P), 256, 0, st>>>(v, P, (uint32_t)k, ns, sh, c->d_seg_off, nullptr, 0, 0);
      c->launches += 1;
      tab = c->d_seg_off;
    }
    const unsigned grid = (unsigned)std::min<size_t>(ns, (size_t)c->num_sms * 8);
    k_dense_fold_apply<T><<<grid, 256, 0, st>>>(v, P, ns, sh, tab, order == PSB_ORDER_RING ? 1 : 0, coef, theta, n,
                                                c->d_flags);
    c->launches += 1;
    PSB_LAUNCH_CHECK(c, "psb_sparse_mean_sgd (dense fold)");
    return PSB_OK;
  }
  if (!tab) {
    PSB_REQUIRE(c, (size_t)P * (nseg + 1) <= c->seg_cap, "sparse apply: segment table exceeds ctx capacity");
    const unsigned gx = (unsigned)((k + 256 * kSegU - 1) / (256 * kSegU));
    k_seg_offsets<<<dim3(gx, (unsigned)P), 256, 0, st>>>(v, P, (uint32_t)k, nseg, seg_shift, c->d_seg_off, nullptr,
                                                         0, 0);
    c->launches += 1;
    tab = c->d_seg_off;
  }
  const uint32_t vcap = c->apply_vcap;
  // TMA-staged entries: f32/f64 top-k payloads (gathered, wire16, or read in
  // place from the peers' arenas) on 16-byte boundaries; q8 values keep the
  // thread-loaded path
  bool direct_ok = true;  // direct view: every rank's arena on 16-byte boundaries
  for (int r = 0; v.wpr && r < (P + v.wpr - 1) / v.wpr; ++r) direct_ok &= ((uintptr_t)v.rank_base[r] & 15) == 0;
  const bool tma = !c->apply_no_tma && !v.q8 && direct_ok && ((uintptr_t)v.base & 15) == 0 &&
                   (v.block_bytes & 15) == 0 && (v.val_off & 15) == 0;
  const uint32_t ib = v.idx16 ? 2 : 4;
  const size_t tcap = c->apply_tma_cap;  // entries per TMA stage (+ the 16-byte widening)
  const uint32_t ci = (uint32_t)psb_align16((tcap + 16 * (size_t)P) * ib);
  const uint32_t cv = (uint32_t)psb_align16((tcap + 8 * (size_t)P) * sizeof(T));
  const size_t smem = (((size_t)P * 8) << (seg_shift - 5)) + (tma ? (size_t)ci + 2 * (size_t)cv : (size_t)vcap * sizeof(T));
  WorkerCoefs ws{};
  if (async_mode)
    for (int q = 0; q < P; ++q) ws.v[q] = wscale_host[q];
  const int PTi = P == 2 || P == 4 || P == 8 ? P : 0;
  // segments of <= 32 entries: one warp each (k_sparse_apply_light), the
  // TMA kernel skips them
  // (P = 2: measured 81 -> 85 us; direct view: the warp's remote row / entry
  // loads are slower than the TMA stage, N = 4 0.421 -> 0.429 ms: both off)
  const uint32_t light = tma && P >= 4 && !v.wpr ? c->apply_light : 0u;
  auto launch = [&](auto kern, T* mo, bool is_tma) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int thr = apply_threads(PTi, is_tma);
    // TMA: persistent CTAs (the stage pipelines a CTA's consecutive
    // segments); otherwise one CTA per segment, many in flight
    unsigned grid = (unsigned)std::min<size_t>(nseg, 1u << 20);
    if (is_tma) {
      int occ = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, thr, smem);
      grid = (unsigned)std::min<size_t>(nseg, (size_t)c->num_sms * (size_t)std::max(occ, 1));
    }
    kern<<<grid, thr, smem, st>>>(v, P, nseg, 0u, nullptr, seg_shift, vcap, ci, cv, is_tma ? light : 0u, tab,
                                  (int)order, dpn, npr, coef, ws, theta, n, mo, nullptr, nullptr, nullptr, c->d_flags);
  };
  if (light) {
    const unsigned lgrid = (unsigned)std::min<size_t>((nseg + 7) / 8, (size_t)c->num_sms * 16);
    if (async_mode)
      k_sparse_apply_light<T, true><<<lgrid, 256, 0, st>>>(v, P, nseg, seg_shift, light, tab, (int)order, dpn, npr,
                                                            coef, ws, theta, n, nullptr, c->d_flags);
    else
      k_sparse_apply_light<T, false><<<lgrid, 256, 0, st>>>(v, P, nseg, seg_shift, light, tab, (int)order, dpn, npr,
                                                             coef, ws, theta, n, mean_out, c->d_flags);
    c->launches += 1;
  }
#define PSB_APPLY_LAUNCH(ASY, MO)                                                                       \
  do {                                                                                                  \
    if (tma) {                                                                                          \
      switch (P) {                                                                                      \
        case 2: launch(k_sparse_apply_bm<T, ASY, 2, true>, MO, true); break;                            \
        case 4: launch(k_sparse_apply_bm<T, ASY, 4, true>, MO, true); break;                            \
        case 8: launch(k_sparse_apply_bm<T, ASY, 8, true>, MO, true); break;                            \
        default: launch(k_sparse_apply_bm<T, ASY, 0, true>, MO, true);                                  \
      }                                                                                                 \
    } else {                                                                                            \
      switch (P) {                                                                                      \
        case 2: launch(k_sparse_apply_bm<T, ASY, 2, false>, MO, false); break;                          \
        case 4: launch(k_sparse_apply_bm<T, ASY, 4, false>, MO, false); break;                          \
        case 8: launch(k_sparse_apply_bm<T, ASY, 8, false>, MO, false); break;                          \
        default: launch(k_sparse_apply_bm<T, ASY, 0, false>, MO, false);                                \
      }                                                                                                 \
    }                                                                                                   \
  } while (0)
  if (async_mode)
    PSB_APPLY_LAUNCH(true, nullptr);
  else
    PSB_APPLY_LAUNCH(false, mean_out);
#undef PSB_APPLY_LAUNCH
  c->launches += 1;
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

template <class T>
psb_status shard_fold_impl(psb_ctx* c, int P, const uint32_t* sidx, const T* sval, const uint32_t* srow,
                           const uint32_t* range, int seg_shift, psb_order order, const psb_topology* topo,
                           double lr, const double* wscale_host, bool async_mode, T* theta, size_t n,
                           uint32_t* list_idx, T* list_val, uint32_t* list_cnt, cudaStream_t st) {
  PayloadView v{};  // flat view: every worker's slice lives in one (idx, val) array pair
  v.base = reinterpret_cast<const uint8_t*>(sidx);
  v.block_bytes = 0;
  v.val_off = (size_t)(reinterpret_cast<const uint8_t*>(sval) - v.base);
  v.scale_off = 0;
  v.q8 = 0;
  uint32_t dpn, npr;
  topo_fields(topo, P, &dpn, &npr);
  const T coef = (T)(-lr);
  const uint32_t vcap = c->apply_vcap;
  const size_t smem = (((size_t)P * 8) << (seg_shift - 5)) + (size_t)vcap * sizeof(T);
  WorkerCoefs ws{};
  if (async_mode)
    for (int q = 0; q < P; ++q) ws.v[q] = wscale_host[q];
  auto launch = [&](auto kern) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    // persistent CTAs over the device-decided segment range
    kern<<<c->num_sms * 4, apply_threads(P == 2 || P == 4 || P == 8 ? P : 0, false), smem, st>>>(
        v, P, 0u, 0u, range, seg_shift, vcap, 0u, 0u, 0u, srow, (int)order, dpn, npr, coef, ws, theta, n, nullptr, list_idx,
        list_val, list_cnt, c->d_flags);
  };
  if (async_mode) {
    switch (P) {
      case 2: launch(k_sparse_apply_bm<T, true, 2, false>); break;
      case 4: launch(k_sparse_apply_bm<T, true, 4, false>); break;
      case 8: launch(k_sparse_apply_bm<T, true, 8, false>); break;
      default: launch(k_sparse_apply_bm<T, true, 0, false>);
    }
  } else {
    switch (P) {
      case 2: launch(k_sparse_apply_bm<T, false, 2, false>); break;
      case 4: launch(k_sparse_apply_bm<T, false, 4, false>); break;
      case 8: launch(k_sparse_apply_bm<T, false, 8, false>); break;
      default: launch(k_sparse_apply_bm<T, false, 0, false>);
    }
  }
  c->launches += 1;
  PSB_LAUNCH_CHECK(c, "shard fold");
  return PSB_OK;
}

// Momentum SGD (north-star a24, this build's rule; include/psb.h):
// m = RN(RN(beta*m) + mean); theta = RN(RN(-lr*m) + theta).  Dense, 20 B/el (f32).
template <class T>
__global__ void __launch_bounds__(256) k_momentum(const T* __restrict__ mean, T* __restrict__ m,
                                                  T* __restrict__ theta, T beta, T coef, size_t n, uint32_t* flags) {
  bool bad = false;
  auto one = [&](size_t i) {
    const T mi = add_rn(mul_rn(beta, m[i]), mean[i]);
    m[i] = mi;
    const T th = add_rn(mul_rn(coef, mi), theta[i]);
    theta[i] = th;
    bad |= !is_finite(th);
  };
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  const size_t t0 = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (sizeof(T) == 4 && ((((uintptr_t)mean) | ((uintptr_t)m) | ((uintptr_t)theta)) & 15) == 0) {
    const size_t nv = n / 4;
    for (size_t v = t0; v < nv; v += stride) {
      const float4 g4 = __ldcs(reinterpret_cast<const float4*>(mean) + v);
      float4 m4 = __ldcs(reinterpret_cast<const float4*>(m) + v);
      float4 t4 = __ldcs(reinterpret_cast<const float4*>(theta) + v);
      const float b = (float)beta, cf = (float)coef;
      m4.x = __fadd_rn(__fmul_rn(b, m4.x), g4.x);
      m4.y = __fadd_rn(__fmul_rn(b, m4.y), g4.y);
      m4.z = __fadd_rn(__fmul_rn(b, m4.z), g4.z);
      m4.w = __fadd_rn(__fmul_rn(b, m4.w), g4.w);
      t4.x = __fadd_rn(__fmul_rn(cf, m4.x), t4.x);
      t4.y = __fadd_rn(__fmul_rn(cf, m4.y), t4.y);
      t4.z = __fadd_rn(__fmul_rn(cf, m4.z), t4.z);
      t4.w = __fadd_rn(__fmul_rn(cf, m4.w), t4.w);
      __stcs(reinterpret_cast<float4*>(m) + v, m4);
      __stcs(reinterpret_cast<float4*>(theta) + v, t4);
      bad |= !is_finite(t4.x) || !is_finite(t4.y) || !is_finite(t4.z) || !is_finite(t4.w);
    }
    for (size_t i = nv * 4 + t0; i < n; i += stride) one(i);
  } else {
    for (size_t i = t0; i < n; i += stride) one(i);
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flags, 1u);
}

// Single-worker top-k momentum step without a dense mean scratch: the mean
// is the payload itself (P = 1: fold of one buffer, scaled by 1/1), already
// sorted by index.  k_tile_starts cuts the payload at 4096-element tiles;
// k_momentum_merge scatters a tile's entries into a zeroed shared-memory tile
// and makes the dense m / theta pass (16 B/el, f32) reading the mean from it.
constexpr int kMomTile = 4096;

__global__ void k_tile_starts(const uint32_t* __restrict__ idx, size_t k, uint32_t* __restrict__ starts,
                              long long ntiles) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t j = (size_t)blockIdx.x * blockDim.x + threadIdx.x; j <= k; j += stride) {
    const long long cur = j < k ? (long long)(idx[j] / kMomTile) : ntiles;
    const long long prev = j > 0 ? (long long)(idx[j - 1] / kMomTile) : -1;
    for (long long t = prev + 1; t <= cur; ++t) starts[t] = (uint32_t)j;
  }
}

template <class T>
__global__ void __launch_bounds__(256) k_momentum_merge(const uint32_t* __restrict__ idx, const T* __restrict__ val,
                                                        const uint32_t* __restrict__ starts, T* __restrict__ m,
                                                        T* __restrict__ theta, T* __restrict__ mean_out, T beta,
                                                        T coef, size_t n, uint32_t* flags) {
  __shared__ __align__(16) T gt[kMomTile];
  for (int e = threadIdx.x; e < kMomTile; e += blockDim.x) gt[e] = T(0);
  bool bad = false;
  const size_t ntiles = (n + kMomTile - 1) / kMomTile;
  const bool vec = sizeof(T) == 4 && ((((uintptr_t)m) | ((uintptr_t)theta) | ((uintptr_t)mean_out)) & 15) == 0;
  for (size_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const size_t lo = t * kMomTile;
    const uint32_t a = starts[t], b = starts[t + 1];
    __syncthreads();  // zeroed tile (first pass / previous un-scatter) visible
    for (uint32_t j = a + threadIdx.x; j < b; j += blockDim.x) gt[idx[j] - lo] = val[j];
    __syncthreads();
    if (vec && lo + kMomTile <= n) {
      constexpr int V = kMomTile / 4 / 256;
      float4 m4[V], t4[V];
#pragma unroll
      for (int u = 0; u < V; ++u) {
        const size_t v = lo / 4 + threadIdx.x + (size_t)u * 256;
        m4[u] = __ldcs(reinterpret_cast<const float4*>(m) + v);
        t4[u] = __ldcs(reinterpret_cast<const float4*>(theta) + v);
      }
      const float bb = (float)beta, cf = (float)coef;
#pragma unroll
      for (int u = 0; u < V; ++u) {
        const int e4 = threadIdx.x + u * 256;
        const float4 g4 = reinterpret_cast<const float4*>(gt)[e4];
        float4 a4 = m4[u], th = t4[u];
        a4.x = __fadd_rn(__fmul_rn(bb, a4.x), g4.x);
        a4.y = __fadd_rn(__fmul_rn(bb, a4.y), g4.y);
        a4.z = __fadd_rn(__fmul_rn(bb, a4.z), g4.z);
        a4.w = __fadd_rn(__fmul_rn(bb, a4.w), g4.w);
        th.x = __fadd_rn(__fmul_rn(cf, a4.x), th.x);
        th.y = __fadd_rn(__fmul_rn(cf, a4.y), th.y);
        th.z = __fadd_rn(__fmul_rn(cf, a4.z), th.z);
        th.w = __fadd_rn(__fmul_rn(cf, a4.w), th.w);
        const size_t v = lo / 4 + e4;
        __stcs(reinterpret_cast<float4*>(m) + v, a4);
        __stcs(reinterpret_cast<float4*>(theta) + v, th);
        if (mean_out) reinterpret_cast<float4*>(mean_out)[v] = g4;
        bad |= !is_finite(th.x) || !is_finite(th.y) || !is_finite(th.z) || !is_finite(th.w);
      }
    } else {
      for (int e = threadIdx.x; e < kMomTile && lo + e < n; e += blockDim.x) {
        const size_t i = lo + e;
        const T mi = add_rn(mul_rn(beta, m[i]), gt[e]);
        m[i] = mi;
        const T th = add_rn(mul_rn(coef, mi), theta[i]);
        theta[i] = th;
        if (mean_out) mean_out[i] = gt[e];
        bad |= !is_finite(th);
      }
    }
    __syncthreads();  // every thread done reading the tile
    for (uint32_t j = a + threadIdx.x; j < b; j += blockDim.x) gt[idx[j] - lo] = T(0);
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flags, 1u);
}

}  // namespace

psb_status psb_momentum_topk1(psb_ctx* c, psb_dtype dt, const uint8_t* payload, size_t k, void* m, void* theta,
                              void* mean_out, double beta, double lr, size_t n, uint32_t* starts_buf,
                              cudaStream_t st) {
  const long long ntiles = (long long)((n + kMomTile - 1) / kMomTile);
  const uint32_t* idx = reinterpret_cast<const uint32_t*>(payload);
  const void* val = payload + psb_align16(k * 4);
  const unsigned g0 = (unsigned)std::max<size_t>(1, std::min<size_t>((k + 1 + 255) / 256, (size_t)c->num_sms * 8));
  k_tile_starts<<<g0, 256, 0, st>>>(idx, k, starts_buf, ntiles);
  const unsigned grid = (unsigned)std::max<long long>(1, std::min<long long>(ntiles, (long long)c->num_sms * 8));
  if (dt == PSB_F32)
    k_momentum_merge<float><<<grid, 256, 0, st>>>(idx, (const float*)val, starts_buf, (float*)m, (float*)theta,
                                                   (float*)mean_out, (float)beta, (float)(-lr), n, c->d_flags);
  else
    k_momentum_merge<double><<<grid, 256, 0, st>>>(idx, (const double*)val, starts_buf, (double*)m, (double*)theta,
                                                    (double*)mean_out, beta, -lr, n, c->d_flags);
  c->launches += 2;
  PSB_LAUNCH_CHECK(c, "psb_momentum_topk1");
  return PSB_OK;
}

extern "C" psb_status psb_momentum_sgd(psb_ctx* c, psb_dtype dt, const void* mean, void* m, void* theta, double beta,
                                       double lr, size_t n, psb_stream_t stream) {
  PSB_REQUIRE(c, c != nullptr, "null ctx");
  PSB_REQUIRE(c, dt == PSB_F32 || dt == PSB_F64, "momentum: bad dtype");
  PSB_REQUIRE(c, mean && m && theta, "momentum: null buffer");
  PSB_REQUIRE(c, lr > 0.0, "HyperParams: learning_rate must be > 0");
  cudaStream_t st = (cudaStream_t)stream;
  const unsigned grid = (unsigned)std::max<size_t>(1, std::min<size_t>((n / 4 + 255) / 256, (size_t)c->num_sms * 8));
  if (dt == PSB_F32)
    k_momentum<float><<<grid, 256, 0, st>>>((const float*)mean, (float*)m, (float*)theta, (float)beta, (float)(-lr),
                                            n, c->d_flags);
  else
    k_momentum<double><<<grid, 256, 0, st>>>((const double*)mean, (double*)m, (double*)theta, beta, -lr, n,
                                             c->d_flags);
  c->launches += 1;
  PSB_LAUNCH_CHECK(c, "psb_momentum_sgd");
  return PSB_OK;
}

psb_status psb_sparse_apply_tab(psb_ctx* c, psb_compressor comp, psb_dtype dt, int P, const void* payloads, size_t k,
                                const uint32_t* tab, psb_order order, const psb_topology* topo, double lr,
                                const double* wscale, int async_mode, void* theta, size_t n, void* mean_out,
                                cudaStream_t st) {
  if (dt == PSB_F64)
    return sparse_impl<double>(c, comp, P, payloads, k, order, topo, lr, wscale, async_mode != 0, (double*)theta, n,
                               (double*)mean_out, st, tab);
  return sparse_impl<float>(c, comp, P, payloads, k, order, topo, lr, wscale, async_mode != 0, (float*)theta, n,
                            (float*)mean_out, st, tab);
}

// wire16 pack: a standard top-k payload block (u32 idx | val) -> (u16 idx &
// (S-1) | val) -- the apply segment of S = 2^seg_shift <= 2^16 indices an
// entry falls in is recovered from the per-segment offset rows.
namespace {
}  // namespace

size_t psb_wire16_bytes(psb_dtype dt, size_t k) {
  return psb_align16(2 * k) + psb_align16((dt == PSB_F64 ? 8 : 4) * k);
}

// P wire16 payloads (blocks of psb_wire16_bytes) + their offset rows -> apply.
psb_status psb_sparse_apply_wire16(psb_ctx* c, psb_dtype dt, int P, const void* payloads, size_t k,
                                   const uint32_t* tab, psb_order order, const psb_topology* topo, double lr,
                                   const double* wscale, int async_mode, void* theta, size_t n, void* mean_out,
                                   cudaStream_t st) {
  PayloadView v{};
  v.base = reinterpret_cast<const uint8_t*>(payloads);
  v.block_bytes = psb_wire16_bytes(dt, k);
  v.val_off = psb_align16(2 * k);
  v.idx16 = 1;
  if (dt == PSB_F64)
    return sparse_impl<double>(c, PSB_COMP_TOPK, P, payloads, k, order, topo, lr, wscale, async_mode != 0,
                               (double*)theta, n, (double*)mean_out, st, tab, &v);
  return sparse_impl<float>(c, PSB_COMP_TOPK, P, payloads, k, order, topo, lr, wscale, async_mode != 0, (float*)theta,
                            n, (float*)mean_out, st, tab, &v);
}

// Direct multi-rank apply: the P payloads (standard, or wire16 when
// `wire16`) and their offset rows are read in place from every rank's
// NVLink-mapped arena (no pull copy; the TMA stage brings them in).
psb_status psb_sparse_apply_direct(psb_ctx* c, psb_compressor comp, psb_dtype dt, int P, int W,
                                   const uint8_t* const* rank_region, size_t k, size_t tab_off, psb_order order,
                                   const psb_topology* topo, double lr, const double* wscale, int async_mode,
                                   void* theta, size_t n, void* mean_out, cudaStream_t st, bool wire16) {
  PayloadView v = make_view(comp, dt, rank_region[c->rank], k);
  if (wire16) {
    v.block_bytes = psb_wire16_bytes(dt, k);
    v.val_off = psb_align16(2 * k);
    v.idx16 = 1;
  }
  v.wpr = W;
  v.tab_off = tab_off;
  for (int r = 0; r < c->nranks; ++r) v.rank_base[r] = rank_region[r];
  const uint32_t* dummy_tab = reinterpret_cast<const uint32_t*>(rank_region[c->rank] + tab_off);
  if (dt == PSB_F64)
    return sparse_impl<double>(c, comp, P, nullptr, k, order, topo, lr, wscale, async_mode != 0, (double*)theta, n,
                               (double*)mean_out, st, dummy_tab, &v);
  return sparse_impl<float>(c, comp, P, nullptr, k, order, topo, lr, wscale, async_mode != 0, (float*)theta, n,
                            (float*)mean_out, st, dummy_tab, &v);
}

psb_status psb_seg_offsets(psb_ctx* c, psb_compressor comp, psb_dtype dt, int nw, const void* payloads, size_t k,
                           uint32_t nseg, int seg_shift, uint32_t* rows, cudaStream_t st, void* out16,
                           size_t out_stride) {
  const PayloadView v = make_view(comp, dt, payloads, k);
  const unsigned gx = (unsigned)((k + 256 * kSegU - 1) / (256 * kSegU));
  k_seg_offsets<<<dim3(gx, (unsigned)nw), 256, 0, st>>>(v, nw, (uint32_t)k, nseg, seg_shift, rows,
                                                        reinterpret_cast<uint8_t*>(out16), out_stride,
                                                        dt == PSB_F64 ? 8 : 4);
  c->launches += 1;
  PSB_LAUNCH_CHECK(c, "segment offsets");
  return PSB_OK;
}

psb_status psb_shard_fold(psb_ctx* c, psb_dtype dt, int P, const uint32_t* sidx, const void* sval,
                          const uint32_t* srow, const uint32_t* range, int seg_shift, psb_order order,
                          const psb_topology* topo, double lr, const double* wscale, int async_mode, void* theta,
                          size_t n, uint32_t* list_idx, void* list_val, uint32_t* list_cnt, cudaStream_t st) {
  if (dt == PSB_F64)
    return shard_fold_impl<double>(c, P, sidx, (const double*)sval, srow, range, seg_shift, order, topo, lr, wscale,
                                   async_mode != 0, (double*)theta, n, list_idx, (double*)list_val, list_cnt, st);
  return shard_fold_impl<float>(c, P, sidx, (const float*)sval, srow, range, seg_shift, order, topo, lr, wscale,
                                async_mode != 0, (float*)theta, n, list_idx, (float*)list_val, list_cnt, st);
}

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

#ifdef PSB_APPLY_TRACE
extern "C" PSB_API void psb_debug_apply_trace(unsigned long long* out8, int reset) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out8, g_apply_trace, sizeof(unsigned long long) * 8);
  if (reset) {
    unsigned long long z[8] = {};
    cudaMemcpyToSymbol(g_apply_trace, z, sizeof(z));
  }
}
#endif

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
