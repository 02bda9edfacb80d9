// psb_topk.cu -- K1: fused error-feedback add + exact top-k selection.
//
// Replaces ef_compress_step(state, g, {topk, k}) (parsim/compression.hpp:146-157)
// and compress_topk (:81-99).  Reference semantics, restated:
//   p = r + g                                    (:150-151)
//   keep the k largest |p|, ties -> lower index  (stable_sort :85-89)
//   emit indices ascending, values p[idx]        (:91, :97)
//   r' = p - decompress(msg) = selected ? +0 : p (:153-154)
//   check_finite(r')                             (:155)
//
// B200 design: a radix select on the magnitude key
// bits(|p|) (monotone for finite values and +-0).  The lowest-index tie-break
// is exact because every candidate list is kept in index order.
//
//   k_topk_begin  1 CTA: reset per-call scratch, zero histograms.
//   k_scan<A>     THE streaming pass (12N bytes: read g, read r, write r).
//                 Predicted mode (the worker's previous call left a key
//                 threshold G = key(T_prev * rho * f)): index-ordered
//                 compaction of every element with key >= G -- CTA b streams a
//                 contiguous index range and appends to its own segment (block
//                 scan per tile, no cross-CTA waits, no histogram atomics) --
//                 and the residual of those candidates is written as +0
//                 speculatively (most of them are selected).  The last CTA
//                 validates the prediction (count >= k, hence T >= G) and
//                 prefix-sums the segment sizes into one logical list.
//                 Cold mode (no prediction): level-1 histogram of key>>19;
//                 the last CTA resolves digit b1 of the k-th key.
//   k_restore     only on a prediction miss: put p back for pass A's candidates.
//   k_scan<A2>    only on a miss: full level-1 histogram pass (reads p).
//   k_scan<D>     only in cold/miss mode: compaction of digit >= b1.
//   k_cand        ONE cooperative kernel for the whole candidate phase
//                 (psb_cand.inl): slices staged in shared memory, grid-wide
//                 barriers instead of kernel boundaries; the exact threshold T
//                 (predicted mode: two levels on key - G, 2048-ulp coarse bins
//                 then ulps; cold mode: the remaining key radix levels),
//                 per-CTA (gt, eq) counts and their scan, then the ordered
//                 write: slot = gt_before + min(eq_before, need_eq); idx/val
//                 out, residual fix-up (+0 or restore p) and, for a single
//                 worker, the fused SGD update of theta[idx].
// Every kernel is launched unconditionally and exits early from device-side
// flags, so the sequence never syncs the host.  Results never depend on the
// prediction: a miss only costs the fallback passes.
#include <cooperative_groups.h>
#include <cuda_pipeline.h>

#include "psb_internal.cuh"
#include "psb_debug.h"

namespace cg = cooperative_groups;

namespace {

template <class T>
struct VecOf;
template <>
struct VecOf<float> {
  static constexpr int W = 4;
};
template <>
struct VecOf<double> {
  static constexpr int W = 2;
};

template <class T>
__host__ __device__ constexpr int tile_elems() {
  return PSB_SCAN_THREADS * 4 * VecOf<T>::W;  // f32: 4096, f64: 2048
}

enum { MODE_A = 0, MODE_A2 = 1, MODE_D = 2, MODE_S = 3 };
enum { DONE_A = 0, DONE_A2 = 1, DONE_S = 2 };
// flags written by another CTA of the same (cooperative) grid: bypass L1
__device__ __forceinline__ uint32_t ld_flag(const uint32_t* p) { return __ldcg(p); }
#ifndef PSB_SECOND_F
#define PSB_SECOND_F 0.97f  // second-chance threshold factor after a prediction miss (tools/sweep_second.sh)
#endif


// key <-> magnitude value, for the predicted threshold key(T * f)
__device__ __forceinline__ unsigned long long scale_key(unsigned long long key, float f, float) {
  return (unsigned long long)__float_as_uint(__fmul_rn(__uint_as_float((uint32_t)key), f));
}
__device__ __forceinline__ unsigned long long scale_key(unsigned long long key, float f, double) {
  return (unsigned long long)__double_as_longlong(__dmul_rn(__longlong_as_double((long long)key), (double)f));
}
__device__ __forceinline__ double to_mag(unsigned long long key, float) {
  return (double)__uint_as_float((uint32_t)key);
}
__device__ __forceinline__ double to_mag(unsigned long long key, double) {
  return __longlong_as_double((long long)key);
}

template <class T>
struct ScanArgs {
  const T* g;  // MODE_A input gradient
  T* r;        // MODE_A residual (EF) or nullptr
  const T* p;  // MODE_A2 / MODE_D source of p (r if EF else g)
  size_t n;
  uint32_t ntiles;
  int vec_ok;
  TopkScratch* s;
  TopkWorker* w;
  uint32_t* hist1;
  uint32_t* tile_cnt;      // candidates of tile t (segment t of the list)
  uint32_t* sb;            // [3][sb_stride] superblock sums of tile_cnt (passes A, S, D)
  uint32_t sb_stride;
  uint32_t* histd;         // pass A (f32): coarse (key - G) histogram of the candidates, for k_cand
  uint32_t* cand_idx;      // tile-segmented candidates: tile t's at [t*TILE, t*TILE + tile_cnt[t])
  T* cand_val;
  uint32_t* flags;
};

__device__ __forceinline__ void ld_vec(const float* p, float (&x)[4]) {
  float4 v = *reinterpret_cast<const float4*>(p);
  x[0] = v.x; x[1] = v.y; x[2] = v.z; x[3] = v.w;
}
__device__ __forceinline__ void ld_vec(const double* p, double (&x)[2]) {
  double2 v = *reinterpret_cast<const double2*>(p);
  x[0] = v.x; x[1] = v.y;
}
__device__ __forceinline__ void ld_vec_stream(const float* p, float (&x)[4]) {
  float4 v = __ldcs(reinterpret_cast<const float4*>(p));
  x[0] = v.x; x[1] = v.y; x[2] = v.z; x[3] = v.w;
}
__device__ __forceinline__ void ld_vec_stream(const double* p, double (&x)[2]) {
  double2 v = __ldcs(reinterpret_cast<const double2*>(p));
  x[0] = v.x; x[1] = v.y;
}
__device__ __forceinline__ void st_vec(float* p, const float (&x)[4]) {
  *reinterpret_cast<float4*>(p) = make_float4(x[0], x[1], x[2], x[3]);
}
__device__ __forceinline__ void st_vec(double* p, const double (&x)[2]) {
  *reinterpret_cast<double2*>(p) = make_double2(x[0], x[1]);
}
__device__ __forceinline__ void st_vec_stream(float* p, const float (&x)[4]) {
  __stcs(reinterpret_cast<float4*>(p), make_float4(x[0], x[1], x[2], x[3]));
}
__device__ __forceinline__ void st_vec_stream(double* p, const double (&x)[2]) {
  __stcs(reinterpret_cast<double2*>(p), make_double2(x[0], x[1]));
}

// Result of resolving one radix level: the bin b holding the need-th largest
// entry, the count above it and its own count.
struct LevelResult {
  int found;
  uint32_t bin;
  unsigned long long above;
  unsigned long long cnt;
  unsigned long long total;  // sum over the explicit bins
};

// Resolve a <= 4096-bin histogram (one whole CTA).  Bins [max(lo,1), nbins)
// are explicit; bin 0 is implicit (the caller derives it from the matching
// total).  `sh` (>= nbins words of shared memory) stages the histogram with
// coalesced loads; all scanning happens in shared memory.
__device__ void resolve_level(const uint32_t* hist, uint32_t nbins, uint32_t lo,
                              unsigned long long need, unsigned long long* sh_warp,
                              LevelResult* out, uint32_t* sh) {
  const uint32_t t = threadIdx.x;
  for (uint32_t b = t; b < nbins; b += blockDim.x)
    sh[b] = (b >= lo && b >= 1) ? __ldcg(hist + b) : 0u;
  if (t == 0) out->found = 0;
  __syncthreads();
  const uint32_t B = nbins >= blockDim.x ? nbins / blockDim.x : 1;
  const uint32_t b0 = t * B;
  unsigned long long sum = 0;
  if (b0 < nbins)
    for (uint32_t b = b0; b < b0 + B; ++b) sum += sh[b];
  unsigned long long total;
  const unsigned long long ex = block_exscan_u64(sum, sh_warp, &total);
  const unsigned long long suf = total - ex - sum;  // count in bins of threads > t
  if (b0 < nbins && suf < need && need <= suf + sum) {
    unsigned long long cum = suf;
    for (int b = (int)(b0 + B) - 1; b >= (int)b0; --b) {
      const uint32_t h = sh[b];
      if (cum + h >= need) {
        out->found = 1;
        out->bin = (uint32_t)b;
        out->above = cum;
        out->cnt = h;
        break;
      }
      cum += h;
    }
  }
  if (t == 0) out->total = total;
  __syncthreads();
}

// Shared-memory histogram increment aggregated across the warp (call with the
// full warp converged): lanes with the same bin elect one leader that adds the
// group's count.  Candidate keys crowd into a few bins near the threshold, so
// plain per-lane atomics would serialize on one address.
__device__ __forceinline__ void hist_add_agg(uint32_t* sh, uint32_t bin, bool active) {
  const uint32_t am = __ballot_sync(0xffffffffu, active);
  if (!active) return;
  const uint32_t grp = __match_any_sync(am, bin);
  if ((int)(threadIdx.x & 31) == __ffs(grp) - 1) atomicAdd(&sh[bin], (uint32_t)__popc(grp));
}

__device__ __forceinline__ bool last_block(uint32_t* counter) {
  __shared__ int am_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) am_last = atomicAdd(counter, 1u) == gridDim.x - 1;
  __syncthreads();
  if (am_last) __threadfence();
  return am_last;
}

__global__ void k_topk_begin(TopkScratch* s, TopkWorker* w, uint32_t* hist1, uint32_t* histr,
                             unsigned long long n, unsigned long long k, int predict) {
  for (int b = threadIdx.x; b < PSB_HIST_BINS; b += blockDim.x) {
    hist1[b] = 0;
    histr[b] = 0;
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < 8; ++i) s->done[i] = 0;
    for (int i = 0; i < 4; ++i) s->tile_ctr[i] = 0;
    s->b1 = 0;
    s->need_full_hist = 0;
    s->need_compact = 0;
    s->nonfinite = 0;
    s->prefix = 0;
    s->need = k;
    s->match = n;
    s->n = n;
    s->k = k;
    s->cand_count = 0;
    s->start_level = 1;
    s->g_key = predict ? w->g_key : 0ull;
    s->z_key = w->z_key > w->g_key ? w->z_key : w->g_key;
    s->g_key2 = 0;
    // pre-zeroing the candidates' residual pays off while most candidates are
    // selected (restores C - k < zero-writes k)
    s->spec_ok = w->last_ratio < 2.0f ? 1u : 0u;
  }
}

// ------------------------------------------------------------------ scan
// Work distribution: tiles are handed out dynamically (one atomic per tile,
// taken one tile ahead so its latency and the next tile's L2 prefetch overlap
// the current tile).  A static contiguous range per CTA left the pass
// tail-bound: with 4 CTAs per SM sharing issue slots unevenly, CTAs with
// equal work ended between 204 and 271 us at 125M (tools/probe_scan_trace.py).
// Each tile compacts its candidates, in index order, into its own segment of
// the list (t*TILE, capacity TILE) and records the count; k_cand turns the
// segments into one contiguous list (grid-wide prefix over the tile counts).
// (A decoupled look-back writing the contiguous list directly from here was
// measured 3x slower: with ~600 tiles in flight every tile waits for its
// predecessors' counts.)
#ifndef PSB_PF
#define PSB_PF 1  // L2 prefetch of the next tile (tools: PSB_PF=0 disables)
#endif

template <class T, int MODE>
__device__ __forceinline__ void scan_body(const ScanArgs<T>& a) {
  typedef KeyOf<T> KO;
  typedef typename KO::K K;
  constexpr int VW = VecOf<T>::W;
  constexpr int TILE = tile_elems<T>();
  constexpr int SH1 = KO::shift(0);

  __shared__ uint32_t sh_hist[PSB_HIST_BINS];
  __shared__ unsigned long long sh_warp[32];
  __shared__ uint32_t sh_nonfinite;
  __shared__ LevelResult sh_res;
  __shared__ uint32_t sh_tile[2];

  // compact: keep key >= gk.  hist: level-1 histogram of every element.
  K gk = 0;
  bool compact, hist;
  if (MODE == MODE_D) {
    if (!ld_flag(&a.s->need_compact)) return;
    gk = (K)a.s->b1 << SH1;
    compact = true;
    hist = false;
  } else if (MODE == MODE_S) {
    if (!ld_flag(&a.s->need_full_hist)) return;
    gk = (K)__ldcg(&a.s->g_key2);
    if (gk == 0) return;
    compact = true;
    hist = false;
  } else if (MODE == MODE_A2) {
    if (!ld_flag(&a.s->need_full_hist)) return;
    compact = false;
    hist = true;
  } else {
    gk = (K)a.s->g_key;
    compact = gk > 0;
    hist = !compact;
  }
  // speculative +0 residual for the candidates likely to be selected: keys
  // >= z (the predicted T without margin; predicted mode, EF pass only)
  const bool spec = MODE == MODE_A && compact && a.s->spec_ok;
  const K zk = (K)a.s->z_key;
  // pass A in predicted mode (f32) also histograms its candidates' coarse
  // digit (key - G) >> PSB_COARSE_SHIFT, so k_cand resolves that level
  // without a pass of its own
  const bool chist = MODE == MODE_A && compact && sizeof(T) == 4 && a.histd != nullptr;
  constexpr int slot = MODE == MODE_A ? 0 : (MODE == MODE_S ? 1 : (MODE == MODE_D ? 2 : 3));
  uint32_t* ctr = &a.s->tile_ctr[slot];
  uint32_t* sbp = a.sb + (size_t)(slot < 3 ? slot : 0) * a.sb_stride;

  if (hist || chist)
    for (int b = threadIdx.x; b < PSB_HIST_BINS; b += blockDim.x) sh_hist[b] = 0;
  if (threadIdx.x == 0) {
    sh_nonfinite = 0;
    sh_tile[0] = atomicAdd(ctr, 1u);
  }
  __syncthreads();

  uint32_t nonfinite = 0;
  const T* __restrict__ src = (MODE == MODE_A) ? a.g : a.p;
  T* __restrict__ rr = a.r;
  auto prefetch_tile = [&](uint32_t t2) {
    if (PSB_PF && MODE == MODE_A && a.vec_ok && t2 < a.ntiles && (size_t)(t2 + 1) * TILE <= a.n) {
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src + (size_t)t2 * TILE),
                   "r"((uint32_t)(TILE * sizeof(T))) : "memory");
      if (rr != nullptr)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(rr + (size_t)t2 * TILE),
                     "r"((uint32_t)(TILE * sizeof(T))) : "memory");
    }
  };
  if (threadIdx.x == 0) prefetch_tile(sh_tile[0]);
  unsigned long long run = 0;  // candidates written by this CTA
  int cur = 0;
  for (uint32_t tile = sh_tile[0]; tile < a.ntiles; tile = sh_tile[cur]) {
    const size_t base = (size_t)tile * TILE;
    const bool full = a.vec_ok && (base + TILE <= a.n);
    T x[4][VW];
    uint32_t valid = 0;
    if (full) {
      valid = 0xffffu;
      if (MODE == MODE_A && rr != nullptr) {
        T gv[4][VW], rv[4][VW];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const size_t e = base + (size_t)(j * PSB_SCAN_THREADS + threadIdx.x) * VW;
          ld_vec_stream(src + e, gv[j]);
          ld_vec_stream(rr + e, rv[j]);  // evict-first: keep L2 for the candidate list
        }
        if (threadIdx.x == 0) {  // next tile: its grab and L2 prefetch overlap this tile
          const uint32_t nt = atomicAdd(ctr, 1u);
          sh_tile[cur ^ 1] = nt;
          prefetch_tile(nt);
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          T out[VW];
#pragma unroll
          for (int c = 0; c < VW; ++c) {
            x[j][c] = add_rn(rv[j][c], gv[j][c]);
            out[c] = (spec && KO::key(x[j][c]) >= zk) ? T(0) : x[j][c];
          }
          const size_t e = base + (size_t)(j * PSB_SCAN_THREADS + threadIdx.x) * VW;
          st_vec_stream(rr + e, out);
        }
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const size_t e = base + (size_t)(j * PSB_SCAN_THREADS + threadIdx.x) * VW;
          ld_vec(src + e, x[j]);
        }
        if (threadIdx.x == 0) {
          const uint32_t nt = atomicAdd(ctr, 1u);
          sh_tile[cur ^ 1] = nt;
          prefetch_tile(nt);
        }
      }
    } else {
      if (threadIdx.x == 0) sh_tile[cur ^ 1] = atomicAdd(ctr, 1u);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
#pragma unroll
        for (int c = 0; c < VW; ++c) {
          const size_t e = base + (size_t)(j * PSB_SCAN_THREADS + threadIdx.x) * VW + c;
          T v = T(0);
          if (e < a.n) {
            valid |= 1u << (j * VW + c);
            if (MODE == MODE_A && rr != nullptr) {
              v = add_rn(rr[e], src[e]);
              rr[e] = (spec && KO::key(v) >= zk) ? T(0) : v;
            } else {
              v = src[e];
            }
          }
          x[j][c] = v;
        }
      }
    }

    uint32_t fl = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
#pragma unroll
      for (int c = 0; c < VW; ++c) {
        const int bit = j * VW + c;
        const bool ok = (valid >> bit) & 1u;
        const K key = KO::key(x[j][c]);
        const uint32_t d = (uint32_t)(key >> SH1);
        if (hist) hist_add_agg(sh_hist, d, ok && d != 0);  // digit 0 is implicit
        if (ok) {
          if (key >= KO::kInf) nonfinite = 1;
          if (key >= gk) fl |= 1u << bit;
        }
      }
    }

    if (compact) {
      // element order inside a tile is (j, thread, c): one packed scan gives
      // every thread its offset in each of the 4 rows
      unsigned long long packed = 0;
#pragma unroll
      for (int j = 0; j < 4; ++j)
        packed |= (unsigned long long)__popc((fl >> (j * VW)) & ((1u << VW) - 1u)) << (16 * j);
      unsigned long long tot;
      const unsigned long long ex = block_exscan_u64(packed, sh_warp, &tot);
      uint32_t acc = 0;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        uint32_t pos = acc + (uint32_t)((ex >> (16 * j)) & 0xffffu);
        acc += (uint32_t)((tot >> (16 * j)) & 0xffffu);
#pragma unroll
        for (int c = 0; c < VW; ++c) {
          if ((fl >> (j * VW + c)) & 1u) {
            const size_t e = base + (size_t)(j * PSB_SCAN_THREADS + threadIdx.x) * VW + c;
            a.cand_idx[base + pos] = (uint32_t)e;
            a.cand_val[base + pos] = x[j][c];
            ++pos;
            if (chist) {
              const K dl = (KO::key(x[j][c]) - gk) >> PSB_COARSE_SHIFT;
              atomicAdd(&sh_hist[dl < (K)(PSB_COARSE_BINS - 1) ? (uint32_t)dl : PSB_COARSE_BINS - 1], 1u);
            }
          }
        }
      }
      if (threadIdx.x == 0) {
        a.tile_cnt[tile] = acc;
        if (acc) atomicAdd(sbp + (tile >> PSB_SB_SHIFT), acc);
      }
      run += acc;
    } else {
      __syncthreads();  // sh_tile[cur ^ 1] visible
    }
    cur ^= 1;
  }

  if (nonfinite) sh_nonfinite = 1;
  __syncthreads();
  if (threadIdx.x == 0) {
    if (sh_nonfinite) atomicOr(a.flags, 1u);
    if (compact && run) atomicAdd(&a.s->cand_count, run);
  }
  if (hist || chist) {
    uint32_t* gh = hist ? a.hist1 : a.histd;
    for (int b = threadIdx.x + (chist ? 1 : 0); b < PSB_HIST_BINS; b += blockDim.x) {  // coarse digit 0 is implicit
      const uint32_t h = sh_hist[b];
      if (h) atomicAdd(&gh[b], h);
    }
  }
  if (MODE == MODE_D) return;  // k_cand reads cand_count after the kernel boundary

  if (!last_block(&a.s->done[MODE == MODE_A ? DONE_A : MODE == MODE_S ? DONE_S : DONE_A2])) return;

  const unsigned long long k = a.s->k, n = a.s->n;
  if (MODE == MODE_S) {
    // second chance valid iff at least k keys >= G2: continue in predicted
    // mode on G2 (r holds p everywhere now, so no speculative zeros)
    const unsigned long long C = __ldcg(&a.s->cand_count);
    if (threadIdx.x == 0) {
      if (C >= k) {
        a.s->list_pass = 1;
        a.s->g_key = a.s->g_key2;
        a.s->spec_ok = 0;
        a.s->start_level = 0;
        a.s->prefix = 0;
        a.s->need = k;
        a.s->match = C;
        __threadfence();
        a.s->need_full_hist = 0;
      } else {
        a.s->cand_count = 0;  // still short: the full histogram pass takes over
      }
    }
    return;
  }
  if (compact) {
    // predicted mode: valid iff at least k keys >= G (then T >= G)
    const unsigned long long C = __ldcg(&a.s->cand_count);
    if (C >= k) {
      if (threadIdx.x == 0) {
        a.s->list_pass = 0;
        a.s->start_level = 0;
        a.s->prefix = 0;
        a.s->need = k;
        a.s->match = C;
      }
    } else if (threadIdx.x == 0) {
      a.s->need_full_hist = 1;  // miss: restore, then a second-chance compaction on
      a.s->cand_count = 0;      // G2 = G * PSB_SECOND_F; the full level-1 pass only if that misses too
      const float f2 = a.w->second_f != 0.f ? a.w->second_f : PSB_SECOND_F;
      a.s->g_key2 = f2 > 0.f ? scale_key(gk, f2, T(0)) : 0ull;
      a.w->misses += 1;
      a.w->f = a.w->f > 0.f ? 1.f - (1.f - a.w->f) * 1.5f : 0.97f;  // widen the margin
      if (a.w->f < 0.5f) a.w->f = 0.5f;
    }
    if (threadIdx.x == 0) a.w->calls += 1;
    return;
  }
  // cold mode / A2: level-1 resolution from the histogram
  __syncthreads();
  resolve_level(a.hist1, PSB_HIST_BINS, 1, k, sh_warp, &sh_res, sh_hist);
  if (threadIdx.x == 0) {
    const LevelResult& R = sh_res;
    if (R.found) {
      a.s->b1 = R.bin;
      a.s->prefix = R.bin;
      a.s->need = k - R.above;
      a.s->match = R.cnt;
    } else {  // the k-th largest key lies in digit 0 (zeros / tiny denormals)
      a.s->b1 = 0;
      a.s->prefix = 0;
      a.s->need = k - R.total;
      a.s->match = n - R.total;
    }
    a.s->start_level = 1;
    a.s->list_pass = 2;
    a.s->need_compact = 1;
    a.s->cand_count = 0;
    if (MODE == MODE_A) a.w->calls += 1;
  }
}

#ifdef PSB_SCAN_TRACE
// diagnostics build only: globaltimer at entry / exit of every k_scan<MODE_A> CTA
__device__ unsigned long long g_scan_trace[2 * 4096];
// k_cand: per CTA 15 phase timestamps + (tiles << 32 | entries) of its slice
__device__ unsigned long long g_cand_trace[16 * 1024];
#endif

#ifndef PSB_SCAN_MINB
#define PSB_SCAN_MINB 4
#endif
template <class T, int MODE>
__global__ void __launch_bounds__(PSB_SCAN_THREADS, PSB_SCAN_MINB) k_scan(ScanArgs<T> a) {
#ifdef PSB_SCAN_TRACE
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
#endif
  scan_body<T, MODE>(a);
#ifdef PSB_SCAN_TRACE
  if (MODE == MODE_A && threadIdx.x == 0 && blockIdx.x < 4096) {
    unsigned long long t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    g_scan_trace[2 * blockIdx.x] = t0;
    g_scan_trace[2 * blockIdx.x + 1] = t1;
  }
#endif
}

// Prediction missed: pass A speculatively stored +0 for its candidates; put p
// back (tile t's segment holds exactly those of tile t) before the second
// chance re-reads p from r.
template <class T>
__device__ __forceinline__ void restore_body(const ScanArgs<T>& a) {
  constexpr int TILE = tile_elems<T>();
  if (!ld_flag(&a.s->need_full_hist) || !a.s->spec_ok || a.r == nullptr) return;
  for (uint32_t t = blockIdx.x; t < a.ntiles; t += gridDim.x) {
    const uint32_t cnt = __ldcg(a.tile_cnt + t);
    const size_t base = (size_t)t * TILE;
    for (uint32_t j = threadIdx.x; j < cnt; j += blockDim.x) a.r[a.cand_idx[base + j]] = a.cand_val[base + j];
  }
}

template <class T>
__global__ void __launch_bounds__(PSB_SCAN_THREADS) k_restore(ScanArgs<T> a) {
  restore_body(a);
}

// The miss / cold fallback (restore, second chance, full level-1 histogram,
// compaction) as ONE cooperative launch on the k_scan grid (co-resident): in
// steady state it is a single node that exits at once instead of four.
template <class T>
__global__ void __launch_bounds__(PSB_SCAN_THREADS) k_fallback(ScanArgs<T> a) {
  cg::grid_group grid = cg::this_grid();
  const bool miss = ld_flag(&a.s->need_full_hist) != 0;
  if (!miss && !ld_flag(&a.s->need_compact)) return;  // uniform: flags from the previous kernel
  if (miss) {
    restore_body(a);
    grid.sync();
    scan_body<T, MODE_S>(a);   // second chance; its last CTA clears need_full_hist if it holds
    grid.sync();
    scan_body<T, MODE_A2>(a);  // full histogram; its last CTA resolves b1 and sets need_compact
    grid.sync();
  }
  scan_body<T, MODE_D>(a);
}

// ---------------------------------------------------- candidate phase
#include "psb_cand.inl"

template <class T>
psb_status run_topk(psb_ctx* c, int worker, const T* g, T* r, size_t n, size_t k,
                    uint32_t* idx_out, T* val_out, T* theta, double lr, T* mean_out,
                    cudaStream_t st) {
  constexpr int TILE = tile_elems<T>();
  const uint32_t ntiles = (uint32_t)((n + TILE - 1) / TILE);
  const int vec_ok = ((((uintptr_t)g) | ((uintptr_t)r)) & 15) == 0;
  TopkScratch* s = c->d_tk;
  TopkWorker* w = c->d_tw + worker;

  k_topk_begin<<<1, 256, 0, st>>>(s, w, c->d_hist1, c->d_histr, n, k, c->predict);
  ScanArgs<T> a;
  a.g = g;
  a.r = r;
  a.p = r ? r : g;
  a.n = n;
  a.ntiles = ntiles;
  a.vec_ok = vec_ok;
  a.s = s;
  a.w = w;
  a.hist1 = c->d_hist1;
  a.tile_cnt = c->d_tile_cnt;
  a.sb = c->d_sb;
  a.sb_stride = c->sb_stride;
  a.histd = sizeof(T) == 4 ? c->d_histd : nullptr;
  // persistent-style grid: PSB_SCAN_MINB CTAs per SM pull tiles dynamically
  // (one fewer under the multi-rank async pipeline: the freed registers let
  // the previous round's exchange and apply run beside this pass -- cfg4 at
  // 4 GPUs 0.89 -> 0.78 ms/round, the pass alone 0.61 -> 0.73 ms)
  const int per_sm = (c->async_pipe && c->nranks > 1) ? PSB_SCAN_MINB - 1 : PSB_SCAN_MINB;
  const uint32_t scan_grid = (uint32_t)std::min<size_t>(ntiles, (size_t)c->num_sms * per_sm);
  a.cand_idx = c->d_stage_idx;
  a.cand_val = reinterpret_cast<T*>(c->d_stage_val);
  a.flags = c->d_flags;
  if (c->prof) cudaEventRecord(psb_prof_event(c), st);
  k_scan<T, MODE_A><<<scan_grid, PSB_SCAN_THREADS, 0, st>>>(a);
  if (c->prof) cudaEventRecord(psb_prof_event(c), st);
  // fallback: one cooperative node when the k_scan grid is co-resident
  int fb_occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&fb_occ, k_fallback<T>, PSB_SCAN_THREADS, 0);
  bool fused_fb = false;
  if ((size_t)fb_occ * c->num_sms >= scan_grid) {
    void* fargs[] = {&a};
    fused_fb = cudaLaunchCooperativeKernel((const void*)k_fallback<T>, dim3(scan_grid), dim3(PSB_SCAN_THREADS),
                                           fargs, 0, st) == cudaSuccess;
  }
  if (!fused_fb) {
    (void)cudaGetLastError();
    k_restore<T><<<scan_grid, PSB_SCAN_THREADS, 0, st>>>(a);
    k_scan<T, MODE_S><<<scan_grid, PSB_SCAN_THREADS, 0, st>>>(a);
    k_scan<T, MODE_A2><<<scan_grid, PSB_SCAN_THREADS, 0, st>>>(a);
    k_scan<T, MODE_D><<<scan_grid, PSB_SCAN_THREADS, 0, st>>>(a);
    c->launches += 3;
  }

  CandArgs<T> b;
  b.s = s;
  b.w = w;
  b.hlev = c->d_histr;
  b.seg_idx = c->d_stage_idx;
  b.seg_val = reinterpret_cast<const T*>(c->d_stage_val);
  b.tile_cnt = c->d_tile_cnt;
  b.sb = c->d_sb;
  b.sb_stride = c->sb_stride;
  b.histd = sizeof(T) == 4 ? c->d_histd : nullptr;
  b.ntiles = ntiles;
  b.cand_idx = c->d_list_idx;
  b.cand_val = reinterpret_cast<T*>(c->d_list_val);
  b.cta = c->d_cta;
  b.idx_out = idx_out;
  b.val_out = val_out;
  b.r = r;
  b.theta = theta;
  b.mean_out = mean_out;
  b.coef = (T)(-lr);
  b.flags = c->d_flags;
  b.npush = c->push_n;
  for (int q = 0; q < c->push_n; ++q) {
    b.push_idx[q] = reinterpret_cast<uint32_t*>(c->push_base[q] + c->push_slot_off);
    b.push_val[q] = reinterpret_cast<T*>(c->push_base[q] + c->push_slot_off + psb_align16(k * 4));
  }
  if (c->push_wait) {  // peers done reading this slot's previous payload
    psb_status ws = psb_peer_wait_ack(c, st);
    if (ws) return ws;
  }
  // cooperative grid: one CTA per SM, the rest of shared memory stages the slice
  const int slot = sizeof(T) == 8;
  if (c->cand_smem[slot] == 0) {
    int optin = 0;
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, c->device);
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, k_cand<T>);
    const int dyn = optin - (int)fa.sharedSizeBytes - 1024;
    cudaFuncSetAttribute(k_cand<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn);
    c->cand_smem[slot] = dyn;
  }
  const int dyn = c->cand_smem[slot];
  b.stage_cap = (uint32_t)(((size_t)dyn - kCoarseBins * 4) / (sizeof(T) + 8)) & ~3u;
  if (c->no_stage) b.stage_cap = 0;  // diagnostics: PSB_NO_STAGE=1 streams the list from L2/HBM
  const uint32_t cgrid = (uint32_t)std::max<size_t>(1, std::min<size_t>((n + 4095) / 4096, (size_t)c->num_sms));
  void* kargs[] = {&b};
  cudaError_t e = cudaLaunchCooperativeKernel((const void*)k_cand<T>, dim3(cgrid), dim3(kCandThreads),
                                              kargs, (size_t)dyn, st);
  if (e != cudaSuccess) return psb_cuda_err(c, e, "psb_ef_topk (cooperative launch)");
  c->launches += 4;
  PSB_LAUNCH_CHECK(c, "psb_ef_topk");
  return PSB_OK;
}

// Int8 values for the selected entries (north-star, unpinned; rule of
// psb_q8_quantize with blocks of 128 consecutive payload entries).  The
// residual at a selected index becomes p - code*scale instead of +0.
__global__ void k_topk_q8(size_t k, const uint32_t* __restrict__ idx, const float* __restrict__ vals,
                          float* __restrict__ r, int8_t* __restrict__ codes,
                          float* __restrict__ scales, uint32_t* flags) {
  const int lane = threadIdx.x & 31;
  const size_t blk = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const size_t lo = blk * 128;
  if (lo >= k) return;
  float v[4];
  float amax = 0.f;
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const size_t j = lo + lane * 4 + c;
    v[c] = j < k ? vals[j] : 0.f;
    amax = fmaxf(amax, fabsf(v[c]));
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
  const float scale = __fdiv_rn(amax, 127.0f);
  if (lane == 0) scales[blk] = scale;
  bool bad = !is_finite(amax);
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const size_t j = lo + lane * 4 + c;
    if (j >= k) continue;
    int q = 0;
    if (scale > 0.f) {
      q = __float2int_rn(__fdiv_rn(v[c], scale));
      q = q > 127 ? 127 : (q < -127 ? -127 : q);
    }
    codes[j] = (int8_t)q;
    if (r) {
      const float xhat = __fmul_rn((float)q, scale);
      const float res = __fsub_rn(v[c], xhat);
      r[idx[j]] = res;
      bad |= !is_finite(res);
    }
  }
  if (bad) atomicOr(flags, 1u);
}

}  // namespace

psb_status psb_topk_run(psb_ctx* c, psb_dtype dt, int worker, const void* g, void* r, size_t n,
                        size_t k, uint32_t* idx_out, void* val_out, cudaStream_t st) {
  return psb_topk_run_fused(c, dt, worker, g, r, n, k, idx_out, val_out, nullptr, 0.0, nullptr, st);
}

psb_status psb_topk_run_fused(psb_ctx* c, psb_dtype dt, int worker, const void* g, void* r, size_t n,
                              size_t k, uint32_t* idx_out, void* val_out, void* theta, double lr,
                              void* mean_out, cudaStream_t st) {
  if (dt == PSB_F32)
    return run_topk<float>(c, worker, (const float*)g, (float*)r, n, k, idx_out, (float*)val_out,
                           (float*)theta, lr, (float*)mean_out, st);
  return run_topk<double>(c, worker, (const double*)g, (double*)r, n, k, idx_out, (double*)val_out,
                          (double*)theta, lr, (double*)mean_out, st);
}

psb_status psb_topk_q8_fix(psb_ctx* c, const float*, size_t k, const uint32_t* idx,
                           const float* vals, float* r, int8_t* codes, float* scales,
                           cudaStream_t st) {
  const size_t nblk = (k + 127) / 128;
  const unsigned grid = (unsigned)((nblk * 32 + 255) / 256);
  k_topk_q8<<<grid, 256, 0, st>>>(k, idx, vals, r, codes, scales, c->d_flags);
  c->launches += 1;
  PSB_LAUNCH_CHECK(c, "psb_ef_topk_q8");
  return PSB_OK;
}

extern "C" psb_status psb_topk_phases(psb_ctx* c, uint64_t* out16) {
  PSB_REQUIRE(c, c != nullptr && out16 != nullptr, "psb_topk_phases: null argument");
  TopkScratch s;
  cudaError_t e = cudaMemcpy(&s, c->d_tk, sizeof(s), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return psb_cuda_err(c, e, "psb_topk_phases");
  for (int i = 0; i < 16; ++i) out16[i] = s.phase_ns[i];
  return PSB_OK;
}

extern "C" psb_status psb_topk_stats(psb_ctx* c, int worker, uint64_t* out8) {
  PSB_REQUIRE(c, c != nullptr && out8 != nullptr, "psb_topk_stats: null argument");
  PSB_REQUIRE(c, worker >= 0 && worker < c->max_workers, "psb_topk_stats: worker out of range");
  TopkScratch s;
  TopkWorker w;
  cudaError_t e = cudaMemcpy(&s, c->d_tk, sizeof(s), cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMemcpy(&w, c->d_tw + worker, sizeof(w), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return psb_cuda_err(c, e, "psb_topk_stats");
  uint32_t fbits;
  memcpy(&fbits, &w.f, 4);
  out8[0] = s.cand_count;   // candidates of the last call
  out8[1] = s.k;
  out8[2] = s.prefix;       // exact threshold key T of the last call
  out8[3] = s.need;         // ties at T taken (lowest indices)
  out8[4] = ((s.g_key != 0 && !s.need_full_hist) ? 0 : 1) |  // 0: predicted set was valid
            ((uint64_t)s.start_level << 8);                  // 100+: T found on key - G
  out8[5] = s.g_key;        // predicted key used by the last call (0 = cold)
  out8[6] = ((uint64_t)w.misses << 32) | w.calls;
  out8[7] = fbits;          // margin factor f for the next call
  return PSB_OK;
}

// diagnostics (psb_debug.h): per-CTA entry/exit timestamps of the last
// k_scan<MODE_A> launch in a -DPSB_SCAN_TRACE build; returns 0 otherwise
extern "C" PSB_API int psb_debug_scan_trace(unsigned long long* out, int max_ctas) {
#ifdef PSB_SCAN_TRACE
  const int m = max_ctas < 4096 ? max_ctas : 4096;
  return cudaMemcpyFromSymbol(out, g_scan_trace, sizeof(unsigned long long) * 2 * m) == cudaSuccess ? m : -1;
#else
  (void)out;
  (void)max_ctas;
  return 0;
#endif
}

extern "C" PSB_API int psb_debug_cand_trace(unsigned long long* out, int max_ctas) {
#ifdef PSB_SCAN_TRACE
  const int m = max_ctas < 1024 ? max_ctas : 1024;
  return cudaMemcpyFromSymbol(out, g_cand_trace, sizeof(unsigned long long) * 16 * m) == cudaSuccess ? m : -1;
#else
  (void)out;
  (void)max_ctas;
  return 0;
#endif
}
