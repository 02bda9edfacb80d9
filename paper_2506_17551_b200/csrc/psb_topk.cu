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
//   k_topk_begin   1 CTA: reset per-call scratch, zero histograms.
//   k_scan<A>      THE streaming pass (12N bytes: read g, read r, write p->r).
//                  Predicted mode (the worker's previous call left a key
//                  threshold G = key(T_prev * f)): index-ordered compaction of
//                  every element with key >= G -- CTA b streams a contiguous
//                  index range and appends to its own segment (block scan per
//                  tile, no cross-CTA waits, no histogram atomics).  The last
//                  CTA validates the prediction (count >= k) and prefix-sums
//                  the segment sizes into one logical index-ordered list.
//                  Cold mode (no prediction): level-1 histogram of key>>19 in
//                  shared memory; the last CTA resolves digit b1 of the k-th key.
//   k_scan<A2>     only if the prediction missed: full histogram pass (reads p).
//   k_scan<D>      only in cold/miss mode: compaction of digit >= b1.
//   k_refine<L>    radix levels over the candidate list (all levels in
//                  predicted mode, levels 2.. in cold mode).
//   k_final_count  per-CTA (gt, eq) counts vs the exact threshold key T; the
//                  last CTA scans the CTA totals and predicts the next G.
//   k_final_write  one packed (gt, eq) block scan per 1024 candidates gives each
//                  element's output slot gt_before + min(eq_before, need_eq);
//                  writes idx/val, r[idx] = +0 and, for a single worker, the
//                  fused SGD update of theta[idx] (no separate apply pass).
// Every kernel is launched unconditionally and exits early from device-side
// flags, so the sequence is CUDA-graph capturable and never syncs the host.
// Results never depend on the prediction: a miss only costs the fallback.
#include "psb_internal.cuh"

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

enum { MODE_A = 0, MODE_A2 = 1, MODE_D = 2 };
enum { DONE_A = 0, DONE_A2 = 1, DONE_R = 2, DONE_F = 3, DONE_D = 4 };

// key <-> magnitude value, for the predicted threshold key(T * f)
__device__ __forceinline__ unsigned long long scale_key(unsigned long long key, float f, float) {
  return (unsigned long long)__float_as_uint(__fmul_rn(__uint_as_float((uint32_t)key), f));
}
__device__ __forceinline__ unsigned long long scale_key(unsigned long long key, float f, double) {
  return (unsigned long long)__double_as_longlong(__dmul_rn(__longlong_as_double((long long)key), (double)f));
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
  uint32_t tpc;       // tiles per CTA: CTA b streams tiles [b*tpc, (b+1)*tpc)
  uint32_t* seg_cnt;  // candidates written by CTA b (segment b of the list)
  uint32_t* seg_pre;  // exclusive prefix of seg_cnt (nseg + 1 entries)
  uint32_t* cand_idx;
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

// Resolve one radix level from a histogram (run by one whole CTA of
// PSB_SCAN_THREADS threads).  Bins [max(lo,1), nbins) hold exact counts.
// Finds the bin b containing the need-th largest entry (found, bin, above =
// count in bins > b, cnt = h[b]).
struct LevelResult {
  int found;
  uint32_t bin;
  unsigned long long above;
  unsigned long long cnt;
  unsigned long long total;  // sum over bins >= max(lo,1)
};

// `sh` is a shared-memory staging area of >= nbins words: the histogram is
// copied in with coalesced, independent loads, then scanned in shared memory.
__device__ void resolve_level(const uint32_t* hist, uint32_t nbins, uint32_t lo,
                              unsigned long long need, unsigned long long* sh_warp,
                              LevelResult* out, uint32_t* sh) {
  const uint32_t t = threadIdx.x;
  for (uint32_t b = t; b < nbins; b += PSB_SCAN_THREADS)
    sh[b] = (b >= lo && b >= 1) ? __ldcg(hist + b) : 0u;
  if (t == 0) out->found = 0;
  __syncthreads();
  const uint32_t B = nbins >= PSB_SCAN_THREADS ? nbins / PSB_SCAN_THREADS : 1;
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

__device__ __forceinline__ bool last_block(uint32_t* counter) {
  __shared__ int am_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) am_last = atomicAdd(counter, 1u) == gridDim.x - 1;
  __syncthreads();
  if (am_last) __threadfence();
  return am_last;
}

// Exclusive prefix of the per-CTA segment counts (run by one whole CTA);
// pre[nseg] = total.  `sh` must hold >= nseg words.
__device__ void seg_prefix(const uint32_t* cnt, uint32_t nseg, uint32_t* pre, uint32_t* sh,
                           unsigned long long* sh_warp) {
  __syncthreads();
  for (uint32_t b = threadIdx.x; b < nseg; b += blockDim.x) sh[b] = __ldcg(cnt + b);
  __syncthreads();
  const uint32_t q = (nseg + PSB_SCAN_THREADS - 1) / PSB_SCAN_THREADS;
  const uint32_t b0 = threadIdx.x * q, b1 = min(nseg, b0 + q);
  unsigned long long local = 0;
  for (uint32_t b = b0; b < b1; ++b) local += sh[b];
  unsigned long long total;
  unsigned long long run = block_exscan_u64(local, sh_warp, &total);
  for (uint32_t b = b0; b < b1; ++b) {
    pre[b] = (uint32_t)run;
    run += sh[b];
  }
  if (threadIdx.x == 0) pre[nseg] = (uint32_t)total;
}

__global__ void k_topk_begin(TopkScratch* s, TopkWorker* w, uint32_t* hist1, uint32_t* histr,
                             unsigned long long n, unsigned long long k, int predict) {
  for (int b = threadIdx.x; b < PSB_HIST_BINS; b += blockDim.x) {
    hist1[b] = 0;
    histr[b] = 0;
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < 8; ++i) s->done[i] = 0;
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
  }
}

// ------------------------------------------------------------------ scan
template <class T, int MODE>
__global__ void __launch_bounds__(PSB_SCAN_THREADS) k_scan(ScanArgs<T> a) {
  typedef KeyOf<T> KO;
  typedef typename KO::K K;
  constexpr int VW = VecOf<T>::W;
  constexpr int TILE = tile_elems<T>();
  constexpr int SH1 = KO::shift(0);

  __shared__ uint32_t sh_hist[PSB_HIST_BINS];
  __shared__ unsigned long long sh_warp[32];
  __shared__ uint32_t sh_nonfinite;
  __shared__ LevelResult sh_res;

  // compact: keep key >= gk.  hist: level-1 histogram of every element.
  K gk = 0;
  bool compact, hist;
  if (MODE == MODE_D) {
    if (!a.s->need_compact) return;
    gk = (K)a.s->b1 << SH1;
    compact = true;
    hist = false;
  } else if (MODE == MODE_A2) {
    if (!a.s->need_full_hist) return;
    compact = false;
    hist = true;
  } else {
    gk = (K)a.s->g_key;
    compact = gk > 0;
    hist = !compact;
  }

  if (hist)
    for (int b = threadIdx.x; b < PSB_HIST_BINS; b += blockDim.x) sh_hist[b] = 0;
  if (threadIdx.x == 0) sh_nonfinite = 0;
  __syncthreads();

  uint32_t nonfinite = 0;
  const T* __restrict__ src = (MODE == MODE_A) ? a.g : a.p;
  T* __restrict__ rr = a.r;

  // CTA b streams a contiguous tile range in index order and appends its
  // candidates to its own segment (capacity = its element count).
  const uint32_t t_lo = blockIdx.x * a.tpc;
  const uint32_t t_hi = min(a.ntiles, t_lo + a.tpc);
  const size_t seg_base = (size_t)t_lo * TILE;
  uint32_t run = 0;  // candidates appended so far (uniform across the CTA)
  for (uint32_t tile = t_lo; tile < t_hi; ++tile) {
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
          ld_vec(rr + e, rv[j]);
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
#pragma unroll
          for (int c = 0; c < VW; ++c) x[j][c] = add_rn(rv[j][c], gv[j][c]);
          const size_t e = base + (size_t)(j * PSB_SCAN_THREADS + threadIdx.x) * VW;
          st_vec(rr + e, x[j]);
        }
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const size_t e = base + (size_t)(j * PSB_SCAN_THREADS + threadIdx.x) * VW;
          ld_vec(src + e, x[j]);
        }
      }
    } else {
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
              rr[e] = v;
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
        if ((valid >> bit) & 1u) {
          const K key = KO::key(x[j][c]);
          if (key >= KO::kInf) nonfinite = 1;
          if (hist) {
            const uint32_t d = (uint32_t)(key >> SH1);
            if (d) atomicAdd(&sh_hist[d], 1u);
          }
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
      uint32_t acc = run;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        uint32_t pos = acc + (uint32_t)((ex >> (16 * j)) & 0xffffu);
        acc += (uint32_t)((tot >> (16 * j)) & 0xffffu);
#pragma unroll
        for (int c = 0; c < VW; ++c) {
          if ((fl >> (j * VW + c)) & 1u) {
            const size_t e = base + (size_t)(j * PSB_SCAN_THREADS + threadIdx.x) * VW + c;
            a.cand_idx[seg_base + pos] = (uint32_t)e;
            a.cand_val[seg_base + pos] = x[j][c];
            ++pos;
          }
        }
      }
      run = acc;
    }
  }

  if (nonfinite) sh_nonfinite = 1;
  __syncthreads();
  if (threadIdx.x == 0) {
    if (sh_nonfinite) atomicOr(a.flags, 1u);
    if (compact) {
      a.seg_cnt[blockIdx.x] = run;
      if (run) atomicAdd(&a.s->cand_count, (unsigned long long)run);
    }
  }
  if (hist) {
    for (int b = threadIdx.x; b < PSB_HIST_BINS; b += blockDim.x) {
      const uint32_t h = sh_hist[b];
      if (h) atomicAdd(&a.hist1[b], h);
    }
  }
  if (MODE == MODE_D) {
    if (last_block(&a.s->done[DONE_D])) seg_prefix(a.seg_cnt, gridDim.x, a.seg_pre, sh_hist, sh_warp);
    return;
  }

  if (!last_block(&a.s->done[MODE == MODE_A ? DONE_A : DONE_A2])) return;

  const unsigned long long k = a.s->k, n = a.s->n;
  if (compact) {
    // predicted mode: valid iff at least k keys >= G (then T >= G)
    const unsigned long long C = __ldcg(&a.s->cand_count);
    if (C >= k) {
      if (threadIdx.x == 0) {
        a.s->start_level = 0;
        a.s->prefix = 0;
        a.s->need = k;
        a.s->match = C;
      }
      seg_prefix(a.seg_cnt, gridDim.x, a.seg_pre, sh_hist, sh_warp);
    } else if (threadIdx.x == 0) {
      a.s->need_full_hist = 1;  // miss: rerun level 1 on all of p, then compact
      a.s->cand_count = 0;
      a.w->misses += 1;
      a.w->f = a.w->f > 0.f ? 1.f - (1.f - a.w->f) * 2.f : 0.98f;  // widen the margin
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
    a.s->need_compact = 1;
    a.s->cand_count = 0;
    if (MODE == MODE_A) a.w->calls += 1;
  }
}

// ---------------------------------------------------- candidate list
template <class T>
struct CandArgs {
  TopkScratch* s;
  TopkWorker* w;
  uint32_t* histr;
  const uint32_t* cand_idx;
  const T* cand_val;
  const uint32_t* seg_pre;  // nseg + 1 exclusive prefixes of the k_scan CTA segments
  uint32_t nseg;
  size_t seg_cap;           // segment stride (= elements streamed by one k_scan CTA)
  unsigned long long* cta;  // per-CTA (gt | eq << 32) totals, then exclusive prefixes
  uint32_t* idx_out;
  T* val_out;
  T* r;
  T* theta;     // fused single-worker SGD update (nullable)
  T* mean_out;  // with theta: dense mean at touched indices (nullable)
  T coef;       // (T)(-lr)
  uint32_t* flags;
};

// Flat view of the segmented candidate list: logical entry e (index order)
// lies in segment s with pre[s] <= e < pre[s+1], physically at
// s*cap + (e - pre[s]).  Work is split evenly over the logical range, so the
// candidate phase is balanced whatever the data's spatial distribution.
struct FlatMap {
  const uint32_t* pre;  // shared-memory copy
  uint32_t nseg;
  size_t cap;
  __device__ __forceinline__ uint32_t seg_of(uint32_t e) const {
    uint32_t lo = 0, hi = nseg;  // pre[lo] <= e < pre[hi]
    while (hi - lo > 1) {
      const uint32_t mid = (lo + hi) >> 1;
      if (pre[mid] <= e) lo = mid;
      else hi = mid;
    }
    return lo;
  }
};

// Loads the segment prefixes into shared memory and returns this CTA's
// logical range (chunks are multiples of 1024 entries).
template <class T>
__device__ __forceinline__ FlatMap flat_begin(const CandArgs<T>& a, uint32_t* sh_pre, uint32_t* lo,
                                              uint32_t* hi) {
  for (uint32_t b = threadIdx.x; b <= a.nseg; b += blockDim.x) sh_pre[b] = a.seg_pre[b];
  __syncthreads();
  const uint32_t C = sh_pre[a.nseg];
  uint32_t chunk = (C + gridDim.x - 1) / gridDim.x;
  chunk = (chunk + 1023u) & ~1023u;
  *lo = min(C, blockIdx.x * chunk);
  *hi = min(C, *lo + chunk);
  FlatMap m;
  m.pre = sh_pre;
  m.nseg = a.nseg;
  m.cap = a.seg_cap;
  return m;
}

// Physical positions of the 4 consecutive logical entries e0..e0+3 (< hi).
__device__ __forceinline__ void flat_pos4(const FlatMap& m, uint32_t e0, uint32_t hi, size_t (&pos)[4]) {
  uint32_t sg = e0 < hi ? m.seg_of(e0) : 0;
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const uint32_t e = e0 + c;
    pos[c] = 0;
    if (e < hi) {
      while (m.pre[sg + 1] <= e) ++sg;
      pos[c] = (size_t)sg * m.cap + (e - m.pre[sg]);
    }
  }
}

template <class T>
__global__ void __launch_bounds__(PSB_SCAN_THREADS) k_refine(CandArgs<T> a, int level) {
  typedef KeyOf<T> KO;
  typedef typename KO::K K;
  __shared__ uint32_t sh_hist[PSB_HIST_BINS];
  __shared__ uint32_t sh_pre[PSB_FINAL_TPC_MAX + 1];
  __shared__ unsigned long long sh_warp[32];
  __shared__ LevelResult sh_res;

  if ((uint32_t)level < a.s->start_level) return;  // resolved by the streaming pass
  const int pshift = level ? KO::shift(level - 1) : (int)(sizeof(K) * 8 - 1);
  const int shift = KO::shift(level);
  const uint32_t nbins = 1u << KO::width(level);
  const K prefix = (K)a.s->prefix;

  for (uint32_t b = threadIdx.x; b < nbins; b += blockDim.x) sh_hist[b] = 0;
  uint32_t lo, hi;
  const FlatMap m = flat_begin(a, sh_pre, &lo, &hi);
  for (uint32_t e0 = lo + 4 * threadIdx.x; e0 < hi; e0 += 4 * PSB_SCAN_THREADS) {
    size_t pos[4];
    flat_pos4(m, e0, hi, pos);
    T v[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) v[c] = e0 + c < hi ? a.cand_val[pos[c]] : T(0);
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const K key = KO::key(v[c]);
      if (e0 + c < hi && (key >> pshift) == prefix) {
        const uint32_t d = (uint32_t)(key >> shift) & (nbins - 1);
        if (d) atomicAdd(&sh_hist[d], 1u);
      }
    }
  }
  __syncthreads();
  for (uint32_t b = threadIdx.x; b < nbins; b += blockDim.x) {
    const uint32_t h = sh_hist[b];
    if (h) atomicAdd(&a.histr[b], h);
  }
  if (!last_block(&a.s->done[DONE_R])) return;

  const unsigned long long need = a.s->need, match = a.s->match;
  __syncthreads();
  resolve_level(a.histr, nbins, 1, need, sh_warp, &sh_res, sh_hist);
  if (threadIdx.x == 0) {
    const LevelResult& R = sh_res;
    uint32_t bin;
    unsigned long long above, cnt;
    if (R.found) {
      bin = R.bin;
      above = R.above;
      cnt = R.cnt;
    } else {
      bin = 0;
      above = R.total;
      cnt = match - R.total;
    }
    a.s->prefix = level ? ((a.s->prefix << KO::width(level)) | bin) : bin;
    a.s->need = need - above;
    a.s->match = cnt;
    a.s->done[DONE_R] = 0;  // next level reuses the counter (stream-ordered)
  }
  __syncthreads();
  for (uint32_t b = threadIdx.x; b < nbins; b += blockDim.x) a.histr[b] = 0;
}

// Counts (key > T, key == T) per CTA chunk; the last CTA turns the totals
// into exclusive prefixes (packed gt | eq << 32; each field < 2^32) -- offsets
// depend only on counts, so the output order is deterministic -- and sets the
// worker's next predicted threshold G = key(T * f), adapting f so the next
// candidate set stays between ~1.1k and ~2k.
template <class T>
__global__ void __launch_bounds__(PSB_SCAN_THREADS) k_final_count(CandArgs<T> a) {
  typedef KeyOf<T> KO;
  typedef typename KO::K K;
  __shared__ unsigned long long sh_c[PSB_FINAL_TPC_MAX];
  __shared__ uint32_t sh_pre[PSB_FINAL_TPC_MAX + 1];
  __shared__ unsigned long long sh_warp[32];
  const K T_key = (K)a.s->prefix;
  uint32_t lo, hi;
  const FlatMap m = flat_begin(a, sh_pre, &lo, &hi);
  uint32_t gt = 0, eq = 0;
  for (uint32_t e0 = lo + 4 * threadIdx.x; e0 < hi; e0 += 4 * PSB_SCAN_THREADS) {
    size_t pos[4];
    flat_pos4(m, e0, hi, pos);
    T v[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) v[c] = e0 + c < hi ? a.cand_val[pos[c]] : T(0);
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const K key = KO::key(v[c]);
      const bool ok = e0 + c < hi;
      gt += ok && key > T_key;
      eq += ok && key == T_key;
    }
  }
  unsigned long long total;
  block_exscan_u64((unsigned long long)gt | ((unsigned long long)eq << 32), sh_warp, &total);
  if (threadIdx.x == 0) a.cta[blockIdx.x] = total;
  if (!last_block(&a.s->done[DONE_F])) return;
  for (uint32_t b = threadIdx.x; b < gridDim.x; b += blockDim.x) sh_c[b] = __ldcg(a.cta + b);
  __syncthreads();
  const uint32_t qb = (gridDim.x + PSB_SCAN_THREADS - 1) / PSB_SCAN_THREADS;
  const uint32_t b0 = threadIdx.x * qb, b1 = min(gridDim.x, b0 + qb);
  unsigned long long local = 0;
  for (uint32_t b = b0; b < b1; ++b) local += sh_c[b];
  unsigned long long run = block_exscan_u64(local, sh_warp, &total);
  for (uint32_t b = b0; b < b1; ++b) {
    const unsigned long long c = sh_c[b];
    a.cta[b] = run;
    run += c;
  }
  if (threadIdx.x == 0) {
    // next call's prediction; candidates this call = a.s->cand_count
    float f = a.w->f > 0.f ? a.w->f : 0.98f;
    const double ratio = (double)__ldcg(&a.s->cand_count) / (double)a.s->k;
    if (a.s->start_level == 0) {            // this call was predicted (and valid)
      if (ratio > 2.0) f = 1.f - (1.f - f) * 0.5f;        // too many candidates: tighten
      else if (ratio < 1.1) f = 1.f - (1.f - f) * 1.5f;   // thin margin: widen
    }
    f = fminf(fmaxf(f, 0.5f), 0.9995f);
    a.w->f = f;
    a.w->g_key = (T_key == 0 || T_key >= KO::kInf) ? 0ull : scale_key(T_key, f, T(0));
  }
}

// One packed (gt, eq) block scan per 1024 candidates: element e is selected
// iff key > T or (key == T and eq_before(e) < need_eq), and lands at slot
// gt_before(e) + min(eq_before(e), need_eq) -- index order preserved.
template <class T>
__global__ void __launch_bounds__(PSB_SCAN_THREADS) k_final_write(CandArgs<T> a) {
  typedef KeyOf<T> KO;
  typedef typename KO::K K;
  __shared__ uint32_t sh_pre[PSB_FINAL_TPC_MAX + 1];
  __shared__ unsigned long long sh_warp[32];
  __shared__ uint32_t sh_bad;
  const K T_key = (K)a.s->prefix;
  const unsigned long long need_eq = a.s->need;
  if (threadIdx.x == 0) sh_bad = 0;
  uint32_t lo, hi;
  const FlatMap m = flat_begin(a, sh_pre, &lo, &hi);
  unsigned long long run = a.cta[blockIdx.x];  // (gt | eq << 32) before this chunk
  bool bad = false;
  for (uint32_t base = lo; base < hi; base += 4 * PSB_SCAN_THREADS) {
    const uint32_t e0 = base + 4 * threadIdx.x;
    size_t pos[4];
    flat_pos4(m, e0, hi, pos);
    T v[4];
    uint32_t id[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      v[c] = e0 + c < hi ? a.cand_val[pos[c]] : T(0);
      id[c] = e0 + c < hi ? a.cand_idx[pos[c]] : 0u;
    }
    uint32_t gtm = 0, eqm = 0;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      if (e0 + c < hi) {
        const K key = KO::key(v[c]);
        gtm |= (key > T_key ? 1u : 0u) << c;
        eqm |= (key == T_key ? 1u : 0u) << c;
      }
    }
    const unsigned long long mine = (unsigned long long)__popc(gtm) | ((unsigned long long)__popc(eqm) << 32);
    unsigned long long tot;
    unsigned long long before = run + block_exscan_u64(mine, sh_warp, &tot);
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const unsigned long long gt_b = before & 0xffffffffull, eq_b = before >> 32;
      const bool gt = (gtm >> c) & 1u, eq = (eqm >> c) & 1u;
      if (gt || (eq && eq_b < need_eq)) {
        const unsigned long long slot = gt_b + (eq_b < need_eq ? eq_b : need_eq);
        const uint32_t i = id[c];
        a.idx_out[slot] = i;
        a.val_out[slot] = v[c];
        if (a.r) a.r[i] = T(0);
        if (a.theta) {
          const T mean = mul_rn(v[c], T(1));  // P = 1: mean = v * (1/1)
          const T th = add_rn(mul_rn(a.coef, mean), a.theta[i]);
          a.theta[i] = th;
          if (a.mean_out) a.mean_out[i] = mean;
          bad |= !is_finite(th);
        }
      }
      before += (unsigned long long)gt | ((unsigned long long)eq << 32);
    }
    run += tot;
  }
  if (bad) sh_bad = 1;
  __syncthreads();
  if (threadIdx.x == 0 && sh_bad) atomicOr(a.flags, 1u);
}

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
  const uint32_t scan_grid0 = (uint32_t)std::min<size_t>(ntiles, (size_t)c->num_sms * 4);
  a.tpc = (ntiles + scan_grid0 - 1) / scan_grid0;
  const uint32_t scan_grid = (ntiles + a.tpc - 1) / a.tpc;
  a.seg_cnt = c->d_seg_cnt;
  a.seg_pre = c->d_seg_pre;
  a.cand_idx = c->d_stage_idx;
  a.cand_val = reinterpret_cast<T*>(c->d_stage_val);
  a.flags = c->d_flags;
  if (c->prof) cudaEventRecord(psb_prof_event(c), st);
  k_scan<T, MODE_A><<<scan_grid, PSB_SCAN_THREADS, 0, st>>>(a);
  if (c->prof) cudaEventRecord(psb_prof_event(c), st);
  k_scan<T, MODE_A2><<<scan_grid, PSB_SCAN_THREADS, 0, st>>>(a);
  k_scan<T, MODE_D><<<scan_grid, PSB_SCAN_THREADS, 0, st>>>(a);

  CandArgs<T> b;
  b.s = s;
  b.w = w;
  b.histr = c->d_histr;
  b.cand_idx = c->d_stage_idx;
  b.cand_val = reinterpret_cast<const T*>(c->d_stage_val);
  b.seg_pre = c->d_seg_pre;
  b.nseg = scan_grid;
  b.seg_cap = (size_t)a.tpc * TILE;
  b.cta = c->d_cta;
  b.idx_out = idx_out;
  b.val_out = val_out;
  b.r = r;
  b.theta = theta;
  b.mean_out = mean_out;
  b.coef = (T)(-lr);
  b.flags = c->d_flags;
  const uint32_t cgrid = (uint32_t)std::max<size_t>(1, std::min<size_t>((n + 4095) / 4096, (size_t)c->num_sms * 4));
  for (int level = 0; level < KeyOf<T>::kLevels; ++level)
    k_refine<T><<<cgrid, PSB_SCAN_THREADS, 0, st>>>(b, level);
  k_final_count<T><<<cgrid, PSB_SCAN_THREADS, 0, st>>>(b);
  k_final_write<T><<<cgrid, PSB_SCAN_THREADS, 0, st>>>(b);
  c->launches += 6 + KeyOf<T>::kLevels;
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
  out8[4] = s.start_level;  // 0: predicted candidate set was valid
  out8[5] = s.g_key;        // predicted key used by the last call (0 = cold)
  out8[6] = ((uint64_t)w.misses << 32) | w.calls;
  out8[7] = fbits;          // margin factor f for the next call
  return PSB_OK;
}
