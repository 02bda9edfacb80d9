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
// B200 design: the selection is a radix select on the
// magnitude key bits(|p|) (monotone for finite values and +-0), with the
// lowest-index tie-break made exact by an index-ordered compaction.
//
//   k_topk_begin   1 CTA: reset per-call scratch, zero histograms.
//   k_scan<A>      THE streaming pass (12N bytes: read g, read r, write p->r).
//                  Level-1 histogram of key>>19 in shared memory and, when the
//                  worker has a predicted level-1 digit G from its previous
//                  call, the index-ordered compaction of every element with
//                  digit >= G into a tile-segmented staging area (tile-local
//                  block scan, no global ordering needed).  The last CTA to
//                  finish resolves level 1 (digit b1 of the k-th largest key)
//                  and validates the prediction (count(digit >= G) >= k).
//   k_scan<A2>     only if the prediction missed: full histogram pass (reads p).
//   k_scan<D>      only if no valid staging exists: compaction of digit >= b1.
//   k_refine<L>    levels 2..: histograms over the staged candidates only.
//   k_final_count  per-tile (gt, eq) counts vs the exact threshold key T; the
//                  last CTA scans them.
//   k_final_write  per-tile ordered write of idx/val; r[idx] = +0.
// Every kernel is launched unconditionally and exits early from device-side
// flags, so the sequence is CUDA-graph capturable and never syncs the host.
#include "psb_internal.cuh"

namespace {

template <class T>
struct VecOf;
template <>
struct VecOf<float> {
  typedef float4 V;
  static constexpr int W = 4;
};
template <>
struct VecOf<double> {
  typedef double2 V;
  static constexpr int W = 2;
};

template <class T>
__host__ __device__ constexpr int tile_elems() {
  return PSB_SCAN_THREADS * 4 * VecOf<T>::W;  // f32: 4096, f64: 2048
}

enum { MODE_A = 0, MODE_A2 = 1, MODE_D = 2 };
enum { DONE_A = 0, DONE_A2 = 1, DONE_R = 2, DONE_F = 3 };

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
  uint32_t* tile_cnt;
  uint32_t* stage_idx;
  T* stage_val;
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
// PSB_SCAN_THREADS threads).  Bins [lo, nbins) hold exact counts; when
// `implicit0`, bin 0 (not counted by the producers) holds match - sum(others).
// Finds the bin b containing the need-th largest entry.  Also finds the bin
// where the cumulative count from the top first reaches `want` (prediction).
// Returns via shared outputs: found, bin, above (count in bins > b), cnt (=h[b]).
struct LevelResult {
  int found;
  uint32_t bin;
  unsigned long long above;
  unsigned long long cnt;
  int want_found;
  uint32_t want_bin;
  unsigned long long total;  // sum over bins >= max(lo,1)
};

__device__ void resolve_level(uint32_t* hist, uint32_t nbins, uint32_t lo,
                              unsigned long long need, unsigned long long want,
                              unsigned long long* sh_warp, LevelResult* out) {
  const uint32_t t = threadIdx.x;
  const uint32_t B = nbins >= PSB_SCAN_THREADS ? nbins / PSB_SCAN_THREADS : 1;
  const uint32_t b0 = t * B;
  unsigned long long sum = 0;
  if (b0 < nbins) {
    for (uint32_t b = b0; b < b0 + B; ++b) {
      uint32_t h = __ldcg(hist + b);
      if (b >= lo && b >= 1) sum += h;
    }
  }
  if (t == 0) {
    out->found = 0;
    out->want_found = 0;
  }
  unsigned long long total;
  unsigned long long ex = block_exscan_u64(sum, sh_warp, &total);
  unsigned long long suf = total - ex - sum;  // count in bins of threads > t
  if (b0 < nbins) {
    if (suf < need && need <= suf + sum) {
      unsigned long long cum = suf;
      for (int b = (int)(b0 + B) - 1; b >= (int)b0; --b) {
        if ((uint32_t)b < lo || b < 1) continue;
        uint32_t h = __ldcg(hist + b);
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
    if (suf < want && want <= suf + sum) {
      unsigned long long cum = suf;
      for (int b = (int)(b0 + B) - 1; b >= (int)b0; --b) {
        if ((uint32_t)b < lo || b < 1) continue;
        uint32_t h = __ldcg(hist + b);
        if (cum + h >= want) {
          out->want_found = 1;
          out->want_bin = (uint32_t)b;
          break;
        }
        cum += h;
      }
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
    s->g_used = predict ? w->g_pred : 0u;
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
  constexpr bool kHist = MODE != MODE_D;

  __shared__ uint32_t sh_hist[kHist ? PSB_HIST_BINS : 1];
  __shared__ unsigned long long sh_warp[32];
  __shared__ uint32_t sh_nonfinite;
  __shared__ LevelResult sh_res;

  uint32_t G;
  bool compact;
  if (MODE == MODE_D) {
    if (!a.s->need_compact) return;
    G = a.s->b1;
    compact = true;
  } else if (MODE == MODE_A2) {
    if (!a.s->need_full_hist) return;
    G = 0;
    compact = false;
  } else {
    G = a.s->g_used;
    compact = G > 0;
  }
  const uint32_t lo_bin = G > 1 ? G : 1;

  if (kHist)
    for (int b = threadIdx.x; b < PSB_HIST_BINS; b += blockDim.x) sh_hist[b] = 0;
  if (threadIdx.x == 0) sh_nonfinite = 0;
  __syncthreads();

  uint32_t nonfinite = 0;
  const T* __restrict__ src = (MODE == MODE_A) ? a.g : a.p;
  T* __restrict__ rr = a.r;

  for (uint32_t tile = blockIdx.x; tile < a.ntiles; tile += gridDim.x) {
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
          const uint32_t d = (uint32_t)(key >> SH1);
          if (kHist && d >= lo_bin) atomicAdd(&sh_hist[d], 1u);
          if (d >= G) fl |= 1u << bit;
        }
      }
    }

    if (compact) {
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
            a.stage_idx[base + pos] = (uint32_t)e;
            a.stage_val[base + pos] = x[j][c];
            ++pos;
          }
        }
      }
      if (threadIdx.x == 0) a.tile_cnt[tile] = acc;
    }
  }

  if (nonfinite) sh_nonfinite = 1;
  __syncthreads();
  if (threadIdx.x == 0 && sh_nonfinite) atomicOr(a.flags, 1u);
  if (kHist) {
    for (int b = threadIdx.x; b < PSB_HIST_BINS; b += blockDim.x) {
      const uint32_t h = sh_hist[b];
      if (h) atomicAdd(&a.hist1[b], h);
    }
  }
  if (MODE == MODE_D) return;

  if (!last_block(&a.s->done[MODE == MODE_A ? DONE_A : DONE_A2])) return;

  // ---- level-1 resolution (last CTA)
  const unsigned long long k = a.s->k, n = a.s->n;
  const unsigned long long want = (2 * k < n) ? 2 * k : n;
  resolve_level(a.hist1, PSB_HIST_BINS, lo_bin, k, want, sh_warp, &sh_res);
  if (threadIdx.x == 0) {
    const LevelResult& R = sh_res;
    uint32_t g_next = 0;
    if (R.want_found) g_next = R.want_bin;
    else if (G > 0) g_next = G > 8 ? G - 8 : 0;
    if (R.found) {
      a.s->b1 = R.bin;
      a.s->prefix = R.bin;
      a.s->need = k - R.above;
      a.s->match = R.cnt;
      a.s->need_compact = (G > 0) ? 0u : 1u;
    } else if (G == 0) {
      // the k-th largest key lies in digit 0 (zeros / tiny denormals)
      a.s->b1 = 0;
      a.s->prefix = 0;
      a.s->need = k - R.total;
      a.s->match = n - R.total;
      a.s->need_compact = 1;
    } else {
      a.s->need_full_hist = 1;  // prediction missed: rerun level 1 on all of p
    }
    a.w->g_pred = g_next;
    a.w->calls += (MODE == MODE_A) ? 1u : 0u;
  }
  // level-1 histogram is consumed; clear it for an A2 rerun
  __syncthreads();
  for (int b = threadIdx.x; b < PSB_HIST_BINS; b += blockDim.x) a.hist1[b] = 0;
}

// ---------------------------------------------------------------- refine
template <class T>
struct StageArgs {
  uint32_t ntiles;
  TopkScratch* s;
  uint32_t* histr;
  const uint32_t* tile_cnt;
  uint32_t* tile_gt;
  uint32_t* tile_eq;
  const uint32_t* stage_idx;
  const T* stage_val;
  uint32_t* idx_out;
  T* val_out;
  T* r;
};

template <class T>
__global__ void __launch_bounds__(PSB_SCAN_THREADS) k_refine(StageArgs<T> a, int level) {
  typedef KeyOf<T> KO;
  typedef typename KO::K K;
  constexpr int TILE = tile_elems<T>();
  __shared__ uint32_t sh_hist[PSB_HIST_BINS];
  __shared__ unsigned long long sh_warp[32];
  __shared__ LevelResult sh_res;

  const int pshift = KO::shift(level - 1);
  const int shift = KO::shift(level);
  const uint32_t nbins = 1u << KO::width(level);
  const K prefix = (K)a.s->prefix;

  for (uint32_t b = threadIdx.x; b < nbins; b += blockDim.x) sh_hist[b] = 0;
  __syncthreads();

  const int lane = threadIdx.x & 31;
  const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t t = warp; t < a.ntiles; t += nwarps) {
    const uint32_t cnt = a.tile_cnt[t];
    const size_t base = (size_t)t * TILE;
    for (uint32_t i = lane; i < cnt; i += 32) {
      const K key = KO::key(a.stage_val[base + i]);
      if ((key >> pshift) == prefix) {
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
  resolve_level(a.histr, nbins, 1, need, 0ull, sh_warp, &sh_res);
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
    a.s->prefix = (a.s->prefix << KO::width(level)) | bin;
    a.s->need = need - above;
    a.s->match = cnt;
    a.s->done[DONE_R] = 0;  // next level reuses the counter (stream-ordered)
  }
  __syncthreads();
  for (uint32_t b = threadIdx.x; b < nbins; b += blockDim.x) a.histr[b] = 0;
}

// --------------------------------------------------------------- final
template <class T>
__global__ void __launch_bounds__(PSB_SCAN_THREADS) k_final_count(StageArgs<T> a) {
  typedef KeyOf<T> KO;
  typedef typename KO::K K;
  constexpr int TILE = tile_elems<T>();
  __shared__ unsigned long long sh_warp[32];
  const K T_key = (K)a.s->prefix;
  const int lane = threadIdx.x & 31;
  const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t t = warp; t < a.ntiles; t += nwarps) {
    const uint32_t cnt = a.tile_cnt[t];
    const size_t base = (size_t)t * TILE;
    uint32_t gt = 0, eq = 0;
    for (uint32_t i = lane; i < cnt; i += 32) {
      const K key = KO::key(a.stage_val[base + i]);
      gt += key > T_key;
      eq += key == T_key;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      gt += __shfl_xor_sync(0xffffffffu, gt, o);
      eq += __shfl_xor_sync(0xffffffffu, eq, o);
    }
    if (lane == 0) {
      a.tile_gt[t] = gt;
      a.tile_eq[t] = eq;
    }
  }
  if (!last_block(&a.s->done[DONE_F])) return;

  // exclusive scan of (gt, eq) over tiles, packed in one u64 (each total < 2^32)
  const uint32_t per = (a.ntiles + blockDim.x - 1) / blockDim.x;
  const uint32_t t0 = threadIdx.x * per;
  const uint32_t t1 = min(a.ntiles, t0 + per);
  unsigned long long local = 0;
  for (uint32_t t = t0; t < t1; ++t)
    local += (unsigned long long)__ldcg(a.tile_gt + t) |
             ((unsigned long long)__ldcg(a.tile_eq + t) << 32);
  unsigned long long total;
  unsigned long long run = block_exscan_u64(local, sh_warp, &total);
  for (uint32_t t = t0; t < t1; ++t) {
    const uint32_t g = __ldcg(a.tile_gt + t), e = __ldcg(a.tile_eq + t);
    a.tile_gt[t] = (uint32_t)(run & 0xffffffffull);
    a.tile_eq[t] = (uint32_t)(run >> 32);
    run += (unsigned long long)g | ((unsigned long long)e << 32);
  }
}

template <class T>
__global__ void __launch_bounds__(PSB_SCAN_THREADS) k_final_write(StageArgs<T> a) {
  typedef KeyOf<T> KO;
  typedef typename KO::K K;
  constexpr int TILE = tile_elems<T>();
  const K T_key = (K)a.s->prefix;
  const unsigned long long need_eq = a.s->need;
  const int lane = threadIdx.x & 31;
  const uint32_t lt_mask = (1u << lane) - 1u;
  const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t t = warp; t < a.ntiles; t += nwarps) {
    const uint32_t cnt = a.tile_cnt[t];
    if (cnt == 0) continue;
    const size_t base = (size_t)t * TILE;
    const unsigned long long eq_off = a.tile_eq[t];
    unsigned long long run_sel = a.tile_gt[t] + (eq_off < need_eq ? eq_off : need_eq);
    unsigned long long run_eq = eq_off;
    for (uint32_t c0 = 0; c0 < cnt; c0 += 32) {
      const uint32_t i = c0 + lane;
      const bool valid = i < cnt;
      T v = T(0);
      uint32_t id = 0;
      K key = 0;
      if (valid) {
        v = a.stage_val[base + i];
        id = a.stage_idx[base + i];
        key = KO::key(v);
      }
      const bool gt = valid && key > T_key;
      const bool eq = valid && key == T_key;
      const uint32_t eqm = __ballot_sync(0xffffffffu, eq);
      const unsigned long long eq_rank = run_eq + __popc(eqm & lt_mask);
      const bool sel = gt || (eq && eq_rank < need_eq);
      const uint32_t selm = __ballot_sync(0xffffffffu, sel);
      if (sel) {
        const unsigned long long pos = run_sel + __popc(selm & lt_mask);
        a.idx_out[pos] = id;
        a.val_out[pos] = v;
        if (a.r) a.r[id] = T(0);
      }
      run_eq += __popc(eqm);
      run_sel += __popc(selm);
    }
  }
}

template <class T>
psb_status run_topk(psb_ctx* c, int worker, const T* g, T* r, size_t n, size_t k,
                    uint32_t* idx_out, T* val_out, cudaStream_t st) {
  constexpr int TILE = tile_elems<T>();
  const uint32_t ntiles = (uint32_t)((n + TILE - 1) / TILE);
  const int vec_ok = ((((uintptr_t)g) | ((uintptr_t)r)) & 15) == 0;
  TopkScratch* s = c->d_tk;
  TopkWorker* w = c->d_tw + worker;

  k_topk_begin<<<1, 256, 0, st>>>(s, w, c->d_hist1, c->d_histr, n, k, 1);
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
  a.stage_idx = c->d_stage_idx;
  a.stage_val = reinterpret_cast<T*>(c->d_stage_val);
  a.flags = c->d_flags;
  const uint32_t scan_grid = (uint32_t)std::min<size_t>(ntiles, (size_t)c->num_sms * 4);
  if (c->prof) cudaEventRecord(psb_prof_event(c), st);
  k_scan<T, MODE_A><<<scan_grid, PSB_SCAN_THREADS, 0, st>>>(a);
  if (c->prof) cudaEventRecord(psb_prof_event(c), st);
  k_scan<T, MODE_A2><<<scan_grid, PSB_SCAN_THREADS, 0, st>>>(a);
  k_scan<T, MODE_D><<<scan_grid, PSB_SCAN_THREADS, 0, st>>>(a);

  StageArgs<T> b;
  b.ntiles = ntiles;
  b.s = s;
  b.histr = c->d_histr;
  b.tile_cnt = c->d_tile_cnt;
  b.tile_gt = c->d_tile_gt;
  b.tile_eq = c->d_tile_eq;
  b.stage_idx = c->d_stage_idx;
  b.stage_val = reinterpret_cast<const T*>(c->d_stage_val);
  b.idx_out = idx_out;
  b.val_out = val_out;
  b.r = r;
  const uint32_t warp_grid =
      (uint32_t)std::max<size_t>(1, std::min<size_t>((ntiles + 7) / 8, (size_t)c->num_sms * 8));
  for (int level = 1; level < KeyOf<T>::kLevels; ++level)
    k_refine<T><<<warp_grid, PSB_SCAN_THREADS, 0, st>>>(b, level);
  k_final_count<T><<<warp_grid, PSB_SCAN_THREADS, 0, st>>>(b);
  k_final_write<T><<<warp_grid, PSB_SCAN_THREADS, 0, st>>>(b);
  c->launches += 6 + (KeyOf<T>::kLevels - 1);
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
  if (dt == PSB_F32)
    return run_topk<float>(c, worker, (const float*)g, (float*)r, n, k, idx_out, (float*)val_out, st);
  return run_topk<double>(c, worker, (const double*)g, (double*)r, n, k, idx_out, (double*)val_out,
                          st);
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
