// psb_cand.inl -- the K1 candidate phase (included by psb_topk.cu inside its
// anonymous namespace; uses its helpers).
//
// One cooperative launch, one CTA per SM, all CTAs co-resident.  Each CTA
// owns an equal slice of the logical (index-ordered) candidate list and, when
// the slice fits (it does for top-k ratios up to a few percent), stages it in
// shared memory once; every following pass -- the threshold levels, the
// (gt, eq) counts and the ordered write -- then runs out of shared memory.
// One grid-wide barrier per level replaces a kernel boundary: after it, EVERY
// CTA resolves the level from the global histogram itself (same data, same
// deterministic result), so no second barrier is needed to broadcast it.
//
// Threshold T:
//   predicted mode (f32): coarse histogram of (key - G) >> kCoarseShift
//     (4096 bins, the top one collecting everything an octave or more above
//     G), then the fine histogram of (key - G) & (2^kCoarseShift - 1) inside
//     the chosen coarse bin.
//   otherwise: the remaining key radix levels (cold mode starts at level 1,
//     f64 and the overflow case at level 0).
// Write: slot = gt_before + min(eq_before, need_eq) from one packed (gt, eq)
//   block scan per sub-tile, so the output keeps index order; then a
//   barrier-free loop does the scattered part (residual fix-up, and the fused
//   single-worker SGD update theta[idx] += (-lr) * (val * 1)).

#ifndef PSB_CAND_THREADS
#define PSB_CAND_THREADS 512
#endif
constexpr int kCandThreads = PSB_CAND_THREADS;
static_assert(4096 % kCandThreads == 0 && kCandThreads % 32 == 0, "level histograms are split evenly over the CTA");
constexpr uint32_t kCoarseBins = 4096;
constexpr int kCoarseShift = 11;  // 2048-ulp coarse bins: 4095 of them span one octave above G
constexpr uint32_t kLevelHist = 4096;  // words per level histogram buffer
constexpr int kHistCoarse = 8, kHistFine = 9, kNumLevelHists = 10;  // radix levels use 0..7

template <class T>
struct CandArgs {
  TopkScratch* s;
  TopkWorker* w;
  uint32_t* hlev;  // kNumLevelHists x kLevelHist global histograms (zero between calls)
  const uint32_t* cand_idx;
  const T* cand_val;
  const uint32_t* seg_cnt;  // candidates per k_scan CTA segment (nseg)
  uint32_t nseg;
  size_t seg_cap;           // segment stride (= elements streamed by one k_scan CTA)
  uint32_t stage_cap;       // entries of the shared-memory staging area
  unsigned long long* cta;  // per-CTA (gt | eq << 32) totals
  uint32_t* idx_out;
  T* val_out;
  T* r;
  T* theta;     // fused single-worker SGD update (nullable)
  T* mean_out;  // with theta: dense mean at touched indices (nullable)
  T coef;       // (T)(-lr)
  uint32_t* flags;
  // NVLink push (multi-rank full exchange): this worker's payload slot in
  // every peer's arena; each CTA copies its contiguous payload range there
  int npush;
  uint32_t* push_idx[PSB_MAX_P];
  T* push_val[PSB_MAX_P];
};

// Flat view of the segmented candidate list: logical entry e (index order)
// lies in segment s with pre[s] <= e < pre[s+1], physically at
// s*cap + (e - pre[s]).
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
  __device__ __forceinline__ size_t phys(uint32_t e, uint32_t* sg) const {
    while (pre[*sg + 1] <= e) ++*sg;
    return (size_t)*sg * cap + (e - pre[*sg]);
  }
};

template <class T>
__global__ void __launch_bounds__(kCandThreads, 1) k_cand(CandArgs<T> a) {
  typedef KeyOf<T> KO;
  typedef typename KO::K K;
  constexpr uint32_t kNoSlot = 0xffffffffu;
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) unsigned char dsm[];
  uint32_t* sh_h = reinterpret_cast<uint32_t*>(dsm);                      // kCoarseBins words
  T* st_val = reinterpret_cast<T*>(dsm + kCoarseBins * 4);                 // stage_cap values
  uint32_t* st_idx = reinterpret_cast<uint32_t*>(st_val + a.stage_cap);    // stage_cap indices
  uint32_t* st_slot = st_idx + a.stage_cap;                                // stage_cap output slots
  __shared__ uint32_t sh_pre[PSB_FINAL_TPC_MAX + 1];
  __shared__ unsigned long long sh_warp[32];
  __shared__ LevelResult sh_res;
  __shared__ uint32_t sh_bad;
  __shared__ unsigned long long sh_base;

  TopkScratch* s = a.s;
  const unsigned long long k = s->k;
  int nphase = 0;
  auto phase = [&]() {  // CTA-0 timestamps for psb_topk_phases diagnostics
    if (blockIdx.x == 0 && threadIdx.x == 0 && nphase < 16) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      s->phase_ns[nphase] = t;
    }
    ++nphase;
  };
  phase();

  // ---- this CTA's slice [lo, hi) of the logical list (multiple of 4 entries)
  // exclusive prefix of the k_scan segment counts, computed by every CTA
  // (no serial last-block pass at the end of k_scan)
  {
    const uint32_t q = (a.nseg + blockDim.x - 1) / blockDim.x;
    const uint32_t b0 = min(a.nseg, threadIdx.x * q), b1 = min(a.nseg, b0 + q);
    unsigned long long loc = 0;
    for (uint32_t b = b0; b < b1; ++b) loc += __ldcg(a.seg_cnt + b);
    unsigned long long tot;
    unsigned long long run0 = block_exscan_u64(loc, sh_warp, &tot);
    for (uint32_t b = b0; b < b1; ++b) {
      sh_pre[b] = (uint32_t)run0;
      run0 += __ldcg(a.seg_cnt + b);
    }
    if (threadIdx.x == 0) {
      sh_pre[a.nseg] = (uint32_t)tot;
      sh_bad = 0;
    }
  }
  __syncthreads();
  FlatMap m;
  m.pre = sh_pre;
  m.nseg = a.nseg;
  m.cap = a.seg_cap;
  const uint32_t C = sh_pre[a.nseg];
  uint32_t chunk = (C + gridDim.x - 1) / gridDim.x;
  chunk = (chunk + 3u) & ~3u;
  const uint32_t lo = min(C, blockIdx.x * chunk), hi = min(C, lo + chunk);
  const uint32_t cnt = hi - lo;
  const bool staged = cnt <= a.stage_cap;
  if (staged && cnt) {
    // copy the slice with cp.async (LDGSTS), all copies in flight at once.
    // Thread t takes entries t, t + blockDim, ... and walks the k_scan
    // segments forward as it goes (one binary search per thread), so a slice
    // spanning hundreds of sparse segments costs no per-segment round trip.
    uint32_t sg = m.seg_of(min(lo + threadIdx.x, hi > 0 ? hi - 1 : 0));
    for (uint32_t j = threadIdx.x; j < cnt; j += blockDim.x) {
      const uint32_t e = lo + j;
      while (sh_pre[sg + 1] <= e) ++sg;
      const size_t src = (size_t)sg * m.cap + (e - sh_pre[sg]);
      __pipeline_memcpy_async(st_val + j, a.cand_val + src, sizeof(T));
      __pipeline_memcpy_async(st_idx + j, a.cand_idx + src, 4);
    }
    __pipeline_commit();
    __pipeline_wait_prior(0);
  }
  __syncthreads();
  phase();

  // Four consecutive entries j0..j0+3 of the slice (j0 local, multiple of 4).
  auto load4 = [&](uint32_t j0, T (&v)[4], uint32_t (&id)[4], bool want_idx) {
    if (staged) {
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        v[c] = j0 + c < cnt ? st_val[j0 + c] : T(0);
        if (want_idx) id[c] = j0 + c < cnt ? st_idx[j0 + c] : 0u;
      }
    } else {
      uint32_t sg = j0 < cnt ? m.seg_of(lo + j0) : 0;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        if (j0 + c < cnt) {
          const size_t p = m.phys(lo + j0 + c, &sg);
          v[c] = a.cand_val[p];
          if (want_idx) id[c] = a.cand_idx[p];
        } else {
          v[c] = T(0);
          if (want_idx) id[c] = 0u;
        }
      }
    }
  };
  // One histogram pass over the slice (digit(key) for matching keys), flushed
  // into global histogram `g`; then the grid barrier; then every CTA resolves
  // the level from `g`: bin holding the need-th largest (bin 0 implicit).
  bool pf_theta = a.theta != nullptr && staged;  // first level pass only
  auto level_pass = [&](uint32_t* g, uint32_t nbins, unsigned long long need, unsigned long long match,
                        auto digit_of, uint32_t* bin, unsigned long long* above,
                        unsigned long long* bcnt) {
    for (uint32_t b = threadIdx.x; b < nbins; b += blockDim.x) sh_h[b] = 0;
    __syncthreads();
    for (uint32_t base = 0; base < cnt; base += 4 * kCandThreads) {
      const uint32_t j0 = base + 4 * threadIdx.x;
      T v[4];
      uint32_t id[4];
      load4(j0, v, id, pf_theta);
      if (pf_theta) {
        // the fused SGD at the end updates theta at the selected indices:
        // pull those sectors into L2 while this pass (sync/atomic-bound) runs
#pragma unroll
        for (int c = 0; c < 4; ++c)
          if (j0 + c < cnt) asm volatile("prefetch.global.L2 [%0];" ::"l"(a.theta + id[c]));
      }
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t d = 0;
        const bool ok = digit_of(KO::key(v[c]), &d) && j0 + c < cnt;
        if (ok) atomicAdd(&sh_h[d], 1u);  // candidate keys spread over the bins: plain smem atomics
      }
    }
    __syncthreads();
    for (uint32_t b = threadIdx.x; b < nbins; b += blockDim.x) {
      const uint32_t h = sh_h[b];
      if (h) atomicAdd(&g[b], h);
    }
    pf_theta = false;
    grid.sync();
    phase();
    resolve_level(g, nbins, 1, need, sh_warp, &sh_res, sh_h);
    *bin = sh_res.found ? sh_res.bin : 0u;
    *above = sh_res.found ? sh_res.above : sh_res.total;
    *bcnt = sh_res.found ? sh_res.cnt : match - sh_res.total;
  };

  const bool pred = s->g_key != 0 && !s->need_full_hist;  // predicted candidate set valid
  const bool spec = pred && s->spec_ok;  // pass A zeroed the residual of candidates with key >= zk
  const K zk = (K)s->z_key;
  auto zeroed = [&](T v) { return spec && KO::key(v) >= zk; };
  uint32_t level = s->start_level;
  K prefix = (K)s->prefix;
  unsigned long long need = s->need, match = s->match;
  bool delta = false;

  // ---- exact threshold T (state identical in every CTA)
  if (sizeof(T) == 4 && pred && level == 0) {
    const K G = (K)s->g_key;
    uint32_t cb;
    unsigned long long above, bcnt;
    // coarse digit min((key - G) >> kCoarseShift, 4095): the top bin collects
    // every key an octave or more above G; digit 0 is implicit (C - others).
    level_pass(a.hlev + kHistCoarse * kLevelHist, kCoarseBins, k, C,
               [&](K key, uint32_t* d) {
                 const K dl = (key - G) >> kCoarseShift;
                 *d = dl < (K)(kCoarseBins - 1) ? (uint32_t)dl : kCoarseBins - 1;
                 return *d != 0;
               },
               &cb, &above, &bcnt);
    if (cb < kCoarseBins - 1) {
      uint32_t fb;
      unsigned long long fabove, fcnt;
      level_pass(a.hlev + kHistFine * kLevelHist, 1u << kCoarseShift, k - above, bcnt,
                 [&](K key, uint32_t* d) {
                   const K dl = key - G;
                   *d = (uint32_t)(dl & ((1u << kCoarseShift) - 1));
                   return (dl >> kCoarseShift) == (K)cb && *d != 0;  // fine digit 0 implicit
                 },
                 &fb, &fabove, &fcnt);
      prefix = G + ((K)cb << kCoarseShift) + (K)fb;  // exact T
      need = k - above - fabove;
      level = KO::kLevels;
      delta = true;
    }  // else T is an octave or more above G: the key radix levels from level 0
  }
  for (; level < (uint32_t)KO::kLevels; ++level) {  // key radix levels
    const int pshift = level ? KO::shift(level - 1) : (int)(sizeof(K) * 8 - 1);
    const int shift = KO::shift(level);
    const uint32_t nbins = 1u << KO::width(level);
    const K pf = prefix;
    uint32_t bin;
    unsigned long long above, bcnt;
    level_pass(a.hlev + level * kLevelHist, nbins, need, match,
               [&](K key, uint32_t* d) {
                 *d = (uint32_t)(key >> shift) & (nbins - 1);
                 return (key >> pshift) == pf && *d != 0;  // digit 0 implicit
               },
               &bin, &above, &bcnt);
    prefix = level ? ((prefix << KO::width(level)) | bin) : bin;
    need -= above;
    match = bcnt;
  }
  const K T_key = prefix;
  const unsigned long long need_eq = need;

  // ---- (gt, eq) counts per CTA; every CTA sums the totals of the CTAs before it.
  // Staged slices: thread t owns the contiguous run [r0, r1) of the slice, so
  // ONE block scan gives every thread its starting (gt, eq) for the write.
  const uint32_t per = (cnt + kCandThreads - 1) / kCandThreads;
  const uint32_t r0 = min(cnt, threadIdx.x * per), r1 = min(cnt, r0 + per);
  unsigned long long my_ex = 0, cta_total = 0;
  if (staged) {
    uint32_t gt = 0, eq = 0;
    for (uint32_t j = r0; j < r1; ++j) {
      const K key = KO::key(st_val[j]);
      gt += key > T_key;
      eq += key == T_key;
    }
    my_ex = block_exscan_u64((unsigned long long)gt | ((unsigned long long)eq << 32), sh_warp, &cta_total);
    if (threadIdx.x == 0) a.cta[blockIdx.x] = cta_total;
  } else {
    uint32_t gt = 0, eq = 0;
    for (uint32_t base = 0; base < cnt; base += 4 * kCandThreads) {
      const uint32_t j0 = base + 4 * threadIdx.x;
      T v[4];
      uint32_t id[4];
      load4(j0, v, id, false);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const K key = KO::key(v[c]);
        gt += j0 + c < cnt && key > T_key;
        eq += j0 + c < cnt && key == T_key;
      }
    }
    unsigned long long total;
    block_exscan_u64((unsigned long long)gt | ((unsigned long long)eq << 32), sh_warp, &total);
    if (threadIdx.x == 0) a.cta[blockIdx.x] = total;
  }
  grid.sync();
  phase();
  {
    unsigned long long part = 0;
    for (uint32_t b = threadIdx.x; b < blockIdx.x; b += blockDim.x) part += __ldcg(a.cta + b);
    unsigned long long total;
    block_exscan_u64(part, sh_warp, &total);
    if (threadIdx.x == 0) sh_base = total;
  }
  // every CTA has read the level histograms: clear them for the next call
  for (uint32_t b = blockIdx.x * blockDim.x + threadIdx.x; b < kNumLevelHists * kLevelHist;
       b += gridDim.x * blockDim.x)
    a.hlev[b] = 0;
  if (blockIdx.x == 0) {
    if (threadIdx.x == 0) {
      s->prefix = T_key;  // diagnostics (psb_topk_stats)
      s->need = need_eq;
      if (delta) s->start_level = 100;  // T found on key - G
      // Next call's prediction G = key(T * rho * f): rho tracks the
      // threshold's drift (error feedback makes it creep up), f is a safety
      // margin adapted so the candidate set stays a little above k.
      TopkWorker* w = a.w;
      float f = w->f > 0.f ? w->f : 0.97f;
      const double ratio = (double)C / (double)k;
      w->last_ratio = (float)ratio;
      if (pred) {
        const double lo = w->ratio_lo > 0.f ? w->ratio_lo : PSB_RATIO_LO;
        const double hi = w->ratio_hi > 0.f ? w->ratio_hi : PSB_RATIO_HI;
        if (ratio > hi) f = 1.f - (1.f - f) * 0.8f;         // loose: tighten
        else if (ratio < lo) f = 1.f - (1.f - f) * 1.25f;  // thin: widen
      }
      f = fminf(fmaxf(f, 0.5f), 0.999f);
      float rho = w->rho > 0.f ? w->rho : 1.f;
      if (w->t_prev != 0 && T_key != 0 && T_key < KO::kInf) {
        const float now = (float)(to_mag(T_key, T(0)) / to_mag((K)w->t_prev, T(0)));
        rho = 0.5f * rho + 0.5f * fminf(fmaxf(now, 0.9f), 1.1f);
      }
      w->f = f;
      w->rho = rho;
      w->t_prev = T_key;
      w->g_key = (T_key == 0 || T_key >= KO::kInf) ? 0ull : scale_key(T_key, f * rho, T(0));
      w->z_key = (T_key == 0 || T_key >= KO::kInf) ? 0ull : scale_key(T_key, rho, T(0));
    }
  }
  __syncthreads();

  // ---- ordered write.  Loop 1: slots (block scans) and the sequential payload
  // writes; loop 2 (staged slices): the scattered updates without barriers.
  unsigned long long run = sh_base;  // (gt | eq << 32) before this slice
  bool bad = false;
  auto scatter = [&](uint32_t id, T v, bool sel) {
    if (sel) {
      if (a.r && !zeroed(v)) a.r[id] = T(0);  // pass A stored p
      if (a.theta) {
        const T mean = mul_rn(v, T(1));  // P = 1: mean = v * (1/1)
        const T t2 = add_rn(mul_rn(a.coef, mean), a.theta[id]);
        a.theta[id] = t2;
        if (a.mean_out) a.mean_out[id] = mean;
        bad |= !is_finite(t2);
      }
    } else if (a.r && zeroed(v)) {
      a.r[id] = v;  // unselected candidate: undo the speculative +0
    }
  };
  if (staged) {
    // the thread's run, in index order: slot = gt_before + min(eq_before, need_eq)
    unsigned long long before = run + my_ex;
    for (uint32_t j = r0; j < r1; ++j) {
      const T v = st_val[j];
      const K key = KO::key(v);
      const bool gt = key > T_key, eq = key == T_key;
      const unsigned long long gt_b = before & 0xffffffffull, eq_b = before >> 32;
      const bool sel = gt || (eq && eq_b < need_eq);
      if (sel) {
        const unsigned long long slot = gt_b + (eq_b < need_eq ? eq_b : need_eq);
        a.idx_out[slot] = st_idx[j];
        a.val_out[slot] = v;
      }
      st_slot[j] = sel ? 1u : kNoSlot;
      before += (unsigned long long)gt | ((unsigned long long)eq << 32);
    }
    run += cta_total;
  }
  for (uint32_t base = 0; base < (staged ? 0u : cnt); base += 4 * kCandThreads) {
    const uint32_t j0 = base + 4 * threadIdx.x;
    T v[4];
    uint32_t id[4];
    load4(j0, v, id, true);
    uint32_t gtm = 0, eqm = 0;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      if (j0 + c < cnt) {
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
      const bool sel = gt || (eq && eq_b < need_eq);
      if (sel) {
        const unsigned long long slot = gt_b + (eq_b < need_eq ? eq_b : need_eq);
        a.idx_out[slot] = id[c];
        a.val_out[slot] = v[c];
      }
      if (j0 + c < cnt) {
        if (staged) st_slot[j0 + c] = sel ? 1u : kNoSlot;
        else scatter(id[c], v[c], sel);
      }
      before += (unsigned long long)gt | ((unsigned long long)eq << 32);
    }
    run += tot;
  }
  phase();
  if (a.npush) {
    // this CTA's selected entries occupy payload slots [s_lo, s_hi) (index
    // order); re-read them from L2 and store them to every peer over NVLink
    // (coalesced 128-byte warp stores, posted: they drain during the scatter)
    const unsigned long long b0 = sh_base;
    const uint32_t s_lo = (uint32_t)((b0 & 0xffffffffull) + min(b0 >> 32, need_eq));
    const uint32_t s_hi = (uint32_t)((run & 0xffffffffull) + min(run >> 32, need_eq));
    __syncthreads();  // the CTA's payload writes are visible to the CTA
    for (uint32_t j = s_lo + threadIdx.x; j < s_hi; j += blockDim.x) {
      const uint32_t id = __ldcg(a.idx_out + j);
      const T v = __ldcg(a.val_out + j);
      for (int q = 0; q < a.npush; ++q) {
        a.push_idx[q][j] = id;
        a.push_val[q][j] = v;
      }
    }
  }
  if (staged) {
    __syncthreads();
    // batches of U entries per thread: all theta loads of a batch are issued
    // before any store (the indices are distinct), so U loads per thread are
    // in flight instead of one dependent round trip per entry
    constexpr int U = 8;
    for (uint32_t j0 = threadIdx.x; j0 < cnt; j0 += U * blockDim.x) {
      uint32_t id[U];
      T v[U], th[U];
      uint32_t selm = 0, actm = 0;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t j = j0 + u * blockDim.x;
        if (j < cnt) {
          actm |= 1u << u;
          id[u] = st_idx[j];
          v[u] = st_val[j];
          if (st_slot[j] != kNoSlot) selm |= 1u << u;
        }
      }
      if (a.theta) {
#pragma unroll
        for (int u = 0; u < U; ++u)
          if ((selm >> u) & 1u) th[u] = a.theta[id[u]];
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (!((actm >> u) & 1u)) continue;
        if ((selm >> u) & 1u) {
          if (a.r && !zeroed(v[u])) a.r[id[u]] = T(0);
          if (a.theta) {
            const T mean = mul_rn(v[u], T(1));  // P = 1: mean = v * (1/1)
            const T t2 = add_rn(mul_rn(a.coef, mean), th[u]);
            a.theta[id[u]] = t2;
            if (a.mean_out) a.mean_out[id[u]] = mean;
            bad |= !is_finite(t2);
          }
        } else if (a.r && zeroed(v[u])) {
          a.r[id[u]] = v[u];  // unselected candidate: undo the speculative +0
        }
      }
    }
  }
  if (bad) sh_bad = 1;
  if (a.npush) __threadfence_system();  // the pushes are visible before the peers are signalled
  __syncthreads();
  if (threadIdx.x == 0 && sh_bad) atomicOr(a.flags, 1u);
  phase();
}
