// psb_cand.inl -- the K1 candidate phase (included by psb_topk.cu inside its
// anonymous namespace; uses its helpers).
//
// One cooperative launch, one CTA per SM, all CTAs co-resident.  Each CTA
// owns an equal slice of the logical (index-ordered) candidate list and, when
// the slice fits (it does for top-k ratios up to a few percent), stages it in
// shared memory once; every following pass -- the threshold levels, the
// (gt, eq) counts and the ordered write -- then runs out of shared memory.
// Grid-wide barriers replace kernel boundaries.
//
// Threshold T:
//   predicted mode (f32): coarse histogram of (key - G) >> kCoarseShift
//     (4096 bins, the top one an implicit overflow), then the fine histogram
//     of (key - G) & (2^kCoarseShift - 1) inside the chosen coarse bin.
//   otherwise: the remaining key radix levels (cold mode starts at level 1,
//     f64 and the overflow case at level 0).
// Write: slot = gt_before + min(eq_before, need_eq) from one packed (gt, eq)
//   block scan per sub-tile, so the output keeps index order; residual
//   fix-up and the fused single-worker SGD update of theta happen here.

constexpr int kCandThreads = 512;
constexpr uint32_t kCoarseBins = 4096;
constexpr int kCoarseShift = 11;  // 2048-ulp coarse bins: 4095 of them span one octave above G

template <class T>
struct CandArgs {
  TopkScratch* s;
  TopkWorker* w;
  uint32_t* histr;  // <= 4096-bin global histogram (coarse, fine or radix level)
  const uint32_t* cand_idx;
  const T* cand_val;
  const uint32_t* seg_pre;  // nseg + 1 exclusive prefixes of the k_scan CTA segments
  uint32_t nseg;
  size_t seg_cap;           // segment stride (= elements streamed by one k_scan CTA)
  uint32_t stage_cap;       // entries of the shared-memory staging area
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
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) unsigned char dsm[];
  uint32_t* sh_h = reinterpret_cast<uint32_t*>(dsm);                  // kCoarseBins words
  T* st_val = reinterpret_cast<T*>(dsm + kCoarseBins * 4);             // stage_cap values
  uint32_t* st_idx = reinterpret_cast<uint32_t*>(st_val + a.stage_cap);  // stage_cap indices
  __shared__ uint32_t sh_pre[PSB_FINAL_TPC_MAX + 1];
  __shared__ unsigned long long sh_warp[32];
  __shared__ LevelResult sh_res;
  __shared__ uint32_t sh_bad;

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
  for (uint32_t b = threadIdx.x; b <= a.nseg; b += blockDim.x) sh_pre[b] = a.seg_pre[b];
  if (threadIdx.x == 0) sh_bad = 0;
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
    // copy the slice segment piece by segment piece with cp.async (LDGSTS):
    // every thread keeps all of its copies in flight, no register round trip
    uint32_t e = lo, sg = m.seg_of(lo);
    while (e < hi) {
      while (sh_pre[sg + 1] <= e) ++sg;
      const uint32_t pe = min(hi, sh_pre[sg + 1]);
      const size_t src = (size_t)sg * m.cap + (e - sh_pre[sg]);
      for (uint32_t j = threadIdx.x; j < pe - e; j += blockDim.x) {
        __pipeline_memcpy_async(st_val + (e - lo + j), a.cand_val + src + j, sizeof(T));
        __pipeline_memcpy_async(st_idx + (e - lo + j), a.cand_idx + src + j, 4);
      }
      e = pe;
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
  // One histogram pass over the slice: digit(key) for matching keys.
  auto hist_pass = [&](uint32_t nbins, auto digit_of) {
    for (uint32_t b = threadIdx.x; b < nbins; b += blockDim.x) sh_h[b] = 0;
    __syncthreads();
    for (uint32_t base = 0; base < cnt; base += 4 * kCandThreads) {
      const uint32_t j0 = base + 4 * threadIdx.x;
      T v[4];
      uint32_t id[4];
      load4(j0, v, id, false);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t d = 0;
        const bool ok = digit_of(KO::key(v[c]), &d) && j0 + c < cnt;
        hist_add_agg(sh_h, d, ok);
      }
    }
    __syncthreads();
    for (uint32_t b = threadIdx.x; b < nbins; b += blockDim.x) {
      const uint32_t h = sh_h[b];
      if (h) atomicAdd(&a.histr[b], h);
    }
  };
  // CTA 0 resolves a level: bin holding the need-th largest (implicit bin 0).
  auto resolve0 = [&](uint32_t nbins, unsigned long long need, unsigned long long match,
                      uint32_t* bin, unsigned long long* above, unsigned long long* bcnt) {
    resolve_level(a.histr, nbins, 1, need, sh_warp, &sh_res, sh_h);
    *bin = sh_res.found ? sh_res.bin : 0u;
    *above = sh_res.found ? sh_res.above : sh_res.total;
    *bcnt = sh_res.found ? sh_res.cnt : match - sh_res.total;
    for (uint32_t b = threadIdx.x; b < nbins; b += blockDim.x) a.histr[b] = 0;
  };

  const bool pred = s->g_key != 0 && !s->need_full_hist;  // predicted candidate set valid
  const bool spec = pred && s->spec_ok;                    // pass A zeroed all candidates
  uint32_t level = s->start_level;

  // ---- exact threshold T
  if (sizeof(T) == 4 && pred && level == 0) {
    const K G = (K)s->g_key;
    // coarse digit min((key - G) >> kCoarseShift, 4095): the top bin collects
    // every key an octave or more above G (overflow); digit 0 is implicit.
    hist_pass(kCoarseBins, [&](K key, uint32_t* d) {
      const K dl = (key - G) >> kCoarseShift;
      *d = dl < (K)(kCoarseBins - 1) ? (uint32_t)dl : kCoarseBins - 1;
      return *d != 0;  // coarse digit 0 is implicit (C - sum of the others)
    });
    grid.sync();
    phase();
    if (blockIdx.x == 0) {
      uint32_t bin;
      unsigned long long above, bcnt;
      resolve0(kCoarseBins, k, C, &bin, &above, &bcnt);
      if (threadIdx.x == 0) {
        if (bin < kCoarseBins - 1) {
          s->b1 = bin;
          s->need = k - above;
          s->match = bcnt;
          s->start_level = 100;  // fine level next
        }  // else T is an octave above G: fall back to the key radix levels
      }
    }
    grid.sync();
    phase();
    level = s->start_level;
    if (level == 100) {
      const K cb = (K)s->b1;
      hist_pass(1u << kCoarseShift, [&](K key, uint32_t* d) {
        const K dl = key - G;
        *d = (uint32_t)(dl & ((1u << kCoarseShift) - 1));
        return (dl >> kCoarseShift) == cb && *d != 0;  // fine digit 0 is implicit
      });
      grid.sync();
      phase();
      if (blockIdx.x == 0) {
        uint32_t bin;
        unsigned long long above, bcnt;
        const unsigned long long need = s->need;
        resolve0(1u << kCoarseShift, need, s->match, &bin, &above, &bcnt);
        if (threadIdx.x == 0) {
          s->prefix = (unsigned long long)(G + (cb << kCoarseShift) + (K)bin);  // exact T
          s->need = need - above;
          s->start_level = KO::kLevels;
        }
      }
      grid.sync();
      phase();
      level = KO::kLevels;
    }
  }
  for (; level < (uint32_t)KO::kLevels; ++level) {  // key radix levels
    const int pshift = level ? KO::shift(level - 1) : (int)(sizeof(K) * 8 - 1);
    const int shift = KO::shift(level);
    const uint32_t nbins = 1u << KO::width(level);
    const K prefix = (K)s->prefix;
    hist_pass(nbins, [&](K key, uint32_t* d) {
      *d = (uint32_t)(key >> shift) & (nbins - 1);
      return (key >> pshift) == prefix && *d != 0;  // digit 0 is implicit
    });
    grid.sync();
    phase();
    if (blockIdx.x == 0) {
      uint32_t bin;
      unsigned long long above, bcnt;
      const unsigned long long need = s->need;
      resolve0(nbins, need, s->match, &bin, &above, &bcnt);
      if (threadIdx.x == 0) {
        s->prefix = level ? ((s->prefix << KO::width(level)) | bin) : bin;
        s->need = need - above;
        s->match = bcnt;
      }
    }
    grid.sync();
    phase();
  }

  // ---- (gt, eq) counts per CTA and their exclusive scan
  const K T_key = (K)s->prefix;
  const unsigned long long need_eq = s->need;
  {
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
  if (blockIdx.x == 0) {
    unsigned long long* sh_c = reinterpret_cast<unsigned long long*>(sh_h);  // gridDim.x <= 2048
    for (uint32_t b = threadIdx.x; b < gridDim.x; b += blockDim.x) sh_c[b] = __ldcg(a.cta + b);
    __syncthreads();
    const uint32_t qb = (gridDim.x + blockDim.x - 1) / blockDim.x;
    const uint32_t b0 = threadIdx.x * qb, b1 = min(gridDim.x, b0 + qb);
    unsigned long long local = 0;
    for (uint32_t b = b0; b < b1; ++b) local += sh_c[b];
    unsigned long long total;
    unsigned long long run = block_exscan_u64(local, sh_warp, &total);
    for (uint32_t b = b0; b < b1; ++b) {
      const unsigned long long c = sh_c[b];
      a.cta[b] = run;
      run += c;
    }
    if (threadIdx.x == 0) {
      // Next call's prediction G = key(T * rho * f): rho tracks the
      // threshold's drift (error feedback makes it creep up), f is a safety
      // margin adapted so the candidate set stays a little above k.
      TopkWorker* w = a.w;
      float f = w->f > 0.f ? w->f : 0.97f;
      const double ratio = (double)C / (double)k;
      w->last_ratio = (float)ratio;
      if (pred) {
        if (ratio > 2.0) f = 1.f - (1.f - f) * 0.8f;         // loose: tighten
        else if (ratio < 1.08) f = 1.f - (1.f - f) * 1.25f;  // thin: widen
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
    }
  }
  grid.sync();
  phase();

  // ---- ordered write
  unsigned long long run = a.cta[blockIdx.x];  // (gt | eq << 32) before this slice
  bool bad = false;
  for (uint32_t base = 0; base < cnt; base += 4 * kCandThreads) {
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
    uint32_t selm = 0;
    unsigned long long slot[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const unsigned long long gt_b = before & 0xffffffffull, eq_b = before >> 32;
      const bool gt = (gtm >> c) & 1u, eq = (eqm >> c) & 1u;
      slot[c] = gt_b + (eq_b < need_eq ? eq_b : need_eq);
      if (gt || (eq && eq_b < need_eq)) selm |= 1u << c;
      before += (unsigned long long)gt | ((unsigned long long)eq << 32);
    }
    // issue the scattered theta loads together (memory-level parallelism)
    T th[4];
    if (a.theta) {
#pragma unroll
      for (int c = 0; c < 4; ++c) th[c] = ((selm >> c) & 1u) ? a.theta[id[c]] : T(0);
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      if ((selm >> c) & 1u) {
        a.idx_out[slot[c]] = id[c];
        a.val_out[slot[c]] = v[c];
        if (a.r && !spec) a.r[id[c]] = T(0);  // cold mode: pass A stored p
        if (a.theta) {
          const T mean = mul_rn(v[c], T(1));  // P = 1: mean = v * (1/1)
          const T t2 = add_rn(mul_rn(a.coef, mean), th[c]);
          a.theta[id[c]] = t2;
          if (a.mean_out) a.mean_out[id[c]] = mean;
          bad |= !is_finite(t2);
        }
      } else if (spec && a.r && j0 + c < cnt) {
        a.r[id[c]] = v[c];  // unselected candidate: undo the speculative +0
      }
    }
    run += tot;
  }
  if (bad) sh_bad = 1;
  __syncthreads();
  if (threadIdx.x == 0 && sh_bad) atomicOr(a.flags, 1u);
  phase();
}
