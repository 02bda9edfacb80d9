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
constexpr uint32_t kCoarseBins = PSB_COARSE_BINS;
constexpr int kCoarseShift = PSB_COARSE_SHIFT;  // 2048-ulp coarse bins: 4095 of them span one octave above G
constexpr uint32_t kLevelHist = 4096;  // words per level histogram buffer
constexpr int kHistCoarse = 8, kHistFine = 9, kNumLevelHists = 10;  // radix levels use 0..7

template <class T>
struct CandArgs {
  TopkScratch* s;
  TopkWorker* w;
  uint32_t* hlev;  // kNumLevelHists x kLevelHist global histograms (zero between calls)
  uint32_t* histd; // coarse (key - G) histogram of pass A's candidates, built by k_scan (f32; zero between calls)
  const uint32_t* seg_idx;   // k_scan's tile-segmented candidates (tile t at t*TILE, tile_cnt[t] entries)
  const T* seg_val;
  const uint32_t* tile_cnt;
  uint32_t* sb;              // [3][sb_stride] superblock sums of tile_cnt (cleared here for the next call)
  uint32_t sb_stride;
  uint32_t ntiles;
  uint32_t* cand_idx;        // the same candidates as one contiguous index-ordered list [0, C)
  T* cand_val;
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
#ifdef PSB_SCAN_TRACE
    if (threadIdx.x == 0 && blockIdx.x < 1024 && nphase < 15) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      g_cand_trace[blockIdx.x * 16 + nphase] = t;
    }
#endif
    ++nphase;
  };
  phase();
#ifdef PSB_SCAN_TRACE
#define TPHASE() phase()
#else
#define TPHASE()
#endif

  // ---- this CTA's slice of the index-ordered list, located without a grid
  // barrier.  Slices are whole k_scan tiles [tb, te), balanced on the cost
  // entries + alpha * tiles (alpha >= 8): a slice covering a sparse stretch
  // of the index space is bounded in tiles, so its tile prefix fits one
  // shared-memory window.  Every CTA scans the superblock sums (64 tiles
  // each), finds the superblocks holding its two boundaries, refines them to
  // tiles with one warp each, then scans its tiles' counts in windows of up to
  // 4095 tiles and copies its entries out of k_scan's tile segments -- into
  // shared memory when the slice fits the stage, else into the contiguous
  // global list at [lo, hi).
  constexpr int TILE = tile_elems<T>();
  constexpr uint32_t kWin = kCoarseBins - 1;  // tiles per prefix window (sh_h)
  constexpr uint32_t kSb = 1u << PSB_SB_SHIFT;
  __shared__ uint32_t sh_bsb[2];                 // superblock holding each boundary
  __shared__ unsigned long long sh_bpre[2];      // entries before that superblock
  __shared__ uint32_t sh_bt[2], sh_be[2];        // boundary tile and entries before it
  if (threadIdx.x == 0) sh_bad = 0;
  const uint32_t pass = __ldcg(&s->list_pass);
  const uint32_t* sbc = a.sb + (size_t)pass * a.sb_stride;
  const uint32_t nsb = (a.ntiles + kSb - 1) >> PSB_SB_SHIFT;
  uint32_t C;
  unsigned long long alpha, total_cost, tgt0, tgt1;
  {
    const uint32_t per = (nsb + blockDim.x - 1) / blockDim.x;
    const uint32_t b0 = min(nsb, threadIdx.x * per), b1 = min(nsb, b0 + per);
    unsigned long long loc = 0;
    for (uint32_t b = b0; b < b1; ++b) loc += __ldcg(sbc + b);
    unsigned long long tot;
    const unsigned long long ex = block_exscan_u64(loc, sh_warp, &tot);
    C = (uint32_t)tot;
    alpha = max(8ull, (tot + 2048ull * gridDim.x - 1) / (2048ull * gridDim.x));
    total_cost = tot + alpha * a.ntiles;
    const unsigned long long q = (total_cost + gridDim.x - 1) / gridDim.x;
    tgt0 = (unsigned long long)blockIdx.x * q;
    tgt1 = tgt0 + q;
    if (threadIdx.x < 2) {
      sh_bsb[threadIdx.x] = nsb;  // boundary at or past the end: the last tile
      sh_bpre[threadIdx.x] = tot;
    }
    __syncthreads();
    unsigned long long e = ex;
    for (uint32_t b = b0; b < b1; ++b) {
      const uint32_t cb = __ldcg(sbc + b);
      const unsigned long long c_lo = e + alpha * ((unsigned long long)b << PSB_SB_SHIFT);
      const unsigned long long c_hi = e + cb + alpha * min((unsigned long long)a.ntiles,
                                                           (unsigned long long)(b + 1) << PSB_SB_SHIFT);
      if (c_lo <= tgt0 && tgt0 < c_hi) {
        sh_bsb[0] = b;
        sh_bpre[0] = e;
      }
      if (c_lo <= tgt1 && tgt1 < c_hi) {
        sh_bsb[1] = b;
        sh_bpre[1] = e;
      }
      e += cb;
    }
  }
  __syncthreads();
  TPHASE();
  if (threadIdx.x < 64) {  // warp q2 refines boundary q2 to a tile
    const int q2 = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const unsigned long long target = q2 ? tgt1 : tgt0;
    const uint32_t b = sh_bsb[q2];
    if (b >= nsb) {
      if (lane == 0) {
        sh_bt[q2] = a.ntiles;
        sh_be[q2] = C;
      }
    } else {
      const uint32_t T0 = b << PSB_SB_SHIFT, nt = min(kSb, a.ntiles - T0);
      const uint32_t i0 = 2 * lane, i1 = 2 * lane + 1;
      const uint32_t c0 = i0 < nt ? __ldcg(a.tile_cnt + T0 + i0) : 0u;
      const uint32_t c1 = i1 < nt ? __ldcg(a.tile_cnt + T0 + i1) : 0u;
      uint32_t incl = c0 + c1;  // entries of this lane's two tiles, scanned over the warp
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      const unsigned long long e0 = sh_bpre[q2] + (incl - c0 - c1);  // entries before tile i0
      const unsigned long long t_cost0 = e0 + alpha * (T0 + i0);
      const unsigned long long t_cost1 = e0 + c0 + alpha * (T0 + i1);
      // boundary = first tile whose start cost reaches the target
      const bool below0 = i0 < nt && t_cost0 < target;
      const bool below1 = i1 < nt && t_cost1 < target;
      const uint32_t nbelow = __popc(__ballot_sync(0xffffffffu, below0)) + __popc(__ballot_sync(0xffffffffu, below1));
      // entries of the tiles before the boundary
      const uint32_t part = (below0 ? c0 : 0u) + (below1 ? c1 : 0u);
      uint32_t sum = part;
#pragma unroll
      for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
      if (lane == 0) {
        sh_bt[q2] = T0 + nbelow;
        sh_be[q2] = (uint32_t)(sh_bpre[q2] + sum);
      }
    }
  }
  __syncthreads();
  TPHASE();
  const uint32_t lo = sh_be[0], hi = sh_be[1];
  const uint32_t tb = sh_bt[0], te = sh_bt[1];
  const uint32_t cnt = hi - lo;
  const bool staged = cnt <= a.stage_cap;
#ifdef PSB_SCAN_TRACE
  if (threadIdx.x == 0 && blockIdx.x < 1024) g_cand_trace[blockIdx.x * 16 + 15] = ((unsigned long long)(te - tb) << 32) | cnt;
#endif
  if (cnt) {
    uint32_t* win = sh_h;  // logical prefix of the window's tiles (kWin + 1 entries)
    unsigned long long pre = lo;
    for (uint32_t ws = tb; ws < te; ws += kWin) {
      const uint32_t nwin = min(kWin, te - ws);
      {
        const uint32_t per = (nwin + blockDim.x - 1) / blockDim.x;
        const uint32_t i0 = min(nwin, threadIdx.x * per), i1 = min(nwin, i0 + per);
        unsigned long long loc = 0;
        for (uint32_t i = i0; i < i1; ++i) loc += __ldcg(a.tile_cnt + ws + i);
        unsigned long long tot;
        unsigned long long r0 = pre + block_exscan_u64(loc, sh_warp, &tot);
        for (uint32_t i = i0; i < i1; ++i) {
          win[i] = (uint32_t)r0;
          r0 += __ldcg(a.tile_cnt + ws + i);
        }
        if (threadIdx.x == 0) win[nwin] = (uint32_t)(pre + tot);
        pre += tot;
      }
      __syncthreads();
      // dense windows (>= 32 entries per tile): one warp per tile, lanes copy
      // the tile's segment; sparse windows: one thread per entry, its tile
      // found by binary search (a warp per near-empty tile idles its lanes).
      // 4-byte cp.async into the stage, plain copies into the global list.
      const uint32_t lane = threadIdx.x & 31, nw = blockDim.x >> 5;
      const uint32_t w_lo = win[0], w_n = win[nwin] - w_lo;
      if (w_n < 32u * nwin) {
        for (uint32_t e = w_lo + threadIdx.x; e < w_lo + w_n; e += blockDim.x) {
          uint32_t l = 0, h = nwin;  // win[l] <= e < win[h]
          while (h - l > 1) {
            const uint32_t m = (l + h) >> 1;
            if (win[m] <= e) l = m;
            else h = m;
          }
          const size_t src = (size_t)(ws + l) * TILE + (e - win[l]);
          if (staged) {
            __pipeline_memcpy_async(st_idx + (e - lo), a.seg_idx + src, 4);
            __pipeline_memcpy_async(st_val + (e - lo), a.seg_val + src, sizeof(T));
          } else {
            a.cand_idx[e] = a.seg_idx[src];
            a.cand_val[e] = a.seg_val[src];
          }
        }
      } else
      for (uint32_t i = threadIdx.x >> 5; i < nwin; i += nw) {
        const uint32_t e0 = win[i], ct = win[i + 1] - e0;
        const size_t src = (size_t)(ws + i) * TILE;
        if (staged) {
          for (uint32_t j = lane; j < ct; j += 32) {
            __pipeline_memcpy_async(st_idx + (e0 - lo) + j, a.seg_idx + src + j, 4);
            __pipeline_memcpy_async(st_val + (e0 - lo) + j, a.seg_val + src + j, sizeof(T));
          }
        } else {
          // into the global list: 8 entries per lane in flight per batch
          constexpr int CU = 8;
          for (uint32_t j0 = lane; j0 < ct; j0 += 32 * CU) {
            uint32_t ci[CU];
            T cv[CU];
#pragma unroll
            for (int u = 0; u < CU; ++u) {
              const uint32_t j = j0 + 32 * u;
              if (j < ct) {
                ci[u] = a.seg_idx[src + j];
                cv[u] = a.seg_val[src + j];
              }
            }
#pragma unroll
            for (int u = 0; u < CU; ++u) {
              const uint32_t j = j0 + 32 * u;
              if (j < ct) {
                a.cand_idx[e0 + j] = ci[u];
                a.cand_val[e0 + j] = cv[u];
              }
            }
          }
        }
      }
      __syncthreads();  // the window is rewritten next
    }
    if (staged) {
      __pipeline_commit();
      TPHASE();
      __pipeline_wait_prior(0);
    }
  }
  __syncthreads();
  if (a.theta != nullptr && staged) {
    // the fused SGD updates theta at the selected indices: start pulling
    // those sectors into L2 now, while the threshold is being resolved --
    // only for the candidates at or above the predicted T (the margin band
    // below it is mostly not selected; cold mode: all)
    const bool pz = s->g_key != 0 && !s->need_full_hist && s->spec_ok;
    const K zk0 = pz ? (K)s->z_key : (K)0;
    for (uint32_t j = threadIdx.x; j < cnt; j += blockDim.x)
      if (KO::key(st_val[j]) >= zk0) asm volatile("prefetch.global.L2 [%0];" ::"l"(a.theta + st_idx[j]));
  }
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
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        if (j0 + c < cnt) {
          v[c] = a.cand_val[lo + j0 + c];
          if (want_idx) id[c] = a.cand_idx[lo + j0 + c];
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
  auto level_pass = [&](uint32_t* g, uint32_t nbins, unsigned long long need, unsigned long long match,
                        auto digit_of, uint32_t* bin, unsigned long long* above,
                        unsigned long long* bcnt) {
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
        if (ok) atomicAdd(&sh_h[d], 1u);  // candidate keys spread over the bins: plain smem atomics
      }
    }
    __syncthreads();
    for (uint32_t b = threadIdx.x; b < nbins; b += blockDim.x) {
      const uint32_t h = sh_h[b];
      if (h) atomicAdd(&g[b], h);
    }
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
    // When the list is pass A's, k_scan already built this histogram while
    // compacting (no pass, no grid barrier here).
    if (pass == 0 && a.histd != nullptr) {
      resolve_level(a.histd, kCoarseBins, 1, k, sh_warp, &sh_res, sh_h);
      cb = sh_res.found ? sh_res.bin : 0u;
      above = sh_res.found ? sh_res.above : sh_res.total;
      bcnt = sh_res.found ? sh_res.cnt : C - sh_res.total;
    } else {
      level_pass(a.hlev + kHistCoarse * kLevelHist, kCoarseBins, k, C,
                 [&](K key, uint32_t* d) {
                   const K dl = (key - G) >> kCoarseShift;
                   *d = dl < (K)(kCoarseBins - 1) ? (uint32_t)dl : kCoarseBins - 1;
                   return *d != 0;
                 },
                 &cb, &above, &bcnt);
    }
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
  {
    // ---- early scatter: every entry whose key differs from T is decided
    // (key > T selected, key < T not); only ties at T wait for their
    // cross-CTA rank.  The theta read-modify-write and the residual fix-ups
    // -- the random-access part of the phase -- run before the count barrier
    // and the ordered write.  Batches of U entries per thread issue all their
    // theta loads before any store (the indices are distinct).
    constexpr int U = 8;
    for (uint32_t j0 = threadIdx.x; j0 < cnt; j0 += U * blockDim.x) {
      uint32_t id[U];
      T v[U], th[U];
      uint32_t selm = 0, actm = 0;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t j = j0 + u * blockDim.x;
        if (j < cnt) {
          v[u] = staged ? st_val[j] : a.cand_val[lo + j];
          const K key = KO::key(v[u]);
          if (key != T_key) {
            actm |= 1u << u;
            id[u] = staged ? st_idx[j] : a.cand_idx[lo + j];
            if (key > T_key) selm |= 1u << u;
          }
        }
      }
#ifdef PSB_DIAG_NO_THETA
      T* const theta_d = nullptr;  // diagnostics build: time the scatter without the theta RMW
#else
      T* const theta_d = a.theta;
#endif
      if (theta_d) {
#pragma unroll
        for (int u = 0; u < U; ++u)
#ifdef PSB_DIAG_THETA_NOLOAD
          th[u] = T(0);
#else
          if ((selm >> u) & 1u) th[u] = a.theta[id[u]];
#endif
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (!((actm >> u) & 1u)) continue;
        if ((selm >> u) & 1u) {
#ifndef PSB_DIAG_NO_RFIX
          if (a.r && !zeroed(v[u])) a.r[id[u]] = T(0);
#endif
          if (theta_d) {
            const T mean = mul_rn(v[u], T(1));  // P = 1: mean = v * (1/1)
            const T t2 = add_rn(mul_rn(a.coef, mean), th[u]);
            
#ifndef PSB_DIAG_THETA_NOSTORE
            a.theta[id[u]] = t2;
#endif

            if (a.mean_out) a.mean_out[id[u]] = mean;
            bad |= !is_finite(t2);
          }
        } else if (a.r && zeroed(v[u])) {
#ifndef PSB_DIAG_NO_RFIX
          a.r[id[u]] = v[u];  // unselected candidate: undo the speculative +0
#endif
        }
      }
    }
  }

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
  // every CTA has read the level histograms and the superblock sums: clear
  // them for the next call
  for (uint32_t b = blockIdx.x * blockDim.x + threadIdx.x; b < kNumLevelHists * kLevelHist;
       b += gridDim.x * blockDim.x)
    a.hlev[b] = 0;
  for (uint32_t b = blockIdx.x * blockDim.x + threadIdx.x; b < 3 * a.sb_stride; b += gridDim.x * blockDim.x)
    a.sb[b] = 0;
  if (a.histd != nullptr)
    for (uint32_t b = blockIdx.x * blockDim.x + threadIdx.x; b < kCoarseBins; b += gridDim.x * blockDim.x)
      a.histd[b] = 0;
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

  // ---- ordered write.  Staged slices: each thread walks its run in index
  // order (slot = gt_before + min(eq_before, need_eq)), records the slot
  // relative to the CTA's first one in shared memory and settles its ties;
  // then the CTA writes its contiguous payload range with coalesced stores.
  // Unstaged slices: 4 entries per thread per block scan, side effects inline.
  unsigned long long run = sh_base;  // (gt | eq << 32) before this slice
  if (staged) {
    const unsigned long long s_lo = (run & 0xffffffffull) + min(run >> 32, need_eq);
    unsigned long long before = run + my_ex;
    for (uint32_t j = r0; j < r1; ++j) {
      const T v = st_val[j];
      const K key = KO::key(v);
      const bool gt = key > T_key, eq = key == T_key;
      const unsigned long long gt_b = before & 0xffffffffull, eq_b = before >> 32;
      const bool sel = gt || (eq && eq_b < need_eq);
      st_slot[j] = sel ? (uint32_t)(gt_b + (eq_b < need_eq ? eq_b : need_eq) - s_lo) : kNoSlot;
      if (eq) scatter(st_idx[j], v, sel);
      before += (unsigned long long)gt | ((unsigned long long)eq << 32);
    }
    run += cta_total;
    __syncthreads();
    for (uint32_t j = threadIdx.x; j < cnt; j += blockDim.x) {
      const uint32_t sl = st_slot[j];
      if (sl != kNoSlot) {
        a.idx_out[s_lo + sl] = st_idx[j];
        a.val_out[s_lo + sl] = st_val[j];
      }
    }
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
      if (j0 + c < cnt && eq) scatter(id[c], v[c], sel);  // ties; the rest went in the early scatter
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
  if (bad) sh_bad = 1;
  if (a.npush) __threadfence_system();  // the pushes are visible before the peers are signalled
  __syncthreads();
  if (threadIdx.x == 0 && sh_bad) atomicOr(a.flags, 1u);
  phase();
}
