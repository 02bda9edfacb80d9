// psb_internal.cuh -- shared definitions for the sm_100a gradient-path kernels.
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>
#include <stdint.h>

#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "psb.h"

#define PSB_MAX_P 32          // payloads folded per apply (worker mask is u32)
#define PSB_HIST_BINS 4096    // widest radix digit (12 bits)
#define PSB_SCAN_THREADS 256  // K1 scan CTA size
#define PSB_ITEMS 16          // elements per thread per K1 tile (f32)
#define PSB_MAX_CTAS 2048  // max CTAs of the cooperative candidate phase

// ------------------------------------------------------------------ K1 state
// Per-call scratch of the top-k selection (reset by k_topk_begin every call).
struct TopkScratch {
  uint32_t done[8];         // last-block counters (one per kernel role)
  uint32_t b1;              // level-1 digit of the k-th largest key
  uint32_t need_full_hist;  // predicted candidate set missed -> full histogram pass
  uint32_t need_compact;    // candidates must be compacted by a separate pass
  uint32_t nonfinite;
  unsigned long long prefix;  // key digits resolved so far
  unsigned long long need;    // entries still to take inside `prefix`
  unsigned long long match;   // entries matching `prefix`
  unsigned long long n;
  unsigned long long k;
  unsigned long long cand_count;  // entries in the candidate list
  unsigned long long g_key;       // predicted key threshold used by this call (0 = none)
  uint32_t start_level;           // first radix level resolved over the candidates
  uint32_t spec_ok;               // predicted mode may pre-zero candidate residuals
  unsigned long long z_key;       // pass A pre-zeroes the residual of keys >= z_key (>= g_key)
  unsigned long long g_key2;      // second-chance threshold after a miss (< g_key; 0 = none)
  unsigned long long phase_ns[16];  // k_cand phase timestamps (globaltimer, CTA 0)
  uint32_t tile_ctr[4];             // dynamic tile counters of the scan passes (A, S, D, A2)
  uint32_t list_pass;               // scan pass whose tile segments hold the final list (0 A, 1 S, 2 D)
};

// K1 tiles per superblock: k_scan sums the tile counts per superblock so the
// candidate phase can locate its slice of the list without a grid barrier.
#define PSB_SB_SHIFT 6
// Coarse histogram of (key - G) >> PSB_COARSE_SHIFT over the predicted
// candidates (2048-ulp bins, the top one collecting an octave and more).
#define PSB_COARSE_BINS 4096
#define PSB_COARSE_SHIFT 11

// candidates / k band of the prediction-margin controller (psb_cand.inl)
#ifndef PSB_RATIO_LO
#define PSB_RATIO_LO 1.08
#endif
#ifndef PSB_RATIO_HI
#define PSB_RATIO_HI 2.0
#endif

// Per-worker persistent selection history: the next call's candidate set is
// {key >= key(T_prev * f)}; f adapts so the set stays a little above k.
struct TopkWorker {
  unsigned long long g_key;  // predicted key threshold for the next call (0 = none)
  unsigned long long t_prev; // threshold key T of the previous call
  float f;                   // margin factor (0 = uninitialised)
  float rho;                 // smoothed step-to-step drift of T (0 = uninitialised)
  uint32_t calls, misses;
  float last_ratio;          // candidates / k of the previous call
  uint32_t pad;
  unsigned long long z_key;  // predicted T without the safety margin (pre-zero boundary)
  float ratio_lo, ratio_hi;  // margin controller band on candidates / k (0 = defaults)
  float second_f;            // second-chance factor after a miss (0 = PSB_SECOND_F, < 0 = off)
  uint32_t pad2;
};

struct psb_ctx {
  int device = 0;
  int num_sms = 148;
  size_t max_n = 0, max_k = 0;
  int max_workers = 1;
  std::string err;
  uint64_t launches = 0;
  // comm
  ncclComm_t comm = nullptr;
  int rank = 0, nranks = 1;
  // flags
  uint32_t* d_flags = nullptr;  // [0] nonfinite
  // K1 scratch
  TopkScratch* d_tk = nullptr;
  TopkWorker* d_tw = nullptr;
  uint32_t* d_hist1 = nullptr;   // level-1 histogram
  uint32_t* d_histr = nullptr;   // refine-level histogram
  uint32_t* d_histd = nullptr;   // (key - G) histogram of the predicted mode
  uint32_t* d_tile_cnt = nullptr;          // candidates per K1 tile (segment) of the scan passes
  uint32_t* d_sb = nullptr;                // [3][sb_stride] superblock sums of the tile counts (passes A, S, D)
  uint32_t sb_stride = 0;
  unsigned long long* d_cta = nullptr;    // per-CTA totals / prefixes
  uint32_t* d_stage_idx = nullptr;  // tile-segmented candidates written by k_scan, capacity max_n
  uint32_t* d_list_idx = nullptr;   // the same, contiguous (k_cand's prologue), capacity max_n
  void* d_list_val = nullptr;
  void* d_stage_val = nullptr;      // f64 capacity
  size_t stage_val_bytes = 0;
  // apply scratch
  uint32_t* d_seg_off = nullptr;  // [max_workers][nseg_max + 1]
  size_t seg_cap = 0;
  // onebit / q8 scratch
  double* d_partials = nullptr;
  size_t partials_cap = 0;
  // exchange buffers (payload gather, q8 shards)
  void* d_gather = nullptr;
  size_t gather_bytes = 0;
  void* d_work = nullptr;  // generic workspace
  size_t work_bytes = 0;
  float* d_qmean = nullptr;
  void* d_mom_mean = nullptr;  // momentum: the step's dense mean
  size_t mom_bytes = 0;
  // kernel timing (psb_profile_*)
  int prof = 0;
  int predict = 1;  // K1 threshold prediction (PSB_NO_PREDICT=1 disables)
  uint32_t apply_vcap = 2048;  // PSB_APPLY_VCAP: staged entries per apply segment
  bool q8_no_pipe = false;       // PSB_Q8_NO_PIPE: the generic q8 reduce only (A/B)
  bool q8_scales_inplace = false;  // PSB_Q8_SCALES_INPLACE: the TMA apply reads remote mean scales in place
  bool q8_direct_apply = false;  // PSB_Q8_DIRECT_APPLY: the q8 apply reads the peers' mean shards in place
  bool apply_no_tma = false;   // PSB_APPLY_NO_TMA: thread-loaded apply entries (A/B)
  // PSB_APPLY_TMA_CAP: entries per TMA stage; 1792 fits a cfg2 segment (at
  // most 1759 entries at P = 2..8) and 4 CTAs per SM
  uint32_t apply_tma_cap = 1792;
  uint32_t apply_light = 32;
  // PSB_DENSE_FOLD_PCT: P payloads with P*k >= pct % of n fold by streaming
  // (k_dense_fold_apply) instead of the bitmap apply (0: off)
  uint32_t dense_fold_pct = 20;  // PSB_APPLY_LIGHT: segments of <= this many entries go one warp each (0: off)
  int q8_no_tma = 0;   // PSB_Q8_NO_TMA=1: register double-buffer kernel for the one-worker q8 step
  int q8_unfused = 0;  // PSB_Q8_UNFUSED=1: single-rank q8 step as quant + reduce (diagnostics)
  // NVLink peer exchange (psb_peer.cu)
  int peer_mode = 1;            // use it when nranks > 1 (PSB_NO_PEER=1 / psb_peer_mode(0): NCCL all-gather)
  void* peer_arena = nullptr;   // own arena: 4 KB flag header + payload slots
  size_t peer_bytes = 0;        // payload capacity of the arenas
  void* peer_base[PSB_MAX_P] = {};  // every rank's arena mapped here (own included)
  int shard_mode = 0;           // sharded multi-rank sparse apply (psb_peer_mode 2 / PSB_SHARD=1)
  int push_mode = 0;            // full exchange: K1 pushes its payload to the peers (psb_peer_mode 3)
  int direct_mode = 2;          // the apply reads the peers' arenas in place: 1 always (psb_peer_mode 4),
                                // 2 auto for top-k f32/f64 (psb_peer_mode 5, the default)
  int no_wire16 = 0;            // PSB_NO_WIRE16=1: 32-bit indices on the NVLink exchange
  // set by the step driver around one worker's K1 call in push mode: the
  // peers' payload-region bases and this worker's slot offset in them
  int push_n = 0;
  uint8_t* push_base[PSB_MAX_P] = {};
  size_t push_slot_off = 0;
  int push_wait = 0;            // K1 waits for the peers' acknowledgement before its write phase
  int no_stage = 0; // PSB_NO_STAGE=1: k_cand reads the list from global memory (diagnostics)
  int cand_smem[2] = {0, 0};  // dynamic shared memory of the cooperative k_cand (f32, f64)
  // bounded-staleness pipeline of psb_async_round (psb_async_pipeline): the
  // exchange + apply of round r runs on apply_st, gated by comp_ev[r % 2],
  // while round r+1 compresses on the caller's stream into the other payload
  // slot (pipe_pl[(r+1) % 2], reused once apply_ev of round r-1 fired)
  int async_pipe = 0;
  cudaStream_t apply_st = nullptr;
  cudaEvent_t comp_ev[2] = {nullptr, nullptr}, apply_ev[2] = {nullptr, nullptr};
  bool apply_pending[2] = {false, false};
  uint64_t pipe_round = 0;
  void* pipe_pl[2] = {nullptr, nullptr};
  size_t pipe_bytes = 0;
  std::vector<cudaEvent_t> prof_ev;  // pairs (start, stop)
  size_t prof_used = 0;
  // psb_profile_read_phase: event pairs around the exchange (1) and the
  // P-payload apply (2) of the steps, recorded while profiling is enabled
  std::vector<cudaEvent_t> prof_ph_ev[3];
  size_t prof_ph_used[3] = {0, 0, 0};
  // step milestones (PSB_STEP_MARKS=1, eager diagnostics: psb_debug_marks)
  int marks_on = 0;
  std::vector<cudaEvent_t> mark_ev;
  size_t marks_used = 0;
};

// Records the next step milestone event (no-op unless PSB_STEP_MARKS=1).
void psb_mark(psb_ctx* c, cudaStream_t st);

// NVLink peer exchange (psb_peer.cu)
// single-worker top-k momentum step straight from the payload; psb_apply.cu
psb_status psb_momentum_topk1(psb_ctx* c, psb_dtype dt, const uint8_t* payload, size_t k, void* m, void* theta,
                              void* mean_out, double beta, double lr, size_t n, uint32_t* starts_buf,
                              cudaStream_t st);
psb_status psb_peer_ensure(psb_ctx* c, size_t payload_bytes, cudaStream_t st);
uint8_t* psb_peer_payload(psb_ctx* c);
psb_status psb_peer_wait_ack(psb_ctx* c, cudaStream_t st);
psb_status psb_peer_exchange(psb_ctx* c, size_t bytes_per_rank, size_t tab_off, size_t tab_words_per_rank,
                             cudaStream_t st);
void psb_peer_destroy(psb_ctx* c);
uint32_t* psb_peer_list_cnt(psb_ctx* c);
void psb_peer_regions(psb_ctx* c, const uint8_t** out);  // every rank's payload region (mapped)
psb_status psb_peer_signal(psb_ctx* c, cudaStream_t st);
psb_status psb_peer_wait_ready(psb_ctx* c, cudaStream_t st);
psb_status psb_peer_put(psb_ctx* c, size_t off, size_t words, cudaStream_t st);
psb_status psb_peer_ack(psb_ctx* c, cudaStream_t st);
void psb_peer_push_targets(psb_ctx* c, size_t slot_off);  // fills push_n / push_base / push_slot_off
psb_status psb_shard_pull(psb_ctx* c, psb_dtype dt, int W, int q8, size_t blk, size_t voff, size_t soff,
                          size_t tab_off, uint32_t nseg, uint32_t* range, uint32_t* sidx, void* sval,
                          uint32_t* srow, size_t max_entries, cudaStream_t st);
psb_status psb_shard_finish(psb_ctx* c, psb_dtype dt, size_t list_off, size_t list_voff, void* theta,
                            size_t max_entries, cudaStream_t st);
// sparse apply pieces (psb_apply.cu)
psb_status psb_seg_offsets(psb_ctx* c, psb_compressor comp, psb_dtype dt, int nw, const void* payloads, size_t k,
                           uint32_t nseg, int seg_shift, uint32_t* rows, cudaStream_t st, void* out16 = nullptr,
                           size_t out_stride = 0);
// P-worker sparse apply with the per-segment offset rows already computed
// (tab: [P][nseg+1] for segments of 2^psb_apply_seg_shift(P); nullptr: compute them)
psb_status psb_sparse_apply_tab(psb_ctx* c, psb_compressor comp, psb_dtype dt, int P, const void* payloads, size_t k,
                                const uint32_t* tab, psb_order order, const psb_topology* topo, double lr,
                                const double* wscale, int async_mode, void* theta, size_t n, void* mean_out,
                                cudaStream_t st);
// wire16 payloads: (u16 in-segment index | val) blocks for the NVLink exchange
size_t psb_wire16_bytes(psb_dtype dt, size_t k);
psb_status psb_sparse_apply_wire16(psb_ctx* c, psb_dtype dt, int P, const void* payloads, size_t k,
                                   const uint32_t* tab, psb_order order, const psb_topology* topo, double lr,
                                   const double* wscale, int async_mode, void* theta, size_t n, void* mean_out,
                                   cudaStream_t st);
psb_status psb_sparse_apply_direct(psb_ctx* c, psb_compressor comp, psb_dtype dt, int P, int W,
                                   const uint8_t* const* rank_region, size_t k, size_t tab_off, psb_order order,
                                   const psb_topology* topo, double lr, const double* wscale, int async_mode,
                                   void* theta, size_t n, void* mean_out, cudaStream_t st, bool wire16);
psb_status psb_shard_fold(psb_ctx* c, psb_dtype dt, int P, const uint32_t* sidx, const void* sval,
                          const uint32_t* srow, const uint32_t* range, int seg_shift, psb_order order,
                          const psb_topology* topo, double lr, const double* wscale, int async_mode, void* theta,
                          size_t n, uint32_t* list_idx, void* list_val, uint32_t* list_cnt, cudaStream_t st);

// Segment size of the P-worker sparse apply: P bitmaps of S bits (x2 with the
// word ranks) within 16 KB of shared memory, 2^10 <= S <= 2^15.
#ifndef PSB_APPLY_BM_BYTES
#define PSB_APPLY_BM_BYTES (16 * 1024)
#endif
static inline int psb_apply_seg_shift(int P) {
  int s = 15;
  while (s > 10 && ((size_t)P * 8) << (s - 5) > PSB_APPLY_BM_BYTES) --s;
  return s;
}

// Segment list of psb_peer_gather: bytes at (rank's payload region + src_off)
// copied to (own payload region + dst_off).
struct PeerSeg {
  int rank;
  size_t src_off, dst_off, bytes;
};
struct PeerSegs {
  PeerSeg s[2 * PSB_MAX_P + 2];
  int n;
};
psb_status psb_peer_gather(psb_ctx* c, const PeerSegs& segs, cudaStream_t st);

// Dense q8 all-reduce views.  Q8Workers: worker q's int8 codes of global
// element e at codes[q][e - e_base] and its block scales at scales[q][blk -
// blk_lo] (local buffers, or the peers' NVLink-mapped arenas).  Q8Shards: the
// requantized mean of element e at codes[rank][e] / scales[rank][e / B] with
// rank = (e / B) / nbs -- the rank that reduced that block shard.
struct Q8Workers {
  const int8_t* codes[PSB_MAX_P];
  const float* scales[PSB_MAX_P];
};
struct Q8Shards {
  const int8_t* codes[PSB_MAX_P];
  const float* scales[PSB_MAX_P];
  size_t nbs;  // blocks per shard (SIZE_MAX: one shard)
};

// Record a profiling event pair around the dominant kernel (no-op unless enabled).
cudaEvent_t psb_prof_event(psb_ctx* c);
// Record one event of phase 1 (exchange) / 2 (apply) on st when profiling.
void psb_prof_mark(psb_ctx* c, int phase, cudaStream_t st);

// ------------------------------------------------------------------- helpers
psb_status psb_set_err(psb_ctx* c, psb_status s, const std::string& msg);
psb_status psb_cuda_err(psb_ctx* c, cudaError_t e, const char* where);

#define PSB_REQUIRE(ctx, cond, msg)                                      \
  do {                                                                   \
    if (!(cond)) return psb_set_err((ctx), PSB_EINVAL, (msg));           \
  } while (0)

#define PSB_LAUNCH_CHECK(ctx, where)                                     \
  do {                                                                   \
    cudaError_t e_ = cudaGetLastError();                                 \
    if (e_ != cudaSuccess) return psb_cuda_err((ctx), e_, (where));      \
  } while (0)

#define CUDA_TRY(c, expr, where)                                  \
  do {                                                            \
    cudaError_t e__ = (expr);                                     \
    if (e__ != cudaSuccess) return psb_cuda_err((c), e__, where); \
  } while (0)

#define NCCL_TRY(c, expr, where)                                                        \
  do {                                                                                  \
    ncclResult_t r__ = (expr);                                                          \
    if (r__ != ncclSuccess)                                                             \
      return psb_set_err((c), PSB_ENCCL, std::string(where) + ": " + ncclGetErrorString(r__)); \
  } while (0)

// ---- 1-D TMA bulk copies into shared memory, completion on an mbarrier
static __device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
static __device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
static __device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
static __device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
static __device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

static inline size_t psb_align16(size_t b) { return (b + 15) & ~(size_t)15; }
static __device__ __forceinline__ size_t psb_align16_d(size_t b) { return (b + 15) & ~(size_t)15; }

// Key of |x|: the magnitude bits, monotone in |x| for finite values and +-0
// (SURVEY.md parity fact 1).
template <class T>
struct KeyOf;
template <>
struct KeyOf<float> {
  typedef uint32_t K;
  static constexpr int kLevels = 3;
  __device__ __forceinline__ static K key(float x) { return __float_as_uint(x) & 0x7fffffffu; }
  __host__ __device__ static constexpr int shift(int l) { return l == 0 ? 19 : (l == 1 ? 8 : 0); }
  __host__ __device__ static constexpr int width(int l) { return l == 0 ? 12 : (l == 1 ? 11 : 8); }
  static constexpr K kInf = 0x7f800000u;
};
template <>
struct KeyOf<double> {
  typedef unsigned long long K;
  static constexpr int kLevels = 6;
  __device__ __forceinline__ static K key(double x) {
    return (unsigned long long)__double_as_longlong(x) & 0x7fffffffffffffffULL;
  }
  __host__ __device__ static constexpr int shift(int l) {
    return l == 0 ? 51 : (l == 1 ? 39 : (l == 2 ? 27 : (l == 3 ? 15 : (l == 4 ? 3 : 0))));
  }
  __host__ __device__ static constexpr int width(int l) { return l == 5 ? 3 : 12; }
  static constexpr K kInf = 0x7ff0000000000000ULL;
};

// IEEE round-to-nearest arithmetic without contraction, per type.
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float sub_rn(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ bool is_finite(float x) {
  return (__float_as_uint(x) & 0x7f800000u) != 0x7f800000u;
}
__device__ __forceinline__ bool is_finite(double x) {
  return ((unsigned long long)__double_as_longlong(x) & 0x7ff0000000000000ULL) !=
         0x7ff0000000000000ULL;
}

// Block-wide exclusive scan of u64 over PSB_SCAN_THREADS threads.  Returns the
// exclusive prefix; *total receives the block total.
__device__ __forceinline__ unsigned long long block_exscan_u64(unsigned long long v,
                                                              unsigned long long* sh_warp,
                                                              unsigned long long* total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  unsigned long long x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sh_warp[wid] = x;
  __syncthreads();
  const int nw = blockDim.x >> 5;
  if (wid == 0) {
    unsigned long long w = lane < nw ? sh_warp[lane] : 0ull;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      unsigned long long y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < nw) sh_warp[lane] = w;  // inclusive warp-total prefix
  }
  __syncthreads();
  unsigned long long warp_excl = wid ? sh_warp[wid - 1] : 0ull;
  *total = sh_warp[nw - 1];
  unsigned long long r = warp_excl + x - v;
  __syncthreads();
  return r;
}

// Launch helpers defined in the .cu files.
// K1 with the single-worker SGD update fused into its final write (theta,
// lr, mean_out nullable): theta[idx] = (-lr) * (val * 1) + theta[idx].
psb_status psb_topk_run_fused(psb_ctx* c, psb_dtype dt, int worker, const void* g, void* r,
                              size_t n, size_t k, uint32_t* idx_out, void* val_out, void* theta,
                              double lr, void* mean_out, cudaStream_t st);
psb_status psb_topk_run(psb_ctx* c, psb_dtype dt, int worker, const void* g, void* r, size_t n,
                        size_t k, uint32_t* idx_out, void* val_out, cudaStream_t st);
psb_status psb_topk_q8_fix(psb_ctx* c, const float* r_unused, size_t k, const uint32_t* idx,
                           const float* vals, float* r, int8_t* codes, float* scales,
                           cudaStream_t st);
