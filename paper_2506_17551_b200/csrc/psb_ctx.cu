// psb_ctx.cu -- context, communicator, argument checks and step drivers.
//
// Step drivers replace the reference's data-parallel step functions:
//   psb_sync_step   <- sync_data_parallel_step  parsim/strategies.hpp:86-121
//   psb_async_round <- async branch of train     parsim/trainer.hpp:244-255
//                      (+ async_step             parsim/strategies.hpp:125-129)
// P = W local virtual workers x R ranks (one process per GPU, NCCL over
// NVLink/NVSwitch).  Worker id = rank*W + w, so the reference's canonical
// worker order is preserved across ranks.
#include <cstdio>
#include <cstring>
#include <vector>

#include <cmath>

#include "psb_internal.cuh"
#include "psb_debug.h"

psb_status psb_q8_quant_launch(psb_ctx* c, const float* x, float* r, size_t n, uint32_t B,
                               int8_t* codes, float* scales, cudaStream_t st);
psb_status psb_q8_reduce_launch(psb_ctx* c, const Q8Workers& wv, int P, size_t blk_lo,
                                size_t blk_hi, size_t n, uint32_t B, psb_order order, uint32_t dpn,
                                uint32_t npr, int8_t* mcodes, float* mscales, double lr,
                                float* theta, float* mean_out, cudaStream_t st);
psb_status psb_q8_step1_launch(psb_ctx* c, const float* g, size_t gstride, float* r, size_t rstride,
                               int P, size_t n, uint32_t B, psb_order order, uint32_t dpn, uint32_t npr,
                               double lr, float* theta, float* mean_out, cudaStream_t st);
psb_status psb_q8_apply_tma_launch(psb_ctx* c, const Q8Shards& ms, const float* scales, size_t n, uint32_t B,
                                   double lr, float* theta, cudaStream_t st);
long long psb_q8_reduce_tma_launch(psb_ctx* c, const Q8Workers& wv, int P, size_t blk_lo, size_t blk_hi, uint32_t B,
                                   int8_t* mcodes, float* mscales, cudaStream_t st);
psb_status psb_q8_apply_launch(psb_ctx* c, const Q8Shards& ms, int R, size_t n, uint32_t B, double lr,
                               float* theta, float* mean_out, cudaStream_t st);

psb_status psb_set_err(psb_ctx* c, psb_status s, const std::string& msg) {
  if (c) c->err = msg;
  return s;
}

psb_status psb_cuda_err(psb_ctx* c, cudaError_t e, const char* where) {
  if (c) c->err = std::string(where) + ": " + cudaGetErrorString(e);
  return PSB_ECUDA;
}


extern "C" int psb_abi_version(void) { return PSB_ABI_VERSION; }

extern "C" const char* psb_status_string(psb_status s) {
  switch (s) {
    case PSB_OK: return "ok";
    case PSB_EINVAL: return "invalid argument";
    case PSB_ENONFINITE: return "non-finite entry";
    case PSB_ECUDA: return "cuda error";
    case PSB_ENCCL: return "nccl error";
    case PSB_ENOMEM: return "out of device memory";
    case PSB_ESTATE: return "invalid ctx state";
  }
  return "unknown";
}

extern "C" size_t psb_payload_bytes(psb_compressor c, psb_dtype dt, size_t k) {
  if (c == PSB_COMP_TOPK) return psb_align16(k * 4) + psb_align16(k * (dt == PSB_F64 ? 8 : 4));
  if (c == PSB_COMP_TOPK_Q8) return psb_align16(k * 4) + psb_align16(k) + psb_align16(((k + 127) / 128) * 4);
  return 0;
}

static size_t tile_f64() { return (size_t)PSB_SCAN_THREADS * 4 * 2; }

extern "C" psb_status psb_ctx_create(psb_ctx** out, int device, size_t max_n, size_t max_k,
                                     int max_workers) {
  if (!out) return PSB_EINVAL;
  *out = nullptr;
  if (max_n < 1 || max_n >= (1ull << 32) || max_k > max_n || max_workers < 1 ||
      max_workers > PSB_MAX_P)
    return PSB_EINVAL;
  psb_ctx* c = new psb_ctx();
  c->device = device;
  c->max_n = max_n;
  c->max_k = max_k < 1 ? 1 : max_k;
  c->max_workers = max_workers;
  if (const char* np = getenv("PSB_NO_PREDICT")) c->predict = np[0] == '0';
  if (const char* ns = getenv("PSB_NO_STAGE")) c->no_stage = ns[0] != '0';
  if (const char* np = getenv("PSB_NO_PEER")) c->peer_mode = np[0] == '0';
  if (const char* sh = getenv("PSB_SHARD")) c->shard_mode = sh[0] != '0';
  if (const char* nw = getenv("PSB_NO_WIRE16")) c->no_wire16 = nw[0] != '0';
  if (const char* pm = getenv("PSB_PEER_MODE")) {  // 0 nccl, 1 pull, 2 shard, 3 push, 4 direct, 5 auto
    const int m = atoi(pm);
    c->peer_mode = m > 0;
    c->shard_mode = m == 2;
    c->push_mode = m == 3;
    c->direct_mode = m == 4 ? 1 : m == 5 ? 2 : 0;
  }
  if (const char* sm = getenv("PSB_STEP_MARKS")) c->marks_on = sm[0] != '0';
  if (const char* qt = getenv("PSB_Q8_NO_TMA")) c->q8_no_tma = qt[0] != '0';
  if (const char* qu = getenv("PSB_Q8_UNFUSED")) c->q8_unfused = qu[0] != '0';
  if (const char* qp = getenv("PSB_Q8_NO_PIPE")) c->q8_no_pipe = qp[0] != '0';
  if (const char* qs = getenv("PSB_Q8_SCALES_INPLACE")) c->q8_scales_inplace = qs[0] != '0';
  if (const char* qd = getenv("PSB_Q8_DIRECT_APPLY")) c->q8_direct_apply = qd[0] != '0';
  if (const char* nt = getenv("PSB_APPLY_NO_TMA")) c->apply_no_tma = nt[0] != '0';
  if (const char* df = getenv("PSB_DENSE_FOLD_PCT")) c->dense_fold_pct = (uint32_t)std::max(0l, atol(df));
  if (const char* al = getenv("PSB_APPLY_LIGHT")) c->apply_light = (uint32_t)std::min(32l, std::max(0l, atol(al)));
  if (const char* tc = getenv("PSB_APPLY_TMA_CAP"))
    c->apply_tma_cap = (uint32_t)std::min(8192l, std::max(64l, atol(tc)));
  if (const char* vc = getenv("PSB_APPLY_VCAP")) c->apply_vcap = (uint32_t)std::min(16384l, std::max(0l, atol(vc))) & ~1u;
  auto fail = [&](cudaError_t e) {
    psb_ctx_destroy(c);
    return e == cudaErrorMemoryAllocation ? PSB_ENOMEM : PSB_ECUDA;
  };
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return fail(e);
  cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device);
  // f32 tiles are 4096 elements, f64 tiles 2048: size for the larger count.
  const size_t ntiles = (max_n + tile_f64() - 1) / tile_f64() + 1;
  const size_t stage_cap = ntiles * tile_f64();
#define ALLOC(ptr, bytes)                                   \
  do {                                                      \
    e = cudaMalloc((void**)&(ptr), (bytes));                \
    if (e != cudaSuccess) return fail(e);                   \
    e = cudaMemset((ptr), 0, (bytes));                      \
    if (e != cudaSuccess) return fail(e);                   \
  } while (0)
  ALLOC(c->d_flags, 64);
  ALLOC(c->d_tk, sizeof(TopkScratch));
  ALLOC(c->d_tw, sizeof(TopkWorker) * max_workers);
  ALLOC(c->d_hist1, sizeof(uint32_t) * PSB_HIST_BINS);
  ALLOC(c->d_histr, sizeof(uint32_t) * PSB_HIST_BINS * 10);  // k_cand level histograms
  ALLOC(c->d_histd, sizeof(uint32_t) * 16384);
  ALLOC(c->d_tile_cnt, sizeof(uint32_t) * ntiles);
  c->sb_stride = (uint32_t)((ntiles >> PSB_SB_SHIFT) + 1);
  ALLOC(c->d_sb, sizeof(uint32_t) * 3 * c->sb_stride);
  ALLOC(c->d_cta, sizeof(unsigned long long) * 2 * PSB_MAX_CTAS);  // (gt, eq) totals | tile-chunk sums
  ALLOC(c->d_stage_idx, sizeof(uint32_t) * stage_cap);
  c->stage_val_bytes = sizeof(double) * stage_cap;
  ALLOC(c->d_stage_val, c->stage_val_bytes);
  ALLOC(c->d_list_idx, sizeof(uint32_t) * stage_cap);
  ALLOC(c->d_list_val, c->stage_val_bytes);
  // segment table: smallest segment is 64 entries (P*S*8 + 4S <= 96 KB, P <= 32)
  c->seg_cap = (size_t)max_workers * (max_n / 64 + 2);
  ALLOC(c->d_seg_off, sizeof(uint32_t) * c->seg_cap);
  c->partials_cap = (size_t)c->num_sms * 4 + 64;
  ALLOC(c->d_partials, sizeof(double) * (c->partials_cap + 1));
#undef ALLOC
  {  // K1 prediction tuning: PSB_RATIO_BAND="lo,hi" (controller band), PSB_SECOND_F (miss second chance)
    float lo = 0.f, hi = 0.f, f2 = 0.f;
    const char* rl = getenv("PSB_RATIO_BAND");
    const char* sf = getenv("PSB_SECOND_F");
    const bool band = rl && sscanf(rl, "%f,%f", &lo, &hi) == 2 && lo > 0.f && hi > lo;
    const bool second = sf && sscanf(sf, "%f", &f2) == 1 && f2 < 1.f;
    if (band || second) {
      std::vector<TopkWorker> tw(max_workers);
      memset(tw.data(), 0, sizeof(TopkWorker) * max_workers);
      for (auto& w : tw) {
        if (band) w.ratio_lo = lo, w.ratio_hi = hi;
        if (second) w.second_f = f2 > 0.f ? f2 : -1.f;
      }
      e = cudaMemcpy(c->d_tw, tw.data(), sizeof(TopkWorker) * max_workers, cudaMemcpyHostToDevice);
      if (e != cudaSuccess) return fail(e);
    }
  }
  *out = c;
  return PSB_OK;
}

extern "C" void psb_ctx_destroy(psb_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  cudaDeviceSynchronize();
  psb_peer_destroy(c);
  for (int i = 0; i < 2; ++i) {
    if (c->comp_ev[i]) cudaEventDestroy(c->comp_ev[i]);
    if (c->apply_ev[i]) cudaEventDestroy(c->apply_ev[i]);
    if (c->pipe_pl[i]) cudaFree(c->pipe_pl[i]);
  }
  if (c->apply_st) cudaStreamDestroy(c->apply_st);
  void* ptrs[] = {c->d_flags,    c->d_tk,        c->d_tw,        c->d_hist1,   c->d_histr,
                  c->d_tile_cnt, c->d_sb, c->d_cta, c->d_list_idx, c->d_list_val,       c->d_histd,       c->d_stage_idx, c->d_stage_val,
                  c->d_seg_off,  c->d_partials,  c->d_gather,    c->d_work,    c->d_qmean,   c->d_mom_mean};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  if (c->comm) ncclCommDestroy(c->comm);
  for (cudaEvent_t e : c->prof_ev) cudaEventDestroy(e);
  for (auto& v : c->prof_ph_ev)
    for (cudaEvent_t e : v) cudaEventDestroy(e);
  delete c;
}

void psb_mark(psb_ctx* c, cudaStream_t st) {
  if (!c->marks_on) return;
  if (c->marks_used == c->mark_ev.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    c->mark_ev.push_back(e);
  }
  cudaEventRecord(c->mark_ev[c->marks_used++], st);
}

// Milliseconds between consecutive milestones recorded since the last call.
extern "C" PSB_API int psb_debug_marks(psb_ctx* c, float* out, int max) {
  if (!c) return 0;
  cudaDeviceSynchronize();
  int m = 0;
  for (size_t i = 1; i < c->marks_used && m < max; ++i, ++m) cudaEventElapsedTime(out + m, c->mark_ev[i - 1], c->mark_ev[i]);
  c->marks_used = 0;
  return m;
}

cudaEvent_t psb_prof_event(psb_ctx* c) {
  if (c->prof_used == c->prof_ev.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    c->prof_ev.push_back(e);
  }
  return c->prof_ev[c->prof_used++];
}

void psb_prof_mark(psb_ctx* c, int phase, cudaStream_t st) {
  if (!c->prof || phase < 1 || phase > 2) return;
  auto& v = c->prof_ph_ev[phase];
  size_t& used = c->prof_ph_used[phase];
  if (used == v.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    v.push_back(e);
  }
  cudaEventRecord(v[used++], st);
}

extern "C" psb_status psb_profile_read_phase(psb_ctx* c, int phase, double* total_ms, uint64_t* pairs_out) {
  PSB_REQUIRE(c, c != nullptr && total_ms && pairs_out, "psb_profile_read_phase: null argument");
  PSB_REQUIRE(c, phase >= 0 && phase <= 2, "psb_profile_read_phase: phase must be 0, 1 or 2");
  if (phase == 0) return psb_profile_read(c, total_ms, pairs_out);
  auto& v = c->prof_ph_ev[phase];
  const size_t pairs = c->prof_ph_used[phase] / 2;
  double t = 0.0;
  for (size_t i = 0; i < pairs; ++i) {
    CUDA_TRY(c, cudaEventSynchronize(v[2 * i + 1]), "psb_profile_read_phase");
    float ms = 0.f;
    CUDA_TRY(c, cudaEventElapsedTime(&ms, v[2 * i], v[2 * i + 1]), "psb_profile_read_phase");
    t += ms;
  }
  *total_ms = t;
  *pairs_out = pairs;
  c->prof_ph_used[phase] = 0;
  return PSB_OK;
}

extern "C" psb_status psb_profile_enable(psb_ctx* c, int enable) {
  PSB_REQUIRE(c, c != nullptr, "null ctx");
  c->prof = enable ? 1 : 0;
  return PSB_OK;
}

extern "C" psb_status psb_profile_read(psb_ctx* c, double* total_ms, uint64_t* launches) {
  PSB_REQUIRE(c, c != nullptr && total_ms && launches, "psb_profile_read: null argument");
  double t = 0.0;
  const size_t pairs = c->prof_used / 2;
  for (size_t i = 0; i < pairs; ++i) {
    CUDA_TRY(c, cudaEventSynchronize(c->prof_ev[2 * i + 1]), "psb_profile_read");
    float ms = 0.f;
    CUDA_TRY(c, cudaEventElapsedTime(&ms, c->prof_ev[2 * i], c->prof_ev[2 * i + 1]), "psb_profile_read");
    t += ms;
  }
  *total_ms = t;
  *launches = pairs;
  c->prof_used = 0;
  return PSB_OK;
}

extern "C" const char* psb_last_error(const psb_ctx* c) { return c ? c->err.c_str() : "null ctx"; }

extern "C" uint64_t psb_launch_count(const psb_ctx* c) { return c ? c->launches : 0; }

extern "C" psb_status psb_check(psb_ctx* c, psb_stream_t stream) {
  if (!c) return PSB_EINVAL;
  CUDA_TRY(c, cudaStreamSynchronize((cudaStream_t)stream), "psb_check");
  if (c->apply_st) CUDA_TRY(c, cudaStreamSynchronize(c->apply_st), "psb_check (async apply stream)");
  uint32_t flags = 0;
  CUDA_TRY(c, cudaMemcpy(&flags, c->d_flags, sizeof(uint32_t), cudaMemcpyDeviceToHost), "psb_check");
  if (c->comm) {
    ncclResult_t ae = ncclSuccess;
    ncclCommGetAsyncError(c->comm, &ae);
    if (ae != ncclSuccess && ae != ncclInProgress)
      return psb_set_err(c, PSB_ENCCL, std::string("nccl async: ") + ncclGetErrorString(ae));
  }
  if (flags) {
    CUDA_TRY(c, cudaMemset(c->d_flags, 0, sizeof(uint32_t)), "psb_check");
    if (flags & 8u) return psb_set_err(c, PSB_ESTATE, "peer exchange: timed out waiting for a peer rank");
    if (flags & 16u) return psb_set_err(c, PSB_EINVAL, "wire_decode: truncated input");
    if (flags & 32u) return psb_set_err(c, PSB_EINVAL, "wire_decode: message exceeds the output capacity");
    if (flags & 64u) return psb_set_err(c, PSB_EINVAL, "wire_decode: index exceeds the 32-bit range");
    if (flags & 128u) return psb_set_err(c, PSB_EINVAL, "bpr_batch_gradient: triple index out of range");
    if (flags & 2u) return psb_set_err(c, PSB_EINVAL, "decompress: index out of range for dim");
    if (flags & 4u) return psb_set_err(c, PSB_EINVAL, "decompress: indices not strictly increasing");
    return psb_set_err(c, PSB_ENONFINITE, "ef_compress_step residual: non-finite entry");
  }
  return PSB_OK;
}

// -------------------------------------------------------------- communicator
extern "C" psb_status psb_comm_unique_id(void* uid_out) {
  if (!uid_out) return PSB_EINVAL;
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return PSB_ENCCL;
  std::memcpy(uid_out, &id, sizeof(id));
  return PSB_OK;
}

extern "C" psb_status psb_comm_init(psb_ctx* c, int rank, int nranks, const void* uid) {
  PSB_REQUIRE(c, c != nullptr, "null ctx");
  PSB_REQUIRE(c, nranks >= 1 && rank >= 0 && rank < nranks, "psb_comm_init: bad rank/size");
  c->rank = rank;
  c->nranks = nranks;
  if (nranks == 1) return PSB_OK;
  PSB_REQUIRE(c, uid != nullptr, "psb_comm_init: null unique id");
  ncclUniqueId id;
  std::memcpy(&id, uid, sizeof(id));
  CUDA_TRY(c, cudaSetDevice(c->device), "psb_comm_init");
  NCCL_TRY(c, ncclCommInitRank(&c->comm, nranks, id, rank), "ncclCommInitRank");
  return PSB_OK;
}

extern "C" int psb_comm_rank(const psb_ctx* c) { return c ? c->rank : -1; }
extern "C" int psb_comm_size(const psb_ctx* c) { return c ? c->nranks : -1; }

extern "C" psb_status psb_allgather(psb_ctx* c, void* buf, size_t bytes_per_rank, psb_stream_t stream) {
  PSB_REQUIRE(c, c != nullptr, "null ctx");
  if (c->nranks == 1) return PSB_OK;
  if (!c->comm) return psb_set_err(c, PSB_ESTATE, "psb_allgather: communicator not initialised");
  uint8_t* b = reinterpret_cast<uint8_t*>(buf);
  NCCL_TRY(c, ncclAllGather(b + (size_t)c->rank * bytes_per_rank, b, bytes_per_rank, ncclUint8, c->comm,
                            (cudaStream_t)stream),
           "ncclAllGather");
  return PSB_OK;
}

// ------------------------------------------------------------ compressors
static psb_status ensure(psb_ctx* c, void** p, size_t* have, size_t need, const char* what) {
  if (*have >= need) return PSB_OK;
  if (*p) cudaFree(*p);
  *p = nullptr;
  *have = 0;
  cudaError_t e = cudaMalloc(p, need);
  if (e != cudaSuccess) return psb_set_err(c, PSB_ENOMEM, std::string(what) + ": out of device memory");
  *have = need;
  return PSB_OK;
}

extern "C" psb_status psb_ef_topk(psb_ctx* c, psb_dtype dt, int worker, const void* g, void* r,
                                  size_t n, size_t k, uint32_t* idx_out, void* val_out,
                                  psb_stream_t stream) {
  PSB_REQUIRE(c, c != nullptr, "null ctx");
  PSB_REQUIRE(c, dt == PSB_F32 || dt == PSB_F64, "psb_ef_topk: bad dtype");
  PSB_REQUIRE(c, k >= 1 && k <= n,
              "compress_topk: k out of range (k=" + std::to_string(k) + ", dim=" + std::to_string(n) + ")");
  PSB_REQUIRE(c, n <= c->max_n, "ef_compress_step: n exceeds ctx max_n");
  PSB_REQUIRE(c, worker >= 0 && worker < c->max_workers, "psb_ef_topk: worker out of range");
  PSB_REQUIRE(c, g && idx_out && val_out, "psb_ef_topk: null pointer");
  return psb_topk_run(c, dt, worker, g, r, n, k, idx_out, val_out, (cudaStream_t)stream);
}

extern "C" psb_status psb_ef_topk_q8(psb_ctx* c, int worker, const float* g, float* r, size_t n,
                                     size_t k, uint32_t* idx_out, int8_t* codes_out,
                                     float* scales_out, psb_stream_t stream) {
  PSB_REQUIRE(c, c != nullptr, "null ctx");
  PSB_REQUIRE(c, k >= 1 && k <= n,
              "compress_topk: k out of range (k=" + std::to_string(k) + ", dim=" + std::to_string(n) + ")");
  PSB_REQUIRE(c, n <= c->max_n && k <= c->max_k, "psb_ef_topk_q8: size exceeds ctx capacity");
  PSB_REQUIRE(c, g && idx_out && codes_out && scales_out, "psb_ef_topk_q8: null pointer");
  psb_status s = ensure(c, &c->d_work, &c->work_bytes, sizeof(float) * c->max_k, "topk_q8 values");
  if (s) return s;
  float* vals = reinterpret_cast<float*>(c->d_work);
  s = psb_topk_run(c, PSB_F32, worker, g, r, n, k, idx_out, vals, (cudaStream_t)stream);
  if (s) return s;
  return psb_topk_q8_fix(c, nullptr, k, idx_out, vals, r, codes_out, scales_out, (cudaStream_t)stream);
}

// --------------------------------------------------------------- drivers
static psb_status check_desc(psb_ctx* c, const psb_step_desc* d) {
  PSB_REQUIRE(c, c != nullptr, "null ctx");
  PSB_REQUIRE(c, d != nullptr, "null step descriptor");
  PSB_REQUIRE(c, d->workers >= 1, "WorkerGroup: no workers");
  PSB_REQUIRE(c, (size_t)d->workers * c->nranks <= (size_t)c->max_workers,
              "sync_data_parallel_step: P exceeds ctx max_workers");
  PSB_REQUIRE(c, d->n >= 1 && d->n <= c->max_n, "sync_data_parallel_step: n out of range for ctx");
  // any finite rate, as sync_data_parallel_step itself (strategies.hpp:86-113;
  // HyperParams::validate is the caller's check).  lr < 0 differs from the
  // reference's dense vec_axpy only in the sign of untouched -0 entries.
  PSB_REQUIRE(c, std::isfinite(d->lr), "sync_data_parallel_step: learning rate must be finite");
  PSB_REQUIRE(c, d->g && d->theta, "sync_data_parallel_step: null buffer");
  if (d->compressor == PSB_COMP_TOPK || d->compressor == PSB_COMP_TOPK_Q8) {
    PSB_REQUIRE(c, d->k >= 1 && d->k <= d->n,
                "compress_topk: k out of range (k=" + std::to_string(d->k) + ", dim=" + std::to_string(d->n) + ")");
    PSB_REQUIRE(c, d->k <= c->max_k, "sync_data_parallel_step: k exceeds ctx max_k");
  }
  if (d->compressor == PSB_COMP_TOPK_Q8 || d->compressor == PSB_COMP_Q8)
    PSB_REQUIRE(c, d->dtype == PSB_F32, "8-bit compressors are f32 only");
  if (d->topo.devices_per_node)
    PSB_REQUIRE(c, d->topo.racks >= 1 && d->topo.nodes_per_rack >= 1, "Topology: counts must be >= 1");
  return PSB_OK;
}

// Compress this rank's W workers into their payload slots of the gather
// buffer and exchange; on return the gather buffer holds all P payloads.
// fuse_apply (P == 1, sync, top-k): the SGD update of the single payload is
// done inside K1's final write (psb_topk_run_fused), no separate apply pass.
//
// Multi-rank over NVLink peer memory, two modes (psb_peer.cu):
//   full    -- every rank pulls all P payloads, then applies them all;
//   sharded -- (ShardPlan non-null on return .on) rank r folds only segments
//              [seg_lo, seg_hi) of the index space: the producer also writes
//              its payloads' per-segment offsets into its arena; shard_apply
//              pulls the matching slices, folds them into theta and an update
//              list, and applies the other ranks' lists.
struct ShardPlan {
  bool on = false;         // sharded apply
  bool tab_ready = false;  // full exchange: every worker's offset rows are in the arena
  bool ack_after_apply = false;  // push mode: acknowledge the peers' payloads once applied
  bool direct = false;           // direct mode: apply from the peers' arenas in place
  bool wire16 = false;           // the arena holds wire16 payloads (u16 in-segment indices)
  int seg_shift = 0;
  uint32_t nseg = 0;
  size_t blk = 0, tab_off = 0, list_off = 0, list_voff = 0, cap = 0;
};

static psb_status compress_and_gather(psb_ctx* c, const psb_step_desc* d, cudaStream_t st,
                                      uint8_t** payloads_out, bool fuse_apply = false,
                                      ShardPlan* plan = nullptr) {
  const int W = d->workers, P = W * c->nranks;
  const size_t es = d->dtype == PSB_F64 ? 8 : 4;
  const size_t blk = psb_payload_bytes(d->compressor, d->dtype, d->k);
  // multi-rank: payloads go straight into this rank's slots of its NVLink
  // peer arena (psb_peer.cu); single rank / PSB_NO_PEER: the gather buffer
  const bool peer = c->nranks > 1 && c->peer_mode;
  const bool shard = peer && plan != nullptr && c->shard_mode && d->mean_out == nullptr && d->theta && P >= 2;
  // full exchange pushed by K1 itself (top-k values; the q8 payload is finished after K1)
  const bool push = peer && !shard && c->push_mode && d->compressor == PSB_COMP_TOPK && plan != nullptr;
  // direct: the apply reads every peer's arena in place (no pull copy)
  // (auto, the default: direct for top-k f32/f64, whose apply stages the
  // remote entries by TMA; pull for top-k int8)
  const bool direct = peer && !shard && !push && plan != nullptr && P >= 2 &&
                      (c->direct_mode == 1 || (c->direct_mode == 2 && d->compressor == PSB_COMP_TOPK));
  // pull / direct mode, top-k f32/f64: the arena slots carry wire16 payloads
  // (u16 in-segment index | value: 6 instead of 8 bytes per entry on
  // NVLink); K1 writes the standard payload into local scratch and k_seg_offsets
  // converts
  const bool wire16 = peer && !shard && !push && plan != nullptr && P >= 2 &&
                      d->compressor == PSB_COMP_TOPK && !c->no_wire16;
  const size_t pblk = wire16 ? psb_wire16_bytes(d->dtype, d->k) : blk;  // arena slot stride
  psb_status s;
  uint8_t* gb;
  uint8_t* kb = nullptr;  // this rank's first K1 output slot (arena, or the wire16 scratch)
  if (peer) {
    auto al = [](size_t b) { return (b + 255) & ~(size_t)255; };
    size_t region = al(pblk * P);
    if (plan && P >= 2) {
      // per-segment offset rows of every worker's payload, computed by its
      // producer and exchanged with it (the consumer skips k_seg_offsets)
      ShardPlan& sp = *plan;
      sp.blk = blk;
      sp.seg_shift = psb_apply_seg_shift(P);
      sp.nseg = (uint32_t)((d->n + ((size_t)1 << sp.seg_shift) - 1) >> sp.seg_shift);
      sp.tab_off = region;
      region += al(sizeof(uint32_t) * P * (sp.nseg + 1));
    }
    if (shard) {
      ShardPlan& sp = *plan;
      sp.on = true;
      sp.cap = std::min((size_t)P * d->k, d->n);
      sp.list_off = region;
      region += al(sizeof(uint32_t) * sp.cap);
      sp.list_voff = region;
      region += al(es * sp.cap);
    }
    s = psb_peer_ensure(c, region, st);
    if (s) return s;
    gb = psb_peer_payload(c);
    psb_mark(c, st);
    if (!push) {
      s = psb_peer_wait_ack(c, st);  // peers done with our previous payloads / update list
      if (s) return s;
    }
    if (direct) plan->direct = true;
    psb_mark(c, st);
    kb = gb + (size_t)c->rank * W * blk;
    if (wire16) {
      s = ensure(c, &c->d_gather, &c->gather_bytes, blk * W, "wire16 scratch");
      if (s) return s;
      kb = reinterpret_cast<uint8_t*>(c->d_gather);
    }
  } else {
    s = ensure(c, &c->d_gather, &c->gather_bytes, blk * P, "payload gather buffer");
    if (s) return s;
    gb = reinterpret_cast<uint8_t*>(c->d_gather);
    kb = gb + (size_t)c->rank * W * blk;
  }
  for (int w = 0; w < W; ++w) {
    const int gid = c->rank * W + w;
    uint8_t* slot = kb + (size_t)w * blk;
    const void* g = reinterpret_cast<const uint8_t*>(d->g) + (size_t)w * d->n * es;
    void* r = d->r ? reinterpret_cast<uint8_t*>(d->r) + (size_t)w * d->n * es : nullptr;
    uint32_t* idx = reinterpret_cast<uint32_t*>(slot);
    if (push) {
      psb_peer_push_targets(c, (size_t)gid * blk);
      c->push_wait = w == 0;  // K1 waits for the peers' acknowledgement before its first push
    }
    if (d->compressor == PSB_COMP_TOPK) {
      if (fuse_apply)
        s = psb_topk_run_fused(c, d->dtype, w, g, r, d->n, d->k, idx, slot + psb_align16(d->k * 4),
                               d->theta, d->lr, d->mean_out, st);
      else
        s = psb_topk_run(c, d->dtype, w, g, r, d->n, d->k, idx, slot + psb_align16(d->k * 4), st);
    } else {
      int8_t* codes = reinterpret_cast<int8_t*>(slot + psb_align16(d->k * 4));
      float* scales = reinterpret_cast<float*>(slot + psb_align16(d->k * 4) + psb_align16(d->k));
      s = psb_ef_topk_q8(c, w, (const float*)g, (float*)r, d->n, d->k, idx, codes, scales,
                         (psb_stream_t)st);
    }
    c->push_n = 0;
    c->push_wait = 0;
    if (s) return s;
  }
  psb_mark(c, st);
  const bool tabs = peer && plan && P >= 2;
  if (tabs) {
    const ShardPlan& sp = *plan;
    uint32_t* tab = reinterpret_cast<uint32_t*>(gb + sp.tab_off) + (size_t)c->rank * W * (sp.nseg + 1);
    // the offset rows and (wire16) the arena payloads in one pass over K1's output
    s = psb_seg_offsets(c, d->compressor, d->dtype, W, kb, d->k, sp.nseg, sp.seg_shift, tab, st,
                        wire16 ? gb + (size_t)c->rank * W * pblk : nullptr, pblk);
    if (s) return s;
    if (wire16) plan->wire16 = true;
    psb_mark(c, st);
  }
  if (push) {
    // payloads are already in every peer's arena; push the offset rows, signal, wait
    const ShardPlan& sp = *plan;
    s = psb_peer_put(c, sp.tab_off + sizeof(uint32_t) * (size_t)c->rank * W * (sp.nseg + 1),
                     (size_t)W * (sp.nseg + 1), st);
    if (s) return s;
    s = psb_peer_signal(c, st);
    if (s) return s;
    s = psb_peer_wait_ready(c, st);
    if (s) return s;
    plan->tab_ready = true;
    plan->ack_after_apply = true;
    psb_mark(c, st);
  } else if (shard) {
    s = psb_peer_signal(c, st);
    if (s) return s;
    psb_mark(c, st);
  } else if (direct) {
    s = psb_peer_signal(c, st);
    if (s) return s;
    s = psb_peer_wait_ready(c, st);
    if (s) return s;
    plan->ack_after_apply = true;
    psb_mark(c, st);
  } else if (peer) {
    psb_prof_mark(c, 1, st);
    s = psb_peer_exchange(c, (size_t)W * pblk, tabs ? plan->tab_off : 0,
                          tabs ? (size_t)W * (plan->nseg + 1) : 0, st);
    psb_prof_mark(c, 1, st);
    if (s) return s;
    if (tabs) plan->tab_ready = true;
    psb_mark(c, st);
  } else if (c->nranks > 1) {
    if (!c->comm) return psb_set_err(c, PSB_ESTATE, "sync step: communicator not initialised");
    psb_prof_mark(c, 1, st);
    NCCL_TRY(c, ncclAllGather(gb + (size_t)c->rank * W * blk, gb, (size_t)W * blk, ncclUint8, c->comm, st),
             "ncclAllGather(payloads)");
    psb_prof_mark(c, 1, st);
  }
  *payloads_out = gb;
  return PSB_OK;
}

// Sharded apply after compress_and_gather (plan.on): pull this rank's slices,
// fold them (theta + update list), publish, apply the other ranks' lists.
static psb_status shard_apply(psb_ctx* c, const psb_step_desc* d, const ShardPlan& sp, const double* wscale,
                              bool async_mode, cudaStream_t st) {
  const int W = d->workers, P = W * c->nranks;
  const size_t es = d->dtype == PSB_F64 ? 8 : 4;
  // local scratch: flat slices (idx | val) of up to P*k entries, P rows of up
  // to nseg+1 offsets, the device-decided segment range
  auto al = [](size_t b) { return (b + 255) & ~(size_t)255; };
  const size_t cap = (size_t)P * d->k;
  const size_t o_val = al(sizeof(uint32_t) * cap);
  const size_t o_row = o_val + al(es * cap);
  const size_t o_rng = o_row + al(sizeof(uint32_t) * P * ((size_t)sp.nseg + 1));
  const size_t total = o_rng + 256;
  psb_status s = ensure(c, &c->d_gather, &c->gather_bytes, total, "shard scratch");
  if (s) return s;
  uint8_t* ws = reinterpret_cast<uint8_t*>(c->d_gather);
  uint32_t* sidx = reinterpret_cast<uint32_t*>(ws);
  void* sval = ws + o_val;
  uint32_t* srow = reinterpret_cast<uint32_t*>(ws + o_row);
  uint32_t* range = reinterpret_cast<uint32_t*>(ws + o_rng);
  const size_t voff = psb_align16(d->k * 4);
  const size_t soff = voff + psb_align16(d->k);
  s = psb_shard_pull(c, d->dtype, W, d->compressor == PSB_COMP_TOPK_Q8, sp.blk, voff, soff, sp.tab_off, sp.nseg,
                     range, sidx, sval, srow, (size_t)W * d->k, st);
  if (s) return s;
  psb_mark(c, st);
  uint8_t* region = psb_peer_payload(c);
  s = psb_shard_fold(c, d->dtype, P, sidx, sval, srow, range, sp.seg_shift, d->order, &d->topo, d->lr,
                     wscale, async_mode, d->theta, d->n, reinterpret_cast<uint32_t*>(region + sp.list_off),
                     region + sp.list_voff, psb_peer_list_cnt(c), st);
  if (s) return s;
  psb_mark(c, st);
  s = psb_shard_finish(c, d->dtype, sp.list_off, sp.list_voff, d->theta, sp.cap, st);
  psb_mark(c, st);
  return s;
}

// Dense q8 all-reduce across ranks over NVLink peer memory (the default for
// nranks > 1; psb_peer_mode 0 keeps the NCCL all-to-all + all-gather).  Each
// rank quantizes its W workers straight into its arena; after one flag round
// every rank reduces its block shard reading all P workers' codes and scales
// in place from the peers' arenas (the reduce-scatter is the reduce kernel's
// own NVLink loads), requantizes the mean into its arena; after a second flag
// round it applies SGD reading each block's mean from the rank that reduced it
// (the all-gather is the apply's own NVLink loads).  No staging copies; the
// fold order, requantization and update are those of the NCCL path.
static psb_status q8_step_nvlink(psb_ctx* c, const psb_step_desc* d, cudaStream_t st, size_t n_pad, size_t nbs,
                                 uint32_t dpn, uint32_t npr) {
  const int W = d->workers, R = c->nranks, P = W * R;
  const uint32_t B = d->q8_block ? d->q8_block : 256;
  const size_t n = d->n, nb = (n + B - 1) / B;
  const size_t shard = nbs * B;
  auto al = [](size_t b) { return (b + 255) & ~(size_t)255; };
  // arena: local codes [W][n_pad] | local scales [W][R*nbs] | mean codes [n_pad]
  //        | mean scales [R*nbs] | pulled codes [P][shard] | pulled scales [P][nbs]
  const size_t o_lc = 0;
  const size_t o_ls = o_lc + al((size_t)W * n_pad);
  const size_t o_mc = o_ls + al(sizeof(float) * W * R * nbs);
  const size_t o_ms = o_mc + al(n_pad);
  const size_t o_xc = o_ms + al(sizeof(float) * R * nbs);
  const size_t o_xs = o_xc + al((size_t)P * shard);
  const size_t total = o_xs + al(sizeof(float) * P * nbs);
  psb_status s = psb_peer_ensure(c, total, st);
  if (s) return s;
  uint8_t* own = psb_peer_payload(c);
  psb_mark(c, st);
  s = psb_peer_wait_ack(c, st);  // peers done reading our previous codes / mean
  if (s) return s;
  psb_mark(c, st);
  if (c->prof) cudaEventRecord(psb_prof_event(c), st);
  for (int w = 0; w < W; ++w) {
    const float* g = reinterpret_cast<const float*>(d->g) + (size_t)w * n;
    float* r = d->r ? reinterpret_cast<float*>(d->r) + (size_t)w * n : nullptr;
    s = psb_q8_quant_launch(c, g, r, n, B, reinterpret_cast<int8_t*>(own + o_lc) + (size_t)w * n_pad,
                            reinterpret_cast<float*>(own + o_ls) + (size_t)w * R * nbs, st);
    if (s) return s;
  }
  if (c->prof) cudaEventRecord(psb_prof_event(c), st);
  psb_mark(c, st);
  auto lo_of = [&](int q) { return std::min(nb, (size_t)q * nbs); };
  auto hi_of = [&](int q) { return std::min(nb, (size_t)(q + 1) * nbs); };
  const size_t blk_lo = lo_of(c->rank), blk_hi = hi_of(c->rank);
  // ---- reduce-scatter: pull every remote worker's codes and scales of our
  // shard over NVLink, fold all P workers in order, requantize our shard
  psb_prof_mark(c, 1, st);
  s = psb_peer_signal(c, st);
  if (!s) s = psb_peer_wait_ready(c, st);
  if (s) return s;
  psb_mark(c, st);
  const bool plain = d->order == PSB_ORDER_NAIVE || (d->order == PSB_ORDER_HIER && dpn >= (uint32_t)P);
  if (!c->q8_no_tma && plain && (P == 2 || P == 4 || P == 8) && (B == 128 || B == 256 || (B == 512 && P == 2))) {
    // the reduce reads every worker's codes and scales of our shard in place
    // (TMA bulk copies from the peers' arenas): no pull into local memory
    const uint8_t* regions[PSB_MAX_P];
    psb_peer_regions(c, regions);
    Q8Workers wr{};
    for (int q = 0; q < P; ++q) {
      const uint8_t* base = regions[q / W];
      wr.codes[q] = reinterpret_cast<const int8_t*>(base + o_lc) + (size_t)(q % W) * n_pad + blk_lo * B;
      wr.scales[q] = reinterpret_cast<const float*>(base + o_ls) + (size_t)(q % W) * R * nbs + blk_lo;
    }
    psb_mark(c, st);
    long long tiles = 0;
    if (blk_hi > blk_lo)
      tiles = psb_q8_reduce_tma_launch(c, wr, P, blk_lo, blk_hi, B, reinterpret_cast<int8_t*>(own + o_mc),
                                       reinterpret_cast<float*>(own + o_ms), st);
    if (tiles < 0) return psb_set_err(c, PSB_ECUDA, "q8 TMA reduce launch");
    const size_t done = blk_lo + (size_t)tiles * 8;
    if (done < blk_hi) {  // ragged tail: direct loads
      Q8Workers wt = wr;
      for (int q = 0; q < P; ++q) {
        wt.codes[q] += (size_t)tiles * 8 * B;
        wt.scales[q] += (size_t)tiles * 8;
      }
      s = psb_q8_reduce_launch(c, wt, P, done, blk_hi, n, B, d->order, dpn, npr,
                               reinterpret_cast<int8_t*>(own + o_mc), reinterpret_cast<float*>(own + o_ms), d->lr,
                               nullptr, nullptr, st);
      if (s) return s;
    }
    psb_mark(c, st);
  } else {
  PeerSegs sg{};
  for (int q = 0; q < P; ++q) {
    if (q / W == c->rank || blk_hi <= blk_lo) continue;
    const int w = q % W;
    sg.s[sg.n++] = {q / W, o_lc + (size_t)w * n_pad + blk_lo * B, o_xc + (size_t)q * shard, (blk_hi - blk_lo) * B};
    sg.s[sg.n++] = {q / W, o_ls + sizeof(float) * ((size_t)w * R * nbs + blk_lo), o_xs + sizeof(float) * q * nbs,
                    sizeof(float) * (blk_hi - blk_lo)};
  }
  s = psb_peer_gather(c, sg, st);
  if (s) return s;
  psb_mark(c, st);
  Q8Workers wv{};
  for (int q = 0; q < P; ++q) {
    if (q / W == c->rank) {
      wv.codes[q] = reinterpret_cast<const int8_t*>(own + o_lc) + (size_t)(q % W) * n_pad + blk_lo * B;
      wv.scales[q] = reinterpret_cast<const float*>(own + o_ls) + (size_t)(q % W) * R * nbs + blk_lo;
    } else {
      wv.codes[q] = reinterpret_cast<const int8_t*>(own + o_xc) + (size_t)q * shard;
      wv.scales[q] = reinterpret_cast<const float*>(own + o_xs) + (size_t)q * nbs;
    }
  }
  s = psb_q8_reduce_launch(c, wv, P, blk_lo, blk_hi, n, B, d->order, dpn, npr,
                           reinterpret_cast<int8_t*>(own + o_mc), reinterpret_cast<float*>(own + o_ms), d->lr,
                           nullptr, nullptr, st);
  if (s) return s;
  psb_mark(c, st);
  }
  // ---- all-gather: pull every other rank's requantized shard into place
  s = psb_peer_signal(c, st);
  if (!s) s = psb_peer_wait_ready(c, st);
  if (s) return s;
  psb_mark(c, st);
  Q8Shards ms{};
  int ms_r = 1;
  const bool tma_apply = !c->q8_no_tma && B <= 512 && d->theta != nullptr && d->mean_out == nullptr &&
                         ((uintptr_t)d->theta & 15) == 0;
  if (tma_apply) {
    // gather only the other ranks' mean scales (4 B per block); the TMA apply
    // streams theta and reads every shard's mean codes in place over NVLink
    const float* lscales = nullptr;  // nullptr: the scales are read in place too
    if (!c->q8_scales_inplace) {
      PeerSegs sm{};
      for (int q = 0; q < R; ++q) {
        if (q == c->rank || hi_of(q) <= lo_of(q)) continue;
        sm.s[sm.n++] = {q, o_ms + sizeof(float) * lo_of(q), o_ms + sizeof(float) * lo_of(q),
                        sizeof(float) * (hi_of(q) - lo_of(q))};
      }
      s = psb_peer_gather(c, sm, st);
      if (s) return s;
      lscales = reinterpret_cast<const float*>(own + o_ms);
    }
    const uint8_t* regions[PSB_MAX_P];
    psb_peer_regions(c, regions);
    for (int q = 0; q < R; ++q) {
      ms.codes[q] = reinterpret_cast<const int8_t*>(regions[q] + o_mc);
      ms.scales[q] = reinterpret_cast<const float*>(regions[q] + o_ms);
    }
    ms.nbs = nbs;
    psb_mark(c, st);
    psb_prof_mark(c, 1, st);
    psb_prof_mark(c, 2, st);
    s = psb_q8_apply_tma_launch(c, ms, lscales, n, B, d->lr, reinterpret_cast<float*>(d->theta), st);
    psb_prof_mark(c, 2, st);
    if (!s) s = psb_peer_ack(c, st);  // done reading the peers' arenas for this step
    psb_mark(c, st);
    return s;
  }
  if (c->q8_direct_apply) {
    // the apply reads every other rank's requantized shard in place over
    // NVLink (no pull of the mean), acknowledging once it is done
    const uint8_t* regions[PSB_MAX_P];
    psb_peer_regions(c, regions);
    for (int q = 0; q < R; ++q) {
      ms.codes[q] = reinterpret_cast<const int8_t*>(regions[q] + o_mc);
      ms.scales[q] = reinterpret_cast<const float*>(regions[q] + o_ms);
    }
    ms.nbs = nbs;
    ms_r = R;
    psb_mark(c, st);
    psb_prof_mark(c, 1, st);
  } else {
    PeerSegs sm{};
    for (int q = 0; q < R; ++q) {
      if (q == c->rank || hi_of(q) <= lo_of(q)) continue;
      sm.s[sm.n++] = {q, o_mc + lo_of(q) * B, o_mc + lo_of(q) * B, (hi_of(q) - lo_of(q)) * B};
      sm.s[sm.n++] = {q, o_ms + sizeof(float) * lo_of(q), o_ms + sizeof(float) * lo_of(q),
                      sizeof(float) * (hi_of(q) - lo_of(q))};
    }
    s = psb_peer_gather(c, sm, st);
    if (!s) s = psb_peer_ack(c, st);  // done reading the peers' arenas for this step
    if (s) return s;
    psb_mark(c, st);
    psb_prof_mark(c, 1, st);
    ms.codes[0] = reinterpret_cast<const int8_t*>(own + o_mc);
    ms.scales[0] = reinterpret_cast<const float*>(own + o_ms);
    ms.nbs = (size_t)-1;
  }
  psb_prof_mark(c, 2, st);
  s = psb_q8_apply_launch(c, ms, ms_r, n, B, d->lr, reinterpret_cast<float*>(d->theta),
                          reinterpret_cast<float*>(d->mean_out), st);
  psb_prof_mark(c, 2, st);
  if (!s && c->q8_direct_apply) s = psb_peer_ack(c, st);
  psb_mark(c, st);
  return s;
}

static psb_status q8_step(psb_ctx* c, const psb_step_desc* d, cudaStream_t st) {
  const int W = d->workers, R = c->nranks, P = W * R;
  const uint32_t B = d->q8_block ? d->q8_block : 256;
  PSB_REQUIRE(c, B == 128 || B == 256 || B == 512 || B == 1024, "q8: block must be 128, 256, 512 or 1024");
  const size_t n = d->n;
  const size_t nb = (n + B - 1) / B;
  // blocks per shard, a multiple of 8 (8-block TMA tiles and 32-byte scale
  // copies start on shard boundaries; the fold is per element, so shard
  // boundaries never change a result)
  const size_t nbs = (((nb + R - 1) / R) + 7) & ~(size_t)7;
  const size_t shard_elems = nbs * B;
  const size_t n_pad = (size_t)R * shard_elems;  // >= n
  // workspace: local codes W*n_pad | local scales W*R*nbs | recv codes P*shard | recv scales P*nbs
  //            | mean codes n_pad | mean scales R*nbs   (each region 256-aligned)
  auto al = [](size_t b) { return (b + 255) & ~(size_t)255; };
  const size_t o_lc = 0;
  const size_t o_ls = o_lc + al((size_t)W * n_pad);
  const size_t o_rc = o_ls + al(sizeof(float) * W * R * nbs);
  const size_t o_rs = o_rc + al((size_t)P * shard_elems);
  const size_t o_mc = o_rs + al(sizeof(float) * P * nbs);
  const size_t o_ms = o_mc + al(n_pad);
  const size_t total = o_ms + al(sizeof(float) * R * nbs);
  psb_status s = ensure(c, &c->d_gather, &c->gather_bytes, total, "q8 workspace");
  if (s) return s;
  uint8_t* ws = reinterpret_cast<uint8_t*>(c->d_gather);
  int8_t* lcodes = reinterpret_cast<int8_t*>(ws + o_lc);
  float* lscales = reinterpret_cast<float*>(ws + o_ls);
  int8_t* rcodes = reinterpret_cast<int8_t*>(ws + o_rc);
  float* rscales = reinterpret_cast<float*>(ws + o_rs);
  int8_t* mcodes = reinterpret_cast<int8_t*>(ws + o_mc);
  float* mscales = reinterpret_cast<float*>(ws + o_ms);
  uint32_t dpn, npr;
  if (d->topo.devices_per_node == 0) {
    dpn = (uint32_t)P;
    npr = 1;
  } else {
    dpn = d->topo.devices_per_node;
    npr = d->topo.nodes_per_rack;
  }
  if (R == 1 && d->theta && !c->q8_unfused && (P == 1 || d->order != PSB_ORDER_RING)) {
    // single rank: quantize, fold, requantize and apply in one pass
    return psb_q8_step1_launch(c, reinterpret_cast<const float*>(d->g), n, reinterpret_cast<float*>(d->r), n, P,
                               n, B, d->order, dpn, npr, d->lr, reinterpret_cast<float*>(d->theta),
                               reinterpret_cast<float*>(d->mean_out), st);
  }
  if (R > 1 && c->peer_mode) return q8_step_nvlink(c, d, st, n_pad, nbs, dpn, npr);
  const bool prof_quant = R > 1;  // multi-rank: the quantizer is the dominant kernel
  if (prof_quant && c->prof) cudaEventRecord(psb_prof_event(c), st);
  for (int w = 0; w < W; ++w) {
    const float* g = reinterpret_cast<const float*>(d->g) + (size_t)w * n;
    float* r = d->r ? reinterpret_cast<float*>(d->r) + (size_t)w * n : nullptr;
    s = psb_q8_quant_launch(c, g, r, n, B, lcodes + (size_t)w * n_pad, lscales + (size_t)w * R * nbs, st);
    if (s) return s;
  }
  if (prof_quant && c->prof) cudaEventRecord(psb_prof_event(c), st);
  float* theta = reinterpret_cast<float*>(d->theta);
  float* mean_out = reinterpret_cast<float*>(d->mean_out);
  if (R == 1) {
    Q8Workers wv{};
    for (int q = 0; q < P; ++q) {
      wv.codes[q] = lcodes + (size_t)q * n_pad;
      wv.scales[q] = lscales + (size_t)q * R * nbs;
    }
    return psb_q8_reduce_launch(c, wv, P, 0, nb, n, B, d->order, dpn, npr, mcodes, mscales, d->lr, theta,
                                mean_out, st);
  }
  if (!c->comm) return psb_set_err(c, PSB_ESTATE, "q8 step: communicator not initialised");
  // all-to-all of block shards: worker gid's shard q goes to rank q, slot gid
  psb_prof_mark(c, 1, st);
  NCCL_TRY(c, ncclGroupStart(), "ncclGroupStart");
  for (int peer = 0; peer < R; ++peer) {
    for (int w = 0; w < W; ++w) {
      const int gid_src = c->rank * W + w;  // my worker, sent to peer
      NCCL_TRY(c, ncclSend(lcodes + (size_t)w * n_pad + (size_t)peer * shard_elems, shard_elems, ncclInt8,
                           peer, c->comm, st), "ncclSend(codes)");
      NCCL_TRY(c, ncclSend(lscales + (size_t)w * R * nbs + (size_t)peer * nbs, nbs, ncclFloat32, peer,
                           c->comm, st), "ncclSend(scales)");
      (void)gid_src;
    }
    for (int w = 0; w < W; ++w) {
      const int gid = peer * W + w;  // peer's worker w, my shard
      NCCL_TRY(c, ncclRecv(rcodes + (size_t)gid * shard_elems, shard_elems, ncclInt8, peer, c->comm, st),
               "ncclRecv(codes)");
      NCCL_TRY(c, ncclRecv(rscales + (size_t)gid * nbs, nbs, ncclFloat32, peer, c->comm, st),
               "ncclRecv(scales)");
    }
  }
  NCCL_TRY(c, ncclGroupEnd(), "ncclGroupEnd");
  psb_prof_mark(c, 1, st);
  const size_t blk_lo = (size_t)c->rank * nbs;
  const size_t blk_hi = std::min(nb, blk_lo + nbs);
  Q8Workers wv{};
  for (int q = 0; q < P; ++q) {
    wv.codes[q] = rcodes + (size_t)q * shard_elems;
    wv.scales[q] = rscales + (size_t)q * nbs;
  }
  s = psb_q8_reduce_launch(c, wv, P, blk_lo, blk_hi, n, B, d->order, dpn, npr, mcodes, mscales, d->lr, nullptr,
                           nullptr, st);
  if (s) return s;
  psb_prof_mark(c, 1, st);
  NCCL_TRY(c, ncclGroupStart(), "ncclGroupStart");
  NCCL_TRY(c, ncclAllGather(mcodes + blk_lo * B, mcodes, shard_elems, ncclInt8, c->comm, st),
           "ncclAllGather(codes)");
  NCCL_TRY(c, ncclAllGather(mscales + blk_lo, mscales, nbs, ncclFloat32, c->comm, st),
           "ncclAllGather(scales)");
  NCCL_TRY(c, ncclGroupEnd(), "ncclGroupEnd");
  psb_prof_mark(c, 1, st);
  Q8Shards ms{};
  ms.codes[0] = mcodes;
  ms.scales[0] = mscales;
  ms.nbs = (size_t)-1;
  return psb_q8_apply_launch(c, ms, 1, n, B, d->lr, theta, mean_out, st);
}

// The step on a validated descriptor; theta == NULL computes only the mean
// (into mean_out) -- the momentum path uses that.
static psb_status sync_step_core(psb_ctx* c, const psb_step_desc* d, psb_stream_t stream) {
  psb_status s = PSB_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const int W = d->workers, P = W * c->nranks;
  const size_t es = d->dtype == PSB_F64 ? 8 : 4;
  switch (d->compressor) {
    case PSB_COMP_TOPK:
    case PSB_COMP_TOPK_Q8: {
      uint8_t* pl = nullptr;
      const bool fuse = P == 1 && d->compressor == PSB_COMP_TOPK && d->theta != nullptr;
      ShardPlan sp;
      s = compress_and_gather(c, d, st, &pl, fuse, &sp);
      if (s || fuse) return s;
      if (sp.on) return shard_apply(c, d, sp, nullptr, false, st);
      psb_prof_mark(c, 2, st);
      if (sp.direct) {
        const uint8_t* regions[PSB_MAX_P];
        psb_peer_regions(c, regions);
        s = psb_sparse_apply_direct(c, d->compressor, d->dtype, P, d->workers, regions, d->k, sp.tab_off, d->order,
                                    &d->topo, d->lr, nullptr, 0, d->theta, d->n, d->mean_out, st, sp.wire16);
      } else if (sp.wire16)
        s = psb_sparse_apply_wire16(c, d->dtype, P, pl, d->k, reinterpret_cast<const uint32_t*>(pl + sp.tab_off),
                                    d->order, &d->topo, d->lr, nullptr, 0, d->theta, d->n, d->mean_out, st);
      else if (sp.tab_ready)
        s = psb_sparse_apply_tab(c, d->compressor, d->dtype, P, pl, d->k,
                                 reinterpret_cast<const uint32_t*>(pl + sp.tab_off), d->order, &d->topo, d->lr,
                                 nullptr, 0, d->theta, d->n, d->mean_out, st);
      else
        s = psb_sparse_mean_sgd(c, d->compressor, d->dtype, P, pl, d->k, d->order, &d->topo, d->lr,
                                d->theta, d->n, d->mean_out, stream);
      psb_prof_mark(c, 2, st);
      if (!s && sp.ack_after_apply) s = psb_peer_ack(c, st);
      psb_mark(c, st);
      return s;
    }
    case PSB_COMP_ONEBIT: {
      const size_t nw = (d->n + 31) / 32;
      const size_t words_bytes = (sizeof(uint32_t) * nw * P + 255) & ~(size_t)255;
      s = ensure(c, &c->d_gather, &c->gather_bytes, words_bytes + sizeof(double) * P, "onebit buffers");
      if (s) return s;
      uint32_t* words = reinterpret_cast<uint32_t*>(c->d_gather);
      double* scales = reinterpret_cast<double*>(reinterpret_cast<uint8_t*>(c->d_gather) + words_bytes);
      for (int w = 0; w < W; ++w) {
        const int gid = c->rank * W + w;
        const void* g = reinterpret_cast<const uint8_t*>(d->g) + (size_t)w * d->n * es;
        void* r = d->r ? reinterpret_cast<uint8_t*>(d->r) + (size_t)w * d->n * es : nullptr;
        s = psb_ef_onebit(c, d->dtype, g, r, d->n, words + (size_t)gid * nw, scales + gid, stream);
        if (s) return s;
      }
      if (c->nranks > 1) {
        if (!c->comm) return psb_set_err(c, PSB_ESTATE, "sync step: communicator not initialised");
        NCCL_TRY(c, ncclGroupStart(), "ncclGroupStart");
        NCCL_TRY(c, ncclAllGather(words + (size_t)c->rank * W * nw, words, (size_t)W * nw, ncclUint32,
                                  c->comm, st), "ncclAllGather(sign words)");
        NCCL_TRY(c, ncclAllGather(scales + (size_t)c->rank * W, scales, (size_t)W, ncclFloat64, c->comm, st),
                 "ncclAllGather(scales)");
        NCCL_TRY(c, ncclGroupEnd(), "ncclGroupEnd");
      }
      return psb_onebit_mean_sgd(c, d->dtype, P, words, scales, d->order, &d->topo, d->lr, d->theta,
                                 d->n, d->mean_out, stream);
    }
    case PSB_COMP_NONE: {
      // no compression: allreduce_mean of the raw buffers (strategies.hpp:94-95);
      // exact reference order requires all P dense buffers -> allgather them.
      const void* bufs = d->g;
      if (c->nranks > 1) {
        s = ensure(c, &c->d_gather, &c->gather_bytes, es * d->n * P, "dense gather buffer");
        if (s) return s;
        uint8_t* gb = reinterpret_cast<uint8_t*>(c->d_gather);
        CUDA_TRY(c, cudaMemcpyAsync(gb + (size_t)c->rank * W * d->n * es, d->g, (size_t)W * d->n * es,
                                    cudaMemcpyDeviceToDevice, st), "dense copy");
        if (!c->comm) return psb_set_err(c, PSB_ESTATE, "sync step: communicator not initialised");
        NCCL_TRY(c, ncclAllGather(gb + (size_t)c->rank * W * d->n * es, gb, (size_t)W * d->n * es, ncclUint8,
                                  c->comm, st), "ncclAllGather(dense)");
        bufs = gb;
      }
      return psb_dense_mean_sgd(c, d->dtype, P, bufs, d->order, &d->topo, d->lr, d->theta, d->n,
                                d->mean_out, stream);
    }
    case PSB_COMP_Q8:
      return q8_step(c, d, st);
  }
  return psb_set_err(c, PSB_EINVAL, "compress: unknown compressor kind");
}

extern "C" psb_status psb_sync_step(psb_ctx* c, const psb_step_desc* d, psb_stream_t stream) {
  psb_status s = check_desc(c, d);
  if (s) return s;
  if (!d->m) return sync_step_core(c, d, stream);
  // momentum SGD: the step's aggregated mean into a zeroed dense scratch,
  // then one dense pass m = beta*m + mean; theta = (-lr)*m + theta
  PSB_REQUIRE(c, d->compressor != PSB_COMP_Q8, "momentum: not supported with the dense q8 compressor");
  cudaStream_t st = (cudaStream_t)stream;
  const size_t es = d->dtype == PSB_F64 ? 8 : 4;
  static const bool no_merge = getenv("PSB_MOM_NO_MERGE") && atoi(getenv("PSB_MOM_NO_MERGE"));
  if (!no_merge && c->nranks == 1 && d->workers == 1 && d->compressor == PSB_COMP_TOPK) {
    // one payload: its sorted (index, value) list is the mean; no dense scratch
    s = ensure(c, &c->d_mom_mean, &c->mom_bytes, sizeof(uint32_t) * (d->n / 4096 + 2), "momentum tile table");
    if (s) return s;
    uint8_t* pl = nullptr;
    s = compress_and_gather(c, d, st, &pl, false, nullptr);
    if (s) return s;
    s = psb_momentum_topk1(c, d->dtype, pl, d->k, d->m, d->theta, d->mean_out, d->beta, d->lr, d->n,
                           reinterpret_cast<uint32_t*>(c->d_mom_mean), st);
    psb_mark(c, st);
    return s;
  }
  s = ensure(c, &c->d_mom_mean, &c->mom_bytes, es * d->n, "momentum mean buffer");
  if (s) return s;
  CUDA_TRY(c, cudaMemsetAsync(c->d_mom_mean, 0, es * d->n, st), "momentum");
  psb_step_desc d2 = *d;
  d2.theta = nullptr;
  d2.mean_out = c->d_mom_mean;
  d2.m = nullptr;
  s = sync_step_core(c, &d2, stream);
  if (s) return s;
  s = psb_momentum_sgd(c, d->dtype, c->d_mom_mean, d->m, d->theta, d->beta, d->lr, d->n, stream);
  if (s) return s;
  if (d->mean_out)
    CUDA_TRY(c, cudaMemcpyAsync(d->mean_out, c->d_mom_mean, es * d->n, cudaMemcpyDeviceToDevice, st), "momentum");
  return PSB_OK;
}

extern "C" psb_status psb_async_pipeline(psb_ctx* c, int enable) {
  PSB_REQUIRE(c, c != nullptr, "null ctx");
  if (enable && !c->apply_st) {
    CUDA_TRY(c, cudaSetDevice(c->device), "psb_async_pipeline");
    // highest priority: the exchange / apply CTAs are scheduled ahead of the
    // next round's compression as SM resources free up
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    CUDA_TRY(c, cudaStreamCreateWithPriority(&c->apply_st, cudaStreamNonBlocking, hi), "psb_async_pipeline");
    for (int i = 0; i < 2; ++i) {
      CUDA_TRY(c, cudaEventCreateWithFlags(&c->comp_ev[i], cudaEventDisableTiming), "psb_async_pipeline");
      CUDA_TRY(c, cudaEventCreateWithFlags(&c->apply_ev[i], cudaEventDisableTiming), "psb_async_pipeline");
    }
  }
  c->async_pipe = enable ? 1 : 0;
  return PSB_OK;
}

extern "C" psb_status psb_async_sync(psb_ctx* c, psb_stream_t stream) {
  PSB_REQUIRE(c, c != nullptr, "null ctx");
  for (int i = 0; i < 2; ++i)
    if (c->apply_pending[i]) {
      CUDA_TRY(c, cudaStreamWaitEvent((cudaStream_t)stream, c->apply_ev[i], 0), "psb_async_sync");
      c->apply_pending[i] = false;
    }
  return PSB_OK;
}

// One pipelined round (psb_async_pipeline on): compress on `st` into the
// round's payload slot, then exchange + apply on the ctx's apply stream.
// Every stage is bitwise the serial round's (the same kernels in the same
// order per buffer): only the cross-round overlap differs.
static psb_status async_round_pipelined(psb_ctx* c, const psb_step_desc* d, const double* scale,
                                        cudaStream_t st) {
  const int W = d->workers, R = c->nranks, P = W * R;
  const size_t blk = psb_payload_bytes(d->compressor, d->dtype, d->k);
  const int slot = (int)(c->pipe_round & 1);
  const size_t need = blk * (size_t)W;
  if (c->pipe_bytes < need) {
    // grow: nothing may still read the old slots
    CUDA_TRY(c, cudaStreamSynchronize(st), "async pipeline");
    CUDA_TRY(c, cudaStreamSynchronize(c->apply_st), "async pipeline");
    for (int i = 0; i < 2; ++i) {
      if (c->pipe_pl[i]) cudaFree(c->pipe_pl[i]);
      c->pipe_pl[i] = nullptr;
      c->apply_pending[i] = false;
    }
    for (int i = 0; i < 2; ++i)
      if (cudaMalloc(&c->pipe_pl[i], need) != cudaSuccess)
        return psb_set_err(c, PSB_ENOMEM, "async pipeline: out of device memory");
    c->pipe_bytes = need;
  }
  // ---- compress (caller's stream): this slot's previous apply must be done
  if (c->apply_pending[slot]) {
    CUDA_TRY(c, cudaStreamWaitEvent(st, c->apply_ev[slot], 0), "async pipeline");
    c->apply_pending[slot] = false;
  }
  uint8_t* kb = reinterpret_cast<uint8_t*>(c->pipe_pl[slot]);
  const size_t es = d->dtype == PSB_F64 ? 8 : 4;
  psb_status s;
  for (int w = 0; w < W; ++w) {
    uint8_t* pslot = kb + (size_t)w * blk;
    const void* g = reinterpret_cast<const uint8_t*>(d->g) + (size_t)w * d->n * es;
    void* r = d->r ? reinterpret_cast<uint8_t*>(d->r) + (size_t)w * d->n * es : nullptr;
    uint32_t* idx = reinterpret_cast<uint32_t*>(pslot);
    if (d->compressor == PSB_COMP_TOPK) {
      s = psb_topk_run(c, d->dtype, w, g, r, d->n, d->k, idx, pslot + psb_align16(d->k * 4), st);
    } else {
      int8_t* codes = reinterpret_cast<int8_t*>(pslot + psb_align16(d->k * 4));
      float* scales = reinterpret_cast<float*>(pslot + psb_align16(d->k * 4) + psb_align16(d->k));
      s = psb_ef_topk_q8(c, w, (const float*)g, (float*)r, d->n, d->k, idx, codes, scales, (psb_stream_t)st);
    }
    if (s) return s;
  }
  CUDA_TRY(c, cudaEventRecord(c->comp_ev[slot], st), "async pipeline");
  // ---- exchange + apply (apply stream, in round order)
  cudaStream_t as = c->apply_st;
  CUDA_TRY(c, cudaStreamWaitEvent(as, c->comp_ev[slot], 0), "async pipeline");
  const uint8_t* pl = kb;
  if (R > 1 && c->peer_mode && P >= 2) {
    // NVLink pull: this rank's payloads (wire16 for f32/f64 top-k) and their
    // per-segment offset rows into its arena, signal, pull the peers', apply
    auto al = [](size_t b) { return (b + 255) & ~(size_t)255; };
    const bool wire16 = d->compressor == PSB_COMP_TOPK && !c->no_wire16;
    const size_t pblk = wire16 ? psb_wire16_bytes(d->dtype, d->k) : blk;
    const int seg_shift = psb_apply_seg_shift(P);
    const uint32_t nseg = (uint32_t)((d->n + ((size_t)1 << seg_shift) - 1) >> seg_shift);
    const size_t tab_off = al(pblk * P);
    const size_t region = tab_off + al(sizeof(uint32_t) * P * (nseg + 1));
    s = psb_peer_ensure(c, region, as);
    if (s) return s;
    uint8_t* gb = psb_peer_payload(c);
    s = psb_peer_wait_ack(c, as);
    if (s) return s;
    uint32_t* tab = reinterpret_cast<uint32_t*>(gb + tab_off) + (size_t)c->rank * W * (nseg + 1);
    s = psb_seg_offsets(c, d->compressor, d->dtype, W, kb, d->k, nseg, seg_shift, tab, as,
                        wire16 ? gb + (size_t)c->rank * W * pblk : nullptr, pblk);
    if (s) return s;
    for (int w = 0; w < W && !wire16; ++w) {
      const int gid = c->rank * W + w;
      s = cudaMemcpyAsync(gb + (size_t)gid * pblk, kb + (size_t)w * blk, blk, cudaMemcpyDeviceToDevice, as) ==
                    cudaSuccess
                ? PSB_OK
                : psb_set_err(c, PSB_ECUDA, "async pipeline: payload copy");
      if (s) return s;
    }
    psb_prof_mark(c, 1, as);
    s = psb_peer_exchange(c, (size_t)W * pblk, tab_off, (size_t)W * (nseg + 1), as);
    psb_prof_mark(c, 1, as);
    if (s) return s;
    const uint32_t* tabs = reinterpret_cast<const uint32_t*>(gb + tab_off);
    if (wire16)
      s = psb_sparse_apply_wire16(c, d->dtype, P, gb, d->k, tabs, PSB_ORDER_NAIVE, nullptr, 0.0, scale, 1, d->theta,
                                  d->n, nullptr, as);
    else
      s = psb_sparse_apply_tab(c, d->compressor, d->dtype, P, gb, d->k, tabs, PSB_ORDER_NAIVE, nullptr, 0.0, scale,
                               1, d->theta, d->n, nullptr, as);
  } else {
    if (R > 1) {
      // NCCL all-gather of the payloads (psb_peer_mode 0)
      s = ensure(c, &c->d_gather, &c->gather_bytes, blk * P, "payload gather buffer");
      if (s) return s;
      uint8_t* gb = reinterpret_cast<uint8_t*>(c->d_gather);
      CUDA_TRY(c, cudaMemcpyAsync(gb + (size_t)c->rank * W * blk, kb, blk * W, cudaMemcpyDeviceToDevice, as),
               "async pipeline");
      if (!c->comm) return psb_set_err(c, PSB_ESTATE, "async round: communicator not initialised");
      NCCL_TRY(c, ncclAllGather(gb + (size_t)c->rank * W * blk, gb, (size_t)W * blk, ncclUint8, c->comm, as),
               "ncclAllGather(payloads)");
      pl = gb;
    }
    s = psb_sparse_async_apply(c, d->compressor, d->dtype, P, pl, d->k, scale, d->theta, d->n, (psb_stream_t)as);
  }
  if (s) return s;
  CUDA_TRY(c, cudaEventRecord(c->apply_ev[slot], as), "async pipeline");
  c->apply_pending[slot] = true;
  c->pipe_round += 1;
  return PSB_OK;
}

extern "C" psb_status psb_async_round(psb_ctx* c, const psb_step_desc* d, uint32_t staleness_bound,
                                      uint64_t* global_updates, psb_stream_t stream) {
  psb_status s = check_desc(c, d);
  if (s) return s;
  PSB_REQUIRE(c, global_updates != nullptr, "psb_async_round: null global_updates");
  PSB_REQUIRE(c, d->m == nullptr, "psb_async_round: momentum is defined for sync steps only");
  PSB_REQUIRE(c, d->compressor == PSB_COMP_TOPK || d->compressor == PSB_COMP_TOPK_Q8,
              "psb_async_round: sparse compressors only");
  cudaStream_t st = (cudaStream_t)stream;
  const int P = d->workers * c->nranks;
  std::vector<double> scale(P);
  const uint64_t g0 = *global_updates;
  for (int p = 0; p < P; ++p) {
    const uint64_t bound = (uint64_t)staleness_bound + 1;
    const uint64_t tau = std::min<uint64_t>(g0 + (uint64_t)p, (uint64_t)p % bound);
    scale[p] = d->lr / (1.0 + (double)tau);  // strategies.hpp:127
  }
  // pipelined rounds (pull or NCCL exchange; the push / sharded / direct
  // modes run serially)
  if (c->async_pipe && (c->nranks == 1 || c->peer_mode <= 1)) {
    s = async_round_pipelined(c, d, scale.data(), st);
    if (s) return s;
    *global_updates = g0 + (uint64_t)P;
    return PSB_OK;
  }
  s = psb_async_sync(c, stream);  // a serial round after pipelined ones
  if (s) return s;
  uint8_t* pl = nullptr;
  ShardPlan sp;
  s = compress_and_gather(c, d, st, &pl, false, &sp);
  if (s) return s;
  if (sp.on) s = shard_apply(c, d, sp, scale.data(), true, st);
  else if (sp.direct) {
    const uint8_t* regions[PSB_MAX_P];
    psb_peer_regions(c, regions);
    s = psb_sparse_apply_direct(c, d->compressor, d->dtype, P, d->workers, regions, d->k, sp.tab_off, PSB_ORDER_NAIVE,
                                nullptr, 0.0, scale.data(), 1, d->theta, d->n, nullptr, st, sp.wire16);
    if (!s) s = psb_peer_ack(c, st);
  } else if (sp.wire16) {
    s = psb_sparse_apply_wire16(c, d->dtype, P, pl, d->k, reinterpret_cast<const uint32_t*>(pl + sp.tab_off),
                                PSB_ORDER_NAIVE, nullptr, 0.0, scale.data(), 1, d->theta, d->n, nullptr, st);
    if (!s && sp.ack_after_apply) s = psb_peer_ack(c, st);
  } else if (sp.tab_ready) {
    s = psb_sparse_apply_tab(c, d->compressor, d->dtype, P, pl, d->k, reinterpret_cast<const uint32_t*>(pl + sp.tab_off),
                             PSB_ORDER_NAIVE, nullptr, 0.0, scale.data(), 1, d->theta, d->n, nullptr, st);
    if (!s && sp.ack_after_apply) s = psb_peer_ack(c, st);
  }
  else s = psb_sparse_async_apply(c, d->compressor, d->dtype, P, pl, d->k, scale.data(), d->theta, d->n, stream);
  if (s) return s;
  *global_updates = g0 + (uint64_t)P;
  return PSB_OK;
}
