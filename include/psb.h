/*
 * psb.h -- C ABI of the B200-native data-parallel gradient path
 *          (compress -> aggregate -> apply) of arXiv 2506.17551.
 *
 * Drop-in boundary.  The reference (parsim, header-only C++20) has no C ABI;
 * its interface is the C++ API in namespace parsim.  Each entry
 * point below names the reference function it replaces (file:line under
 * /root/reference/proj/include/parsim).  A host binding (ctypes, the C++
 * facade in include/parsim_b200.hpp, or a cgo/JNI stub)
 * calls these with plain device pointers and sizes; no torch types appear.
 *
 * Conventions
 *   - All array arguments are DEVICE pointers unless marked (host).
 *   - Every call is stream-ordered on `stream` (a cudaStream_t; NULL = legacy
 *     default stream) and returns immediately.  Argument errors are reported
 *     synchronously (PSB_EINVAL, text in psb_last_error(), same wording as the
 *     reference's detail::require messages).  Data-dependent errors (a
 *     non-finite residual or parameter, parsim/numerics.hpp:57-61) raise a
 *     device flag that psb_check() turns into PSB_ENONFINITE.
 *   - The caller owns g, r (error-feedback residual), theta and all outputs;
 *     the ctx owns every scratch buffer (allocated once in psb_ctx_create,
 *     none per call) and the NCCL communicator.
 *   - A ctx is bound to one device and one stream at a time; not thread-safe.
 *   - Index type is u32: n must be < 2^32.
 *   - f32 is the production type; f64 instantiations exist for bit-exact
 *     parity with the f64 reference.
 */
#ifndef PSB_H_
#define PSB_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PSB_ABI_VERSION 1

#if defined(__GNUC__)
#define PSB_API __attribute__((visibility("default")))
#else
#define PSB_API
#endif

typedef struct psb_ctx psb_ctx;
typedef struct CUstream_st* psb_stream_t; /* == cudaStream_t */

typedef enum {
  PSB_OK = 0,
  PSB_EINVAL = 1,     /* precondition failed (reference: std::invalid_argument) */
  PSB_ENONFINITE = 2, /* non-finite residual/parameter (reference: check_finite) */
  PSB_ECUDA = 3,
  PSB_ENCCL = 4,
  PSB_ENOMEM = 5,
  PSB_ESTATE = 6 /* ctx misuse (e.g. collective without psb_comm_init) */
} psb_status;

typedef enum { PSB_F32 = 0, PSB_F64 = 1 } psb_dtype;

/* CollectiveAlgorithm fold orders, parsim/collectives.hpp:41, 68-128.
 * pipelined_ring folds like ring (collectives.hpp:142-143). */
typedef enum { PSB_ORDER_NAIVE = 0, PSB_ORDER_RING = 1, PSB_ORDER_HIER = 2 } psb_order;

/* CompressorKind, parsim/compression.hpp:20 (none/onebit/topk), plus the
 * north-star additions with no reference code: top-k with int8
 * values and the dense 8-bit block quantizer. */
typedef enum {
  PSB_COMP_NONE = 0,
  PSB_COMP_ONEBIT = 1,
  PSB_COMP_TOPK = 2,
  PSB_COMP_TOPK_Q8 = 3,
  PSB_COMP_Q8 = 4
} psb_compressor;

typedef enum { PSB_DIST_UNIFORM = 0, PSB_DIST_LLMREC = 1, PSB_DIST_TIES = 2 } psb_dist;

/* Topology grouping used by the hierarchical fold, parsim/collectives.hpp:18-39. */
typedef struct {
  uint32_t racks;
  uint32_t nodes_per_rack;
  uint32_t devices_per_node;
} psb_topology;

/* ------------------------------------------------------------ context */
PSB_API int psb_abi_version(void);
PSB_API const char* psb_status_string(psb_status s);

/* Allocates all workspace for gradients up to max_n elements, top-k up to
 * max_k, and up to max_workers payloads per step (P = local workers x ranks). */
PSB_API psb_status psb_ctx_create(psb_ctx** out, int device, size_t max_n, size_t max_k, int max_workers);
PSB_API void psb_ctx_destroy(psb_ctx* ctx);
PSB_API const char* psb_last_error(const psb_ctx* ctx);

/* Synchronizes `stream` and converts device error flags raised since the
 * last check into a status (PSB_ENONFINITE), clearing them. */
PSB_API psb_status psb_check(psb_ctx* ctx, psb_stream_t stream);

/* Number of the ctx's own kernels launched so far (for launch accounting). */
PSB_API uint64_t psb_launch_count(const psb_ctx* ctx);

/* Kernel timing for roofline accounting: when enabled, every launch of the
 * K1 streaming pass (the EF add + level-1 histogram kernel, the path's
 * dominant kernel) is bracketed by CUDA events on its launching stream.
 * psb_profile_read synchronizes, returns the summed duration (ms) and launch
 * count since the last read, and clears them. */
PSB_API psb_status psb_profile_enable(psb_ctx* ctx, int enable);
PSB_API psb_status psb_profile_read(psb_ctx* ctx, double* total_ms, uint64_t* launches);
/* Same for a phase of the multi-rank steps: 0 = the K1 streaming pass (as
 * psb_profile_read), 1 = the exchange (NVLink signal + pull, or the NCCL
 * collectives; wait for the slowest peer included), 2 = the P-payload apply.
 * Returns the summed ms and the number of event pairs since the last read. */
PSB_API psb_status psb_profile_read_phase(psb_ctx* ctx, int phase, double* total_ms, uint64_t* pairs);

/* Diagnostics of the last K1 call and of `worker`'s threshold prediction:
 * out[0] candidates, [1] k, [2] threshold key T, [3] ties taken at T,
 * [4] first radix level resolved over candidates (0 = prediction valid),
 * [5] predicted key used (0 = cold), [6] misses << 32 | calls, [7] bits of
 * the margin factor f.  Synchronous (copies from the device). */
PSB_API psb_status psb_topk_stats(psb_ctx* ctx, int worker, uint64_t* out8);
/* GPU timestamps (ns) of the candidate-phase milestones of the last K1 call
 * (diagnostics; entries after the last milestone are stale). */
PSB_API psb_status psb_topk_phases(psb_ctx* ctx, uint64_t* out16);

/* Bytes of one worker's top-k payload block: u32 idx[k] | pad16 | val[k] | pad16
 * (TOPK, val of dtype) or u32 idx[k] | pad16 | i8 code[k] | pad16 |
 * f32 scale[ceil(k/128)] | pad16 (TOPK_Q8). */
PSB_API size_t psb_payload_bytes(psb_compressor c, psb_dtype dt, size_t k);

/* -------------------------------------------------------- communicator
 * One rank per GPU, NCCL over NVLink/NVSwitch.  uid is 128 bytes (host). */
PSB_API psb_status psb_comm_unique_id(void* uid_out);
PSB_API psb_status psb_comm_init(psb_ctx* ctx, int rank, int nranks, const void* uid);
PSB_API int psb_comm_rank(const psb_ctx* ctx);
PSB_API int psb_comm_size(const psb_ctx* ctx);
/* In-place allgather: buf holds nranks blocks of bytes_per_rank; this rank's
 * block is at buf + rank*bytes_per_rank. */
PSB_API psb_status psb_allgather(psb_ctx* ctx, void* buf, size_t bytes_per_rank, psb_stream_t stream);
/* Sparse exchange + apply of psb_sync_step / psb_async_round with nranks > 1,
 * over NVLink peer memory (CUDA IPC arenas, device-side sequence flags, set
 * up collectively on first use) unless mode 0:
 *   5 (default) auto: 4 for top-k f32/f64, 1 for top-k int8;
 *   1 pull: after K1 every rank copies the peers' payloads (and their
 *     producer-computed per-segment offset rows) into its arena, each CTA
 *     waiting only for its own peer, then applies all P payloads;
 *   3 push: K1 stores each CTA's finished payload range straight into every
 *     peer's arena (top-k f32/f64; top-k int8 falls back to 1), then every
 *     rank applies all P payloads from its own arena;
 *   2 sharded: each rank pulls only the payload entries of its share of the
 *     index space (balanced on the device), folds them into theta and an
 *     update list, then applies the other ranks' lists;
 *   4 direct: no copy -- the apply reads every peer's wire16 payload and
 *     offset rows in place from its arena over NVLink, its TMA stage
 *     bringing the next segment's remote entries in while it folds the
 *     current one (the fastest measured on B200 for top-k f32: DESIGN.md
 *     section 4);
 *   0 NCCL all-gather of the payloads, then the full apply.
 * Results are bitwise identical in every mode.  Environment at ctx creation: PSB_NO_PEER=1 -> 0,
 * PSB_SHARD=1 -> 2, PSB_PEER_MODE=<n> -> n.  Steps with mean_out never shard. */
PSB_API psb_status psb_peer_mode(psb_ctx* ctx, int mode);
/* 1 once the peer arenas are mapped. */
PSB_API int psb_peer_active(const psb_ctx* ctx);

/* -------------------------------------------------------- wire format
 * wire_encode / wire_decode (parsim/compression.hpp:159-239), little-endian:
 *   DENSE   u64 dim | dim x f64
 *   SIGNBIT u64 dim | f64 scale | ceil(dim/8) sign bytes (bit i%8 of byte i/8)
 *   TOPK    u64 dim | u64 count | count x (u64 index, f64 value)
 * Device buffers; values widen to f64 on encode, round to the payload dtype
 * on decode.  Encode outputs 16-byte aligned (dense: 8). */
typedef enum { PSB_WIRE_DENSE = 0, PSB_WIRE_SIGNBIT = 1, PSB_WIRE_TOPK = 2 } psb_wire_kind;
PSB_API size_t psb_wire_bytes(psb_wire_kind kind, uint64_t dim, size_t k);
PSB_API psb_status psb_wire_encode_topk(psb_ctx* ctx, psb_dtype dt, uint64_t dim, const uint32_t* idx,
                                const void* val, size_t k, void* out, psb_stream_t stream);
/* Synchronizes the stream; errors as the reference: "wire_decode: truncated
 * input", plus capacity (count > k_cap) and the 32-bit index range. */
PSB_API psb_status psb_wire_decode_topk(psb_ctx* ctx, psb_dtype dt, const void* in, size_t nbytes, size_t k_cap,
                                uint32_t* idx, void* val, uint64_t* dim_out, size_t* count_out,
                                psb_stream_t stream);
PSB_API psb_status psb_wire_encode_signbit(psb_ctx* ctx, uint64_t dim, const uint32_t* words, const double* scale,
                                   void* out, psb_stream_t stream);
PSB_API psb_status psb_wire_encode_dense(psb_ctx* ctx, psb_dtype dt, const void* x, uint64_t dim, void* out,
                                 psb_stream_t stream);

/* ------------------------------------------- gradient producer (BPR)
 * bpr_batch_gradient + bpr_batch_loss (parsim/trainer.hpp:98-138) for the
 * reference's matrix-factorisation recommender; flat theta = user rows then
 * item rows, dim columns (trainer.hpp:86-91).  Triples (user, pos, neg) are
 * device u32 arrays of length B.  grad ([users+items][dim], dtype) is fully
 * written (zeros outside the touched rows); loss_out (device double, nullable)
 * gets the batch-mean loss.  Every row's contributions are folded in batch
 * order as the reference does; exp() is the device's (<= 1 ulp from glibc). */
PSB_API psb_status psb_bpr_gradient(psb_ctx* ctx, psb_dtype dt, const void* theta, uint32_t users, uint32_t items,
                            uint32_t dim, const uint32_t* user, const uint32_t* pos, const uint32_t* neg,
                            uint32_t B, void* grad, double* loss_out, psb_stream_t stream);

/* Sampled ranking of evaluate_topk (trainer.hpp:269-324): for each of R test
 * records (user, true item) and its ncand candidate items (u32, 0xffffffff =
 * padding), rank = 1 + #{c : s(c) > s(true) or (s(c) == s(true) and c < true)}
 * with the reference's sequential f64 dot-product scores (bit-exact). */
PSB_API psb_status psb_rank_candidates(psb_ctx* ctx, psb_dtype dt, const void* theta, uint32_t users, uint32_t dim,
                               uint32_t R, const uint32_t* rec_user, const uint32_t* rec_item,
                               const uint32_t* cands, uint32_t ncand, uint32_t* rank_out, psb_stream_t stream);

/* ---------------------------------------------------------- generator
 * Counter-based synthetic gradients, identical bits to
 * oracle/psb_oracle.c:orc_generate.  Input generation only. */
PSB_API psb_status psb_generate(psb_dist dist, uint64_t seed, uint32_t rank, uint32_t step, size_t n,
                        float* out, psb_stream_t stream);

/* -------------------------------------------------------- compressors */

/* K1: ef_compress_step with the top-k compressor (compression.hpp:146-157 ->
 * compress_topk :81-99).  p = r + g; the k entries of largest |p| (ties to
 * the lower index) are emitted with indices ascending; r := (selected ? +0 : p).
 * r == NULL: transient zero residual (strategies.hpp:97-102), p = g, nothing
 * written back -- with g as input this is compress_topk itself.
 * `worker` in [0, max_workers) keys the per-worker selection history used to
 * predict the threshold (results never depend on it).  idx_out: u32[k];
 * val_out: dtype[k]. */
PSB_API psb_status psb_ef_topk(psb_ctx* ctx, psb_dtype dt, int worker, const void* g, void* r, size_t n,
                       size_t k, uint32_t* idx_out, void* val_out, psb_stream_t stream);

/* K1 + int8 values (north-star, unpinned): the selected values p[idx] are
 * quantized in blocks of 128 consecutive payload entries with the 8-bit rule
 * of psb_q8_quantize; r := (selected ? p - code*scale : p). */
PSB_API psb_status psb_ef_topk_q8(psb_ctx* ctx, int worker, const float* g, float* r, size_t n, size_t k,
                          uint32_t* idx_out, int8_t* codes_out, float* scales_out,
                          psb_stream_t stream);

/* 1-bit sign compressor with EF: compress_onebit (compression.hpp:67-77) on
 * p = r + g.  words_out: u32[ceil(n/32)], bit i%32 of word i/32 = (p_i >= 0)
 * (little-endian identical to the reference sign_bytes); scale_out: one f64
 * (device) = sum|p_i| / n (fixed-shape deterministic reduction); r := p -
 * (+-scale) in dtype. */
PSB_API psb_status psb_ef_onebit(psb_ctx* ctx, psb_dtype dt, const void* g, void* r, size_t n,
                         uint32_t* words_out, double* scale_out, psb_stream_t stream);

/* 8-bit block quantizer (north-star, no reference code; spec in
 * oracle/psb_oracle.c:orc_q8_quant): per block of `block` elements scale =
 * absmax/127, code = rint(p/scale) in [-127,127]; r (nullable) := p - code*scale. */
PSB_API psb_status psb_q8_quantize(psb_ctx* ctx, const float* x, float* r, size_t n, uint32_t block,
                           int8_t* codes, float* scales, psb_stream_t stream);
PSB_API psb_status psb_q8_dequantize(psb_ctx* ctx, const int8_t* codes, const float* scales, size_t n,
                             uint32_t block, float* out, psb_stream_t stream);

/* decompress of one top-k payload into a dense vector (compression.hpp:113-142):
 * out (n, pre-zeroed by the caller) receives val at idx.  Index validation
 * (idx < n, strictly increasing) raises a device flag reported by psb_check as
 * PSB_EINVAL ("decompress: index out of range" / "indices not strictly increasing"). */
PSB_API psb_status psb_decompress_topk(psb_ctx* ctx, psb_dtype dt, const uint32_t* idx, const void* val,
                               size_t k, size_t n, void* out, psb_stream_t stream);

/* ------------------------------------------------- aggregate + apply */

/* decompress + allreduce_mean + vec_axpy(-lr, mean, theta) for P top-k
 * payload blocks (strategies.hpp:105-112, collectives.hpp:135-148,
 * numerics.hpp:70-78), without materializing dense messages.  payloads: P
 * blocks of psb_payload_bytes(PSB_COMP_TOPK or TOPK_Q8, dt, k) in worker order.
 * The mean at each touched index is folded over the P dense values (+0 where a
 * worker did not select the index) in the configured order, so results are
 * bit-identical to the reference's dense fold; theta is updated in place with
 * a separate multiply and add (no FMA).  Untouched entries are unchanged
 * (bitwise, as (-lr)*(+0) + theta == theta).  mean_out (nullable, dense n,
 * pre-zeroed by the caller) receives the mean at touched indices.
 * theta == NULL computes the mean only (allreduce_mean without the update);
 * the same holds for psb_dense_mean_sgd and psb_onebit_mean_sgd. */
PSB_API psb_status psb_sparse_mean_sgd(psb_ctx* ctx, psb_compressor c, psb_dtype dt, int P,
                               const void* payloads, size_t k, psb_order order,
                               const psb_topology* topo, double lr, void* theta, size_t n,
                               void* mean_out, psb_stream_t stream);

/* Eq. 12 async application of P payloads in worker order: theta :=
 * (-eta_p/(1+tau_p)) * decompress(msg_p) + theta for p = 0..P-1
 * (strategies.hpp:125-129 applied as in trainer.hpp:245-254).
 * scale_per_worker (host, P doubles) = eta/(1+tau_p). */
PSB_API psb_status psb_sparse_async_apply(psb_ctx* ctx, psb_compressor c, psb_dtype dt, int P,
                                  const void* payloads, size_t k, const double* scale_per_worker,
                                  void* theta, size_t n, psb_stream_t stream);

/* compressor none: allreduce_mean over P dense buffers [P][n] + SGD. */
PSB_API psb_status psb_dense_mean_sgd(psb_ctx* ctx, psb_dtype dt, int P, const void* bufs, psb_order order,
                              const psb_topology* topo, double lr, void* theta, size_t n,
                              void* mean_out, psb_stream_t stream);

/* 1-bit: words [P][ceil(n/32)], scales (device, P doubles) -> mean + SGD. */
PSB_API psb_status psb_onebit_mean_sgd(psb_ctx* ctx, psb_dtype dt, int P, const uint32_t* words,
                               const double* scales, psb_order order, const psb_topology* topo,
                               double lr, void* theta, size_t n, void* mean_out,
                               psb_stream_t stream);

/* Momentum SGD pass (north-star a24, this build's rule -- no reference code):
 * m = RN(RN(beta*m) + mean); theta = RN(RN(-lr*m) + theta), dense over n. */
PSB_API psb_status psb_momentum_sgd(psb_ctx* ctx, psb_dtype dt, const void* mean, void* m, void* theta,
                            double beta, double lr, size_t n, psb_stream_t stream);

/* ------------------------------------------------------- step drivers */
typedef struct {
  psb_compressor compressor;
  psb_dtype dtype;
  size_t n;          /* gradient length */
  size_t k;          /* top-k per worker (TOPK, TOPK_Q8) */
  uint32_t q8_block; /* block size for PSB_COMP_Q8 (e.g. 256) */
  int workers;       /* local virtual workers W: g and r hold W rows of n */
  const void* g;     /* [W][n] this rank's gradients */
  void* r;           /* [W][n] EF residuals, or NULL (no error feedback) */
  void* theta;       /* [n] replica of the parameters (identical on all ranks) */
  double lr;
  psb_order order;
  psb_topology topo; /* for PSB_ORDER_HIER; zeros = flat (devices_per_node = P) */
  void* mean_out;    /* optional dense [n] aggregated mean (parity/debug) */
  /* Momentum SGD (north-star a24; NO reference code -- the rule is this
   * build's, restated in oracle/psb_oracle.c:orc_momentum): when m is
   * non-NULL, with the aggregated mean g^ of the step,
   *   m = RN(RN(beta * m) + g^);  theta = RN(RN(-lr * m) + theta)
   * as a dense pass over n (sync steps, compressors NONE / ONEBIT / TOPK /
   * TOPK_Q8).  Zero-initialised trailing fields keep plain SGD. */
  void* m;           /* [n] momentum buffer (caller-owned, persistent), or NULL */
  double beta;
} psb_step_desc;

/* sync_data_parallel_step (strategies.hpp:86-121) across W local workers x
 * nranks ranks (P = W * nranks, worker id = rank*W + w): per-worker EF
 * compression, one exchange (NCCL allgather of payloads, or the dense 8-bit
 * all-to-all + allgather for PSB_COMP_Q8), then the fused mean + SGD apply.
 * theta is updated in place identically on every rank. */
PSB_API psb_status psb_sync_step(psb_ctx* ctx, const psb_step_desc* d, psb_stream_t stream);

/* One round of the bounded-staleness async loop (trainer.hpp:244-255) for the
 * P workers: each worker's EF-compressed message is applied in worker order
 * with scale lr/(1+tau_p), tau_p = min(*global_updates + p, p mod (s+1))
 * where s = staleness_bound (s = 3 reproduces the reference's fixed pattern).
 * *global_updates (host, in/out) advances by P. */
PSB_API psb_status psb_async_round(psb_ctx* ctx, const psb_step_desc* d, uint32_t staleness_bound,
                           uint64_t* global_updates, psb_stream_t stream);

/* Bounded-staleness pipeline of psb_async_round (the async branch's overlap,
 * driven by CUDA streams and events instead of host threads): with enable =
 * 1, round r's exchange + apply run on a ctx-owned stream, gated by an event
 * recorded after round r's compression on `stream`, so round r+1's
 * compression overlaps round r's apply; payload slots are double-buffered
 * (round r+2 waits for round r's apply).  theta is then up to one round
 * behind `stream`: psb_async_sync makes `stream` wait for every pending
 * apply (call it before reading theta, and before ending a CUDA-graph capture
 * of rounds).  Results are bitwise those of serial rounds (same kernels, same
 * per-buffer order).  Pull (mode 1) and NCCL (mode 0) exchanges pipeline;
 * the other peer modes run serially.  psb_check drains the apply stream. */
PSB_API psb_status psb_async_pipeline(psb_ctx* ctx, int enable);
PSB_API psb_status psb_async_sync(psb_ctx* ctx, psb_stream_t stream);

#ifdef __cplusplus
}
#endif

#endif /* PSB_H_ */
