/*
 * psb_oracle.c -- CPU restatement of the reference data-parallel gradient path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the checker, never the product:
 * only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load it.  The product path (paper_2506_17551_b200 + libpsb.so) never links
 * or calls it and fails loudly when the CUDA library is missing.
 *
 * Every function restates one piece of the reference (parsim, header-only
 * C++20, /root/reference/proj/include/parsim) and cites the lines it follows.
 * Built with -ffp-contract=off so a*x+y is a separate multiply and add, as in
 * the reference on x86-64 (SURVEY.md App. A trap 5).
 *
 * Parity pinning: tests/test_oracle.py checks this restatement bit-for-bit
 * against the reference itself (oracle/_ref/libparsim_ref.so, compiled from
 * the unmodified headers by oracle/Makefile) and against the golden fixtures
 * in tests/golden/ that were generated from it.  The 8-bit block quantizer
 * and int8 top-k values have no reference code: for those this
 * file IS the spec ("parity unpinned" against the reference, pinned against
 * this restatement), see DESIGN.md section "Unpinned semantics".
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_EINVAL 1
#define ORC_ENONFINITE 2

/* ---------------------------------------------------------------- PRNG */

/* mix64: parsim/numerics.hpp:181-186 (SplitMix64 finalizer). */
uint64_t orc_mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

/* SeededRng::next_u64 stream: parsim/numerics.hpp:152-162.  KAT in
 * proj/tests/test_numerics.cpp:66-77. */
void orc_splitmix_stream(uint64_t seed, size_t n, uint64_t* out) {
  uint64_t s = seed;
  for (size_t i = 0; i < n; ++i) {
    s += 0x9E3779B97F4A7C15ULL;
    uint64_t z = s;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    out[i] = z ^ (z >> 31);
  }
}

/* ------------------------------------------------ synthetic gradients
 * Counter-based generator (SURVEY.md 8d "Synthetic inputs"); the device
 * kernel psb_generate implements the same integer/fp32 recipe, so host and
 * device produce identical bits.  dist: 0 uniform, 1 LLM-rec, 2 ties.      */
static inline float u24(uint64_t h) { return (float)(h >> 40) * 0x1.0p-24f; }

static inline float irwin4(uint64_t base, uint64_t i) {
  float a = u24(orc_mix64(base + 4 * i + 0));
  float b = u24(orc_mix64(base + 4 * i + 1));
  float c = u24(orc_mix64(base + 4 * i + 2));
  float d = u24(orc_mix64(base + 4 * i + 3));
  return ((a + b) + (c + d)) - 2.0f;
}

void orc_generate(int dist, uint64_t seed, uint32_t rank, uint32_t step, size_t n, float* out) {
  uint64_t base = orc_mix64(seed ^ (((uint64_t)rank << 32) | (uint64_t)step));
  uint64_t base_row = orc_mix64(base ^ 0x5851F42D4C957F2DULL);
  size_t n_emb = (n * 3 / 5) & ~(size_t)63;
  for (size_t i = 0; i < n; ++i) {
    float g;
    if (dist == 0) {
      g = 2.0f * u24(orc_mix64(base + i)) - 1.0f;
    } else if (dist == 2) {
      uint64_t v = orc_mix64(base + i) >> 40;
      int bucket = (int)((v * 5) >> 24);
      g = (float)(bucket - 2) * 0.25f;
    } else {
      float z = irwin4(base, i) * 1.7320508e-3f;
      if (i < n_emb) {
        uint64_t row = i >> 6;
        uint64_t zr = orc_mix64(base_row + 2 * row) >> 40;
        if (((zr * 20) >> 24) < 19) {
          g = 0.0f;
        } else {
          uint64_t e = ((orc_mix64(base_row + 2 * row + 1) >> 40) * 7) >> 24;
          g = z * ldexpf(1.0f, -(int)e);
        }
      } else {
        g = z;
      }
    }
    out[i] = g;
  }
}

/* ------------------------------------------------------------ top-k
 * compress_topk: parsim/compression.hpp:81-99.  The reference stable-sorts
 * all indices by |g| descending (:85-89; stability = lower index wins a tie),
 * keeps k (:90), sorts them ascending (:91) and gathers g[idx] (:97).
 * Restated as a sort on (bits(|x|) descending, index ascending), which is the
 * same total order for finite values and +-0 (parity fact 1). */
typedef struct {
  uint64_t key;
  uint32_t idx;
} orc_kv;

static int kv_cmp(const void* a, const void* b) {
  const orc_kv* x = (const orc_kv*)a;
  const orc_kv* y = (const orc_kv*)b;
  if (x->key != y->key) return x->key > y->key ? -1 : 1;
  return x->idx < y->idx ? -1 : (x->idx > y->idx ? 1 : 0);
}

static int u32_cmp(const void* a, const void* b) {
  uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
  return x < y ? -1 : (x > y ? 1 : 0);
}

static uint64_t key_f32(float x) {
  uint32_t u;
  memcpy(&u, &x, 4);
  return u & 0x7fffffffu;
}
static uint64_t key_f64(double x) {
  uint64_t u;
  memcpy(&u, &x, 8);
  return u & 0x7fffffffffffffffULL;
}

static int topk_indices(const void* x, int is64, size_t n, size_t k, uint32_t* idx) {
  if (k < 1 || k > n) return ORC_EINVAL; /* compression.hpp:82-84 */
  orc_kv* kv = (orc_kv*)malloc(n * sizeof(orc_kv));
  if (!kv) return ORC_EINVAL;
  for (size_t i = 0; i < n; ++i) {
    kv[i].key = is64 ? key_f64(((const double*)x)[i]) : key_f32(((const float*)x)[i]);
    kv[i].idx = (uint32_t)i;
  }
  qsort(kv, n, sizeof(orc_kv), kv_cmp);
  for (size_t j = 0; j < k; ++j) idx[j] = kv[j].idx;
  free(kv);
  qsort(idx, k, sizeof(uint32_t), u32_cmp);
  return ORC_OK;
}

int orc_topk_f32(const float* x, size_t n, size_t k, uint32_t* idx, float* val) {
  int st = topk_indices(x, 0, n, k, idx);
  if (st) return st;
  for (size_t j = 0; j < k; ++j) val[j] = x[idx[j]];
  return ORC_OK;
}

int orc_topk_f64(const double* x, size_t n, size_t k, uint32_t* idx, double* val) {
  int st = topk_indices(x, 1, n, k, idx);
  if (st) return st;
  for (size_t j = 0; j < k; ++j) val[j] = x[idx[j]];
  return ORC_OK;
}

/* ef_compress_step with the top-k compressor: parsim/compression.hpp:146-157.
 * p = r + g (:150-151), msg = compress_topk(p) (:152), r' = p - decompress(msg)
 * (:153-154), i.e. +0.0 at selected positions and p elsewhere (parity fact 2),
 * check_finite(r') (:155).  r == NULL means a transient zero residual
 * (parsim/strategies.hpp:97-102): p = g and nothing is written back. */
int orc_ef_topk_f32(const float* g, float* r, size_t n, size_t k, uint32_t* idx, float* val) {
  float* p = (float*)malloc(n * sizeof(float));
  int nonfinite = 0;
  for (size_t i = 0; i < n; ++i) p[i] = r ? (r[i] + g[i]) : g[i];
  int st = orc_topk_f32(p, n, k, idx, val);
  if (st) {
    free(p);
    return st;
  }
  for (size_t j = 0; j < k; ++j) p[idx[j]] = p[idx[j]] - p[idx[j]]; /* x - x = +0 */
  for (size_t i = 0; i < n; ++i) {
    if (!isfinite(p[i])) nonfinite = 1;
    if (r) r[i] = p[i];
  }
  free(p);
  return nonfinite ? ORC_ENONFINITE : ORC_OK;
}

int orc_ef_topk_f64(const double* g, double* r, size_t n, size_t k, uint32_t* idx, double* val) {
  double* p = (double*)malloc(n * sizeof(double));
  int nonfinite = 0;
  for (size_t i = 0; i < n; ++i) p[i] = r ? (r[i] + g[i]) : g[i];
  int st = orc_topk_f64(p, n, k, idx, val);
  if (st) {
    free(p);
    return st;
  }
  for (size_t j = 0; j < k; ++j) p[idx[j]] = p[idx[j]] - p[idx[j]];
  for (size_t i = 0; i < n; ++i) {
    if (!isfinite(p[i])) nonfinite = 1;
    if (r) r[i] = p[i];
  }
  free(p);
  return nonfinite ? ORC_ENONFINITE : ORC_OK;
}

/* ------------------------------------------------------------- 1-bit
 * compress_onebit: parsim/compression.hpp:67-77.  scale = l1_norm(p)/dim with
 * l1_norm a sequential f64 left fold (parsim/numerics.hpp:96-101); sign bit
 * set iff p >= 0 (:74, sign(0) = +1).  Bits are packed into little-endian
 * u32 words: bit i%32 of word i/32, byte-identical to the reference's
 * sign_bytes (bit i%8 of byte i/8, compression.hpp:31-40).  decompress gives
 * +-scale (:113-120); the residual is p - (+-scale) (:153-154).  The f32
 * variant uses (float)scale as the decompressed magnitude. */
int orc_ef_onebit_f32(const float* g, float* r, size_t n, uint32_t* words, double* scale_out) {
  if (n == 0) return ORC_EINVAL;
  float* p = (float*)malloc(n * sizeof(float));
  double l1 = 0.0;
  for (size_t i = 0; i < n; ++i) {
    p[i] = r ? (r[i] + g[i]) : g[i];
    l1 += fabs((double)p[i]);
  }
  double scale = l1 / (double)n;
  float s = (float)scale;
  memset(words, 0, ((n + 31) / 32) * sizeof(uint32_t));
  int nonfinite = 0;
  for (size_t i = 0; i < n; ++i) {
    int pos = p[i] >= 0.0f;
    if (pos) words[i / 32] |= (1u << (i % 32));
    float res = p[i] - (pos ? s : -s);
    if (!isfinite(res)) nonfinite = 1;
    if (r) r[i] = res;
  }
  *scale_out = scale;
  free(p);
  return nonfinite ? ORC_ENONFINITE : ORC_OK;
}

int orc_ef_onebit_f64(const double* g, double* r, size_t n, uint32_t* words, double* scale_out) {
  if (n == 0) return ORC_EINVAL;
  double* p = (double*)malloc(n * sizeof(double));
  double l1 = 0.0;
  for (size_t i = 0; i < n; ++i) {
    p[i] = r ? (r[i] + g[i]) : g[i];
    l1 += fabs(p[i]);
  }
  double scale = l1 / (double)n;
  memset(words, 0, ((n + 31) / 32) * sizeof(uint32_t));
  int nonfinite = 0;
  for (size_t i = 0; i < n; ++i) {
    int pos = p[i] >= 0.0;
    if (pos) words[i / 32] |= (1u << (i % 32));
    double res = p[i] - (pos ? scale : -scale);
    if (!isfinite(res)) nonfinite = 1;
    if (r) r[i] = res;
  }
  *scale_out = scale;
  free(p);
  return nonfinite ? ORC_ENONFINITE : ORC_OK;
}

/* ------------------------------------------------------- fold orders
 * allreduce_mean: parsim/collectives.hpp:135-154, with the three canonical
 * orders: naive (:68-73), ring (:77-94; pipelined_ring -> ring, :142-143) and
 * hierarchical (:99-128).  The mean is sum * (1/P) (:71, :92, :126).
 * bufs is P rows of n.  order: 0 naive, 1 ring, 2 hierarchical. */
#define FOLD_BODY(T)                                                              \
  if (P < 1) return ORC_EINVAL;                                                   \
  const T inv = (T)(1.0 / (double)P);                                             \
  if (order == 0) {                                                               \
    for (size_t i = 0; i < n; ++i) {                                              \
      T acc = bufs[i];                                                            \
      for (int p = 1; p < P; ++p) acc = acc + bufs[(size_t)p * n + i];            \
      out[i] = acc * inv;                                                         \
    }                                                                             \
  } else if (order == 1) {                                                        \
    for (int j = 0; j < P; ++j) {                                                 \
      size_t lo = (size_t)j * n / (size_t)P, hi = (size_t)(j + 1) * n / (size_t)P; \
      int start = (j + 1) % P;                                                    \
      for (size_t i = lo; i < hi; ++i) {                                          \
        T acc = bufs[(size_t)start * n + i];                                      \
        for (int s = 1; s < P; ++s) acc = acc + bufs[(size_t)((start + s) % P) * n + i]; \
        out[i] = acc * inv;                                                       \
      }                                                                           \
    }                                                                             \
  } else if (order == 2) {                                                        \
    if (dpn < 1 || npr < 1) return ORC_EINVAL;                                    \
    size_t per_rack = (size_t)dpn * npr;                                          \
    size_t nodes = ((size_t)P + dpn - 1) / dpn;                                   \
    size_t npru = (per_rack + dpn - 1) / dpn;                                     \
    for (size_t i = 0; i < n; ++i) {                                              \
      T total = 0, rack = 0;                                                      \
      int have_total = 0;                                                         \
      for (size_t nb = 0; nb < nodes; nb += npru) {                               \
        int have_rack = 0;                                                        \
        for (size_t nd = nb; nd < nodes && nd < nb + npru; ++nd) {                \
          size_t base = nd * dpn;                                                 \
          T node = bufs[base * n + i];                                            \
          for (size_t p = base + 1; p < base + dpn && p < (size_t)P; ++p)         \
            node = node + bufs[p * n + i];                                        \
          rack = have_rack ? rack + node : node;                                  \
          have_rack = 1;                                                          \
        }                                                                         \
        total = have_total ? total + rack : rack;                                 \
        have_total = 1;                                                           \
      }                                                                           \
      out[i] = total * inv;                                                       \
    }                                                                             \
  } else {                                                                        \
    return ORC_EINVAL;                                                            \
  }                                                                               \
  return ORC_OK;

int orc_fold_mean_f32(int order, int P, size_t n, const float* bufs, uint32_t dpn, uint32_t npr,
                      float* out) {
  FOLD_BODY(float)
}

int orc_fold_mean_f64(int order, int P, size_t n, const double* bufs, uint32_t dpn, uint32_t npr,
                      double* out) {
  FOLD_BODY(double)
}

/* -------------------------------------------------------------- SGD
 * vec_axpy(-lr, mean, theta): parsim/numerics.hpp:70-78 (a*x + y, separate
 * multiply and add) + check_finite (:76).  In place on theta.  The f32
 * variant rounds a once to float. */
int orc_axpy_f32(double a, const float* x, float* y, size_t n) {
  float af = (float)a;
  int nonfinite = 0;
  for (size_t i = 0; i < n; ++i) {
    float prod = af * x[i];
    y[i] = prod + y[i];
    if (!isfinite(y[i])) nonfinite = 1;
  }
  return nonfinite ? ORC_ENONFINITE : ORC_OK;
}

int orc_axpy_f64(double a, const double* x, double* y, size_t n) {
  int nonfinite = 0;
  for (size_t i = 0; i < n; ++i) {
    double prod = a * x[i];
    y[i] = prod + y[i];
    if (!isfinite(y[i])) nonfinite = 1;
  }
  return nonfinite ? ORC_ENONFINITE : ORC_OK;
}

/* async_step: parsim/strategies.hpp:125-129.  scale = eta/(1+tau) in f64
 * (:127), then vec_axpy(-scale, g, theta) (:128). */
double orc_async_scale(double eta, uint64_t tau) { return eta / (1.0 + (double)tau); }

/* ---------------------------------------------- 8-bit block quantizer
 * NO REFERENCE CODE (multi-bit quantization is a non-goal):
 * this restatement is the spec the CUDA kernel is pinned to.
 *   per block of B consecutive elements (last block may be short):
 *     absmax = max |p_i|;  scale = absmax / 127.0f   (IEEE f32 division)
 *     q_i = scale > 0 ? clamp(rint(p_i / scale), -127, 127) : 0
 *           (IEEE f32 division; rint = round-half-to-even)
 *     xhat_i = (float)q_i * scale;  EF: r_i = p_i - xhat_i
 * p = r + g when r != NULL (error feedback, compression.hpp:150-151 shape). */
int orc_q8_quant(const float* x, float* r, size_t n, uint32_t block, int8_t* codes, float* scales) {
  if (block == 0) return ORC_EINVAL;
  int nonfinite = 0;
  size_t nb = (n + block - 1) / block;
  float* p = (float*)malloc((size_t)block * sizeof(float));
  for (size_t b = 0; b < nb; ++b) {
    size_t lo = b * block, hi = lo + block < n ? lo + block : n;
    float amax = 0.0f;
    for (size_t i = lo; i < hi; ++i) {
      p[i - lo] = r ? (r[i] + x[i]) : x[i];
      float a = fabsf(p[i - lo]);
      if (!isfinite(a)) nonfinite = 1;
      if (a > amax) amax = a;
    }
    float scale = amax / 127.0f;
    scales[b] = scale;
    for (size_t i = lo; i < hi; ++i) {
      int q = 0;
      if (scale > 0.0f) {
        float t = rintf(p[i - lo] / scale);
        q = t > 127.0f ? 127 : (t < -127.0f ? -127 : (int)t);
      }
      codes[i] = (int8_t)q;
      if (r) {
        float xhat = (float)q * scale;
        r[i] = p[i - lo] - xhat;
      }
    }
  }
  free(p);
  return nonfinite ? ORC_ENONFINITE : ORC_OK;
}

void orc_q8_dequant(const int8_t* codes, const float* scales, size_t n, uint32_t block, float* out) {
  for (size_t i = 0; i < n; ++i) out[i] = (float)codes[i] * scales[i / block];
}

/* ------------------------------------------------------------ wire format
 * parsim/compression.hpp:159-239, little-endian throughout:
 *   Dense:   u64 dim | dim x f64
 *   SignBit: u64 dim | f64 scale | ceil(dim/8) sign bytes (bit i%8 of byte i/8)
 *   TopK:    u64 dim | u64 count | count x (u64 index, f64 value)
 * Values are carried as f64 (the reference's DenseVector); f32 payloads widen
 * exactly.  Decoders return -1 on truncation ("wire_decode: truncated ..."). */
static void put_u64(uint8_t* o, uint64_t v) {
  for (int b = 0; b < 8; ++b) o[b] = (uint8_t)(v >> (8 * b));
}
static uint64_t get_u64(const uint8_t* i) {
  uint64_t v = 0;
  for (int b = 0; b < 8; ++b) v |= (uint64_t)i[b] << (8 * b);
  return v;
}
static void put_f64(uint8_t* o, double v) {
  uint64_t u;
  memcpy(&u, &v, 8);
  put_u64(o, u);
}
static double get_f64(const uint8_t* i) {
  uint64_t u = get_u64(i);
  double v;
  memcpy(&v, &u, 8);
  return v;
}

size_t orc_wire_encode_topk(uint64_t dim, const uint32_t* idx, const double* val, size_t k, uint8_t* out) {
  put_u64(out, dim);
  put_u64(out + 8, (uint64_t)k);
  for (size_t j = 0; j < k; ++j) {
    put_u64(out + 16 + 16 * j, idx[j]);
    put_f64(out + 24 + 16 * j, val[j]);
  }
  return 16 + 16 * k;
}

/* count of the message, or -1 if truncated; idx/val may be NULL to query */
long long orc_wire_decode_topk(const uint8_t* in, size_t nbytes, uint64_t* dim, uint64_t* idx, double* val) {
  if (nbytes < 16) return -1;
  *dim = get_u64(in);
  const uint64_t count = get_u64(in + 8);
  if (count > (nbytes - 16) / 16) return -1;
  if (idx && val)
    for (uint64_t j = 0; j < count; ++j) {
      idx[j] = get_u64(in + 16 + 16 * j);
      val[j] = get_f64(in + 24 + 16 * j);
    }
  return (long long)count;
}

size_t orc_wire_encode_signbit(uint64_t dim, double scale, const uint32_t* words, uint8_t* out) {
  put_u64(out, dim);
  put_f64(out + 8, scale);
  const size_t nb = (size_t)((dim + 7) / 8);
  for (size_t b = 0; b < nb; ++b) out[16 + b] = (uint8_t)(words[b / 4] >> (8 * (b % 4)));
  return 16 + nb;
}

size_t orc_wire_encode_dense(uint64_t dim, const double* x, uint8_t* out) {
  put_u64(out, dim);
  for (uint64_t i = 0; i < dim; ++i) put_f64(out + 8 + 8 * i, x[i]);
  return 8 + 8 * (size_t)dim;
}

/* ------------------------------------------------------------ momentum SGD
 * North-star a24, NO reference code: this build's rule, with
 * the reference's no-FMA convention (separate RN multiply and add):
 *   m = RN(RN(beta * m) + mean);  theta = RN(RN(-lr * m) + theta)          */
void orc_momentum_f32(const float* mean, float* m, float* theta, double beta, double lr, size_t n) {
  const float b = (float)beta, c = (float)(-lr);
  for (size_t i = 0; i < n; ++i) {
    volatile float t = b * m[i];
    m[i] = t + mean[i];
    volatile float u = c * m[i];
    theta[i] = u + theta[i];
  }
}
void orc_momentum_f64(const double* mean, double* m, double* theta, double beta, double lr, size_t n) {
  const double c = -lr;
  for (size_t i = 0; i < n; ++i) {
    volatile double t = beta * m[i];
    m[i] = t + mean[i];
    volatile double u = c * m[i];
    theta[i] = u + theta[i];
  }
}
