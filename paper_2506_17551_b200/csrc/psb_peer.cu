// psb_peer.cu -- payload exchange over NVLink peer memory (CUDA IPC).
//
// Replaces the NCCL all-gather of the compressed payloads (the reference's
// message exchange: every worker's (indices, values) reach every replica,
// parsim/strategies.hpp:104-112) with a pull over NVLink/NVSwitch:
//   * every rank owns one "arena" (cudaMalloc, exported with CUDA IPC and
//     mapped by every peer): a 4 KB header of flags followed by the P payload
//     slots, laid out exactly like the gather buffer (slot gid = worker id);
//   * a rank's compressor writes its payloads straight into its own slots;
//   * k_peer_signal bumps the rank's device-side sequence number and
//     publishes it into every peer's header (st.release.sys);
//   * k_peer_pull waits until every peer has published the same sequence
//     number, copies the peers' slots from their arenas into its own (int4
//     loads over NVLink, all SMs), then acknowledges to every peer;
//   * k_peer_wait_ack, launched before the next compression, waits until
//     every peer has acknowledged the previous payload, so a slot is never
//     rewritten while a peer is still reading it.
// The sequence numbers live on the device, so captured CUDA graphs can be
// replayed any number of times.  All waits are bounded (~10 s): on timeout
// the kernel sets flag bit 3 and psb_check reports PSB_ESTATE instead of
// hanging.
#include <cstdio>
#include <cstdlib>

#include "psb_internal.cuh"
#include "psb_debug.h"

namespace {

constexpr size_t kHdrBytes = 4096;
#ifndef PSB_PULL_U
#define PSB_PULL_U 4  // int4 loads in flight per thread in the pull
#endif
#ifndef PSB_PULL_CTAS
#define PSB_PULL_CTAS 4  // pull CTAs per SM
#endif
// header words: [0,32) ready[p]: p's payloads of seq are in place
//               [32,64) ackp[p]: p has finished reading our payloads of seq
//               [64,96) upd[p]: p's update list of seq is complete (sharded apply)
//               [96,128) acku[p]: p has finished reading our update list of seq
//               128 local seq, 129/130 last-CTA counters, 131 update-list length
constexpr int kReady = 0, kAck = 32, kUpd = 64, kAckU = 96, kSeq = 128, kCtr = 129, kCtr2 = 130,
              kListCnt = 131;
constexpr unsigned long long kSpinNs = 10ull * 1000 * 1000 * 1000;

struct PeerPtrs {
  uint8_t* base[PSB_MAX_P];  // every rank's arena (own one included)
};

__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned long long now_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// Waits until hdr[slot0 + p] >= target for every peer p != rank; false on timeout.
__device__ bool wait_all(const uint32_t* hdr, int slot0, int R, int rank, uint32_t target) {
  const unsigned long long t0 = now_ns();
  for (int p = 0; p < R; ++p) {
    if (p == rank) continue;
    while ((int32_t)(ld_acquire_sys(hdr + slot0 + p) - target) < 0) {
      if (now_ns() - t0 > kSpinNs) return false;
      __nanosleep(64);
    }
  }
  return true;
}

// Step start: every peer is done with our previous payloads and update list;
// then the list may be reset.
__global__ void k_peer_wait_ack(uint32_t* hdr, int R, int rank, uint32_t* flags) {
  const uint32_t s = hdr[kSeq];
  if (!wait_all(hdr, kAck, R, rank, s) || !wait_all(hdr, kAckU, R, rank, s)) atomicOr(flags, 8u);
  hdr[kListCnt] = 0;
}

// Last CTA out (counter word ctr) publishes value s into slot0 + rank of every peer.
__device__ void last_cta_publish(const PeerPtrs& pp, int R, int rank, int ctr, int slot0, int slot1,
                                 uint32_t s) {
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t* hdr = reinterpret_cast<uint32_t*>(pp.base[rank]);
    __threadfence();
    if (atomicAdd(hdr + ctr, 1u) == gridDim.x - 1) {
      hdr[ctr] = 0;
      __threadfence_system();
      for (int p = 0; p < R; ++p) {
        if (p == rank) continue;
        uint32_t* ph = reinterpret_cast<uint32_t*>(pp.base[p]);
        st_release_sys(ph + slot0 + rank, s);
        if (slot1 >= 0) st_release_sys(ph + slot1 + rank, s);
      }
    }
  }
}

__global__ void k_peer_signal(PeerPtrs pp, int R, int rank) {
  uint32_t* hdr = reinterpret_cast<uint32_t*>(pp.base[rank]);
  const uint32_t s = hdr[kSeq] + 1;
  hdr[kSeq] = s;
  __threadfence_system();  // payload writes (earlier kernels) before the flag
  for (int p = 0; p < R; ++p)
    if (p != rank) st_release_sys(reinterpret_cast<uint32_t*>(pp.base[p]) + kReady + rank, s);
}

// Copies every peer's rank range [p*bpr, (p+1)*bpr) of the payload region
// from its arena into ours (bpr is a multiple of 16), plus, when tw > 0, its
// tw words of per-segment offset rows at tab_off + p*tw*4; then acknowledges.
// CTAs are dealt round-robin to the peers and each waits only for its own
// peer, so a fast peer's payload moves while a slower one still compresses.
__global__ void __launch_bounds__(256) k_peer_pull(PeerPtrs pp, int R, int rank, size_t bpr, size_t tab_off,
                                                   size_t tw, uint32_t* flags) {
  uint32_t* hdr = reinterpret_cast<uint32_t*>(pp.base[rank]);
  const uint32_t s = hdr[kSeq];
  const int npeer = R - 1;
  const int pi = (int)(blockIdx.x % npeer);
  const int p = pi + (pi >= rank);
  const uint32_t cta = blockIdx.x / npeer;                                        // CTA index among p's
  const uint32_t ncta = (gridDim.x - pi + npeer - 1) / npeer;                     // CTAs serving p
  __shared__ int ok;
  if (threadIdx.x == 0) {
    const unsigned long long t0 = now_ns();
    ok = 1;
    while ((int32_t)(ld_acquire_sys(hdr + kReady + p) - s) < 0) {
      if (now_ns() - t0 > kSpinNs) {
        ok = 0;
        break;
      }
      __nanosleep(64);
    }
  }
  __syncthreads();
  if (!ok) {
    if (threadIdx.x == 0) atomicOr(flags, 8u);
  } else {
    const size_t nv = bpr / 16;
    const size_t stride = (size_t)ncta * blockDim.x;
    const uint8_t* src = pp.base[p] + kHdrBytes + (size_t)p * bpr;
    uint8_t* dst = pp.base[rank] + kHdrBytes + (size_t)p * bpr;
    constexpr int U = PSB_PULL_U;
    for (size_t t0 = (size_t)cta * blockDim.x + threadIdx.x; t0 < nv; t0 += U * stride) {
      int4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (t0 + u * stride < nv) v[u] = __ldcs(reinterpret_cast<const int4*>(src) + t0 + u * stride);
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (t0 + u * stride < nv) __stcg(reinterpret_cast<int4*>(dst) + t0 + u * stride, v[u]);
    }
    if (tw) {
      const uint32_t* ts = reinterpret_cast<const uint32_t*>(pp.base[p] + kHdrBytes + tab_off) + (size_t)p * tw;
      uint32_t* td = reinterpret_cast<uint32_t*>(pp.base[rank] + kHdrBytes + tab_off) + (size_t)p * tw;
      for (size_t t = (size_t)cta * blockDim.x + threadIdx.x; t < tw; t += stride) td[t] = ts[t];
    }
  }
  // last CTA out acknowledges to every peer (no update list in this mode)
  last_cta_publish(pp, R, rank, kCtr, kAck, kAckU, s);
}

// ------------------------------------------------------ sharded apply
// Rank r folds only the segments [seg_lo, seg_hi) of the index space; it
// pulls from every worker's payload just the entries inside them (the
// producer's per-segment offsets tell where), folds them locally into theta
// and an update list (index, new theta), and every rank then applies the
// other ranks' lists.  NVLink traffic per rank: ~W*k payload entries in, the
// other shards' update lists in -- instead of all P payloads.
struct ShardArgs {
  PeerPtrs pp;
  int R, rank, W, P, q8;
  size_t blk, voff, soff;  // payload block layout (psb_payload_bytes)
  size_t tab_off;          // per-worker segment offset rows, from the payload region start
  uint32_t nseg;
  uint32_t* range;         // [seg_lo, seg_hi) of this rank, written by k_shard_plan
  uint32_t* sidx;  // local flat slices: indices
  void* sval;      //                    values (T)
  uint32_t* srow;  // P x (seg_hi - seg_lo + 1) offsets into the flat slices
  uint32_t* flags;
};

__device__ __forceinline__ const uint32_t* shard_tab(const ShardArgs& a, int q) {
  return reinterpret_cast<const uint32_t*>(a.pp.base[q / a.W] + kHdrBytes + a.tab_off) + (size_t)q * (a.nseg + 1);
}

// Balanced shard boundaries (one CTA, every rank computes the same ones):
// rank r takes segments [b_r, b_{r+1}) with b_r the first segment whose
// cumulative entry count over all P workers, cum(s) = sum_q tab_q[s], reaches
// r*P*k/R.  cum is sampled at 1024 points, then the bracketing interval is
// searched exactly.
__global__ void __launch_bounds__(1024) k_shard_plan(ShardArgs a, uint32_t k) {
  uint32_t* hdr = reinterpret_cast<uint32_t*>(a.pp.base[a.rank]);
  __shared__ int ok;
  __shared__ unsigned long long samp[1025];
  __shared__ uint32_t bnd[2];
  if (threadIdx.x == 0) ok = wait_all(hdr, kReady, a.R, a.rank, hdr[kSeq]);
  __syncthreads();
  if (!ok) {
    if (threadIdx.x == 0) atomicOr(a.flags, 8u);
    return;
  }
  // cost model: entries + one average segment's worth per segment (the
  // per-segment fixed cost of the fold), so sparse regions get fewer segments
  const unsigned long long avg = ((unsigned long long)a.P * k + a.nseg - 1) / a.nseg;
  auto cum = [&](uint32_t sg) {
    unsigned long long c = 0;
    for (int q = 0; q < a.P; ++q) c += shard_tab(a, q)[sg];
    return c + avg * sg;
  };
  const uint32_t t = threadIdx.x;
  const uint32_t ns = a.nseg;
  samp[t] = cum((uint32_t)((unsigned long long)t * ns / 1024));
  if (t == 0) samp[1024] = (unsigned long long)a.P * k + avg * ns;
  __syncthreads();
  const unsigned long long total = (unsigned long long)a.P * k + avg * ns;
  for (int side = 0; side < 2; ++side) {
    const int r = a.rank + side;
    const unsigned long long target = total * (unsigned long long)r / (unsigned long long)a.R;
    if (r == 0 || r == a.R) {
      if (t == 0) bnd[side] = r == 0 ? 0u : ns;
      continue;
    }
    // last sample below target: the boundary lies in (s_i, s_{i+1}]
    __shared__ uint32_t si;
    if (t < 1024 && samp[t] < target && samp[t + 1] >= target) si = t;
    if (t == 0 && samp[0] >= target) si = 0xffffffffu;
    __syncthreads();
    if (si == 0xffffffffu) {
      if (t == 0) bnd[side] = 0;
    } else {
      const uint32_t lo = (uint32_t)((unsigned long long)si * ns / 1024);
      const uint32_t hi = si + 1 == 1024 ? ns : (uint32_t)((unsigned long long)(si + 1) * ns / 1024);
      if (t == 0) bnd[side] = hi;
      __syncthreads();
      for (uint32_t sg = lo + 1 + t; sg < hi; sg += blockDim.x)
        if (cum(sg) >= target) atomicMin(&bnd[side], sg);
    }
    __syncthreads();
  }
  if (t == 0) {
    a.range[0] = bnd[0];
    a.range[1] = max(bnd[0], bnd[1]);
  }
}

template <class T>
__global__ void __launch_bounds__(256) k_shard_pull(ShardArgs a) {
  uint32_t* hdr = reinterpret_cast<uint32_t*>(a.pp.base[a.rank]);
  const uint32_t s = hdr[kSeq];
  const uint32_t seg_lo = a.range[0], seg_hi = a.range[1];
  __shared__ uint32_t s_a[PSB_MAX_P], s_base[PSB_MAX_P + 1];  // (peers are ready: k_shard_plan waited)
  auto tab = [&](int q) { return shard_tab(a, q); };
  auto block = [&](int q) { return a.pp.base[q / a.W] + kHdrBytes + (size_t)q * a.blk; };
  if (threadIdx.x < 32) {
    const int q = threadIdx.x;
    uint32_t len = 0, lo = 0;
    if (q < a.P) {
      lo = tab(q)[seg_lo];
      len = tab(q)[seg_hi] - lo;
    }
    uint32_t incl = len;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
      if (q >= o) incl += t;
    }
    if (q < a.P) {
      s_a[q] = lo;
      s_base[q + 1] = incl;
    }
    if (q == 0) s_base[0] = 0;
  }
  __syncthreads();
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  const size_t gt = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  // rows, rebased onto the flat slices
  const uint32_t nr = seg_hi - seg_lo + 1;
  for (size_t t = gt; t < (size_t)a.P * nr; t += stride) {
    const int q = (int)(t / nr);
    const uint32_t sj = (uint32_t)(t - (size_t)q * nr);
    a.srow[t] = s_base[q] + (tab(q)[seg_lo + sj] - s_a[q]);
  }
  // entries; a batch issues all of its remote loads first
  const uint32_t total = s_base[a.P];
  T* sval = reinterpret_cast<T*>(a.sval);
  constexpr int U = 4;
  for (size_t e0 = gt; e0 < total; e0 += U * stride) {
    uint32_t id[U];
    T v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const size_t e = e0 + u * stride;
      if (e < total) {
        int q = 0;
        while (q + 1 < a.P && s_base[q + 1] <= e) ++q;
        const uint32_t j = s_a[q] + (uint32_t)(e - s_base[q]);
        const uint8_t* b = block(q);
        id[u] = reinterpret_cast<const uint32_t*>(b)[j];
        if (a.q8) {
          const int8_t code = reinterpret_cast<const int8_t*>(b + a.voff)[j];
          v[u] = (T)__fmul_rn((float)code, reinterpret_cast<const float*>(b + a.soff)[j >> 7]);
        } else {
          v[u] = reinterpret_cast<const T*>(b + a.voff)[j];
        }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const size_t e = e0 + u * stride;
      if (e < total) {
        a.sidx[e] = id[u];
        sval[e] = v[u];
      }
    }
  }
  last_cta_publish(a.pp, a.R, a.rank, kCtr, kAck, -1, s);  // done with the peers' payloads
}

// Our update list is complete: publish it.
__global__ void k_peer_publish_upd(PeerPtrs pp, int R, int rank) {
  const uint32_t s = reinterpret_cast<uint32_t*>(pp.base[rank])[kSeq];
  __threadfence_system();
  for (int p = 0; p < R; ++p)
    if (p != rank) st_release_sys(reinterpret_cast<uint32_t*>(pp.base[p]) + kUpd + rank, s);
}

// theta[idx] = new value, for every other rank's update list (remote reads).
template <class T>
__global__ void __launch_bounds__(256) k_shard_scatter(PeerPtrs pp, int R, int rank, size_t list_off,
                                                       size_t list_voff, T* __restrict__ theta, uint32_t* flags) {
  uint32_t* hdr = reinterpret_cast<uint32_t*>(pp.base[rank]);
  const uint32_t s = hdr[kSeq];
  __shared__ int ok;
  __shared__ uint32_t s_base[PSB_MAX_P + 1];
  if (threadIdx.x == 0) ok = wait_all(hdr, kUpd, R, rank, s);
  __syncthreads();
  if (!ok) {
    if (threadIdx.x == 0) atomicOr(flags, 8u);
    return;
  }
  if (threadIdx.x < 32) {
    const int q = threadIdx.x;
    uint32_t len = 0;
    if (q < R && q != rank) len = ld_acquire_sys(reinterpret_cast<const uint32_t*>(pp.base[q]) + kListCnt);
    uint32_t incl = len;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
      if (q >= o) incl += t;
    }
    if (q < R) s_base[q + 1] = incl;
    if (q == 0) s_base[0] = 0;
  }
  __syncthreads();
  const uint32_t total = s_base[R];
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  constexpr int U = 8;
  for (size_t e0 = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e0 < total; e0 += U * stride) {
    uint32_t id[U];
    T v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const size_t e = e0 + u * stride;
      if (e < total) {
        int q = 0;
        while (q + 1 < R && s_base[q + 1] <= e) ++q;
        const size_t j = e - s_base[q];
        const uint8_t* b = pp.base[q] + kHdrBytes;
        id[u] = __ldcs(reinterpret_cast<const uint32_t*>(b + list_off) + j);
        v[u] = __ldcs(reinterpret_cast<const T*>(b + list_voff) + j);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (e0 + u * stride < total) theta[id[u]] = v[u];
  }
  last_cta_publish(pp, R, rank, kCtr2, kAckU, -1, s);  // done with the peers' lists
}

PeerPtrs peer_ptrs(const psb_ctx* c) {
  PeerPtrs pp{};
  for (int p = 0; p < c->nranks; ++p) pp.base[p] = reinterpret_cast<uint8_t*>(c->peer_base[p]);
  return pp;
}

void peer_release(psb_ctx* c) {
  for (int p = 0; p < PSB_MAX_P; ++p) {
    if (p != c->rank && c->peer_base[p]) cudaIpcCloseMemHandle(c->peer_base[p]);
    c->peer_base[p] = nullptr;
  }
  if (c->peer_arena) cudaFree(c->peer_arena);
  c->peer_arena = nullptr;
  c->peer_bytes = 0;
}

}  // namespace

// Collective: every rank calls it with the same payload-region size.
psb_status psb_peer_ensure(psb_ctx* c, size_t payload_bytes, cudaStream_t st) {
  if (c->peer_bytes >= payload_bytes) return PSB_OK;
  if (!c->comm) return psb_set_err(c, PSB_ESTATE, "peer exchange: communicator not initialised");
  CUDA_TRY(c, cudaSetDevice(c->device), "peer arena");
  if (c->peer_arena) {
    // every rank done with the old arenas before any is unmapped
    CUDA_TRY(c, cudaDeviceSynchronize(), "peer arena");
    NCCL_TRY(c, ncclAllReduce(c->d_flags + 3, c->d_flags + 3, 1, ncclUint32, ncclMax, c->comm, st),
             "ncclAllReduce(barrier)");
    CUDA_TRY(c, cudaStreamSynchronize(st), "peer arena");
    peer_release(c);
  }
  const size_t bytes = kHdrBytes + ((payload_bytes + 255) & ~(size_t)255);
  void* arena = nullptr;
  if (cudaMalloc(&arena, bytes) != cudaSuccess) return psb_set_err(c, PSB_ENOMEM, "peer arena: out of device memory");
  c->peer_arena = arena;
  CUDA_TRY(c, cudaMemset(arena, 0, kHdrBytes), "peer arena");
  cudaIpcMemHandle_t h;
  CUDA_TRY(c, cudaIpcGetMemHandle(&h, arena), "cudaIpcGetMemHandle");
  // exchange the handles over the communicator
  const size_t hb = sizeof(cudaIpcMemHandle_t);
  uint8_t* d_h = nullptr;
  CUDA_TRY(c, cudaMalloc(&d_h, hb * c->nranks), "peer handles");
  std::vector<uint8_t> all(hb * c->nranks);
  cudaError_t e = cudaMemcpy(d_h + hb * c->rank, &h, hb, cudaMemcpyHostToDevice);
  ncclResult_t nr = ncclSuccess;
  if (e == cudaSuccess) nr = ncclAllGather(d_h + hb * c->rank, d_h, hb, ncclUint8, c->comm, st);
  if (e == cudaSuccess && nr == ncclSuccess) e = cudaStreamSynchronize(st);
  if (e == cudaSuccess && nr == ncclSuccess) e = cudaMemcpy(all.data(), d_h, hb * c->nranks, cudaMemcpyDeviceToHost);
  cudaFree(d_h);
  if (nr != ncclSuccess) return psb_set_err(c, PSB_ENCCL, std::string("peer handles: ") + ncclGetErrorString(nr));
  if (e != cudaSuccess) return psb_cuda_err(c, e, "peer handles");
  for (int p = 0; p < c->nranks; ++p) {
    if (p == c->rank) {
      c->peer_base[p] = arena;
      continue;
    }
    cudaIpcMemHandle_t hp;
    std::memcpy(&hp, all.data() + hb * p, hb);
    e = cudaIpcOpenMemHandle(&c->peer_base[p], hp, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) {
      c->peer_base[p] = nullptr;
      peer_release(c);
      return psb_cuda_err(c, e, "cudaIpcOpenMemHandle");
    }
  }
  c->peer_bytes = payload_bytes;
  return PSB_OK;
}

uint8_t* psb_peer_payload(psb_ctx* c) { return reinterpret_cast<uint8_t*>(c->peer_arena) + kHdrBytes; }

psb_status psb_peer_wait_ack(psb_ctx* c, cudaStream_t st) {
  k_peer_wait_ack<<<1, 1, 0, st>>>(reinterpret_cast<uint32_t*>(c->peer_arena), c->nranks, c->rank, c->d_flags);
  c->launches += 1;
  PSB_LAUNCH_CHECK(c, "peer wait");
  return PSB_OK;
}

psb_status psb_peer_exchange(psb_ctx* c, size_t bytes_per_rank, size_t tab_off, size_t tab_words_per_rank,
                             cudaStream_t st) {
  if (bytes_per_rank % 16) return psb_set_err(c, PSB_EINVAL, "peer exchange: rank range not 16-byte aligned");
  const PeerPtrs pp = peer_ptrs(c);
  k_peer_signal<<<1, 1, 0, st>>>(pp, c->nranks, c->rank);
  const size_t npeer = (size_t)c->nranks - 1;
  const size_t per = std::max<size_t>(1, std::min<size_t>((bytes_per_rank / 16 + 1023) / 1024,
                                                          (size_t)c->num_sms * PSB_PULL_CTAS / npeer));
  k_peer_pull<<<(unsigned)(per * npeer), 256, 0, st>>>(pp, c->nranks, c->rank, bytes_per_rank, tab_off,
                                                        tab_words_per_rank, c->d_flags);
  c->launches += 2;
  PSB_LAUNCH_CHECK(c, "peer exchange");
  return PSB_OK;
}

void psb_peer_destroy(psb_ctx* c) { peer_release(c); }

namespace {
__global__ void k_peer_wait_ready(uint32_t* hdr, int R, int rank, uint32_t* flags) {
  if (!wait_all(hdr, kReady, R, rank, hdr[kSeq])) atomicOr(flags, 8u);
}
// Done reading the peers' payloads (push mode: after the apply).
__global__ void k_peer_ack(PeerPtrs pp, int R, int rank) {
  const uint32_t s = reinterpret_cast<uint32_t*>(pp.base[rank])[kSeq];
  __threadfence_system();
  for (int p = 0; p < R; ++p) {
    if (p == rank) continue;
    uint32_t* ph = reinterpret_cast<uint32_t*>(pp.base[p]);
    st_release_sys(ph + kAck + rank, s);
    st_release_sys(ph + kAckU + rank, s);
  }
}
}  // namespace

namespace {
// Stores [off, off + words) of our payload region into every peer's region.
__global__ void k_peer_put(PeerPtrs pp, int R, int rank, size_t off, size_t words) {
  const uint32_t* src = reinterpret_cast<const uint32_t*>(pp.base[rank] + kHdrBytes + off);
  for (size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x; t < words; t += (size_t)gridDim.x * blockDim.x) {
    const uint32_t v = src[t];
    for (int p = 0; p < R; ++p)
      if (p != rank) reinterpret_cast<uint32_t*>(pp.base[p] + kHdrBytes + off)[t] = v;
  }
  __threadfence_system();
}
}  // namespace

namespace {
// Segment copy from the peers' (NVLink-mapped) payload regions into ours: one
// grid row per segment, int4 loads with PSB_PULL_U in flight per thread (u32
// copies for a segment that is not 16-byte aligned).  The caller has waited
// for the peers' readiness flags.
__global__ void __launch_bounds__(256) k_peer_gather(PeerPtrs pp, int rank, PeerSegs sg) {
  const PeerSeg g = sg.s[blockIdx.y];
  const uint8_t* src = pp.base[g.rank] + kHdrBytes + g.src_off;
  uint8_t* dst = pp.base[rank] + kHdrBytes + g.dst_off;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  if (((g.src_off | g.dst_off | g.bytes) & 15) == 0) {
    const size_t nv = g.bytes / 16;
    constexpr int U = PSB_PULL_U;
    for (size_t t0 = (size_t)blockIdx.x * blockDim.x + threadIdx.x; t0 < nv; t0 += U * stride) {
      int4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (t0 + u * stride < nv) v[u] = __ldcs(reinterpret_cast<const int4*>(src) + t0 + u * stride);
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (t0 + u * stride < nv) reinterpret_cast<int4*>(dst)[t0 + u * stride] = v[u];
    }
  } else {
    const size_t nw = g.bytes / 4;
    for (size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x; t < nw; t += stride)
      reinterpret_cast<uint32_t*>(dst)[t] = reinterpret_cast<const uint32_t*>(src)[t];
  }
}
}  // namespace

psb_status psb_peer_gather(psb_ctx* c, const PeerSegs& segs, cudaStream_t st) {
  if (segs.n <= 0) return PSB_OK;
  size_t mx = 0;
  for (int i = 0; i < segs.n; ++i) {
    if (segs.s[i].bytes % 4) return psb_set_err(c, PSB_EINVAL, "peer gather: segment not a multiple of 4 bytes");
    mx = std::max(mx, segs.s[i].bytes);
  }
  const unsigned gx = (unsigned)std::max<size_t>(
      1, std::min<size_t>((mx / 16 + 255) / 256, (size_t)c->num_sms * PSB_PULL_CTAS / (size_t)segs.n + 1));
  k_peer_gather<<<dim3(gx, (unsigned)segs.n), 256, 0, st>>>(peer_ptrs(c), c->rank, segs);
  c->launches += 1;
  PSB_LAUNCH_CHECK(c, "peer gather");
  return PSB_OK;
}

psb_status psb_peer_put(psb_ctx* c, size_t off, size_t words, cudaStream_t st) {
  const unsigned grid = (unsigned)std::max<size_t>(1, std::min<size_t>((words + 255) / 256, (size_t)c->num_sms));
  k_peer_put<<<grid, 256, 0, st>>>(peer_ptrs(c), c->nranks, c->rank, off, words);
  c->launches += 1;
  PSB_LAUNCH_CHECK(c, "peer put");
  return PSB_OK;
}

psb_status psb_peer_wait_ready(psb_ctx* c, cudaStream_t st) {
  k_peer_wait_ready<<<1, 1, 0, st>>>(reinterpret_cast<uint32_t*>(c->peer_arena), c->nranks, c->rank, c->d_flags);
  c->launches += 1;
  PSB_LAUNCH_CHECK(c, "peer wait ready");
  return PSB_OK;
}

psb_status psb_peer_ack(psb_ctx* c, cudaStream_t st) {
  k_peer_ack<<<1, 1, 0, st>>>(peer_ptrs(c), c->nranks, c->rank);
  c->launches += 1;
  PSB_LAUNCH_CHECK(c, "peer ack");
  return PSB_OK;
}

void psb_peer_push_targets(psb_ctx* c, size_t slot_off) {
  c->push_n = 0;
  for (int p = 0; p < c->nranks; ++p)
    if (p != c->rank) c->push_base[c->push_n++] = reinterpret_cast<uint8_t*>(c->peer_base[p]) + kHdrBytes;
  c->push_slot_off = slot_off;
}

void psb_peer_regions(psb_ctx* c, const uint8_t** out) {
  for (int p = 0; p < c->nranks; ++p) out[p] = reinterpret_cast<const uint8_t*>(c->peer_base[p]) + kHdrBytes;
}

uint32_t* psb_peer_list_cnt(psb_ctx* c) { return reinterpret_cast<uint32_t*>(c->peer_arena) + kListCnt; }

psb_status psb_peer_signal(psb_ctx* c, cudaStream_t st) {
  k_peer_signal<<<1, 1, 0, st>>>(peer_ptrs(c), c->nranks, c->rank);
  c->launches += 1;
  PSB_LAUNCH_CHECK(c, "peer signal");
  return PSB_OK;
}

psb_status psb_shard_pull(psb_ctx* c, psb_dtype dt, int W, int q8, size_t blk, size_t voff, size_t soff,
                          size_t tab_off, uint32_t nseg, uint32_t* range, uint32_t* sidx, void* sval,
                          uint32_t* srow, size_t max_entries, cudaStream_t st) {
  ShardArgs a;
  a.pp = peer_ptrs(c);
  a.R = c->nranks;
  a.rank = c->rank;
  a.W = W;
  a.P = W * c->nranks;
  a.q8 = q8;
  a.blk = blk;
  a.voff = voff;
  a.soff = soff;
  a.tab_off = tab_off;
  a.nseg = nseg;
  a.range = range;
  a.sidx = sidx;
  a.sval = sval;
  a.srow = srow;
  a.flags = c->d_flags;
  const unsigned grid = (unsigned)std::max<size_t>(1, std::min<size_t>((max_entries + 1023) / 1024,
                                                                         (size_t)c->num_sms * 4));
  k_shard_plan<<<1, 1024, 0, st>>>(a, (uint32_t)(max_entries / (size_t)W));
  if (dt == PSB_F64) k_shard_pull<double><<<grid, 256, 0, st>>>(a);
  else k_shard_pull<float><<<grid, 256, 0, st>>>(a);
  c->launches += 2;
  PSB_LAUNCH_CHECK(c, "shard pull");
  return PSB_OK;
}

psb_status psb_shard_finish(psb_ctx* c, psb_dtype dt, size_t list_off, size_t list_voff, void* theta,
                            size_t max_entries, cudaStream_t st) {
  const PeerPtrs pp = peer_ptrs(c);
  k_peer_publish_upd<<<1, 1, 0, st>>>(pp, c->nranks, c->rank);
  const unsigned grid = (unsigned)std::max<size_t>(1, std::min<size_t>((max_entries + 1023) / 1024,
                                                                         (size_t)c->num_sms * 4));
  const int reps = c->marks_on && getenv("PSB_SCATTER_TWICE") ? 2 : 1;  // diagnostics: time a wait-free rerun
  for (int rep = 0; rep < reps; ++rep) {
    if (rep) psb_mark(c, st);
    if (dt == PSB_F64)
      k_shard_scatter<double><<<grid, 256, 0, st>>>(pp, c->nranks, c->rank, list_off, list_voff,
                                                    reinterpret_cast<double*>(theta), c->d_flags);
    else
      k_shard_scatter<float><<<grid, 256, 0, st>>>(pp, c->nranks, c->rank, list_off, list_voff,
                                                   reinterpret_cast<float*>(theta), c->d_flags);
  }
  c->launches += 2;
  PSB_LAUNCH_CHECK(c, "shard scatter");
  return PSB_OK;
}

extern "C" psb_status psb_peer_mode(psb_ctx* c, int mode) {
  PSB_REQUIRE(c, c != nullptr, "null ctx");
  PSB_REQUIRE(c, mode >= 0 && mode <= 5, "psb_peer_mode: mode must be 0..5");
  c->peer_mode = mode > 0;
  c->shard_mode = mode == 2;
  c->push_mode = mode == 3;
  c->direct_mode = mode == 4 ? 1 : mode == 5 ? 2 : 0;
  return PSB_OK;
}

extern "C" int psb_peer_active(const psb_ctx* c) { return c && c->peer_arena ? 1 : 0; }

// ------------------------------------------------------------ diagnostics
namespace {
__global__ void __launch_bounds__(256) k_copy16(int4* __restrict__ dst, const int4* __restrict__ src, size_t nv) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  constexpr int U = 4;
  for (size_t i0 = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i0 < nv; i0 += U * stride) {
    int4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (i0 + u * stride < nv) v[u] = __ldcs(src + i0 + u * stride);
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (i0 + u * stride < nv) __stcs(dst + i0 + u * stride, v[u]);
  }
}
}  // namespace

// SM-driven 16-byte copy (either pointer may live on a peer GPU of the same
// process after cudaDeviceEnablePeerAccess); for NVLink bandwidth probes.
extern "C" PSB_API int psb_debug_copy16(void* dst, const void* src, size_t bytes, int ctas, void* stream) {
  k_copy16<<<ctas, 256, 0, (cudaStream_t)stream>>>(reinterpret_cast<int4*>(dst), reinterpret_cast<const int4*>(src),
                                                   bytes / 16);
  return (int)cudaGetLastError();
}
extern "C" PSB_API int psb_debug_enable_peer(int dev, int peer) {
  int cur = 0;
  cudaGetDevice(&cur);
  cudaSetDevice(dev);
  cudaError_t e = cudaDeviceEnablePeerAccess(peer, 0);
  cudaSetDevice(cur);
  return e == cudaErrorPeerAccessAlreadyEnabled ? 0 : (int)e;
}

namespace {
__global__ void __launch_bounds__(256) k_debug_scatter(float* __restrict__ theta, const uint32_t* __restrict__ idx,
                                                       const float* __restrict__ val, size_t cnt) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  constexpr int U = 8;
  for (size_t e0 = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e0 < cnt; e0 += U * stride) {
    uint32_t id[U];
    float v[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (e0 + u * stride < cnt) {
        id[u] = __ldcs(idx + e0 + u * stride);
        v[u] = __ldcs(val + e0 + u * stride);
      }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (e0 + u * stride < cnt) theta[id[u]] = v[u];
  }
}
}  // namespace

// theta[idx[j]] = val[j] (the update-list scatter of the sharded apply, lists
// anywhere in the peer-mapped address space); for bandwidth probes.
extern "C" PSB_API int psb_debug_scatter(float* theta, const uint32_t* idx, const float* val, size_t cnt, int ctas,
                                         void* stream) {
  k_debug_scatter<<<ctas, 256, 0, (cudaStream_t)stream>>>(theta, idx, val, cnt);
  return (int)cudaGetLastError();
}

// Diagnostics: `iters` bare payload exchanges of bytes_per_rank (arena set up
// on first use; every rank must call it together).
extern "C" PSB_API psb_status psb_debug_exchange(psb_ctx* c, size_t bytes_per_rank, int iters, psb_stream_t stream) {
  PSB_REQUIRE(c, c != nullptr && c->nranks > 1, "debug exchange: needs a multi-rank ctx");
  cudaStream_t st = (cudaStream_t)stream;
  psb_status s = psb_peer_ensure(c, bytes_per_rank * c->nranks, st);
  if (s) return s;
  for (int i = 0; i < iters; ++i) {
    s = psb_peer_wait_ack(c, st);
    if (s) return s;
    s = psb_peer_exchange(c, bytes_per_rank, 0, 0, st);
    if (s) return s;
  }
  return PSB_OK;
}

// ---- diagnostics: device timestamps at step boundaries (graph-capturable;
// the slot index advances on the device)
namespace {
__device__ unsigned long long g_stamps[4096];
__device__ unsigned int g_nstamps;
__global__ void k_stamp() {
  const unsigned int i = atomicAdd(&g_nstamps, 1u);
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  if (i < 4096) g_stamps[i] = t;
}
}  // namespace

extern "C" PSB_API psb_status psb_debug_stamp(psb_ctx* c, psb_stream_t stream) {
  PSB_REQUIRE(c, c != nullptr, "null ctx");
  k_stamp<<<1, 1, 0, (cudaStream_t)stream>>>();
  PSB_LAUNCH_CHECK(c, "debug stamp");
  return PSB_OK;
}

extern "C" PSB_API int psb_debug_stamps(unsigned long long* out, int max) {
  unsigned int n = 0;
  if (cudaMemcpyFromSymbol(&n, g_nstamps, sizeof(n)) != cudaSuccess) return -1;
  const int m = (int)std::min<unsigned int>(n, (unsigned int)std::min(max, 4096));
  if (m > 0 && cudaMemcpyFromSymbol(out, g_stamps, sizeof(unsigned long long) * m) != cudaSuccess) return -1;
  const unsigned int z = 0;
  cudaMemcpyToSymbol(g_nstamps, &z, sizeof(z));
  return m;
}
