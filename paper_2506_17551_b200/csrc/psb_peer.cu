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

#include "psb_internal.cuh"

namespace {

constexpr size_t kHdrBytes = 4096;
// header words: [0, 32) ready[p], [32, 64) ack[p], 64 local seq, 65 pull CTA counter
constexpr int kReady = 0, kAck = 32, kSeq = 64, kCtr = 65;
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

__global__ void k_peer_wait_ack(uint32_t* hdr, int R, int rank, uint32_t* flags) {
  if (!wait_all(hdr, kAck, R, rank, hdr[kSeq])) atomicOr(flags, 8u);
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
// from its arena into ours, then acknowledges.  bpr is a multiple of 16.
__global__ void __launch_bounds__(256) k_peer_pull(PeerPtrs pp, int R, int rank, size_t bpr, uint32_t* flags) {
  uint32_t* hdr = reinterpret_cast<uint32_t*>(pp.base[rank]);
  const uint32_t s = hdr[kSeq];
  __shared__ int ok;
  if (threadIdx.x == 0) ok = wait_all(hdr, kReady, R, rank, s);
  __syncthreads();
  if (!ok) {
    if (threadIdx.x == 0) atomicOr(flags, 8u);
    return;
  }
  const size_t v_per = bpr / 16;  // int4 per rank range
  const size_t total = v_per * (size_t)(R - 1);
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  constexpr int U = 4;
  for (size_t t0 = (size_t)blockIdx.x * blockDim.x + threadIdx.x; t0 < total; t0 += U * stride) {
    int4 v[U];
    int4* dst[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const size_t t = t0 + u * stride;
      dst[u] = nullptr;
      if (t < total) {
        int pi = (int)(t / v_per);
        const size_t j = t - (size_t)pi * v_per;
        const int p = pi + (pi >= rank);  // skip our own range
        const size_t off = kHdrBytes + (size_t)p * bpr + j * 16;
        v[u] = __ldcs(reinterpret_cast<const int4*>(pp.base[p] + off));
        dst[u] = reinterpret_cast<int4*>(pp.base[rank] + off);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (dst[u]) *dst[u] = v[u];
  }
  // last CTA out acknowledges to every peer
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(hdr + kCtr, 1u) == gridDim.x - 1) {
      hdr[kCtr] = 0;
      __threadfence_system();
      for (int p = 0; p < R; ++p)
        if (p != rank) st_release_sys(reinterpret_cast<uint32_t*>(pp.base[p]) + kAck + rank, s);
    }
  }
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

psb_status psb_peer_exchange(psb_ctx* c, size_t bytes_per_rank, cudaStream_t st) {
  if (bytes_per_rank % 16) return psb_set_err(c, PSB_EINVAL, "peer exchange: rank range not 16-byte aligned");
  const PeerPtrs pp = peer_ptrs(c);
  k_peer_signal<<<1, 1, 0, st>>>(pp, c->nranks, c->rank);
  const size_t v = bytes_per_rank / 16 * (size_t)(c->nranks - 1);
  const unsigned grid = (unsigned)std::max<size_t>(1, std::min<size_t>((v + 1023) / 1024, (size_t)c->num_sms * 4));
  k_peer_pull<<<grid, 256, 0, st>>>(pp, c->nranks, c->rank, bytes_per_rank, c->d_flags);
  c->launches += 2;
  PSB_LAUNCH_CHECK(c, "peer exchange");
  return PSB_OK;
}

void psb_peer_destroy(psb_ctx* c) { peer_release(c); }

extern "C" psb_status psb_peer_mode(psb_ctx* c, int on) {
  PSB_REQUIRE(c, c != nullptr, "null ctx");
  c->peer_mode = on ? 1 : 0;
  return PSB_OK;
}

extern "C" int psb_peer_active(const psb_ctx* c) { return c && c->peer_arena ? 1 : 0; }
