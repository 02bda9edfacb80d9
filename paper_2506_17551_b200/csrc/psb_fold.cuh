// psb_fold.cuh -- the reference's canonical fold orders, per element.
//
// allreduce_mean (parsim/collectives.hpp:135-154) reduces P dense buffers in a
// fixed order and scales by 1/P:
//   naive        acc = b0; acc += b1 .. b_{P-1}                     (:68-73)
//   ring         chunk j = [j*n/P, (j+1)*n/P) folds b_{(j+1)%P}, b_{(j+2)%P}, ...  (:77-94)
//   hierarchical fold devices_per_node contiguous workers per node, nodes per
//                rack, then racks                                    (:99-128)
// get(q) returns worker q's dense value at this index (+0 where a sparse
// worker did not select it), so the result is bitwise the reference's.
#pragma once
#include "psb_internal.cuh"

// The ring chunk containing index i, cached: consecutive indices almost always
// share a chunk (chunks are n/P long), so the 64-bit divisions run only when
// the chunk changes.
struct RingChunk {
  size_t lo = 1, hi = 0;  // current chunk [lo, hi) (empty initially)
  int start = 0;          // first worker folded for this chunk: (j + 1) % P
  __device__ __forceinline__ int start_for(size_t i, size_t n, int P) {
    if (i < lo || i >= hi) {
      uint32_t j = (uint32_t)((i * (size_t)P) / n);
      while (j + 1 < (uint32_t)P && ((size_t)(j + 1) * n) / (size_t)P <= i) ++j;
      while (j > 0 && ((size_t)j * n) / (size_t)P > i) --j;
      lo = ((size_t)j * n) / (size_t)P;
      hi = ((size_t)(j + 1) * n) / (size_t)P;
      start = (int)((j + 1) % (uint32_t)P);
    }
    return start;
  }
};

// Fold with an explicit ring start (ignored by the other orders).
template <class T, class Get>
__device__ __forceinline__ T fold_sum_start(const Get& get, int P, int order, int ring_start, uint32_t dpn,
                                            uint32_t npr) {
  T acc;
  if (order == PSB_ORDER_RING) {
    acc = get(ring_start);
    for (int s = 1; s < P; ++s) {
      int q = ring_start + s;
      if (q >= P) q -= P;
      acc = add_rn(acc, get(q));
    }
  } else if (order == PSB_ORDER_HIER && dpn < (uint32_t)P) {
    const uint32_t nodes = ((uint32_t)P + dpn - 1) / dpn;
    T total = T(0);
    bool have_total = false;
    for (uint32_t nb = 0; nb < nodes; nb += npr) {
      T rack = T(0);
      bool have_rack = false;
      for (uint32_t nd = nb; nd < nodes && nd < nb + npr; ++nd) {
        const uint32_t base = nd * dpn;
        T node = get((int)base);
        for (uint32_t p = base + 1; p < base + dpn && p < (uint32_t)P; ++p) node = add_rn(node, get((int)p));
        rack = have_rack ? add_rn(rack, node) : node;
        have_rack = true;
      }
      total = have_total ? add_rn(total, rack) : rack;
      have_total = true;
    }
    acc = total;
  } else {
    // naive, and hierarchical with a single node (devices_per_node >= P),
    // which folds in plain worker order (collectives.hpp:105-111).
    acc = get(0);
    for (int q = 1; q < P; ++q) acc = add_rn(acc, get(q));
  }
  return acc;
}

template <class T, class Get>
__device__ __forceinline__ T fold_sum(const Get& get, int P, int order, size_t i, size_t n, uint32_t dpn,
                                      uint32_t npr) {
  RingChunk rc;
  const int start = order == PSB_ORDER_RING ? rc.start_for(i, n, P) : 0;
  return fold_sum_start<T>(get, P, order, start, dpn, npr);
}
