// topk.cuh — warp-resident sorted top-k list.
//
// Order = numpy's stable argsort of the distance row (knn.py:46, 77):
// ascending distance, ties broken by ascending index, NaN after everything.
// The list holds K = 32*KPL slots; slot g = s*32 + lane lives in register
// (d[s], i[s]) of that lane.  Insertion is warp-synchronous: position by
// ballot/popc, shift by shuffles — no shared memory, no atomics.
#pragma once
#include "common.cuh"

namespace sd {

template <typename T>
__device__ __forceinline__ bool key_less(T d1, int64_t i1, T d2, int64_t i2) {
  if (d1 < d2) return true;
  if (d1 > d2) return false;
  const bool n1 = d1 != d1, n2 = d2 != d2;
  if (n1 != n2) return n2;
  return i1 < i2;
}

template <typename T, int KPL>
struct WarpTopK {
  T d[KPL];
  int64_t i[KPL];
  T thr_d;          // the k-th entry, refreshed after every insertion (rare):
  int64_t thr_i;    // the common offer is a compare and a vote, no shuffles

  __device__ __forceinline__ void init() {
#pragma unroll
    for (int s = 0; s < KPL; ++s) {
      d[s] = T(NAN);
      i[s] = INT64_MAX;
    }
    thr_d = T(NAN);
    thr_i = INT64_MAX;
  }

  // current k-th entry (the admission threshold)
  __device__ __forceinline__ void kth(int k, T& td, int64_t& ti) const {
    const int s = (k - 1) >> 5, l = (k - 1) & 31;
    T dd = d[0];
    int64_t ii = i[0];
#pragma unroll
    for (int q = 1; q < KPL; ++q)
      if (q == s) { dd = d[q]; ii = i[q]; }
    td = __shfl_sync(0xffffffffu, dd, l);
    ti = __shfl_sync(0xffffffffu, ii, l);
  }

  // insert a warp-uniform candidate (only the first k slots are meaningful)
  __device__ __forceinline__ void insert(T cd, int64_t ci, int k) {
    const unsigned lane = lane_id();
    int pos = 0;
#pragma unroll
    for (int s = 0; s < KPL; ++s) {
      const bool lt = (s * 32 + int(lane) < k) && key_less(d[s], i[s], cd, ci);
      pos += __popc(__ballot_sync(0xffffffffu, lt));
    }
    if (pos >= k) return;
    T carry_d = T(0);
    int64_t carry_i = 0;
#pragma unroll
    for (int s = 0; s < KPL; ++s) {
      T up_d = __shfl_up_sync(0xffffffffu, d[s], 1);
      int64_t up_i = __shfl_up_sync(0xffffffffu, i[s], 1);
      const T last_d = __shfl_sync(0xffffffffu, d[s], 31);
      const int64_t last_i = __shfl_sync(0xffffffffu, i[s], 31);
      if (lane == 0) { up_d = carry_d; up_i = carry_i; }
      const int g = s * 32 + int(lane);
      if (g == pos) { d[s] = cd; i[s] = ci; }
      else if (g > pos) { d[s] = up_d; i[s] = up_i; }
      carry_d = last_d;
      carry_i = last_i;
    }
  }

  // offer one candidate per lane (valid lanes only), in lane order
  __device__ __forceinline__ void offer(bool valid, T cd, int64_t ci, int k) {
    const T td = thr_d;
    const int64_t ti = thr_i;
    unsigned mask = __ballot_sync(0xffffffffu, valid && key_less(cd, ci, td, ti));
    const bool inserted = mask != 0u;
    while (mask) {
      const int src = __ffs(mask) - 1;
      mask &= mask - 1;
      const T sd_ = __shfl_sync(0xffffffffu, cd, src);
      const int64_t si = __shfl_sync(0xffffffffu, ci, src);
      insert(sd_, si, k);
    }
    if (inserted) kth(k, thr_d, thr_i);
  }

  __device__ __forceinline__ void store(int k, T* od, int64_t* oi, int64_t base) const {
#pragma unroll
    for (int s = 0; s < KPL; ++s) {
      const int g = s * 32 + int(lane_id());
      if (g < k) { od[g] = d[s]; oi[g] = i[s] + base; }
    }
  }
};

}  // namespace sd
