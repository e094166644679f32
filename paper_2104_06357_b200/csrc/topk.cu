// topk.cu — select_topk over dense distance rows (knn.py:41-47, 76-79) and
// the merge of per-shard candidate lists after the NCCL all-gather
// (SURVEY.md §8e).  k <= 128 runs one warp per row with the register list
// of topk.cuh; larger k uses a stable segmented sort of (distance, index),
// which is numpy's argsort(kind="stable") order by construction.
#include <algorithm>
#include <cub/cub.cuh>
#include "common.cuh"
#include "prep.cuh"
#include "topk.cuh"

namespace sd {

template <typename T, int KPL>
__global__ void topk_rows_kernel(const T* __restrict__ dist, int64_t m, int64_t n, int64_t ldd, int k,
                                 int64_t base, T* __restrict__ od, int64_t* __restrict__ oi) {
  const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t r = warp; r < m; r += nw) {
    WarpTopK<T, KPL> top;
    top.init();
    const T* row = dist + r * ldd;
    for (int64_t q = 0; q < n; q += 32) {
      const int64_t j = q + lane_id();
      const bool valid = j < n;
      top.offer(valid, valid ? row[j] : T(0), j, k);
    }
    top.store(k, od + r * k, oi + r * k, base);
  }
}

template <typename T, int KPL>
__global__ void topk_merge_kernel(const T* __restrict__ cd, const int64_t* __restrict__ ci, int64_t m,
                                  int lists, int k, T* __restrict__ od, int64_t* __restrict__ oi) {
  const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t r = warp; r < m; r += nw) {
    WarpTopK<T, KPL> top;
    top.init();
    for (int g = 0; g < lists; ++g) {
      const T* d = cd + (int64_t(g) * m + r) * k;
      const int64_t* ix = ci + (int64_t(g) * m + r) * k;
      for (int q = 0; q < k; q += 32) {
        const int j = q + int(lane_id());
        const bool valid = j < k;
        top.offer(valid, valid ? d[j] : T(0), valid ? ix[j] : 0, k);
      }
    }
    top.store(k, od + r * k, oi + r * k, 0);
  }
}

// top-k of column chunk g of every row (warp per (g, row), chunk lists
// [g][m][k] with global column ids) — a few long rows spread over many warps
template <typename T, int KPL>
__global__ void topk_chunks_kernel(const T* __restrict__ dist, int64_t m, int64_t n, int64_t ldd, int k,
                                   int64_t chunk, int64_t nchunks, T* __restrict__ cd, int64_t* __restrict__ ci) {
  const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t w = warp; w < m * nchunks; w += nw) {
    const int64_t g = w / m, r = w - g * m;
    WarpTopK<T, KPL> top;
    top.init();
    const T* row = dist + r * ldd;
    const int64_t j0 = g * chunk, j1 = tmin<int64_t>(n, j0 + chunk);
    for (int64_t q = j0; q < j1; q += 32) {
      const int64_t j = q + lane_id();
      const bool valid = j < j1;
      top.offer(valid, valid ? row[j] : T(0), j, k);
    }
    top.store(k, cd + w * k, ci + w * k, 0);
  }
}

// od[rowmap[r]] = rows r of the compact lists, indices + base
template <typename T>
__global__ void scatter_rows_kernel(const T* __restrict__ sd_, const int64_t* __restrict__ si, int64_t m, int k,
                                    const int32_t* __restrict__ rowmap, int64_t base, T* __restrict__ od,
                                    int64_t* __restrict__ oi) {
  for (int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; q < m * k; q += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r = q / k, t = q - r * k;
    const int64_t o = int64_t(rowmap[r]) * k + t;
    od[o] = sd_[q];
    oi[o] = si[q] + base;
  }
}

template <typename T>
__global__ void gather_first_k(const T* __restrict__ sd_, const int64_t* __restrict__ si, int64_t m,
                               int64_t seg, int k, int64_t base, T* __restrict__ od, int64_t* __restrict__ oi) {
  const int64_t total = m * k;
  for (int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; q < total; q += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r = q / k, t = q - r * k;
    od[q] = sd_[r * seg + t];
    oi[q] = si[r * seg + t] + base;
  }
}

template <typename T>
__global__ void iota_rows(const T* __restrict__ src, int64_t m, int64_t n, int64_t lds, T* __restrict__ keys,
                          int64_t* __restrict__ ids, int64_t* __restrict__ offs) {
  const int64_t total = m * n;
  for (int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; q < total; q += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r = q / n, j = q - r * n;
    keys[q] = src[r * lds + j];
    ids[q] = ids ? j : 0;
  }
  for (int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; r <= m; r += int64_t(gridDim.x) * blockDim.x)
    offs[r] = r * n;
}

template <typename T>
static int sorted_topk(const T* dist, int64_t m, int64_t n, int64_t ldd, int k, int64_t base, T* od,
                       int64_t* oi, cudaStream_t st) {
  Scratch keys, keys_o, ids, ids_o, offs, tmp;
  SD_TRY(keys.alloc(sizeof(T) * m * n, st));
  SD_TRY(keys_o.alloc(sizeof(T) * m * n, st));
  SD_TRY(ids.alloc(sizeof(int64_t) * m * n, st));
  SD_TRY(ids_o.alloc(sizeof(int64_t) * m * n, st));
  SD_TRY(offs.alloc(sizeof(int64_t) * (m + 1), st));
  const int blocks = int(std::min<int64_t>((m * n + 255) / 256, int64_t(num_sms()) * 16));
  iota_rows<T><<<std::max(1, blocks), 256, 0, st>>>(dist, m, n, ldd, keys.as<T>(), ids.as<int64_t>(), offs.as<int64_t>());
  SD_LAUNCH_CHECK();
  size_t tb = 0;
  cub::DeviceSegmentedSort::StableSortPairs(nullptr, tb, keys.as<T>(), keys_o.as<T>(), ids.as<int64_t>(),
                                            ids_o.as<int64_t>(), m * n, m, offs.as<int64_t>(),
                                            offs.as<int64_t>() + 1, st);
  SD_TRY(tmp.alloc(tb, st));
  SD_CUDA_TRY(cub::DeviceSegmentedSort::StableSortPairs(tmp.ptr, tb, keys.as<T>(), keys_o.as<T>(), ids.as<int64_t>(),
                                                        ids_o.as<int64_t>(), m * n, m, offs.as<int64_t>(),
                                                        offs.as<int64_t>() + 1, st));
  const int gb = int(std::min<int64_t>((m * k + 255) / 256, int64_t(num_sms()) * 16));
  gather_first_k<T><<<std::max(1, gb), 256, 0, st>>>(keys_o.as<T>(), ids_o.as<int64_t>(), m, n, k, base, od, oi);
  SD_LAUNCH_CHECK();
  return SD_OK;
}

int topk_rows(const void* dist, int64_t m, int64_t n, int64_t ldd, int dtype, int k, int64_t base,
              void* od, int64_t* oi, cudaStream_t st) {
  if (k > n) { set_error("k exceeds the number of candidates"); return SD_E_K_TOO_LARGE; }
  if (k < 0) { set_error("k must be non-negative"); return SD_E_INVALID; }
  if (m == 0 || k == 0) return SD_OK;
  return SD_DISPATCH_DTYPE(dtype, T, [&]() -> int {
    const T* d = static_cast<const T*>(dist);
    const int blocks = int(std::min<int64_t>((m * 32 + 255) / 256, int64_t(num_sms()) * 16));
    if (k <= 32) topk_rows_kernel<T, 1><<<blocks, 256, 0, st>>>(d, m, n, ldd, k, base, static_cast<T*>(od), oi);
    else if (k <= 128) topk_rows_kernel<T, 4><<<blocks, 256, 0, st>>>(d, m, n, ldd, k, base, static_cast<T*>(od), oi);
    else return sorted_topk<T>(d, m, n, ldd, k, base, static_cast<T*>(od), oi, st);
    SD_LAUNCH_CHECK();
    return SD_OK;
  });
}

// top-k of a few long dense rows (the hybrid path's heavy kNN queries):
// column chunks over ~8 waves of warps, their lists merged, the results
// scattered to rows rowmap[r] of (od, oi) with indices + base.  k <= 128.
int topk_rows_scatter(const void* dist, int64_t m, int64_t n, int64_t ldd, int dtype, int k, int64_t base,
                      const int32_t* rowmap, void* od, int64_t* oi, cudaStream_t st) {
  if (m == 0 || k == 0) return SD_OK;
  if (k > 128) { set_error("chunked top-k supports k <= 128"); return SD_E_INVALID; }
  const int64_t want = std::max<int64_t>(1, int64_t(num_sms()) * 64 / std::max<int64_t>(1, m));
  const int64_t chunk = std::max<int64_t>(int64_t(k) * 32, (n + want - 1) / want);
  const int64_t nchunks = (n + chunk - 1) / chunk;
  const size_t es = dtype == SD_F64 ? 8 : 4;
  Scratch cd, ci, md, mi;
  SD_TRY(cd.alloc(es * size_t(m * nchunks * k), st));
  SD_TRY(ci.alloc(sizeof(int64_t) * size_t(m * nchunks * k), st));
  SD_TRY(md.alloc(es * size_t(m * k), st));
  SD_TRY(mi.alloc(sizeof(int64_t) * size_t(m * k), st));
  SD_TRY(SD_DISPATCH_DTYPE(dtype, T, [&]() -> int {
    const T* d = static_cast<const T*>(dist);
    const int blocks = int(std::min<int64_t>((m * nchunks * 32 + 255) / 256, int64_t(num_sms()) * 16));
    if (k <= 32) topk_chunks_kernel<T, 1><<<blocks, 256, 0, st>>>(d, m, n, ldd, k, chunk, nchunks, cd.as<T>(), ci.as<int64_t>());
    else topk_chunks_kernel<T, 4><<<blocks, 256, 0, st>>>(d, m, n, ldd, k, chunk, nchunks, cd.as<T>(), ci.as<int64_t>());
    SD_LAUNCH_CHECK();
    return SD_OK;
  }));
  SD_TRY(topk_merge(cd.ptr, ci.as<int64_t>(), m, int(nchunks), k, dtype, md.ptr, mi.as<int64_t>(), st));
  return SD_DISPATCH_DTYPE(dtype, T, [&]() -> int {
    const int blocks = int(std::min<int64_t>((m * k + 255) / 256, int64_t(num_sms()) * 8));
    scatter_rows_kernel<T><<<std::max(1, blocks), 256, 0, st>>>(md.as<T>(), mi.as<int64_t>(), m, k, rowmap, base,
                                                               static_cast<T*>(od), oi);
    SD_LAUNCH_CHECK();
    return SD_OK;
  });
}

int topk_merge(const void* cd, const int64_t* ci, int64_t m, int lists, int k, int dtype, void* od,
               int64_t* oi, cudaStream_t st) {
  if (m == 0 || k == 0) return SD_OK;
  if (lists < 1) { set_error("need at least one candidate list"); return SD_E_INVALID; }
  return SD_DISPATCH_DTYPE(dtype, T, [&]() -> int {
    const int blocks = int(std::min<int64_t>((m * 32 + 255) / 256, int64_t(num_sms()) * 16));
    if (k <= 32)
      topk_merge_kernel<T, 1><<<blocks, 256, 0, st>>>(static_cast<const T*>(cd), ci, m, lists, k, static_cast<T*>(od), oi);
    else if (k <= 128)
      topk_merge_kernel<T, 4><<<blocks, 256, 0, st>>>(static_cast<const T*>(cd), ci, m, lists, k, static_cast<T*>(od), oi);
    else { set_error("merge supports k <= 128"); return SD_E_INVALID; }
    SD_LAUNCH_CHECK();
    return SD_OK;
  });
}

}  // namespace sd
