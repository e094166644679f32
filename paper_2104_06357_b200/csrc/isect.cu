// isect.cu — the fused intersection path.
//
// Alg. 3 of the paper probes every nonzero of B once per query row, i.e.
// m·nnz(B) probes, although only |A_i ∩ B_j| of the nnz(B_j) probes of a pair
// can hit (≈ d_A·d_B/k: 0.4 of 154 on the MovieLens shape).  On B200 the
// hot path is instead output-stationary over a J-blocked inverted index:
//
//   index (built once per B, cached):  B^T split into tiles of TJ index rows;
//     for tile t and column c the postings (j - t·TJ : u16, b_jc : T) are
//     contiguous, located by colptr[t·n_cols + c] (u32).
//   kernel: one warp per query row i (dynamic queue, longest rows first);
//     for each tile t the warp owns a TJ-cell accumulator in shared memory,
//     walks A_i's columns in ascending order and scatter-adds the
//     contribution of every posting of column c (distinct cells within a
//     column, __syncwarp between columns => each cell accumulates in
//     ascending column order, deterministic, no atomics), then runs the
//     metric epilogue on the TJ cells and writes them coalesced — or, for
//     kNN, offers them to a warp-register top-k list (no distance matrix).
//
// HBM traffic is the output write plus posting reads, which stay L2-resident
// per tile (DESIGN.md §7 byte model).
#include <cstdlib>
#include <mutex>
#include <vector>
#include <cub/cub.cuh>
#include "common.cuh"
#include "metric.cuh"
#include "prep.cuh"
#include "topk.cuh"
#include "isect_kernel.cuh"

#include "index.cuh"
#include "hybrid.cuh"

namespace sd {

int default_tile(int dtype) {
  const int64_t t = knob(SD_TUNE_TILE);  // experiment override
  if (t >= 128 && t <= 65536 && t % 128 == 0) return int(dtype == SD_F64 ? t / 2 : t);
  return dtype == SD_F64 ? 2048 : 4096;
}

__global__ void index_count_kernel(const int64_t* __restrict__ ptr, const int32_t* __restrict__ idx,
                                   int64_t n_rows, int tile, int64_t n_cols, uint32_t* counts) {
  const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t r = warp; r < n_rows; r += nw) {
    const int64_t base = (r / tile) * n_cols;
    for (int64_t e = ptr[r] + lane_id(); e < ptr[r + 1]; e += 32) atomicAdd(&counts[base + idx[e]], 1u);
  }
}

// kNN: every query's shared k-th-distance bound starts at +inf
template <typename K>
__global__ void fill_key_kernel(K* __restrict__ k, int64_t n, K v) {
  for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < n; e += int64_t(gridDim.x) * blockDim.x) k[e] = v;
}

// per-tile sums of row degrees and squared row degrees (collision estimate)
__global__ void tile_degree_kernel(const int64_t* __restrict__ ptr, int64_t n_rows, int tile, double* sums) {
  for (int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < n_rows; r += int64_t(gridDim.x) * blockDim.x) {
    const double d = double(ptr[r + 1] - ptr[r]);
    atomicAdd(&sums[2 * (r / tile)], d);
    atomicAdd(&sums[2 * (r / tile) + 1], d * d);
  }
}

template <typename T>
__global__ void index_scatter_kernel(const int64_t* __restrict__ ptr, const int32_t* __restrict__ idx,
                                     const T* __restrict__ val, int64_t n_rows, int tile, int64_t n_cols,
                                     const uint32_t* __restrict__ colptr, uint32_t* cursor,
                                     Posting<T>* __restrict__ post) {
  const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t r = warp; r < n_rows; r += nw) {
    const int64_t t = r / tile;
    const int64_t base = t * n_cols;
    for (int64_t e = ptr[r] + lane_id(); e < ptr[r + 1]; e += 32) {
      const int64_t key = base + idx[e];
      const uint32_t pos = colptr[key] + atomicAdd(&cursor[key], 1u);
      Posting<T> q;
      q.j = uint32_t(r - t * tile);
      q.v = val[e];
      if constexpr (sizeof(T) == 8) q.pad = 0;
      post[pos] = q;
    }
  }
}

int index_build(const sd_csr* b, int dtype, int tile, sd_index** out, cudaStream_t st) {
  if (tile <= 0) tile = default_tile(dtype);
  if (tile > 65536) { set_error("tile_rows must be <= 65536"); return SD_E_INVALID; }
  if (b->nnz >= (int64_t(1) << 32)) { set_error("index nnz must be < 2^32"); return SD_E_INVALID; }
  const int64_t n_tiles = std::max<int64_t>(1, (b->n_rows + tile - 1) / tile);
  const int64_t n_keys = n_tiles * b->n_cols;
  const size_t es = dtype == SD_F64 ? 8 : 4;
  sd_index* ix = new sd_index();
  ix->n_rows = b->n_rows; ix->n_cols = b->n_cols; ix->nnz = b->nnz;
  ix->tile = tile; ix->n_tiles = n_tiles; ix->dtype = dtype;
  auto fail = [&](int code) { sd_index_free(ix); return code; };
  const size_t ps = dtype == SD_F64 ? sizeof(Posting<double>) : sizeof(Posting<float>);
  (void)es;
  if (cudaMalloc(&ix->colptr, sizeof(uint32_t) * (n_keys + 1)) != cudaSuccess ||
      cudaMalloc(&ix->post, ps * std::max<int64_t>(1, b->nnz)) != cudaSuccess) {
    set_error("cudaMalloc failed for the inverted index");
    return fail(SD_E_CUDA);
  }
  ix->bytes = int64_t(sizeof(uint32_t) * (n_keys + 1) + ps * b->nnz);
  Scratch counts;
  if (counts.alloc(sizeof(uint32_t) * (n_keys + 1), st) != SD_OK) return fail(SD_E_CUDA);
  if (cudaMemsetAsync(counts.ptr, 0, sizeof(uint32_t) * (n_keys + 1), st) != cudaSuccess) return fail(SD_E_CUDA);
  const int blocks = int(std::min<int64_t>((std::max<int64_t>(b->n_rows, 1) * 32 + 255) / 256, int64_t(num_sms()) * 16));
  if (b->n_rows > 0 && b->nnz > 0) {
    index_count_kernel<<<blocks, 256, 0, st>>>(b->indptr, b->indices, b->n_rows, tile, b->n_cols, counts.as<uint32_t>());
    if (cudaGetLastError() != cudaSuccess) { set_error("index count kernel failed"); return fail(SD_E_CUDA); }
  }
  size_t tmp_bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, counts.as<uint32_t>(), ix->colptr, n_keys + 1, st);
  Scratch tmp;
  if (tmp.alloc(tmp_bytes, st) != SD_OK) return fail(SD_E_CUDA);
  if (cub::DeviceScan::ExclusiveSum(tmp.ptr, tmp_bytes, counts.as<uint32_t>(), ix->colptr, n_keys + 1, st) != cudaSuccess) {
    set_error("index scan failed");
    return fail(SD_E_CUDA);
  }
  if (cudaMemsetAsync(counts.ptr, 0, sizeof(uint32_t) * (n_keys + 1), st) != cudaSuccess) return fail(SD_E_CUDA);
  if (b->n_rows > 0 && b->nnz > 0) {
    int rc = SD_DISPATCH_DTYPE(dtype, T, [&]() -> int {
      index_scatter_kernel<T><<<blocks, 256, 0, st>>>(b->indptr, b->indices, static_cast<const T*>(b->values),
                                                      b->n_rows, tile, b->n_cols, ix->colptr,
                                                      counts.as<uint32_t>(), static_cast<Posting<T>*>(ix->post));
      SD_LAUNCH_CHECK();
      return SD_OK;
    });
    if (rc != SD_OK) return fail(rc);
  }
  if (b->n_rows > 0 && b->nnz > 0) {  // collision estimate (one small D2H at build time)
    Scratch sums;
    if (sums.alloc(sizeof(double) * 2 * n_tiles, st) != SD_OK) return fail(SD_E_CUDA);
    if (cudaMemsetAsync(sums.ptr, 0, sizeof(double) * 2 * n_tiles, st) != cudaSuccess) return fail(SD_E_CUDA);
    tile_degree_kernel<<<int(std::min<int64_t>((b->n_rows + 255) / 256, 4096)), 256, 0, st>>>(
        b->indptr, b->n_rows, tile, sums.as<double>());
    count_launch();
    std::vector<double> h(2 * n_tiles);
    if (cudaGetLastError() != cudaSuccess ||
        cudaMemcpyAsync(h.data(), sums.ptr, sizeof(double) * 2 * n_tiles, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess) {
      set_error("index collision estimate failed");
      return fail(SD_E_CUDA);
    }
    double sq = 0.0, dd = 0.0;
    for (int64_t t = 0; t < n_tiles; ++t) { dd += h[2 * t] * h[2 * t]; sq += h[2 * t + 1]; }
    ix->collide = dd > 0.0 ? sq / dd : 0.0;
  }
  // the chebyshev top-K masks and the hybrid heavy-row block are built on the
  // first call that needs them (ensure_cheb, ensure_hybrid)
  *out = ix;
  return SD_OK;
}

// chebyshev's copy of the postings with the rank of every posting's value in
// its index row (top-CHEB_K by |value|, else 255) packed into bits 16..23 of
// the row id, so the sweep loads one record per posting; the rank comes from
// the per-entry ranks: the posting's column follows from its (tile, column)
// key range, its entry from a binary search in the sorted row
template <typename T>
__global__ void cheb_rank_kernel(const uint32_t* __restrict__ colptr, const Posting<T>* __restrict__ post,
                                 int64_t n_keys, int64_t n_cols, int tile, const int64_t* __restrict__ bptr,
                                 const int32_t* __restrict__ bidx, const uint8_t* __restrict__ rank,
                                 Posting<T>* __restrict__ post_cheb) {
  for (int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < n_keys; k += int64_t(gridDim.x) * blockDim.x) {
    const int64_t base = (k / n_cols) * tile;
    const int32_t c = int32_t(k % n_cols);
    for (uint32_t p = colptr[k]; p < colptr[k + 1]; ++p) {
      Posting<T> q = post[p];
      const int64_t j = base + q.j;
      int64_t lo = bptr[j], hi = bptr[j + 1];
      while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (bidx[mid] < c) lo = mid + 1; else hi = mid;
      }
      q.j |= uint32_t(rank[lo]) << 16;
      post_cheb[p] = q;
    }
  }
}

// Chebyshev's per-row top-CHEB_K |values| and ranked postings, once per index.
int ensure_cheb(sd_index* ix, const sd_csr* b, cudaStream_t st) {
  std::lock_guard<std::mutex> lock(ix->mu);
  if (ix->topb) return SD_OK;
  const size_t es = ix->dtype == SD_F64 ? 8 : 4;
  const size_t ps = ix->dtype == SD_F64 ? sizeof(Posting<double>) : sizeof(Posting<float>);
  void* topb = nullptr;
  void* post_cheb = nullptr;
  if (cudaMalloc(&topb, es * CHEB_K * std::max<int64_t>(1, ix->n_rows)) != cudaSuccess ||
      cudaMalloc(&post_cheb, ps * std::max<int64_t>(1, ix->nnz)) != cudaSuccess) {
    if (topb) cudaFree(topb);
    set_error("cudaMalloc failed for the chebyshev masks");
    return SD_E_CUDA;
  }
  Scratch rank;
  int rc = rank.alloc(std::max<int64_t>(1, ix->nnz), st);
  if (rc == SD_OK) rc = row_topk(b, ix->dtype, rank.as<uint8_t>(), topb, st);
  if (rc == SD_OK && ix->nnz > 0) {
    const int64_t n_keys = ix->n_tiles * ix->n_cols;
    const int blocks = int(std::min<int64_t>((n_keys + 255) / 256, int64_t(num_sms()) * 16));
    rc = SD_DISPATCH_DTYPE(ix->dtype, T, [&]() -> int {
      cheb_rank_kernel<T><<<std::max(1, blocks), 256, 0, st>>>(ix->colptr, static_cast<const Posting<T>*>(ix->post),
                                                               n_keys, ix->n_cols, ix->tile, b->indptr, b->indices,
                                                               rank.as<uint8_t>(), static_cast<Posting<T>*>(post_cheb));
      SD_LAUNCH_CHECK();
      return SD_OK;
    });
  }
  if (rc != SD_OK) { cudaFree(topb); cudaFree(post_cheb); return rc; }
  ix->topb = topb;
  ix->post_cheb = post_cheb;
  ix->bytes += int64_t(es * CHEB_K * ix->n_rows + ps * ix->nnz);
  return SD_OK;
}

// The hybrid heavy-row block, on the first dot-family (HYB_DOT) or manhattan
// (HYB_MINSUM) call (index rows of degree >= n_cols/32; hybrid.cu).
int ensure_hybrid(sd_index* ix, const sd_csr* b, int kind, cudaStream_t st) {
  std::lock_guard<std::mutex> lock(ix->mu);
  return hybrid_index_build(b, ix->dtype, ix, kind, st);
}

// post_cos[p] = post[p] with the value times 1/||b_row|| (the tile of a
// posting follows from its (tile, column) key range)
template <typename T>
__global__ void post_scale_kernel(const uint32_t* __restrict__ colptr, const Posting<T>* __restrict__ post,
                                  int64_t n_keys, int64_t n_cols, int tile, const T* __restrict__ inv,
                                  Posting<T>* __restrict__ out) {
  for (int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < n_keys; k += int64_t(gridDim.x) * blockDim.x) {
    const int64_t base = (k / n_cols) * tile;
    for (uint32_t p = colptr[k]; p < colptr[k + 1]; ++p) {
      Posting<T> q = post[p];
      q.v = mul_rn(q.v, inv[base + q.j]);
      out[p] = q;
    }
  }
}

static int ensure_post_cos(sd_index* ix, const void* inv, cudaStream_t st) {
  std::lock_guard<std::mutex> lock(ix->mu);
  if (ix->post_cos) return SD_OK;
  const size_t ps = ix->dtype == SD_F64 ? sizeof(Posting<double>) : sizeof(Posting<float>);
  void* buf = nullptr;
  if (cudaMalloc(&buf, ps * std::max<int64_t>(1, ix->nnz)) != cudaSuccess) {
    set_error("cudaMalloc failed for the scaled cosine postings");
    return SD_E_CUDA;
  }
  const int64_t n_keys = ix->n_tiles * ix->n_cols;
  const int blocks = int(std::min<int64_t>((n_keys + 255) / 256, int64_t(num_sms()) * 16));
  const int rc = SD_DISPATCH_DTYPE(ix->dtype, T, [&]() -> int {
    post_scale_kernel<T><<<std::max(1, blocks), 256, 0, st>>>(ix->colptr, static_cast<const Posting<T>*>(ix->post),
                                                              n_keys, ix->n_cols, ix->tile, static_cast<const T*>(inv),
                                                              static_cast<Posting<T>*>(buf));
    SD_LAUNCH_CHECK();
    return SD_OK;
  });
  if (rc != SD_OK) { cudaFree(buf); return rc; }
  ix->post_cos = buf;
  ix->bytes += int64_t(ps) * ix->nnz;
  return SD_OK;
}

// Work plan (one CTA, no library sort): queries ordered by descending
// floor(log2(degree)) (LPT), each split into items of `tpi` consecutive tiles
// so that every item costs about total/(8·warps) — a power-law query of
// degree 25k is spread over up to n_tiles warps instead of serialising on one.
__global__ void __launch_bounds__(1024) plan_kernel(const int64_t* __restrict__ ptr, int64_t m, int64_t n_tiles,
                                                    int64_t band, int64_t warps, int64_t epi_cost, int tile_major,
                                                    const int32_t* __restrict__ skip,
                                                    int32_t* __restrict__ order, int32_t* __restrict__ tpi,
                                                    int64_t* __restrict__ item_off, int32_t* __restrict__ item_pos) {
  __shared__ unsigned int hist[64];
  __shared__ unsigned int base[64];
  __shared__ unsigned long long total;
  if (threadIdx.x < 64) hist[threadIdx.x] = 0;
  if (threadIdx.x == 0) total = 0;
  __syncthreads();
  // degree buckets with warp-aggregated shared atomics (power-law queries
  // crowd a few buckets: one atomic per distinct bucket in the warp)
  const unsigned lane = threadIdx.x & 31u;
  const unsigned lt = (1u << lane) - 1u;
  unsigned long long local = 0;
  for (int64_t r0 = 0; r0 < m; r0 += blockDim.x) {  // warp-uniform trip count
    const int64_t r = r0 + threadIdx.x;
    const bool ok = r < m;
    const int64_t d = ok ? ptr[r + 1] - ptr[r] : 0;
    const int b = d > 0 ? 63 - __clzll(d) : 0;
    const unsigned grp = __match_any_sync(0xffffffffu, ok ? unsigned(63 - b) : 64u + lane);
    if (ok && (grp & lt) == 0u) atomicAdd(&hist[63 - b], unsigned(__popc(grp)));
    if (ok && (!skip || skip[r] < 0)) local += (unsigned long long)(d + epi_cost);
  }
  atomicAdd(&total, local);
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned int acc = 0;
    for (int b = 0; b < 64; ++b) { base[b] = acc; acc += hist[b]; }
  }
  __syncthreads();
  for (int64_t r0 = 0; r0 < m; r0 += blockDim.x) {
    const int64_t r = r0 + threadIdx.x;
    const bool ok = r < m;
    const int64_t d = ok ? ptr[r + 1] - ptr[r] : 0;
    const int b = d > 0 ? 63 - __clzll(d) : 0;
    const unsigned grp = __match_any_sync(0xffffffffu, ok ? unsigned(63 - b) : 64u + lane);
    const int leader = __ffs(grp) - 1;
    unsigned pos0 = 0;
    if (ok && int(lane) == leader) pos0 = atomicAdd(&base[63 - b], unsigned(__popc(grp)));
    pos0 = __shfl_sync(0xffffffffu, pos0, leader);
    if (ok) order[pos0 + __popc(grp & lt)] = int32_t(r);
  }
  __syncthreads();
  if (tile_major) {  // items (tile t, position p) ordered tile-major: item = t * m + p
    for (int64_t q = threadIdx.x; q < m; q += blockDim.x) { tpi[q] = 1; item_off[q] = q * n_tiles; }
    if (threadIdx.x == 0) item_off[m] = m * n_tiles;
    return;
  }
  // items of one band (the list repeats for every band of `band` tiles)
  const int64_t target = tmax<int64_t>(1, int64_t(total) * band / tmax<int64_t>(1, warps * 8));
  // contiguous chunk per thread: items per position, then a block scan
  const int64_t chunk = (m + blockDim.x - 1) / blockDim.x;
  const int64_t lo = tmin<int64_t>(m, int64_t(threadIdx.x) * chunk), hi = tmin<int64_t>(m, lo + chunk);
  int64_t sum = 0;
  // 8 positions at a time: their row ids, then their degrees, are loaded
  // together (one round trip each instead of one per position); the item
  // count of each position is parked in item_off until the scan
  for (int64_t q0 = lo; q0 < hi; q0 += 8) {
    int64_t r[8], d[8];
    bool sk[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) r[u] = q0 + u < hi ? order[q0 + u] : 0;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      d[u] = q0 + u < hi ? ptr[r[u] + 1] - ptr[r[u]] : 0;
      sk[u] = q0 + u < hi && skip && skip[r[u]] >= 0;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (q0 + u < hi) {
        const int64_t t = tmin<int64_t>(band, tmax<int64_t>(1, target / (d[u] + epi_cost)));
        const int64_t cnt = sk[u] ? 0 : (band + t - 1) / t;  // rows of the hybrid path get no items
        tpi[q0 + u] = int32_t(t);
        item_off[q0 + u] = cnt;
        sum += cnt;
      }
    }
  }
  // block-wide exclusive scan of the per-thread item counts
  int64_t off;
  {
    typedef cub::BlockScan<int64_t, 1024> Scan;
    __shared__ typename Scan::TempStorage scan_tmp;
    int64_t total_items;
    Scan(scan_tmp).ExclusiveSum(sum, off, total_items);
    if (threadIdx.x == 0) item_off[m] = total_items;
  }
  for (int64_t q = lo; q < hi; ++q) {
    const int64_t cnt = item_off[q];
    item_off[q] = off;
    for (int64_t it = 0; it < cnt; ++it) item_pos[off + it] = int32_t(q);
    off += cnt;
  }
}

// Per-row statistics of both sides for the fused epilogue (norms for the
// dot family, one-sided sums for NAMM metrics, degrees of A for KL).
int hybrid_kind(int metric) {
  const int ck = metric_contrib(metric);
  return ck == C_MUL ? HYB_DOT : ck == C_ABS ? HYB_MINSUM : -1;
}

bool isect_hybrid_eligible(const sd_index* ix, const sd_metric_desc* md, int topk) {
  const int kind = hybrid_kind(md->metric);
  // kNN too (k <= 128): the heavy queries' dense rows go through a chunked top-k
  if (topk > 128 || kind < 0 || !ix || ix->n_heavy == 0 || !hybrid_enabled()) return false;
  if (!(kind == HYB_DOT ? ix->dot_ready : ix->ms_ready)) return false;
  return ix->n_tiles >= 4 || hybrid_forced();  // small indexes: the sweep is cheap, keep it exact
}

int isect_stats(const sd_csr* a, const sd_csr* b, const sd_index* ix_c, int dtype, const sd_metric_desc* md,
                Scratch& sa_buf, Scratch& sb_buf, Stats* sa, Stats* sb, bool defer_a, cudaStream_t st) {
  const size_t es = dtype == SD_F64 ? 8 : 4;
  if (md->metric == SD_M_CHEBYSHEV) {  // top-K |a| per query row + per-entry ranks; B side lives in the index
    const int64_t stride = stats_stride(std::max<int64_t>(1, a->n_rows));
    const int64_t nnz_span = std::max<int64_t>(1, a->nnz);
    SD_TRY(sa_buf.alloc(es * CHEB_K * stride + nnz_span, st));
    uint8_t* rank = reinterpret_cast<uint8_t*>(static_cast<char*>(sa_buf.ptr) + es * CHEB_K * stride);
    // top values K-major with row stride `stride`: row_topk writes [r * n_rows + row]
    sd_csr a2 = *a;
    SD_TRY(row_topk(&a2, dtype, rank, sa_buf.ptr, st));
    sa->s[0] = sa_buf.ptr;
    sa->s[2] = rank;
    if (!ix_c) { set_error("chebyshev fused path needs the index"); return SD_E_INVALID; }
    SD_TRY(ensure_cheb(const_cast<sd_index*>(ix_c), b, st));
    sb->s[0] = ix_c->topb;
    return SD_OK;
  }
  const int64_t ns = metric_stats_count(md->metric);
  if (ns == 0) return SD_OK;
  SD_TRY(sa_buf.alloc(es * ns * stats_stride(std::max<int64_t>(1, a->n_rows)), st));
  if (defer_a) {  // slot q of the buffer holds statistic q (metric_stats' layout for dot-family metrics)
    for (int64_t q = 0; q < ns && q < 3; ++q)
      sa->s[q] = static_cast<char*>(sa_buf.ptr) + size_t(q) * size_t(stats_stride(std::max<int64_t>(1, a->n_rows))) * es;
  } else {
    SD_TRY(metric_stats(a, dtype, md, true, sa_buf.ptr, sa, st));
  }
  if (md->metric == SD_M_KL) return SD_OK;
  sd_index* ix = const_cast<sd_index*>(ix_c);
  if (ix == nullptr) {
    SD_TRY(sb_buf.alloc(es * ns * stats_stride(std::max<int64_t>(1, b->n_rows)), st));
    return metric_stats(b, dtype, md, false, sb_buf.ptr, sb, st);
  }
  const double pk = is_namm(md->metric) ? md->p : 0.0;
  std::lock_guard<std::mutex> lock(ix->mu);
  for (auto& e : ix->stat_cache)
    if (e.metric == md->metric && e.p == pk) { *sb = e.stats; return SD_OK; }
  sd_index::StatEntry e{md->metric, pk, nullptr, Stats()};
  if (cudaMalloc(&e.buf, es * ns * stats_stride(std::max<int64_t>(1, b->n_rows))) != cudaSuccess) {
    set_error("cudaMalloc failed for index statistics");
    return SD_E_CUDA;
  }
  const int rc = metric_stats(b, dtype, md, false, e.buf, &e.stats, st);
  if (rc != SD_OK) { cudaFree(e.buf); return rc; }
  ix->stat_cache.push_back(e);
  *sb = e.stats;
  return SD_OK;
}

// Fused pairwise distances / kNN over the intersection path.
int isect_run(const sd_csr* a, const sd_csr* b, const sd_index* ix, int dtype, const sd_metric_desc* md,
              const Stats& sa, const Stats& sb, void* out, int64_t ldo, int topk, int64_t index_base,
              void* out_d, int64_t* out_i, uint32_t* flags, PhaseTimer* tm, bool a_stats_deferred,
              cudaStream_t st) {
  const int ck = metric_contrib(md->metric);
  if (ck < 0) { set_error("metric not decomposable over intersections"); return SD_E_UNSUPPORTED; }
  if (ix->dtype != dtype || ix->n_rows != b->n_rows || ix->n_cols != b->n_cols) {
    set_error("index does not match B / dtype");
    return SD_E_INVALID;
  }
  const int64_t m = a->n_rows;
  if (m == 0 || b->n_rows == 0) return SD_OK;
  if (m >= (int64_t(1) << 31)) { set_error("too many query rows"); return SD_E_INVALID; }
  const size_t es = dtype == SD_F64 ? 8 : 4;
  const int64_t per_warp = int64_t(ix->tile) * (int64_t(es) + isect_second_bytes(ck, int64_t(es)));
  const bool hyb = isect_hybrid_eligible(ix, md, topk);
  // with the hybrid gather in the sweep's shadow (hybrid.cu) the sweep leaves
  // room for its 128-thread block on every SM: 12 warps (192 KB, 48 K registers)
  const int64_t wcap = hyb && knob(SD_TUNE_GATHER_SHADOW) != 0 ? 12 : ISECT_MAX_WARPS;
  const int W = int(std::min<int64_t>(wcap, (smem_optin_bytes() - 2048) / per_warp));
  if (W < 1) { set_error("index tile does not fit shared memory"); return SD_E_INVALID; }
  const int64_t warps = int64_t(num_sms()) * W;
  // bands of tiles whose postings fit the L2 together, so the index streams
  // from HBM about once while every query sweeps the resident band; bands are
  // split evenly (no short tail band).  SD_ISECT_BAND overrides (tuning).
  const int tile_major = int(knob(SD_TUNE_ISECT_PLAN));  // experiment override: 1 = tile-major items
  // cosine over postings pre-divided by the index-row norms (built once per index)
  const bool cos_scaled = md->metric == SD_M_COSINE && sb.s[1] != nullptr && knob(SD_TUNE_COS_RAW) == 0;
  if (cos_scaled) SD_TRY(ensure_post_cos(const_cast<sd_index*>(ix), sb.s[1], st));
  // hybrid path (hybrid.cu, hminsum.cu): heavy query rows of dot-family
  // metrics and manhattan are computed densely; the sweep skips them
  // (declared before the hybrid state: its destructor makes the caller's
  // stream wait for the side streams before these buffers are released)
  Scratch order, tpi, item_off, item_pos, counter, cand_d, cand_i;
  HybridState hs;
  if (hyb) SD_TRY(hybrid_classify(a, ix, dtype, hybrid_kind(md->metric), hs, st));
  const int64_t be0 = knob(SD_TUNE_ISECT_BAND);
  // bytes the sweep streams: postings + their (tile, column) ranges (not the
  // hybrid block or the other metric's posting copy, which it never touches)
  const int64_t post_bytes = std::max<int64_t>(
      1, ix->nnz * int64_t(dtype == SD_F64 ? sizeof(Posting<double>) : sizeof(Posting<float>)) +
             int64_t(sizeof(uint32_t)) * (ix->n_tiles * ix->n_cols + 1));
  // once the hybrid path takes the heavy query rows, a band's postings take
  // about a fifth of the L2 (C2 cosine: bands of 100 MB 2.37 ms, 50 MB 2.28,
  // 25 MB 2.21, 12 MB 2.43) — the rest holds the streaming output.
  // Otherwise whole-L2 bands: with heavy rows in the sweep (C2 manhattan 4.9
  // vs 5.9 ms) smaller bands cost more than they save.
  const int64_t ld = knob(SD_TUNE_ISECT_L2_DIV);
  // Dense-ish indexes (long posting lists per (tile, column), C4: ~280) also
  // prefer the small bands (C4 46.4 -> 39.6 ms).
  const bool long_lists = ix->nnz > 64 * ix->n_tiles * ix->n_cols;
  const int64_t div = ld > 0 ? ld : (topk == 0 && (hyb || long_lists) ? 5 : 1);
  // kNN: bands of ~2.5 L2 — every item of a band starts an empty top-k list
  // and leaves one to merge, so fewer, longer items win over L2 residency
  // (C5 with the shared bound: 1 L2 23.1 ms, 2.5 L2 21.6, whole index 22.3)
  const int64_t band_bytes = std::max<int64_t>(
      1, topk > 0 && ld <= 0 ? l2_bytes() * 5 / 2 : l2_bytes() / std::max<int64_t>(1, div));
  const int64_t n_bands0 = (post_bytes + band_bytes - 1) / band_bytes;
  const int64_t auto_band = (ix->n_tiles + n_bands0 - 1) / n_bands0;
  const int64_t band0 = std::max<int64_t>(1, std::min<int64_t>(ix->n_tiles, be0 > 0 ? be0 : auto_band));
  const int64_t max_items = m * band0 * ((ix->n_tiles + band0 - 1) / band0);
  SD_TRY(order.alloc(sizeof(int32_t) * m, st));
  SD_TRY(tpi.alloc(sizeof(int32_t) * m, st));
  SD_TRY(item_off.alloc(sizeof(int64_t) * (m + 1), st));
  SD_TRY(item_pos.alloc(sizeof(int32_t) * max_items, st));
  SD_TRY(counter.alloc(sizeof(unsigned int), st));
  SD_CUDA_TRY(cudaMemsetAsync(counter.ptr, 0, sizeof(unsigned int), st));
  const int64_t band = band0;
  // On the hybrid path the work plan and the deferred query statistics only
  // need the classification: they run on a side stream, off the critical
  // path (the host's read of the heavy count, the dense block and the gather
  // proceed meanwhile); the sweep waits for them.
  cudaStream_t ps = st;
  if (hyb) {
    cudaStream_t s1 = side_stream(1);
    if (s1) {
      ps = s1;
      hs.main = st;
      SD_CUDA_TRY(cudaEventCreateWithFlags(&hs.cls, cudaEventDisableTiming));
      SD_CUDA_TRY(cudaEventRecord(hs.cls, st));
      SD_CUDA_TRY(cudaStreamWaitEvent(ps, hs.cls, 0));
    }
  }
  if (a_stats_deferred) {
    Stats tmp;
    SD_TRY(metric_stats(a, dtype, md, true, const_cast<void*>(sa.s[0]), &tmp, ps));
  }
  plan_kernel<<<1, 1024, 0, ps>>>(a->indptr, m, ix->n_tiles, band, warps, ix->tile / 16, tile_major,
                                  hyb ? hs.qid.as<int32_t>() : nullptr,
                                  order.as<int32_t>(), tpi.as<int32_t>(), item_off.as<int64_t>(),
                                  item_pos.as<int32_t>());
  SD_LAUNCH_CHECK();
  if (ps != st) {
    SD_CUDA_TRY(cudaEventCreateWithFlags(&hs.stats_done, cudaEventDisableTiming));
    SD_CUDA_TRY(cudaEventRecord(hs.stats_done, ps));
  }
  if (hyb) {
    if (tm) tm->begin(PH_PASS2);
    SD_TRY(hybrid_prepare(a, b, ix, dtype, hybrid_kind(md->metric), hs, st));
    if (tm) tm->end(PH_PASS2);
    if (hs.nhq > 0 && hs.join) {  // the dense block's sums (dqh) are complete at this point of st
      SD_CUDA_TRY(cudaEventCreateWithFlags(&hs.dense_done, cudaEventDisableTiming));
      SD_CUDA_TRY(cudaEventRecord(hs.dense_done, st));
    }
  }
  if (ps != st) SD_CUDA_TRY(cudaStreamWaitEvent(st, hs.stats_done, 0));
  Scratch kth;
  if (topk > 0) {
    SD_TRY(kth.alloc(8 * size_t(m), st));
    const int blocks = int(std::min<int64_t>((m + 255) / 256, int64_t(num_sms()) * 4));
    if (dtype == SD_F64)
      fill_key_kernel<long long><<<blocks, 256, 0, st>>>(kth.as<long long>(), m, 0x7ff0000000000000LL);
    else
      fill_key_kernel<int><<<blocks, 256, 0, st>>>(kth.as<int>(), m, 0x7f800000);
    SD_LAUNCH_CHECK();
    SD_TRY(cand_d.alloc(es * size_t(max_items) * topk, st));
    SD_TRY(cand_i.alloc(sizeof(int64_t) * size_t(max_items) * topk, st));
  }
  return SD_DISPATCH_DTYPE(dtype, T, [&]() -> int {
    IsectArgs<T> args;
    args.a_ptr = a->indptr; args.a_idx = a->indices; args.a_val = static_cast<const T*>(a->values);
    args.m = m;
    args.colptr = ix->colptr; args.post = static_cast<const Posting<T>*>(ix->post);
    args.tile = ix->tile; args.n_tiles = ix->n_tiles; args.n = ix->n_rows; args.n_cols = ix->n_cols;
    args.sa0 = static_cast<const T*>(sa.s[0]); args.sa1 = static_cast<const T*>(sa.s[1]);
    args.sb0 = static_cast<const T*>(sb.s[0]); args.sb1 = static_cast<const T*>(sb.s[1]);
    args.order = order.as<int32_t>(); args.tpi = tpi.as<int32_t>();
    args.item_off = item_off.as<int64_t>(); args.item_pos = item_pos.as<int32_t>();
    args.counter = counter.as<unsigned int>();
    args.tile_major = tile_major;
    args.skip = hs.nhq > 0 ? hs.qid.as<int32_t>() : nullptr;
    args.cos_scaled = cos_scaled ? 1 : 0;
    if (cos_scaled) args.post = static_cast<const Posting<T>*>(ix->post_cos);
    args.debug = int(knob(SD_TUNE_ISECT_DEBUG));
    args.band = band;
    args.strict = md->strict;
    args.k = T(a->n_cols); args.p = T(md->p);
    args.out = static_cast<T*>(out); args.ldo = ldo; args.flags = flags;
    args.topk = topk;
    args.heavy_compact = 0;
    args.cand_d = cand_d.as<T>(); args.cand_i = cand_i.as<int64_t>();
    args.kth = kth.as<typename OrdKey<T>::type>();
    args.a_rank = static_cast<const uint8_t*>(sa.s[2]);
    if (md->metric == SD_M_CHEBYSHEV) args.post = static_cast<const Posting<T>*>(ix->post_cheb);
    args.topa = static_cast<const T*>(sa.s[0]);
    args.topb = static_cast<const T*>(ix->topb);
    args.b_ptr = b->indptr; args.b_idx = b->indices; args.b_val = static_cast<const T*>(b->values);
    if (tm) tm->begin(PH_PASS1);
    SD_TRY(isect_launch(args, md->metric, W, st));
    // pairwise: the heavy rows' epilogue writes rows the sweep does not touch —
    // on side stream 0 after the gather and the dense block, it fills the SMs
    // the sweep's CTAs release at its tail instead of waiting for all of them
    if (topk == 0 && hs.nhq > 0 && hs.dense_done) {
      cudaStream_t side = side_stream(0);
      SD_CUDA_TRY(cudaStreamWaitEvent(side, hs.dense_done, 0));
      SD_TRY(isect_heavy_rows(args, md->metric, hs.hq.as<int32_t>(), hs.nhq, ix->hid, hs.dqh.as<T>(), ix->hpad,
                              hs.dlh.as<T>(), hs.qpad, side));
      SD_CUDA_TRY(cudaEventRecord(hs.join, side));  // (re-recorded: the caller's stream joins below)
      SD_CUDA_TRY(cudaStreamWaitEvent(st, hs.join, 0));
    }
    if (hs.nhq > 0 && knob(SD_TUNE_GATHER_SHADOW) != 0) SD_TRY(hybrid_gather(a, b, ix, dtype, hs, st));
    if (tm) tm->end(PH_PASS1);
    // kNN: the sweep's per-item lists are merged first (the heavy queries get
    // empty lists there), then the heavy queries' dense rows are selected
    if (topk > 0) SD_TRY(isect_merge(args, index_base, static_cast<T*>(out_d), out_i, st));
    if (hs.nhq > 0 && !(topk == 0 && hs.dense_done)) {
      if (tm) tm->begin(PH_EXPANSION);  // includes any wait for the side-stream gather
      SD_TRY(hs.wait(st));
      if (topk > 0) {  // dense rows [nhq][n] of the heavy queries, then their top-k
        const int64_t ldt = (ix->n_rows + 3) / 4 * 4;
        Scratch rowsbuf;
        SD_TRY(rowsbuf.alloc(es * size_t(hs.nhq) * size_t(ldt), st));
        IsectArgs<T> dense_rows = args;
        dense_rows.out = rowsbuf.as<T>();
        dense_rows.ldo = ldt;
        dense_rows.heavy_compact = 1;
        SD_TRY(isect_heavy_rows(dense_rows, md->metric, hs.hq.as<int32_t>(), hs.nhq, ix->hid, hs.dqh.as<T>(),
                                ix->hpad, hs.dlh.as<T>(), hs.qpad, st));
        SD_TRY(topk_rows_scatter(rowsbuf.ptr, hs.nhq, ix->n_rows, ldt, dtype, topk, index_base,
                                 hs.hq.as<int32_t>(), out_d, out_i, st));
      } else {
        SD_TRY(isect_heavy_rows(args, md->metric, hs.hq.as<int32_t>(), hs.nhq, ix->hid, hs.dqh.as<T>(), ix->hpad,
                                hs.dlh.as<T>(), hs.qpad, st));
      }
      if (tm) tm->end(PH_EXPANSION);
    }
    return SD_OK;
  });
}

}  // namespace sd

int sd_index_free(sd_index* ix) {
  if (!ix) return SD_OK;
  if (ix->colptr) cudaFree(ix->colptr);
  if (ix->post) cudaFree(ix->post);
  if (ix->post_cheb) cudaFree(ix->post_cheb);
  if (ix->topb) cudaFree(ix->topb);
  if (ix->post_cos) cudaFree(ix->post_cos);
  if (ix->dimg) cudaFree(ix->dimg);
  for (auto& e : ix->stat_cache) cudaFree(e.buf);
  sd::hybrid_index_free(ix);
  delete ix;
  return SD_OK;
}

int64_t sd_index_bytes(const sd_index* ix) { return ix ? ix->bytes : 0; }
int sd_index_tile_rows(const sd_index* ix) { return ix ? ix->tile : 0; }
int64_t sd_index_heavy_rows(const sd_index* ix) { return ix ? ix->n_heavy : 0; }
int sd_index_hybrid_blocks(const sd_index* ix) {
  if (!ix) return 0;
  return (ix->dot_ready ? 1 : 0) | (ix->ms_ready ? 2 : 0) | (ix->dimg ? 4 : 0) | (ix->dplanes == 2 ? 8 : 0) |
         (ix->dimg && ix->dints ? 16 : 0);
}
