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
#include <cub/cub.cuh>
#include "common.cuh"
#include "metric.cuh"
#include "prep.cuh"
#include "topk.cuh"

struct sd_index {
  int64_t n_rows = 0, n_cols = 0, nnz = 0;
  int tile = 0;
  int64_t n_tiles = 0;
  int dtype = 0;
  uint32_t* colptr = nullptr;  // [n_tiles * n_cols + 1]
  uint16_t* post_j = nullptr;  // [nnz] row id within tile
  void* post_v = nullptr;      // [nnz] value
  int64_t bytes = 0;
};

namespace sd {

int default_tile(int dtype) { return dtype == SD_F64 ? 2048 : 4096; }

__global__ void index_count_kernel(const int64_t* __restrict__ ptr, const int32_t* __restrict__ idx,
                                   int64_t n_rows, int tile, int64_t n_cols, uint32_t* counts) {
  const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t r = warp; r < n_rows; r += nw) {
    const int64_t base = (r / tile) * n_cols;
    for (int64_t e = ptr[r] + lane_id(); e < ptr[r + 1]; e += 32) atomicAdd(&counts[base + idx[e]], 1u);
  }
}

template <typename T>
__global__ void index_scatter_kernel(const int64_t* __restrict__ ptr, const int32_t* __restrict__ idx,
                                     const T* __restrict__ val, int64_t n_rows, int tile, int64_t n_cols,
                                     const uint32_t* __restrict__ colptr, uint32_t* cursor,
                                     uint16_t* __restrict__ pj, T* __restrict__ pv) {
  const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t r = warp; r < n_rows; r += nw) {
    const int64_t t = r / tile;
    const int64_t base = t * n_cols;
    for (int64_t e = ptr[r] + lane_id(); e < ptr[r + 1]; e += 32) {
      const int64_t key = base + idx[e];
      const uint32_t pos = colptr[key] + atomicAdd(&cursor[key], 1u);
      pj[pos] = uint16_t(r - t * tile);
      pv[pos] = val[e];
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
  if (cudaMalloc(&ix->colptr, sizeof(uint32_t) * (n_keys + 1)) != cudaSuccess ||
      cudaMalloc(&ix->post_j, sizeof(uint16_t) * std::max<int64_t>(1, b->nnz)) != cudaSuccess ||
      cudaMalloc(&ix->post_v, es * std::max<int64_t>(1, b->nnz)) != cudaSuccess) {
    set_error("cudaMalloc failed for the inverted index");
    return fail(SD_E_CUDA);
  }
  ix->bytes = int64_t(sizeof(uint32_t) * (n_keys + 1) + (2 + es) * b->nnz);
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
                                                      counts.as<uint32_t>(), ix->post_j, static_cast<T*>(ix->post_v));
      SD_LAUNCH_CHECK();
      return SD_OK;
    });
    if (rc != SD_OK) return fail(rc);
  }
  *out = ix;
  return SD_OK;
}

// ---------------------------------------------------------------- kernel

template <typename T>
struct IsectArgs {
  const int64_t* a_ptr;
  const int32_t* a_idx;
  const T* a_val;
  int64_t m;
  const uint32_t* colptr;
  const uint16_t* pj;
  const T* pv;
  int tile;
  int64_t n_tiles, n, n_cols;
  const T* sa0; const T* sa1; const T* sb0; const T* sb1;
  const int32_t* order;
  unsigned int* counter;
  int metric, strict;
  T k, p;
  T* out;
  int64_t ldo;
  uint32_t* flags;
  int topk;
  int64_t index_base;
  T* out_d;
  int64_t* out_i;
};

constexpr int ISECT_U = 8;  // columns whose first postings are in flight at once

template <typename T, int CK>
__device__ __forceinline__ T fused_value(const IsectArgs<T>& a, T acc, T cnt, T ra0, T ra1, T rb0, T rb1,
                                         uint32_t& flags) {
  if constexpr (CK == C_KL) {
    if (cnt != ra0) {  // some column of A_i is absent from B_j (metrics.py:352-366)
      if (a.strict) flags |= SD_FLAG_KL_UNCOVERED;
      return Num<T>::big();
    }
    return acc;
  } else if constexpr (CK == C_MUL) {
    return expand_cell<T>(a.metric, acc, ra0, ra1, rb0, rb1, a.k, a.p, flags);
  } else {
    T x = add_rn(add_rn(ra0, rb0), acc);
    x = x < T(0) ? T(0) : x;  // cancellation residue of the union decomposition
    return expand_cell<T>(a.metric, x, T(0), T(0), T(0), T(0), a.k, a.p, flags);
  }
}

template <typename T, int CK, int KPL>
__global__ void __launch_bounds__(512) isect_kernel(const IsectArgs<T> a) {
  extern __shared__ __align__(16) unsigned char smem[];
  constexpr bool KL = CK == C_KL;
  constexpr unsigned FULL = 0xffffffffu;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int TJ = a.tile;
  T* acc = reinterpret_cast<T*>(smem) + size_t(warp) * TJ * (KL ? 2 : 1);
  T* cnt = acc + TJ;
  const T p = a.p;
  uint32_t flags = 0;

  while (true) {
    unsigned qi = 0;
    if (lane == 0) qi = atomicAdd(a.counter, 1u);
    qi = __shfl_sync(FULL, qi, 0);
    if (int64_t(qi) >= a.m) break;
    const int64_t i = a.order ? int64_t(a.order[qi]) : int64_t(qi);
    const int64_t abeg = a.a_ptr[i], aend = a.a_ptr[i + 1];
    const T ra0 = a.sa0 ? a.sa0[i] : T(0);
    const T ra1 = a.sa1 ? a.sa1[i] : T(0);
    WarpTopK<T, (KPL > 0 ? KPL : 1)> top;
    if constexpr (KPL > 0) top.init();

    for (int64_t t = 0; t < a.n_tiles; ++t) {
      const int64_t j0 = t * TJ;
      const int nt = int(tmin<int64_t>(TJ, a.n - j0));
      for (int q = lane; q < nt; q += 32) {
        acc[q] = T(0);
        if constexpr (KL) cnt[q] = T(0);
      }
      __syncwarp();
      const uint32_t* cp = a.colptr + t * a.n_cols;
      for (int64_t base = abeg; base < aend; base += 32) {
        const int64_t e = base + lane;
        const bool valid = e < aend;
        const int32_t c = valid ? a.a_idx[e] : 0;
        const T av = valid ? a.a_val[e] : T(0);
        const uint32_t pb = valid ? cp[c] : 0u;
        const uint32_t pe = valid ? cp[c + 1] : 0u;
        const int ncol = int(tmin<int64_t>(32, aend - base));
        for (int q0 = 0; q0 < ncol; q0 += ISECT_U) {
          uint32_t b0[ISECT_U], b1[ISECT_U];
          T x[ISECT_U], y[ISECT_U];
          int jl[ISECT_U];
#pragma unroll
          for (int u = 0; u < ISECT_U; ++u) {
            const int q = (q0 + u) & 31;
            b0[u] = __shfl_sync(FULL, pb, q);
            b1[u] = __shfl_sync(FULL, pe, q);
            x[u] = __shfl_sync(FULL, av, q);
            if (q0 + u >= ncol) b1[u] = b0[u];
            const uint32_t pp = b0[u] + lane;
            jl[u] = 0;
            y[u] = T(0);
            if (pp < b1[u]) {
              jl[u] = a.pj[pp];
              y[u] = a.pv[pp];
            }
          }
#pragma unroll
          for (int u = 0; u < ISECT_U; ++u) {
            const uint32_t pp = b0[u] + lane;
            if (pp < b1[u]) {
              acc[jl[u]] = add_rn(acc[jl[u]], contrib<CK, T>(x[u], y[u], p));
              if constexpr (KL) cnt[jl[u]] = add_rn(cnt[jl[u]], T(1));
              for (uint32_t p2 = pp + 32; p2 < b1[u]; p2 += 32) {
                const int j2 = a.pj[p2];
                acc[j2] = add_rn(acc[j2], contrib<CK, T>(x[u], a.pv[p2], p));
                if constexpr (KL) cnt[j2] = add_rn(cnt[j2], T(1));
              }
            }
            __syncwarp();
          }
        }
      }
      // epilogue over the tile's cells
      for (int q = 0; q < nt; q += 32) {
        const int l = q + lane;
        const bool valid = l < nt;
        const int64_t j = j0 + l;
        T d = T(0);
        if (valid) {
          const T rb0 = a.sb0 ? a.sb0[j] : T(0);
          const T rb1 = a.sb1 ? a.sb1[j] : T(0);
          d = fused_value<T, CK>(a, acc[l], KL ? cnt[l] : T(0), ra0, ra1, rb0, rb1, flags);
        }
        if constexpr (KPL > 0) {
          top.offer(valid, d, j, a.topk);
        } else {
          if (valid) a.out[i * a.ldo + j] = d;
        }
      }
      __syncwarp();
    }
    if constexpr (KPL > 0) top.store(a.topk, a.out_d + i * a.topk, a.out_i + i * a.topk, a.index_base);
  }
  flags = __reduce_or_sync(FULL, flags);
  if (flags && lane == 0) atomicOr(a.flags, flags);
}

template <typename T, int CK, int KPL>
static int launch_isect(IsectArgs<T>& args, cudaStream_t st) {
  const int64_t optin = smem_optin_bytes() - static_smem((const void*)isect_kernel<T, CK, KPL>);
  const int64_t per_warp = int64_t(args.tile) * sizeof(T) * (CK == C_KL ? 2 : 1);
  int W = int(std::min<int64_t>(16, (optin - 1024) / per_warp));
  if (W < 1) { set_error("index tile does not fit shared memory"); return SD_E_INVALID; }
  const size_t smem = size_t(W) * per_warp;
  SD_TRY(prepare_smem(isect_kernel<T, CK, KPL>, smem, "isect_kernel"));
  int per_sm = 0;
  SD_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, isect_kernel<T, CK, KPL>, W * 32, smem));
  per_sm = std::max(1, per_sm);
  const int64_t warps_needed = args.m;
  int64_t blocks = std::min<int64_t>(int64_t(num_sms()) * per_sm, (warps_needed + W - 1) / W);
  blocks = std::max<int64_t>(1, blocks);
  isect_kernel<T, CK, KPL><<<unsigned(blocks), W * 32, smem, st>>>(args);
  SD_LAUNCH_CHECK();
  return SD_OK;
}

// Query schedule: rows ordered by descending floor(log2(degree)) so the
// dynamic queue hands out the longest rows first (LPT).  One CTA: bucket
// histogram, scan, scatter — no library sort in the hot path.
__global__ void __launch_bounds__(1024) degree_order_kernel(const int64_t* __restrict__ ptr, int64_t m,
                                                            int32_t* __restrict__ order) {
  __shared__ unsigned int hist[64];
  __shared__ unsigned int base[64];
  if (threadIdx.x < 64) hist[threadIdx.x] = 0;
  __syncthreads();
  for (int64_t r = threadIdx.x; r < m; r += blockDim.x) {
    const int64_t d = ptr[r + 1] - ptr[r];
    const int b = d > 0 ? 63 - __clzll(d) : 0;   // floor(log2 d)
    atomicAdd(&hist[63 - b], 1u);                // descending degree
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned int acc = 0;
    for (int b = 0; b < 64; ++b) { base[b] = acc; acc += hist[b]; }
  }
  __syncthreads();
  for (int64_t r = threadIdx.x; r < m; r += blockDim.x) {
    const int64_t d = ptr[r + 1] - ptr[r];
    const int b = d > 0 ? 63 - __clzll(d) : 0;
    order[atomicAdd(&base[63 - b], 1u)] = int32_t(r);
  }
}

static int degree_order(const sd_csr* a, cudaStream_t st, Scratch& order_buf) {
  SD_TRY(order_buf.alloc(sizeof(int32_t) * std::max<int64_t>(1, a->n_rows), st));
  degree_order_kernel<<<1, 1024, 0, st>>>(a->indptr, a->n_rows, order_buf.as<int32_t>());
  SD_LAUNCH_CHECK();
  return SD_OK;
}

// Per-row statistics of both sides for the fused epilogue (norms for the
// dot family, one-sided sums for NAMM metrics, degrees of A for KL).
int isect_stats(const sd_csr* a, const sd_csr* b, int dtype, const sd_metric_desc* md, Scratch& sa_buf,
                Scratch& sb_buf, Stats* sa, Stats* sb, cudaStream_t st) {
  const size_t es = dtype == SD_F64 ? 8 : 4;
  const int64_t ns = metric_stats_count(md->metric);
  if (ns == 0) return SD_OK;
  SD_TRY(sa_buf.alloc(es * ns * std::max<int64_t>(1, a->n_rows), st));
  SD_TRY(metric_stats(a, dtype, md, true, sa_buf.ptr, sa, st));
  if (md->metric != SD_M_KL) {
    SD_TRY(sb_buf.alloc(es * ns * std::max<int64_t>(1, b->n_rows), st));
    SD_TRY(metric_stats(b, dtype, md, false, sb_buf.ptr, sb, st));
  }
  return SD_OK;
}

// Fused pairwise distances / kNN over the intersection path.
int isect_run(const sd_csr* a, const sd_csr* b, const sd_index* ix, int dtype, const sd_metric_desc* md,
              const Stats& sa, const Stats& sb, void* out, int64_t ldo, int topk, int64_t index_base,
              void* out_d, int64_t* out_i, uint32_t* flags, cudaStream_t st) {
  const int ck = metric_contrib(md->metric);
  if (ck < 0) { set_error("metric not decomposable over intersections"); return SD_E_UNSUPPORTED; }
  if (ix->dtype != dtype || ix->n_rows != b->n_rows || ix->n_cols != b->n_cols) {
    set_error("index does not match B / dtype");
    return SD_E_INVALID;
  }
  if (a->n_rows == 0 || b->n_rows == 0) return SD_OK;
  Scratch order, counter;
  SD_TRY(degree_order(a, st, order));
  SD_TRY(counter.alloc(sizeof(unsigned int), st));
  SD_CUDA_TRY(cudaMemsetAsync(counter.ptr, 0, sizeof(unsigned int), st));
  return SD_DISPATCH_DTYPE(dtype, T, [&]() -> int {
    IsectArgs<T> args;
    args.a_ptr = a->indptr; args.a_idx = a->indices; args.a_val = static_cast<const T*>(a->values);
    args.m = a->n_rows;
    args.colptr = ix->colptr; args.pj = ix->post_j; args.pv = static_cast<const T*>(ix->post_v);
    args.tile = ix->tile; args.n_tiles = ix->n_tiles; args.n = ix->n_rows; args.n_cols = ix->n_cols;
    args.sa0 = static_cast<const T*>(sa.s[0]); args.sa1 = static_cast<const T*>(sa.s[1]);
    args.sb0 = static_cast<const T*>(sb.s[0]); args.sb1 = static_cast<const T*>(sb.s[1]);
    args.order = order.as<int32_t>();
    args.counter = counter.as<unsigned int>();
    args.metric = md->metric; args.strict = md->strict;
    args.k = T(a->n_cols); args.p = T(md->p);
    args.out = static_cast<T*>(out); args.ldo = ldo; args.flags = flags;
    args.topk = topk; args.index_base = index_base;
    args.out_d = static_cast<T*>(out_d); args.out_i = out_i;
    auto go = [&](auto ck_tag) -> int {
      constexpr int CK = decltype(ck_tag)::value;
      if (topk <= 0) return launch_isect<T, CK, 0>(args, st);
      if (topk <= 32) return launch_isect<T, CK, 1>(args, st);
      return launch_isect<T, CK, 4>(args, st);
    };
    switch (ck) {
      case C_MUL: return go(std::integral_constant<int, C_MUL>());
      case C_KL: return go(std::integral_constant<int, C_KL>());
      case C_ABS: return go(std::integral_constant<int, C_ABS>());
      case C_ABSPOW: return go(std::integral_constant<int, C_ABSPOW>());
      case C_CANBERRA: return go(std::integral_constant<int, C_CANBERRA>());
      case C_MISMATCH: return go(std::integral_constant<int, C_MISMATCH>());
      default: return go(std::integral_constant<int, C_JS>());
    }
  });
}

}  // namespace sd

int sd_index_free(sd_index* ix) {
  if (!ix) return SD_OK;
  if (ix->colptr) cudaFree(ix->colptr);
  if (ix->post_j) cudaFree(ix->post_j);
  if (ix->post_v) cudaFree(ix->post_v);
  delete ix;
  return SD_OK;
}

int64_t sd_index_bytes(const sd_index* ix) { return ix ? ix->bytes : 0; }
int sd_index_tile_rows(const sd_index* ix) { return ix ? ix->tile : 0; }
