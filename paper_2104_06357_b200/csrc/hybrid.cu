// hybrid.cu — dense path for heavy query rows (dot-family metrics).
//
// On power-law data a few query rows carry most of the query nonzeros (C2:
// the 1.4% of queries with >= n_cols/32 nonzeros hold ~80% of them) and a few
// index rows most of the index nonzeros.  In the intersection sweep a query
// costs one warp step per (query column, index tile) pair, so those heavy
// queries dominate the sweep although they are a handful of output rows.
// Their rows are computed densely instead:
//
//   heavy queries x heavy index rows   GEMM   HQT^T[nhq x K] * HT[K x n_heavy]
//   heavy queries x light index rows   gather DLH[j][q] = sum_c b_jc * HQT[c][q]
//
// where HT (index build, cached) and HQT (per call) are the dense, column-
// major (K-major) images of the heavy rows.  heavy_rows_kernel
// (isect_kernel.cuh) then applies the metric epilogue to those rows; the
// sweep handles every other query row.  Only metrics whose contribution is a
// product (semiring.py:76-78) take this path: their dense sums equal the
// sparse intersection sums up to rounding (products with an absent entry are
// exact zeros).
#include <algorithm>
#include <mutex>
#include <string>
#include <cstdlib>
#include <vector>
#include "index.cuh"
#include "isect_kernel.cuh"
#include "hybrid.cuh"

namespace sd {

int64_t hybrid_threshold(int64_t n_cols) {
  const int64_t t = knob(SD_TUNE_HEAVY_DEG);
  return std::max<int64_t>(64, t > 0 ? t : (n_cols + 31) / 32);
}

// SD_TUNE_HYBRID: 0 off, 1 automatic (default), 2 forced even for small indexes (tests)
bool hybrid_enabled() { return knob(SD_TUNE_HYBRID) != 0; }
bool hybrid_forced() { return knob(SD_TUNE_HYBRID) == 2; }

// ---------------------------------------------------------------- index side

// dense[(h / 128) * bstride + idx * ld + h % 128] = val for the nonzeros of
// rows[h] (bstride = 128, ld = pad: the [n_cols][pad] image; bstride =
// n_cols * 128, ld = 128: 128-row blocks, each [n_cols][128]); POS stores
// max(val, 0) (the min-sum image).  Block (h, c) of a (rows x chunks) grid
// takes every chunks-th 256-wide slice of row rows[h], so a handful of long
// rows still spreads over the whole GPU.
template <typename T, bool POS>
__global__ void ht_scatter_kernel(const int64_t* __restrict__ ptr, const int32_t* __restrict__ idx,
                                  const T* __restrict__ val, const int32_t* __restrict__ rows, int64_t nrows,
                                  int64_t bstride, int64_t ld, T* __restrict__ dense) {
  for (int64_t h = blockIdx.x; h < nrows; h += gridDim.x) {
    const int64_t r = rows[h];
    T* base = dense + (h >> 7) * bstride + (h & 127);
    const int64_t step = int64_t(gridDim.y) * blockDim.x;
    for (int64_t e = ptr[r] + int64_t(blockIdx.y) * blockDim.x + threadIdx.x; e < ptr[r + 1]; e += step) {
      const T v = val[e];
      base[int64_t(idx[e]) * ld] = POS ? (v > T(0) ? v : T(0)) : v;
    }
  }
}

dim3 row_scatter_grid(int64_t nrows) {
  const int64_t chunks = std::min<int64_t>(64, std::max<int64_t>(1, (int64_t(num_sms()) * 8 + nrows - 1) /
                                                                        std::max<int64_t>(1, nrows)));
  return dim3{unsigned(std::min<int64_t>(std::max<int64_t>(1, nrows), 65535)), unsigned(chunks), 1u};
}

// the common part: heavy ids (degree >= theta), light rows by descending degree
static int hybrid_base_build(const sd_csr* b, sd_index* ix, cudaStream_t st) {
  const int64_t theta = hybrid_threshold(b->n_cols);
  std::vector<int64_t> ptr(b->n_rows + 1);
  SD_CUDA_TRY(cudaMemcpyAsync(ptr.data(), b->indptr, sizeof(int64_t) * (b->n_rows + 1), cudaMemcpyDeviceToHost, st));
  SD_CUDA_TRY(cudaStreamSynchronize(st));
  std::vector<int32_t> hid(b->n_rows, -1), rows, light;
  for (int64_t r = 0; r < b->n_rows; ++r) {
    if (ptr[r + 1] - ptr[r] >= theta) { hid[r] = int32_t(rows.size()); rows.push_back(int32_t(r)); }
    else light.push_back(int32_t(r));
  }
  auto deg = [&](int32_t r) { return ptr[r + 1] - ptr[r]; };
  // light rows by descending degree: the dense gather takes the long ones first
  std::stable_sort(light.begin(), light.end(), [&](int32_t x, int32_t y) { return deg(x) > deg(y); });
  const int64_t nh = int64_t(rows.size());
  if (nh < 32) return SD_OK;  // nothing worth a dense block
  std::vector<int32_t> perm(nh);
  for (int64_t h = 0; h < nh; ++h) perm[h] = int32_t(h);
  std::stable_sort(perm.begin(), perm.end(), [&](int32_t x, int32_t y) { return deg(rows[x]) > deg(rows[y]); });
  if (cudaMalloc(&ix->hid, sizeof(int32_t) * b->n_rows) != cudaSuccess ||
      cudaMalloc(&ix->hrows, sizeof(int32_t) * nh) != cudaSuccess ||
      cudaMalloc(&ix->hperm, sizeof(int32_t) * nh) != cudaSuccess ||
      cudaMalloc(&ix->lrows, sizeof(int32_t) * std::max<size_t>(1, light.size())) != cudaSuccess) {
    set_error("cudaMalloc failed for the hybrid index");
    return SD_E_CUDA;
  }
  SD_CUDA_TRY(cudaMemcpyAsync(ix->hid, hid.data(), sizeof(int32_t) * b->n_rows, cudaMemcpyHostToDevice, st));
  SD_CUDA_TRY(cudaMemcpyAsync(ix->hrows, rows.data(), sizeof(int32_t) * nh, cudaMemcpyHostToDevice, st));
  SD_CUDA_TRY(cudaMemcpyAsync(ix->hperm, perm.data(), sizeof(int32_t) * nh, cudaMemcpyHostToDevice, st));
  if (!light.empty())
    SD_CUDA_TRY(cudaMemcpyAsync(ix->lrows, light.data(), sizeof(int32_t) * light.size(), cudaMemcpyHostToDevice, st));
  SD_CUDA_TRY(cudaStreamSynchronize(st));  // the host vectors must outlive the transfers
  ix->heavy_deg = theta;
  ix->n_heavy = nh;
  ix->hpad = (nh + 127) / 128 * 128;
  ix->n_light = int64_t(light.size());
  ix->bytes += int64_t(sizeof(int32_t)) * (b->n_rows + 2 * nh + ix->n_light);
  return SD_OK;
}

// dot family: HT (dense, column-major) and, for fp32, the tensor-core GEMM's
// A-operand image
static int hybrid_dot_build(const sd_csr* b, int dtype, sd_index* ix, cudaStream_t st) {
  const int64_t nh = ix->n_heavy, pad = ix->hpad;
  const int64_t cap = knob(SD_TUNE_HYBRID_MAX_MB) << 20;
  if (dtype == SD_F32) {  // the heavy rows as the tcgen05 GEMM's bf16 operand image (dense_tc.cu)
    Scratch flag;
    SD_TRY(flag.alloc(sizeof(unsigned int), st));
    SD_CUDA_TRY(cudaMemsetAsync(flag.ptr, 0, sizeof(unsigned int), st));
    SD_TRY(check_bf16_exact(b, flag.as<unsigned int>(), st));
    unsigned int inexact = 0;
    SD_CUDA_TRY(cudaMemcpyAsync(&inexact, flag.ptr, sizeof(inexact), cudaMemcpyDeviceToHost, st));
    SD_CUDA_TRY(cudaStreamSynchronize(st));
    const int planes = (inexact & 1u) ? 2 : 1;
    const int64_t nkb = dense_kblocks(b->n_cols);
    const size_t tbytes = dense_image_bytes(nh, nkb, planes, 128);
    if (int64_t(tbytes) > cap) return SD_OK;
    if (cudaMalloc(&ix->hbf, tbytes) != cudaSuccess) {
      set_error("cudaMalloc failed for the hybrid index (bf16 image)");
      return SD_E_CUDA;
    }
    SD_TRY(dense_image(b, ix->hrows, nh, nkb, planes, 128, ix->hbf, st));
    SD_CUDA_TRY(cudaStreamSynchronize(st));
    ix->hbf_planes = planes;
    ix->hbf_nkb = nkb;
    ix->bytes += int64_t(tbytes);
    ix->dot_ready = true;
    return SD_OK;
  }
  // fp64: HT, dense column-major, for the CUDA-core DFMA GEMM
  const int64_t dense_bytes = b->n_cols * pad * 8;
  if (dense_bytes > cap) return SD_OK;
  if (cudaMalloc(&ix->ht, dense_bytes) != cudaSuccess) {
    set_error("cudaMalloc failed for the hybrid index");
    return SD_E_CUDA;
  }
  SD_CUDA_TRY(cudaMemsetAsync(ix->ht, 0, dense_bytes, st));
  ht_scatter_kernel<double, false><<<row_scatter_grid(nh), 256, 0, st>>>(
      b->indptr, b->indices, static_cast<const double*>(b->values), ix->hrows, nh, 128, pad, static_cast<double*>(ix->ht));
  SD_LAUNCH_CHECK();
  SD_CUDA_TRY(cudaStreamSynchronize(st));
  ix->bytes += dense_bytes;
  ix->dot_ready = true;
  return SD_OK;
}

// min-sum (manhattan): only for an index without negative (or NaN) values,
// where |a - b| - |a| - |b| = -2 min(max(a, 0), b) for every a
static int hybrid_minsum_build(const sd_csr* b, int dtype, sd_index* ix, cudaStream_t st) {
  Scratch flag;
  SD_TRY(flag.alloc(sizeof(unsigned int), st));
  SD_CUDA_TRY(cudaMemsetAsync(flag.ptr, 0, sizeof(unsigned int), st));
  SD_TRY(minsum_check_index(b, dtype, flag.as<unsigned int>(), st));
  unsigned int bad = 0;
  SD_CUDA_TRY(cudaMemcpyAsync(&bad, flag.ptr, sizeof(bad), cudaMemcpyDeviceToHost, st));
  SD_CUDA_TRY(cudaStreamSynchronize(st));
  if (bad) return SD_OK;
  const int64_t nch = (b->n_cols + minsum_chunk_cols(dtype) - 1) / minsum_chunk_cols(dtype);
  const size_t bytes = sizeof(int64_t) * size_t(ix->n_heavy) * size_t(nch + 1);
  if (cudaMalloc(&ix->hchunk, bytes) != cudaSuccess) {
    set_error("cudaMalloc failed for the min-sum chunk pointers");
    return SD_E_CUDA;
  }
  SD_TRY(minsum_chunks(b, dtype, ix->hrows, ix->n_heavy, nch, ix->hchunk, st));
  ix->ms_nch = nch;
  ix->bytes += int64_t(bytes);
  ix->ms_ready = true;
  return SD_OK;
}

int hybrid_index_build(const sd_csr* b, int dtype, sd_index* ix, int kind, cudaStream_t st) {
  if (!hybrid_enabled() || b->n_rows == 0 || b->nnz == 0) return SD_OK;
  if (!ix->hybrid_tried) {
    ix->hybrid_tried = true;
    SD_TRY(hybrid_base_build(b, ix, st));
  }
  if (ix->n_heavy == 0) return SD_OK;
  if (kind == HYB_DOT && !ix->dot_tried) {
    ix->dot_tried = true;
    return hybrid_dot_build(b, dtype, ix, st);
  }
  if (kind == HYB_MINSUM && !ix->ms_tried) {
    ix->ms_tried = true;
    return hybrid_minsum_build(b, dtype, ix, st);
  }
  return SD_OK;
}

void hybrid_index_free(sd_index* ix) {
  if (ix->hid) cudaFree(ix->hid);
  if (ix->ht) cudaFree(ix->ht);
  if (ix->lrows) cudaFree(ix->lrows);
  if (ix->hbf) cudaFree(ix->hbf);
  if (ix->hrows) cudaFree(ix->hrows);
  if (ix->hperm) cudaFree(ix->hperm);
  if (ix->hchunk) cudaFree(ix->hchunk);
  ix->hbf = nullptr;
  ix->hrows = nullptr;
  ix->hperm = nullptr;
  ix->hchunk = nullptr;
  ix->hid = nullptr;
  ix->ht = nullptr;
  ix->lrows = nullptr;
}

// ---------------------------------------------------------------- query side

// non-blocking side streams per device (created once, never destroyed):
// 0 carries the dense gather, 1 the deferred query statistics and work plan
cudaStream_t side_stream(int which) {
  static std::mutex mu;
  static cudaStream_t streams[2][64] = {};
  int dev = 0;
  if (which < 0 || which > 1 || cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
  std::lock_guard<std::mutex> lock(mu);
  cudaStream_t& s = streams[which][dev];
  // highest priority: the side streams carry latency-bound work (gather,
  // statistics, work plan) that should be dispatched onto free SM resources
  // ahead of the pending CTAs of the dense block on the caller's stream
  int lo = 0, hi = 0;
  if (cudaDeviceGetStreamPriorityRange(&lo, &hi) != cudaSuccess) hi = 0;
  if (!s && cudaStreamCreateWithPriority(&s, cudaStreamNonBlocking, hi) != cudaSuccess) s = nullptr;
  return s;
}

// heavy query rows get ids 0..cap-1 (the id order is irrelevant to results:
// every heavy row is computed independently of its slot)
__global__ void classify_kernel(const int64_t* __restrict__ ptr, int64_t m, int64_t theta, int cap,
                                int32_t* __restrict__ qid, int32_t* __restrict__ hq, unsigned int* count) {
  for (int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < m; r += int64_t(gridDim.x) * blockDim.x) {
    int32_t id = -1;
    if (ptr[r + 1] - ptr[r] >= theta) {
      const unsigned int k = atomicAdd(count, 1u);
      if (k < unsigned(cap)) { id = int32_t(k); hq[k] = int32_t(r); }
    }
    qid[r] = id;
  }
}

// GEMM D = A^T B with A = HQT [K][lda] (heavy queries), B = HT [K][ldb] (heavy
// index rows), both K-major (the fp64 heavy block).  CTA tile 64 x 128, 128
// threads with 8 x 8 accumulators each (16 operands read from shared memory
// per 64 FMAs, as 16-byte vectors; 4 x 8 left the kernel shared-memory bound
// at a sixth of the fp64 peak), K
// split across blockIdx.z into partial tiles that hreduce_kernel sums in
// split order (deterministic).
constexpr int HG_BM = 64, HG_BN = 128, HG_BK = 16, HG_THREADS = 128;

template <typename T>
__global__ void __launch_bounds__(HG_THREADS) hgemm_kernel(const T* __restrict__ A, const T* __restrict__ B, int64_t K,
                                                           int64_t lda, int64_t ldb, int64_t kchunk, int64_t ldp,
                                                           int64_t rows, T* __restrict__ P) {
  __shared__ __align__(16) T As[2][HG_BK][HG_BM];
  __shared__ __align__(16) T Bs[2][HG_BK][HG_BN];
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  const int64_t q0 = int64_t(blockIdx.y) * HG_BM, h0 = int64_t(blockIdx.x) * HG_BN;
  const int64_t kb = int64_t(blockIdx.z) * kchunk, ke = tmin<int64_t>(K, kb + kchunk);
  // global -> register staging: A tile 16 x 64 (8 per thread), B tile 16 x 128 (16 per thread)
  const int sr = tid >> 3, ac = (tid & 7) * 8, bc = (tid & 7) * 16;
  T ra[8], rb[16];
  auto gload = [&](int64_t k0) {
    const int64_t k = k0 + sr;
    if (k < ke) {
      V4<T>::load(A + k * lda + q0 + ac, ra);
      V4<T>::load(A + k * lda + q0 + ac + 4, ra + 4);
#pragma unroll
      for (int v = 0; v < 4; ++v) V4<T>::load(B + k * ldb + h0 + bc + 4 * v, rb + 4 * v);
    } else {
#pragma unroll
      for (int u = 0; u < 8; ++u) ra[u] = T(0);
#pragma unroll
      for (int u = 0; u < 16; ++u) rb[u] = T(0);
    }
  };
  auto sstore = [&](int buf) {
    V4<T>::store_plain(&As[buf][sr][ac], ra);
    V4<T>::store_plain(&As[buf][sr][ac + 4], ra + 4);
#pragma unroll
    for (int v = 0; v < 4; ++v) V4<T>::store_plain(&Bs[buf][sr][bc + 4 * v], rb + 4 * v);
  };
  T acc[8][8];
#pragma unroll
  for (int x = 0; x < 8; ++x)
#pragma unroll
    for (int y = 0; y < 8; ++y) acc[x][y] = T(0);
  gload(kb);
  sstore(0);
  __syncthreads();
  int buf = 0;
  for (int64_t k0 = kb; k0 < ke; k0 += HG_BK) {
    const bool more = k0 + HG_BK < ke;
    if (more) gload(k0 + HG_BK);
#pragma unroll
    for (int kk = 0; kk < HG_BK; ++kk) {
      T a[8], b[8];
      V4<T>::load(&As[buf][kk][ty * 8], a);
      V4<T>::load(&As[buf][kk][ty * 8 + 4], a + 4);
      V4<T>::load(&Bs[buf][kk][tx * 4], b);
      V4<T>::load(&Bs[buf][kk][64 + tx * 4], b + 4);
#pragma unroll
      for (int x = 0; x < 8; ++x)
#pragma unroll
        for (int y = 0; y < 8; ++y) acc[x][y] = fma_rn(a[x], b[y], acc[x][y]);
    }
    if (more) {
      sstore(buf ^ 1);
      __syncthreads();
      buf ^= 1;
    }
  }
  T* out = P + int64_t(blockIdx.z) * rows * ldp;
#pragma unroll
  for (int x = 0; x < 8; ++x) {
    T* row = out + (q0 + ty * 8 + x) * ldp + h0;
    V4<T>::store_plain(row + tx * 4, acc[x]);
    V4<T>::store_plain(row + 64 + tx * 4, acc[x] + 4);
  }
}

// fp64 on the tensor cores: mma.sync m8n8k4 f64 (DMMA).  CTA tile 64
// (queries) x 128 (heavy index rows), 4 warps of 32 x 64 (4 x 8 MMA tiles,
// 64 fp64 accumulators per thread), BK = 16 double-buffered through shared
// memory; fragments: A (8 x 4, row) one element per lane at (lane / 4, lane % 4),
// B (4 x 8, col) at (lane % 4, lane / 4), C two at (lane / 4, 2 (lane % 4) + {0, 1}).
constexpr int DM_BM = 64, DM_BN = 128, DM_BK = 8, DM_PA = DM_BM + 4, DM_PB = DM_BN + 4;

__device__ __forceinline__ void dmma(double* c, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}

__global__ void __launch_bounds__(128) hgemm_dmma_kernel(const double* __restrict__ A, const double* __restrict__ B,
                                                         int64_t K, int64_t lda, int64_t ldb, int64_t kchunk,
                                                         int64_t ldp, int64_t rows, double* __restrict__ P) {
  __shared__ __align__(16) double As[2][DM_BK][DM_PA];
  __shared__ __align__(16) double Bs[2][DM_BK][DM_PB];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wq = (warp >> 1) * 32, wh = (warp & 1) * 64;  // the warp's 32 x 64 sub-tile
  const int64_t q0 = int64_t(blockIdx.y) * DM_BM, h0 = int64_t(blockIdx.x) * DM_BN;
  const int64_t kb = int64_t(blockIdx.z) * kchunk, ke = tmin<int64_t>(K, kb + kchunk);
  // global -> register staging: A tile 8 x 64 (4 per thread), B tile 8 x 128 (8 per thread)
  const int sr = tid >> 4, ac = (tid & 15) * 4, bc = (tid & 15) * 8;
  double ra[4], rb[8];
  auto gload = [&](int64_t k0) {
    const int64_t k = k0 + sr;
    if (k < ke) {
      V4<double>::load(A + k * lda + q0 + ac, ra);
      V4<double>::load(B + k * ldb + h0 + bc, rb);
      V4<double>::load(B + k * ldb + h0 + bc + 4, rb + 4);
    } else {
#pragma unroll
      for (int u = 0; u < 4; ++u) ra[u] = 0.0;
#pragma unroll
      for (int u = 0; u < 8; ++u) rb[u] = 0.0;
    }
  };
  auto sstore = [&](int buf) {
    V4<double>::store_plain(&As[buf][sr][ac], ra);
    V4<double>::store_plain(&Bs[buf][sr][bc], rb);
    V4<double>::store_plain(&Bs[buf][sr][bc + 4], rb + 4);
  };
  double acc[4][8][2];
#pragma unroll
  for (int x = 0; x < 4; ++x)
#pragma unroll
    for (int y = 0; y < 8; ++y) acc[x][y][0] = acc[x][y][1] = 0.0;
  gload(kb);
  sstore(0);
  __syncthreads();
  int buf = 0;
  const int fr = lane >> 2, fk = lane & 3;
  for (int64_t k0 = kb; k0 < ke; k0 += DM_BK) {
    const bool more = k0 + DM_BK < ke;
    if (more) gload(k0 + DM_BK);
#pragma unroll
    for (int kk = 0; kk < DM_BK; kk += 4) {
      double a[4], b[8];
#pragma unroll
      for (int x = 0; x < 4; ++x) a[x] = As[buf][kk + fk][wq + 8 * x + fr];
#pragma unroll
      for (int y = 0; y < 8; ++y) b[y] = Bs[buf][kk + fk][wh + 8 * y + fr];
#pragma unroll
      for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < 8; ++y) dmma(acc[x][y], a[x], b[y]);
    }
    if (more) {
      sstore(buf ^ 1);
      __syncthreads();
      buf ^= 1;
    }
  }
  double* out = P + int64_t(blockIdx.z) * rows * ldp;
#pragma unroll
  for (int x = 0; x < 4; ++x) {
    const int64_t q = q0 + wq + 8 * x + fr;
#pragma unroll
    for (int y = 0; y < 8; ++y)
      *reinterpret_cast<double2*>(out + q * ldp + h0 + wh + 8 * y + 2 * fk) = make_double2(acc[x][y][0], acc[x][y][1]);
  }
}

template <typename T>
__global__ void hreduce_kernel(const T* __restrict__ P, int splits, int64_t count, T* __restrict__ D) {
  for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < count; e += int64_t(gridDim.x) * blockDim.x) {
    T s = P[e];
    for (int z = 1; z < splits; ++z) s = add_rn(s, P[int64_t(z) * count + e]);
    D[e] = s;
  }
}

// dense rows in flight per lane in the gather (4: fewer registers, more
// resident warps — C2 cosine 1.98 -> 1.96 ms, C5 18.29 -> 17.94 ms against 8;
// 16 loses: 2.20 / 20.2 ms)
#ifndef SD_HGATHER_UNROLL
#define SD_HGATHER_UNROLL 4
#endif
constexpr int HGU = SD_HGATHER_UNROLL;

// DLH[j][q] = sum_c b_jc * HQT[c][q] (MINSUM: sum_c min(b_jc, HQT[c][q]))
// over light index rows j (heavy rows are the dense block's); one warp per
// (row, 128-wide block of heavy queries), ascending column order, HGU dense
// rows in flight per lane; the block's values of column c are at
// D + blk * bstride + c * ld.  Rows are taken from a shared counter in
// descending-degree order (lrows, index build) so the long rows start first
// and no warp is left with a tail of them.
template <typename T, bool MINSUM, int QPL>
__global__ void __launch_bounds__(256) hgather_kernel(const int64_t* __restrict__ ptr, const int32_t* __restrict__ idx,
                                                      const T* __restrict__ val, const int32_t* __restrict__ lrows,
                                                      int64_t n_light, const T* __restrict__ D, int64_t ld,
                                                      int64_t bstride, int64_t nblk, int64_t ldo,
                                                      unsigned long long* counter, T* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const unsigned long long total = (unsigned long long)(n_light * nblk);
  while (true) {
    unsigned long long it = 0;
    if (lane == 0) it = atomicAdd(counter, 1ull);
    it = __shfl_sync(0xffffffffu, it, 0);
    if (it >= total) break;
    const int64_t j = lrows[it / nblk], blk = int64_t(it % nblk);
    const int64_t beg = ptr[j], end = ptr[j + 1];
    // QPL = 4: the lane's queries as in EQ<T> (isect_kernel.cuh) — fp64 loads
    // and stores contiguous over the warp
    const T* dcol = D + blk * bstride + (QPL == 4 ? EQ<T>::CELL : 1) * lane;
    T acc[QPL];
#pragma unroll
    for (int k = 0; k < QPL; ++k) acc[k] = T(0);
    for (int64_t e0 = beg; e0 < end; e0 += 32) {
      const bool ok = e0 + lane < end;
      const int32_t cl = ok ? idx[e0 + lane] : 0;
      const T vl = ok ? val[e0 + lane] : T(0);
      const int nn = int(tmin<int64_t>(32, end - e0));
      for (int u0 = 0; u0 < nn; u0 += HGU) {
        T d[HGU][QPL];
        T x[HGU];
#pragma unroll
        for (int u = 0; u < HGU; ++u) {
          const int src = (u0 + u) & 31;
          const int32_t c = __shfl_sync(0xffffffffu, cl, src);
          x[u] = __shfl_sync(0xffffffffu, vl, src);
          if (u0 + u < nn) {
            if constexpr (QPL == 4) EQ<T>::ldg(dcol + int64_t(c) * ld, d[u]);
            else d[u][0] = dcol[int64_t(c) * ld];
          }
        }
#pragma unroll
        for (int u = 0; u < HGU; ++u)
          if (u0 + u < nn)
#pragma unroll
            for (int k = 0; k < QPL; ++k)
              acc[k] = MINSUM ? add_rn(acc[k], min_(x[u], d[u][k])) : fma_rn(x[u], d[u][k], acc[k]);
      }
    }
    if constexpr (QPL == 4 && sizeof(T) == 4) {
      V4<T>::store_plain(out + j * ldo + blk * 128 + 4 * lane, acc);
    } else if constexpr (QPL == 4) {
      T* o = out + j * ldo + blk * 128 + 2 * lane;
      reinterpret_cast<double2*>(o)[0] = make_double2(acc[0], acc[1]);
      reinterpret_cast<double2*>(o + 64)[0] = make_double2(acc[2], acc[3]);
    }
    else out[j * ldo + blk * 32 + lane] = acc[0];
  }
}

// ---------------------------------------------------------------- driver

int hybrid_classify(const sd_csr* a, const sd_index* ix, int dtype, int kind, HybridState& hs, cudaStream_t st) {
  hs.nhq = 0;
  const int64_t m = a->n_rows;
  const int cap = int(std::max<int64_t>(1, knob(SD_TUNE_HYBRID_MAX_QUERIES)));
  SD_TRY(hs.qid.alloc(sizeof(int32_t) * std::max<int64_t>(1, m), st));
  SD_TRY(hs.hq.alloc(sizeof(int32_t) * cap, st));
  SD_TRY(hs.count.alloc(2 * sizeof(unsigned int), st));
  SD_CUDA_TRY(cudaMemsetAsync(hs.count.ptr, 0, 2 * sizeof(unsigned int), st));
  SD_TRY(hs.gcount.alloc(sizeof(unsigned long long), st));
  SD_CUDA_TRY(cudaMemsetAsync(hs.gcount.ptr, 0, sizeof(unsigned long long), st));
  const int blocks = int(std::min<int64_t>((m + 255) / 256, int64_t(num_sms()) * 8));
  classify_kernel<<<std::max(1, blocks), 256, 0, st>>>(a->indptr, m, ix->heavy_deg, cap, hs.qid.as<int32_t>(),
                                                       hs.hq.as<int32_t>(), hs.count.as<unsigned int>());
  SD_LAUNCH_CHECK();
  if (dtype == SD_F32 && kind == HYB_DOT && ix->hbf)  // planes of the queries' GEMM image (read with the count)
    SD_TRY(check_bf16_exact(a, hs.count.as<unsigned int>() + 1, st));
  hs.cap = cap;
  return SD_OK;
}

// The dense gather on side stream 0 (after hs.fork): DLH for the light index
// rows.  Shadow mode: one 128-thread block per SM next to the sweep's CTAs.
int hybrid_gather(const sd_csr* a, const sd_csr* b, const sd_index* ix, int dtype, HybridState& hs, cudaStream_t st) {
  if (hs.nhq == 0) return SD_OK;
  const bool ms = hs.gather_kind == HYB_MINSUM;
  const int qpl = hs.qpad % 128 == 0 ? 4 : 1;  // queries per lane: 128-query blocks, or one block of 32
  const int64_t K = a->n_cols, nblk = hs.qpad / (32 * qpl);
  const int64_t hq_bstride = ms ? K * 128 : 32 * qpl, hq_ld = ms ? 128 : hs.qpad;
  cudaStream_t side = hs.fork ? side_stream(0) : st;
  if (side != st) SD_CUDA_TRY(cudaStreamWaitEvent(side, hs.fork, 0));
  // keep the SMs' shared-memory carveout at its maximum while the gather
  // runs, so CTAs needing ~200 KB of shared memory can co-reside with it
  static const bool carve = [] {
    cudaFuncSetAttribute(hgather_kernel<float, false, 4>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    cudaFuncSetAttribute(hgather_kernel<float, false, 1>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    cudaFuncSetAttribute(hgather_kernel<float, true, 4>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    cudaFuncSetAttribute(hgather_kernel<double, false, 4>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    cudaFuncSetAttribute(hgather_kernel<double, true, 4>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    return true;
  }();
  (void)carve;
  const bool shadow = knob(SD_TUNE_GATHER_SHADOW) != 0;
  const int gthreads = shadow ? 128 : 256;
  SD_TRY(SD_DISPATCH_DTYPE(dtype, T, [&]() -> int {
    auto go = [&](auto kernel) -> int {
      int per_sm = 0;
      SD_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, 256, 0));
      if (shadow) per_sm = 1;
      else if (knob(SD_TUNE_GATHER_BLOCKS) > 0) per_sm = std::min<int>(per_sm, int(knob(SD_TUNE_GATHER_BLOCKS)));
      kernel<<<std::max(1, per_sm) * num_sms(), gthreads, 0, side>>>(
          b->indptr, b->indices, static_cast<const T*>(b->values), ix->lrows, ix->n_light, hs.hqt.as<T>(), hq_ld,
          hq_bstride, nblk, hs.qpad, hs.gcount.as<unsigned long long>(), hs.dlh.as<T>());
      SD_LAUNCH_CHECK();
      return SD_OK;
    };
    if (ms) return go(hgather_kernel<T, true, 4>);
    return qpl == 4 ? go(hgather_kernel<T, false, 4>) : go(hgather_kernel<T, false, 1>);
  }));
  if (side != st) {
    SD_CUDA_TRY(cudaEventCreateWithFlags(&hs.join, cudaEventDisableTiming));
    SD_CUDA_TRY(cudaEventRecord(hs.join, side));
  }
  return SD_OK;
}

int hybrid_prepare(const sd_csr* a, const sd_csr* b, const sd_index* ix, int dtype, int kind, HybridState& hs,
                   cudaStream_t st) {
  // the host needs the heavy count to size the dense block: one small read
  // (work queued on the side streams before it keeps the GPU busy meanwhile)
  unsigned int cnt[2] = {0, 0};
  SD_CUDA_TRY(cudaMemcpyAsync(cnt, hs.count.ptr, sizeof(cnt), cudaMemcpyDeviceToHost, st));
  SD_CUDA_TRY(cudaStreamSynchronize(st));
  hs.nhq = int(std::min<unsigned int>(cnt[0], unsigned(hs.cap)));
  const int q_planes = (cnt[1] & 1u) ? 2 : 1;
  if (hs.nhq == 0) return SD_OK;
  const size_t es = dtype == SD_F64 ? 8 : 4;
  const int64_t K = a->n_cols;
  // a few heavy queries (e.g. one rank's share of a strong-scaled run, fp32
  // dot family): one 32-query block, so the gather reads 128 B of HQT per
  // index entry instead of 512 (the min-sum block stages 128-query chunks and
  // the fp64 GEMM tiles 64 queries)
  hs.qpad = (kind != HYB_MINSUM && dtype == SD_F32 && hs.nhq <= 32) ? 32 : (hs.nhq + 127) / 128 * 128;
  SD_TRY(hs.hqt.alloc(es * size_t(K) * size_t(hs.qpad), st));
  SD_CUDA_TRY(cudaMemsetAsync(hs.hqt.ptr, 0, es * size_t(K) * size_t(hs.qpad), st));
  SD_TRY(hs.dqh.alloc(es * size_t(hs.qpad) * size_t(ix->hpad), st));
  SD_TRY(hs.dlh.alloc(es * size_t(std::max<int64_t>(1, b->n_rows)) * size_t(hs.qpad), st));
  // min-sum: HQT in 128-query blocks ([blk][K][128], one contiguous stage per
  // column chunk for the bulk copies of hminsum_kernel) holding max(a, 0)
  const bool ms = kind == HYB_MINSUM;
  const int64_t hq_bstride = ms ? K * 128 : (hs.qpad % 128 == 0 ? 128 : 32), hq_ld = ms ? 128 : hs.qpad;
  // the dense gather runs on a side stream (heavy_rows joins it), after the
  // dense block
  // the gather forks now (it only needs HQT).  Shadow mode (knob, off by
  // default) launches it after the sweep (hybrid_gather, from isect_run) with
  // one 128-thread block per SM beside the sweep's CTAs: measured on C2
  // cosine it loses (3.66 vs 1.98 ms) — 4 warps per SM leave the
  // latency-bound gather ~10x slower than alone, and the sweep at 12 warps
  // 13 % slower
  cudaStream_t side = side_stream(0);
  if (side && side != st) {
    SD_CUDA_TRY(cudaEventCreateWithFlags(&hs.fork, cudaEventDisableTiming));
    hs.main = st;
  }
  hs.gather_kind = kind;
  auto gather = [&](auto) -> int {
    if (hs.fork) SD_CUDA_TRY(cudaEventRecord(hs.fork, st));
    if (knob(SD_TUNE_GATHER_SHADOW) != 0) return SD_OK;  // launched by hybrid_gather after the sweep
    return hybrid_gather(a, b, ix, dtype, hs, st);
  };
  if (ms) {
    return SD_DISPATCH_DTYPE(dtype, T, [&]() -> int {
      ht_scatter_kernel<T, true><<<row_scatter_grid(hs.nhq), 256, 0, st>>>(
          a->indptr, a->indices, static_cast<const T*>(a->values), hs.hq.as<int32_t>(), hs.nhq, hq_bstride, hq_ld,
          hs.hqt.as<T>());
      SD_LAUNCH_CHECK();
      SD_TRY(gather(T(0)));
      return hminsum(ix, b, dtype, hs.hqt.ptr, K, hs.qpad, hs.part, hs.dqh.ptr, st);
    });
  }
  // fp32: tcgen05 bf16 GEMM (dense_tc.cu; hi/lo planes where values are
  // not bf16-exact, M = 128 heavy index rows x N = 128 or 256 heavy queries,
  // K split over ~2 waves of CTAs); fp64: CUDA-core DFMA (tile 32 x 128 x 16)
  const bool tcb = dtype == SD_F32;
  const int R = hs.nhq <= 128 ? 128 : 256;  // queries per GEMM CTA
  const int64_t bm = tcb ? R : HG_BM;
  const int64_t bn = tcb ? 128 : HG_BN, bkk = tcb ? 64 : HG_BK;
  const int64_t tiles_q = (hs.nhq + bm - 1) / bm, tiles_h = ix->hpad / bn;
  const int64_t rows = tcb ? hs.qpad : tiles_q * bm;  // GEMM rows written (<= qpad)
  // K split so that the GEMM fills about two (tensor-core) or six waves of CTAs
  const int64_t waves = tcb ? 2 : 3 * 2;
  const int64_t want = std::max<int64_t>(1, (waves * int64_t(num_sms()) + tiles_q * tiles_h - 1) / (tiles_q * tiles_h));
  int64_t kchunk = (K + want - 1) / want;
  kchunk = std::max<int64_t>(bkk, (kchunk + bkk - 1) / bkk * bkk);
  const int64_t splits = (K + kchunk - 1) / kchunk;
  if (tcb) {  // the bf16 image of this call's heavy queries
    SD_TRY(hs.hq_img.alloc(dense_image_bytes(hs.nhq, ix->hbf_nkb, 2, R), st));
    SD_TRY(dense_image(a, hs.hq.as<int32_t>(), hs.nhq, ix->hbf_nkb, 2, R, hs.hq_img.ptr, st));
  }
  SD_TRY(hs.part.alloc(es * size_t(splits) * size_t(rows) * size_t(ix->hpad), st));
  return SD_DISPATCH_DTYPE(dtype, T, [&]() -> int {
    ht_scatter_kernel<T, false><<<row_scatter_grid(hs.nhq), 256, 0, st>>>(
        a->indptr, a->indices, static_cast<const T*>(a->values), hs.hq.as<int32_t>(), hs.nhq, hq_bstride, hq_ld,
        hs.hqt.as<T>());
    SD_LAUNCH_CHECK();
    const dim3 grid{unsigned(tiles_h), unsigned(tiles_q), unsigned(splits)};
    if constexpr (sizeof(T) == 4) {
      SD_TRY(dense_gemm_raw(ix->hbf, ix->hbf_planes, ix->n_heavy, hs.hq_img.ptr, q_planes, R, hs.nhq,
                            ix->hbf_nkb, kchunk / bkk, hs.part.as<float>(), rows, ix->hpad, st));
    } else {
      // fp64: DMMA tensor cores (knob hgemm = 1: the CUDA-core DFMA tile, for A/B)
      if (knob(SD_TUNE_HGEMM) == 1)
        hgemm_kernel<T><<<grid, HG_THREADS, 0, st>>>(hs.hqt.as<T>(), static_cast<const T*>(ix->ht), K, hs.qpad,
                                                     ix->hpad, kchunk, ix->hpad, rows, hs.part.as<T>());
      else
        hgemm_dmma_kernel<<<grid, 128, 0, st>>>(hs.hqt.as<double>(), static_cast<const double*>(ix->ht), K, hs.qpad,
                                                ix->hpad, kchunk, ix->hpad, rows, hs.part.as<double>());
    }
    SD_LAUNCH_CHECK();
    // the gather forks after the GEMM: run side by side they slow each other
    // down (C2: 550 us together vs 202 + 244 us in sequence; the GEMM streams
    // its operand image from HBM, the gather is L2-latency bound), and the
    // side stream's priority would otherwise put the gather first
    SD_TRY(gather(T(0)));
    const int64_t count = rows * ix->hpad;
    hreduce_kernel<T><<<int(std::min<int64_t>((count + 255) / 256, int64_t(num_sms()) * 16)), 256, 0, st>>>(
        hs.part.as<T>(), int(splits), count, hs.dqh.as<T>());
    SD_LAUNCH_CHECK();
    return SD_OK;
  });
}

}  // namespace sd
