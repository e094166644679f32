// hminsum.cu — the hybrid path's dense block for manhattan (hybrid.cu).
//
// Manhattan's union decomposition adds, per intersecting column, the
// contribution |a - b| - |a| - |b| (metric.cuh contrib<C_ABS>).  When no index
// value is negative (checked once per index) that is exactly
// -2 min(max(a, 0), b) for every query value a, and 0 wherever either side is
// absent — so heavy query rows can be summed densely like the dot family:
//
//   heavy queries x heavy index rows   hminsum_kernel  dqh[q][h] = sum_c min(HQT+[c][q], B[h][c])
//   heavy queries x light index rows   hgather_kernel<T, MINSUM> (hybrid.cu)
//
// and heavy_rows_kernel finishes d = S_A + S_B - 2 * sum.  There is no
// tensor-core form of a min-sum, so the heavy block is sparse over the index
// rows (their CSR entries, ~17 % of the dense block on C2) and dense over the
// queries:
//
//   * the columns are cut into chunks of CW (128 fp32 / 64 fp64); the queries'
//     values of a chunk, HQT+[c0:c0+CW][128 queries], are one contiguous 64 KB
//     block (HQT is stored in 128-query blocks) moved into shared memory by a
//     single bulk copy (TMA engine) on an mbarrier, three stages in flight;
//   * a CTA owns 64 heavy index rows (16 warps x 4, interleaved over the
//     degree-ordered heavy ids so the warps carry similar work) and a group of
//     consecutive chunks; for each chunk a warp walks its rows' entries of
//     that chunk (per-(row, chunk) CSR offsets, hchunk, built once per index):
//     32 entries per coalesced load, each broadcast by shuffle, the lane's 4
//     query values read with one 16-byte shared load, 4 min-adds per lane
//     into register accumulators;
//   * partial sums per chunk group are written [group][h][q] and summed in
//     group order by msreduce_kernel (deterministic, no atomics).
//
// Bound: shared-memory bandwidth — 128 values x sizeof(T) per CSR entry of the
// heavy rows (C2: 20.8 M entries x 512 B = 10.6 GB at ~128 B/clk/SM).
#include <algorithm>
#include "common.cuh"
#include "hybrid.cuh"
#include "index.cuh"
#include "isect_kernel.cuh"
#include "tma.cuh"

namespace sd {

namespace {

constexpr int MS_STAGE_BYTES = 65536;
constexpr int MS_STAGES = 3;
constexpr int MS_WARPS = 16;
constexpr int MS_RPW = 4;                  // heavy rows per warp
constexpr int MS_HB = MS_WARPS * MS_RPW;   // heavy rows per CTA

template <typename T>
constexpr int ms_cw() { return MS_STAGE_BYTES / (128 * int(sizeof(T))); }

// hchunk[h * (nch + 1) + k] = first entry of heavy row h with column >= k * cw
// (k = nch: the row's end); B's rows are sorted by column (canonical CSR)
__global__ void hchunk_kernel(const int64_t* __restrict__ ptr, const int32_t* __restrict__ idx,
                              const int32_t* __restrict__ hrows, int64_t nh, int64_t nch, int64_t cw,
                              int64_t* __restrict__ hchunk) {
  const int64_t total = nh * (nch + 1);
  for (int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < total; t += int64_t(gridDim.x) * blockDim.x) {
    const int64_t h = t / (nch + 1), k = t - h * (nch + 1);
    const int64_t r = hrows[h];
    int64_t lo = ptr[r], hi = ptr[r + 1];
    const int64_t c = k * cw;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (int64_t(idx[mid]) < c) lo = mid + 1; else hi = mid;
    }
    hchunk[t] = lo;
  }
}

// flag = 1 if some value is negative or NaN
template <typename T>
__global__ void not_nonneg_kernel(const T* __restrict__ v, int64_t n, unsigned int* flag) {
  bool bad = false;
  for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < n; e += int64_t(gridDim.x) * blockDim.x)
    bad |= !(v[e] >= T(0));
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1u);
}

// grid (ceil(nh / 64), groups, qpad / 128); 512 threads; dynamic shared
// memory MS_STAGES x 64 KB.  D = HQT+ in 128-query blocks: block qb's column
// c values at D + (qb * n_cols + c) * 128.
template <typename T>
__global__ void __launch_bounds__(MS_WARPS * 32, 1) hminsum_kernel(
    const int64_t* __restrict__ hchunk, int64_t nch, const int32_t* __restrict__ hperm, int64_t nh,
    const int32_t* __restrict__ bidx, const T* __restrict__ bval, const T* __restrict__ D, int64_t n_cols,
    int64_t G, int64_t hpad, int64_t qpad, T* __restrict__ part) {
  constexpr int CW = ms_cw<T>();
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) unsigned long long full[MS_STAGES];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t g = blockIdx.y, qb = blockIdx.z;
  const int64_t k0 = g * G, k1 = tmin<int64_t>(nch, k0 + G);
  const T* Dq = D + qb * n_cols * 128;
  const uint32_t sbase = uint32_t(__cvta_generic_to_shared(smem));
  const uint32_t fb = uint32_t(__cvta_generic_to_shared(&full[0]));
  if (threadIdx.x == 0) {
    for (int s = 0; s < MS_STAGES; ++s) mbar_init(fb + 8 * s, 1);
    mbar_fence_init();
  }
  __syncthreads();
  auto issue = [&](int64_t k) {
    const int s = int((k - k0) % MS_STAGES);
    const int64_t c0 = k * CW;
    const uint32_t bytes = uint32_t(tmin<int64_t>(CW, n_cols - c0)) * 128u * uint32_t(sizeof(T));
    mbar_expect_tx(fb + 8 * s, bytes);
    bulk_g2s(sbase + uint32_t(s) * MS_STAGE_BYTES, Dq + c0 * 128, bytes, fb + 8 * s);
  };
  if (threadIdx.x == 0)
    for (int64_t k = k0; k < tmin<int64_t>(k1, k0 + MS_STAGES); ++k) issue(k);
  int32_t hs[MS_RPW];
#pragma unroll
  for (int u = 0; u < MS_RPW; ++u) {
    const int64_t p = int64_t(blockIdx.x) * MS_HB + u * MS_WARPS + warp;
    hs[u] = p < nh ? hperm[p] : -1;
  }
  T acc[MS_RPW][4];
#pragma unroll
  for (int u = 0; u < MS_RPW; ++u)
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[u][q] = T(0);
  for (int64_t k = k0; k < k1; ++k) {
    const int s = int((k - k0) % MS_STAGES);
    mbar_wait(fb + 8 * s, uint32_t(((k - k0) / MS_STAGES) & 1));
    const uint32_t sq = sbase + uint32_t(s) * MS_STAGE_BYTES + uint32_t(lane) * 4u * uint32_t(sizeof(T));
    const int32_t c0 = int32_t(k * CW);
#pragma unroll
    for (int u = 0; u < MS_RPW; ++u) {
      if (hs[u] < 0) continue;  // warp-uniform
      const int64_t* hc = hchunk + int64_t(hs[u]) * (nch + 1) + k;
      const int64_t beg = hc[0], end = hc[1];
      for (int64_t e0 = beg; e0 < end; e0 += 32) {
        const bool ok = e0 + lane < end;
        const int32_t cl = ok ? bidx[e0 + lane] - c0 : 0;
        const T vl = ok ? bval[e0 + lane] : T(0);
        const int nn = int(tmin<int64_t>(32, end - e0));
        int t = 0;
        for (; t + 4 <= nn; t += 4) {
          T d[4][4], x[4];
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            const int32_t c = __shfl_sync(0xffffffffu, cl, t + v);
            x[v] = __shfl_sync(0xffffffffu, vl, t + v);
            lds4(sq + uint32_t(c) * 128u * uint32_t(sizeof(T)), d[v]);
          }
#pragma unroll
          for (int v = 0; v < 4; ++v)
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[u][q] = add_rn(acc[u][q], min_(x[v], d[v][q]));
        }
        for (; t < nn; ++t) {
          T d[4];
          const int32_t c = __shfl_sync(0xffffffffu, cl, t);
          const T x = __shfl_sync(0xffffffffu, vl, t);
          lds4(sq + uint32_t(c) * 128u * uint32_t(sizeof(T)), d);
#pragma unroll
          for (int q = 0; q < 4; ++q) acc[u][q] = add_rn(acc[u][q], min_(x, d[q]));
        }
      }
    }
    __syncthreads();  // every warp is done with stage s
    if (threadIdx.x == 0 && k + MS_STAGES < k1) issue(k + MS_STAGES);
  }
  T* out = part + g * hpad * qpad + qb * 128 + 4 * lane;
#pragma unroll
  for (int u = 0; u < MS_RPW; ++u)
    if (hs[u] >= 0) V4<T>::store_plain(out + int64_t(hs[u]) * qpad, acc[u]);
}

// dqh[q][h] = sum over groups (in order) of part[g][h][q]
template <typename T>
__global__ void msreduce_kernel(const T* __restrict__ part, int64_t groups, int64_t nh, int64_t hpad, int64_t qpad,
                                T* __restrict__ dqh) {
  const int64_t count = nh * qpad;
  for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < count; e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t h = e / qpad, q = e - h * qpad;
    T s = part[e];
    for (int64_t g = 1; g < groups; ++g) s = add_rn(s, part[g * hpad * qpad + e]);
    dqh[q * hpad + h] = s;
  }
}

}  // namespace

int64_t minsum_chunk_cols(int dtype) { return dtype == SD_F64 ? ms_cw<double>() : ms_cw<float>(); }

int minsum_check_index(const sd_csr* b, int dtype, unsigned int* flag, cudaStream_t st) {
  if (b->nnz == 0) return SD_OK;
  return SD_DISPATCH_DTYPE(dtype, T, [&]() -> int {
    const int blocks = int(tmin<int64_t>((b->nnz + 255) / 256, int64_t(num_sms()) * 8));
    not_nonneg_kernel<T><<<blocks, 256, 0, st>>>(static_cast<const T*>(b->values), b->nnz, flag);
    SD_LAUNCH_CHECK();
    return SD_OK;
  });
}

int minsum_chunks(const sd_csr* b, int dtype, const int32_t* hrows, int64_t nh, int64_t nch, int64_t* hchunk,
                  cudaStream_t st) {
  const int64_t total = nh * (nch + 1);
  const int blocks = int(tmin<int64_t>((total + 255) / 256, int64_t(num_sms()) * 16));
  hchunk_kernel<<<std::max(1, blocks), 256, 0, st>>>(b->indptr, b->indices, hrows, nh, nch, minsum_chunk_cols(dtype),
                                                     hchunk);
  SD_LAUNCH_CHECK();
  return SD_OK;
}

int hminsum(const sd_index* ix, const sd_csr* b, int dtype, const void* hqt, int64_t n_cols, int64_t qpad,
            Scratch& part, void* dqh, cudaStream_t st) {
  const int64_t nh = ix->n_heavy, nch = ix->ms_nch;
  const int64_t hblocks = (nh + MS_HB - 1) / MS_HB, qblocks = qpad / 128;
  // chunk groups: about 4 waves of one-CTA-per-SM blocks (fewer partials than
  // one group per chunk, enough CTAs to balance)
  const int64_t want = std::max<int64_t>(1, (4 * int64_t(num_sms()) + hblocks * qblocks - 1) / (hblocks * qblocks));
  const int64_t G = std::max<int64_t>(MS_STAGES, (nch + want - 1) / want);
  const int64_t groups = (nch + G - 1) / G;
  const size_t es = dtype == SD_F64 ? 8 : 4;
  SD_TRY(part.alloc(es * size_t(groups) * size_t(ix->hpad) * size_t(qpad), st));
  const size_t smem = size_t(MS_STAGES) * MS_STAGE_BYTES;
  return SD_DISPATCH_DTYPE(dtype, T, [&]() -> int {
    SD_TRY(prepare_smem(hminsum_kernel<T>, smem, "hminsum_kernel"));
    const dim3 grid{unsigned(hblocks), unsigned(groups), unsigned(qblocks)};
    hminsum_kernel<T><<<grid, MS_WARPS * 32, smem, st>>>(ix->hchunk, nch, ix->hperm, nh, b->indices,
                                                         static_cast<const T*>(b->values), static_cast<const T*>(hqt),
                                                         n_cols, G, ix->hpad, qpad, part.as<T>());
    SD_LAUNCH_CHECK();
    const int64_t count = nh * qpad;
    msreduce_kernel<T><<<int(std::min<int64_t>((count + 255) / 256, int64_t(num_sms()) * 16)), 256, 0, st>>>(
        part.as<T>(), groups, nh, ix->hpad, qpad, static_cast<T*>(dqh));
    SD_LAUNCH_CHECK();
    return SD_OK;
  });
}

}  // namespace sd
