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
//   * a CTA owns 60 heavy index rows (20 warps x 3, a stratified sample of
//     the degree-ordered heavy ids so CTAs and warps carry similar work) and a
//     group of consecutive chunks (their per-(row, chunk) CSR offsets, hchunk,
//     built once per index, staged in shared memory); for each chunk a warp
//     walks its rows' entries of that chunk: 32 entries per coalesced load
//     (prefetched one chunk ahead), each broadcast by shuffle, the lane's 4
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
template <typename T>
constexpr int ms_stages() { return sizeof(T) == 4 ? 3 : 2; }  // fp64: its staging area needs the room
#ifndef SD_MS_WARPS
#define SD_MS_WARPS 20
#endif
#ifndef SD_MS_RPW
#define SD_MS_RPW 3
#endif
#ifndef SD_MS_UNROLL
#define SD_MS_UNROLL 8
#endif
// 20 consumer warps x 3 rows: the block is latency-bound on its shared loads,
// so more warps beat more rows per warp (C2 fp32 583 -> 527 us; measured
// 16 x 4, 20 x 3, 22 x 3, 31 x 2: 583 / 527 / 544 / 553 us)
constexpr int MS_WARPS = SD_MS_WARPS;      // consumer warps (plus one producer warp)
constexpr int MS_RPW = SD_MS_RPW;          // heavy rows per warp
constexpr int MS_HB = MS_WARPS * MS_RPW;   // heavy rows per CTA
constexpr int MS_UNROLL = SD_MS_UNROLL;    // staged entries per step (rows padded to a multiple)
constexpr int MS_MAX_G = 32;               // chunks per CTA (their pointers: MS_HB x 33 x 8 B of shared memory)

template <typename T>
constexpr int ms_cw() { return MS_STAGE_BYTES / (128 * int(sizeof(T))); }

// acc[q] += min(x, d[q]), q < 4 — fp32 with two packed f32x2 adds (FADD2:
// each element rounded like add.rn.f32), fp64 scalar
__device__ __forceinline__ void minadd4(float* acc, float x, const float* d) {
  const float m0 = fminf(x, d[0]), m1 = fminf(x, d[1]), m2 = fminf(x, d[2]), m3 = fminf(x, d[3]);
  uint64_t a01, a23, b01, b23;
  asm("mov.b64 %0, {%1, %2};" : "=l"(a01) : "f"(acc[0]), "f"(acc[1]));
  asm("mov.b64 %0, {%1, %2};" : "=l"(a23) : "f"(acc[2]), "f"(acc[3]));
  asm("mov.b64 %0, {%1, %2};" : "=l"(b01) : "f"(m0), "f"(m1));
  asm("mov.b64 %0, {%1, %2};" : "=l"(b23) : "f"(m2), "f"(m3));
  asm("add.rn.f32x2 %0, %0, %1;" : "+l"(a01) : "l"(b01));
  asm("add.rn.f32x2 %0, %0, %1;" : "+l"(a23) : "l"(b23));
  asm("mov.b64 {%0, %1}, %2;" : "=f"(acc[0]), "=f"(acc[1]) : "l"(a01));
  asm("mov.b64 {%0, %1}, %2;" : "=f"(acc[2]), "=f"(acc[3]) : "l"(a23));
}
__device__ __forceinline__ void minadd4(double* acc, double x, const double* d) {
#pragma unroll
  for (int q = 0; q < 4; ++q) acc[q] = __dadd_rn(acc[q], fmin(x, d[q]));
}

// one staged entry of a heavy row: byte offset of its column's query values
// in the stage, and the index value (read back as one broadcast shared load)
template <typename T> struct MsEntry;
template <> struct __align__(8) MsEntry<float> { uint32_t off; float v; };
template <> struct __align__(16) MsEntry<double> { uint32_t off, pad; double v; };

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

// grid (ceil(nh / MS_HB), groups, qpad / 128); (MS_WARPS + 1) x 32 threads; dynamic shared
// memory ms_stages x 64 KB + the CTA's chunk pointers + per-warp entry staging.  D = HQT+ in 128-query
// blocks: block qb's column c values at D + (qb * n_cols + c) * 128.  CTA b
// takes the degree-ordered heavy positions b, b + hblocks, b + 2 hblocks, ...
// (a stratified sample of the degrees: every CTA carries about the same work).
template <typename T>
__global__ void __launch_bounds__((MS_WARPS + 1) * 32, 1) hminsum_kernel(
    const int64_t* __restrict__ hchunk, int64_t nch, const int32_t* __restrict__ hperm, int64_t nh,
    const int32_t* __restrict__ bidx, const T* __restrict__ bval, const T* __restrict__ D, int64_t n_cols,
    int64_t G, int64_t hpad, int64_t qpad, T* __restrict__ part) {
  constexpr int CW = ms_cw<T>();
  constexpr int MS_STAGES = ms_stages<T>();
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) unsigned long long bars[6];  // full[3], empty[3]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t g = blockIdx.y, qb = blockIdx.z, hb = gridDim.x;
  const int64_t k0 = g * G, k1 = tmin<int64_t>(nch, k0 + G);
  const int gs = int(k1 - k0) + 1;  // chunk pointers per row
  const T* Dq = D + qb * n_cols * 128;
  const uint32_t sbase = uint32_t(__cvta_generic_to_shared(smem));
  const uint32_t fb = uint32_t(__cvta_generic_to_shared(&bars[0])), eb = fb + 24;
  int64_t* hcs = reinterpret_cast<int64_t*>(smem + MS_STAGES * MS_STAGE_BYTES);  // [MS_HB][gs]
  if (threadIdx.x == 0) {
    for (int s = 0; s < MS_STAGES; ++s) {
      mbar_init(fb + 8 * s, 1);
      mbar_init(eb + 8 * s, MS_WARPS);
    }
    mbar_fence_init();
  }
  auto heavy_of = [&](int r) -> int32_t {  // local row r = u * MS_WARPS + warp
    const int64_t p = int64_t(r) * hb + blockIdx.x;
    return p < nh ? hperm[p] : -1;
  };
  for (int e = threadIdx.x; e < MS_HB * gs; e += blockDim.x) {
    const int r = e / gs, t = e - r * gs;
    const int32_t h = heavy_of(r);
    hcs[e] = h >= 0 ? hchunk[int64_t(h) * (nch + 1) + k0 + t] : 0;
  }
  __syncthreads();
  if (warp == MS_WARPS) {
    // producer warp: refills a stage once all consumer warps released it, so
    // the consumers drift apart by up to MS_STAGES - 1 chunks instead of
    // meeting at a block-wide barrier every chunk
    if (lane == 0) {
      for (int64_t k = k0; k < k1; ++k) {
        const int64_t i = k - k0;
        const int s = int(i % MS_STAGES);
        if (i >= MS_STAGES) mbar_wait(eb + 8 * s, uint32_t(((i / MS_STAGES) - 1) & 1));
        const int64_t c0 = k * CW;
        const uint32_t bytes = uint32_t(tmin<int64_t>(CW, n_cols - c0)) * 128u * uint32_t(sizeof(T));
        mbar_expect_tx(fb + 8 * s, bytes);
        bulk_g2s(sbase + uint32_t(s) * MS_STAGE_BYTES, Dq + c0 * 128, bytes, fb + 8 * s);
      }
    }
    return;
  }
  int32_t hs[MS_RPW];
#pragma unroll
  for (int u = 0; u < MS_RPW; ++u) hs[u] = heavy_of(u * MS_WARPS + warp);
  // the first 32 entries of every row's chunk, fetched one chunk ahead so the
  // global loads overlap the previous chunk's min-adds
  int32_t cc[MS_RPW];
  T cv[MS_RPW];
  auto fetch = [&](int64_t k, int32_t* pc, T* pv) {
#pragma unroll
    for (int u = 0; u < MS_RPW; ++u) {
      pc[u] = 0;
      pv[u] = T(0);
      if (hs[u] >= 0 && k < k1) {
        const int64_t* hr = hcs + (u * MS_WARPS + warp) * gs + (k - k0);
        const int64_t e = hr[0] + lane;
        if (e < hr[1]) { pc[u] = bidx[e]; pv[u] = bval[e]; }
      }
    }
  };
  fetch(k0, cc, cv);
  T acc[MS_RPW][4];
#pragma unroll
  for (int u = 0; u < MS_RPW; ++u)
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[u][q] = T(0);
  // per-warp staging of the prefetched entries: [MS_RPW][32]
  MsEntry<T>* stg = reinterpret_cast<MsEntry<T>*>(hcs + MS_HB * gs) + warp * (MS_RPW * 32);
  constexpr uint32_t ROWB = 128u * uint32_t(sizeof(T));  // bytes of one column's query values
  for (int64_t k = k0; k < k1; ++k) {
    const int32_t c0 = int32_t(k * CW);
    // this chunk's first 32 entries per row into the warp's staging area
    // (padding lanes: offset 0, value 0 -> min(0, d) = 0 adds nothing)
    __syncwarp();  // the previous chunk's reads of the staging area are done
#pragma unroll
    for (int u = 0; u < MS_RPW; ++u) {
      const int64_t* hr = hcs + (u * MS_WARPS + warp) * gs + (k - k0);
      const bool ok = hs[u] >= 0 && hr[0] + lane < hr[1];
      MsEntry<T> en;
      en.off = ok ? uint32_t(cc[u] - c0) * ROWB : 0u;
      if constexpr (sizeof(T) == 8) en.pad = 0;
      en.v = ok ? cv[u] : T(0);
      stg[u * 32 + lane] = en;
    }
    __syncwarp();
    fetch(k + 1, cc, cv);  // next chunk's entries: in flight during this chunk
    const int64_t i = k - k0;
    const int s = int(i % MS_STAGES);
    mbar_wait(fb + 8 * s, uint32_t((i / MS_STAGES) & 1));
    // the lane's 4 queries: 4l..4l+3 (fp32), 2l, 2l+1, 64+2l, 65+2l (fp64: each
    // 16-byte shared load contiguous over the warp, EQ<T> in isect_kernel.cuh)
    const uint32_t sq = sbase + uint32_t(s) * MS_STAGE_BYTES + uint32_t(lane) * uint32_t(EQ<T>::CELL * sizeof(T));
#pragma unroll
    for (int u = 0; u < MS_RPW; ++u) {
      if (hs[u] < 0) continue;  // warp-uniform
      const int64_t* hr = hcs + (u * MS_WARPS + warp) * gs + (k - k0);
      const int64_t beg = hr[0], end = hr[1];
      const int nn = int(tmin<int64_t>(32, end - beg));
      const MsEntry<T>* row = stg + u * 32;
      if constexpr (sizeof(T) == 4) {
        // fp32: two staged entries per 16-byte broadcast load (4.5 instead of 5
        // shared wavefronts per entry), steps of 8 and a last step of 4 when at
        // most 4 entries remain (the zero padding costs wavefronts too)
        auto step = [&](int t, auto nv) {
          constexpr int NV = decltype(nv)::value;
          T d[NV][4];
          uint32_t off[NV];
          T x[NV];
#pragma unroll
          for (int v = 0; v < NV; v += 2) {
            const uint4 w = *reinterpret_cast<const uint4*>(row + t + v);  // 16-byte aligned pair
            off[v] = w.x; x[v] = __uint_as_float(w.y);
            off[v + 1] = w.z; x[v + 1] = __uint_as_float(w.w);
            EQ<T>::lds(sq + off[v], d[v]);
            EQ<T>::lds(sq + off[v + 1], d[v + 1]);
          }
#pragma unroll
          for (int v = 0; v < NV; ++v) minadd4(acc[u], x[v], d[v]);
        };
        int t = 0;
        for (; t + 4 < nn; t += MS_UNROLL) step(t, std::integral_constant<int, MS_UNROLL>{});
        if (t < nn) step(t, std::integral_constant<int, 4>{});
      } else {
        for (int t = 0; t < nn; t += MS_UNROLL) {  // padded to a multiple of MS_UNROLL
          T d[MS_UNROLL][4];
          MsEntry<T> en[MS_UNROLL];
#pragma unroll
          for (int v = 0; v < MS_UNROLL; ++v) {
            en[v] = row[t + v];
            EQ<T>::lds(sq + en[v].off, d[v]);
          }
#pragma unroll
          for (int v = 0; v < MS_UNROLL; ++v) minadd4(acc[u], en[v].v, d[v]);
        }
      }
      for (int64_t e0 = beg + 32; e0 < end; e0 += 32) {  // long rows: entries beyond the staged 32
        const bool ok = e0 + lane < end;
        const uint32_t ol = ok ? uint32_t(bidx[e0 + lane] - c0) * ROWB : 0u;
        const T vl = ok ? bval[e0 + lane] : T(0);
        const int n2 = int(tmin<int64_t>(32, end - e0));
        for (int t = 0; t < n2; ++t) {
          T d[4];
          const uint32_t o = __shfl_sync(0xffffffffu, ol, t);
          const T x = __shfl_sync(0xffffffffu, vl, t);
          EQ<T>::lds(sq + o, d);
          minadd4(acc[u], x, d);
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(eb + 8 * s);  // this warp is done with stage s
  }
  T* out = part + g * hpad * qpad + qb * 128 + EQ<T>::CELL * lane;
#pragma unroll
  for (int u = 0; u < MS_RPW; ++u) {
    if (hs[u] < 0) continue;
    T* o = out + int64_t(hs[u]) * qpad;
    if constexpr (sizeof(T) == 4) {
      V4<T>::store_plain(o, acc[u]);
    } else {
      reinterpret_cast<double2*>(o)[0] = make_double2(acc[u][0], acc[u][1]);
      reinterpret_cast<double2*>(o + 64)[0] = make_double2(acc[u][2], acc[u][3]);
    }
  }
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
  // chunk groups: 3-6 waves of one-CTA-per-SM blocks (fewer partials than
  // one group per chunk, enough CTAs to balance), the count whose last wave
  // is fullest; at most MS_MAX_G chunks per group (their pointers sit in
  // shared memory)
  const int64_t sms = num_sms(), per = hblocks * qblocks;
  int64_t groups = 0;
  double best = 1e30;
  for (int64_t gg = std::max<int64_t>(1, (3 * sms) / per); gg <= std::max<int64_t>(1, (6 * sms + per - 1) / per); ++gg) {
    const int64_t G0 = (nch + gg - 1) / gg;
    if (G0 > MS_MAX_G) continue;
    const int64_t ctas = per * ((nch + G0 - 1) / G0);
    const double waste = double((ctas + sms - 1) / sms * sms) / double(ctas);
    if (waste < best - 1e-9) { best = waste; groups = gg; }
  }
  if (groups == 0) groups = (nch + MS_MAX_G - 1) / MS_MAX_G;
  const int64_t G = (nch + groups - 1) / groups;
  groups = (nch + G - 1) / G;
  const size_t es = dtype == SD_F64 ? 8 : 4;
  SD_TRY(part.alloc(es * size_t(groups) * size_t(ix->hpad) * size_t(qpad), st));
  return SD_DISPATCH_DTYPE(dtype, T, [&]() -> int {
    const size_t smem = size_t(ms_stages<T>()) * MS_STAGE_BYTES + size_t(MS_HB) * size_t(G + 1) * sizeof(int64_t) +
                        size_t(MS_WARPS) * MS_RPW * 32 * sizeof(MsEntry<T>);
    SD_TRY(prepare_smem(hminsum_kernel<T>, smem, "hminsum_kernel"));
    const dim3 grid{unsigned(hblocks), unsigned(groups), unsigned(qblocks)};
    hminsum_kernel<T><<<grid, (MS_WARPS + 1) * 32, smem, st>>>(ix->hchunk, nch, ix->hperm, nh, b->indices,
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
