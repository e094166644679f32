// prep.cu — per-row statistics and element-wise preparation kernels.
//
// Row reductions run one thread per row and accumulate SEQUENTIALLY in
// ascending column order.  The fused intersection kernel (isect.cu) accumulates
// its per-cell dot products in the same ascending order, so ||a||^2 and
// <a,a> are bitwise equal and self-distances of the expanded metrics come
// out exactly 0, as they do in the reference (hard part 4).
#include "common.cuh"
#include "prep.cuh"
#include "semiring.cuh"

namespace sd {

template <typename T, int KIND, int SR>
__device__ __forceinline__ T stat_term(T v, T p) {
  if constexpr (KIND == SD_STAT_L0) return T(1);
  else if constexpr (KIND == SD_STAT_L1) return abs_(v);
  else if constexpr (KIND == SD_STAT_L2 || KIND == SD_STAT_L2SQ) return mul_rn(v, v);
  else if constexpr (KIND == SD_STAT_SUM) return v;
  else if constexpr (KIND == STAT_ONESIDED_A) return product_a0<SR, T>(v, p);
  else return product_0b<SR, T>(v, p);  // STAT_ONESIDED_B
}

// Sequential ascending sums (the association order of the fused kernel's
// per-cell accumulation).  A warp owns 32 consecutive rows: short rows are
// summed by their own lane; each long row (power-law tail) is then summed by
// the whole warp — chunks of 256 values loaded coalesced (next chunk in flight
// while the current one is summed), staged in shared memory and added in
// order by lane 0 — so a 25k-entry row costs ~its FADD chain, not 25k
// dependent global loads.
constexpr int STAT_LONG = 64;
constexpr int STAT_CHUNK = 256;
constexpr int64_t STAT_BLOCKED = 2048;  // longer rows: 32 lane-blocked partial sums
constexpr int STAT_WARPS = 4;

// LONG = false: one lane per row, rows of <= STAT_LONG entries (all rows for
// L0).  LONG = true: one warp per row, the longer rows — a second launch so
// that the long rows of power-law data run side by side, not one after
// another inside the warp that owns their 32-row group.
template <typename T, int KIND, int SR, bool LONG>
__global__ void __launch_bounds__(STAT_WARPS * 32) row_stat_kernel(const int64_t* __restrict__ ptr,
                                                                   const T* __restrict__ val, int64_t n_rows,
                                                                   T p, T* __restrict__ out, T* __restrict__ out2) {
  __shared__ __align__(16) T stage[STAT_WARPS][STAT_CHUNK];
  const unsigned lane = lane_id();
  const int w = threadIdx.x >> 5;
  const int64_t nwarps = int64_t(gridDim.x) * STAT_WARPS;
  const int64_t gwarp = int64_t(blockIdx.x) * STAT_WARPS + w;
  for (int64_t r0 = LONG ? gwarp : gwarp * 32; r0 < n_rows; r0 += LONG ? nwarps : nwarps * 32) {
    const int64_t r = LONG ? r0 : r0 + lane;
    const bool ok = r < n_rows && (!LONG || lane == 0);
    const int64_t beg = ok ? ptr[r] : 0, end = ok ? ptr[r + 1] : 0;
    const bool mine = LONG ? end - beg > STAT_LONG : (KIND == SD_STAT_L0 || end - beg <= STAT_LONG);
    if (LONG && !__any_sync(0xffffffffu, ok && mine)) continue;
    T s = T(0);
    if constexpr (KIND == SD_STAT_L0) {
      s = T(end - beg);
    } else if (!LONG && end - beg <= STAT_LONG) {
      int64_t e = beg;
      for (; e + 8 <= end; e += 8) {
        T t[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) t[u] = stat_term<T, KIND, SR>(__ldg(val + e + u), p);
#pragma unroll
        for (int u = 0; u < 8; ++u) s = add_rn(s, t[u]);
      }
      for (; e < end; ++e) s = add_rn(s, stat_term<T, KIND, SR>(__ldg(val + e), p));
    }
    if constexpr (KIND != SD_STAT_L0 && LONG) {
      unsigned long_mask = __ballot_sync(0xffffffffu, ok && end - beg > STAT_LONG);
      while (long_mask) {
        const int src = __ffs(long_mask) - 1;
        long_mask &= long_mask - 1;
        const int64_t lb = __shfl_sync(0xffffffffu, beg, src), le = __shfl_sync(0xffffffffu, end, src);
        T ls = T(0);
        if (le - lb > STAT_BLOCKED) {
          // very long (power-law) rows: each lane sums one contiguous 1/32 of the
          // row in order, lane 0 adds the 32 partials in order — deterministic,
          // a 32x shorter dependency chain than the strictly sequential sum
          const int64_t len = le - lb, per = (len + 31) / 32;
          const int64_t cb = lb + tmin<int64_t>(len, int64_t(lane) * per), ce = tmin<int64_t>(le, cb + per);
          T part = T(0);
          int64_t e = cb;
          for (; e + 8 <= ce; e += 8) {
            T t[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) t[u] = stat_term<T, KIND, SR>(__ldg(val + e + u), p);
#pragma unroll
            for (int u = 0; u < 8; ++u) part = add_rn(part, t[u]);
          }
          for (; e < ce; ++e) part = add_rn(part, stat_term<T, KIND, SR>(__ldg(val + e), p));
          for (int l = 0; l < 32; ++l) ls = add_rn(ls, __shfl_sync(0xffffffffu, part, l));
          if (int(lane) == src) s = ls;
          continue;
        }
        T nxt[STAT_CHUNK / 32];
#pragma unroll
        for (int k = 0; k < STAT_CHUNK / 32; ++k) {
          const int64_t e = lb + k * 32 + lane;
          nxt[k] = e < le ? __ldg(val + e) : T(0);
        }
        for (int64_t c = lb; c < le; c += STAT_CHUNK) {
          __syncwarp();
#pragma unroll
          for (int k = 0; k < STAT_CHUNK / 32; ++k) stage[w][k * 32 + lane] = nxt[k];
          __syncwarp();
#pragma unroll
          for (int k = 0; k < STAT_CHUNK / 32; ++k) {  // next chunk in flight during the serial sum
            const int64_t e = c + STAT_CHUNK + k * 32 + lane;
            nxt[k] = e < le ? __ldg(val + e) : T(0);
          }
          if (lane == 0) {  // loads batched 8 ahead: the chain runs at FADD latency
            const int cnt = int(tmin<int64_t>(STAT_CHUNK, le - c));
            int q = 0;
            for (; q + 8 <= cnt; q += 8) {
              T t[8];
#pragma unroll
              for (int u = 0; u < 8; ++u) t[u] = stat_term<T, KIND, SR>(stage[w][q + u], p);
#pragma unroll
              for (int u = 0; u < 8; ++u) ls = add_rn(ls, t[u]);
            }
            for (; q < cnt; ++q) ls = add_rn(ls, stat_term<T, KIND, SR>(stage[w][q], p));
          }
        }
        ls = __shfl_sync(0xffffffffu, ls, 0);
        if (int(lane) == src) s = ls;
      }
    }
    if constexpr (KIND == SD_STAT_L2) s = sqrt_rn(s);
    if (ok && mine) {
      out[r] = s;
      if constexpr (KIND == SD_STAT_L2)  // optional 1/||row|| (0 for empty rows), same pass
        if (out2) out2[r] = s > T(0) ? div_rn(T(1), s) : T(0);
    }
  }
}

template <typename T, int KIND, int SR>
static int launch_stat(const sd_csr* m, T p, void* out, cudaStream_t st, void* out2 = nullptr) {
  if (m->n_rows == 0) return SD_OK;
  const int64_t warps = (m->n_rows + 31) / 32;
  int blocks = int(tmin<int64_t>((warps + STAT_WARPS - 1) / STAT_WARPS, int64_t(num_sms()) * 16));
  row_stat_kernel<T, KIND, SR, false><<<blocks, STAT_WARPS * 32, 0, st>>>(
      m->indptr, static_cast<const T*>(m->values), m->n_rows, p, static_cast<T*>(out), static_cast<T*>(out2));
  SD_LAUNCH_CHECK();
  if constexpr (KIND != SD_STAT_L0) {
    const int lblocks = int(tmin<int64_t>((m->n_rows + STAT_WARPS - 1) / STAT_WARPS, int64_t(num_sms()) * 32));
    row_stat_kernel<T, KIND, SR, true><<<lblocks, STAT_WARPS * 32, 0, st>>>(
        m->indptr, static_cast<const T*>(m->values), m->n_rows, p, static_cast<T*>(out), static_cast<T*>(out2));
    SD_LAUNCH_CHECK();
  }
  return SD_OK;
}

int row_stat_l2_inv(const sd_csr* m, int dtype, void* l2, void* inv, cudaStream_t st) {
  return SD_DISPATCH_DTYPE(dtype, T, [&]() -> int { return launch_stat<T, SD_STAT_L2, 0>(m, T(0), l2, st, inv); });
}

int row_stat(const sd_csr* m, int dtype, int kind, int semiring, double p, void* out,
             cudaStream_t st) {
  return SD_DISPATCH_DTYPE(dtype, T, [&]() -> int {
    const T pp = T(p);
    switch (kind) {
      case SD_STAT_L0: return launch_stat<T, SD_STAT_L0, 0>(m, pp, out, st);
      case SD_STAT_L1: return launch_stat<T, SD_STAT_L1, 0>(m, pp, out, st);
      case SD_STAT_L2: return launch_stat<T, SD_STAT_L2, 0>(m, pp, out, st);
      case SD_STAT_L2SQ: return launch_stat<T, SD_STAT_L2SQ, 0>(m, pp, out, st);
      case SD_STAT_SUM: return launch_stat<T, SD_STAT_SUM, 0>(m, pp, out, st);
      case STAT_ONESIDED_A:
        return SD_DISPATCH_SEMIRING(semiring, SR, [&]() -> int { return launch_stat<T, STAT_ONESIDED_A, SR>(m, pp, out, st); });
      case STAT_ONESIDED_B:
        return SD_DISPATCH_SEMIRING(semiring, SR, [&]() -> int { return launch_stat<T, STAT_ONESIDED_B, SR>(m, pp, out, st); });
      default:
        set_error("unknown row statistic kind");
        return SD_E_INVALID;
    }
  });
}

// Per-row top-K by |value| (ties -> lower entry index): rank[e] in [0, K) for
// the K largest entries of each row, 255 otherwise; top[r * n_rows + row] =
// the r-th largest |value| (0 beyond the row's degree).  Used by the fused
// Chebyshev path (max over the union needs the largest one-sided entries).
template <typename T>
__global__ void row_topk_kernel(const int64_t* __restrict__ ptr, const T* __restrict__ val, int64_t n_rows,
                                uint8_t* __restrict__ rank, T* __restrict__ top) {
  const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  const unsigned lane = lane_id();
  for (int64_t row = warp; row < n_rows; row += nw) {
    const int64_t beg = ptr[row], end = ptr[row + 1];
    for (int64_t e = beg + lane; e < end; e += 32) rank[e] = 255;
    __syncwarp();
    T prev_k = Num<T>::inf();
    int64_t prev_e = -1;
    for (int r = 0; r < CHEB_K; ++r) {
      // next entry in (|v| desc, e asc) order after (prev_k, prev_e)
      T best_k = T(-1);
      int64_t best_e = INT64_MAX;
      for (int64_t e = beg + lane; e < end; e += 32) {
        const T k = abs_(val[e]);
        const bool after = k < prev_k || (k == prev_k && e > prev_e);
        if (after && (k > best_k || (k == best_k && e < best_e))) { best_k = k; best_e = e; }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const T ok = __shfl_xor_sync(0xffffffffu, best_k, o);
        const int64_t oe = __shfl_xor_sync(0xffffffffu, best_e, o);
        if (ok > best_k || (ok == best_k && oe < best_e)) { best_k = ok; best_e = oe; }
      }
      if (lane == 0) top[int64_t(r) * n_rows + row] = best_e == INT64_MAX ? T(0) : best_k;
      if (best_e == INT64_MAX) {  // row exhausted
        for (int rr = r + 1 + int(lane); rr < CHEB_K; rr += 32) top[int64_t(rr) * n_rows + row] = T(0);
        break;
      }
      if (lane == 0) rank[best_e] = uint8_t(r);
      prev_k = best_k;
      prev_e = best_e;
    }
  }
}

int row_topk(const sd_csr* m, int dtype, uint8_t* rank, void* top, cudaStream_t st) {
  if (m->n_rows == 0) return SD_OK;
  return SD_DISPATCH_DTYPE(dtype, T, [&]() -> int {
    const int blocks = int(tmin<int64_t>((m->n_rows * 32 + 255) / 256, int64_t(num_sms()) * 16));
    row_topk_kernel<T><<<blocks, 256, 0, st>>>(m->indptr, static_cast<const T*>(m->values), m->n_rows, rank,
                                               static_cast<T*>(top));
    SD_LAUNCH_CHECK();
    return SD_OK;
  });
}

__global__ void coo_rows_kernel(const int64_t* __restrict__ ptr, int64_t n_rows,
                                int64_t* __restrict__ rows) {
  const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t r = warp; r < n_rows; r += nwarps)
    for (int64_t e = ptr[r] + lane_id(); e < ptr[r + 1]; e += 32) rows[e] = r;
}

int csr_to_coo(const sd_csr* m, int64_t* rows, cudaStream_t st) {
  if (m->n_rows == 0 || m->nnz == 0) return SD_OK;
  int blocks = int(tmin<int64_t>((m->n_rows * 32 + 255) / 256, int64_t(num_sms()) * 16));
  coo_rows_kernel<<<blocks, 256, 0, st>>>(m->indptr, m->n_rows, rows);
  SD_LAUNCH_CHECK();
  return SD_OK;
}

template <typename T>
__global__ void negative_kernel(const T* __restrict__ v, int64_t n, uint32_t* flags) {
  bool neg = false;
  for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < n;
       e += int64_t(gridDim.x) * blockDim.x)
    neg |= v[e] < T(0);
  if (__any_sync(0xffffffffu, neg) && lane_id() == 0) atomicOr(flags, SD_FLAG_NEGATIVE);
}

int check_nonnegative(const sd_csr* m, int dtype, uint32_t* flags, cudaStream_t st) {
  if (m->nnz == 0) return SD_OK;
  return SD_DISPATCH_DTYPE(dtype, T, [&]() -> int {
    int blocks = int(tmin<int64_t>((m->nnz + 255) / 256, int64_t(num_sms()) * 8));
    negative_kernel<T><<<blocks, 256, 0, st>>>(static_cast<const T*>(m->values), m->nnz, flags);
    SD_LAUNCH_CHECK();
    return SD_OK;
  });
}

template <typename T>
__global__ void sqrt_kernel(const T* __restrict__ v, int64_t n, T* __restrict__ out) {
  for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < n;
       e += int64_t(gridDim.x) * blockDim.x)
    out[e] = sqrt_rn(v[e]);
}

int sqrt_values(const sd_csr* m, int dtype, void* out, cudaStream_t st) {
  if (m->nnz == 0) return SD_OK;
  return SD_DISPATCH_DTYPE(dtype, T, [&]() -> int {
    int blocks = int(tmin<int64_t>((m->nnz + 255) / 256, int64_t(num_sms()) * 8));
    sqrt_kernel<T><<<blocks, 256, 0, st>>>(static_cast<const T*>(m->values), m->nnz,
                                           static_cast<T*>(out));
    SD_LAUNCH_CHECK();
    return SD_OK;
  });
}

template <typename T>
__global__ void fill_kernel(T* __restrict__ out, int64_t m, int64_t n, int64_t ldo, T value) {
  const int64_t total = m * n;
  for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = e / n, j = e - i * n;
    out[i * ldo + j] = value;
  }
}

int fill(void* out, int64_t m, int64_t n, int64_t ldo, int dtype, double value, cudaStream_t st) {
  if (m == 0 || n == 0) return SD_OK;
  return SD_DISPATCH_DTYPE(dtype, T, [&]() -> int {
    int blocks = int(tmin<int64_t>((m * n + 255) / 256, int64_t(num_sms()) * 16));
    fill_kernel<T><<<blocks, 256, 0, st>>>(static_cast<T*>(out), m, n, ldo, T(value));
    SD_LAUNCH_CHECK();
    return SD_OK;
  });
}

}  // namespace sd
