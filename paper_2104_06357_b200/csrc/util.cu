// util.cu — device-backed utilities of the drop-in surface that are not the
// distance sweep itself:
//   * segment_reduce (sparse.py:31-53) with numpy's exact reduceat association,
//   * mix32 and the open-addressing HashAccumulator (hashtable.py:12-106),
//   * elementwise semiring products (Semiring.product_op, semiring.py:36-119),
//   * the dense brute-force arbiter of `verify` (oracle.py:35-190 formulas),
//   * validate_and_canonicalize (sparse.py:135-202): validation with the
//     reference's error order, stable (row, column) sort, duplicates summed
//     in input order with numpy's association, zeros dropped.
#include <cub/cub.cuh>
#include "common.cuh"
#include "semiring.cuh"

namespace sd {

// ---------------------------------------------------------------- segment_reduce

// numpy's pairwise summation (umath loops_utils: blocks of < 8 summed in
// order from -0.0, <= 128 with 8 interleaved accumulators, longer halved at
// a multiple of 8).  add.reduceat evaluates a segment as v[0] + pw(v[1:]).
template <typename T>
__device__ T pw_sum(const T* a, int64_t n) {
  if (n < 8) {
    T res = T(-0.0);
    for (int64_t i = 0; i < n; ++i) res = add_rn(res, a[i]);
    return res;
  }
  if (n <= 128) {
    T r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = a[j];
    int64_t i = 8;
    for (; i < n - (n % 8); i += 8)
#pragma unroll
      for (int j = 0; j < 8; ++j) r[j] = add_rn(r[j], a[i + j]);
    T res = add_rn(add_rn(add_rn(r[0], r[1]), add_rn(r[2], r[3])), add_rn(add_rn(r[4], r[5]), add_rn(r[6], r[7])));
    for (; i < n; ++i) res = add_rn(res, a[i]);
    return res;
  }
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  return add_rn(pw_sum(a, n2), pw_sum(a + n2, n - n2));
}

template <typename T>
__device__ __forceinline__ T np_max(T a, T b) { return (a != a || a >= b) ? a : b; }  // NaN propagates
template <typename T>
__device__ __forceinline__ T np_min(T a, T b) { return (a != a || a <= b) ? a : b; }

template <typename T>
__global__ void segment_reduce_kernel(const T* __restrict__ v, const int64_t* __restrict__ bounds, int64_t n_seg,
                                      int ufunc, T identity, T* __restrict__ out) {
  for (int64_t s = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; s < n_seg; s += int64_t(gridDim.x) * blockDim.x) {
    const int64_t b = bounds[s], e = bounds[s + 1];
    if (b >= e) { out[s] = identity; continue; }
    T r = v[b];
    if (ufunc == SD_UFUNC_ADD) {
      if (e - b > 1) r = add_rn(r, pw_sum(v + b + 1, e - b - 1));
    } else {
      for (int64_t i = b + 1; i < e; ++i)
        r = ufunc == SD_UFUNC_MAXIMUM ? np_max(r, v[i]) : ufunc == SD_UFUNC_MINIMUM ? np_min(r, v[i]) : mul_rn(r, v[i]);
    }
    out[s] = r;
  }
}

// ---------------------------------------------------------------- hashing

__global__ void mix32_kernel(const int64_t* __restrict__ keys, int64_t n, uint64_t* __restrict__ out) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    out[i] = uint64_t(mix32(uint32_t(uint64_t(keys[i]) & 0xffffffffull)));
}

constexpr int64_t EMPTY_SLOT = INT64_MAX;  // hashtable.py:12

// HashAccumulator.build (hashtable.py:43-63): keys placed in insertion order by
// linear probing from mix32(key) % capacity — one thread, so the table layout
// is exactly the reference's (capacities are <= 16384 entries).
__global__ void hash_build_kernel(const int64_t* __restrict__ keys, const double* __restrict__ vals, int64_t n,
                                  int64_t cap, int64_t* __restrict__ tk, double* __restrict__ tv) {
  for (int64_t h = threadIdx.x; h < cap; h += blockDim.x) tk[h] = EMPTY_SLOT;
  __syncthreads();
  if (threadIdx.x != 0) return;
  for (int64_t i = 0; i < n; ++i) {
    int64_t h = int64_t(mix32(uint32_t(uint64_t(keys[i]) & 0xffffffffull)) % uint64_t(cap));
    while (tk[h] != EMPTY_SLOT) h = h + 1 == cap ? 0 : h + 1;
    tk[h] = keys[i];
    tv[h] = vals[i];
  }
}

// HashAccumulator.probe_many (hashtable.py:80-106): one thread per query key.
__global__ void hash_probe_kernel(const int64_t* __restrict__ tk, const double* __restrict__ tv, int64_t cap,
                                  const int64_t* __restrict__ q, int64_t n, double* __restrict__ ov,
                                  uint8_t* __restrict__ of) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t key = q[i];
    int64_t h = int64_t(mix32(uint32_t(uint64_t(key) & 0xffffffffull)) % uint64_t(cap));
    double v = 0.0;
    uint8_t f = 0;
    for (int64_t step = 0; step < cap; ++step) {
      const int64_t k = tk[h];
      if (k == key) { v = tv[h]; f = 1; break; }
      if (k == EMPTY_SLOT) break;
      h = h + 1 == cap ? 0 : h + 1;
    }
    ov[i] = v;
    of[i] = f;
  }
}

// ---------------------------------------------------------------- semiring products

template <int SR>
__global__ void semiring_apply_kernel(const double* __restrict__ x, const double* __restrict__ y, int64_t n,
                                      double p, double* __restrict__ out) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    out[i] = product<SR, double>(x[i], y[i], p);
}

// ---------------------------------------------------------------- dense arbiter

// One thread per (i, j): the textbook formula over all k columns of the two
// dense rows (oracle.py:35-154), sharing no code with the sparse kernels.
__global__ void dense_pairwise_kernel(const double* __restrict__ da, const double* __restrict__ db, int64_t m,
                                      int64_t n, int64_t k, int metric, double p, int strict,
                                      double* __restrict__ out, uint32_t* flags) {
  uint32_t f = 0;
  for (int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; q < m * n; q += int64_t(gridDim.x) * blockDim.x) {
    const double* a = da + (q / n) * k;
    const double* b = db + (q % n) * k;
    double r = 0.0;
    switch (metric) {
      case SD_M_MANHATTAN: for (int64_t c = 0; c < k; ++c) r += fabs(a[c] - b[c]); break;
      case SD_M_CHEBYSHEV: for (int64_t c = 0; c < k; ++c) r = fmax(r, fabs(a[c] - b[c])); break;
      case SD_M_MINKOWSKI:
        for (int64_t c = 0; c < k; ++c) r += pow(fabs(a[c] - b[c]), p);
        r = pow(r, 1.0 / p);
        break;
      case SD_M_CANBERRA:
        for (int64_t c = 0; c < k; ++c) {
          const double den = fabs(a[c]) + fabs(b[c]);
          r += den > 0 ? fabs(a[c] - b[c]) / den : 0.0;
        }
        break;
      case SD_M_HAMMING: {
        int64_t cnt = 0;
        for (int64_t c = 0; c < k; ++c) cnt += a[c] != b[c];
        r = k ? double(cnt) / double(k) : 0.0;
        break;
      }
      case SD_M_EUCLIDEAN:
        for (int64_t c = 0; c < k; ++c) r += (a[c] - b[c]) * (a[c] - b[c]);
        r = sqrt(r);
        break;
      case SD_M_DOT: for (int64_t c = 0; c < k; ++c) r += a[c] * b[c]; break;
      case SD_M_COSINE: {
        double aa = 0, bb = 0, ab = 0;
        for (int64_t c = 0; c < k; ++c) { aa += a[c] * a[c]; bb += b[c] * b[c]; ab += a[c] * b[c]; }
        const double na = sqrt(aa), nb = sqrt(bb);
        r = (na == 0 && nb == 0) ? 0.0 : (na == 0 || nb == 0) ? 1.0 : 1.0 - ab / (na * nb);
        break;
      }
      case SD_M_CORRELATION: {
        double sa = 0, sb = 0;
        bool nz = false;
        for (int64_t c = 0; c < k; ++c) { sa += a[c]; sb += b[c]; nz |= a[c] != 0 || b[c] != 0; }
        const double ma = k ? sa / double(k) : 0.0, mb = k ? sb / double(k) : 0.0;
        double va = 0, vb = 0, cab = 0;
        for (int64_t c = 0; c < k; ++c) {
          const double x = a[c] - ma, y = b[c] - mb;
          va += x * x; vb += y * y; cab += x * y;
        }
        r = (va == 0 || vb == 0) ? (nz ? 1.0 : 0.0) : 1.0 - cab / sqrt(va * vb);
        break;
      }
      case SD_M_DICE:
      case SD_M_JACCARD: {
        double ca = 0, cb = 0, ab = 0;
        for (int64_t c = 0; c < k; ++c) { ca += a[c] != 0; cb += b[c] != 0; ab += a[c] * b[c]; }
        if (metric == SD_M_DICE) {
          r = ca + cb == 0 ? 0.0 : 1.0 - 2.0 * ab / (ca + cb);
        } else {
          const double den = ca + cb - ab;
          r = den <= 0 ? (ca + cb == 0 ? 0.0 : 1.0) : 1.0 - ab / den;
        }
        break;
      }
      case SD_M_RUSSELRAO: {
        double ab = 0;
        for (int64_t c = 0; c < k; ++c) ab += a[c] * b[c];
        r = k ? (double(k) - ab) / double(k) : 0.0;
        break;
      }
      case SD_M_HELLINGER: {
        double s = 0;
        for (int64_t c = 0; c < k; ++c) {
          if (a[c] < 0 || b[c] < 0) f |= SD_FLAG_NEGATIVE;
          s += sqrt(a[c] * b[c]);
        }
        r = 1.0 - sqrt(s);
        break;
      }
      case SD_M_KL: {
        bool uncovered = false;
        for (int64_t c = 0; c < k; ++c) {
          if (a[c] < 0 || b[c] < 0) f |= SD_FLAG_NEGATIVE;
          if (a[c] > 0 && b[c] == 0) uncovered = true;
          if (a[c] > 0 && b[c] != 0) r += a[c] * log(a[c] / b[c]);
        }
        if (uncovered) {
          if (strict) f |= SD_FLAG_KL_UNCOVERED;
          r = 1e308;
        }
        break;
      }
      case SD_M_JENSENSHANNON: {
        for (int64_t c = 0; c < k; ++c) {
          if (a[c] < 0 || b[c] < 0) f |= SD_FLAG_NEGATIVE;
          const double mu = 0.5 * (a[c] + b[c]);
          const double smu = mu > 0 ? mu : 1.0;
          r += (a[c] > 0 ? a[c] * log(a[c] / smu) : 0.0) + (b[c] > 0 ? b[c] * log(b[c] / smu) : 0.0);
        }
        r = sqrt(fmax(r, 0.0) / 2.0);
        break;
      }
      default: break;
    }
    out[q] = r;
  }
  f = __reduce_or_sync(0xffffffffu, f);
  if (f && lane_id() == 0) atomicOr(flags, f);
}

static int grid_for(int64_t n) { return int(tmax<int64_t>(1, tmin<int64_t>((n + 255) / 256, int64_t(num_sms()) * 16))); }

// ---------------------------------------------------------------- canonicalize

// first offending positions (atomicMin): [0] negative indptr entry, [1] row
// where indptr decreases, [2] entry whose column is outside [0, n_cols)
__global__ void canon_check_kernel(const int64_t* __restrict__ ptr, int64_t n_rows, const int64_t* __restrict__ idx,
                                   int64_t nnz, int64_t n_cols, unsigned long long* first) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; r <= n_rows; r += stride) {
    if (ptr[r] < 0) atomicMin(&first[0], (unsigned long long)r);
    if (r < n_rows && ptr[r + 1] < ptr[r]) atomicMin(&first[1], (unsigned long long)r);
  }
  for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < nnz; e += stride)
    if (idx[e] < 0 || idx[e] >= n_cols) atomicMin(&first[2], (unsigned long long)e);
}

// row of entry `pos` (searchsorted(indptr, pos, 'right') - 1) and its column
__global__ void canon_locate_kernel(const int64_t* __restrict__ ptr, int64_t n_rows, const int64_t* __restrict__ idx,
                                    int64_t pos, int64_t* out) {
  int64_t lo = 0, hi = n_rows + 1;  // first r with ptr[r] > pos
  while (lo < hi) {
    const int64_t mid = (lo + hi) / 2;
    if (ptr[mid] > pos) hi = mid; else lo = mid + 1;
  }
  out[0] = lo - 1;
  out[1] = idx[pos];
}

__global__ void canon_keys_kernel(const int64_t* __restrict__ ptr, int64_t n_rows, const int64_t* __restrict__ idx,
                                  int64_t n_cols, uint64_t* __restrict__ keys, int64_t* __restrict__ order) {
  const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t r = warp; r < n_rows; r += nw)
    for (int64_t e = ptr[r] + lane_id(); e < ptr[r + 1]; e += 32) {
      keys[e] = uint64_t(r) * uint64_t(n_cols > 0 ? n_cols : 1) + uint64_t(idx[e]);
      order[e] = e;
    }
}

// run heads of the sorted keys
__global__ void canon_heads_kernel(const uint64_t* __restrict__ keys, int64_t nnz, uint8_t* __restrict__ head) {
  for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < nnz; e += int64_t(gridDim.x) * blockDim.x)
    head[e] = e == 0 || keys[e] != keys[e - 1];
}

// one run of equal keys -> its value (add.reduceat association, input order) and keep flag
__global__ void canon_runs_kernel(const uint64_t* __restrict__ keys, const int64_t* __restrict__ order,
                                  const double* __restrict__ vals, const int64_t* __restrict__ starts,
                                  const int64_t* __restrict__ n_runs_p, int64_t nnz, uint64_t* __restrict__ rkey,
                                  double* __restrict__ rval, uint8_t* __restrict__ keep, double* __restrict__ scratch) {
  const int64_t n_runs = *n_runs_p;
  for (int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < n_runs; r += int64_t(gridDim.x) * blockDim.x) {
    const int64_t b = starts[r], e = r + 1 < n_runs ? starts[r + 1] : nnz;
    for (int64_t i = b; i < e; ++i) scratch[i] = vals[order[i]];
    double v = scratch[b];
    if (e - b > 1) v = add_rn(v, pw_sum(scratch + b + 1, e - b - 1));
    rkey[r] = keys[b];
    rval[r] = v;
    keep[r] = v != 0.0;
  }
}

__global__ void canon_split_kernel(const uint64_t* __restrict__ key, const int64_t* __restrict__ n_p, int64_t n_cols,
                                   int64_t* __restrict__ cols, unsigned int* __restrict__ counts) {
  const int64_t n = *n_p;
  const uint64_t nc = uint64_t(n_cols > 0 ? n_cols : 1);
  for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < n; e += int64_t(gridDim.x) * blockDim.x) {
    const uint64_t r = key[e] / nc;
    cols[e] = int64_t(key[e] - r * nc);
    atomicAdd(&counts[r], 1u);
  }
}

__global__ void canon_indptr_kernel(const unsigned int* __restrict__ counts, int64_t n_rows, int64_t* __restrict__ ptr) {
  // sequential prefix over rows by one block (rows of a single ingest call; the
  // scan is negligible next to the sort)
  __shared__ int64_t carry;
  if (threadIdx.x == 0) { carry = 0; ptr[0] = 0; }
  __syncthreads();
  typedef cub::BlockScan<int64_t, 256> Scan;
  __shared__ typename Scan::TempStorage tmp;
  for (int64_t base = 0; base < n_rows; base += 256) {
    const int64_t r = base + threadIdx.x;
    const int64_t c = r < n_rows ? int64_t(counts[r]) : 0;
    int64_t incl, total;
    Scan(tmp).InclusiveSum(c, incl, total);
    if (r < n_rows) ptr[r + 1] = carry + incl;
    __syncthreads();
    if (threadIdx.x == 0) carry += total;
    __syncthreads();
  }
}

}  // namespace sd

using namespace sd;

extern "C" {

int sd_segment_reduce(const void* values, int64_t n_values, const int64_t* bounds, int64_t n_segments, int dtype,
                      int ufunc, double identity, void* out, sd_stream_t stream) {
  if (n_segments < 0 || n_values < 0) { set_error("negative sizes"); return SD_E_INVALID; }
  if (ufunc < SD_UFUNC_ADD || ufunc > SD_UFUNC_MULTIPLY) { set_error("unsupported ufunc"); return SD_E_UNSUPPORTED; }
  if (n_segments == 0) return SD_OK;
  cudaStream_t st = as_stream(stream);
  return SD_DISPATCH_DTYPE(dtype, T, [&]() -> int {
    segment_reduce_kernel<T><<<grid_for(n_segments), 256, 0, st>>>(static_cast<const T*>(values), bounds, n_segments,
                                                                   ufunc, T(identity), static_cast<T*>(out));
    SD_LAUNCH_CHECK();
    return SD_OK;
  });
}

int sd_mix32(const int64_t* keys, int64_t n, uint64_t* out, sd_stream_t stream) {
  if (n <= 0) return SD_OK;
  mix32_kernel<<<grid_for(n), 256, 0, as_stream(stream)>>>(keys, n, out);
  SD_LAUNCH_CHECK();
  return SD_OK;
}

int sd_hash_build(const int64_t* keys, const double* values, int64_t n, int64_t capacity, int64_t* table_keys,
                  double* table_values, sd_stream_t stream) {
  if (capacity < 1) { set_error("capacity must be at least 1"); return SD_E_INVALID; }
  if (n >= capacity) { set_error("entries cannot fit the capacity"); return SD_E_INVALID; }
  hash_build_kernel<<<1, 256, 0, as_stream(stream)>>>(keys, values, n, capacity, table_keys, table_values);
  SD_LAUNCH_CHECK();
  return SD_OK;
}

int sd_hash_probe(const int64_t* table_keys, const double* table_values, int64_t capacity, const int64_t* queries,
                  int64_t n, double* out_values, uint8_t* out_found, sd_stream_t stream) {
  if (capacity < 1) { set_error("capacity must be at least 1"); return SD_E_INVALID; }
  if (n <= 0) return SD_OK;
  hash_probe_kernel<<<grid_for(n), 256, 0, as_stream(stream)>>>(table_keys, table_values, capacity, queries, n,
                                                                out_values, out_found);
  SD_LAUNCH_CHECK();
  return SD_OK;
}

int sd_semiring_apply(int semiring, double p, const double* x, const double* y, int64_t n, double* out,
                      sd_stream_t stream) {
  if (n <= 0) return SD_OK;
  cudaStream_t st = as_stream(stream);
  return SD_DISPATCH_SEMIRING(semiring, SR, [&]() -> int {
    semiring_apply_kernel<SR><<<grid_for(n), 256, 0, st>>>(x, y, n, p, out);
    SD_LAUNCH_CHECK();
    return SD_OK;
  });
}

int sd_dense_pairwise(const double* da, const double* db, int64_t m, int64_t n, int64_t k,
                      const sd_metric_desc* md, double* out, uint32_t* dev_flags, sd_stream_t stream) {
  if (!md || md->metric < 0 || md->metric > SD_M_MINKOWSKI) { set_error("unknown metric id"); return SD_E_INVALID; }
  if (m <= 0 || n <= 0) return SD_OK;
  dense_pairwise_kernel<<<grid_for(m * n), 256, 0, as_stream(stream)>>>(da, db, m, n, k, md->metric, md->p,
                                                                        md->strict, out, dev_flags);
  SD_LAUNCH_CHECK();
  return SD_OK;
}

int sd_canonicalize(int64_t n_rows, int64_t n_cols, int64_t nnz, const int64_t* indptr, const int64_t* indices,
                    const double* values, int64_t* out_indptr, int64_t* out_indices, double* out_values,
                    int64_t* out_nnz, sd_invalid* why, sd_stream_t stream) {
  cudaStream_t st = as_stream(stream);
  if (why) *why = sd_invalid{0, 0, 0, 0, 0};
  auto invalid = [&](int kind, int64_t row, int64_t column, int64_t value) {
    if (why) *why = sd_invalid{kind, 0, row, column, value};
    set_error("CSR validation failed");
    return SD_E_INVALID;
  };
  if (n_rows < 0 || n_cols < 0 || nnz < 0) { set_error("matrix dimensions must be non-negative"); return SD_E_INVALID; }
  *out_nnz = 0;
  // 1. validation, in the reference's order (sparse.py:135-170)
  Scratch first;
  SD_TRY(first.alloc(3 * sizeof(unsigned long long), st));
  SD_CUDA_TRY(cudaMemsetAsync(first.ptr, 0xff, 3 * sizeof(unsigned long long), st));
  canon_check_kernel<<<grid_for(std::max<int64_t>(n_rows + 1, nnz)), 256, 0, st>>>(
      indptr, n_rows, indices, nnz, n_cols, first.as<unsigned long long>());
  SD_LAUNCH_CHECK();
  unsigned long long h[3];
  int64_t ends[2];
  SD_CUDA_TRY(cudaMemcpyAsync(h, first.ptr, sizeof(h), cudaMemcpyDeviceToHost, st));
  SD_CUDA_TRY(cudaMemcpyAsync(&ends[0], indptr, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  SD_CUDA_TRY(cudaMemcpyAsync(&ends[1], indptr + n_rows, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  SD_CUDA_TRY(cudaStreamSynchronize(st));
  if (h[0] != ~0ull) {
    const int64_t pos = int64_t(h[0]);
    int64_t off = 0;
    SD_CUDA_TRY(cudaMemcpy(&off, indptr + pos, sizeof(int64_t), cudaMemcpyDeviceToHost));
    return invalid(SD_INVALID_NEGATIVE_OFFSET, std::max<int64_t>(0, std::min<int64_t>(pos, n_rows - 1)), 0, off);
  }
  if (ends[0] != 0) return invalid(SD_INVALID_INDPTR_START, 0, 0, ends[0]);
  if (h[1] != ~0ull) return invalid(SD_INVALID_DECREASING, int64_t(h[1]), 0, 0);
  if (ends[1] != nnz) return invalid(SD_INVALID_NNZ, 0, 0, ends[1]);
  if (h[2] != ~0ull) {
    Scratch loc;
    SD_TRY(loc.alloc(2 * sizeof(int64_t), st));
    canon_locate_kernel<<<1, 1, 0, st>>>(indptr, n_rows, indices, int64_t(h[2]), loc.as<int64_t>());
    SD_LAUNCH_CHECK();
    int64_t rc[2];
    SD_CUDA_TRY(cudaMemcpyAsync(rc, loc.ptr, sizeof(rc), cudaMemcpyDeviceToHost, st));
    SD_CUDA_TRY(cudaStreamSynchronize(st));
    return invalid(SD_INVALID_COLUMN, rc[0], rc[1], n_cols);
  }
  if (n_rows > 0) SD_CUDA_TRY(cudaMemsetAsync(out_indptr, 0, sizeof(int64_t) * (n_rows + 1), st));
  else SD_CUDA_TRY(cudaMemsetAsync(out_indptr, 0, sizeof(int64_t), st));
  if (nnz == 0) return SD_OK;
  // 2. stable sort by key = row * n_cols + column (sparse.py:172-176)
  Scratch keys, keys2, ord, ord2, tmp;
  SD_TRY(keys.alloc(sizeof(uint64_t) * nnz, st));
  SD_TRY(keys2.alloc(sizeof(uint64_t) * nnz, st));
  SD_TRY(ord.alloc(sizeof(int64_t) * nnz, st));
  SD_TRY(ord2.alloc(sizeof(int64_t) * nnz, st));
  canon_keys_kernel<<<grid_for(n_rows * 32), 256, 0, st>>>(indptr, n_rows, indices, n_cols, keys.as<uint64_t>(),
                                                           ord.as<int64_t>());
  SD_LAUNCH_CHECK();
  int end_bit = 1;
  while (end_bit < 64 && (uint64_t(1) << end_bit) <= uint64_t(n_rows) * uint64_t(std::max<int64_t>(1, n_cols)))
    ++end_bit;
  size_t tbytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tbytes, keys.as<uint64_t>(), keys2.as<uint64_t>(), ord.as<int64_t>(),
                                  ord2.as<int64_t>(), nnz, 0, end_bit, st);
  SD_TRY(tmp.alloc(tbytes, st));
  SD_CUDA_TRY(cub::DeviceRadixSort::SortPairs(tmp.ptr, tbytes, keys.as<uint64_t>(), keys2.as<uint64_t>(),
                                              ord.as<int64_t>(), ord2.as<int64_t>(), nnz, 0, end_bit, st));
  // 3. runs of equal keys, summed in input order; zeros dropped (sparse.py:177-185)
  Scratch head, starts, nruns, rkey, rval, keep, scratch, nkept, iota;
  SD_TRY(head.alloc(nnz, st));
  SD_TRY(starts.alloc(sizeof(int64_t) * nnz, st));
  SD_TRY(nruns.alloc(sizeof(int64_t), st));
  canon_heads_kernel<<<grid_for(nnz), 256, 0, st>>>(keys2.as<uint64_t>(), nnz, head.as<uint8_t>());
  SD_LAUNCH_CHECK();
  cub::CountingInputIterator<int64_t> count_it(0);
  size_t sbytes = 0;
  cub::DeviceSelect::Flagged(nullptr, sbytes, count_it, head.as<uint8_t>(), starts.as<int64_t>(), nruns.as<int64_t>(),
                             nnz, st);
  Scratch stmp;
  SD_TRY(stmp.alloc(sbytes, st));
  SD_CUDA_TRY(cub::DeviceSelect::Flagged(stmp.ptr, sbytes, count_it, head.as<uint8_t>(), starts.as<int64_t>(),
                                         nruns.as<int64_t>(), nnz, st));
  SD_TRY(rkey.alloc(sizeof(uint64_t) * nnz, st));
  SD_TRY(rval.alloc(sizeof(double) * nnz, st));
  SD_TRY(keep.alloc(nnz, st));
  SD_TRY(scratch.alloc(sizeof(double) * nnz, st));
  SD_CUDA_TRY(cudaMemsetAsync(keep.ptr, 0, nnz, st));
  canon_runs_kernel<<<grid_for(nnz), 256, 0, st>>>(keys2.as<uint64_t>(), ord2.as<int64_t>(), values,
                                                   starts.as<int64_t>(), nruns.as<int64_t>(), nnz, rkey.as<uint64_t>(),
                                                   rval.as<double>(), keep.as<uint8_t>(), scratch.as<double>());
  SD_LAUNCH_CHECK();
  // 4. compaction of the kept runs, then column ids and row pointers
  SD_TRY(nkept.alloc(sizeof(int64_t), st));
  Scratch ckey;
  SD_TRY(ckey.alloc(sizeof(uint64_t) * nnz, st));
  size_t cbytes = 0;
  cub::DeviceSelect::Flagged(nullptr, cbytes, rkey.as<uint64_t>(), keep.as<uint8_t>(), ckey.as<uint64_t>(),
                             nkept.as<int64_t>(), nnz, st);
  Scratch ctmp;
  SD_TRY(ctmp.alloc(cbytes, st));
  SD_CUDA_TRY(cub::DeviceSelect::Flagged(ctmp.ptr, cbytes, rkey.as<uint64_t>(), keep.as<uint8_t>(), ckey.as<uint64_t>(),
                                         nkept.as<int64_t>(), nnz, st));
  SD_CUDA_TRY(cub::DeviceSelect::Flagged(ctmp.ptr, cbytes, rval.as<double>(), keep.as<uint8_t>(), out_values,
                                         nkept.as<int64_t>(), nnz, st));
  Scratch counts;
  SD_TRY(counts.alloc(sizeof(unsigned int) * std::max<int64_t>(1, n_rows), st));
  SD_CUDA_TRY(cudaMemsetAsync(counts.ptr, 0, sizeof(unsigned int) * std::max<int64_t>(1, n_rows), st));
  canon_split_kernel<<<grid_for(nnz), 256, 0, st>>>(ckey.as<uint64_t>(), nkept.as<int64_t>(), n_cols, out_indices,
                                                    counts.as<unsigned int>());
  SD_LAUNCH_CHECK();
  canon_indptr_kernel<<<1, 256, 0, st>>>(counts.as<unsigned int>(), n_rows, out_indptr);
  SD_LAUNCH_CHECK();
  SD_CUDA_TRY(cudaMemcpyAsync(out_nnz, nkept.ptr, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  SD_CUDA_TRY(cudaStreamSynchronize(st));
  return SD_OK;
}

}  // extern "C"
