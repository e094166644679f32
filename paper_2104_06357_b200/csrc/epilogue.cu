// epilogue.cu — metric table, per-row statistics for a metric, and the
// element-wise expansion kernel (expansion_apply, metrics.py:287-300; the
// expansion/post-scale phase of pairwise_distances_detail, metrics.py:368-374).
#include "common.cuh"
#include "metric.cuh"
#include "prep.cuh"

namespace sd {

// Table 1 (metrics.py:183-270): metric -> semiring of its engine passes.
int metric_semiring(int metric) {
  switch (metric) {
    case SD_M_KL: return SD_SR_KL_TERM;
    case SD_M_CANBERRA: return SD_SR_CANBERRA;
    case SD_M_CHEBYSHEV: return SD_SR_ABS_DIFF_MAX;
    case SD_M_HAMMING: return SD_SR_MISMATCH;
    case SD_M_JENSENSHANNON: return SD_SR_JS_TERM;
    case SD_M_MANHATTAN: return SD_SR_ABS_DIFF;
    case SD_M_MINKOWSKI: return SD_SR_ABS_DIFF_POW;
    default: return SD_SR_DOT;
  }
}

bool metric_two_pass(int metric) { return is_namm(metric); }

// number of per-row statistic arrays the epilogue reads for a metric
int64_t metric_stats_count(int metric) {
  switch (metric) {
    case SD_M_CORRELATION: case SD_M_COSINE: return 2;
    case SD_M_DICE: case SD_M_EUCLIDEAN: case SD_M_JACCARD: case SD_M_KL: return 1;
    default: return is_namm(metric) ? 1 : 0;
  }
}

// statistics the element-wise expansion (sd_expand) reads
int64_t metric_expand_stats_count(int metric) {
  return metric == SD_M_COSINE ? 1 : metric_stats_count(metric);
}

// Fill `buf` (n_rows * metric_stats_count values) with the statistics
// `expand_cell` expects for this side (metrics.py:314-317).  For NAMM metrics
// the single statistic is the one-sided sum used by the fused path.
int metric_stats(const sd_csr* m, int dtype, const sd_metric_desc* md, bool a_side, void* buf,
                 Stats* out, cudaStream_t st) {
  const size_t es = dtype == SD_F64 ? 8 : 4;
  char* b = static_cast<char*>(buf);
  const int64_t n = m->n_rows;
  // slots start on 32-byte boundaries: the fused epilogue reads them 4 values at a time
  auto slot = [&](int q) { return static_cast<void*>(b + size_t(q) * size_t(stats_stride(n)) * es); };
  switch (md->metric) {
    case SD_M_CORRELATION:
      SD_TRY(row_stat(m, dtype, SD_STAT_SUM, 0, 0.0, slot(0), st));
      SD_TRY(row_stat(m, dtype, SD_STAT_L2SQ, 0, 0.0, slot(1), st));
      out->s[0] = slot(0); out->s[1] = slot(1);
      return SD_OK;
    case SD_M_COSINE:  // s1 = 1/l2 for the fused epilogue
      SD_TRY(row_stat_l2_inv(m, dtype, slot(0), slot(1), st));
      out->s[0] = slot(0); out->s[1] = slot(1);
      return SD_OK;
    case SD_M_DICE: case SD_M_JACCARD: case SD_M_KL:
      SD_TRY(row_stat(m, dtype, SD_STAT_L0, 0, 0.0, slot(0), st));
      out->s[0] = slot(0);
      return SD_OK;
    case SD_M_EUCLIDEAN:
      SD_TRY(row_stat(m, dtype, SD_STAT_L2SQ, 0, 0.0, slot(0), st));
      out->s[0] = slot(0);
      return SD_OK;
    default:
      if (is_namm(md->metric)) {
        SD_TRY(row_stat(m, dtype, a_side ? STAT_ONESIDED_A : STAT_ONESIDED_B,
                        metric_semiring(md->metric), md->p, slot(0), st));
        out->s[0] = slot(0);
      }
      return SD_OK;
  }
}

template <typename T>
__global__ void expand_kernel(T* __restrict__ d, int64_t m, int64_t n, int64_t ldo, int metric,
                              const T* __restrict__ a0, const T* __restrict__ a1,
                              const T* __restrict__ b0, const T* __restrict__ b1,
                              const T* __restrict__ miss, int strict, int stage, T k, T p, uint32_t* flags) {
  uint32_t f = 0;
  const int64_t total = m * n;
  for (int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; q < total;
       q += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = q / n, j = q - i * n;
    T* cell = d + i * ldo + j;
    if (miss) {  // KL coverage from the miss-count pass (metrics.py:352-366)
      if (miss[i * ldo + j] > T(0)) {
        if (strict) f |= SD_FLAG_KL_UNCOVERED;
        *cell = Num<T>::big();
        continue;
      }
    }
    *cell = expand_stage<T>(metric, stage, *cell, a0 ? a0[i] : T(0), a1 ? a1[i] : T(0), b0 ? b0[j] : T(0),
                            b1 ? b1[j] : T(0), k, p, f);
  }
  f = __reduce_or_sync(0xffffffffu, f);
  if (f && lane_id() == 0) atomicOr(flags, f);
}

int expand(void* dots, int64_t m, int64_t n, int64_t ldo, int dtype, const sd_metric_desc* md,
           int64_t n_cols, const Stats& sa, const Stats& sb, const void* miss, uint32_t* flags,
           cudaStream_t st) {
  if (m == 0 || n == 0) return SD_OK;
  return SD_DISPATCH_DTYPE(dtype, T, [&]() -> int {
    const int blocks = int(std::min<int64_t>((m * n + 255) / 256, int64_t(num_sms()) * 16));
    expand_kernel<T><<<blocks, 256, 0, st>>>(
        static_cast<T*>(dots), m, n, ldo, md->metric, static_cast<const T*>(sa.s[0]),
        static_cast<const T*>(sa.s[1]), static_cast<const T*>(sb.s[0]), static_cast<const T*>(sb.s[1]),
        static_cast<const T*>(miss), md->strict, md->stages, T(n_cols), T(md->p), flags);
    SD_LAUNCH_CHECK();
    return SD_OK;
  });
}

}  // namespace sd
