// prep.cuh — internal entry points shared by the translation units.
#pragma once
#include "common.cuh"

namespace sd {

// rows per statistic slot, rounded so every slot is 32-byte aligned
inline int64_t stats_stride(int64_t n) { return (n + 3) & ~int64_t(3); }

struct Stats {  // per-row statistics the metric epilogue reads (metric.cuh layout)
  const void* s[3] = {nullptr, nullptr, nullptr};
};

// internal statistic kinds beyond sd_stat_kind: one-sided NAMM sums
//   S_A[i] = sum_c ⊗(a_ic, 0)   and   S_B[j] = sum_c ⊗(0, b_jc)
constexpr int STAT_ONESIDED_A = 16;
constexpr int STAT_ONESIDED_B = 17;


int row_stat(const sd_csr* m, int dtype, int kind, int semiring, double p, void* out,
             cudaStream_t st);
int csr_to_coo(const sd_csr* m, int64_t* rows, cudaStream_t st);
// ||row||_2 and 1/||row||_2 (0 for empty rows) in one pass: the fused cosine
// epilogue multiplies by reciprocals instead of dividing
int row_stat_l2_inv(const sd_csr* m, int dtype, void* l2, void* inv, cudaStream_t st);
// fused Chebyshev: per-row top-CHEB_K entries by |value|
constexpr int CHEB_K = 16;
int row_topk(const sd_csr* m, int dtype, uint8_t* rank, void* top, cudaStream_t st);
int check_nonnegative(const sd_csr* m, int dtype, uint32_t* flags, cudaStream_t st);
int sqrt_values(const sd_csr* m, int dtype, void* out, cudaStream_t st);
int fill(void* out, int64_t m, int64_t n, int64_t ldo, int dtype, double value, cudaStream_t st);

// engine.cu
int engine_pass(const sd_csr* a, const sd_csr* b, int dtype, int semiring, double p, int pass,
                const sd_strategy* strategy, void* out, int64_t ldo, sd_report* report,
                cudaStream_t st);
void reference_report(const int64_t* degrees, int64_t n_rows, const sd_strategy* strategy,
                      int64_t swept_nnz, sd_report* rep);

// epilogue.cu
int metric_stats(const sd_csr* m, int dtype, const sd_metric_desc* md, bool a_side, void* buf,
                 Stats* out, cudaStream_t st);
int64_t metric_stats_count(int metric);
int64_t metric_expand_stats_count(int metric);
int expand(void* dots, int64_t m, int64_t n, int64_t ldo, int dtype, const sd_metric_desc* md,
           int64_t n_cols, const Stats& sa, const Stats& sb, const void* miss,
           uint32_t* flags, cudaStream_t st);

// Device times of the phases of one call (sd_pairwise's phase_ms): events on
// the call's stream, read once at the end.
struct PhaseTimer {
  float* out;
  cudaStream_t st;
  cudaEvent_t ev[8] = {};
  bool used[4] = {false, false, false, false};
  PhaseTimer(float* o, cudaStream_t s) : out(o), st(s) {
    if (out)
      for (auto& e : ev) cudaEventCreate(&e);
  }
  ~PhaseTimer() {
    if (out)
      for (auto& e : ev) cudaEventDestroy(e);
  }
  void begin(int ph) { if (out) { cudaEventRecord(ev[2 * ph], st); used[ph] = true; } }
  void end(int ph) { if (out) cudaEventRecord(ev[2 * ph + 1], st); }
  int finish() {
    if (!out) return SD_OK;
    SD_CUDA_TRY(cudaStreamSynchronize(st));
    for (int ph = 0; ph < 4; ++ph) {
      out[ph] = 0.f;
      if (used[ph]) SD_CUDA_TRY(cudaEventElapsedTime(&out[ph], ev[2 * ph], ev[2 * ph + 1]));
    }
    return SD_OK;
  }
};
enum { PH_NORMS = 0, PH_PASS1 = 1, PH_PASS2 = 2, PH_EXPANSION = 3 };

int metric_semiring(int metric);
int default_tile(int dtype);
int index_build(const sd_csr* b, int dtype, int tile, sd_index** out, cudaStream_t st);
// defer_a: only lay out the query-side statistics (isect_run computes them)
int isect_stats(const sd_csr* a, const sd_csr* b, const sd_index* ix, int dtype, const sd_metric_desc* md,
                Scratch& sa_buf, Scratch& sb_buf, Stats* sa, Stats* sb, bool defer_a, cudaStream_t st);
// could isect_run take the hybrid path (it then computes deferred query statistics)?
bool isect_hybrid_eligible(const sd_index* ix, const sd_metric_desc* md, int topk);
int hybrid_kind(int metric);  // HYB_DOT, HYB_MINSUM or -1 (no dense heavy-row path)
// dense_tc.cu: dense-index mode (the whole matrix as one tensor-core GEMM)
bool dense_eligible(const sd_csr* b, const sd_metric_desc* md, int dtype, int topk);
int ensure_dense(sd_index* ix, const sd_csr* b, cudaStream_t st);
int dense_run(const sd_csr* a, const sd_csr* b, const sd_index* ix, const sd_metric_desc* md, const Stats& sa,
              const Stats& sb, void* out, int64_t ldo, uint32_t* flags, cudaStream_t st);
int isect_run(const sd_csr* a, const sd_csr* b, const sd_index* ix, int dtype, const sd_metric_desc* md,
              const Stats& sa, const Stats& sb, void* out, int64_t ldo, int topk, int64_t index_base,
              void* out_d, int64_t* out_i, uint32_t* flags, PhaseTimer* tm, bool a_stats_deferred,
              cudaStream_t st);
int topk_rows(const void* dist, int64_t m, int64_t n, int64_t ldd, int dtype, int k, int64_t base,
              void* od, int64_t* oi, cudaStream_t st);
int topk_rows_scatter(const void* dist, int64_t m, int64_t n, int64_t ldd, int dtype, int k, int64_t base,
                      const int32_t* rowmap, void* od, int64_t* oi, cudaStream_t st);
int topk_merge(const void* cd, const int64_t* ci, int64_t m, int lists, int k, int dtype, void* od,
               int64_t* oi, cudaStream_t st);
bool metric_two_pass(int metric);

}  // namespace sd
