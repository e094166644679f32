// index.cuh — the J-blocked inverted index of B (isect.cu) and its dense
// heavy-row block for the hybrid path (hybrid.cu).
#pragma once
#include <mutex>
#include <vector>
#include "common.cuh"
#include "prep.cuh"

struct sd_index {
  // per-row statistics of the index rows, computed once per (metric, p) and
  // owned by the index (they are a property of B, like the postings)
  struct StatEntry {
    int metric;
    double p;
    void* buf;
    sd::Stats stats;
  };
  std::mutex mu;
  std::vector<StatEntry> stat_cache;
  int64_t n_rows = 0, n_cols = 0, nnz = 0;
  int tile = 0;
  int64_t n_tiles = 0;
  int dtype = 0;
  uint32_t* colptr = nullptr;  // [n_tiles * n_cols + 1]
  void* post = nullptr;        // [nnz] Posting<T> (row id within tile, value)
  // chebyshev (built on the first chebyshev call: ensure_cheb)
  void* post_cheb = nullptr;   // [nnz] postings with the value's rank in its B row (top-CHEB_K, else 255) in bits 16..23 of j
  void* topb = nullptr;        // [CHEB_K][n_rows] largest |values| per B row
  int64_t bytes = 0;
  // cosine: a copy of `post` with every value divided by its row's L2 norm,
  // built on the first cosine call (the epilogue then needs no index-row statistic)
  void* post_cos = nullptr;
  // probability that two random postings of one tile belong to the same row
  // (sum over tiles of sum d_j^2 / sum over tiles of (sum d_j)^2): why packing
  // several columns into one warp step does not pay on power-law indexes
  //
  double collide = 0.0;
  // hybrid path (hybrid.cu): rows of degree >= heavy_deg, densely as HT
  // (built on the first dot-family call: ensure_hybrid)
  // The common part (heavy ids, light rows) is built once; the dot-family
  // images (HT, the GEMM operand image) and the min-sum chunk pointers on the
  // first call of a metric that needs them.
  bool hybrid_tried = false;
  int64_t heavy_deg = 0, n_heavy = 0, hpad = 0;
  int32_t* hid = nullptr;  // [n_rows]: heavy id or -1
  int32_t* hrows = nullptr;  // [n_heavy] index row of each heavy id
  int32_t* hperm = nullptr;  // [n_heavy] heavy ids by descending degree (min-sum CTA balance)
  int32_t* lrows = nullptr;  // [n_light] the other rows, by descending degree
  int64_t n_light = 0;
  // dot family (C_MUL)
  bool dot_tried = false, dot_ready = false;
  void* ht = nullptr;      // [n_cols][hpad] T: HT[c][h] = B[heavy row h][c]
  void* hbf = nullptr;       // fp32: the heavy rows as the tcgen05 GEMM's bf16 operand image (dense_tc.cu)
  int hbf_planes = 0;        // 1 (values bf16-exact) or 2 (hi, lo)
  int64_t hbf_nkb = 0;       // its K blocks of 64 columns
  // min-sum (C_ABS, manhattan; only when every value of B is >= 0)
  bool ms_tried = false, ms_ready = false;
  int64_t* hchunk = nullptr;  // [n_heavy][ms_nch + 1] first CSR entry of each column chunk (hminsum.cu)
  int64_t ms_nch = 0;
  // dense-index mode (dense_tc.cu, built on the first eligible call): every
  // row as bf16 planes in the tensor-core operand layout
  void* dimg = nullptr;
  int dplanes = 0;      // 1 (values bf16-exact) or 2 (hi, lo)
  bool dints = false;   // every value a small integer (|v| <= 16)
  int64_t dnkb = 0;     // K blocks of 64 columns
};

namespace sd {
// hybrid.cu
enum HybridKind { HYB_DOT = 0, HYB_MINSUM = 1 };
int hybrid_index_build(const sd_csr* b, int dtype, sd_index* ix, int kind, cudaStream_t st);
// isect.cu: lazily built parts of the index (thread-safe, once)
int ensure_cheb(sd_index* ix, const sd_csr* b, cudaStream_t st);
int ensure_hybrid(sd_index* ix, const sd_csr* b, int kind, cudaStream_t st);
void hybrid_index_free(sd_index* ix);
}  // namespace sd
