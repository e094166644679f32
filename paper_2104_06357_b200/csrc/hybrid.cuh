// hybrid.cuh — per-call state of the dense path for heavy query rows (hybrid.cu).
#pragma once
#include "common.cuh"

struct sd_index;

namespace sd {

struct HybridState {
  cudaEvent_t fork = nullptr;  // the gather's side-stream fork / join (hybrid_prepare)
  cudaEvent_t join = nullptr;
  cudaStream_t main = nullptr;  // the caller's stream (scratch below is freed on it)
  cudaEvent_t cls = nullptr;         // classification done (side-stream plan / statistics start)
  cudaEvent_t dense_done = nullptr;  // the dense block's sums complete on the caller's stream
  cudaEvent_t stats_done = nullptr;  // deferred query statistics + work plan (isect_run) finished
  // the caller's stream waits for the side stream (before heavy_rows and
  // before any of this state's scratch is released on it)
  int wait(cudaStream_t st) {
    if (join && cudaStreamWaitEvent(st, join, 0) != cudaSuccess) return SD_E_CUDA;
    return SD_OK;
  }
  ~HybridState() {  // runs before the Scratch members free their buffers on `main`
    if (join && main) cudaStreamWaitEvent(main, join, 0);
    if (stats_done && main) cudaStreamWaitEvent(main, stats_done, 0);
    if (fork) cudaEventDestroy(fork);
    if (cls) cudaEventDestroy(cls);
    if (dense_done) cudaEventDestroy(dense_done);
    if (stats_done) cudaEventDestroy(stats_done);
    if (join) cudaEventDestroy(join);
  }
  int nhq = 0;          // heavy query rows of this call (ids 0..nhq-1)
  int cap = 0;          // most heavy query rows one call takes
  int gather_kind = 0;  // HYB_DOT / HYB_MINSUM (hybrid_gather)
  int64_t qpad = 0;     // nhq rounded up to 128
  Scratch qid;          // [m] heavy id of each query row or -1
  Scratch hq;           // [cap] query row of each heavy id
  Scratch count;        // [2]: heavy count, the queries' bf16-exactness flags
  Scratch gcount;       // work counter of the dense gather
  Scratch hqt;          // [n_cols][qpad] dense heavy query rows
  Scratch hq_img;       // the same rows as the tensor-core GEMM's bf16 operand image
  Scratch part;         // GEMM K-split partials
  Scratch dqh;          // [qpad][hpad] heavy query x heavy index row sums
  Scratch dlh;          // [n][qpad] light index row x heavy query sums
};

int64_t hybrid_threshold(int64_t n_cols);
cudaStream_t side_stream(int which);  // per-device side streams (nullptr if unavailable)
dim3 row_scatter_grid(int64_t nrows);  // grid of the per-row scatter kernels
// dense_tc.cu (fp32 tcgen05 bf16 GEMM): operand images of selected CSR rows,
// then P[z][q][h] (q < prow, h < ldp) = sum over split z's K blocks (`per` each)
int check_bf16_exact(const sd_csr* m, unsigned int* flag, cudaStream_t st);  // bit 0 inexact, bit 1 non-integer
int64_t dense_kblocks(int64_t n_cols);
size_t dense_image_bytes(int64_t nrows, int64_t nkb, int planes, int R);
int dense_image(const sd_csr* m, const int32_t* rows, int64_t nrows, int64_t nkb, int planes, int R, void* img,
                cudaStream_t st);
int dense_gemm_raw(const void* aimg, int pa, int64_t na, const void* bimg, int pb, int R, int64_t nq, int64_t nkb,
                   int64_t per, float* part, int64_t prow, int64_t ldp, cudaStream_t st);
bool hybrid_enabled();
bool hybrid_forced();
// classify query rows (heavy ids in hs.qid / hs.hq, count on the device) ...
int hybrid_classify(const sd_csr* a, const sd_index* ix, int dtype, int kind, HybridState& hs, cudaStream_t st);
// ... then read the count and run the dense block (GEMM or min-sum, kind =
// HYB_DOT / HYB_MINSUM) + gather for the heavy ones (no-op when none)
int hybrid_prepare(const sd_csr* a, const sd_csr* b, const sd_index* ix, int dtype, int kind, HybridState& hs,
                   cudaStream_t st);
// the dense gather (side stream); in shadow mode called by isect_run after the sweep's launch
int hybrid_gather(const sd_csr* a, const sd_csr* b, const sd_index* ix, int dtype, HybridState& hs, cudaStream_t st);
// hminsum.cu (manhattan): columns per chunk, index-side chunk pointers and
// value check, and dqh[q][h] = sum_c min(HQT+[c][q], B[heavy row h][c])
int64_t minsum_chunk_cols(int dtype);
int minsum_check_index(const sd_csr* b, int dtype, unsigned int* flag, cudaStream_t st);
int minsum_chunks(const sd_csr* b, int dtype, const int32_t* hrows, int64_t nh, int64_t nch, int64_t* hchunk,
                  cudaStream_t st);
int hminsum(const sd_index* ix, const sd_csr* b, int dtype, const void* hqt, int64_t n_cols, int64_t qpad,
            Scratch& part, void* dqh, cudaStream_t st);

}  // namespace sd
