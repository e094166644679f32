/*
 * semidist_b200.h — C ABI of the B200-native sparse semiring distance library
 * (libsemidist_b200.so, sm_100a).
 *
 * This is the drop-in boundary for the hot path of the reference package
 * `semidist` (/root/reference/pkg/src/semidist).  The reference is pure
 * Python/NumPy, so there is no native interface to replace: each entry point
 * below replaces one Python function of the reference and the Python shim
 * (paper_2104_06357_b200/_lib.py) binds it through ctypes exactly as a
 * maintainer of the reference would.
 *
 * Conventions
 *   - Every pointer inside an sd_csr and every output pointer is a DEVICE
 *     pointer; the caller owns all of them.  Scratch memory is taken
 *     stream-ordered (cudaMallocAsync) from the current device's pool and
 *     returned before the call's work completes on `stream`.
 *   - All work is enqueued on `stream`; functions return without
 *     synchronising unless documented otherwise.
 *   - Every entry returns an sd_status; sd_last_error() gives a thread-local
 *     message for the last non-OK status.
 *   - Deterministic: for a fixed input, device and dtype every output bit is
 *     reproducible run to run (no floating-point atomics anywhere).
 */
#ifndef SEMIDIST_B200_H
#define SEMIDIST_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SD_ABI_VERSION 1

#if defined(__GNUC__)
#define SD_API __attribute__((visibility("default")))
#else
#define SD_API
#endif

typedef void* sd_stream_t; /* a cudaStream_t (0 = legacy default stream) */

/* status codes -> Python exceptions (errors.py:4-76) */
typedef enum {
  SD_OK = 0,
  SD_E_DIM = 1,              /* DimensionMismatch            (errors.py:39)  */
  SD_E_DOMAIN_NEG = 2,       /* DomainError: negative input  (metrics.py:308-311) */
  SD_E_DOMAIN_RADICAND = 3,  /* DomainError: radicand < -tol (metrics.py:93-99) */
  SD_E_KL_UNCOVERED = 4,     /* DomainError: strict KL miss  (metrics.py:359-364) */
  SD_E_K_TOO_LARGE = 5,      /* KTooLarge                    (knn.py:56-57, 44-45) */
  SD_E_INVALID = 6,          /* ValueError: bad shape/argument */
  SD_E_UNSUPPORTED = 7,      /* NotImplementedError: semiring without a device functor */
  SD_E_CUDA = 8,             /* RuntimeError: CUDA failure */
  SD_E_DOMAIN_PARAM = 9      /* DomainError: minkowski p < 1 or non-finite (metrics.py:244-251) */
} sd_status;

typedef enum { SD_F32 = 0, SD_F64 = 1 } sd_dtype;

/* Canonical CSR (sparse.py:56-94) in HBM. */
typedef struct {
  int64_t n_rows;
  int64_t n_cols;
  int64_t nnz;
  const int64_t* indptr;  /* [n_rows+1], indptr[0] == 0 */
  const int32_t* indices; /* [nnz], strictly ascending per row */
  const void* values;     /* [nnz] of sd_dtype, no stored zeros */
} sd_csr;

/* Semirings: the fixed functor set of semiring.py:76-119 plus the KL
 * miss counter of metrics.py:303-305.  Values follow that order. */
typedef enum {
  SD_SR_DOT = 0,          /* x*y, +, 0, annihilating         semiring.py:76-78  */
  SD_SR_MIN_PLUS = 1,     /* x+y, min, +inf                  semiring.py:81-83  */
  SD_SR_ABS_DIFF = 2,     /* |x-y|, +, 0                     semiring.py:86-87  */
  SD_SR_ABS_DIFF_POW = 3, /* |x-y|^p, +, 0                   semiring.py:90-97  */
  SD_SR_ABS_DIFF_MAX = 4, /* |x-y|, max, 0                   semiring.py:100-101 */
  SD_SR_CANBERRA = 5,     /* |x-y|/(|x|+|y|), +, 0           semiring.py:104-106 */
  SD_SR_MISMATCH = 6,     /* x!=y, +, 0                      semiring.py:109-110 */
  SD_SR_JS_TERM = 7,      /* x log(x/mu)+y log(y/mu), +, 0   semiring.py:113-115 */
  SD_SR_KL_TERM = 8,      /* x log(x/y), +, 0, annihilating  semiring.py:118-119 */
  SD_SR_MISS_COUNT = 9    /* 1, +, 0                         metrics.py:303-305 */
} sd_semiring;

/* Metrics in METRIC_NAMES order (metrics.py:31-35). */
typedef enum {
  SD_M_CORRELATION = 0, SD_M_COSINE = 1, SD_M_DICE = 2, SD_M_DOT = 3,
  SD_M_EUCLIDEAN = 4, SD_M_HELLINGER = 5, SD_M_JACCARD = 6, SD_M_KL = 7,
  SD_M_RUSSELRAO = 8, SD_M_CANBERRA = 9, SD_M_CHEBYSHEV = 10,
  SD_M_HAMMING = 11, SD_M_JENSENSHANNON = 12, SD_M_MANHATTAN = 13,
  SD_M_MINKOWSKI = 14
} sd_metric;

/* Execution strategy (engine.py:53-77). */
typedef enum {
  SD_STRAT_NAIVE = 0, /* Alg. 2: per-pair sorted merge       engine.py:270-311 */
  SD_STRAT_DENSE = 1, /* Alg. 3, dense SMEM row accumulator  engine.py:195-267 */
  SD_STRAT_HASH = 2,  /* Alg. 3, SMEM open-addressing table + chunking          */
  SD_STRAT_AUTO = 3   /* per-row choice by degree against the SMEM budget       */
} sd_strategy_kind;

typedef struct {
  int32_t kind;                 /* sd_strategy_kind */
  int32_t accumulator_capacity; /* hash only; chunk budget = floor(load*capacity) */
  double max_load_factor;       /* (0, 1], default 0.5 */
} sd_strategy;

/* WorkspaceReport (engine.py:80-99). */
typedef struct {
  int64_t peak_accumulator_entries;
  int64_t workspace_elements;
  int64_t chunks_executed;
} sd_report;

/* Metric request for the fused entry points. */
typedef struct {
  int32_t metric;          /* sd_metric */
  int32_t strict;          /* KL: 1 = uncovered pair -> SD_FLAG_KL_UNCOVERED, 0 = saturate */
  double p;                /* minkowski order */
  int32_t pre_transformed; /* 1: a, b (and index) already carry the metric's value
                              transform (sqrt for hellinger, metrics.py:332-338) */
  int32_t stages;          /* sd_expand only: 0 expansion + post-scale, 1 expansion only
                              (MetricSpec.expansion), 2 post-scale only (MetricSpec.post_scale) */
} sd_metric_desc;

/* Row statistic kinds for sd_row_stat (sparse.py:257-273). */
typedef enum {
  SD_STAT_L0 = 0, SD_STAT_L1 = 1, SD_STAT_L2 = 2, SD_STAT_L2SQ = 3, SD_STAT_SUM = 4
} sd_stat_kind;

/* Device flag bits written by the fused kernels (one uint32 word). */
#define SD_FLAG_RADICAND 0x1u
#define SD_FLAG_KL_UNCOVERED 0x2u
#define SD_FLAG_NEGATIVE 0x4u

typedef struct sd_index sd_index; /* opaque J-blocked inverted index of B */

/* Tuning knobs (experiments, tests).  Each knob's default is read ONCE,
 * when the library loads, from the environment variable named in the
 * comment; sd_tune overrides it for the rest of the process.  No entry
 * point reads the environment per call. */
typedef enum {
  SD_TUNE_TILE = 0,            /* SD_TILE: index tile rows (fp32; fp64 halves), 0 = default */
  SD_TUNE_ISECT_PLAN = 1,      /* SD_ISECT_PLAN: 1 = tile-major work items */
  SD_TUNE_COS_RAW = 2,         /* SD_COS_RAW: 1 = cosine over unscaled postings */
  SD_TUNE_ISECT_DEBUG = 3,     /* SD_ISECT_DEBUG: 1 skip sweep, 2 skip epilogue (timing only) */
  SD_TUNE_ISECT_BAND = 4,      /* SD_ISECT_BAND: tiles per L2 band, 0 = automatic */
  SD_TUNE_ISECT_L2_DIV = 5,    /* SD_ISECT_L2_DIV: band = L2 / div, 0 = automatic */
  SD_TUNE_HEAVY_DEG = 6,       /* SD_HEAVY_DEG: heavy-row degree threshold, 0 = n_cols/32 */
  SD_TUNE_HYBRID = 7,          /* SD_HYBRID: 0 off, 1 automatic, 2 forced on small indexes */
  SD_TUNE_HYBRID_MAX_MB = 8,   /* SD_HYBRID_MAX_MB: largest heavy-row image (MiB; fp32 bf16 planes, fp64 HT) */
  SD_TUNE_HYBRID_MAX_QUERIES = 9, /* SD_HYBRID_MAX_QUERIES: heavy query rows per call */
  SD_TUNE_HGEMM = 10,          /* SD_HGEMM: fp64 heavy block, 1 = CUDA-core DFMA tile instead of DMMA (fp32: tcgen05) */
  SD_TUNE_DENSE = 11,          /* SD_DENSE: dense-index tensor-core mode, 0 off, 1 automatic, 2 forced */
  SD_TUNE_DENSE_MAX_MB = 12,   /* SD_DENSE_MAX_MB: largest dense index image (MiB) */
  SD_TUNE_GATHER_SHADOW = 13,  /* SD_GATHER_SHADOW (experiment): 1 = hybrid gather co-resident with the sweep
                                  (one 128-thread block per SM, sweep capped at 12 warps); default 0 = gather on
                                  every SM first (C2 cosine 1.98 ms vs 3.66 ms co-resident) */
  SD_TUNE_GATHER_BLOCKS = 14,  /* SD_GATHER_BLOCKS: hybrid gather 256-thread blocks per SM, 0 = as many as fit */
  SD_TUNE_COUNT = 15
} sd_tune_knob;

/* ---------------------------------------------------------------- misc */
SD_API int sd_version(void);
/* Set knob `knob` to `value`; the old value goes to *previous (nullable). */
SD_API int sd_tune(int knob, int64_t value, int64_t* previous);
SD_API const char* sd_last_error(void);
/* Cumulative number of kernels this library has launched in the process. */
SD_API uint64_t sd_launch_count(void);
/* Largest dynamic shared memory per block on `device` (opt-in), bytes. */
SD_API int sd_smem_budget(int device, int64_t* bytes);

/* ---------------------------------------------------------------- prep */
/* Per-row statistic (row_norms / row_signed_sums, sparse.py:257-273). */
SD_API int sd_row_stat(const sd_csr* m, int dtype, int kind, void* out, sd_stream_t stream);
/* CSR -> COO row ids (coo_row_ids, sparse.py:78-81). */
SD_API int sd_csr_to_coo(const sd_csr* m, int64_t* rows_out, sd_stream_t stream);
/* Sets SD_FLAG_NEGATIVE in *dev_flags if any value < 0 (metrics.py:308-311). */
SD_API int sd_check_nonnegative(const sd_csr* m, int dtype, uint32_t* dev_flags, sd_stream_t stream);
/* values_out[e] = sqrt(values[e]) (Hellinger value transform, metrics.py:205-207). */
SD_API int sd_sqrt_values(const sd_csr* m, int dtype, void* values_out, sd_stream_t stream);
/* out[i, j] = value for an m x n row-major block with leading dim ldo
 * (allocate_output, engine.py:167-169). */
SD_API int sd_fill(void* out, int64_t m, int64_t n, int64_t ldo, int dtype, double value,
            sd_stream_t stream);

/* -------------------------------------------------------------- engine */
/* One sweep of the generalized pairwise SpMV into a caller-initialised
 * m x n output (row-major, leading dimension ldo):
 *   pass 1 == pairwise_spmv_pass1 (engine.py:314-333)
 *   pass 2 == pairwise_spmv_pass2 (engine.py:336-353, zero-mask complement)
 * `p` is the exponent for SD_SR_ABS_DIFF_POW.  `report` (host, may be NULL)
 * receives the WorkspaceReport of this pass.  Synchronises `stream` only to
 * read A/B row degrees for the staging plan. */
SD_API int sd_pass(const sd_csr* a, const sd_csr* b, int dtype, int semiring, double p,
            int pass, const sd_strategy* strategy, void* out, int64_t ldo,
            sd_report* report, sd_stream_t stream);

/* ---------------------------------------------------------- fast path */
/* Build the J-blocked inverted index of B (B^T split into row tiles of
 * `tile_rows` index rows).  tile_rows = 0 picks the default for dtype. */
SD_API int sd_index_build(const sd_csr* b, int dtype, int tile_rows, sd_index** out,
                   sd_stream_t stream);
SD_API int sd_index_free(sd_index* index);
SD_API int64_t sd_index_bytes(const sd_index* index);
SD_API int sd_index_tile_rows(const sd_index* index);
/* Index rows held densely for the hybrid path (heavy query rows of dot-family
 * metrics, hybrid.cu); 0 when the index has no heavy-row block. */
SD_API int64_t sd_index_heavy_rows(const sd_index* index);
/* Dense blocks built so far: bit 0 the dot family's heavy-row block (HT +
 * tensor-core operand image), bit 1 manhattan's min-sum chunk pointers
 * (hminsum.cu; only for an index without negative values), bit 2 the
 * dense-index image (dense_tc.cu), bit 3 set when that image holds two bf16
 * planes (hi, lo), bit 4 when every index value is a small integer.  Same
 * reference role as above. */
SD_API int sd_index_hybrid_blocks(const sd_index* index);

/* Full distance matrix for one catalog metric (pairwise_distances,
 * metrics.py:320-381): out[i*ldo + j] for i < a.n_rows, j < b.n_rows.
 * `index` may be NULL (built internally) and is only used by the
 * intersection path.  `strategy` NULL or kind AUTO selects the fused
 * intersection path for (+)-reduced metrics and the two-pass engine for
 * chebyshev; DENSE/HASH/NAIVE force the engine.  Domain violations set bits
 * in *dev_flags (device word, caller zeroes it).  `report` (host, nullable)
 * receives the engine's WorkspaceReport.  `phase_ms` (host, nullable, 4
 * floats) receives device times of the phases {norms, pass1, pass2,
 * expansion} of metrics.py:325-374 measured with CUDA events; passing it
 * synchronises `stream`.  On the fused path "pass1" is the intersection
 * kernel alone, "pass2" the one-sided NAMM sums that replace the complement
 * sweep or, for dot-family metrics, the dense path of the
 * heavy query rows (GEMM + gather, hybrid.cu), and "expansion" the epilogue
 * of those heavy rows. */
SD_API int sd_pairwise(const sd_csr* a, const sd_csr* b, const sd_index* index, int dtype,
                const sd_metric_desc* metric, const sd_strategy* strategy,
                void* out, int64_t ldo, uint32_t* dev_flags, sd_report* report,
                float* phase_ms, sd_stream_t stream);

/* Element-wise expansion + post-scale over a dots matrix in place
 * (expansion_apply, metrics.py:287-300).  stats_a/stats_b are the per-row
 * statistics the metric needs, in the order documented in DESIGN.md §4. */
SD_API int sd_expand(void* dots, int64_t m, int64_t n, int64_t ldo, int dtype,
              const sd_metric_desc* metric, int64_t n_cols,
              const void* const* stats_a, const void* const* stats_b,
              uint32_t* dev_flags, sd_stream_t stream);

/* ----------------------------------------------------------------- kNN */
/* k nearest index rows per query with fused top-k (kneighbors,
 * knn.py:50-94): ascending distance, ties -> lower index.  Indices written
 * are index_base + local row.  k <= 128. */
SD_API int sd_knn(const sd_csr* queries, const sd_csr* index_rows, const sd_index* index,
           int dtype, const sd_metric_desc* metric, int k, int64_t index_base,
           void* out_dist, int64_t* out_idx, uint32_t* dev_flags, sd_stream_t stream);
/* Row-wise top-k over a dense m x n distance block (select_topk, knn.py:41-47). */
SD_API int sd_topk_rows(const void* dist, int64_t m, int64_t n, int64_t ldd, int dtype, int k,
                 int64_t index_base, void* out_dist, int64_t* out_idx,
                 sd_stream_t stream);
/* Merge `lists` sorted candidate lists of length k per query (layout
 * [lists][m][k], e.g. after an all-gather of per-shard results) into the
 * global top-k with the same (distance, index) order. */
SD_API int sd_topk_merge(const void* cand_dist, const int64_t* cand_idx, int64_t m, int lists,
                  int k, int dtype, void* out_dist, int64_t* out_idx, sd_stream_t stream);

/* ------------------------------------------- drop-in utilities (device) */
/* numpy ufuncs segment_reduce supports (sparse.py:31-53). */
typedef enum {
  SD_UFUNC_ADD = 0, SD_UFUNC_MAXIMUM = 1, SD_UFUNC_MINIMUM = 2, SD_UFUNC_MULTIPLY = 3
} sd_ufunc;
/* out[s] = ufunc.reduce(values[bounds[s]:bounds[s+1]]), identity for empty
 * segments (segment_reduce, sparse.py:31-53), with numpy's association:
 * add.reduceat is v[0] + pairwise_sum(v[1:]), so results are BITWISE those
 * of the reference.  The caller has checked that bounds tile the values. */
SD_API int sd_segment_reduce(const void* values, int64_t n_values, const int64_t* bounds,
                      int64_t n_segments, int dtype, int ufunc, double identity, void* out,
                      sd_stream_t stream);
/* mix32 of the low 32 bits of each key (hashtable.py:21-29). */
SD_API int sd_mix32(const int64_t* keys, int64_t n, uint64_t* out, sd_stream_t stream);
/* HashAccumulator.build (hashtable.py:43-63): table_keys/values[capacity],
 * empty slots hold INT64_MAX (EMPTY_SLOT, hashtable.py:12); n < capacity. */
SD_API int sd_hash_build(const int64_t* keys, const double* values, int64_t n, int64_t capacity,
                  int64_t* table_keys, double* table_values, sd_stream_t stream);
/* HashAccumulator.probe_many (hashtable.py:80-106). */
SD_API int sd_hash_probe(const int64_t* table_keys, const double* table_values, int64_t capacity,
                  const int64_t* queries, int64_t n, double* out_values, uint8_t* out_found,
                  sd_stream_t stream);
/* out[i] = ⊗(x[i], y[i]) of a semiring (Semiring.product_op, semiring.py:36-119). */
SD_API int sd_semiring_apply(int semiring, double p, const double* x, const double* y, int64_t n,
                      double* out, sd_stream_t stream);
/* Dense brute-force arbiter (oracle.py:35-190): out[i*n+j] = the textbook
 * formula of `metric` over all k columns of dense rows da[i], db[j]; the
 * engine-independent check behind `verify` (verification.py:54-71). */
SD_API int sd_dense_pairwise(const double* da, const double* db, int64_t m, int64_t n, int64_t k,
                      const sd_metric_desc* metric, double* out, uint32_t* dev_flags,
                      sd_stream_t stream);

/* Why sd_canonicalize rejected its input (sparse.py:135-170 error order). */
typedef enum {
  SD_INVALID_NONE = 0,
  SD_INVALID_NEGATIVE_OFFSET = 1, /* NegativeOffset(row, offset=value)        */
  SD_INVALID_INDPTR_START = 2,    /* NonMonotonicIndptr(0): indptr[0] = value  */
  SD_INVALID_DECREASING = 3,      /* NonMonotonicIndptr(row)                   */
  SD_INVALID_NNZ = 4,             /* ValueError: indptr[-1] = value != nnz      */
  SD_INVALID_COLUMN = 5           /* IndexOutOfBounds(row, column, n_cols=value) */
} sd_invalid_kind;

typedef struct {
  int32_t kind; /* sd_invalid_kind */
  int32_t pad;
  int64_t row;
  int64_t column;
  int64_t value;
} sd_invalid;

/* validate_and_canonicalize (sparse.py:135-202) on device: validates a raw
 * CSR triple (int64 indptr/indices, float64 values) in the reference's error
 * order (status SD_E_INVALID, details in *why), then sorts each row's
 * columns (stable), sums duplicates in input order with numpy's reduceat
 * association (bitwise the reference's values), drops the zeros and writes
 * the canonical CSR into out_* (capacity nnz entries; out_indptr n_rows+1).
 * *out_nnz (host) receives the canonical entry count; synchronises `stream`. */
SD_API int sd_canonicalize(int64_t n_rows, int64_t n_cols, int64_t nnz, const int64_t* indptr,
                    const int64_t* indices, const double* values, int64_t* out_indptr,
                    int64_t* out_indices, double* out_values, int64_t* out_nnz, sd_invalid* why,
                    sd_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* SEMIDIST_B200_H */
