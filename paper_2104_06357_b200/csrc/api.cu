// api.cu — extern "C" entry points of libsemidist_b200.so (include/semidist_b200.h).
//
// Orchestration mirrors pairwise_distances_detail (metrics.py:320-375) and
// kneighbors_detail (knn.py:50-82); every piece of arithmetic runs in the
// kernels of prep.cu / engine.cu / isect.cu / epilogue.cu / topk.cu.
#include <atomic>
#include <cstdlib>
#include <cmath>
#include <mutex>
#include <string>
#include <vector>
#include "common.cuh"
#include "metric.cuh"
#include "prep.cuh"
#include "index.cuh"
#include "hybrid.cuh"
#include "index.cuh"
#include "hybrid.cuh"

namespace sd {

static thread_local std::string g_error;
void set_error(const std::string& msg) { g_error = msg; }
static std::atomic<uint64_t> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

// Tuning knobs: environment defaults read once (first use), sd_tune afterwards.
static std::atomic<int64_t> g_knobs[SD_TUNE_COUNT];
static std::once_flag g_knobs_once;

static void init_knobs() {
  auto env = [](const char* name, int64_t dflt) -> int64_t {
    const char* e = getenv(name);
    return e ? atoll(e) : dflt;
  };
  g_knobs[SD_TUNE_TILE] = env("SD_TILE", 0);
  g_knobs[SD_TUNE_ISECT_PLAN] = env("SD_ISECT_PLAN", 0);
  g_knobs[SD_TUNE_COS_RAW] = getenv("SD_COS_RAW") ? 1 : 0;
  g_knobs[SD_TUNE_ISECT_DEBUG] = env("SD_ISECT_DEBUG", 0);
  g_knobs[SD_TUNE_ISECT_BAND] = env("SD_ISECT_BAND", 0);
  g_knobs[SD_TUNE_ISECT_L2_DIV] = env("SD_ISECT_L2_DIV", 0);
  g_knobs[SD_TUNE_HEAVY_DEG] = env("SD_HEAVY_DEG", 0);
  g_knobs[SD_TUNE_HYBRID] = env("SD_HYBRID", 1);
  g_knobs[SD_TUNE_HYBRID_MAX_MB] = env("SD_HYBRID_MAX_MB", 8192);
  g_knobs[SD_TUNE_HYBRID_MAX_QUERIES] = env("SD_HYBRID_MAX_QUERIES", 1024);
  g_knobs[SD_TUNE_DENSE] = env("SD_DENSE", 1);
  g_knobs[SD_TUNE_DENSE_MAX_MB] = env("SD_DENSE_MAX_MB", 32768);
  g_knobs[SD_TUNE_GATHER_SHADOW] = env("SD_GATHER_SHADOW", 0);
  g_knobs[SD_TUNE_GATHER_BLOCKS] = env("SD_GATHER_BLOCKS", 0);
  const char* g = getenv("SD_HGEMM");
  g_knobs[SD_TUNE_HGEMM] = !g ? 0 : std::string(g) == "simt" ? 1 : std::string(g) == "mma" ? 2 : atoll(g);
}

int64_t knob(int k) {
  std::call_once(g_knobs_once, init_knobs);
  return (k >= 0 && k < SD_TUNE_COUNT) ? g_knobs[k].load(std::memory_order_relaxed) : 0;
}

// device attributes, cached per device (queried on every launch otherwise)
static int device_attr(cudaDeviceAttr attr, int fallback) {
  constexpr int kMaxDev = 64;
  static std::atomic<int> cache[3][kMaxDev];
  const int slot = attr == cudaDevAttrMultiProcessorCount ? 0
                 : attr == cudaDevAttrMaxSharedMemoryPerBlockOptin ? 1 : 2;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDev) return fallback;
  int v = cache[slot][dev].load(std::memory_order_relaxed);
  if (v > 0) return v;
  if (slot == 0) {
    // scratch comes from the device's default stream-ordered pool: keep freed
    // blocks in the pool across synchronisations instead of returning them to
    // the driver (each call's large scratch would otherwise be re-mapped)
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t keep = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
  }
  if (cudaDeviceGetAttribute(&v, attr, dev) != cudaSuccess || v <= 0) return fallback;
  cache[slot][dev].store(v, std::memory_order_relaxed);
  return v;
}

int num_sms() { return device_attr(cudaDevAttrMultiProcessorCount, 148); }
int64_t smem_optin_bytes() { return device_attr(cudaDevAttrMaxSharedMemoryPerBlockOptin, 227 * 1024); }
int64_t l2_bytes() { return device_attr(cudaDevAttrL2CacheSize, 126 * 1024 * 1024); }

static int check_csr(const sd_csr* m, const char* what) {
  if (!m) { set_error(std::string(what) + " is NULL"); return SD_E_INVALID; }
  if (m->n_rows < 0 || m->n_cols < 0 || m->nnz < 0) { set_error(std::string(what) + " has negative dims"); return SD_E_INVALID; }
  if (m->n_cols >= (int64_t(1) << 31)) { set_error(std::string(what) + ": n_cols must fit int32"); return SD_E_INVALID; }
  if (m->n_rows > 0 && !m->indptr) { set_error(std::string(what) + ".indptr is NULL"); return SD_E_INVALID; }
  return SD_OK;
}

static int check_metric(const sd_metric_desc* md) {
  if (!md || md->metric < 0 || md->metric > SD_M_MINKOWSKI) { set_error("unknown metric id"); return SD_E_INVALID; }
  if (md->metric == SD_M_MINKOWSKI && (!std::isfinite(md->p) || md->p < 1.0)) {
    set_error("minkowski requires finite p >= 1");
    return SD_E_DOMAIN_PARAM;
  }
  return SD_OK;
}

static bool needs_nonneg(int metric) {
  return metric == SD_M_KL || metric == SD_M_JENSENSHANNON || metric == SD_M_HELLINGER;
}

// Apply the metric's value transform (hellinger: sqrt, metrics.py:332-338) into scratch.
static int transformed(const sd_csr* in, int dtype, const sd_metric_desc* md, sd_csr* out, Scratch& buf,
                       cudaStream_t st) {
  *out = *in;
  if (md->metric != SD_M_HELLINGER || md->pre_transformed || in->nnz == 0) return SD_OK;
  SD_TRY(buf.alloc((dtype == SD_F64 ? 8 : 4) * size_t(in->nnz), st));
  SD_TRY(sqrt_values(in, dtype, buf.ptr, st));
  out->values = buf.ptr;
  return SD_OK;
}

// Device time of the phases {norms, pass1, pass2, expansion} (metrics.py:325-374).


// The two-pass engine route of pairwise_distances_detail (metrics.py:340-375).
static int engine_pairwise(const sd_csr* a, const sd_csr* b, int dtype, const sd_metric_desc* md,
                           const sd_strategy* strat, void* out, int64_t ldo, uint32_t* flags,
                           sd_report* report, PhaseTimer& tm, cudaStream_t st) {
  const int sr = metric_semiring(md->metric);
  SD_TRY(fill(out, a->n_rows, b->n_rows, ldo, dtype, 0.0, st));
  sd_report r1{}, r2{};
  Stats sa, sb;
  Scratch sabuf, sbbuf;
  const int64_t ns = metric_stats_count(md->metric);
  const size_t es = dtype == SD_F64 ? 8 : 4;
  tm.begin(PH_NORMS);
  if (ns > 0 && !is_namm(md->metric) && md->metric != SD_M_KL) {
    SD_TRY(sabuf.alloc(es * ns * stats_stride(std::max<int64_t>(1, a->n_rows)), st));
    SD_TRY(sbbuf.alloc(es * ns * stats_stride(std::max<int64_t>(1, b->n_rows)), st));
    SD_TRY(metric_stats(a, dtype, md, true, sabuf.ptr, &sa, st));
    SD_TRY(metric_stats(b, dtype, md, false, sbbuf.ptr, &sb, st));
  }
  tm.end(PH_NORMS);
  tm.begin(PH_PASS1);
  SD_TRY(engine_pass(a, b, dtype, sr, md->p, 1, strat, out, ldo, report ? &r1 : nullptr, st));
  tm.end(PH_PASS1);
  Scratch miss;
  tm.begin(PH_PASS2);
  if (metric_two_pass(md->metric)) {
    SD_TRY(engine_pass(a, b, dtype, sr, md->p, 2, strat, out, ldo, report ? &r2 : nullptr, st));
  } else if (md->metric == SD_M_KL && a->n_rows > 0 && b->n_rows > 0) {
    // miss counts share the output's leading dimension (expand reads both with ldo)
    SD_TRY(miss.alloc((dtype == SD_F64 ? 8 : 4) * size_t(a->n_rows) * size_t(ldo), st));
    SD_TRY(fill(miss.ptr, a->n_rows, b->n_rows, ldo, dtype, 0.0, st));
    SD_TRY(engine_pass(a, b, dtype, SD_SR_MISS_COUNT, 0.0, 2, strat, miss.ptr, ldo, report ? &r2 : nullptr, st));
  }
  tm.end(PH_PASS2);
  if (report) {
    report->peak_accumulator_entries = std::max(r1.peak_accumulator_entries, r2.peak_accumulator_entries);
    report->workspace_elements = std::max(r1.workspace_elements, r2.workspace_elements);
    report->chunks_executed = r1.chunks_executed + r2.chunks_executed;
  }
  if (md->metric == SD_M_KL && miss.ptr == nullptr) return SD_OK;
  tm.begin(PH_EXPANSION);
  sd_metric_desc full = *md;  // the distance path always applies expansion and post-scale
  full.stages = 0;
  SD_TRY(expand(out, a->n_rows, b->n_rows, ldo, dtype, &full, a->n_cols, sa, sb, miss.ptr, flags, st));
  tm.end(PH_EXPANSION);
  return SD_OK;
}

// The fused route: statistics, then one intersection kernel with the
// epilogue (or top-k) fused in.
static int fused_run(const sd_csr* a, const sd_csr* b, const sd_index* index, int dtype,
                     const sd_metric_desc* md, void* out, int64_t ldo, int topk, int64_t base, void* out_d,
                     int64_t* out_i, uint32_t* flags, PhaseTimer& tm, cudaStream_t st) {
  sd_index* own = nullptr;
  const sd_index* ix = index;
  if (!ix) {
    SD_TRY(index_build(b, dtype, 0, &own, st));
    ix = own;
  }
  Scratch sabuf, sbbuf;
  Stats sa, sb;
  if (dense_eligible(b, md, dtype, topk)) {  // dense-ish index: one tensor-core GEMM (dense_tc.cu)
    SD_TRY(ensure_dense(const_cast<sd_index*>(ix), b, st));
    tm.begin(PH_NORMS);
    int rc = isect_stats(a, b, ix, dtype, md, sabuf, sbbuf, &sa, &sb, false, st);
    tm.end(PH_NORMS);
    if (rc == SD_OK) {
      tm.begin(PH_PASS1);
      rc = dense_run(a, b, ix, md, sa, sb, out, ldo, flags, st);
      tm.end(PH_PASS1);
    }
    if (own) {
      cudaStreamSynchronize(st);
      sd_index_free(own);
    }
    return rc;
  }
  if (topk <= 128 && hybrid_kind(md->metric) >= 0 && hybrid_enabled())
    SD_TRY(ensure_hybrid(const_cast<sd_index*>(ix), b, hybrid_kind(md->metric), st));
  const int ph_stats = is_namm(md->metric) ? PH_PASS2 : PH_NORMS;
  tm.begin(ph_stats);
  // dot-family metrics that may take the hybrid path compute their query
  // statistics inside isect_run (overlapped with the dense path)
  const bool defer_a = isect_hybrid_eligible(ix, md, topk) && metric_stats_count(md->metric) > 0;
  int rc = isect_stats(a, b, ix, dtype, md, sabuf, sbbuf, &sa, &sb, defer_a, st);
  tm.end(ph_stats);
  if (rc == SD_OK) {
    rc = isect_run(a, b, ix, dtype, md, sa, sb, out, ldo, topk, base, out_d, out_i, flags, &tm, defer_a, st);
  }
  if (own) {
    cudaStreamSynchronize(st);
    sd_index_free(own);
  }
  return rc;
}

}  // namespace sd

using namespace sd;

extern "C" {

int sd_version(void) { return SD_ABI_VERSION; }

int sd_tune(int k, int64_t value, int64_t* previous) {
  if (k < 0 || k >= SD_TUNE_COUNT) { set_error("unknown tuning knob"); return SD_E_INVALID; }
  const int64_t old = knob(k);
  g_knobs[k].store(value, std::memory_order_relaxed);
  if (previous) *previous = old;
  return SD_OK;
}
uint64_t sd_launch_count(void) { return g_launches.load(); }
const char* sd_last_error(void) { return g_error.c_str(); }

int sd_smem_budget(int device, int64_t* bytes) {
  int v = 0;
  SD_CUDA_TRY(cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
  *bytes = v;
  return SD_OK;
}

int sd_row_stat(const sd_csr* m, int dtype, int kind, void* out, sd_stream_t stream) {
  SD_TRY(check_csr(m, "m"));
  if (kind < SD_STAT_L0 || kind > SD_STAT_SUM) { set_error("unknown statistic"); return SD_E_INVALID; }
  return row_stat(m, dtype, kind, 0, 0.0, out, as_stream(stream));
}

int sd_csr_to_coo(const sd_csr* m, int64_t* rows_out, sd_stream_t stream) {
  SD_TRY(check_csr(m, "m"));
  return csr_to_coo(m, rows_out, as_stream(stream));
}

int sd_check_nonnegative(const sd_csr* m, int dtype, uint32_t* dev_flags, sd_stream_t stream) {
  SD_TRY(check_csr(m, "m"));
  return check_nonnegative(m, dtype, dev_flags, as_stream(stream));
}

int sd_sqrt_values(const sd_csr* m, int dtype, void* values_out, sd_stream_t stream) {
  SD_TRY(check_csr(m, "m"));
  return sqrt_values(m, dtype, values_out, as_stream(stream));
}

int sd_fill(void* out, int64_t m, int64_t n, int64_t ldo, int dtype, double value, sd_stream_t stream) {
  if (ldo < n) { set_error("ldo < n"); return SD_E_INVALID; }
  return fill(out, m, n, ldo, dtype, value, as_stream(stream));
}

int sd_pass(const sd_csr* a, const sd_csr* b, int dtype, int semiring, double p, int pass,
            const sd_strategy* strategy, void* out, int64_t ldo, sd_report* report, sd_stream_t stream) {
  SD_TRY(check_csr(a, "a"));
  SD_TRY(check_csr(b, "b"));
  return engine_pass(a, b, dtype, semiring, p, pass, strategy, out, ldo, report, as_stream(stream));
}

int sd_index_build(const sd_csr* b, int dtype, int tile_rows, sd_index** out, sd_stream_t stream) {
  SD_TRY(check_csr(b, "b"));
  if (!out) { set_error("out is NULL"); return SD_E_INVALID; }
  return index_build(b, dtype, tile_rows, out, as_stream(stream));
}

int sd_pairwise(const sd_csr* a, const sd_csr* b, const sd_index* index, int dtype, const sd_metric_desc* md,
                const sd_strategy* strategy, void* out, int64_t ldo, uint32_t* dev_flags, sd_report* report,
                float* phase_ms, sd_stream_t stream) {
  cudaStream_t st = as_stream(stream);
  SD_TRY(check_csr(a, "a"));
  SD_TRY(check_csr(b, "b"));
  SD_TRY(check_metric(md));
  if (a->n_cols != b->n_cols) { set_error("column counts differ"); return SD_E_DIM; }
  if (ldo < b->n_rows) { set_error("ldo < b.n_rows"); return SD_E_INVALID; }
  PhaseTimer tm(phase_ms, st);
  if (needs_nonneg(md->metric)) {
    SD_TRY(check_nonnegative(a, dtype, dev_flags, st));
    SD_TRY(check_nonnegative(b, dtype, dev_flags, st));
  }
  sd_csr a2, b2;
  Scratch abuf, bbuf;
  tm.begin(PH_NORMS);
  SD_TRY(transformed(a, dtype, md, &a2, abuf, st));
  SD_TRY(transformed(b, dtype, md, &b2, bbuf, st));
  tm.end(PH_NORMS);
  const bool engine = (strategy && strategy->kind != SD_STRAT_AUTO) || metric_contrib(md->metric) < 0;
  if (engine) {
    SD_TRY(engine_pairwise(&a2, &b2, dtype, md, strategy, out, ldo, dev_flags, report, tm, st));
    return tm.finish();
  }
  if (report) *report = sd_report{0, 0, 0};
  if (a->n_rows == 0 || b->n_rows == 0) return tm.finish();
  const bool fresh = md->metric == SD_M_HELLINGER && !md->pre_transformed;
  SD_TRY(fused_run(&a2, &b2, fresh ? nullptr : index, dtype, md, out, ldo, 0, 0, nullptr, nullptr, dev_flags, tm, st));
  return tm.finish();
}

int sd_expand(void* dots, int64_t m, int64_t n, int64_t ldo, int dtype, const sd_metric_desc* md, int64_t n_cols,
              const void* const* stats_a, const void* const* stats_b, uint32_t* dev_flags, sd_stream_t stream) {
  SD_TRY(check_metric(md));
  if (md->stages < 0 || md->stages > 2) { set_error("stages must be 0, 1 or 2"); return SD_E_INVALID; }
  Stats sa, sb;
  const int64_t ns = metric_expand_stats_count(md->metric);
  if (!is_namm(md->metric) && md->metric != SD_M_KL && md->stages != 2) {
    for (int64_t q = 0; q < ns; ++q) {
      sa.s[q] = stats_a ? stats_a[q] : nullptr;
      sb.s[q] = stats_b ? stats_b[q] : nullptr;
      if (!sa.s[q] || !sb.s[q]) { set_error("missing per-row statistics for the expansion"); return SD_E_INVALID; }
    }
  }
  return expand(dots, m, n, ldo, dtype, md, n_cols, sa, sb, nullptr, dev_flags, as_stream(stream));
}

int sd_knn(const sd_csr* q, const sd_csr* b, const sd_index* index, int dtype, const sd_metric_desc* md, int k,
           int64_t index_base, void* out_dist, int64_t* out_idx, uint32_t* dev_flags, sd_stream_t stream) {
  cudaStream_t st = as_stream(stream);
  SD_TRY(check_csr(q, "queries"));
  SD_TRY(check_csr(b, "index"));
  SD_TRY(check_metric(md));
  if (q->n_cols != b->n_cols) { set_error("column counts differ"); return SD_E_DIM; }
  if (k > b->n_rows) { set_error("k exceeds the index rows"); return SD_E_K_TOO_LARGE; }
  if (k < 0) { set_error("k must be non-negative"); return SD_E_INVALID; }
  if (k == 0 || q->n_rows == 0) return SD_OK;
  if (needs_nonneg(md->metric)) {
    SD_TRY(check_nonnegative(q, dtype, dev_flags, st));
    SD_TRY(check_nonnegative(b, dtype, dev_flags, st));
  }
  sd_csr q2, b2;
  Scratch qbuf, bbuf;
  SD_TRY(transformed(q, dtype, md, &q2, qbuf, st));
  SD_TRY(transformed(b, dtype, md, &b2, bbuf, st));
  sd_metric_desc md2 = *md;
  md2.pre_transformed = 1;
  const bool fresh = md->metric == SD_M_HELLINGER && !md->pre_transformed;
  if (metric_contrib(md->metric) >= 0 && k <= 128) {
    PhaseTimer tm(nullptr, st);
    return fused_run(&q2, &b2, fresh ? nullptr : index, dtype, &md2, nullptr, 0, k, index_base, out_dist, out_idx,
                     dev_flags, tm, st);
  }
  // materialised route: query batches of distance rows, then row top-k
  const size_t es = dtype == SD_F64 ? 8 : 4;
  const int64_t n = b->n_rows;
  const int64_t budget = int64_t(1) << 30;
  const int64_t rows = std::max<int64_t>(1, std::min<int64_t>(q->n_rows, budget / (int64_t(es) * n)));
  Scratch dist;
  SD_TRY(dist.alloc(es * size_t(rows) * size_t(n), st));
  sd_strategy auto_s{SD_STRAT_AUTO, 0, 0.5};
  for (int64_t s = 0; s < q->n_rows; s += rows) {
    sd_csr qs = q2;
    qs.n_rows = std::min<int64_t>(rows, q->n_rows - s);
    qs.indptr = q2.indptr + s;
    SD_TRY(sd_pairwise(&qs, &b2, fresh ? nullptr : index, dtype, &md2, &auto_s, dist.ptr, n, dev_flags, nullptr,
                       nullptr, stream));
    SD_TRY(topk_rows(dist.ptr, qs.n_rows, n, n, dtype, k, index_base, static_cast<char*>(out_dist) + es * s * k,
                     out_idx + s * k, st));
  }
  return SD_OK;
}

int sd_topk_rows(const void* dist, int64_t m, int64_t n, int64_t ldd, int dtype, int k, int64_t index_base,
                 void* out_dist, int64_t* out_idx, sd_stream_t stream) {
  return topk_rows(dist, m, n, ldd, dtype, k, index_base, out_dist, out_idx, as_stream(stream));
}

int sd_topk_merge(const void* cand_dist, const int64_t* cand_idx, int64_t m, int lists, int k, int dtype,
                  void* out_dist, int64_t* out_idx, sd_stream_t stream) {
  return topk_merge(cand_dist, cand_idx, m, lists, k, dtype, out_dist, out_idx, as_stream(stream));
}

}  // extern "C"
