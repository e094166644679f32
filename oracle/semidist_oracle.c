/*
 * ORACLE — TEST INFRASTRUCTURE ONLY (C restatement, pthreads).
 *
 * The same reference algorithm as oracle/semidist_oracle.py, in C so that the
 * config-scale parity tests (C2 64 queries x 162k rows, C3 32 x
 * 300k, C5 32 x 1M) and bench.py's agreement checks finish in seconds instead
 * of the numpy port's minutes (its pass 2 is a Python loop over every index
 * row).  Used only by tests/, smoke() and bench.py as the CHECKER; the
 * product never loads it.  Built by __graft_entry__.build() / oracle/Makefile
 * into oracle/liboracle_c.so.
 *
 * Source of truth: /root/reference/pkg/src/semidist (pure Python + numpy).
 *   pass 1 (engine.py:195-267, complement=False): stage A row r densely,
 *     every stored entry of every B row j contributes ⊗(A_r[c] or 0, b_jc),
 *     reduced with ⊕ over B_j's entries in storage order, then
 *     out[r, j] = ⊕(out[r, j], partial)                       (engine.py:258-259)
 *   pass 2 (complement=True): stage B row j; entries of A_i whose column is
 *     absent from B_j (probe == 0, the zero mask of engine.py:246-250)
 *     contribute ⊗(a_ic, 0); out[i, j] = ⊕(out[i, j], partial) (engine.py:256-257)
 *   semirings: semiring.py:36-119; expansions / post-scales: metrics.py:93-180;
 *   KL coverage: miss-count pass 2 (metrics.py:303-305, 352-366);
 *   value transform (hellinger sqrt): metrics.py:205-207, 332-338.
 *
 * Pinning: the numpy port is bitwise equal to the reference (tests/golden);
 * this restatement sums sequentially where numpy's reduceat sums pairwise, so
 * it equals the golden vectors to rounding — tests/test_oracle_golden.py
 * checks it against every golden pairwise case (and bit-exact for chebyshev).
 */
#include <math.h>
#include <pthread.h>
#include <stdatomic.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

enum { M_CORRELATION, M_COSINE, M_DICE, M_DOT, M_EUCLIDEAN, M_HELLINGER, M_JACCARD, M_KL, M_RUSSELRAO,
       M_CANBERRA, M_CHEBYSHEV, M_HAMMING, M_JENSENSHANNON, M_MANHATTAN, M_MINKOWSKI };
enum { OK = 0, E_NEGATIVE = 2, E_RADICAND = 3, E_KL_UNCOVERED = 4, E_INVALID = 6, E_NOMEM = 8 };

typedef struct {
  int64_t n_rows, n_cols;
  const int64_t* ptr;
  const int64_t* idx;
  const double* val;
} csr_t;

static const double KL_SATURATION = 1e308;   /* metrics.py:29 */
static const double RADICAND_TOL = 1e-9;     /* metrics.py:27 */

/* ⊗ of semiring.py:36-73 / 90-97 */
static inline double product(int metric, double x, double y, double p) {
  switch (metric) {
    case M_MANHATTAN:
    case M_CHEBYSHEV: return fabs(x - y);
    case M_MINKOWSKI: return pow(fabs(x - y), p);
    case M_CANBERRA: {
      const double den = fabs(x) + fabs(y);
      return den > 0 ? fabs(x - y) / den : 0.0;
    }
    case M_HAMMING: return x != y ? 1.0 : 0.0;
    case M_JENSENSHANNON: {
      const double mu = 0.5 * (x + y);
      const double smu = mu > 0 ? mu : 1.0;
      const double left = x > 0 ? x * log(x / smu) : 0.0;
      const double right = y > 0 ? y * log(y / smu) : 0.0;
      return left + right;
    }
    case M_KL: return x > 0 ? x * log(x / (y > 0 ? y : 1.0)) : 0.0;
    default: return x * y;  /* dot family */
  }
}

static inline double reduce(int metric, double acc, double v) {
  return metric == M_CHEBYSHEV ? (v > acc ? v : acc) : acc + v;
}

static int two_pass(int metric) { return metric >= M_CANBERRA; }

/* ------------------------------------------------ parallel row loop (pthreads) */
typedef struct job {
  const csr_t* a;
  const csr_t* b;
  int metric, count, absolute;
  double p;
  double* out;
  int64_t n_items, chunk, width;
  atomic_llong next;
  atomic_int err;
  void (*body)(struct job*, int64_t, double*);
} job_t;

static void* worker(void* arg) {
  job_t* j = (job_t*)arg;
  double* buf = (double*)calloc((size_t)j->width, sizeof(double));
  if (!buf) { atomic_store(&j->err, E_NOMEM); return NULL; }
  for (;;) {
    const int64_t lo = atomic_fetch_add(&j->next, j->chunk);
    if (lo >= j->n_items) break;
    const int64_t hi = lo + j->chunk < j->n_items ? lo + j->chunk : j->n_items;
    for (int64_t it = lo; it < hi; ++it) j->body(j, it, buf);
  }
  free(buf);
  return NULL;
}

static int run(job_t* j, int threads) {
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  atomic_init(&j->next, 0);
  atomic_init(&j->err, OK);
  pthread_t tid[256];
  int started = 0;
  for (int t = 1; t < threads; ++t)
    if (pthread_create(&tid[started], NULL, worker, j) == 0) ++started;
  worker(j);
  for (int t = 0; t < started; ++t) pthread_join(tid[t], NULL);
  return atomic_load(&j->err);
}

/* one ⊗ term; in magnitude mode its absolute value (conditioning of the sum) */
static inline double term(const job_t* jb, double x, double y) {
  const double t = product(jb->metric, x, y, jb->p);
  return jb->absolute ? fabs(t) : t;
}

/* pass 1 body, staged A row i: out[i, j] ⊕= ⊕_{e in B_j} ⊗(A_i[c_e] or 0, b_e) */
static void pass1_row(job_t* jb, int64_t i, double* buf) {
  const csr_t *a = jb->a, *b = jb->b;
  const int metric = jb->metric;
  for (int64_t e = a->ptr[i]; e < a->ptr[i + 1]; ++e) buf[a->idx[e]] = a->val[e];
  double* row = jb->out + i * b->n_rows;
  for (int64_t j = 0; j < b->n_rows; ++j) {
    const int64_t lo = b->ptr[j], hi = b->ptr[j + 1];
    if (lo == hi) continue;
    double acc = term(jb, buf[b->idx[lo]], b->val[lo]);
    for (int64_t e = lo + 1; e < hi; ++e) acc = reduce(metric, acc, term(jb, buf[b->idx[e]], b->val[e]));
    row[j] = reduce(metric, row[j], acc);
  }
  for (int64_t e = a->ptr[i]; e < a->ptr[i + 1]; ++e) buf[a->idx[e]] = 0.0;
}

/* pass 2 body (zero mask), staged B row j: out[i, j] ⊕= ⊕_{e in A_i, c_e not in B_j} ⊗(a_e, 0).
 * `count` replaces ⊗ by 1 (the KL miss counter, metrics.py:303-305). */
static void pass2_row(job_t* jb, int64_t j, double* buf) {
  const csr_t *a = jb->a, *b = jb->b;
  const int metric = jb->metric;
  for (int64_t e = b->ptr[j]; e < b->ptr[j + 1]; ++e) buf[b->idx[e]] = b->val[e];
  for (int64_t i = 0; i < a->n_rows; ++i) {
    int any = 0;
    double acc = 0.0;
    for (int64_t e = a->ptr[i]; e < a->ptr[i + 1]; ++e) {
      if (buf[a->idx[e]] != 0.0) continue;
      const double t = jb->count ? 1.0 : term(jb, a->val[e], 0.0);
      acc = any ? reduce(metric, acc, t) : t;
      any = 1;
    }
    double* c = jb->out + i * b->n_rows + j;
    if (any) *c = reduce(metric, *c, acc);
  }
  for (int64_t e = b->ptr[j]; e < b->ptr[j + 1]; ++e) buf[b->idx[e]] = 0.0;
}

static int pass(const csr_t* a, const csr_t* b, int metric, double p, int which, int count, int absolute,
                double* out, int threads) {
  job_t j;
  memset(&j, 0, sizeof(j));
  j.a = a; j.b = b; j.metric = metric; j.p = p; j.count = count; j.absolute = absolute; j.out = out;
  j.n_items = which == 1 ? a->n_rows : b->n_rows;
  j.chunk = which == 1 ? 1 : 16;
  j.width = a->n_cols > 0 ? a->n_cols : 1;
  j.body = which == 1 ? pass1_row : pass2_row;
  return run(&j, threads);
}

/* row norms (sparse.py:257-273): kind 0 = l0, 1 = l2sq, 2 = signed sum */
static void norms(const csr_t* m, int kind, double* out) {
  for (int64_t r = 0; r < m->n_rows; ++r) {
    double s = 0.0;
    for (int64_t e = m->ptr[r]; e < m->ptr[r + 1]; ++e)
      s += kind == 0 ? 1.0 : kind == 1 ? m->val[e] * m->val[e] : m->val[e];
    out[r] = s;
  }
}

static int clamp(double* x) {  /* clamp_radicand, metrics.py:93-99 */
  if (*x < -RADICAND_TOL) return E_RADICAND;
  if (*x < 0) *x = 0.0;
  return OK;
}

/* expansions + post-scales (metrics.py:102-180), k = a.n_cols (metrics.py:371-373) */
static int expand(const csr_t* a, const csr_t* b, int metric, double p, double* out) {
  const int64_t m = a->n_rows, n = b->n_rows;
  const double k = (double)a->n_cols;
  double *sa0 = NULL, *sa1 = NULL, *sb0 = NULL, *sb1 = NULL;
  int err = OK;
  if (metric == M_EUCLIDEAN || metric == M_COSINE || metric == M_CORRELATION || metric == M_DICE ||
      metric == M_JACCARD) {
    sa0 = malloc(sizeof(double) * (m ? m : 1)); sa1 = malloc(sizeof(double) * (m ? m : 1));
    sb0 = malloc(sizeof(double) * (n ? n : 1)); sb1 = malloc(sizeof(double) * (n ? n : 1));
    if (!sa0 || !sa1 || !sb0 || !sb1) { err = E_NOMEM; goto done; }
    const int k0 = (metric == M_DICE || metric == M_JACCARD) ? 0 : metric == M_CORRELATION ? 2 : 1;
    norms(a, k0, sa0); norms(b, k0, sb0);
    if (metric == M_CORRELATION) { norms(a, 1, sa1); norms(b, 1, sb1); }
    if (metric == M_COSINE) {
      for (int64_t i = 0; i < m; ++i) sa0[i] = sqrt(sa0[i]);
      for (int64_t j = 0; j < n; ++j) sb0[j] = sqrt(sb0[j]);
    }
  }
  for (int64_t i = 0; i < m && err == OK; ++i) {
    double fa = 0.0;
    if (metric == M_CORRELATION) {
      fa = k * sa1[i] - sa0[i] * sa0[i];
      if ((err = clamp(&fa)) != OK) break;
    }
    for (int64_t j = 0; j < n; ++j) {
      double* c = out + i * n + j;
      const double d = *c;
      switch (metric) {
        case M_EUCLIDEAN: {
          double x = sa0[i] - 2.0 * d + sb0[j];
          if ((err = clamp(&x)) != OK) goto done;
          *c = sqrt(x);
          break;
        }
        case M_COSINE: {
          const double den = sa0[i] * sb0[j];
          *c = den > 0 ? 1.0 - d / den : ((sa0[i] == 0 && sb0[j] == 0) ? 0.0 : 1.0);
          break;
        }
        case M_CORRELATION: {
          double fb = k * sb1[j] - sb0[j] * sb0[j];
          if ((err = clamp(&fb)) != OK) goto done;
          const double den = sqrt(fa * fb);
          const double num = k * d - sa0[i] * sb0[j];
          *c = den > 0 ? 1.0 - num / den : ((sa1[i] == 0 && sb1[j] == 0) ? 0.0 : 1.0);
          break;
        }
        case M_DICE: {
          const double den = sa0[i] + sb0[j];
          *c = den > 0 ? 1.0 - 2.0 * d / den : 0.0;
          break;
        }
        case M_JACCARD: {
          const double den = sa0[i] + sb0[j] - d;
          *c = den > 0 ? 1.0 - d / den : ((sa0[i] == 0 && sb0[j] == 0) ? 0.0 : 1.0);
          break;
        }
        case M_RUSSELRAO: *c = k == 0 ? 0.0 : (k - d) / k; break;
        case M_HELLINGER: {
          double x = d;
          if ((err = clamp(&x)) != OK) goto done;
          *c = 1.0 - sqrt(x);
          break;
        }
        case M_HAMMING: *c = k != 0 ? d / k : 0.0; break;
        case M_JENSENSHANNON: {
          double x = d;
          if ((err = clamp(&x)) != OK) goto done;
          *c = sqrt(x / 2.0);
          break;
        }
        case M_MINKOWSKI: *c = pow(d, 1.0 / p); break;
        default: break;  /* dot, kl, canberra, chebyshev, manhattan */
      }
    }
  }
done:
  free(sa0); free(sa1); free(sb0); free(sb1);
  return err;
}

/* pairwise_distances (metrics.py:320-381), float64, dense m x n row-major `out`.
 * flags bit 0 (magnitude mode, for the parity rule): the passes sum |⊗| and
 * stop before the KL coverage test and the expansion. */
int oracle_pairwise(int64_t m, int64_t n, int64_t n_cols, const int64_t* a_ptr, const int64_t* a_idx,
                    const double* a_val, const int64_t* b_ptr, const int64_t* b_idx, const double* b_val,
                    int metric, double p, int strict, int threads, int flags, double* out) {
  const int absolute = flags & 1;
  if (metric < 0 || metric > M_MINKOWSKI) return E_INVALID;
  csr_t a = {m, n_cols, a_ptr, a_idx, a_val}, b = {n, n_cols, b_ptr, b_idx, b_val};
  const int64_t nnz_a = m ? a_ptr[m] : 0, nnz_b = n ? b_ptr[n] : 0;
  if (metric == M_KL || metric == M_JENSENSHANNON || metric == M_HELLINGER) {  /* metrics.py:308-311 */
    for (int64_t e = 0; e < nnz_a; ++e) if (a_val[e] < 0) return E_NEGATIVE;
    for (int64_t e = 0; e < nnz_b; ++e) if (b_val[e] < 0) return E_NEGATIVE;
  }
  double *ta = NULL, *tb = NULL;
  if (metric == M_HELLINGER) {  /* value transform: sqrt of the stored values */
    ta = malloc(sizeof(double) * (nnz_a ? nnz_a : 1));
    tb = malloc(sizeof(double) * (nnz_b ? nnz_b : 1));
    if (!ta || !tb) { free(ta); free(tb); return E_NOMEM; }
    for (int64_t e = 0; e < nnz_a; ++e) ta[e] = sqrt(a_val[e]);
    for (int64_t e = 0; e < nnz_b; ++e) tb[e] = sqrt(b_val[e]);
    a.val = ta;
    b.val = tb;
  }
  for (int64_t q = 0; q < m * n; ++q) out[q] = 0.0;  /* every ⊕ identity here is 0 */
  int err = pass(&a, &b, metric, p, 1, 0, absolute, out, threads);
  if (err == OK && two_pass(metric)) err = pass(&a, &b, metric, p, 2, 0, absolute, out, threads);
  if (absolute) {
    free(ta);
    free(tb);
    return err;
  }
  if (err == OK && metric == M_KL && m && n) {
    double* miss = calloc((size_t)(m * n), sizeof(double));
    if (!miss) err = E_NOMEM;
    else {
      err = pass(&a, &b, metric, p, 2, 1, 0, miss, threads);
      for (int64_t q = 0; q < m * n && err == OK; ++q) {
        if (miss[q] > 0) {
          if (strict) err = E_KL_UNCOVERED;
          else out[q] = KL_SATURATION;
        }
      }
      free(miss);
    }
  }
  if (err == OK) err = expand(&a, &b, metric, p, out);
  free(ta);
  free(tb);
  return err;
}
