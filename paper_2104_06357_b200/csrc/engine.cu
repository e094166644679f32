// engine.cu — the generalized two-pass pairwise SpMV (paper Alg. 3) and the
// per-pair merge (Alg. 2), for every semiring of the reference.
//
// Reference semantics (engine.py:195-311):
//   pass 1: out[i, j] ⊕= ⊕_{c ∈ B_j} ⊗(A_i[c] or 0, b_jc)          (staged = A rows)
//   pass 2: out[i, j] ⊕= ⊕_{c ∈ A_i, c ∉ B_j} ⊗(a_ic, 0)           (staged = B rows,
//           zero-mask: only probe misses contribute, engine.py:246-250)
//
// B200 design:
//   * A CTA owns a *batch* of staging units and a slice of swept rows.  A unit
//     is one staged row, or one column chunk of a staged row (plan_chunks,
//     engine.py:143-164), or one column window of a dense row wider than SMEM.
//     Up to RMAX units are staged in shared memory at once ("a round") — the
//     swept nonzeros streamed from HBM/L2 are then probed against all of
//     them, amortising the stream over R staged rows instead of the paper's 1.
//   * Unit storage: a dense value window (n_cols or a window of it) or an
//     open-addressing table (int32 key / T value, mix32 hash, linear probe,
//     load <= 50%) — the paper's two accumulators (§3.3.1-3.3.2).
//   * One warp per swept row: lanes stride the row's nonzeros (coalesced),
//     keep one partial per staged unit in registers and finish with a fixed
//     butterfly reduction; the cell is then updated by exactly one lane.
//     All units of one staged row live in one CTA and are applied in chunk
//     order, so every output cell has a single owner and results are
//     deterministic without atomics.
#include <algorithm>
#include <vector>
#include "common.cuh"
#include "prep.cuh"
#include "semiring.cuh"

namespace sd {

struct Unit {
  int64_t row;          // staged row id
  int64_t ebeg, eend;   // entries [ebeg, eend) of the staged row held by this unit
  int32_t clo, chi;     // column window; -1 = take indices[ebeg] / indices[eend]
  int32_t pad0, pad1;
};

constexpr int RMAX = 8;
constexpr int PASS_THREADS = 256;
constexpr int PASS_WARPS = PASS_THREADS / 32;

template <typename T>
struct PassArgs {
  const int64_t* s_ptr; const int32_t* s_idx; const T* s_val;   // staged side
  const int64_t* w_ptr; const int32_t* w_idx; const T* w_val;   // swept side
  int64_t n_swept;
  int32_t n_cols;
  const Unit* units;
  const int64_t* batch_off;   // batch b = units [batch_off[b], batch_off[b+1])
  int R;                      // units per round
  int hash;                   // 0: dense windows, 1: hash tables
  int slot;                   // dense: window width; hash: table capacity (pow2)
  int64_t swept_per_cta;
  T p;
  T* out;
  int64_t ldo;
};

template <typename T>
__device__ __forceinline__ void hash_insert(int32_t* keys, T* vals, int cap, int32_t c, T v) {
  uint32_t h = mix32(uint32_t(c)) & uint32_t(cap - 1);
  while (true) {
    int32_t prev = atomicCAS(&keys[h], -1, c);
    if (prev == -1) { vals[h] = v; return; }
    h = (h + 1) & uint32_t(cap - 1);
  }
}

template <typename T>
__device__ __forceinline__ T hash_probe(const int32_t* keys, const T* vals, int cap, int32_t c,
                                        bool& found) {
  uint32_t h = mix32(uint32_t(c)) & uint32_t(cap - 1);
  while (true) {
    const int32_t k = keys[h];
    if (k == c) { found = true; return vals[h]; }
    if (k < 0) { found = false; return T(0); }
    h = (h + 1) & uint32_t(cap - 1);
  }
}

template <typename T, int SR, int PASS>
__global__ void __launch_bounds__(PASS_THREADS) pass_kernel(const PassArgs<T> a) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ int64_t u_row[RMAX];
  __shared__ int32_t u_lo[RMAX], u_hi[RMAX], u_grp[RMAX];
  __shared__ T red[PASS_WARPS][RMAX];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t ub = a.batch_off[blockIdx.x], ue = a.batch_off[blockIdx.x + 1];
  const int64_t w0 = int64_t(blockIdx.y) * a.swept_per_cta;
  const int64_t w1 = min(a.n_swept, w0 + a.swept_per_cta);
  const int slot = a.slot;
  T* dslot = reinterpret_cast<T*>(smem);
  int32_t* hkeys = reinterpret_cast<int32_t*>(smem);
  T* hvals = reinterpret_cast<T*>(smem + ((size_t(a.R) * slot * 4 + 15) & ~size_t(15)));
  const T p = a.p;

  for (int64_t rs = ub; rs < ue; rs += a.R) {
    const int nr = int(tmin<int64_t>(a.R, ue - rs));
    __syncthreads();  // previous round finished with the slots
    if (threadIdx.x < nr) {
      const Unit u = a.units[rs + threadIdx.x];
      u_row[threadIdx.x] = u.row;
      u_lo[threadIdx.x] = u.clo >= 0 ? u.clo : a.s_idx[u.ebeg];
      u_hi[threadIdx.x] = u.chi >= 0 ? u.chi : a.s_idx[u.eend];
    }
    const int nslot = nr * slot;
    if (!a.hash) {
      for (int e = threadIdx.x; e < nslot; e += blockDim.x) dslot[e] = T(0);
    } else {
      for (int e = threadIdx.x; e < nslot; e += blockDim.x) hkeys[e] = -1;
    }
    __syncthreads();
    if (threadIdx.x == 0) {  // group consecutive units of the same staged row
      for (int r = 0; r < nr; ++r) u_grp[r] = 0;
      int head = 0;
      for (int r = 0; r < nr; ++r) {
        if (r > 0 && u_row[r] != u_row[head]) head = r;
        u_grp[head] += 1;
      }
    }
    for (int r = warp; r < nr; r += PASS_WARPS) {
      const Unit u = a.units[rs + r];
      const int lo = u_lo[r], hi = u_hi[r];
      for (int64_t e = u.ebeg + lane; e < u.eend; e += 32) {
        const int32_t c = a.s_idx[e];
        const T v = a.s_val[e];
        if (!a.hash) {
          if (c >= lo && c < hi) dslot[size_t(r) * slot + (c - lo)] = v;
        } else {
          hash_insert<T>(hkeys + size_t(r) * slot, hvals + size_t(r) * slot, slot, c, v);
        }
      }
    }
    __syncthreads();

    for (int64_t w = w0 + warp; w < w1; w += PASS_WARPS) {
      T acc[RMAX];
#pragma unroll
      for (int r = 0; r < RMAX; ++r) acc[r] = reduce_identity<SR, T>();
      const int64_t eb = a.w_ptr[w], ee = a.w_ptr[w + 1];
      for (int64_t e = eb + lane; e < ee; e += 32) {
        const int32_t c = a.w_idx[e];
        const T v = a.w_val[e];
#pragma unroll
        for (int r = 0; r < RMAX; ++r) {
          if (r < nr && c >= u_lo[r] && c < u_hi[r]) {
            bool found;
            T x;
            if (!a.hash) {
              x = dslot[size_t(r) * slot + (c - u_lo[r])];
              found = x != T(0);
            } else {
              x = hash_probe<T>(hkeys + size_t(r) * slot, hvals + size_t(r) * slot, slot, c, found);
            }
            if constexpr (PASS == 1) {
              acc[r] = reduce_op<SR, T>(acc[r], product<SR, T>(found ? x : T(0), v, p));
            } else {
              if (!found) acc[r] = reduce_op<SR, T>(acc[r], product<SR, T>(v, T(0), p));
            }
          }
        }
      }
#pragma unroll
      for (int r = 0; r < RMAX; ++r) {
        if (r < nr) {
          const T s = warp_reduce<SR, T>(acc[r]);
          if (lane == r) red[warp][r] = s;
        }
      }
      __syncwarp();
      if (lane < nr && u_grp[lane] > 0) {
        const int64_t row = u_row[lane];
        T* cell = PASS == 1 ? a.out + row * a.ldo + w : a.out + w * a.ldo + row;
        T val = *cell;
        for (int q = 0; q < u_grp[lane]; ++q) val = reduce_op<SR, T>(val, red[warp][lane + q]);
        *cell = val;
      }
      __syncwarp();
    }
  }
}

// Alg. 2 (engine.py:270-311): one thread per (i, j), merging the two sorted
// column lists.  Kept as the reference execution strategy ("naive").
template <typename T, int SR, int PASS>
__global__ void naive_kernel(const int64_t* __restrict__ a_ptr, const int32_t* __restrict__ a_idx,
                             const T* __restrict__ a_val, const int64_t* __restrict__ b_ptr,
                             const int32_t* __restrict__ b_idx, const T* __restrict__ b_val,
                             int64_t m, int64_t n, T p, T* __restrict__ out, int64_t ldo) {
  const int64_t total = m * n;
  for (int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; q < total;
       q += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = q / n, j = q - i * n;
    int64_t ia = a_ptr[i], ib = b_ptr[j];
    const int64_t ae = a_ptr[i + 1], be = b_ptr[j + 1];
    T acc = reduce_identity<SR, T>();
    if constexpr (PASS == 1) {
      if (ib == be) continue;
      for (; ib < be; ++ib) {
        const int32_t c = b_idx[ib];
        while (ia < ae && a_idx[ia] < c) ++ia;
        const T x = (ia < ae && a_idx[ia] == c) ? a_val[ia] : T(0);
        acc = reduce_op<SR, T>(acc, product<SR, T>(x, b_val[ib], p));
      }
    } else {
      if (ia == ae) continue;
      for (; ia < ae; ++ia) {
        const int32_t c = a_idx[ia];
        while (ib < be && b_idx[ib] < c) ++ib;
        if (!(ib < be && b_idx[ib] == c)) acc = reduce_op<SR, T>(acc, product<SR, T>(a_val[ia], T(0), p));
      }
    }
    T* cell = out + i * ldo + j;
    *cell = reduce_op<SR, T>(*cell, acc);
  }
}

// ------------------------------------------------------------------ host

// plan_chunks (engine.py:143-164): near-equal spans of at most `budget`.
static void plan_chunks(int64_t degree, int64_t budget, std::vector<std::pair<int64_t, int64_t>>& spans) {
  spans.clear();
  if (degree <= budget) { spans.emplace_back(0, degree); return; }
  const int64_t n = (degree + budget - 1) / budget;
  const int64_t base = degree / n, rem = degree % n;
  int64_t s = 0;
  for (int64_t t = 0; t < n; ++t) {
    const int64_t sz = base + (t < rem ? 1 : 0);
    spans.emplace_back(s, s + sz);
    s += sz;
  }
}

static int64_t ref_chunk_budget(const sd_strategy* st) {
  return int64_t(st->max_load_factor * double(st->accumulator_capacity));
}

// WorkspaceReport the reference would produce for one pass (engine.py:80-99,
// 212-267, 314-353): computed from the staged side's degrees.
void reference_report(const int64_t* deg, int64_t n_rows, const sd_strategy* st, int64_t swept_nnz,
                      sd_report* rep) {
  rep->peak_accumulator_entries = 0;
  rep->workspace_elements = 0;
  rep->chunks_executed = 0;
  if (st->kind == SD_STRAT_NAIVE) return;
  rep->workspace_elements = swept_nnz;
  std::vector<std::pair<int64_t, int64_t>> spans;
  const bool hash = st->kind == SD_STRAT_HASH;
  const int64_t budget = hash ? std::max<int64_t>(1, ref_chunk_budget(st)) : 0;
  for (int64_t r = 0; r < n_rows; ++r) {
    if (hash) {
      plan_chunks(deg[r], budget, spans);
      rep->chunks_executed += int64_t(spans.size());
      for (auto& s : spans) rep->peak_accumulator_entries = std::max(rep->peak_accumulator_entries, s.second - s.first);
    } else {
      rep->chunks_executed += 1;
      rep->peak_accumulator_entries = std::max(rep->peak_accumulator_entries, deg[r]);
    }
  }
}

struct LaunchClass {
  int hash;
  int slot;                 // window width or table capacity
  std::vector<Unit> units;  // grouped by row, rows ascending, chunks in order
};

static int next_pow2(int64_t x) {
  int64_t c = 2;
  while (c < x) c <<= 1;
  return int(c);
}

template <typename T, int SR, int PASS>
static int run_classes(std::vector<LaunchClass>& classes, const sd_csr* staged, const sd_csr* swept,
                       double p, void* out, int64_t ldo, cudaStream_t st) {
  const int64_t optin = smem_optin_bytes() - static_smem((const void*)pass_kernel<T, SR, PASS>);
  const int sms = num_sms();
  for (auto& cls : classes) {
    if (cls.units.empty()) continue;
    const int64_t per_slot = cls.hash ? int64_t(cls.slot) * (4 + sizeof(T)) + 16 : int64_t(cls.slot) * sizeof(T);
    const int64_t soft = std::min<int64_t>(optin, 112 * 1024);
    int R = int(std::max<int64_t>(1, std::min<int64_t>(RMAX, soft / per_slot)));
    if (per_slot * R > optin) R = int(std::max<int64_t>(1, optin / per_slot));
    if (per_slot > optin) { set_error("staging slot exceeds shared memory"); return SD_E_INVALID; }
    // batches: whole rows, at most R units unless a single row needs more (rounds)
    std::vector<int64_t> boff;
    boff.push_back(0);
    const int64_t nu = int64_t(cls.units.size());
    int64_t i = 0, in_batch = 0;
    while (i < nu) {
      int64_t j = i;
      while (j < nu && cls.units[j].row == cls.units[i].row) ++j;
      const int64_t cnt = j - i;
      if (in_batch > 0 && in_batch + cnt > R) { boff.push_back(i); in_batch = 0; }
      in_batch += cnt;
      i = j;
    }
    boff.push_back(nu);
    const int64_t nb = int64_t(boff.size()) - 1;
    Scratch du, db;
    SD_TRY(du.alloc(sizeof(Unit) * nu, st));
    SD_TRY(db.alloc(sizeof(int64_t) * boff.size(), st));
    SD_CUDA_TRY(cudaMemcpyAsync(du.ptr, cls.units.data(), sizeof(Unit) * nu, cudaMemcpyHostToDevice, st));
    SD_CUDA_TRY(cudaMemcpyAsync(db.ptr, boff.data(), sizeof(int64_t) * boff.size(), cudaMemcpyHostToDevice, st));
    const size_t smem = cls.hash ? ((size_t(R) * cls.slot * 4 + 15) & ~size_t(15)) + size_t(R) * cls.slot * sizeof(T)
                                 : size_t(R) * cls.slot * sizeof(T);
    SD_TRY(prepare_smem(pass_kernel<T, SR, PASS>, smem, "pass_kernel"));
    const int per_sm = std::max<int>(1, int(std::min<int64_t>(8, (228 * 1024) / int64_t(smem + 2048))));
    const int64_t target = int64_t(sms) * per_sm * 2;
    int64_t ny = std::max<int64_t>(1, (target + nb - 1) / nb);
    ny = std::min<int64_t>(ny, std::max<int64_t>(1, swept->n_rows / 16));
    ny = std::min<int64_t>(ny, 65535);
    PassArgs<T> args;
    args.s_ptr = staged->indptr; args.s_idx = staged->indices; args.s_val = static_cast<const T*>(staged->values);
    args.w_ptr = swept->indptr; args.w_idx = swept->indices; args.w_val = static_cast<const T*>(swept->values);
    args.n_swept = swept->n_rows;
    args.n_cols = int32_t(staged->n_cols);
    args.units = du.as<Unit>();
    args.batch_off = db.as<int64_t>();
    args.R = R; args.hash = cls.hash; args.slot = cls.slot;
    args.swept_per_cta = (swept->n_rows + ny - 1) / ny;
    args.p = T(p);
    args.out = static_cast<T*>(out);
    args.ldo = ldo;
    const dim3 grid{unsigned(nb), unsigned(ny), 1u};
    pass_kernel<T, SR, PASS><<<grid, PASS_THREADS, smem, st>>>(args);
    SD_LAUNCH_CHECK();
  }
  return SD_OK;
}

template <typename T>
static int build_classes(const sd_csr* staged, const std::vector<int64_t>& ptr, const sd_strategy* strat,
                         std::vector<LaunchClass>& classes) {
  // the pass kernel's own static shared memory (same for every semiring/pass) is not available
  // to the staging slots: size windows and tables from what is left
  const int64_t optin = smem_optin_bytes() - static_smem((const void*)pass_kernel<T, SD_SR_DOT, 1>);
  const int64_t n_cols = staged->n_cols;
  const int64_t n = staged->n_rows;
  const int kind = strat ? strat->kind : SD_STRAT_AUTO;
  // hash tables: 4-byte key + value, <= 50% load, must fit the opt-in budget
  const int64_t max_cap = [&] {
    int64_t c = 2;
    while (c * 2 * int64_t(4 + sizeof(T)) + 16 <= optin) c *= 2;
    return c;
  }();
  const bool dense = kind == SD_STRAT_DENSE || (kind == SD_STRAT_AUTO && n_cols * int64_t(sizeof(T)) <= optin);
  if (dense) {
    const int64_t win = std::max<int64_t>(1, std::min<int64_t>(n_cols, optin / int64_t(sizeof(T))));
    LaunchClass cls;
    cls.hash = 0;
    cls.slot = int(std::max<int64_t>(1, std::min<int64_t>(win, n_cols)));
    for (int64_t r = 0; r < n; ++r)
      for (int64_t w0 = 0; w0 < std::max<int64_t>(n_cols, 1); w0 += win)
        cls.units.push_back(Unit{r, ptr[r], ptr[r + 1], int32_t(w0), int32_t(std::min<int64_t>(n_cols, w0 + win)), 0, 0});
    classes.push_back(std::move(cls));
    return SD_OK;
  }
  int64_t budget = max_cap / 2;
  if (kind == SD_STRAT_HASH) budget = std::min<int64_t>(budget, std::max<int64_t>(1, ref_chunk_budget(strat)));
  // group rows by table capacity class so each launch sizes its slots tightly
  std::vector<std::pair<int64_t, int64_t>> spans;
  std::vector<LaunchClass> by_cap(32);
  for (int64_t r = 0; r < n; ++r) {
    const int64_t deg = ptr[r + 1] - ptr[r];
    plan_chunks(deg, budget, spans);
    int64_t mx = 0;
    for (auto& s : spans) mx = std::max(mx, s.second - s.first);
    const int cap = next_pow2(std::max<int64_t>(2, 2 * mx));
    int lg = 0;
    while ((1 << lg) < cap) ++lg;
    LaunchClass& cls = by_cap[lg];
    cls.hash = 1;
    cls.slot = cap;
    const int64_t ns = int64_t(spans.size());
    for (int64_t t = 0; t < ns; ++t) {
      Unit u{r, ptr[r] + spans[t].first, ptr[r] + spans[t].second,
             t == 0 ? 0 : -1, t == ns - 1 ? int32_t(n_cols) : -1, 0, 0};
      cls.units.push_back(u);
    }
  }
  for (auto& c : by_cap)
    if (!c.units.empty()) classes.push_back(std::move(c));
  return SD_OK;
}

int engine_pass(const sd_csr* a, const sd_csr* b, int dtype, int semiring, double p, int pass,
                const sd_strategy* strategy, void* out, int64_t ldo, sd_report* report,
                cudaStream_t st) {
  if (a->n_cols != b->n_cols) { set_error("column counts differ"); return SD_E_DIM; }
  if (pass != 1 && pass != 2) { set_error("pass must be 1 or 2"); return SD_E_INVALID; }
  if (ldo < b->n_rows) { set_error("ldo smaller than b.n_rows"); return SD_E_INVALID; }
  sd_strategy dflt{SD_STRAT_AUTO, 0, 0.5};
  const sd_strategy* strat = strategy ? strategy : &dflt;
  if (strat->kind == SD_STRAT_HASH && (strat->accumulator_capacity < 1 || ref_chunk_budget(strat) < 1)) {
    set_error("hash strategy needs accumulator_capacity * max_load_factor >= 1");
    return SD_E_INVALID;
  }
  const sd_csr* staged = pass == 1 ? a : b;
  const sd_csr* swept = pass == 1 ? b : a;
  std::vector<int64_t> ptr(size_t(staged->n_rows + 1));
  SD_CUDA_TRY(cudaMemcpyAsync(ptr.data(), staged->indptr, sizeof(int64_t) * ptr.size(), cudaMemcpyDeviceToHost, st));
  SD_CUDA_TRY(cudaStreamSynchronize(st));
  if (report) {
    std::vector<int64_t> deg(size_t(staged->n_rows));
    for (int64_t r = 0; r < staged->n_rows; ++r) deg[r] = ptr[r + 1] - ptr[r];
    reference_report(deg.data(), staged->n_rows, strat, swept->nnz, report);
  }
  if (a->n_rows == 0 || b->n_rows == 0) return SD_OK;
  if (strat->kind == SD_STRAT_NAIVE) {
    return SD_DISPATCH_DTYPE(dtype, T, [&]() -> int {
      return SD_DISPATCH_SEMIRING(semiring, SR, [&]() -> int {
        const int64_t total = a->n_rows * b->n_rows;
        const int blocks = int(std::min<int64_t>((total + 255) / 256, int64_t(num_sms()) * 32));
        if (pass == 1)
          naive_kernel<T, SR, 1><<<blocks, 256, 0, st>>>(a->indptr, a->indices, static_cast<const T*>(a->values),
              b->indptr, b->indices, static_cast<const T*>(b->values), a->n_rows, b->n_rows, T(p),
              static_cast<T*>(out), ldo);
        else
          naive_kernel<T, SR, 2><<<blocks, 256, 0, st>>>(a->indptr, a->indices, static_cast<const T*>(a->values),
              b->indptr, b->indices, static_cast<const T*>(b->values), a->n_rows, b->n_rows, T(p),
              static_cast<T*>(out), ldo);
        SD_LAUNCH_CHECK();
        return SD_OK;
      });
    });
  }
  return SD_DISPATCH_DTYPE(dtype, T, [&]() -> int {
    std::vector<LaunchClass> classes;
    SD_TRY(build_classes<T>(staged, ptr, strat, classes));
    return SD_DISPATCH_SEMIRING(semiring, SR, [&]() -> int {
      if (pass == 1) return run_classes<T, SR, 1>(classes, staged, swept, p, out, ldo, st);
      return run_classes<T, SR, 2>(classes, staged, swept, p, out, ldo, st);
    });
  });
}

}  // namespace sd
