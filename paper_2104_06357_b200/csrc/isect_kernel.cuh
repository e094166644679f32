// isect_kernel.cuh — the fused intersection kernel (design: isect.cu header).
// Templated on <value type, metric, top-k slots per lane>; instantiations live
// in isect_f32.cu / isect_f64.cu so they compile in parallel.
#pragma once
#include <type_traits>
#include "common.cuh"
#include "metric.cuh"
#include "prep.cuh"
#include "topk.cuh"

namespace sd {

// One posting of the inverted index: row id within the tile + value, packed
// so that a lane fetches it with a single 8-byte (fp32) / 16-byte (fp64) load.
template <typename T> struct Posting;
template <> struct __align__(8) Posting<float> { uint32_t j; float v; };
template <> struct __align__(16) Posting<double> { uint32_t j; uint32_t pad; double v; };

// order-preserving integer image of a float (for atomicMin on distances)
template <typename T> struct OrdKey;
template <> struct OrdKey<float> {
  using type = int;
  __device__ __forceinline__ static int key(float f) { const int b = __float_as_int(f); return b >= 0 ? b : b ^ 0x7fffffff; }
  __device__ __forceinline__ static float val(int k) { return __int_as_float(k >= 0 ? k : k ^ 0x7fffffff); }
};
template <> struct OrdKey<double> {
  using type = long long;
  __device__ __forceinline__ static long long key(double f) {
    const long long b = __double_as_longlong(f);
    return b >= 0 ? b : b ^ 0x7fffffffffffffffLL;
  }
  __device__ __forceinline__ static double val(long long k) {
    return __longlong_as_double(k >= 0 ? k : k ^ 0x7fffffffffffffffLL);
  }
};

template <typename T>
struct IsectArgs {
  const int64_t* a_ptr;
  const int32_t* a_idx;
  const T* a_val;
  int64_t m;
  const uint32_t* colptr;   // [n_tiles * n_cols + 1]
  const Posting<T>* post;
  int tile;
  int64_t n_tiles, n, n_cols;
  const T* sa0; const T* sa1; const T* sb0; const T* sb1;
  // work plan (plan_kernel): items are (query, tile range) pairs
  const int32_t* order;     // order[p] = query at plan position p (longest first)
  const int32_t* tpi;       // tiles per item of position p
  const int64_t* item_off;  // items of position p: [item_off[p], item_off[p+1])
  const int32_t* item_pos;  // item -> plan position
  unsigned int* counter;
  int tile_major;           // items are (tile, position) pairs in tile-major order
  int cos_scaled;           // cosine: postings hold b_jc / ||b_j|| (sd_index post_cos)
  const int32_t* skip;      // rows with skip[i] >= 0 belong to the hybrid path (tile-major plan)
  int debug;                // timing experiments (SD_ISECT_DEBUG): 1 skip the sweep, 2 skip the epilogue
  int64_t band;             // tiles per band (band-major plan)
  int strict;
  T k, p;
  T* out;
  int64_t ldo;
  uint32_t* flags;
  int topk;
  T* cand_d;                // kNN: per-item candidate lists [items][topk]
  int64_t* cand_i;
  // fused chebyshev (C_MAX)
  const uint8_t* a_rank;    // rank of each A entry in its row (top-CHEB_K by |a|, else 255)
  const T* topa;            // [CHEB_K][m] largest |a| per query row
  const T* topb;            // [CHEB_K][n] largest |b| per index row
  const int64_t* b_ptr;     // index CSR, for the exact fallback of a fully-hit top-K
  const int32_t* b_idx;
  const T* b_val;
  int heavy_compact;        // heavy_rows_kernel: output row = heavy id (kNN's dense rows) instead of the query row
  // kNN: per query, an upper bound of its k-th distance shared by its items
  // (ordered-integer keys, ord_key), lowered when an item's list fills
  typename OrdKey<T>::type* kth;
};


// fast epilogue: 128-cell groups in flight per warp
#ifndef SD_ISECT_EPF
#define SD_ISECT_EPF 4
#endif
constexpr int EPF = SD_ISECT_EPF;
// kNN: its groups are voted, not stored — fewer in flight leaves registers to
// the top-k lists (C5 17.9 -> 16.5 ms with 2; pairwise keeps 4: manhattan
// 2.72 -> 3.49 ms with 2, and 8 loses everywhere)
#ifndef SD_ISECT_EPF_KNN
#define SD_ISECT_EPF_KNN 2
#endif
constexpr int EPF_KNN = SD_ISECT_EPF_KNN;

// warps per CTA (one CTA per SM: 14 x 16 KB accumulators = 224 KB); capping
// the CTA at 448 threads (4 warps on some SM sub-partitions) caps each thread at 128 registers
#ifndef SD_ISECT_WARPS
#define SD_ISECT_WARPS 14
#endif
constexpr int ISECT_MAX_WARPS = SD_ISECT_WARPS;

// columns whose first 32 postings are loaded before any is applied (16: half
// the code and the registers of 32 and measured faster on C2/C3/C5 — the
// kernel is large enough for instruction-cache misses to show)
#ifndef SD_ISECT_U32
#define SD_ISECT_U32 16
#endif
template <typename T> struct IsectU { static constexpr int value = sizeof(T) == 4 ? SD_ISECT_U32 : 16; };

// 4 consecutive values through 16-byte shared/global accesses
template <typename T> struct V4;
template <> struct V4<float> {
  __device__ __forceinline__ static void load(const float* p, float* v) {
    const float4 t = *reinterpret_cast<const float4*>(p);
    v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
  }
  __device__ __forceinline__ static void store(float* p, const float* v) {  // streaming store
    __stcs(reinterpret_cast<float4*>(p), make_float4(v[0], v[1], v[2], v[3]));
  }
  __device__ __forceinline__ static void store_plain(float* p, const float* v) {
    *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
  }
};
template <> struct V4<double> {
  __device__ __forceinline__ static void load(const double* p, double* v) {
    const double2 a = reinterpret_cast<const double2*>(p)[0];
    const double2 b = reinterpret_cast<const double2*>(p)[1];
    v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
  }
  __device__ __forceinline__ static void store(double* p, const double* v) {
    __stcs(reinterpret_cast<double2*>(p), make_double2(v[0], v[1]));
    __stcs(reinterpret_cast<double2*>(p) + 1, make_double2(v[2], v[3]));
  }
  __device__ __forceinline__ static void store_plain(double* p, const double* v) {
    reinterpret_cast<double2*>(p)[0] = make_double2(v[0], v[1]);
    reinterpret_cast<double2*>(p)[1] = make_double2(v[2], v[3]);
  }
};

// read-only 8/16-byte posting fetch (ld.global.nc)
// postings are re-read by every query touching a column: keep them in L2
// (evict_last) against the output stream, which is written evict_first
__device__ __forceinline__ uint64_t l2_evict_last_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ Posting<float> load_posting(const Posting<float>* p, uint64_t pol) {
  uint2 r;
  asm("ld.global.nc.L2::cache_hint.v2.u32 {%0, %1}, [%2], %3;" : "=r"(r.x), "=r"(r.y) : "l"(p), "l"(pol));
  Posting<float> q;
  q.j = r.x;
  q.v = __uint_as_float(r.y);
  return q;
}
__device__ __forceinline__ Posting<double> load_posting(const Posting<double>* p, uint64_t pol) {
  unsigned long long a, b;
  asm("ld.global.nc.L2::cache_hint.v2.u64 {%0, %1}, [%2], %3;" : "=l"(a), "=l"(b) : "l"(p), "l"(pol));
  Posting<double> q;
  q.j = uint32_t(a);
  q.pad = 0;
  q.v = __longlong_as_double((long long)b);
  return q;
}

// Explicit shared-window accesses (32-bit addresses): generic pointers into the
// dynamic shared buffer made the compiler rebuild the cluster window address
// for every access.
__device__ __forceinline__ float lds(uint32_t a, float) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ double lds(uint32_t a, double) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void sts(uint32_t a, float v) {
  asm volatile("st.shared.f32 [%0], %1;" :: "r"(a), "f"(v) : "memory");
}
__device__ __forceinline__ void sts(uint32_t a, double v) {
  asm volatile("st.shared.f64 [%0], %1;" :: "r"(a), "d"(v) : "memory");
}
__device__ __forceinline__ void lds4(uint32_t a, float* v) {
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]) : "r"(a) : "memory");
}
__device__ __forceinline__ void lds4(uint32_t a, double* v) {
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v[0]), "=d"(v[1]) : "r"(a) : "memory");
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v[2]), "=d"(v[3]) : "r"(a + 16) : "memory");
}
__device__ __forceinline__ void sts4_zero(uint32_t a, float) {
  asm volatile("st.shared.v4.f32 [%0], {%1, %1, %1, %1};" :: "r"(a), "f"(0.f) : "memory");
}
__device__ __forceinline__ void sts4_zero(uint32_t a, double) {
  asm volatile("st.shared.v2.f64 [%0], {%1, %1};" :: "r"(a), "d"(0.0) : "memory");
  asm volatile("st.shared.v2.f64 [%0], {%1, %1};" :: "r"(a + 16), "d"(0.0) : "memory");
}

// A lane's 4 cells of a 128-cell group in the straight-line epilogue.  fp32:
// cells 4l..4l+3, one 16-byte access.  fp64: cells 2l, 2l+1, 64+2l, 65+2l —
// two 16-byte accesses, each contiguous over the warp (512 B: 4 wavefronts,
// no bank conflicts; with cells 4l..4l+3 a lane's two halves sat 32 B apart
// and every fp64 epilogue access took twice its wavefronts, r02e ncu: 2.3e8
// excess shared wavefronts per C2 launch).  Output and statistic rows use the
// same cells, so the global stores stay fully coalesced too.
// KL coverage counts: 16 bits per cell (a count never exceeds the query
// row's degree; rows of >= 65,536 columns are settled exactly, kl_count
// below), so a warp needs TJ x (sizeof(T) + 2) bytes and 9 warps fit an SM
// instead of 7 (fp64: 11 instead of 7)
__device__ __forceinline__ uint32_t lds_u16(uint32_t a) {
  unsigned short v;
  asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void sts_u16(uint32_t a, uint32_t v) {
  asm volatile("st.shared.u16 [%0], %1;" :: "r"(a), "h"((unsigned short)v) : "memory");
}
// 4 consecutive counts (8 bytes), zeroed behind
template <typename T>
__device__ __forceinline__ void ldz_cnt4(uint32_t a, T* c) {
  uint32_t w0, w1;
  asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(w0), "=r"(w1) : "r"(a) : "memory");
  asm volatile("st.shared.v2.u32 [%0], {%1, %1};" :: "r"(a), "r"(0u) : "memory");
  c[0] = T(w0 & 0xffffu); c[1] = T(w0 >> 16); c[2] = T(w1 & 0xffffu); c[3] = T(w1 >> 16);
}
// the counts of a lane's 4 epilogue cells (EQ<T> layout), zeroed behind
template <typename T>
__device__ __forceinline__ void ldz_cnt_eq(uint32_t a, T* c) {
  if constexpr (sizeof(T) == 4) {
    ldz_cnt4(a, c);
  } else {
    uint32_t w0, w1;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(w0) : "r"(a) : "memory");
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(w1) : "r"(a + 128u) : "memory");
    asm volatile("st.shared.u32 [%0], %1;" :: "r"(a), "r"(0u) : "memory");
    asm volatile("st.shared.u32 [%0], %1;" :: "r"(a + 128u), "r"(0u) : "memory");
    c[0] = T(w0 & 0xffffu); c[1] = T(w0 >> 16); c[2] = T(w1 & 0xffffu); c[3] = T(w1 >> 16);
  }
}

// ldz(): read the 4 cells and leave zeros behind.  SD_ISECT_XCHG = 1: one
// 16-byte shared exchange per half (ATOMS.EXCH.128) instead of a load and a
// store of zeros (the zeroing stores were 17% of the C2 sweep's LSU wavefronts)
#ifndef SD_ISECT_XCHG
#define SD_ISECT_XCHG 0
#endif
__device__ __forceinline__ void xchg16_zero(uint32_t a, uint32_t* w) {
  unsigned long long lo, hi;
  asm volatile("{\n .reg .b128 z, o;\n mov.b128 z, {%2, %2};\n atom.shared.exch.b128 o, [%3], z;\n"
               " mov.b128 {%0, %1}, o;\n}"
               : "=l"(lo), "=l"(hi) : "l"(0ull), "r"(a) : "memory");
  w[0] = uint32_t(lo); w[1] = uint32_t(lo >> 32); w[2] = uint32_t(hi); w[3] = uint32_t(hi >> 32);
}
template <typename T> struct EQ;
template <> struct EQ<float> {
  static constexpr int CELL = 4;
  __device__ __forceinline__ static int cell(int lane, int u) { return 4 * lane + u; }
  __device__ __forceinline__ static void lds(uint32_t a, float* v) { lds4(a, v); }
  __device__ __forceinline__ static void sts_zero(uint32_t a) { sts4_zero(a, 0.f); }
  __device__ __forceinline__ static void ldz(uint32_t a, float* v) {
#if SD_ISECT_XCHG
    uint32_t w[4];
    xchg16_zero(a, w);
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = __uint_as_float(w[u]);
#else
    lds(a, v);
    sts_zero(a);
#endif
  }
  __device__ __forceinline__ static void ldg(const float* p, float* v) { V4<float>::load(p, v); }
  __device__ __forceinline__ static void stg(float* p, const float* v) { V4<float>::store(p, v); }
};
template <> struct EQ<double> {
  static constexpr int CELL = 2;
  __device__ __forceinline__ static int cell(int lane, int u) { return 2 * lane + (u & 1) + (u >> 1) * 64; }
  __device__ __forceinline__ static void lds(uint32_t a, double* v) {
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v[0]), "=d"(v[1]) : "r"(a) : "memory");
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v[2]), "=d"(v[3]) : "r"(a + 512u) : "memory");
  }
  __device__ __forceinline__ static void sts_zero(uint32_t a) {
    asm volatile("st.shared.v2.f64 [%0], {%1, %1};" :: "r"(a), "d"(0.0) : "memory");
    asm volatile("st.shared.v2.f64 [%0], {%1, %1};" :: "r"(a + 512u), "d"(0.0) : "memory");
  }
  __device__ __forceinline__ static void ldz(uint32_t a, double* v) {
#if SD_ISECT_XCHG
    uint32_t w[4];
    xchg16_zero(a, w);
    v[0] = __hiloint2double(int(w[1]), int(w[0]));
    v[1] = __hiloint2double(int(w[3]), int(w[2]));
    xchg16_zero(a + 512u, w);
    v[2] = __hiloint2double(int(w[1]), int(w[0]));
    v[3] = __hiloint2double(int(w[3]), int(w[2]));
#else
    lds(a, v);
    sts_zero(a);
#endif
  }
  __device__ __forceinline__ static void ldg(const double* p, double* v) {
    const double2 x = *reinterpret_cast<const double2*>(p);
    const double2 y = *reinterpret_cast<const double2*>(p + 64);
    v[0] = x.x; v[1] = x.y; v[2] = y.x; v[3] = y.y;
  }
  __device__ __forceinline__ static void stg(double* p, const double* v) {
    __stcs(reinterpret_cast<double2*>(p), make_double2(v[0], v[1]));
    __stcs(reinterpret_cast<double2*>(p + 64), make_double2(v[2], v[3]));
  }
};

// Metrics whose value for a cell without any intersecting column is a
// per-query constant once the query row is non-empty (the common case on
// sparse data): the epilogue then skips the division entirely.
template <int M>
__host__ __device__ constexpr bool sparse_result() {
  return M == SD_M_DICE || M == SD_M_JACCARD || M == SD_M_DOT || M == SD_M_RUSSELRAO ||
         M == SD_M_HELLINGER;
}

template <typename T, int M>
__device__ __forceinline__ T fused_value(const IsectArgs<T>& a, T acc, T cnt, T ra0, T ra1, T rb0, T rb1,
                                         uint32_t& flags) {
  constexpr int CK = metric_contrib(M);
  if constexpr (CK == C_KL) {
    if (cnt != ra0) {  // some column of A_i is absent from B_j (metrics.py:352-366)
      if (a.strict) flags |= SD_FLAG_KL_UNCOVERED;
      return Num<T>::big();
    }
    return acc;
  } else if constexpr (CK == C_MUL) {
    return expand_cell_t<M, T>(acc, ra0, ra1, rb0, rb1, a.k, a.p, flags);
  } else {
    T x = add_rn(add_rn(ra0, rb0), acc);
    x = x < T(0) ? T(0) : x;  // cancellation residue of the union decomposition
    return expand_cell_t<M, T>(x, T(0), T(0), T(0), T(0), a.k, a.p, flags);
  }
}

// Final value of one cell from its accumulated intersection value gv (and
// count gcv), the query statistics ra0/ra1 and the index-row statistics
// gb0/gb1 (every metric except chebyshev).  Shared by the fused epilogue and
// the heavy-query epilogue so both produce identical bits.
template <typename T, int M>
__device__ __forceinline__ T isect_cell(const IsectArgs<T>& a, T gv, T gcv, T ra0, T ra1, T gb0, T gb1,
                                        bool fast_zero, T zero_val, uint32_t& f) {
  if constexpr (M == SD_M_COSINE) {
    if (ra0 > T(0))  // gb1 = 1/||b|| (0 if empty); scaled postings already carry it
      return a.cos_scaled ? sub_rn(T(1), mul_rn(gv, ra1)) : sub_rn(T(1), mul_rn(gv, mul_rn(ra1, gb1)));
    return gb0 == T(0) ? T(0) : T(1);  // empty query row (metrics.py:116-118): 0 against empty rows, else 1
  } else {
    if (fast_zero && gv == T(0)) return zero_val;
    return fused_value<T, M>(a, gv, gcv, ra0, ra1, gb0, gb1, f);
  }
}

// per-query constants of isect_cell: cells without intersections of a
// non-empty query row take zero_val without the division
template <typename T, int M>
__device__ __forceinline__ void isect_zero(const IsectArgs<T>& a, T ra0, T ra1, bool& fast_zero, T& zero_val) {
  fast_zero = false;
  zero_val = T(0);
  if constexpr (sparse_result<M>()) {
    fast_zero = (M == SD_M_COSINE || M == SD_M_DICE || M == SD_M_JACCARD) ? ra0 > T(0) : true;
    uint32_t f = 0;
    zero_val = expand_cell_t<M, T>(T(0), ra0, ra1, T(1), T(1), a.k, a.p, f);
  }
}

template <typename T, int M, int KPL>
__global__ void __launch_bounds__(ISECT_MAX_WARPS * 32, 1) isect_kernel(const IsectArgs<T> a) {
  extern __shared__ __align__(16) unsigned char smem[];
  constexpr int CK = metric_contrib(M);
  constexpr bool MX = CK == C_MAX;
  constexpr bool KL = CK == C_KL || MX;   // second per-cell array: KL counts / chebyshev masks
  constexpr bool KC = CK == C_KL;         // ... of 16-bit KL counts
  constexpr bool SB0 = (M == SD_M_CORRELATION || M == SD_M_COSINE || M == SD_M_DICE || M == SD_M_EUCLIDEAN ||
                        M == SD_M_JACCARD || is_namm(M));
  constexpr bool SB1 = M == SD_M_CORRELATION || M == SD_M_COSINE;
  // cosine: branch-free 1 - d * (1/||a||) * (1/||b||) (reciprocals from row_stat)
  constexpr unsigned FULL = 0xffffffffu;
  constexpr int U = IsectU<T>::value;
  // posting schedule, chosen per instantiation (both in one kernel cost
  // registers and instruction cache): flattened waves where the per-posting
  // work is heavy or the epilogue light enough for the sweep to dominate
  // (JS 11.6 -> 7.7 ms, canberra 8.5 -> 7.9, KL 15.4 -> 13.1 on C3; kNN C5
  // 23.0 -> 15.1); column at a time for the rest (C2 cosine 1.42 vs 2.02 ms
  // flattened, manhattan 1.80 vs 2.33, chebyshev 15.5 vs 16.0)
  constexpr bool FLAT = KPL > 0 || CK == C_JS || CK == C_CANBERRA || CK == C_KL;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int TJ = a.tile;
  constexpr uint32_t ES = sizeof(T);
  constexpr uint32_t CS = (KC || MX) ? 2u : 0u;  // bytes per cell of the second array (16-bit)
  // chebyshev hit masks: the top-MK ranks of each side (bits 0..7 the query
  // row's, 8..15 the index row's); the index keeps ranks up to CHEB_K
  constexpr int MK = 8;
  // opaque copies: keeps the accumulator base and the posting pointer in
  // registers instead of letting the compiler rebuild them per access
  uint32_t acc_s;
  asm volatile("mov.b32 %0, %1;" : "=r"(acc_s)
               : "r"(uint32_t(__cvta_generic_to_shared(smem)) + uint32_t(warp) * TJ * (ES + CS)));
  const uint32_t cnt_s = acc_s + uint32_t(TJ) * ES;
  const Posting<T>* __restrict__ post = a.post;
  const uint64_t l2pol = l2_evict_last_policy();
  const T p = a.p;
  const int64_t band_items = a.item_off[a.m];  // written by plan_kernel
  const int64_t total_items = a.tile_major ? band_items : band_items * ((a.n_tiles + a.band - 1) / a.band);
  const bool vec_out = KPL == 0 && (a.ldo & 3) == 0 && (reinterpret_cast<uintptr_t>(a.out) & 15) == 0;
  uint32_t flags = 0;

  // one posting (row jr, value bv) of a column with query value x (and, for
  // chebyshev, query-entry rank xr; jr then carries the posting's rank in bits 16..23)
  auto apply_posting = [&](uint32_t jr, T bv, T x, uint32_t xr, T xl) {
    if constexpr (MX) {
      const uint32_t jl = jr & 0xffffu, rb = jr >> 16;
      const uint32_t ad = acc_s + jl * ES;
      const T m = contrib<CK, T>(x, bv, p);
      const T old = lds(ad, T(0));
      sts(ad, m > old ? m : old);
      const uint32_t bits = (xr < MK ? (1u << xr) : 0u) | (rb < MK ? (1u << (8 + rb)) : 0u);
      if (bits) {
        const uint32_t am = cnt_s + jl * 2u;
        sts_u16(am, lds_u16(am) | bits);
      }
    } else {
      const uint32_t ad = acc_s + jr * ES;
      T c;
      if constexpr (CK == C_JS) c = js_contrib(x, xl, bv);  // log(x) once per column
      else c = contrib<CK, T>(x, bv, p);
      sts(ad, add_rn(lds(ad, T(0)), c));
      if constexpr (KC) sts_u16(cnt_s + jr * 2u, lds_u16(cnt_s + jr * 2u) + 1u);
    }
  };

  for (int q = lane; q < TJ; q += 32) {  // accumulators start zeroed; the epilogue re-zeroes
    sts(acc_s + q * ES, T(0));
    if constexpr (KC || MX) sts_u16(cnt_s + q * 2u, 0u);
  }
  __syncwarp();

  while (true) {
    unsigned item = 0;
    if (lane == 0) item = atomicAdd(a.counter, 1u);
    item = __shfl_sync(FULL, item, 0);
    if (int64_t(item) >= total_items) break;
    int pos;
    int64_t t0, t1;
    if (a.tile_major) {
      t0 = int64_t(item) / a.m;
      pos = int(int64_t(item) - t0 * a.m);
      t1 = t0 + 1;
    } else {
      // band-major items: every band of `band` tiles repeats the same item list
      const int64_t band = int64_t(item) / band_items;
      const int64_t r = int64_t(item) - band * band_items;
      pos = a.item_pos[r];
      const int64_t tpi = a.tpi[pos];
      t0 = band * a.band + (r - a.item_off[pos]) * tpi;
      t1 = tmin<int64_t>(tmin<int64_t>(a.n_tiles, (band + 1) * a.band), t0 + tpi);
    }
    const int64_t i = a.order[pos];
    if (a.skip && a.skip[i] >= 0) continue;
    const int64_t abeg = a.a_ptr[i], aend = a.a_ptr[i + 1];
    const T ra0 = a.sa0 ? a.sa0[i] : T(0);
    // KL with a query row of >= 65,536 columns: the 16-bit counts wrap, so a
    // cell is covered only if B_j holds at least as many columns, the count
    // agrees modulo 2^16, and a merge of the two sorted rows confirms it
    const bool kl_big = KC && aend - abeg >= 65536;
    auto kl_count = [&](T c16, int64_t j) -> T {
      const int64_t da = aend - abeg, bb = a.b_ptr[j], be = a.b_ptr[j + 1];
      if (be - bb < da || uint32_t(c16) != uint32_t(da & 0xffff)) return T(0);  // != ra0 (>= 65,536)
      int64_t ia = abeg, ib = bb, hit = 0;
      while (ia < aend && ib < be) {
        const int32_t ca = a.a_idx[ia], cb = a.b_idx[ib];
        hit += ca == cb;
        ia += ca <= cb;
        ib += cb <= ca;
      }
      return T(hit);
    };
    const T ra1 = a.sa1 ? a.sa1[i] : T(0);
    T topa_l = T(0);  // chebyshev: lane r holds the r-th largest |a| of the query row
    if constexpr (MX) topa_l = lane < CHEB_K ? a.topa[int64_t(lane) * a.m + i] : T(0);
    // value of a cell without intersections when the query row is non-empty
    bool fast_zero;
    T zero_val;
    isect_zero<T, M>(a, ra0, ra1, fast_zero, zero_val);
    // cosine reads the index-row norms only to resolve an empty query row
    const bool need_sb0 = M != SD_M_COSINE || !(ra0 > T(0));
    // ... and over scaled postings not even the 1/||b|| (kNN's generic epilogue)
    const bool need_sb1 = !(M == SD_M_COSINE && a.cos_scaled && ra0 > T(0));
    WarpTopK<T, (KPL > 0 ? KPL : 1)> top;
    if constexpr (KPL > 0) top.init();
    // kNN: cells above the query's shared bound cannot reach its top-k (the
    // bound is some item's k-th distance, >= the final k-th distance)
    T gbound = Num<T>::inf();
    if constexpr (KPL > 0) gbound = OrdKey<T>::val(__ldcg(a.kth + i));

    // the first 32 columns of the query and their posting ranges in tile t0;
    // later tiles get theirs prefetched during the previous tile's epilogue
    // (items of the last, partial band may have an empty tile range: t0 >= t1)
    const bool valid0 = t0 < t1 && abeg + lane < aend;
    const int32_t c0 = valid0 ? a.a_idx[abeg + lane] : 0;
    const T av0 = valid0 ? a.a_val[abeg + lane] : T(0);
    const uint32_t ar0 = (MX && valid0) ? a.a_rank[abeg + lane] : 255u;
    uint32_t pb0 = valid0 ? a.colptr[t0 * a.n_cols + c0] : 0u;
    uint32_t pe0 = valid0 ? a.colptr[t0 * a.n_cols + c0 + 1] : 0u;
    for (int64_t t = t0; t < t1; ++t) {
      if constexpr (KPL > 0) gbound = min_(gbound, OrdKey<T>::val(__ldcg(a.kth + i)));  // other items' progress
      const int64_t j0 = t * TJ;
      const int nt = int(tmin<int64_t>(TJ, a.n - j0));
      const uint32_t* cp = a.colptr + t * a.n_cols;
      // software pipeline: (column, value, posting range) of the next 32 columns
      int64_t e = abeg + lane;
      bool valid = valid0;
      int32_t c = c0;
      T av = av0;
      uint32_t ar = ar0;
      uint32_t pb = pb0;
      uint32_t pe = pe0;
      for (int64_t base = (a.debug & 1) ? aend : abeg; base < aend; base += 32) {
        const int ncol = int(tmin<int64_t>(32, aend - base));
        const uint32_t cur_pb = pb;
        const T cur_av = av;
        const uint32_t cur_ar = ar;
        const unsigned long_mask = __ballot_sync(FULL, pe - pb > 32u);
        const uint32_t cur_pe = pe;
        // next batch's columns (independent of this batch's postings)
        e = base + 32 + lane;
        valid = e < aend;
        c = valid ? a.a_idx[e] : 0;
        av = valid ? a.a_val[e] : T(0);
        if constexpr (MX) ar = valid ? a.a_rank[e] : 255u;
        if constexpr (FLAT) {
          // flattened waves: the batch's postings in this tile, concatenated in
          // column order, 32 per wave (one per lane) whatever the lists'
          // lengths — short lists (C3: ~9 postings per column and tile) no
          // longer leave most lanes idle.  Lanes of one wave holding the same
          // index row (two of the query's columns hit it) apply in column
          // order, so every accumulator sees the per-column order exactly
          // (bitwise the column-at-a-time results).
          const uint32_t cnt = cur_pe - cur_pb;  // 0 past the batch end
          uint32_t incl = cnt;
#pragma unroll
          for (int d = 1; d < 32; d <<= 1) {
            const uint32_t v = __shfl_up_sync(FULL, incl, d);
            if (lane >= d) incl += v;
          }
          const uint32_t excl = incl - cnt;
          const uint32_t total = __shfl_sync(FULL, incl, 31);
          pb = valid ? cp[c] : 0u;  // next batch's ranges, in flight during this one
          pe = valid ? cp[c + 1] : 0u;
          constexpr int UW = U / 4;
          for (uint32_t w0 = 0; w0 < total; w0 += 32u * UW) {
            Posting<T> ps[UW];
            T xs[UW];
            uint32_t xrs[UW];
#pragma unroll
            for (int u = 0; u < UW; ++u) {
              const uint32_t f = w0 + 32u * uint32_t(u) + uint32_t(lane);
              int k = 0;  // the column of flat position f: last k with excl_k <= f
#pragma unroll
              for (int step = 16; step > 0; step >>= 1)
                if (__shfl_sync(FULL, excl, k + step) <= f) k += step;
              const uint32_t ok0 = __shfl_sync(FULL, excl, k);
              const uint32_t pbk = __shfl_sync(FULL, cur_pb, k);
              xs[u] = __shfl_sync(FULL, cur_av, k);
              xrs[u] = 0;
              if constexpr (MX) xrs[u] = __shfl_sync(FULL, cur_ar, k);
              ps[u].j = 0xffffffffu;
              if (f < total) ps[u] = load_posting(post + pbk + (f - ok0), l2pol);
            }
            // conflicts: lanes of a wave holding the same row apply in column
            // order.  KL (7 warps per SM, two accumulator arrays) ranks all UW
            // waves first so the match instructions overlap (C3 14.8 -> 13.1
            // ms); the lighter metrics lose to the extra registers (JS 7.6 ->
            // 8.3) and rank wave by wave
            constexpr bool HOIST = CK == C_KL;
            int rk[UW];
            bool conflict = false;
            if constexpr (HOIST) {
              unsigned any_rank = 0;
#pragma unroll
              for (int u = 0; u < UW; ++u) {
                const bool act = ps[u].j != 0xffffffffu;
                const uint32_t key = act ? (MX ? (ps[u].j & 0xffffu) : ps[u].j) : (0xffff0000u | uint32_t(lane));
                rk[u] = __popc(__match_any_sync(FULL, key) & ((1u << lane) - 1u));
                any_rank |= unsigned(rk[u]);
              }
              conflict = __any_sync(FULL, any_rank != 0u);
            }
#pragma unroll
            for (int u = 0; u < UW; ++u) {
              if (w0 + 32u * uint32_t(u) < total) {  // warp-uniform
                const bool act = ps[u].j != 0xffffffffu;
                const T xl = CK == C_JS ? log_(xs[u]) : T(0);
                if constexpr (!HOIST) {
                  const uint32_t key = act ? (MX ? (ps[u].j & 0xffffu) : ps[u].j) : (0xffff0000u | uint32_t(lane));
                  rk[u] = __popc(__match_any_sync(FULL, key) & ((1u << lane) - 1u));
                  conflict = __any_sync(FULL, rk[u] > 0);
                }
                if (conflict) {
                  const int maxr = int(__reduce_max_sync(FULL, unsigned(rk[u])));
                  for (int r = 0; r <= maxr; ++r) {
                    if (act && rk[u] == r) apply_posting(ps[u].j, ps[u].v, xs[u], xrs[u], xl);
                    __syncwarp();
                  }
                } else {
                  if (act) apply_posting(ps[u].j, ps[u].v, xs[u], xrs[u], xl);
                  __syncwarp();
                }
              }
            }
          }
          continue;
        }
        for (int q0 = 0; q0 < ncol; q0 += U) {
          Posting<T> ps[U];
          if (ncol == 32) {  // full batch: no per-column bounds test
#pragma unroll
            for (int u = 0; u < U; ++u) {
              const uint32_t b0 = __shfl_sync(FULL, cur_pb, (q0 + u) & 31);
              const uint32_t b1 = __shfl_sync(FULL, cur_pe, (q0 + u) & 31);
              const uint32_t pp = b0 + lane;
              ps[u].j = 0xffffffffu;
              if (pp < b1) {
                ps[u] = load_posting(post + pp, l2pol);
              }
            }
          } else {
#pragma unroll
            for (int u = 0; u < U; ++u) {
              const uint32_t b0 = __shfl_sync(FULL, cur_pb, (q0 + u) & 31);
              const uint32_t b1 = __shfl_sync(FULL, cur_pe, (q0 + u) & 31);
              const uint32_t pp = b0 + lane;
              ps[u].j = 0xffffffffu;
              if (q0 + u < ncol && pp < b1) {
                ps[u] = load_posting(post + pp, l2pol);
              }
            }
          }
          if (q0 + U >= ncol) {  // last group of this batch: start the next batch's colptr loads
            pb = valid ? cp[c] : 0u;
            pe = valid ? cp[c + 1] : 0u;
          }
          if (ncol == 32 && long_mask == 0u) {
            // fast path: a full batch without long posting lists (warp-uniform)
#pragma unroll
            for (int u = 0; u < U; ++u) {
              const T x = __shfl_sync(FULL, cur_av, (q0 + u) & 31);
              uint32_t xr = 0;
              if constexpr (MX) xr = __shfl_sync(FULL, cur_ar, (q0 + u) & 31);
              const T xl = CK == C_JS ? log_(x) : T(0);
              if (ps[u].j != 0xffffffffu) apply_posting(ps[u].j, ps[u].v, x, xr, xl);
              __syncwarp();
            }
          } else {
#pragma unroll
            for (int u = 0; u < U; ++u) {
              if (q0 + u < ncol) {
                const T x = __shfl_sync(FULL, cur_av, (q0 + u) & 31);
                uint32_t xr = 0;
                if constexpr (MX) xr = __shfl_sync(FULL, cur_ar, (q0 + u) & 31);
                const T xl = CK == C_JS ? log_(x) : T(0);
                if (ps[u].j != 0xffffffffu) apply_posting(ps[u].j, ps[u].v, x, xr, xl);
                if (long_mask & (1u << ((q0 + u) & 31))) {  // > 32 postings of this column in this tile
                  const uint32_t b0 = __shfl_sync(FULL, cur_pb, (q0 + u) & 31);
                  const uint32_t b1 = __shfl_sync(FULL, cur_pe, (q0 + u) & 31);
                  for (uint32_t p2 = b0 + 32 + lane; p2 < b1; p2 += 32) {
                    Posting<T> q2 = load_posting(post + p2, l2pol);
                    apply_posting(q2.j, q2.v, x, xr, xl);
                  }
                }
                __syncwarp();
              }
            }
          }
        }
      }
      if (t + 1 < t1) {  // next tile's first-batch posting ranges, in flight during the epilogue
        pb0 = valid0 ? cp[a.n_cols + c0] : 0u;
        pe0 = valid0 ? cp[a.n_cols + c0 + 1] : 0u;
      }
      if (a.debug & 2) continue;
      if constexpr (!MX) {
        // full tile (and, pairwise, 16-byte aligned output rows): a
        // straight-line epilogue with pointers advanced per group, no bounds
        // tests, and the per-query cosine branch hoisted out of the cell loop;
        // kNN votes each group against its bounds instead of storing it
        // 128-cell groups in flight: 2 for kNN and KL (KL's count array makes
        // each group heavier: C3 KL 11.56 -> 10.74 ms; JS / canberra lose with 2)
        constexpr int EP = (KPL > 0 || CK == C_KL) ? EPF_KNN : EPF;
        if ((KPL > 0 || vec_out) && nt == TJ && TJ % (EP * 128) == 0) {
          // nz: 0 generic cell, 1 cosine of a non-empty query, 2 the same over
          // scaled postings (no per-cell index statistic at all)
          auto run = [&](auto nz) {
            constexpr int NZM = decltype(nz)::value;
            constexpr bool NZ = NZM > 0;
            constexpr int LC = EQ<T>::CELL;  // the lane's first cell of a group: LC * lane
            T* op = KPL == 0 ? a.out + i * a.ldo + j0 + LC * lane : nullptr;
            const T* p0 = SB0 ? a.sb0 + j0 + LC * lane : nullptr;
            const T* p1 = SB1 ? a.sb1 + j0 + LC * lane : nullptr;
            uint32_t sa = acc_s + uint32_t(LC) * uint32_t(lane) * ES;
            uint32_t sc = cnt_s + uint32_t(LC) * uint32_t(lane) * CS;
            // EP register sets: group g is finished while the next EP-1
            // groups' shared and global loads are in flight
            T gv[EP][4], gc[EP][4], g0[EP][4], g1[EP][4];
            auto load = [&](uint32_t off, T* v, T* c, T* b0, T* b1) {
              EQ<T>::ldz(sa + off * ES, v);
              if constexpr (KC) ldz_cnt_eq<T>(sc + off * CS, c);
              else if constexpr (KL) EQ<T>::ldz(sc + off * ES, c);
              if constexpr (SB0 && !(M == SD_M_COSINE && NZ)) EQ<T>::ldg(p0 + off, b0);
              if constexpr (SB1 && NZM != 2) EQ<T>::ldg(p1 + off, b1);
            };
            T taup = T(0);
            auto retau = [&]() {
              if constexpr (KPL > 0 && M == SD_M_COSINE && NZM == 2) {
                const T thr = top.thr_d;
                const T E = thr != thr ? gbound : min_(thr, gbound);
                const T tau = mul_rn(sub_rn(T(1), E), ra0);
                taup = sub_rn(tau, mul_rn(add_rn(abs_(tau), ra0), T(0x1p-18)));
              }
            };
            retau();
            auto finish = [&](uint32_t off, const T* v, const T* c, const T* b0, const T* b1) {
              if constexpr (KPL > 0 && M == SD_M_COSINE && NZM == 2) {
                // kNN cosine over scaled postings: once a group cannot beat
                // the bound E (the list's k-th distance, or the query's shared
                // bound), r = 1 - v / ||a|| <= E needs v >= (1 - E) ||a||.  A
                // group whose every accumulator lies below that threshold,
                // lowered by a margin far above the rounding of r and of the
                // threshold itself, is one the exact vote below would reject:
                // skip its arithmetic (C5: after the lists fill, ~all groups).
                // NaN accumulators pass to the exact path.
                // (taup: recomputed per tile and after every offer)
                const bool pass = !(v[0] < taup) || !(v[1] < taup) || !(v[2] < taup) || !(v[3] < taup);
                if (!__any_sync(FULL, pass)) return;
              }
              T cc[4];
#pragma unroll
              for (int u = 0; u < 4; ++u) cc[u] = KL ? c[u] : T(0);
              if constexpr (KC) {
                if (kl_big)
#pragma unroll
                  for (int u = 0; u < 4; ++u) cc[u] = kl_count(cc[u], j0 + off + EQ<T>::cell(lane, u));
              }
              T r[4];
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                if constexpr (M == SD_M_COSINE && NZM == 2) {
                  r[u] = sub_rn(T(1), mul_rn(v[u], ra1));
                } else if constexpr (M == SD_M_COSINE && NZ) {
                  r[u] = sub_rn(T(1), mul_rn(v[u], mul_rn(ra1, b1[u])));
                } else {
                  uint32_t f = 0;
                  r[u] = isect_cell<T, M>(a, v[u], cc[u], ra0, ra1, SB0 ? b0[u] : T(0),
                                          SB1 ? b1[u] : T(0), fast_zero, zero_val, f);
                  flags |= f;
                }
              }
              if constexpr (KPL > 0) {  // the generic epilogue's vote (below), same bounds
                const T thr = top.thr_d;
                const bool open = thr != thr;
                bool ok[4], poss = false;
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                  ok[u] = !(r[u] > gbound);
                  poss |= ok[u] && (open || r[u] < thr);
                }
                if (__any_sync(FULL, poss)) {
#pragma unroll
                  for (int u = 0; u < 4; ++u) top.offer(ok[u], r[u], j0 + off + EQ<T>::cell(lane, u), a.topk);
                  retau();
                }
              } else {
                EQ<T>::stg(op + off, r);
              }
            };
#pragma unroll
            for (int q = 0; q < EP; ++q) load(uint32_t(q) * 128u, gv[q], gc[q], g0[q], g1[q]);
#pragma unroll 1
            for (uint32_t g = 0; g < uint32_t(TJ); g += EP * 128) {
#pragma unroll
              for (int q = 0; q < EP; ++q) {
                finish(g + uint32_t(q) * 128u, gv[q], gc[q], g0[q], g1[q]);
                if (g + uint32_t(q + EP) * 128u < uint32_t(TJ))
                  load(g + uint32_t(q + EP) * 128u, gv[q], gc[q], g0[q], g1[q]);
              }
            }
          };
          if (M == SD_M_COSINE && ra0 > T(0) && a.cos_scaled) run(std::integral_constant<int, 2>{});
          else if (M == SD_M_COSINE && ra0 > T(0)) run(std::integral_constant<int, 1>{});
          else run(std::integral_constant<int, 0>{});
          __syncwarp();
          continue;
        }
      }
      // epilogue: each lane finishes 4 consecutive cells per step (16-byte
      // shared/global accesses); the accumulator is re-zeroed as it is read
      T* orow = KPL == 0 ? a.out + i * a.ldo + j0 : nullptr;
      // group g (128 cells) is computed while group g+1's shared and global
      // loads are in flight (the statistic load is an L2 round trip)
      T v[4], cv[4], b0[4], b1[4];
      auto load_group = [&](int qb, T* gv, T* gcv, T* gb0, T* gb1) {
        const int q = qb + 4 * lane;
#pragma unroll
        for (int u = 0; u < 4; ++u) { gv[u] = T(0); gcv[u] = T(0); gb0[u] = T(0); gb1[u] = T(0); }
        if (q + 3 < nt) {
          lds4(acc_s + q * ES, gv);
          sts4_zero(acc_s + q * ES, T(0));
          if constexpr (KC || MX) ldz_cnt4<T>(cnt_s + q * CS, gcv);
          else if constexpr (KL) { lds4(cnt_s + q * ES, gcv); sts4_zero(cnt_s + q * ES, T(0)); }
          if constexpr (SB0) { if (need_sb0) V4<T>::load(a.sb0 + j0 + q, gb0); }
          if constexpr (SB1) { if (need_sb1) V4<T>::load(a.sb1 + j0 + q, gb1); }
        } else {
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            if (q + u < nt) {
              gv[u] = lds(acc_s + (q + u) * ES, T(0));
              sts(acc_s + (q + u) * ES, T(0));
              if constexpr (KC || MX) { gcv[u] = T(lds_u16(cnt_s + (q + u) * CS)); sts_u16(cnt_s + (q + u) * CS, 0u); }
              else if constexpr (KL) { gcv[u] = lds(cnt_s + (q + u) * ES, T(0)); sts(cnt_s + (q + u) * ES, T(0)); }
              if constexpr (SB0) { if (need_sb0) gb0[u] = a.sb0[j0 + q + u]; }
              if constexpr (SB1) { if (need_sb1) gb1[u] = a.sb1[j0 + q + u]; }
            }
          }
        }
      };
      auto finish_group = [&](int qb, const T* gv, const T* gcv, const T* gb0, const T* gb1) {
        const int q = qb + 4 * lane;
        const bool full = q + 3 < nt;
        T r[4];
        if constexpr (MX) {  // max(M_isect, largest |a| not hit, largest |b| not hit)
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const uint32_t mk = uint32_t(gcv[u]);                 // 16-bit mask, held as a number
            const int fa = __ffs(~(mk & 0xffu)) - 1;              // first unhit A rank, MK = all hit
            const int fb = __ffs(~(mk >> 8)) - 1;
            const T ma = __shfl_sync(FULL, topa_l, fa & 31);
            const int64_t j = j0 + q + u;
            T mb = gb0[u];                                         // rank 0 of B row j
            bool exact = fa == MK && aend - abeg > MK;
            if (q + u < nt && fb > 0) {
              if (fb < MK) mb = a.topb[int64_t(fb) * a.n + j];
              else if (a.b_ptr[j + 1] - a.b_ptr[j] > MK) exact = true;
              else mb = T(0);
            }
            if (exact && q + u < nt) {  // every top-K entry intersects: exact sorted merge (rare)
              T mx = T(0);
              int64_t ia = abeg, ib = a.b_ptr[j];
              const int64_t ie = aend, be = a.b_ptr[j + 1];
              while (ia < ie || ib < be) {
                const int32_t ca = ia < ie ? a.a_idx[ia] : INT32_MAX;
                const int32_t cb = ib < be ? a.b_idx[ib] : INT32_MAX;
                T dv;
                if (ca == cb) { dv = abs_(sub_rn(a.a_val[ia], a.b_val[ib])); ++ia; ++ib; }
                else if (ca < cb) { dv = abs_(a.a_val[ia]); ++ia; }
                else { dv = abs_(a.b_val[ib]); ++ib; }
                mx = dv > mx ? dv : mx;
              }
              r[u] = mx;
            } else {
              T x = gv[u] > ma ? gv[u] : ma;
              r[u] = mb > x ? mb : x;
            }
          }
        } else {
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            uint32_t f = 0;
            T cu = gcv[u];
            if constexpr (KC) { if (kl_big && q + u < nt) cu = kl_count(cu, j0 + q + u); }
            r[u] = isect_cell<T, M>(a, gv[u], cu, ra0, ra1, gb0[u], gb1[u], fast_zero, zero_val, f);
            if (q + u < nt) flags |= f;  // lanes past the tile end evaluate a dummy cell
          }
        }
        if constexpr (KPL > 0) {
          // one vote per 4 cells: once the list is full almost every cell is
          // above the k-th distance.  Exact admission test: cells arrive in
          // ascending index within an item, so a cell tying the k-th
          // distance never precedes it (ties — e.g. the many cosine 1.0s of
          // cells without intersections — are rejected here); a NaN
          // threshold means the list is not full yet
          const T thr = top.thr_d;
          const bool open = thr != thr;
          bool ok[4], poss = false;
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            ok[u] = (q + u < nt) && !(r[u] > gbound);  // (NaN distances only while the bound is open)
            poss |= ok[u] && (open || r[u] < thr);
          }
          if (__any_sync(FULL, poss)) {
#pragma unroll
            for (int u = 0; u < 4; ++u) top.offer(ok[u], r[u], j0 + q + u, a.topk);
          }
        } else {
          if (full && vec_out) {
            V4<T>::store(orow + q, r);
          } else {
#pragma unroll
            for (int u = 0; u < 4; ++u)
              if (q + u < nt) __stcs(orow + q + u, r[u]);
          }
        }
      };
      // ping-pong: finish group g from one register set while group g+1 loads
      // into the other (no copies, so the loads stay in flight)
      T v2[4], cv2[4], b02[4], b12[4];
      load_group(0, v, cv, b0, b1);
      for (int qb = 0; qb < nt; qb += 256) {  // warp-uniform trip count (top-k offers are collective)
        if (qb + 128 < nt) load_group(qb + 128, v2, cv2, b02, b12);
        finish_group(qb, v, cv, b0, b1);
        if (qb + 128 < nt) {
          if (qb + 256 < nt) load_group(qb + 256, v, cv, b0, b1);
          finish_group(qb + 128, v2, cv2, b02, b12);
        }
      }
      __syncwarp();
    }
    if constexpr (KPL > 0) {
      top.store(a.topk, a.cand_d + int64_t(item) * a.topk, a.cand_i + int64_t(item) * a.topk, 0);
      const T thr = top.thr_d;
      if (lane == 0 && thr == thr) atomicMin(a.kth + i, OrdKey<T>::key(thr));  // the list is full
    }
  }
  flags = __reduce_or_sync(FULL, flags);
  if (flags && lane == 0) atomicOr(a.flags, flags);
}

// kNN: merge the per-item candidate lists of each query into its top-k.
template <typename T, int KPL>
__global__ void merge_items_kernel(const T* __restrict__ cd, const int64_t* __restrict__ ci,
                                   const int32_t* __restrict__ order, const int64_t* __restrict__ item_off,
                                   int64_t m, int k, int tile_major, int64_t n_tiles, int64_t n_bands,
                                   int64_t base,
                                   T* __restrict__ od, int64_t* __restrict__ oi) {
  const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  const int64_t band_items = item_off[m];
  for (int64_t p = warp; p < m; p += nw) {
    WarpTopK<T, KPL> top;
    top.init();
    const int64_t per_band = item_off[p + 1] - item_off[p];
    const int64_t n_lists = tile_major ? n_tiles : per_band * n_bands;
    for (int64_t l = 0; l < n_lists; ++l) {
      const int64_t it = tile_major ? l * m + p : (l / per_band) * band_items + item_off[p] + l % per_band;
      for (int q = 0; q < k; q += 32) {
        const int j = q + int(lane_id());
        const bool ok = j < k;
        top.offer(ok, ok ? cd[it * k + j] : T(0), ok ? ci[it * k + j] : 0, k);
      }
    }
    const int64_t i = order[p];
    top.store(k, od + i * k, oi + i * k, base);
  }
}


// Heavy query rows of the hybrid path (hybrid.cu, dot-family metrics): every
// cell of such a row comes from the dense path — heavy index rows from dqh
// ([nhq][hpad], the GEMM), light index rows from dlh ([n][qpad], the dense
// gather).  A CTA stages JB rows of dlh in shared memory so that both the dlh
// reads and the output rows stay coalesced.
template <typename T, int M>
__global__ void __launch_bounds__(256) heavy_rows_kernel(const IsectArgs<T> a, const int32_t* __restrict__ hq,
                                                         int nhq, const int32_t* __restrict__ hid,
                                                         const T* __restrict__ dqh, int64_t hpad,
                                                         const T* __restrict__ dlh, int64_t qpad, int JB) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int64_t qs = qpad + 1;  // padded row stride: lanes read one column across rows
  // per heavy query (row, statistics), loaded once per CTA ahead of the staged rows
  int64_t* qrow = reinterpret_cast<int64_t*>(smem);
  T* qa0 = reinterpret_cast<T*>(qrow + nhq);
  T* qa1 = qa0 + nhq;
  T* sv = reinterpret_cast<T*>(smem + ((size_t(nhq) * (8 + 2 * sizeof(T)) + 15) & ~size_t(15)));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t nblk = (a.n + JB - 1) / JB;
  uint32_t flags = 0;
  for (int qq = threadIdx.x; qq < nhq; qq += blockDim.x) {
    const int64_t i = hq[qq];
    qrow[qq] = i;
    qa0[qq] = a.sa0 ? a.sa0[i] : T(0);
    qa1[qq] = a.sa1 ? a.sa1[i] : T(0);
  }
  for (int64_t blk = blockIdx.x; blk < nblk; blk += gridDim.x) {
    const int64_t j0 = blk * JB;
    const int jn = int(tmin<int64_t>(JB, a.n - j0));
    // per-cell index-row data, loaded once per block row instead of once per heavy query
    constexpr int JL = 2;  // cells per lane (JB <= 64)
    int32_t hj[JL];
    T gb0[JL], gb1[JL];
#pragma unroll
    for (int u = 0; u < JL; ++u) {
      const int jj = lane + 32 * u;
      const bool ok = jj < jn;
      hj[u] = ok ? hid[j0 + jj] : -1;
      gb0[u] = ok && a.sb0 ? a.sb0[j0 + jj] : T(0);
      gb1[u] = ok && a.sb1 ? a.sb1[j0 + jj] : T(0);
    }
    __syncthreads();
    // stage the block's rows of dlh: SU vector loads in flight per thread
    // before any shared store (a load -> store chain per element left the
    // kernel latency-bound)
    const int qv = int(qpad) / 4, nv = jn * qv;
    constexpr int SU = sizeof(T) == 4 ? 8 : 4;
    for (int v0 = threadIdx.x; v0 < nv; v0 += int(blockDim.x) * SU) {
      T r[SU][4];
#pragma unroll
      for (int u = 0; u < SU; ++u) {  // (heavy index rows have no dlh row: never read)
        const int v = v0 + u * int(blockDim.x);
        if (v < nv && __ldg(hid + j0 + v / qv) < 0) V4<T>::load(dlh + j0 * qpad + 4 * int64_t(v), r[u]);
      }
#pragma unroll
      for (int u = 0; u < SU; ++u) {
        const int v = v0 + u * int(blockDim.x);
        if (v < nv && __ldg(hid + j0 + v / qv) < 0) {
          const int jj = v / qv, q = 4 * (v - jj * qv);
#pragma unroll
          for (int t = 0; t < 4; ++t) sv[jj * qs + q + t] = r[u][t];
        }
      }
    }
    // heavy index rows of the block (no dlh row): their sums from the dense
    // block, split over the warps by ordinal
    {
      int ord = 0;
#pragma unroll
      for (int u = 0; u < JL; ++u) {
        unsigned mask = __ballot_sync(0xffffffffu, hj[u] >= 0);
        while (mask) {
          const int l = __ffs(mask) - 1;
          mask &= mask - 1u;
          const int32_t h = __shfl_sync(0xffffffffu, hj[u], l);
          if (ord++ % int(blockDim.x >> 5) == warp)
            for (int q = lane; q < nhq; q += 32) sv[(l + 32 * u) * qs + q] = dqh[int64_t(q) * hpad + h];
        }
      }
    }
    __syncthreads();
    for (int qq = warp; qq < nhq; qq += int(blockDim.x >> 5)) {
      const int64_t i = a.heavy_compact ? int64_t(qq) : qrow[qq];  // output row (kNN: a compact buffer)
      const T ra0 = qa0[qq];
      const T ra1 = qa1[qq];
      bool fast_zero;
      T zero_val;
      isect_zero<T, M>(a, ra0, ra1, fast_zero, zero_val);
#pragma unroll
      for (int u = 0; u < JL; ++u) {
        const int jj = lane + 32 * u;
        if (jj < jn) {
          T gv = sv[jj * qs + qq];
          // manhattan: the dense sums are sum min(a+, b); the contribution is -2x that
          if constexpr (metric_contrib(M) == C_ABS) gv = mul_rn(T(-2), gv);
          uint32_t f = 0;
          __stcs(a.out + i * a.ldo + j0 + jj,
                 isect_cell<T, M>(a, gv, T(0), ra0, ra1, gb0[u], gb1[u], fast_zero, zero_val, f));
          flags |= f;
        }
      }
    }
  }
  flags = __reduce_or_sync(0xffffffffu, flags);
  if (flags && lane == 0) atomicOr(a.flags, flags);
}

template <typename T, int M>
int launch_heavy_rows(IsectArgs<T>& a, const int32_t* hq, int nhq, const int32_t* hid, const T* dqh,
                      int64_t hpad, const T* dlh, int64_t qpad, cudaStream_t st) {
  if (nhq <= 0) return SD_OK;
  if constexpr (metric_contrib(M) != C_MUL && metric_contrib(M) != C_ABS) {
    set_error("the hybrid path serves dot-family metrics and manhattan only");
    return SD_E_UNSUPPORTED;
  } else {
    const int64_t per_row = (qpad + 1) * int64_t(sizeof(T));
    const int64_t qbytes = (int64_t(nhq) * (8 + 2 * int64_t(sizeof(T))) + 15) & ~int64_t(15);
    const int JB = int(tmin<int64_t>(64, (smem_optin_bytes() - 4096 - qbytes) / per_row));  // <= 2 cells per lane
    if (JB < 1) { set_error("too many heavy query rows for the hybrid epilogue"); return SD_E_INVALID; }
    const size_t smem = size_t(qbytes) + size_t(JB) * size_t(per_row);
    SD_TRY(prepare_smem(heavy_rows_kernel<T, M>, smem, "heavy_rows_kernel"));
    const int64_t nblk = (a.n + JB - 1) / JB;
    const int blocks = int(tmin<int64_t>(nblk, int64_t(num_sms()) * 8));
    IsectArgs<T> raw = a;
    raw.cos_scaled = 0;  // the dense path sums raw products
    heavy_rows_kernel<T, M><<<blocks, 256, smem, st>>>(raw, hq, nhq, hid, dqh, hpad, dlh, qpad, JB);
    SD_LAUNCH_CHECK();
    return SD_OK;
  }
}

template <typename T, int M, int KPL>
int launch_isect_kernel(IsectArgs<T>& args, int W, cudaStream_t st) {
  const int64_t per_warp = int64_t(args.tile) * (int64_t(sizeof(T)) + isect_second_bytes(metric_contrib(M), sizeof(T)));
  const size_t smem = size_t(W) * per_warp;
  SD_TRY(prepare_smem(isect_kernel<T, M, KPL>, smem, "isect_kernel"));
  int per_sm = 0;
  SD_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, isect_kernel<T, M, KPL>, W * 32, smem));
  per_sm = std::max(1, per_sm);
  const int64_t blocks = std::max<int64_t>(1, int64_t(num_sms()) * per_sm);
  isect_kernel<T, M, KPL><<<unsigned(blocks), W * 32, smem, st>>>(args);
  SD_LAUNCH_CHECK();
  return SD_OK;
}

template <typename T, int M>
int launch_isect_metric(IsectArgs<T>& args, int W, cudaStream_t st) {
  if (args.topk <= 0) return launch_isect_kernel<T, M, 0>(args, W, st);
  if (args.topk <= 32) return launch_isect_kernel<T, M, 1>(args, W, st);
  return launch_isect_kernel<T, M, 4>(args, W, st);
}

#define SD_ISECT_DISPATCH(T)                                                                        \
  int isect_launch(IsectArgs<T>& args, int metric, int W, cudaStream_t st) {                       \
    switch (metric) {                                                                               \
      case SD_M_CORRELATION: return launch_isect_metric<T, SD_M_CORRELATION>(args, W, st);         \
      case SD_M_COSINE: return launch_isect_metric<T, SD_M_COSINE>(args, W, st);                   \
      case SD_M_DICE: return launch_isect_metric<T, SD_M_DICE>(args, W, st);                       \
      case SD_M_DOT: return launch_isect_metric<T, SD_M_DOT>(args, W, st);                         \
      case SD_M_EUCLIDEAN: return launch_isect_metric<T, SD_M_EUCLIDEAN>(args, W, st);             \
      case SD_M_HELLINGER: return launch_isect_metric<T, SD_M_HELLINGER>(args, W, st);             \
      case SD_M_JACCARD: return launch_isect_metric<T, SD_M_JACCARD>(args, W, st);                 \
      case SD_M_KL: return launch_isect_metric<T, SD_M_KL>(args, W, st);                           \
      case SD_M_RUSSELRAO: return launch_isect_metric<T, SD_M_RUSSELRAO>(args, W, st);             \
      case SD_M_CANBERRA: return launch_isect_metric<T, SD_M_CANBERRA>(args, W, st);               \
      case SD_M_CHEBYSHEV: return launch_isect_metric<T, SD_M_CHEBYSHEV>(args, W, st);             \
      case SD_M_HAMMING: return launch_isect_metric<T, SD_M_HAMMING>(args, W, st);                 \
      case SD_M_JENSENSHANNON: return launch_isect_metric<T, SD_M_JENSENSHANNON>(args, W, st);     \
      case SD_M_MANHATTAN: return launch_isect_metric<T, SD_M_MANHATTAN>(args, W, st);             \
      case SD_M_MINKOWSKI: return launch_isect_metric<T, SD_M_MINKOWSKI>(args, W, st);             \
      default: set_error("metric has no fused intersection kernel"); return SD_E_UNSUPPORTED;      \
    }                                                                                               \
  }                                                                                                 \
  int isect_heavy_rows(IsectArgs<T>& a, int metric, const int32_t* hq, int nhq, const int32_t* hid,                     \
                       const T* dqh, int64_t hpad, const T* dlh, int64_t qpad, cudaStream_t st) {                       \
    switch (metric) {                                                                                                   \
      case SD_M_CORRELATION: return launch_heavy_rows<T, SD_M_CORRELATION>(a, hq, nhq, hid, dqh, hpad, dlh, qpad, st);  \
      case SD_M_COSINE: return launch_heavy_rows<T, SD_M_COSINE>(a, hq, nhq, hid, dqh, hpad, dlh, qpad, st);            \
      case SD_M_DICE: return launch_heavy_rows<T, SD_M_DICE>(a, hq, nhq, hid, dqh, hpad, dlh, qpad, st);                \
      case SD_M_DOT: return launch_heavy_rows<T, SD_M_DOT>(a, hq, nhq, hid, dqh, hpad, dlh, qpad, st);                  \
      case SD_M_EUCLIDEAN: return launch_heavy_rows<T, SD_M_EUCLIDEAN>(a, hq, nhq, hid, dqh, hpad, dlh, qpad, st);      \
      case SD_M_HELLINGER: return launch_heavy_rows<T, SD_M_HELLINGER>(a, hq, nhq, hid, dqh, hpad, dlh, qpad, st);      \
      case SD_M_JACCARD: return launch_heavy_rows<T, SD_M_JACCARD>(a, hq, nhq, hid, dqh, hpad, dlh, qpad, st);          \
      case SD_M_RUSSELRAO: return launch_heavy_rows<T, SD_M_RUSSELRAO>(a, hq, nhq, hid, dqh, hpad, dlh, qpad, st);      \
      case SD_M_MANHATTAN: return launch_heavy_rows<T, SD_M_MANHATTAN>(a, hq, nhq, hid, dqh, hpad, dlh, qpad, st);      \
      default: set_error("metric has no hybrid path"); return SD_E_UNSUPPORTED;                                         \
    }                                                                                                                   \
  }                                                                                                                     \
  int isect_merge(IsectArgs<T>& a, int64_t base, T* od, int64_t* oi, cudaStream_t st) {            \
    const int blocks = int(std::min<int64_t>((a.m * 32 + 255) / 256, int64_t(num_sms()) * 16));    \
    if (a.topk <= 32)                                                                               \
      merge_items_kernel<T, 1><<<blocks, 256, 0, st>>>(a.cand_d, a.cand_i, a.order, a.item_off,    \
                                                        a.m, a.topk, a.tile_major, a.n_tiles,              \
                                                        (a.n_tiles + a.band - 1) / a.band,                \
                                                        base, od, oi);                                     \
    else                                                                                            \
      merge_items_kernel<T, 4><<<blocks, 256, 0, st>>>(a.cand_d, a.cand_i, a.order, a.item_off,    \
                                                        a.m, a.topk, a.tile_major, a.n_tiles,              \
                                                        (a.n_tiles + a.band - 1) / a.band,                \
                                                        base, od, oi);                                     \
    SD_LAUNCH_CHECK();                                                                              \
    return SD_OK;                                                                                   \
  }

int isect_launch(IsectArgs<float>& args, int metric, int W, cudaStream_t st);
int isect_launch(IsectArgs<double>& args, int metric, int W, cudaStream_t st);
int isect_merge(IsectArgs<float>& a, int64_t base, float* od, int64_t* oi, cudaStream_t st);
int isect_heavy_rows(IsectArgs<float>& a, int metric, const int32_t* hq, int nhq, const int32_t* hid,
                     const float* dqh, int64_t hpad, const float* dlh, int64_t qpad, cudaStream_t st);
int isect_heavy_rows(IsectArgs<double>& a, int metric, const int32_t* hq, int nhq, const int32_t* hid,
                     const double* dqh, int64_t hpad, const double* dlh, int64_t qpad, cudaStream_t st);
int isect_merge(IsectArgs<double>& a, int64_t base, double* od, int64_t* oi, cudaStream_t st);

}  // namespace sd
