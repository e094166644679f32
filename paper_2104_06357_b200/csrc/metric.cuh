// metric.cuh — Table-1 catalog on device (metrics.py:102-270).
//
// expand_cell() is the element-wise epilogue of pairwise_distances_detail
// (metrics.py:368-374): expansion (metrics.py:102-159) then post-scale
// (metrics.py:162-180), written with the reference's operation order.
//
// For the fused intersection path (isect.cu) every (+)-reduced metric is
// evaluated from intersecting columns only:
//   dot family:  acc = Σ_{c∈A_i∩B_j} a·b                      (exact pass-1 value)
//   kl:          acc = Σ_{c∈A_i∩B_j} a·log(a/b), cnt = |A_i∩B_j|; covered iff cnt == |A_i|
//   NAMM (+):    union sum = S_A[i] + S_B[j] + Σ_{c∈A_i∩B_j} (⊗(a,b) − ⊗(a,0) − ⊗(0,b))
//                with S_A[i] = Σ_c ⊗(a_ic,0), S_B[j] = Σ_c ⊗(0,b_jc)  (Eq. 5 union decomposition)
#pragma once
#include "common.cuh"
#include "semiring.cuh"

namespace sd {

// NEGATIVE_RADICAND_TOLERANCE (metrics.py:27).  float64 uses the reference's
// absolute 1e-9 exactly (same error behaviour: a radicand below -1e-9 raises
// DomainError).  float32 — a precision the reference does not have — also
// admits the fp32 rounding residue of the cancelled terms, 64·eps·scale
// (DESIGN.md §5).
template <typename T>
__device__ __forceinline__ T clamp_radicand(T x, T scale, uint32_t& flags) {
  const T tol = sizeof(T) == 8 ? T(1e-9) : fmax(T(1e-9), T(64) * Num<T>::eps() * scale);
  if (x < -tol) flags |= SD_FLAG_RADICAND;
  return x < T(0) ? T(0) : x;
}

template <typename T>
__device__ __forceinline__ T root_p(T x, T p) {
  // numpy `x ** (1/p)` (metrics.py:166-172); 1/p == 0.5 and 1 hit numpy's exact fast paths
  const T inv = div_rn(T(1), p);
  if (inv == T(1)) return x;
  if (inv == T(0.5)) return sqrt_rn(x);
  return pow_(x, inv);
}

// Per-row statistics layout (s0, s1) for each metric, both sides:
//   correlation: s0 = signed sum, s1 = l2sq     cosine: s0 = l2
//   dice, jaccard: s0 = l0                        euclidean: s0 = l2sq
//   kl (A side): s0 = l0 (coverage test)          NAMM (fused path): s0 = one-sided sum
template <int M, typename T>
__device__ __forceinline__ T expand_cell_t(T d, T a0, T a1, T b0, T b1, T k, T p, uint32_t& flags) {
  if constexpr (M == SD_M_CORRELATION) {  // metrics.py:121-132
    T fa = clamp_radicand(sub_rn(mul_rn(k, a1), mul_rn(a0, a0)), mul_rn(k, a1), flags);
    T fb = clamp_radicand(sub_rn(mul_rn(k, b1), mul_rn(b0, b0)), mul_rn(k, b1), flags);
    T denom = sqrt_rn(mul_rn(fa, fb));
    T num = sub_rn(mul_rn(k, d), mul_rn(a0, b0));
    if (denom > T(0)) return sub_rn(T(1), div_rn(num, denom));
    return (a1 == T(0) && b1 == T(0)) ? T(0) : T(1);
  } else if constexpr (M == SD_M_COSINE) {  // metrics.py:112-118
    T denom = mul_rn(a0, b0);
    if (denom > T(0)) return sub_rn(T(1), div_rn(d, denom));
    return (a0 == T(0) && b0 == T(0)) ? T(0) : T(1);
  } else if constexpr (M == SD_M_DICE) {  // metrics.py:135-140
    T denom = add_rn(a0, b0);
    return denom > T(0) ? sub_rn(T(1), div_rn(mul_rn(T(2), d), denom)) : T(0);
  } else if constexpr (M == SD_M_DOT || M == SD_M_KL) {  // metrics.py:102-103
    return d;
  } else if constexpr (M == SD_M_EUCLIDEAN) {  // metrics.py:106-109 + _sqrt_post 162-163
    T x = add_rn(sub_rn(a0, mul_rn(T(2), d)), b0);
    return sqrt_rn(clamp_radicand(x, add_rn(a0, b0), flags));
  } else if constexpr (M == SD_M_HELLINGER) {  // metrics.py:158-159
    return sub_rn(T(1), sqrt_rn(clamp_radicand(d, T(1), flags)));
  } else if constexpr (M == SD_M_JACCARD) {  // metrics.py:143-149
    T denom = sub_rn(add_rn(a0, b0), d);
    if (denom > T(0)) return sub_rn(T(1), div_rn(d, denom));
    return (a0 == T(0) && b0 == T(0)) ? T(0) : T(1);
  } else if constexpr (M == SD_M_RUSSELRAO) {  // metrics.py:152-155
    return k == T(0) ? T(0) : div_rn(sub_rn(k, d), k);
  } else if constexpr (M == SD_M_HAMMING) {  // _mean_post, metrics.py:175-176
    return k != T(0) ? div_rn(d, k) : T(0);
  } else if constexpr (M == SD_M_JENSENSHANNON) {  // _js_post, metrics.py:179-180
    return sqrt_rn(div_rn(clamp_radicand(d, T(0), flags), T(2)));
  } else if constexpr (M == SD_M_MINKOWSKI) {  // _root_post, metrics.py:166-172
    return root_p(d, p);
  } else {  // canberra, chebyshev, manhattan: identity
    return d;
  }
}

// runtime-dispatched form (element-wise expansion kernel, expansion_apply)
template <typename T>
__device__ __forceinline__ T expand_cell(int metric, T d, T a0, T a1, T b0, T b1, T k, T p, uint32_t& flags) {
  switch (metric) {
    case SD_M_CORRELATION: return expand_cell_t<SD_M_CORRELATION, T>(d, a0, a1, b0, b1, k, p, flags);
    case SD_M_COSINE: return expand_cell_t<SD_M_COSINE, T>(d, a0, a1, b0, b1, k, p, flags);
    case SD_M_DICE: return expand_cell_t<SD_M_DICE, T>(d, a0, a1, b0, b1, k, p, flags);
    case SD_M_EUCLIDEAN: return expand_cell_t<SD_M_EUCLIDEAN, T>(d, a0, a1, b0, b1, k, p, flags);
    case SD_M_HELLINGER: return expand_cell_t<SD_M_HELLINGER, T>(d, a0, a1, b0, b1, k, p, flags);
    case SD_M_JACCARD: return expand_cell_t<SD_M_JACCARD, T>(d, a0, a1, b0, b1, k, p, flags);
    case SD_M_RUSSELRAO: return expand_cell_t<SD_M_RUSSELRAO, T>(d, a0, a1, b0, b1, k, p, flags);
    case SD_M_HAMMING: return expand_cell_t<SD_M_HAMMING, T>(d, a0, a1, b0, b1, k, p, flags);
    case SD_M_JENSENSHANNON: return expand_cell_t<SD_M_JENSENSHANNON, T>(d, a0, a1, b0, b1, k, p, flags);
    case SD_M_MINKOWSKI: return expand_cell_t<SD_M_MINKOWSKI, T>(d, a0, a1, b0, b1, k, p, flags);
    default: return d;
  }
}

// One stage of the epilogue (sd_metric_desc.stages): 0 both, 1 the expansion
// alone (MetricSpec.expansion), 2 the post-scale alone (MetricSpec.post_scale).
// Euclidean is the only metric with both (metrics.py:200-202); every other
// metric has one of them, which expand_cell applies in full.
template <typename T>
__device__ __forceinline__ T expand_stage(int metric, int stage, T d, T a0, T a1, T b0, T b1, T k, T p,
                                          uint32_t& flags) {
  const bool has_post = metric == SD_M_EUCLIDEAN || metric == SD_M_HAMMING || metric == SD_M_JENSENSHANNON ||
                        metric == SD_M_MINKOWSKI;
  const bool has_exp = metric <= SD_M_RUSSELRAO;  // the dot family, kl (identity)
  if (stage == 1) {
    if (!has_exp) return d;
    if (metric == SD_M_EUCLIDEAN) return clamp_radicand(add_rn(sub_rn(a0, mul_rn(T(2), d)), b0), add_rn(a0, b0), flags);
  } else if (stage == 2) {
    if (!has_post) return d;
    if (metric == SD_M_EUCLIDEAN) return sqrt_rn(d);
  }
  return expand_cell<T>(metric, d, a0, a1, b0, b1, k, p, flags);
}

// ---- contributions of one intersecting column for the fused path
enum ContribKind { C_MUL = 0, C_KL = 1, C_ABS = 2, C_ABSPOW = 3, C_CANBERRA = 4, C_MISMATCH = 5, C_JS = 6,
                   C_MAX = 7 /* chebyshev: running max over intersections + top-K hit masks */ };

__host__ __device__ constexpr int metric_contrib(int metric) {
  switch (metric) {
    case SD_M_KL: return C_KL;
    case SD_M_MANHATTAN: return C_ABS;
    case SD_M_MINKOWSKI: return C_ABSPOW;
    case SD_M_CANBERRA: return C_CANBERRA;
    case SD_M_HAMMING: return C_MISMATCH;
    case SD_M_JENSENSHANNON: return C_JS;
    case SD_M_CHEBYSHEV: return C_MAX;
    default: return C_MUL;
  }
}

// bytes per accumulator cell of the fused kernel's second array: 16-bit KL
// coverage counts, 16-bit chebyshev hit masks (top-8 ranks of each side),
// none else
__host__ __device__ constexpr int64_t isect_second_bytes(int ck, int64_t es) {
  return (ck == C_KL || ck == C_MAX) ? 2 : 0;
}

__host__ __device__ inline int contrib_semiring(int ck) {
  switch (ck) {
    case C_MUL: return SD_SR_DOT;
    case C_KL: return SD_SR_KL_TERM;
    case C_ABS: return SD_SR_ABS_DIFF;
    case C_ABSPOW: return SD_SR_ABS_DIFF_POW;
    case C_CANBERRA: return SD_SR_CANBERRA;
    case C_MISMATCH: return SD_SR_MISMATCH;
    default: return SD_SR_JS_TERM;
  }
}

template <int CK, typename T>
__device__ __forceinline__ T contrib(T a, T b, T p) {
  if constexpr (CK == C_MUL) {
    return mul_rn(a, b);
  } else if constexpr (CK == C_KL && sizeof(T) == 4) {
    // fp32 fused path: the quotient by the fast reciprocal-multiply division
    // (<= 2 ulp; the log of the rounded quotient is off by ~u_T absolutely
    // either way, which the parity rule's KL slack allows), huge divisors
    // pre-scaled into the approximate divide's range
    if (!(a > T(0))) return T(0);
    const T y = b > T(0) ? b : T(1);
    const T sc = y > T(1e30) ? T(0x1p-64) : T(1);
    return mul_rn(a, log_(__fdividef(a * sc, y * sc)));
  } else if constexpr (CK == C_KL) {
    return product<SD_SR_KL_TERM, T>(a, b, p);
  } else if constexpr (CK == C_MAX) {
    return abs_(sub_rn(a, b));
  } else if constexpr (CK == C_CANBERRA && sizeof(T) == 4) {
    // fp32 fused path: |a-b| / (|a|+|b|) with the fast reciprocal-multiply
    // division (<= 2 ulp of a ratio in [0, 1], inside the fp32 tolerance; the
    // IEEE division's special-case branch dominated the posting loop), huge
    // pairs pre-scaled so the approximate divide stays in range; equal values
    // still give exactly -2 (0 / d = 0)
    const T num = abs_(sub_rn(a, b)), den = add_rn(abs_(a), abs_(b));
    const T sc = den > T(1e30) ? T(0x1p-64) : T(1);
    const T r = den > T(0) ? __fdividef(num * sc, den * sc) : T(0);
    return sub_rn(sub_rn(r, product_a0<SD_SR_CANBERRA, T>(a, p)), product_0b<SD_SR_CANBERRA, T>(b, p));
  } else {
    constexpr int SR = CK == C_ABS ? SD_SR_ABS_DIFF
                     : CK == C_ABSPOW ? SD_SR_ABS_DIFF_POW
                     : CK == C_CANBERRA ? SD_SR_CANBERRA
                     : CK == C_MISMATCH ? SD_SR_MISMATCH : SD_SR_JS_TERM;
    const T both = product<SR, T>(a, b, p);
    const T left = product_a0<SR, T>(a, p);
    const T right = product_0b<SR, T>(b, p);
    return sub_rn(sub_rn(both, left), right);
  }
}

// Jensen-Shannon's intersection term without divisions: with s = x + y,
// ⊗(x,y) − ⊗(x,0) − ⊗(0,y) = x·log(2x/s) + y·log(2y/s) − (x+y)·log 2
//                          = x·(log x − log s) + y·(log y − log s)
// (x, y > 0: stored entries of nonnegative rows); lx = log x is computed once
// per query column.  Two logs per posting instead of two logs and two
// divisions; same value up to rounding (the union decomposition is a
// restatement within tolerance anyway).
template <typename T>
__device__ __forceinline__ T js_contrib(T x, T lx, T y) {
  const T ls = log_(add_rn(x, y));
  const T gen = add_rn(mul_rn(x, sub_rn(lx, ls)), mul_rn(y, sub_rn(log_(y), ls)));
  // x == y: ⊗(x,x) = 0 exactly, and −x·log 2 − x·log 2 cancels the one-sided
  // sums (product_a0's x·log 2) bit for bit: identical rows get distance
  // exactly 0, as in the reference (a select, not a branch: no divergence)
  const T e = mul_rn(x, log_(T(2)));
  return x == y ? sub_rn(sub_rn(T(0), e), e) : gen;
}

__host__ __device__ constexpr bool is_namm(int metric) {
  return metric >= SD_M_CANBERRA && metric <= SD_M_MINKOWSKI;
}

}  // namespace sd
