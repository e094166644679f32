// semiring.cuh — device functors for the fixed semiring set of the reference
// (/root/reference/pkg/src/semidist/semiring.py:36-119, metrics.py:303-305).
//
// Each product reproduces the numpy expression of the reference operation by
// operation (same guards, same operation order, IEEE-rounded ops, no FMA),
// so fp64 products are bitwise those of the reference up to libm ulp
// differences in log/pow.
#pragma once
#include "common.cuh"

namespace sd {

enum ReduceKind { RED_SUM = 0, RED_MAX = 1, RED_MIN = 2 };

template <int SR> struct SemiringTraits;
#define SD_SR_TRAITS(ID, RED, ANNIH)                      \
  template <> struct SemiringTraits<ID> {                 \
    static constexpr int reduce = RED;                    \
    static constexpr bool annihilating = ANNIH;           \
  };
SD_SR_TRAITS(SD_SR_DOT, RED_SUM, true)
SD_SR_TRAITS(SD_SR_MIN_PLUS, RED_MIN, false)
SD_SR_TRAITS(SD_SR_ABS_DIFF, RED_SUM, false)
SD_SR_TRAITS(SD_SR_ABS_DIFF_POW, RED_SUM, false)
SD_SR_TRAITS(SD_SR_ABS_DIFF_MAX, RED_MAX, false)
SD_SR_TRAITS(SD_SR_CANBERRA, RED_SUM, false)
SD_SR_TRAITS(SD_SR_MISMATCH, RED_SUM, false)
SD_SR_TRAITS(SD_SR_JS_TERM, RED_SUM, false)
SD_SR_TRAITS(SD_SR_KL_TERM, RED_SUM, true)
SD_SR_TRAITS(SD_SR_MISS_COUNT, RED_SUM, false)
#undef SD_SR_TRAITS

// |x|^p as numpy evaluates `np.abs(d) ** p` for a Python-float p: numpy's
// scalar-power fast paths (p == 1, 2) are exact, everything else is pow().
template <typename T>
__device__ __forceinline__ T pow_p(T d, T p) {
  if (p == T(1)) return d;
  if (p == T(2)) return mul_rn(d, d);
  return pow_(d, p);
}

// ⊗(x, y); x is always the left (A-side) operand.
template <int SR, typename T>
__device__ __forceinline__ T product(T x, T y, T p) {
  if constexpr (SR == SD_SR_DOT) {
    return mul_rn(x, y);                                   // semiring.py:77
  } else if constexpr (SR == SD_SR_MIN_PLUS) {
    return add_rn(x, y);                                   // semiring.py:82
  } else if constexpr (SR == SD_SR_ABS_DIFF || SR == SD_SR_ABS_DIFF_MAX) {
    return abs_(sub_rn(x, y));                             // semiring.py:36-37
  } else if constexpr (SR == SD_SR_ABS_DIFF_POW) {
    return pow_p(abs_(sub_rn(x, y)), p);                   // semiring.py:93-94
  } else if constexpr (SR == SD_SR_CANBERRA) {             // semiring.py:40-44
    T num = abs_(sub_rn(x, y));
    T den = add_rn(abs_(x), abs_(y));
    return den > T(0) ? div_rn(num, den) : T(0);
  } else if constexpr (SR == SD_SR_MISMATCH) {
    return x != y ? T(1) : T(0);                           // semiring.py:47-48
  } else if constexpr (SR == SD_SR_JS_TERM) {              // semiring.py:51-62
    T mu = mul_rn(T(0.5), add_rn(x, y));
    T safe_mu = mu > T(0) ? mu : T(1);
    T left = x > T(0) ? mul_rn(x, log_(div_rn(x, safe_mu))) : T(0);
    T right = y > T(0) ? mul_rn(y, log_(div_rn(y, safe_mu))) : T(0);
    return add_rn(left, right);
  } else if constexpr (SR == SD_SR_KL_TERM) {              // semiring.py:65-73
    T safe_y = y > T(0) ? y : T(1);
    return x > T(0) ? mul_rn(x, log_(div_rn(x, safe_y))) : T(0);
  } else {  // SD_SR_MISS_COUNT, metrics.py:303-305
    return T(1);
  }
}

template <int SR, typename T>
__device__ __forceinline__ T reduce_identity() {
  if constexpr (SemiringTraits<SR>::reduce == RED_MIN) return Num<T>::inf();
  else return T(0);
}

template <int SR, typename T>
__device__ __forceinline__ T reduce_op(T a, T b) {
  if constexpr (SemiringTraits<SR>::reduce == RED_SUM) return add_rn(a, b);
  else if constexpr (SemiringTraits<SR>::reduce == RED_MAX) return a > b ? a : (b != b ? b : (a != a ? a : b));
  else return a < b ? a : (b != b ? b : (a != a ? a : b));
}

// Warp all-reduce with a fixed butterfly order (deterministic).
template <int SR, typename T>
__device__ __forceinline__ T warp_reduce(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = reduce_op<SR, T>(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// One-sided terms ⊗(x, 0) and ⊗(0, y) of a single stored entry (the union
// decomposition's correction terms and one-sided row sums).  The JS term
// reduces to x·log 2 whenever x/2 is exact (normal x): the same value as the
// general formula (mu = x/2, x/mu == 2) without its division and log.
// Canberra's is |x| / |x| = 1 exactly for any finite non-zero x.
template <int SR, typename T>
__device__ __forceinline__ T product_a0(T x, T p) {
  if constexpr (SR == SD_SR_JS_TERM) {
    if (x >= T(2) * Num<T>::min_normal()) return mul_rn(x, log_(T(2)));
  } else if constexpr (SR == SD_SR_CANBERRA) {
    if (x != T(0) && abs_(x) <= Num<T>::max_finite()) return T(1);
  }
  return product<SR, T>(x, T(0), p);
}
template <int SR, typename T>
__device__ __forceinline__ T product_0b(T y, T p) {
  if constexpr (SR == SD_SR_JS_TERM) {
    if (y >= T(2) * Num<T>::min_normal()) return mul_rn(y, log_(T(2)));
  } else if constexpr (SR == SD_SR_CANBERRA) {
    if (y != T(0) && abs_(y) <= Num<T>::max_finite()) return T(1);
  }
  return product<SR, T>(T(0), y, p);
}

}  // namespace sd

#define SD_DISPATCH_SEMIRING(sr, SR, ...)                                          \
  [&]() -> int {                                                                   \
    switch (sr) {                                                                  \
      case SD_SR_DOT: { constexpr int SR = SD_SR_DOT; return __VA_ARGS__(); }      \
      case SD_SR_MIN_PLUS: { constexpr int SR = SD_SR_MIN_PLUS; return __VA_ARGS__(); } \
      case SD_SR_ABS_DIFF: { constexpr int SR = SD_SR_ABS_DIFF; return __VA_ARGS__(); } \
      case SD_SR_ABS_DIFF_POW: { constexpr int SR = SD_SR_ABS_DIFF_POW; return __VA_ARGS__(); } \
      case SD_SR_ABS_DIFF_MAX: { constexpr int SR = SD_SR_ABS_DIFF_MAX; return __VA_ARGS__(); } \
      case SD_SR_CANBERRA: { constexpr int SR = SD_SR_CANBERRA; return __VA_ARGS__(); } \
      case SD_SR_MISMATCH: { constexpr int SR = SD_SR_MISMATCH; return __VA_ARGS__(); } \
      case SD_SR_JS_TERM: { constexpr int SR = SD_SR_JS_TERM; return __VA_ARGS__(); } \
      case SD_SR_KL_TERM: { constexpr int SR = SD_SR_KL_TERM; return __VA_ARGS__(); } \
      case SD_SR_MISS_COUNT: { constexpr int SR = SD_SR_MISS_COUNT; return __VA_ARGS__(); } \
      default: ::sd::set_error("semiring has no device functor");                  \
               return SD_E_UNSUPPORTED;                                            \
    }                                                                              \
  }()
