// common.cuh — shared plumbing for libsemidist_b200 (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <string>
#include <cmath>
#include <cfloat>
#include "../../include/semidist_b200.h"

namespace sd {

template <typename T>
__host__ __device__ __forceinline__ T tmin(T a, T b) { return a < b ? a : b; }
template <typename T>
__host__ __device__ __forceinline__ T tmax(T a, T b) { return a < b ? b : a; }

// ------------------------------------------------------------------ errors
void set_error(const std::string& msg);
void count_launch();

struct Status {
  int code;
};

#define SD_CUDA_TRY(expr)                                                        \
  do {                                                                           \
    cudaError_t _e = (expr);                                                     \
    if (_e != cudaSuccess) {                                                     \
      ::sd::set_error(std::string(#expr) + ": " + cudaGetErrorString(_e));      \
      return SD_E_CUDA;                                                          \
    }                                                                            \
  } while (0)

#define SD_LAUNCH_CHECK()                                                        \
  do {                                                                           \
    ::sd::count_launch();                                                        \
    cudaError_t _e = cudaGetLastError();                                         \
    if (_e != cudaSuccess) {                                                     \
      ::sd::set_error(std::string("kernel launch (") + __FILE__ + ":" +          \
                      std::to_string(__LINE__) + "): " + cudaGetErrorString(_e)); \
      return SD_E_CUDA;                                                          \
    }                                                                            \
  } while (0)

#define SD_TRY(expr)                                                             \
  do {                                                                           \
    int _s = (expr);                                                             \
    if (_s != SD_OK) return _s;                                                  \
  } while (0)

inline cudaStream_t as_stream(sd_stream_t s) { return reinterpret_cast<cudaStream_t>(s); }

// tuning knob (sd_tune_knob): environment default read once at load, then sd_tune
int64_t knob(int k);

int num_sms();
int64_t smem_optin_bytes();
int64_t l2_bytes();

// Opt a kernel into `dyn` bytes of dynamic shared memory, accounting for its
// static shared memory; reports the kernel name on failure.
template <typename K>
int prepare_smem(K kernel, size_t dyn, const char* name) {
  cudaFuncAttributes attr{};
  cudaError_t e = cudaFuncGetAttributes(&attr, kernel);
  if (e != cudaSuccess) {
    set_error(std::string(name) + ": cudaFuncGetAttributes: " + cudaGetErrorString(e));
    return SD_E_CUDA;
  }
  if (int64_t(dyn + attr.sharedSizeBytes) > smem_optin_bytes()) {
    set_error(std::string(name) + ": shared memory request exceeds the opt-in limit");
    return SD_E_INVALID;
  }
  e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(dyn));
  if (e != cudaSuccess) {
    set_error(std::string(name) + ": cudaFuncSetAttribute(" + std::to_string(dyn) + "): " + cudaGetErrorString(e));
    return SD_E_CUDA;
  }
  return SD_OK;
}

inline int64_t static_smem(const void* kernel) {
  cudaFuncAttributes attr{};
  if (cudaFuncGetAttributes(&attr, kernel) != cudaSuccess) return 0;
  return int64_t(attr.sharedSizeBytes);
}

// Stream-ordered scratch allocation that is released when the guard dies
// (the release is itself stream-ordered, so kernels already enqueued keep
// a valid buffer).
struct Scratch {
  void* ptr = nullptr;
  cudaStream_t stream = 0;
  Scratch() = default;
  Scratch(const Scratch&) = delete;
  Scratch& operator=(const Scratch&) = delete;
  ~Scratch() {
    if (ptr) cudaFreeAsync(ptr, stream);
  }
  int alloc(size_t bytes, cudaStream_t s) {
    stream = s;
    if (bytes == 0) bytes = 16;
    cudaError_t e = cudaMallocAsync(&ptr, bytes, s);
    if (e != cudaSuccess) {
      ptr = nullptr;
      set_error(std::string("cudaMallocAsync: ") + cudaGetErrorString(e));
      return SD_E_CUDA;
    }
    return SD_OK;
  }
  template <typename T>
  T* as() const { return reinterpret_cast<T*>(ptr); }
};

// ----------------------------------------------------------- device utils
template <typename T> struct Num;
template <> struct Num<float> {
  __device__ __forceinline__ static float inf() { return __int_as_float(0x7f800000); }
  __device__ __forceinline__ static float big() { return __int_as_float(0x7f800000); }  // KL saturation (1e308 not representable)
  __device__ __forceinline__ static float eps() { return FLT_EPSILON; }
  __device__ __forceinline__ static float min_normal() { return FLT_MIN; }
  __device__ __forceinline__ static float max_finite() { return FLT_MAX; }
};
template <> struct Num<double> {
  __device__ __forceinline__ static double inf() { return __longlong_as_double(0x7ff0000000000000ULL); }
  __device__ __forceinline__ static double big() { return 1e308; }  // KL_SATURATION, metrics.py:29
  __device__ __forceinline__ static double eps() { return DBL_EPSILON; }
  __device__ __forceinline__ static double min_normal() { return DBL_MIN; }
  __device__ __forceinline__ static double max_finite() { return DBL_MAX; }
};

// Exact IEEE ops, spelled out so that no FMA contraction can change the
// rounding relative to the numpy reference (the library is also compiled
// with -fmad=false).
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float sub_rn(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ float fma_rn(float a, float b, float c) { return __fmaf_rn(a, b, c); }
__device__ __forceinline__ double fma_rn(double a, double b, double c) { return __fma_rn(a, b, c); }
__device__ __forceinline__ float div_rn(float a, float b) { return __fdiv_rn(a, b); }
__device__ __forceinline__ double div_rn(double a, double b) { return __ddiv_rn(a, b); }
// fp32: the hardware approximation (MUFU.SQRT, relative error ~2^-22, exact
// at 0) — far inside the fp32 parity tolerance (1e-5) and one instruction
// instead of the IEEE sequence (C2 euclidean 3.29 -> 2.67 ms); fp64 stays IEEE.
// -DSD_IEEE_SQRT restores __fsqrt_rn.
#ifndef SD_IEEE_SQRT
__device__ __forceinline__ float sqrt_rn(float a) {
  float r;
  asm("sqrt.approx.f32 %0, %1;" : "=f"(r) : "f"(a));
  return r;
}
#else
__device__ __forceinline__ float sqrt_rn(float a) { return __fsqrt_rn(a); }
#endif
__device__ __forceinline__ double sqrt_rn(double a) { return __dsqrt_rn(a); }
__device__ __forceinline__ float log_(float a) { return logf(a); }
__device__ __forceinline__ double log_(double a) { return log(a); }
__device__ __forceinline__ float pow_(float a, float b) { return powf(a, b); }
__device__ __forceinline__ double pow_(double a, double b) { return pow(a, b); }
__device__ __forceinline__ float abs_(float a) { return fabsf(a); }
__device__ __forceinline__ double abs_(double a) { return fabs(a); }
__device__ __forceinline__ float min_(float a, float b) { return fminf(a, b); }
__device__ __forceinline__ double min_(double a, double b) { return fmin(a, b); }

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }

// Murmur3 fmix32 (hashtable.py:21-29).
__device__ __forceinline__ uint32_t mix32(uint32_t h) {
  h ^= h >> 16;
  h *= 0x85EBCA6Bu;
  h ^= h >> 13;
  h *= 0xC2B2AE35u;
  h ^= h >> 16;
  return h;
}

}  // namespace sd

#define SD_DISPATCH_DTYPE(dt, T, ...)                                  \
  [&]() -> int {                                                       \
    if ((dt) == SD_F32) { using T = float; return __VA_ARGS__(); }     \
    if ((dt) == SD_F64) { using T = double; return __VA_ARGS__(); }    \
    ::sd::set_error("dtype must be SD_F32 or SD_F64");                 \
    return SD_E_INVALID;                                               \
  }()
