// Shared device/host helpers for the bcmg B200 library (sm_100a).
//
// Element types follow the reference's four-type enum (reference
// pkg/src/bcmg/core.py:61-121): real32=0, real64=1, complex64=2,
// complex128=3.  All arithmetic runs in FP64 (DMMA tensor cores for the
// contractions), storage stays in the caller's type.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>

namespace bcmg {

enum DType : int { R32 = 0, R64 = 1, C64 = 2, C128 = 3 };

inline int dtype_size(int dt) {
  switch (dt) {
    case R32: return 4;
    case R64: return 8;
    case C64: return 8;
    case C128: return 16;
  }
  return 0;
}
inline bool dtype_complex(int dt) { return dt == C64 || dt == C128; }

// Error codes: the stable registry of the reference's binding surface
// (reference pkg/frontend/src/errors.ts:9-23) plus a CUDA/NCCL runtime code.
enum Err : int {
  OK = 0,
  NOT_POSITIVE_DEFINITE = 1,
  CONFIG = 2,
  NO_CONVERGENCE = 3,
  OUT_OF_MEMORY = 4,
  CHECK_FAILED = 5,
  STALE_SESSION = 6,
  IO = 7,
  CUDA = 8,
};

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define BCMG_CUDA(call)                                                              \
  do {                                                                               \
    cudaError_t e_ = (call);                                                         \
    if (e_ != cudaSuccess) {                                                         \
      int code_ = (e_ == cudaErrorMemoryAllocation) ? ::bcmg::OUT_OF_MEMORY : ::bcmg::CUDA; \
      throw ::bcmg::Error(code_, std::string(#call) + ": " + cudaGetErrorString(e_)); \
    }                                                                                \
  } while (0)

// Every kernel launch of the library goes through BCMG_CHECK_LAUNCH, which
// also counts it (bcmg_launch_count(): evidence that the native path ran).
// BCMG_DEBUG_SYNC=1 synchronises after every launch and names the failing one.
void note_launch(const char* file, int line);
#define BCMG_CHECK_LAUNCH()                      \
  do {                                           \
    BCMG_CUDA(cudaGetLastError());               \
    ::bcmg::note_launch(__FILE__, __LINE__);     \
  } while (0)

// ---------------------------------------------------------------- storage traits
// Storage type S <-> compute value.  Real types compute in double; complex
// types compute in double2 (re, im).
template <class S> struct Traits;
template <> struct Traits<float> {
  static constexpr bool cplx = false;
  static constexpr int code = R32;
};
template <> struct Traits<double> {
  static constexpr bool cplx = false;
  static constexpr int code = R64;
};
template <> struct Traits<float2> {
  static constexpr bool cplx = true;
  static constexpr int code = C64;
};
template <> struct Traits<double2> {
  static constexpr bool cplx = true;
  static constexpr int code = C128;
};

__host__ __device__ __forceinline__ double2 to_c(float v) { return make_double2(v, 0.0); }
__host__ __device__ __forceinline__ double2 to_c(double v) { return make_double2(v, 0.0); }
__host__ __device__ __forceinline__ double2 to_c(float2 v) { return make_double2(v.x, v.y); }
__host__ __device__ __forceinline__ double2 to_c(double2 v) { return v; }

template <class S> __host__ __device__ __forceinline__ S from_c(double2 v);
template <> __host__ __device__ __forceinline__ float from_c<float>(double2 v) { return (float)v.x; }
template <> __host__ __device__ __forceinline__ double from_c<double>(double2 v) { return v.x; }
template <> __host__ __device__ __forceinline__ float2 from_c<float2>(double2 v) {
  return make_float2((float)v.x, (float)v.y);
}
template <> __host__ __device__ __forceinline__ double2 from_c<double2>(double2 v) { return v; }

__host__ __device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__host__ __device__ __forceinline__ double2 cmulc(double2 a, double2 b) {  // a * conj(b)
  return make_double2(a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y);
}
__host__ __device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }

// Dispatch a templated functor over the four storage types.
template <class F>
inline void dispatch_dtype(int dt, F&& f) {
  switch (dt) {
    case R32: f(float{}); break;
    case R64: f(double{}); break;
    case C64: f(float2{}); break;
    case C128: f(double2{}); break;
    default: throw Error(CONFIG, "unknown element-type code " + std::to_string(dt));
  }
}

}  // namespace bcmg
