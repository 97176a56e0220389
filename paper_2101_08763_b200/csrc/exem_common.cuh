// exem_common.cuh -- shared helpers for the sm_100a kernels and the C-ABI.
//
// Status/error plumbing mirrors the reference's exception hierarchy
// (pkg/src/exembatch/errors.py:4-41) through the EXEM_* codes declared in
// include/exem_b200.h.
#pragma once

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdarg>
#include <cstdio>

#include "../../include/exem_b200.h"

namespace exem {

// ---------------------------------------------------------------- errors
void set_error(const char *fmt, ...);
int fail(int code, const char *fmt, ...);
void count_launch();

#define EXEM_LAUNCH_CHECK(what)                                                \
  do {                                                                         \
    ::exem::count_launch();                                                    \
    cudaError_t _e = cudaGetLastError();                                       \
    if (_e != cudaSuccess)                                                     \
      return ::exem::fail(EXEM_ERR_CUDA, "%s: %s", what,                       \
                          cudaGetErrorString(_e));                             \
  } while (0)

// ---------------------------------------------------------------- layout
constexpr int kPointPad = 256;  // ld of the SIMT layout and TC row padding
constexpr int kDimPad = 8;      // SIMT k-chunk (BK)
constexpr int kTcConst = 6;     // folded constant columns in the TC operands
constexpr int kTcKChunk = 64;   // bf16/f16 elements per 128-byte swizzle row

inline int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }
inline bool aligned(const void *p, uintptr_t a) {
  return ((uintptr_t)p & (a - 1)) == 0;
}
inline int64_t ceil_div(int64_t x, int64_t m) { return (x + m - 1) / m; }

// ---------------------------------------------------------------- types
template <int DT> struct Traits;
template <> struct Traits<EXEM_F16> {
  using S = __half;
  using C = float;
  static constexpr bool kDirect = true;  // objective.py:76-80 direct form
};
template <> struct Traits<EXEM_BF16> {
  using S = __nv_bfloat16;
  using C = float;
  static constexpr bool kDirect = true;
};
template <> struct Traits<EXEM_F32> {
  using S = float;
  using C = float;
  static constexpr bool kDirect = false;  // objective.py:83-90 GEMM form
};
template <> struct Traits<EXEM_F64> {
  using S = double;
  using C = double;
  static constexpr bool kDirect = false;
};

__device__ __forceinline__ float to_c(__half x) { return __half2float(x); }
__device__ __forceinline__ float to_c(__nv_bfloat16 x) {
  return __bfloat162float(x);
}
__device__ __forceinline__ float to_c(float x) { return x; }
__device__ __forceinline__ double to_c(double x) { return x; }

template <typename S> __device__ __forceinline__ S from_d(double x);
template <> __device__ __forceinline__ __half from_d<__half>(double x) {
  return __double2half(x);
}
template <>
__device__ __forceinline__ __nv_bfloat16 from_d<__nv_bfloat16>(double x) {
  return __double2bfloat16(x);
}
template <> __device__ __forceinline__ float from_d<float>(double x) {
  return (float)x;
}
template <> __device__ __forceinline__ double from_d<double>(double x) {
  return x;
}

// ------------------------------------------- vt element type
// vt holds the compute type, or (dtype | EXEM_VT_STORAGE, half tags only)
// the 2-byte storage values themselves; kernels widen in registers.
template <int DT, bool VS> struct VtOf {
  using T = typename Traits<DT>::C;
};
template <> struct VtOf<EXEM_F16, true> { using T = __half; };
template <> struct VtOf<EXEM_BF16, true> { using T = __nv_bfloat16; };

// exact narrowing of a value that came from the storage type
template <typename T> __device__ __forceinline__ T to_vt(float x);
template <> __device__ __forceinline__ float to_vt<float>(float x) { return x; }
template <> __device__ __forceinline__ __half to_vt<__half>(float x) {
  return __float2half_rn(x);
}
template <> __device__ __forceinline__ __nv_bfloat16 to_vt<__nv_bfloat16>(float x) {
  return __float2bfloat16_rn(x);
}
template <typename T> __device__ __forceinline__ T to_vt(double x);
template <> __device__ __forceinline__ double to_vt<double>(double x) { return x; }

template <typename T> __device__ __forceinline__ T tmax(T a, T b);
template <> __device__ __forceinline__ float tmax(float a, float b) {
  return fmaxf(a, b);
}
template <> __device__ __forceinline__ double tmax(double a, double b) {
  return fmax(a, b);
}
template <typename T> __device__ __forceinline__ T tmin(T a, T b);
template <> __device__ __forceinline__ float tmin(float a, float b) {
  return fminf(a, b);
}
template <> __device__ __forceinline__ double tmin(double a, double b) {
  return fmin(a, b);
}
template <typename T> __device__ __forceinline__ T tinf();
template <> __device__ __forceinline__ float tinf<float>() { return __int_as_float(0x7f800000); }
template <> __device__ __forceinline__ double tinf<double>() {
  return __longlong_as_double(0x7ff0000000000000ll);
}

// ------------------------------------------- folded constant columns (TC)
// A per-row constant t >= 0 (h = (||v||^2 - m)/2 or b = ||c||^2/2) rides in
// three storage-type pieces that the other operand multiplies by its "ones"
// columns [kFoldScale, 1, 1]:  t = p0*kFoldScale + p1 + p2.  binary16 tops
// out at 65504, so its first piece is t / 2^11 (exact power-of-two scale;
// t up to 1.3e8, i.e. ||v||^2 < 2.6e8, checked on the host before the TC
// path is chosen); the residues stay below 2^15.  bfloat16 has the fp32
// range and keeps the scale at 1.
template <typename S> struct FoldScale { static constexpr double v = 1.0; };
template <> struct FoldScale<__half> { static constexpr double v = 2048.0; };

template <typename S>
__device__ __forceinline__ void fold_pieces(double t, double (&p)[3]) {
  constexpr double sc = FoldScale<S>::v;
  p[0] = (double)to_c(from_d<S>(t / sc));
  const double r1 = t - p[0] * sc;
  p[1] = (double)to_c(from_d<S>(r1));
  p[2] = (double)to_c(from_d<S>(r1 - p[1]));
}
// value of ones column `piece` (0..2) of the opposite operand
template <typename S>
__device__ __forceinline__ double fold_one(int piece) {
  return piece == 0 ? FoldScale<S>::v : 1.0;
}

// Distance in the reference's per-precision form.
//  GEMM form (f32/f64, objective.py:83-89): out=-2x; out+=b2; out+=e2; max 0
template <typename T>
__device__ __forceinline__ T gemm_form(T dot, T a, T b) {
  T o = T(-2) * dot;
  o = o + a;
  o = o + b;
  return tmax(o, T(0));
}

// ---------------------------------------------------------------- reductions
// Deterministic block sum: fixed xor-shuffle tree, then fixed smem order.
template <int NT>
__device__ __forceinline__ double block_sum(double v, double *sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) sh[w] = v;
  __syncthreads();
  double r = 0.0;
  if (w == 0) {
    r = (lane < NT / 32) ? sh[lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
  }
  __syncthreads();
  return r;  // valid in warp 0
}

// block_sum<256> of 256 point values held two per thread by a 128-thread
// block (thread t: points 2t, 2t+1), bit for bit: each warp rebuilds the
// two 32-point warps of block_sum<256> it covers with shuffles, runs the
// same xor trees, and warp 0 combines the 8 warp sums in the same order.
__device__ __forceinline__ double pair_block_sum(double v0, double v1,
                                                 double *sh) {
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int src_a = lane >> 1, src_b = 16 + (lane >> 1);
  const double a0 = __shfl_sync(0xffffffffu, v0, src_a);
  const double a1 = __shfl_sync(0xffffffffu, v1, src_a);
  const double b0 = __shfl_sync(0xffffffffu, v0, src_b);
  const double b1 = __shfl_sync(0xffffffffu, v1, src_b);
  double va = (lane & 1) ? a1 : a0, vb = (lane & 1) ? b1 : b0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    va += __shfl_xor_sync(0xffffffffu, va, o);
    vb += __shfl_xor_sync(0xffffffffu, vb, o);
  }
  if (lane == 0) {
    sh[2 * w] = va;
    sh[2 * w + 1] = vb;
  }
  __syncthreads();
  double r = 0.0;
  if (w == 0) {
    r = lane < 8 ? sh[lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
  }
  __syncthreads();
  return r;  // valid in warp 0
}

// cp.async helpers (16-byte global -> shared)
__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s),
               "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;\n" ::);
}
template <int N> __device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

}  // namespace exem

// Dispatch a dtype tag to a template body (no runtime multi-backend: one
// kernel instantiation per precision).
// EXEM_DISPATCH plus the vt element flag: VS is a constexpr bool (true only
// for a half tag carrying EXEM_VT_STORAGE)
#define EXEM_DISPATCH_VT(dtype, DT, VS, ...)                                   \
  do {                                                                         \
    const int _tag = (int)(dtype) & ~EXEM_VT_STORAGE;                          \
    const bool _vs = ((int)(dtype) & EXEM_VT_STORAGE) != 0;                    \
    if (_vs && _tag != EXEM_F16 && _tag != EXEM_BF16)                          \
      return ::exem::fail(EXEM_ERR_ARG,                                        \
                          "EXEM_VT_STORAGE needs a bf16/f16 tag (got %d)",     \
                          _tag);                                               \
    switch (_tag) {                                                            \
      case EXEM_F16:                                                           \
        if (_vs) { constexpr int DT = EXEM_F16; constexpr bool VS = true;      \
                   __VA_ARGS__; }                                              \
        else { constexpr int DT = EXEM_F16; constexpr bool VS = false;         \
               __VA_ARGS__; }                                                  \
        break;                                                                 \
      case EXEM_BF16:                                                          \
        if (_vs) { constexpr int DT = EXEM_BF16; constexpr bool VS = true;     \
                   __VA_ARGS__; }                                              \
        else { constexpr int DT = EXEM_BF16; constexpr bool VS = false;        \
               __VA_ARGS__; }                                                  \
        break;                                                                 \
      case EXEM_F32: { constexpr int DT = EXEM_F32; constexpr bool VS = false; \
                       __VA_ARGS__; break; }                                   \
      case EXEM_F64: { constexpr int DT = EXEM_F64; constexpr bool VS = false; \
                       __VA_ARGS__; break; }                                   \
      default:                                                                 \
        return ::exem::fail(EXEM_ERR_ARG, "unknown dtype tag %d", _tag);       \
    }                                                                          \
  } while (0)

#define EXEM_DISPATCH(dtype, DT, ...)                                          \
  switch (dtype) {                                                             \
    case EXEM_F16: { constexpr int DT = EXEM_F16; __VA_ARGS__; break; }        \
    case EXEM_BF16: { constexpr int DT = EXEM_BF16; __VA_ARGS__; break; }      \
    case EXEM_F32: { constexpr int DT = EXEM_F32; __VA_ARGS__; break; }        \
    case EXEM_F64: { constexpr int DT = EXEM_F64; __VA_ARGS__; break; }        \
    default:                                                                   \
      return ::exem::fail(EXEM_ERR_ARG, "unknown dtype tag %d", (int)dtype);   \
  }
