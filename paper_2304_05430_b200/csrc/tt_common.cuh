// Shared device/host helpers for libtt_b200 (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <cmath>

#include "../../include/tt_b200.h"

namespace tt {

// ---------------------------------------------------------------- errors --
void set_error(const char* fmt, ...);
int check_launch(const char* what);

#define TT_REQUIRE(cond, ...)        \
  do {                               \
    if (!(cond)) {                   \
      ::tt::set_error(__VA_ARGS__);  \
      return TT_EINVAL;              \
    }                                \
  } while (0)

#define TT_CUDA(call)                                                           \
  do {                                                                          \
    cudaError_t e__ = (call);                                                   \
    if (e__ != cudaSuccess) {                                                   \
      ::tt::set_error("%s failed: %s", #call, cudaGetErrorString(e__));        \
      return TT_ECUDA;                                                          \
    }                                                                           \
  } while (0)

inline cudaStream_t as_stream(tt_stream_t s) { return reinterpret_cast<cudaStream_t>(s); }

inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

int sm_count();

// Raise a kernel's dynamic shared-memory limit to at least `smem` -- never
// lower it: host threads scoring concurrently launch the same kernel with
// different sizes, and a lowered limit fails the larger launch -- and report
// its resident CTAs per SM for (threads, smem).  Both are cached per
// (device, kernel): the CUDA calls cost microseconds of host time a
// one-program scoring call would otherwise pay every time (tt_base.cu).
int kernel_smem(const void* kern, size_t smem);
int kernel_occupancy(const void* kern, int threads, size_t smem, int* per_sm);

// ------------------------------------------------------------ arithmetic --
// Activations.  float: ex2.approx-based exp + approximate reciprocal, error a
// few ulp (well inside the 1e-5 score tolerance; tanh.approx's 5e-4 is not).
// double: libdevice exp/tanh, matching numpy to ~1 ulp.
template <typename R>
struct Act;

template <>
struct Act<float> {
  // MUFU ex2 / rcp in their flush-to-zero forms: the same two SFU ops as
  // __expf / __fdividef without the denormal-range fix-ups, which these
  // activations never need (1 + e^{...} >= 1; e^{x} below 2^-126 is 0 here
  // as in any fp32 sum it is added to).
  static __device__ __forceinline__ float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
  }
  static __device__ __forceinline__ float rcp(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
  }
  static __device__ __forceinline__ float sigmoid(float x) {
    return rcp(1.0f + ex2(-1.4426950408889634f * x));
  }
  static __device__ __forceinline__ float tanh(float x) {
    // 1 - 2/(e^{2x}+1): exact limits at +-inf, absolute error ~1e-7.
    return 1.0f - 2.0f * rcp(ex2(2.8853900817779268f * x) + 1.0f);
  }
  static __device__ __forceinline__ float exp(float x) { return ex2(1.4426950408889634f * x); }
  static __device__ __forceinline__ float softplus(float x) {
    // log(1 + e^x) computed as max(x,0) + log1p(e^-|x|)  (np.logaddexp(0, x))
    return fmaxf(x, 0.0f) + log1pf(__expf(-fabsf(x)));
  }
  static __device__ __forceinline__ float rsqrt(float x) { return rsqrtf(x); }
};

template <>
struct Act<double> {
  static __device__ __forceinline__ double sigmoid(double x) {
    // tuner.py:27-33 split form
    if (x >= 0.0) return 1.0 / (1.0 + ::exp(-x));
    double e = ::exp(x);
    return e / (1.0 + e);
  }
  static __device__ __forceinline__ double tanh(double x) { return ::tanh(x); }
  static __device__ __forceinline__ double exp(double x) { return ::exp(x); }
  static __device__ __forceinline__ double softplus(double x) {
    return fmax(x, 0.0) + log1p(::exp(-fabs(x)));
  }
  static __device__ __forceinline__ double rsqrt(double x) { return 1.0 / ::sqrt(x); }
};

// Explicitly fused multiply-add: an expression like a*b + c*d leaves the
// compiler free to contract either product, and the choice can differ between
// template instances (tile sizes) -- spelling the FMA out keeps a program's
// arithmetic identical in every instance.
__device__ __forceinline__ float fma_rn(float a, float b, float c) { return __fmaf_rn(a, b, c); }
__device__ __forceinline__ double fma_rn(double a, double b, double c) { return __fma_rn(a, b, c); }

// ------------------------------------------------------------- reductions --
template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <typename T>
__device__ __forceinline__ T warp_max(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    T w = __shfl_xor_sync(0xffffffffu, v, o);
    v = w > v ? w : v;
  }
  return v;
}

// Named barrier over `count` threads (multiple of 32); id 0 is __syncthreads.
// The non-.aligned form: warp-specialised kernels meet on one barrier id from
// different code locations (e.g. recurrence warps and prefetch warps), which
// the .aligned form (bar.sync) does not allow (PTX ISA: every thread of the
// CTA must execute the same aligned barrier instruction; compute-sanitizer
// synccheck flags it).
__device__ __forceinline__ void named_barrier(int id, int count) {
  asm volatile("barrier.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

// Software grid barrier for cooperative (co-resident) launches.  `ctr` is a
// zero-initialised counter; `target` advances by gridDim.x per barrier.
__device__ __forceinline__ void grid_barrier(unsigned int* ctr, unsigned int& target) {
  __syncthreads();
  target += gridDim.x;
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(ctr, 1u);
    unsigned int v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
    } while (v < target);
    __threadfence();
  }
  __syncthreads();
}

}  // namespace tt
