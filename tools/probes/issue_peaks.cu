// Issue-rate peaks of the pipes the scoring / PCA kernels are bound by
// (BASELINE.md §3 asks for the MUFU peak to be measured, not assumed):
//   MUFU.TANH (tanh.approx.f32), MUFU.EX2 (ex2.approx.f32), FP32 FFMA and
//   FP64 DFMA -- ops/s for the whole GPU.  (The rcp chain v = 1/v is folded
//   to a 2-cycle identity by the compiler and is not reported.)
// Every thread runs 8 independent dependency chains (enough ILP to saturate
// the pipe), all SMs x 8 CTAs x 256 threads, timed with CUDA events.
// Note: cudaDevAttrClockRate reports the boost clock; the run's actual SM
// clock is sampled by the caller (nvidia-smi) if per-clock rates matter.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o issue_peaks issue_peaks.cu && ./issue_peaks
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kIters = 4096;
constexpr int kChains = 8;

template <int OP>
__device__ __forceinline__ float op(float x) {
  float y;
  if constexpr (OP == 0) asm volatile("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  if constexpr (OP == 1) asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  if constexpr (OP == 2) asm volatile("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  if constexpr (OP == 3) y = fmaf(x, 0.999999f, 1e-7f);
  return y;
}

template <int OP>
__global__ void kern(float* out, float seed) {
  float v[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) v[c] = seed + 0.01f * (threadIdx.x + c);
  for (int i = 0; i < kIters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) v[c] = op<OP>(v[c]);
  }
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += v[c];
  if (s == 12345.f) out[threadIdx.x] = s;
}

__global__ void kern_d(double* out, double seed) {
  double v[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) v[c] = seed + 0.01 * (threadIdx.x + c);
  for (int i = 0; i < kIters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) v[c] = fma(v[c], 0.999999, 1e-7);
  }
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += v[c];
  if (s == 12345.0) out[threadIdx.x] = s;
}

template <typename F>
double time_ops(F launch, double ops) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  launch();
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a);
    launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  return ops / (best * 1e-3);
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);  // kHz
  float* out;
  cudaMalloc(&out, 4096 * sizeof(double));
  const int grid = sms * 8, block = 256;
  const double ops = (double)grid * block * kIters * kChains;
  const double hz = clk * 1e3;
  const char* names[4] = {"mufu_tanh", "mufu_ex2", "mufu_rcp", "fp32_ffma"};
  double r[5];
  r[0] = time_ops([&] { kern<0><<<grid, block>>>(out, 0.3f); }, ops);
  r[1] = time_ops([&] { kern<1><<<grid, block>>>(out, 0.3f); }, ops);
  r[2] = time_ops([&] { kern<2><<<grid, block>>>(out, 1.3f); }, ops);
  r[3] = time_ops([&] { kern<3><<<grid, block>>>(out, 0.3f); }, ops);
  r[4] = time_ops([&] { kern_d<<<grid, block>>>((double*)out, 0.3); }, ops);
  printf("{\"sms\": %d, \"clock_mhz\": %.0f", sms, hz / 1e6);
  for (int i = 0; i < 4; ++i)
    printf(", \"%s_ops_per_s\": %.4g, \"%s_per_sm_per_clk\": %.2f", names[i], r[i], names[i],
           r[i] / sms / hz);
  printf(", \"fp64_dfma_ops_per_s\": %.4g, \"fp64_dfma_per_sm_per_clk\": %.2f", r[4], r[4] / sms / hz);
  printf(", \"fp32_tflops\": %.2f}\n", 2 * r[3] / 1e12);
  return 0;
}
