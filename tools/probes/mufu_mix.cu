// MUFU throughput for rcp.approx and an ex2/rcp mix (the LSTM epilogue's
// instruction mix): 8 independent chains per thread, x = mufu(fma(x, a, b)),
// 148 x 8 blocks of 256 threads.  Prints ops per SM per clock at the clock
// the driver reports.
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void k(float* out, int iters, float a, float b) {
  float x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3f + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      float y = fmaf(x[i], a, b), z;
      if constexpr (OP == 0) asm volatile("rcp.approx.ftz.f32 %0, %1;" : "=f"(z) : "f"(y));
      if constexpr (OP == 1) asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(z) : "f"(y));
      if constexpr (OP == 2) {  // 5 ex2 : 3 rcp
        if (i < 5) asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(z) : "f"(y));
        else asm volatile("rcp.approx.ftz.f32 %0, %1;" : "=f"(z) : "f"(y));
      }
      x[i] = z;
    }
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 12345.f) out[0] = s;
}

template <int OP>
static void run(const char* name, int sms, double mhz) {
  float* out;
  cudaMalloc(&out, 4);
  const int iters = 4096, blocks = sms * 8, threads = 256;
  k<OP><<<blocks, threads>>>(out, 16, 0.999f, 0.001f);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<OP><<<blocks, threads>>>(out, iters, 0.999f, 0.001f);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double ops = (double)blocks * threads * iters * 8;
  printf("{\"op\": \"%s\", \"ops_per_s\": %.4g, \"per_sm_per_clk\": %.2f}\n", name, ops / (ms * 1e-3),
         ops / (ms * 1e-3) / sms / (mhz * 1e6));
  cudaFree(out);
}

int main() {
  int dev = 0, sms = 0, khz = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, dev);
  const double mhz = khz / 1000.0;
  run<0>("rcp.approx.ftz", sms, mhz);
  run<1>("ex2.approx.ftz", sms, mhz);
  run<2>("ex2:rcp 5:3", sms, mhz);
  return 0;
}
