// Per-step latency of the v4 recurrences in isolation (1 CTA, 256 threads,
// warps 0..3 = two directions x two warps), clock64 around T steps.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../include -I../../paper_2304_05430_b200/csrc \
//        -o recprobe recprobe.cu && ./recprobe
#include <cstdio>
#include "tt_tuner_fast.cuh"

using namespace tt;

__global__ void __launch_bounds__(256, 1) probe(const float* Wh, int T, long long* out) {
  extern __shared__ float sm[];
  const int TM = 32;
  float* xz = sm;                       // [2][TM][128]
  float* S = xz + 2 * TM * kFG;         // [TM][64]
  float* gc = S + TM * kFD;             // [2][TM][128]
  float* cs = gc + 2 * TM * kFG;        // [2][TM][32]
  float* hb = cs + 2 * TM * kFH;        // 256
  float* gex = hb + 256;                // 512
  float* dS = gex + 512;                // [TM][64]
  float* dZ = dS + TM * kFD;            // [2][TM][128]
  float* Sg = dZ + 2 * TM * kFG;        // scratch "global" (smem here)
  float* Hg = Sg + TM * kFD;
  float* dZg = Hg + 2 * TM * kFH;
  for (int i = threadIdx.x; i < 2 * TM * kFG; i += 256) xz[i] = 0.01f * (i % 7);
  for (int i = threadIdx.x; i < TM * kFD; i += 256) dS[i] = 0.001f * (i % 5);
  __syncthreads();
  const int warp = threadIdx.x >> 5;
  if (warp < 4) {
    WReg w;
    load_wh_cols(w, Wh, warp & 1);
    __syncwarp();
    long long t0 = clock64();
    fast_rec_fwd(w, warp >> 1, warp & 1, T, TM, xz, S, Sg, Hg + (warp >> 1) * TM * kFH, gc, cs, hb, gex);
    long long t1 = clock64();
    WReg wr;
    load_wh_row(wr, Wh, warp & 1);
    named_barrier(1, 128);
    long long t2 = clock64();
    fast_rec_bwd(wr, warp >> 1, warp & 1, T, TM, gc, cs, dS, dZ, dZg + (warp >> 1) * TM * kFG, gex);
    long long t3 = clock64();
    if ((threadIdx.x & 31) == 0) {
      out[warp * 2] = t1 - t0;
      out[warp * 2 + 1] = t3 - t2;
    }
  }
}

int main() {
  float* Wh;
  long long* out;
  cudaMalloc(&Wh, 32 * 128 * 4);
  cudaMemset(Wh, 0, 32 * 128 * 4);
  cudaMalloc(&out, 64 * 8);
  const int smem = 200 * 1024;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int T : {1, 4, 8, 16, 32}) {
    for (int rep = 0; rep < 3; ++rep) probe<<<1, 256, smem>>>(Wh, T, out);
    cudaDeviceSynchronize();
    long long h[8];
    cudaMemcpy(h, out, 64, cudaMemcpyDeviceToHost);
    printf("T=%2d  fwd %6lld cyc (%.0f/step)   bwd %6lld cyc (%.0f/step)\n", T, h[0], h[0] / (double)T,
           h[1], h[1] / (double)T);
  }
  cudaError_t e = cudaGetLastError();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
