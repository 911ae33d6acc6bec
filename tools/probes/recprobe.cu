// Per-step latency of the v4 recurrences in isolation (1 CTA, 256 threads,
// warps 0..3 = two directions x two warps), clock64 around T steps.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../include -I../../paper_2304_05430_b200/csrc \
//        -o recprobe recprobe.cu && ./recprobe
#include <cstdio>
#include "tt_tuner_fast.cuh"

using namespace tt;

__device__ __forceinline__ void rec_fwd_v2(const WReg& w, int dir, int sub, int T, int TM,
                                             const float* xz, float* S, float* Sg, float* Hg,
                                             float* gc, float* cs, float* hb, float* gex) {
  const int j = threadIdx.x & 31;
  float c = 0.f;
  float* hm = hb + (dir * 2 + sub) * 2 * kFH;          // [parity][32]
  float* gx_me = gex + (dir * 2 + sub) * 2 * 2 * kFH;  // [parity][64]
  const float* gx_ot = gex + (dir * 2 + (sub ^ 1)) * 2 * 2 * kFH;
  hm[j] = 0.f;
  __syncwarp();
  for (int s = 0; s < T; ++s) {
    const int par = s & 1;
    const int t = dir == 0 ? s : T - 1 - s;
    const float* xr = xz + ((int64_t)dir * TM + t) * kFG + 2 * sub * kFH;
    float a[8] = {xr[j], 0.f, 0.f, 0.f, xr[kFH + j], 0.f, 0.f, 0.f};
    const float4* h4 = reinterpret_cast<const float4*>(hm + par * kFH);
#pragma unroll
    for (int m = 0; m < kFH / 4; ++m) {
      const float4 u = h4[m];
      const int q = m & 3;
      a[q] = fmaf(u.x, w[4 * m + 0], a[q]);
      a[4 + q] = fmaf(u.x, w[kFH + 4 * m + 0], a[4 + q]);
      a[q] = fmaf(u.y, w[4 * m + 1], a[q]);
      a[4 + q] = fmaf(u.y, w[kFH + 4 * m + 1], a[4 + q]);
      a[q] = fmaf(u.z, w[4 * m + 2], a[q]);
      a[4 + q] = fmaf(u.z, w[kFH + 4 * m + 2], a[4 + q]);
      a[q] = fmaf(u.w, w[4 * m + 3], a[q]);
      a[4 + q] = fmaf(u.w, w[kFH + 4 * m + 3], a[4 + q]);
    }
    const float a00 = (a[0] + a[1]) + (a[2] + a[3]), a01 = 0.f;
    const float a10 = (a[4] + a[5]) + (a[6] + a[7]), a11 = 0.f;
    const float z0 = a00 + a01, z1 = a10 + a11;
    // sub 0: (i, f) = sigmoid; sub 1: g = tanh, o = sigmoid
    const float v0 = sub == 0 ? fsig(z0) : ftanh(z0);
    const float v1 = fsig(z1);
    float* gr = gc + ((int64_t)dir * TM + t) * kFG + 2 * sub * kFH;
    gr[j] = v0;
    gr[kFH + j] = v1;
    gx_me[par * 2 * kFH + j] = v0;
    gx_me[par * 2 * kFH + kFH + j] = v1;
    named_barrier(2 + dir, 64);
    const float o0 = gx_ot[par * 2 * kFH + j], o1 = gx_ot[par * 2 * kFH + kFH + j];
    const float gi = sub == 0 ? v0 : o0, gf = sub == 0 ? v1 : o1;
    const float gg = sub == 0 ? o0 : v0, go = sub == 0 ? o1 : v1;
    c = gf * c + gi * gg;
    const float h = go * ftanh(c);
    hm[(par ^ 1) * kFH + j] = h;
    if (sub == 0) {
      S[(int64_t)t * kFD + dir * kFH + j] = h;
      Sg[(int64_t)t * kFD + dir * kFH + j] = h;
      cs[((int64_t)dir * TM + t) * kFH + j] = c;
    } else {
      // h_prev rows of the stacked exchange, in the direction's order
      if (s == 0) Hg[(int64_t)t * kFH + j] = 0.f;
      if (s + 1 < T) Hg[(int64_t)(dir == 0 ? t + 1 : t - 1) * kFH + j] = h;
    }
    __syncwarp();
  }
}



__device__ __forceinline__ float atanh_(float x) { float y; asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ float asig(float x) { return fmaf(0.5f, atanh_(0.5f * x), 0.5f); }
__device__ __forceinline__ void rec_fwd_v3(const WReg& w, int dir, int sub, int T, int TM,
                                             const float* xz, float* S, float* Sg, float* Hg,
                                             float* gc, float* cs, float* hb, float* gex) {
  const int j = threadIdx.x & 31;
  float c = 0.f;
  float* hm = hb + (dir * 2 + sub) * 2 * kFH;          // [parity][32]
  float* gx_me = gex + (dir * 2 + sub) * 2 * 2 * kFH;  // [parity][64]
  const float* gx_ot = gex + (dir * 2 + (sub ^ 1)) * 2 * 2 * kFH;
  hm[j] = 0.f;
  __syncwarp();
  for (int s = 0; s < T; ++s) {
    const int par = s & 1;
    const int t = dir == 0 ? s : T - 1 - s;
    const float* xr = xz + ((int64_t)dir * TM + t) * kFG + 2 * sub * kFH;
    float a[8] = {xr[j], 0.f, 0.f, 0.f, xr[kFH + j], 0.f, 0.f, 0.f};
    const float4* h4 = reinterpret_cast<const float4*>(hm + par * kFH);
#pragma unroll
    for (int m = 0; m < kFH / 4; ++m) {
      const float4 u = h4[m];
      const int q = m & 3;
      a[q] = fmaf(u.x, w[4 * m + 0], a[q]);
      a[4 + q] = fmaf(u.x, w[kFH + 4 * m + 0], a[4 + q]);
      a[q] = fmaf(u.y, w[4 * m + 1], a[q]);
      a[4 + q] = fmaf(u.y, w[kFH + 4 * m + 1], a[4 + q]);
      a[q] = fmaf(u.z, w[4 * m + 2], a[q]);
      a[4 + q] = fmaf(u.z, w[kFH + 4 * m + 2], a[4 + q]);
      a[q] = fmaf(u.w, w[4 * m + 3], a[q]);
      a[4 + q] = fmaf(u.w, w[kFH + 4 * m + 3], a[4 + q]);
    }
    const float a00 = (a[0] + a[1]) + (a[2] + a[3]), a01 = 0.f;
    const float a10 = (a[4] + a[5]) + (a[6] + a[7]), a11 = 0.f;
    const float z0 = a00 + a01, z1 = a10 + a11;
    // sub 0: (i, f) = sigmoid; sub 1: g = tanh, o = sigmoid
    const float v0 = sub == 0 ? fsig(z0) : ftanh(z0);
    const float v1 = fsig(z1);
    float* gr = gc + ((int64_t)dir * TM + t) * kFG + 2 * sub * kFH;

    gx_me[par * 2 * kFH + j] = v0;
    gx_me[par * 2 * kFH + kFH + j] = v1;
    named_barrier(2 + dir, 64);
    const float o0 = gx_ot[par * 2 * kFH + j], o1 = gx_ot[par * 2 * kFH + kFH + j];
    const float gi = sub == 0 ? v0 : o0, gf = sub == 0 ? v1 : o1;
    const float gg = sub == 0 ? o0 : v0, go = sub == 0 ? o1 : v1;
    c = gf * c + gi * gg;
    const float h = go * ftanh(c);
    hm[(par ^ 1) * kFH + j] = h;

    __syncwarp();
  }
}



__device__ __forceinline__ void rec_fwd_v4(const WReg& w, int dir, int sub, int T, int TM,
                                             const float* xz, float* S, float* Sg, float* Hg,
                                             float* gc, float* cs, float* hb, float* gex) {
  const int j = threadIdx.x & 31;
  float c = 0.f;
  float* hm = hb + (dir * 2 + sub) * 2 * kFH;          // [parity][32]
  float* gx_me = gex + (dir * 2 + sub) * 2 * 2 * kFH;  // [parity][64]
  const float* gx_ot = gex + (dir * 2 + (sub ^ 1)) * 2 * 2 * kFH;
  hm[j] = 0.f;
  __syncwarp();
  for (int s = 0; s < T; ++s) {
    const int par = s & 1;
    const int t = dir == 0 ? s : T - 1 - s;
    const float* xr = xz + ((int64_t)dir * TM + t) * kFG + 2 * sub * kFH;
    float a[8] = {xr[j], 0.f, 0.f, 0.f, xr[kFH + j], 0.f, 0.f, 0.f};
    const float4* h4 = reinterpret_cast<const float4*>(hm + par * kFH);
#pragma unroll
    for (int m = 0; m < kFH / 4; ++m) {
      const float4 u = h4[m];
      const int q = m & 3;
      a[q] = fmaf(u.x, w[4 * m + 0], a[q]);
      a[4 + q] = fmaf(u.x, w[kFH + 4 * m + 0], a[4 + q]);
      a[q] = fmaf(u.y, w[4 * m + 1], a[q]);
      a[4 + q] = fmaf(u.y, w[kFH + 4 * m + 1], a[4 + q]);
      a[q] = fmaf(u.z, w[4 * m + 2], a[q]);
      a[4 + q] = fmaf(u.z, w[kFH + 4 * m + 2], a[4 + q]);
      a[q] = fmaf(u.w, w[4 * m + 3], a[q]);
      a[4 + q] = fmaf(u.w, w[kFH + 4 * m + 3], a[4 + q]);
    }
    const float a00 = (a[0] + a[1]) + (a[2] + a[3]), a01 = 0.f;
    const float a10 = (a[4] + a[5]) + (a[6] + a[7]), a11 = 0.f;
    const float z0 = a00 + a01, z1 = a10 + a11;
    // sub 0: (i, f) = sigmoid; sub 1: g = tanh, o = sigmoid
    const float v0 = sub == 0 ? asig(z0) : atanh_(z0);
    const float v1 = asig(z1);
    float* gr = gc + ((int64_t)dir * TM + t) * kFG + 2 * sub * kFH;
    gr[j] = v0;
    gr[kFH + j] = v1;
    gx_me[par * 2 * kFH + j] = v0;
    gx_me[par * 2 * kFH + kFH + j] = v1;
    named_barrier(2 + dir, 64);
    const float o0 = gx_ot[par * 2 * kFH + j], o1 = gx_ot[par * 2 * kFH + kFH + j];
    const float gi = sub == 0 ? v0 : o0, gf = sub == 0 ? v1 : o1;
    const float gg = sub == 0 ? o0 : v0, go = sub == 0 ? o1 : v1;
    c = gf * c + gi * gg;
    const float h = go * atanh_(c);
    hm[(par ^ 1) * kFH + j] = h;
    if (sub == 0) {
      S[(int64_t)t * kFD + dir * kFH + j] = h;
      Sg[(int64_t)t * kFD + dir * kFH + j] = h;
      cs[((int64_t)dir * TM + t) * kFH + j] = c;
    } else {
      // h_prev rows of the stacked exchange, in the direction's order
      if (s == 0) Hg[(int64_t)t * kFH + j] = 0.f;
      if (s + 1 < T) Hg[(int64_t)(dir == 0 ? t + 1 : t - 1) * kFH + j] = h;
    }
    __syncwarp();
  }
}



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
    named_barrier(1, 128);
    long long t4 = clock64();
    rec_fwd_v2(w, warp >> 1, warp & 1, T, TM, xz, S, Sg, Hg + (warp >> 1) * TM * kFH, gc, cs, hb, gex);
    long long t5 = clock64();
    if ((threadIdx.x & 31) == 0) out[16 + warp] = t5 - t4;
    named_barrier(1, 128);
    long long t6 = clock64();
    rec_fwd_v3(w, warp >> 1, warp & 1, T, TM, xz, S, Sg, Hg + (warp >> 1) * TM * kFH, gc, cs, hb, gex);
    long long t7 = clock64();
    named_barrier(1, 128);
    long long t8 = clock64();
    rec_fwd_v4(w, warp >> 1, warp & 1, T, TM, xz, S, Sg, Hg + (warp >> 1) * TM * kFH, gc, cs, hb, gex);
    long long t9 = clock64();
    if ((threadIdx.x & 31) == 0) { out[20 + warp] = t7 - t6; out[24 + warp] = t9 - t8; }
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
    long long h[32];
    cudaMemcpy(h, out, 32 * 8, cudaMemcpyDeviceToHost);
    printf("T=%2d  fwd %6lld cyc (%.0f/step)   bwd %6lld cyc (%.0f/step)   fwd_v2 %.0f v3(no stores) %.0f v4(approx) %.0f\n", T, h[0],
           h[0] / (double)T, h[1], h[1] / (double)T, h[16] / (double)T, h[20] / (double)T, h[24] / (double)T);
  }
  cudaError_t e = cudaGetLastError();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
