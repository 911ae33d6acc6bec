// L2 staging probe: how long does a CTA take to pull ~48 KB that 16 other
// CTAs just wrote, via cp.async (16 B) vs ld.global.cg + st.shared?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2probe l2probe.cu && ./l2probe
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned ld_acq(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void cpa16(float* s, const float* g) {
  unsigned sa = (unsigned)__cvta_generic_to_shared(s);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(g) : "memory");
}

constexpr int kSlotFloats = 11520;  // 46 KB per slot
constexpr int kRowsPerSlot = 10, kRowFloats = 112;  // what one job reads per slot

__global__ void __launch_bounds__(256, 1) probe(float* slots, unsigned* ctr, unsigned long long* out,
                                                int mode, int rounds) {
  extern __shared__ float sm[];
  const int tid = threadIdx.x;
  for (int rd = 0; rd < rounds; ++rd) {
    // writers: CTAs 0..15 fill their slot
    if (blockIdx.x < 16) {
      float* s = slots + (size_t)blockIdx.x * kSlotFloats;
      for (int i = tid; i < kSlotFloats; i += 256) s[i] = (float)(i + rd);
      __syncthreads();
      if (tid == 0) { __threadfence(); atomicAdd(ctr, 1u); }
    }
    if (tid == 0) while (ld_acq(ctr) < 16u * (rd + 1)) {}
    __syncthreads();
    unsigned long long t0 = gtime();
    // reader: 16 slots x 10 rows x 112 floats (row stride 128 floats), offset by CTA
    const int off = (blockIdx.x % 8) * 8;
    if (mode == 0) {
      for (int k = 0; k < 16; ++k) {
        const float* s = slots + (size_t)k * kSlotFloats + off;
        for (int i = tid; i < kRowsPerSlot * (kRowFloats / 4); i += 256) {
          const int r = i / (kRowFloats / 4), q = i % (kRowFloats / 4);
          cpa16(sm + (k * kRowsPerSlot + r) * kRowFloats + q * 4, s + r * 128 * 8 + q * 4);
        }
      }
      asm volatile("cp.async.wait_all;" ::: "memory");
    } else if (mode == 1) {
      // flat: all (slot,row,chunk) items, 8 loads in flight per thread
      const int per = kRowsPerSlot * (kRowFloats / 4), tot = 16 * per;
      for (int i0 = tid; i0 < tot; i0 += 256 * 8) {
        float4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int i = i0 + u * 256;
          if (i < tot) {
            const int k = i / per, rem = i % per, r = rem / (kRowFloats / 4), q = rem % (kRowFloats / 4);
            v[u] = __ldcg(reinterpret_cast<const float4*>(slots + (size_t)k * kSlotFloats + off + r * 128 * 8 + q * 4));
          }
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int i = i0 + u * 256;
          if (i < tot) *reinterpret_cast<float4*>(sm + i * 4) = v[u];
        }
      }
    } else {
      // flat cp.async
      const int per = kRowsPerSlot * (kRowFloats / 4), tot = 16 * per;
      for (int i = tid; i < tot; i += 256) {
        const int k = i / per, rem = i % per, r = rem / (kRowFloats / 4), q = rem % (kRowFloats / 4);
        cpa16(sm + i * 4, slots + (size_t)k * kSlotFloats + off + r * 128 * 8 + q * 4);
      }
      asm volatile("cp.async.wait_all;" ::: "memory");
    }
    __syncthreads();
    unsigned long long t1 = gtime();
    if (tid == 0) out[(size_t)rd * gridDim.x + blockIdx.x] = t1 - t0;
    // everyone done before the next round's writes
    __syncthreads();
    if (tid == 0) { __threadfence(); atomicAdd(ctr + 1, 1u); while (ld_acq(ctr + 1) < gridDim.x * (rd + 1)) {} }
    __syncthreads();
  }
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  float* slots;
  unsigned* ctr;
  unsigned long long* out;
  const int rounds = 20;
  cudaMalloc(&slots, 16 * kSlotFloats * 4 + 4096);
  cudaMalloc(&ctr, 64);
  cudaMalloc(&out, rounds * nsm * 8);
  const int smem = 16 * kRowsPerSlot * kRowFloats * 4;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int mode = 0; mode < 3; ++mode) {
    cudaMemset(ctr, 0, 64);
    void* args[] = {&slots, &ctr, &out, (void*)&mode, (void*)&rounds};
    cudaError_t e = cudaLaunchCooperativeKernel((void*)probe, nsm, 256, args, 200 * 1024, 0);
    cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
    std::vector<unsigned long long> h(rounds * nsm);
    cudaMemcpy(h.data(), out, h.size() * 8, cudaMemcpyDeviceToHost);
    std::vector<unsigned long long> v(h.begin() + 5 * nsm, h.end());
    std::sort(v.begin(), v.end());
    printf("mode %d (%s): %d KB per CTA: median %.2f us  p90 %.2f us  max %.2f us\n", mode,
           mode == 0 ? "cp.async per-slot loops" : mode == 1 ? "ldcg x8 in flight" : "cp.async flat",
           smem / 1024, v[v.size() / 2] / 1e3, v[v.size() * 9 / 10] / 1e3, v.back() / 1e3);
  }
  return 0;
}
