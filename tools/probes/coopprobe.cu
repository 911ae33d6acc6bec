// Can two cooperative kernels (half the SMs each, two streams, one process)
// run concurrently and hand flags to each other?  Bounded spins: no hang.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o coopprobe coopprobe.cu && ./coopprobe
#include <cstdio>
__global__ void pingpong(unsigned* mine, unsigned* other, int rounds, int* ok) {
  for (int r = 1; r <= rounds; ++r) {
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence_system();
      atomicAdd(other + blockIdx.x % 4, 0);  // touch
      asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(other + 64 + blockIdx.x), "r"((unsigned)r) : "memory");
      long long spins = 0;
      unsigned v;
      do {
        asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(mine + 64 + blockIdx.x) : "memory");
      } while (v < (unsigned)r && ++spins < 20000000);
      if (v < (unsigned)r) atomicExch(ok, 0);
    }
    __syncthreads();
  }
}
int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned *a, *b;
  int* ok;
  cudaMalloc(&a, 4096);
  cudaMalloc(&b, 4096);
  cudaMalloc(&ok, 4);
  cudaMemset(a, 0, 4096);
  cudaMemset(b, 0, 4096);
  int one = 1;
  cudaMemcpy(ok, &one, 4, cudaMemcpyHostToDevice);
  cudaStream_t s1, s2;
  cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
  cudaFuncSetAttribute(pingpong, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  const int grid = sms / 2, rounds = 1000;
  void* args1[] = {&a, &b, (void*)&rounds, &ok};
  void* args2[] = {&b, &a, (void*)&rounds, &ok};
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, s1);
  cudaError_t r1 = cudaLaunchCooperativeKernel((void*)pingpong, grid, 256, args1, 160 * 1024, s1);
  cudaError_t r2 = cudaLaunchCooperativeKernel((void*)pingpong, grid, 256, args2, 160 * 1024, s2);
  cudaDeviceSynchronize();
  cudaEventRecord(e1, s1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  int h = 0;
  cudaMemcpy(&h, ok, 4, cudaMemcpyDeviceToHost);
  printf("launch %s / %s, ok=%d, %.3f ms for %d rounds (%.2f us/round)  err=%s\n", cudaGetErrorString(r1),
         cudaGetErrorString(r2), h, ms, rounds, ms * 1000 / rounds, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
