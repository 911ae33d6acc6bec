// K2 pruning statistics (sampling.py:37-59 filter_invalid + data.py:440-446
// throughput + numpy's linear quantile), bit-exact in float64.
//
// One CTA per task.  Throughput tp = double(flops) / cost (IEEE division,
// round-to-nearest int64->double, like Python's int / float).  The two order
// statistics the linear quantile needs are found by an 8-pass MSB radix
// select over order-preserving 64-bit keys (smem histograms with integer
// atomics -> order independent), then numpy's _lerp is evaluated with
// explicit round-to-nearest operations (no FMA contraction):
//   vi = (n-1)*q ; lo = floor(vi) ; t = vi - lo ; d = b - a
//   thr = t >= 0.5 ? b - d*(1-t) : a + d*t      (vi >= n-1 -> max)
// Survivors are valid records with tp >= thr; the task is kept iff
// survivors >= min_records.
#include "tt_ops.cuh"

namespace tt {

__device__ __forceinline__ double tput(const int64_t* flops, const double* cost, int64_t i) {
  return __ddiv_rn(__ll2double_rn(flops[i]), cost[i]);
}

__device__ __forceinline__ unsigned long long okey(double v) {
  if (v == 0.0) v = 0.0;  // -0 and +0 compare equal in np.sort
  const unsigned long long b = (unsigned long long)__double_as_longlong(v);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

__device__ __forceinline__ double unkey(unsigned long long k) {
  const unsigned long long b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
  return __longlong_as_double((long long)b);
}

// k-th smallest (0-based) key among valid records of [a, a+n)
__device__ unsigned long long radix_select(const int64_t* flops, const double* cost,
                                           const uint8_t* valid, int64_t a, int64_t n, int64_t k,
                                           unsigned int* hist) {
  unsigned long long prefix = 0, mask = 0;
  for (int shift = 56; shift >= 0; shift -= 8) {
    for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
      if (!valid[a + i]) continue;
      const unsigned long long key = okey(tput(flops, cost, a + i));
      if ((key & mask) == prefix) atomicAdd(&hist[(key >> shift) & 0xff], 1u);
    }
    __syncthreads();
    // every thread scans the 256 bins (cheap, avoids another barrier round)
    int64_t run = 0;
    int bin = 255;
    for (int b = 0; b < 256; ++b) {
      const int64_t c = hist[b];
      if (run + c > k) {
        bin = b;
        break;
      }
      run += c;
    }
    k -= run;
    prefix |= (unsigned long long)bin << shift;
    mask |= 0xffull << shift;
    __syncthreads();
  }
  return prefix;
}

__global__ void __launch_bounds__(256) prune_stats_kernel(
    const int64_t* __restrict__ flops, const double* __restrict__ cost,
    const uint8_t* __restrict__ valid, const int64_t* __restrict__ toff, double q, int min_records,
    double* __restrict__ thr_out, uint8_t* __restrict__ keep, int32_t* __restrict__ surv_out,
    uint8_t* __restrict__ task_keep) {
  __shared__ unsigned int hist[256];
  __shared__ int red[8];
  const int task = blockIdx.x;
  const int64_t a = toff[task];
  const int64_t n = toff[task + 1] - a;
  // count valid records
  int cnt = 0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) cnt += valid[a + i] ? 1 : 0;
  cnt = warp_sum(cnt);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = cnt;
  __syncthreads();
  int64_t nv = 0;
  for (int w = 0; w < 8; ++w) nv += red[w];
  __syncthreads();
  if (nv == 0) {
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) keep[a + i] = 0;
    if (threadIdx.x == 0) {
      thr_out[task] = __longlong_as_double(0x7ff8000000000000ll);
      surv_out[task] = 0;
      task_keep[task] = 0;
    }
    return;
  }
  const double vi = __dmul_rn((double)(nv - 1), q);
  double thr;
  if (vi >= (double)(nv - 1)) {
    thr = unkey(radix_select(flops, cost, valid, a, n, nv - 1, hist));
  } else if (vi < 0.0) {
    thr = unkey(radix_select(flops, cost, valid, a, n, 0, hist));
  } else {
    const double lo = floor(vi);
    const double t = __dsub_rn(vi, lo);
    const double va = unkey(radix_select(flops, cost, valid, a, n, (int64_t)lo, hist));
    const double vb = unkey(radix_select(flops, cost, valid, a, n, (int64_t)lo + 1, hist));
    const double d = __dsub_rn(vb, va);
    thr = t >= 0.5 ? __dsub_rn(vb, __dmul_rn(d, __dsub_rn(1.0, t))) : __dadd_rn(va, __dmul_rn(d, t));
  }
  int s = 0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x)
    s += (valid[a + i] && tput(flops, cost, a + i) >= thr) ? 1 : 0;
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  int64_t surv = 0;
  for (int w = 0; w < 8; ++w) surv += red[w];
  const bool tk = surv >= min_records;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x)
    keep[a + i] = (tk && valid[a + i] && tput(flops, cost, a + i) >= thr) ? 1 : 0;
  if (threadIdx.x == 0) {
    thr_out[task] = thr;
    surv_out[task] = (int32_t)surv;
    task_keep[task] = tk ? 1 : 0;
  }
}

}  // namespace tt

using namespace tt;

extern "C" {

size_t tt_prune_workspace_bytes(int64_t n_records) {
  (void)n_records;
  return 0;
}

int tt_prune_stats(const int64_t* flops, const double* cost, const uint8_t* valid,
                   const int64_t* toff, int32_t n_tasks, double q, int32_t min_records,
                   double* thr, uint8_t* keep, int32_t* surv, uint8_t* task_keep, void* ws,
                   size_t ws_bytes, tt_stream_t st) {
  (void)ws;
  (void)ws_bytes;
  TT_REQUIRE(n_tasks >= 0, "prune: negative task count");
  TT_REQUIRE(q >= 0.0 && q < 1.0, "prune: quantile must be in [0, 1)");
  if (n_tasks == 0) return TT_OK;
  prune_stats_kernel<<<n_tasks, 256, 0, as_stream(st)>>>(flops, cost, valid, toff, q, min_records,
                                                          thr, keep, surv, task_keep);
  return check_launch("prune stats");
}

}  // extern "C"
