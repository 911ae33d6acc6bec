// Device building blocks shared by the fused training kernels and the
// standalone entry points: Adam update and the pairwise logistic loss.
#pragma once

#include "tt_common.cuh"

namespace tt {

// Exact-rounding arithmetic helpers: the float64 build must reproduce the
// reference's numpy evaluation order without FMA contraction.
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double div_rn(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float sub_rn(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ float div_rn(float a, float b) { return __fdiv_rn(a, b); }
__device__ __forceinline__ double sqrt_rn(double a) { return __dsqrt_rn(a); }
__device__ __forceinline__ float sqrt_rn(float a) { return __fsqrt_rn(a); }

struct AdamHyper {
  double lr, b1, b2, eps;
};

// optim.py:40-46, one element, in the reference's operation order:
//   m = m*b1 + (1-b1)*g ; v = v*b2 + ((1-b2)*g)*g
//   p = p - (lr * (m/c1)) / (sqrt(v/c2) + eps)
template <typename R>
__device__ __forceinline__ void adam_update(R& p, R g, R& m, R& v, const AdamHyper& h, double c1,
                                            double c2) {
  const R b1 = (R)h.b1, b2 = (R)h.b2, ob1 = (R)(1.0 - h.b1), ob2 = (R)(1.0 - h.b2);
  m = add_rn(mul_rn(m, b1), mul_rn(ob1, g));
  v = add_rn(mul_rn(v, b2), mul_rn(mul_rn(ob2, g), g));
  const R mh = div_rn(m, (R)c1);
  const R vh = div_rn(v, (R)c2);
  p = sub_rn(p, div_rn(mul_rn((R)h.lr, mh), add_rn(sqrt_rn(vh), (R)h.eps)));
}

// Pairwise logistic loss over one minibatch held in shared memory
// (mlp.py:25-35).  All threads of the block participate; writes dscore[k]
// for k < n and returns the loss to every thread.  Deterministic: the loss
// sum is reduced in a fixed tree order.  `red` must hold blockDim.x values.
template <typename R>
__device__ R rank_loss_block(const R* y, const R* s, int n, R* dscore, R* red) {
  if (n <= 32 && blockDim.x >= 32 * 4) {
    // small minibatch (the B = 16 training case): one pair per lane, rows
    // k = warp, warp + W, ..; per-row shuffle sums, rows summed in order.
    // `red` needs 2 n + 2 values.
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, W = blockDim.x >> 5;
    for (int k = warp; k < n; k += W) {
      const R yk = y[k], sk = s[k];
      R d = 0, part = 0, pairs = 0;
      if (lane < n) {
        const R yj = y[lane], sj = s[lane];
        if (yj > yk) d = (R)1 / ((R)1 + Act<R>::exp(sj - sk));
        if (yk > yj) {
          const R mg = sk - sj;
          d -= (R)1 / ((R)1 + Act<R>::exp(mg));
          part = Act<R>::softplus(-mg);
          pairs = (R)1;
        }
      }
      d = warp_sum(d);
      part = warp_sum(part);
      pairs = warp_sum(pairs);
      if (lane == 0) {
        dscore[k] = d;
        red[k] = part;
        red[n + k] = pairs;
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      R tp = 0, np = 0;
      for (int k = 0; k < n; ++k) {
        tp += red[k];
        np += red[n + k];
      }
      red[2 * n] = tp;
      red[2 * n + 1] = np;
    }
    __syncthreads();
    const R np = red[2 * n + 1];
    if ((int)threadIdx.x < n) dscore[threadIdx.x] = np == (R)0 ? (R)0 : dscore[threadIdx.x] / np;
    const R out = np == (R)0 ? (R)0 : red[2 * n] / np;
    __syncthreads();
    return out;
  }
  R part = 0;
  int pairs = 0;
  for (int k = threadIdx.x; k < n; k += blockDim.x) {
    const R yk = y[k], sk = s[k];
    R gin = 0, gout = 0;
    for (int j = 0; j < n; ++j) {
      const R yj = y[j], sj = s[j];
      if (yj > yk) {  // pair (j, k): j ranked above k, margin s_j - s_k
        gin += (R)1 / ((R)1 + Act<R>::exp(sj - sk));
      }
      if (yk > yj) {  // pair (k, j)
        const R mg = sk - sj;
        gout += (R)1 / ((R)1 + Act<R>::exp(mg));
        part += Act<R>::softplus(-mg);
        ++pairs;
      }
    }
    dscore[k] = gin - gout;  // scaled by 1/n_pairs below
  }
  // block-wide reductions (fixed order)
  red[threadIdx.x] = part;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  const R loss_sum = red[0];
  __syncthreads();
  red[threadIdx.x] = (R)pairs;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  const R npairs = red[0];
  __syncthreads();
  if (npairs == (R)0) {
    for (int k = threadIdx.x; k < n; k += blockDim.x) dscore[k] = 0;
    __syncthreads();
    return 0;
  }
  for (int k = threadIdx.x; k < n; k += blockDim.x) dscore[k] = dscore[k] / npairs;
  __syncthreads();
  return loss_sum / npairs;
}

// MSE over one minibatch in shared memory (tuner.py:373-375).
template <typename R>
__device__ R mse_block(const R* y, const R* s, int n, R* dscore, R* red) {
  R part = 0;
  for (int k = threadIdx.x; k < n; k += blockDim.x) {
    const R d = s[k] - y[k];
    part += d * d;
    dscore[k] = (R)2 * d / (R)n;
  }
  red[threadIdx.x] = part;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  const R out = red[0] / (R)n;
  __syncthreads();
  return out;
}

}  // namespace tt
