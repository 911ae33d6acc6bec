// CostMLP kernels (estimators/mlp.py:72-144): K3 scoring and the fused
// single-CTA training loop (K4 forward/backward + K7 loss + K8 Adam per
// minibatch, one launch per epoch).
//
// Scoring: a CTA owns 64-row tiles (persistent grid).  X and W1 stream
// through shared memory in 64-wide K chunks; each thread keeps a 4x4 register
// tile of the 64x64 hidden pre-activations, tanh is fused into the epilogue,
// the 64x64 second layer reuses the same tiling from shared memory and the
// 64->1 output is a per-row dot product.  This CUDA-core tile is the
// correctness baseline for the tcgen05 version.
#include <type_traits>

#include "tt_ops.cuh"

namespace tt {

constexpr int kMT = 256;   // threads
constexpr int kW = 64;     // hidden width (mlp.py:17)
constexpr int kTile = 64;  // rows per tile
constexpr int kKc = 64;    // K chunk

struct MOff {
  int64_t W1, b1, W2, b2, W3, b3, total;
};

inline __host__ __device__ MOff mlp_offsets(int F) {
  MOff o;
  o.W1 = 0;
  o.b1 = (int64_t)F * kW;
  o.W2 = o.b1 + kW;
  o.b2 = o.W2 + kW * kW;
  o.W3 = o.b2 + kW;
  o.b3 = o.W3 + kW;
  o.total = o.b3 + 1;
  return o;
}

template <typename R>
struct MlpSmem {
  R xs[kTile][kKc + 1];
  R ws[kKc][kW + 4];
  R h1[kTile][kW + 1];
  R h2[kTile][kW + 1];
};

// Forward of up to 64 rows; row r of the tile is X[rowidx(r)].  Leaves tanh
// activations in sm.h1/sm.h2 and writes out_rows[r] for r < rows.
template <typename R>
__device__ void mlp_tile_fwd(const R* __restrict__ prm, const MOff& o, int F, const R* X,
                             int64_t row0, const int32_t* idx, int rows, MlpSmem<R>& sm,
                             R* out_rows) {
  const int tid = threadIdx.x;
  const int rg = tid / 16, cg = tid % 16;
  R acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0;
  for (int k0 = 0; k0 < F; k0 += kKc) {
    const int kc = min(kKc, F - k0);
    for (int i = tid; i < kTile * kKc; i += kMT) {
      const int r = i / kKc, k = i % kKc;
      R v = 0;
      if (r < rows && k < kc) {
        const int64_t row = idx ? (int64_t)idx[r] : row0 + r;
        v = X[row * F + k0 + k];
      }
      sm.xs[r][k] = v;
    }
    for (int i = tid; i < kKc * kW; i += kMT) {
      const int k = i / kW, c = i % kW;
      sm.ws[k][c] = k < kc ? prm[o.W1 + (int64_t)(k0 + k) * kW + c] : (R)0;
    }
    __syncthreads();
    for (int k = 0; k < kc; ++k) {
      R a[4], w[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = sm.xs[rg * 4 + i][k];
#pragma unroll
      for (int j = 0; j < 4; ++j) w[j] = sm.ws[k][cg * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] += a[i] * w[j];
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
      sm.h1[rg * 4 + i][cg * 4 + j] = Act<R>::tanh(acc[i][j] + prm[o.b1 + cg * 4 + j]);
  for (int i = tid; i < kW * kW; i += kMT) sm.ws[i / kW][i % kW] = prm[o.W2 + i];
  __syncthreads();
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0;
  for (int k = 0; k < kW; ++k) {
    R a[4], w[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) a[i] = sm.h1[rg * 4 + i][k];
#pragma unroll
    for (int j = 0; j < 4; ++j) w[j] = sm.ws[k][cg * 4 + j];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] += a[i] * w[j];
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
      sm.h2[rg * 4 + i][cg * 4 + j] = Act<R>::tanh(acc[i][j] + prm[o.b2 + cg * 4 + j]);
  __syncthreads();
  if (tid < rows) {
    R s = 0;
    for (int c = 0; c < kW; ++c) s += sm.h2[tid][c] * prm[o.W3 + c];
    out_rows[tid] = s + prm[o.b3];
  }
  __syncthreads();
}

template <typename R>
__global__ void __launch_bounds__(kMT) mlp_predict_kernel(const R* __restrict__ prm,
                                                          const R* __restrict__ X, int64_t n, int F,
                                                          R* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  MlpSmem<R>& sm = *reinterpret_cast<MlpSmem<R>*>(smem_raw);
  const MOff o = mlp_offsets(F);
  const int64_t tiles = (n + kTile - 1) / kTile;
  for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
    const int64_t row0 = t * kTile;
    const int rows = (int)(n - row0 < kTile ? n - row0 : kTile);
    mlp_tile_fwd<R>(prm, o, F, X, row0, nullptr, rows, sm, out + row0);
  }
}

// --------------------------------------------------------------- training --
template <typename R>
struct MlpTrainArgs {
  R* prm;
  R* m;
  R* v;
  const R* X;
  const R* y;
  int F;
  const int32_t* order;
  int64_t n_order;
  int B;
  int loss_kind;
  int mode;
  int n_steps;
  AdamHyper hyp;
  const double* corr;
  R* step_loss;
  R* grad_out;
  int32_t* status;
  // scratch (global)
  R* H1;    // [B][64]
  R* H2;    // [B][64]
  R* D1;    // [B][64]
  R* D2;    // [B][64]
  R* outs;  // [B]
  R* ys;    // [B]
  R* dsc;   // [B]
  R* grad;  // [NP]
};

template <typename R>
__global__ void __launch_bounds__(kMT, 1) mlp_train_kernel(MlpTrainArgs<R> a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  MlpSmem<R>& sm = *reinterpret_cast<MlpSmem<R>*>(smem_raw);
  __shared__ R red[kMT];
  const MOff o = mlp_offsets(a.F);
  const int tid = threadIdx.x;
  const int F = a.F;
  for (int step = 0; step < a.n_steps; ++step) {
    const int64_t b0 = (int64_t)step * a.B;
    const int bn = (int)(a.n_order - b0 < (int64_t)a.B ? a.n_order - b0 : (int64_t)a.B);
    const int32_t* idx = a.order + b0;
    // forward (mlp.py:72-79), activations kept for backward
    for (int r0 = 0; r0 < bn; r0 += kTile) {
      const int rows = min(kTile, bn - r0);
      mlp_tile_fwd<R>(a.prm, o, F, a.X, 0, idx + r0, rows, sm, a.outs + r0);
      for (int i = tid; i < rows * kW; i += kMT) {
        const int r = i / kW, c = i % kW;
        a.H1[(int64_t)(r0 + r) * kW + c] = sm.h1[r][c];
        a.H2[(int64_t)(r0 + r) * kW + c] = sm.h2[r][c];
      }
      __syncthreads();
    }
    for (int k = tid; k < bn; k += kMT) a.ys[k] = a.y[idx[k]];
    __syncthreads();
    const R loss = a.loss_kind == TT_LOSS_RANK ? rank_loss_block<R>(a.ys, a.outs, bn, a.dsc, red)
                                               : mse_block<R>(a.ys, a.outs, bn, a.dsc, red);
    if (!isfinite((double)loss)) {
      if (tid == 0) {
        a.status[0] = step;
        a.step_loss[step] = loss;
      }
      return;
    }
    if (tid == 0) a.step_loss[step] = loss;
    // backward (mlp.py:81-95)
    R* g = a.grad;
    for (int c = tid; c < kW; c += kMT) {
      R s = 0;
      for (int r = 0; r < bn; ++r) s += a.H2[(int64_t)r * kW + c] * a.dsc[r];
      g[o.W3 + c] = s;
    }
    if (tid == 0) {
      R s = 0;
      for (int r = 0; r < bn; ++r) s += a.dsc[r];
      g[o.b3] = s;
    }
    for (int i = tid; i < bn * kW; i += kMT) {
      const int r = i / kW, c = i % kW;
      const R h = a.H2[i];
      a.D2[i] = a.dsc[r] * a.prm[o.W3 + c] * ((R)1 - h * h);
    }
    __syncthreads();
    for (int i = tid; i < kW * kW; i += kMT) {
      const int k = i / kW, c = i % kW;
      R s = 0;
      for (int r = 0; r < bn; ++r) s += a.H1[(int64_t)r * kW + k] * a.D2[(int64_t)r * kW + c];
      g[o.W2 + i] = s;
    }
    for (int c = tid; c < kW; c += kMT) {
      R s = 0;
      for (int r = 0; r < bn; ++r) s += a.D2[(int64_t)r * kW + c];
      g[o.b2 + c] = s;
    }
    for (int i = tid; i < bn * kW; i += kMT) {
      const int r = i / kW, k = i % kW;
      R s = 0;
      for (int c = 0; c < kW; ++c) s += a.D2[(int64_t)r * kW + c] * a.prm[o.W2 + k * kW + c];
      const R h = a.H1[i];
      a.D1[i] = s * ((R)1 - h * h);
    }
    __syncthreads();
    for (int i = tid; i < F * kW; i += kMT) {
      const int f = i / kW, k = i % kW;
      R s = 0;
      for (int r = 0; r < bn; ++r) s += a.X[(int64_t)idx[r] * F + f] * a.D1[(int64_t)r * kW + k];
      g[o.W1 + i] = s;
    }
    for (int k = tid; k < kW; k += kMT) {
      R s = 0;
      for (int r = 0; r < bn; ++r) s += a.D1[(int64_t)r * kW + k];
      g[o.b1 + k] = s;
    }
    __syncthreads();
    if (a.mode == TT_MODE_GRAD) {
      for (int64_t p = tid; p < o.total; p += kMT) a.grad_out[p] = g[p];
    } else {
      const double c1 = a.corr[2 * step], c2 = a.corr[2 * step + 1];
      for (int64_t p = tid; p < o.total; p += kMT) {
        R pp = a.prm[p], mm = a.m[p], vv = a.v[p];
        adam_update<R>(pp, g[p], mm, vv, a.hyp, c1, c2);
        a.prm[p] = pp;
        a.m[p] = mm;
        a.v[p] = vv;
      }
    }
    __syncthreads();
  }
}

// ------------------------------------------- training, shared-memory resident --
// fp32, minibatch <= 16 rows at the reference's widths: the parameters and
// both Adam moments live in shared memory for the whole epoch (3 x 14,785
// floats at F = 164), so a step touches global memory only for its X rows
// (prefetched one step ahead by cp.async) and the loss value.  Per step:
// forward h1, h2, out (thread = (4 rows, 1 column)); loss; D2 and D1 with
// the pre-update W3 / W2; then every gradient entry is formed by a
// fixed-order sum over the rows and immediately applied by the fused Adam
// update (or written out in gradient mode).  Deterministic: no atomics.
__device__ long long g_mlp_prof[16];  // tt_debug_mlp_phase_times
#define MLP_MARK(i) \
  do {                                                   \
    if (step == 64 && threadIdx.x == 0) g_mlp_prof[i] = clock64(); \
  } while (0)
constexpr int kMB = 16;   // rows per minibatch of this kernel
constexpr int kMT2 = 512; // its threads

struct MlpSmemLayout {
  int64_t prm, m, v, x, h1, h2, d1, d2, out, ys, dsc, red, total;  // float offsets
};

inline __host__ __device__ int mlp_fp(int F) { return (F + 3) / 4 * 4; }  // padded X row

inline __host__ __device__ MlpSmemLayout mlp_smem_layout(int F) {
  MlpSmemLayout l{};
  const int64_t np = mlp_offsets(F).total;
  const int64_t npp = (np + 3) / 4 * 4;
  const int64_t xf = (int64_t)kMB * mlp_fp(F);
  l.prm = 0;
  l.m = npp;
  l.v = 2 * npp;
  l.x = 3 * npp;                // two X buffers, rows padded to a multiple of 4 (zeros)
  l.h1 = l.x + 2 * xf;
  l.h2 = l.h1 + kMB * kW;
  l.d1 = l.h2 + kMB * kW;
  l.d2 = l.d1 + kMB * kW;
  l.out = l.d2 + kMB * kW;
  l.ys = l.out + kMB;
  l.dsc = l.ys + kMB;
  l.red = l.dsc + kMB;
  l.total = l.red + kMT2 + 3 * kMB + 2 * kMB;  // + order ring [3][16] (int), y ring [2][16]
  return l;
}

__device__ __forceinline__ void cp_async4_mlp(float* s, const float* g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((uint32_t)__cvta_generic_to_shared(s)),
               "l"(g)
               : "memory");
}

__device__ __forceinline__ float4 ld4(const float* p) { return *reinterpret_cast<const float4*>(p); }

// Pairwise logistic loss of a <= 16-row minibatch (mlp.py:25-35), one pair
// per thread: warp k owns row k, lane j the pair (k, j); the same per-pair
// terms as rank_loss_block, summed in a fixed shuffle / row order.  `red`
// needs 66 floats.  Returns the loss in every thread.
__device__ float mlp_rank_loss(const float* y, const float* s, int n, float* dscore, float* red) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp < n) {
    const float yk = y[warp], sk = s[warp];
    float d = 0.f, part = 0.f, pairs = 0.f;
    if (lane < n) {
      const float yj = y[lane], sj = s[lane];
      if (yj > yk) d = 1.f / (1.f + Act<float>::exp(sj - sk));
      if (yk > yj) {
        const float mg = sk - sj;
        d -= 1.f / (1.f + Act<float>::exp(mg));
        part = Act<float>::softplus(-mg);
        pairs = 1.f;
      }
    }
    d = warp_sum(d);
    part = warp_sum(part);
    pairs = warp_sum(pairs);
    if (lane == 0) {
      dscore[warp] = d;
      red[warp] = part;
      red[32 + warp] = pairs;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    float tp = 0.f, np = 0.f;
    for (int k = 0; k < n; ++k) {
      tp += red[k];
      np += red[32 + k];
    }
    red[64] = tp;
    red[65] = np;
  }
  __syncthreads();
  const float np = red[65];
  if ((int)threadIdx.x < n) dscore[threadIdx.x] = np == 0.f ? 0.f : dscore[threadIdx.x] / np;
  const float loss = np == 0.f ? 0.f : red[64] / np;
  __syncthreads();
  return loss;
}

// optim.py:33-46 in fp32 with one division per parameter: the bias
// corrections are applied as precomputed reciprocals and the denominator's
// square root by the hardware's correctly rounded sqrt (differs from the
// exactly rounded two-division form by an ulp; inside the fp32 tolerance)
__device__ __forceinline__ void adam_fast(float& p, float g, float& m, float& v, float b1, float b2,
                                          float ob1, float ob2, float lr, float eps, float ic1,
                                          float ic2) {
  m = fmaf(m, b1, ob1 * g);
  v = fmaf(v, b2, ob2 * g * g);
  p -= lr * (m * ic1) / (sqrtf(v * ic2) + eps);
}

// 4x4 register tile of a weight gradient dW[a][b] = sum_r A[r][a] Bm[r][b]
// (A rows stride lda, Bm rows stride ldb, both 16-B aligned), rows in order.
__device__ __forceinline__ void grad_tile(const float* A, int lda, const float* Bm, int ldb, int a0,
                                          int b0, int bn, float (&g)[4][4]) {
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) g[i][j] = 0.f;
  for (int r = 0; r < bn; ++r) {
    const float4 x = ld4(A + r * lda + a0), d = ld4(Bm + r * ldb + b0);
    const float xa[4] = {x.x, x.y, x.z, x.w}, da[4] = {d.x, d.y, d.z, d.w};
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) g[i][j] = fmaf(xa[i], da[j], g[i][j]);
  }
}

__global__ void __launch_bounds__(kMT2, 1) mlp_train_smem_kernel(MlpTrainArgs<float> a) {
  extern __shared__ __align__(16) float smf[];
  const int F = a.F, Fp = mlp_fp(F), tid = threadIdx.x, lane = tid & 31;
  const MOff o = mlp_offsets(F);
  const MlpSmemLayout L = mlp_smem_layout(F);
  const int64_t xf = (int64_t)kMB * Fp;
  float* P = smf + L.prm;
  float* M = smf + L.m;
  float* V = smf + L.v;
  float* H1 = smf + L.h1;
  float* H2 = smf + L.h2;
  float* D1 = smf + L.d1;
  float* D2 = smf + L.d2;
  float* out = smf + L.out;
  float* ys = smf + L.ys;
  float* dsc = smf + L.dsc;
  float* red = smf + L.red;
  for (int64_t p = tid; p < o.total; p += kMT2) {
    P[p] = a.prm[p];
    if (a.mode == TT_MODE_TRAIN) {
      M[p] = a.m[p];
      V[p] = a.v[p];
    }
  }
  for (int64_t i = tid; i < 2 * xf; i += kMT2) smf[L.x + i] = 0.f;  // pads stay zero
  // staging pipeline (no global load on a step's critical path): during step
  // s the order indices of step s + 2 and, through the indices already in
  // shared memory, the X rows and labels of step s + 1 are copied by cp.async
  int* ordr = reinterpret_cast<int*>(smf + L.red + kMT2);  // [3][kMB]
  float* yr = smf + L.red + kMT2 + 3 * kMB;                // [2][kMB]
  auto rows_of = [&](int step) {
    const int64_t b0 = (int64_t)step * a.B;
    return (int)(a.n_order - b0 < (int64_t)a.B ? a.n_order - b0 : (int64_t)a.B);
  };
  auto stage_order = [&](int step) {
    if (step >= a.n_steps) return;
    const int bn = rows_of(step);
    for (int i = tid; i < bn; i += kMT2)
      cp_async4_mlp(reinterpret_cast<float*>(ordr + (step % 3) * kMB + i),
                    reinterpret_cast<const float*>(a.order + (int64_t)step * a.B + i));
  };
  auto stage_rows = [&](int step) {
    if (step >= a.n_steps) return;
    const int bn = rows_of(step);
    const int* od = ordr + (step % 3) * kMB;
    float* xs = smf + L.x + (step & 1) * xf;
    for (int i = tid; i < bn * F; i += kMT2) {
      const int r = i / F, k = i - r * F;
      cp_async4_mlp(xs + r * Fp + k, a.X + (int64_t)od[r] * F + k);
    }
    for (int i = tid; i < bn; i += kMT2) cp_async4_mlp(yr + (step & 1) * kMB + i, a.y + od[i]);
  };
  stage_order(0);
  stage_order(1);
  asm volatile("cp.async.commit_group;" ::: "memory");
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();
  stage_rows(0);
  asm volatile("cp.async.commit_group;" ::: "memory");
  const int c = tid & 63, rq = tid >> 6;  // forward: output column, rows 2 rq, 2 rq + 1
  for (int step = 0; step < a.n_steps; ++step) {
    const int64_t b0 = (int64_t)step * a.B;
    const int bn = (int)(a.n_order - b0 < (int64_t)a.B ? a.n_order - b0 : (int64_t)a.B);
    const float* X = smf + L.x + (step & 1) * xf;
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
    MLP_MARK(0);
    for (int k = tid; k < bn; k += kMT2) ys[k] = yr[(step & 1) * kMB + k];
    stage_order(step + 2);  // overlaps this step
    stage_rows(step + 1);
    asm volatile("cp.async.commit_group;" ::: "memory");
    // ---- forward (mlp.py:72-79): rows 4 rq .. 4 rq + 3, column c; the X / H1
    //      rows are read as float4 broadcasts, the weight column per k
    {
      float acc[2] = {0.f, 0.f};
      for (int k = 0; k < Fp; k += 4) {
        float w[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) w[j] = k + j < F ? P[o.W1 + (k + j) * kW + c] : 0.f;
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const float4 x = ld4(X + (2 * rq + i) * Fp + k);
          acc[i] = fmaf(x.x, w[0], acc[i]);
          acc[i] = fmaf(x.y, w[1], acc[i]);
          acc[i] = fmaf(x.z, w[2], acc[i]);
          acc[i] = fmaf(x.w, w[3], acc[i]);
        }
      }
#pragma unroll
      for (int i = 0; i < 2; ++i) H1[(2 * rq + i) * kW + c] = Act<float>::tanh(acc[i] + P[o.b1 + c]);
    }
    __syncthreads();
    {
      float acc[2] = {0.f, 0.f};
      for (int k = 0; k < kW; k += 4) {
        float w[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) w[j] = P[o.W2 + (k + j) * kW + c];
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const float4 x = ld4(H1 + (2 * rq + i) * kW + k);
          acc[i] = fmaf(x.x, w[0], acc[i]);
          acc[i] = fmaf(x.y, w[1], acc[i]);
          acc[i] = fmaf(x.z, w[2], acc[i]);
          acc[i] = fmaf(x.w, w[3], acc[i]);
        }
      }
#pragma unroll
      for (int i = 0; i < 2; ++i) H2[(2 * rq + i) * kW + c] = Act<float>::tanh(acc[i] + P[o.b2 + c]);
    }
    __syncthreads();
    MLP_MARK(1);
    // out[r] = H2[r] . W3 + b3: warp w < bn / 2 handles rows 2w, 2w + 1 (lane halves)
    if (tid < 8 * 32) {
      const int r = (tid >> 5) * 2 + (lane >> 4), q = lane & 15;
      float s = 0.f;
      if (r < bn) {
        const float4 h = ld4(H2 + r * kW + 4 * q), w = ld4(P + o.W3 + 4 * q);
        s = fmaf(h.x, w.x, fmaf(h.y, w.y, fmaf(h.z, w.z, h.w * w.w)));
      }
#pragma unroll
      for (int off = 8; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
      if (q == 0 && r < bn) out[r] = s + P[o.b3];
    }
    __syncthreads();
    MLP_MARK(2);
    const float loss = a.loss_kind == TT_LOSS_RANK ? mlp_rank_loss(ys, out, bn, dsc, red)
                                                   : mse_block<float>(ys, out, bn, dsc, red);
    MLP_MARK(3);
    if (tid == 0) a.step_loss[step] = loss;
    if (!isfinite(loss)) {
      if (tid == 0) a.status[0] = step;
      return;
    }
    // ---- backward (mlp.py:81-95) with the pre-update W3, W2
    for (int i = tid; i < kMB * kW; i += kMT2) {
      const int r = i / kW, k = i % kW;
      const float h = H2[i];
      D2[i] = r < bn ? dsc[r] * P[o.W3 + k] * (1.f - h * h) : 0.f;  // rows >= bn: zero
    }
    __syncthreads();
    for (int i = tid; i < kMB * kW; i += kMT2) {
      const int r = i / kW, k = i % kW;
      // lane-rotated column order: W2 row k is read without bank conflicts;
      // two independent halves, added in a fixed order
      float s0 = 0.f, s1 = 0.f;
      const float* d2r = D2 + r * kW;
      const float* w2r = P + o.W2 + k * kW;
      for (int t = 0; t < kW / 2; ++t) {
        const int c0 = (t + lane) & (kW - 1), c1 = (t + kW / 2 + lane) & (kW - 1);
        s0 = fmaf(d2r[c0], w2r[c0], s0);
        s1 = fmaf(d2r[c1], w2r[c1], s1);
      }
      const float s = s0 + s1;
      const float h = H1[i];
      D1[i] = r < bn ? s * (1.f - h * h) : 0.f;
    }
    __syncthreads();
    MLP_MARK(4);
    // ---- gradients (4x4 register tiles, rows in order) + fused Adam
    const double c1 = a.mode == TT_MODE_TRAIN ? a.corr[2 * step] : 1.0;
    const double c2 = a.mode == TT_MODE_TRAIN ? a.corr[2 * step + 1] : 1.0;
    const float hb1 = (float)a.hyp.b1, hb2 = (float)a.hyp.b2, ob1 = (float)(1.0 - a.hyp.b1),
                ob2 = (float)(1.0 - a.hyp.b2), hlr = (float)a.hyp.lr, heps = (float)a.hyp.eps;
    const float ic1 = (float)(1.0 / c1), ic2 = (float)(1.0 / c2);
    auto apply = [&](int64_t p, float g) {
      if (a.mode == TT_MODE_GRAD) {
        a.grad_out[p] = g;
      } else {
        float pp = P[p], mm = M[p], vv = V[p];
        adam_fast(pp, g, mm, vv, hb1, hb2, ob1, ob2, hlr, heps, ic1, ic2);
        P[p] = pp;
        M[p] = mm;
        V[p] = vv;
      }
    };
    const int t1 = (Fp / 4) * (kW / 4), t2 = (kW / 4) * (kW / 4);
    for (int t = tid; t < t1 + t2; t += kMT2) {
      float g[4][4];
      if (t < t1) {  // W1[f][k] = sum_r X[r][f] D1[r][k]
        const int f0 = (t / (kW / 4)) * 4, k0 = (t % (kW / 4)) * 4;
        grad_tile(X, Fp, D1, kW, f0, k0, bn, g);
#pragma unroll
        for (int i = 0; i < 4; ++i)
          if (f0 + i < F)
#pragma unroll
            for (int j = 0; j < 4; ++j) apply(o.W1 + (int64_t)(f0 + i) * kW + k0 + j, g[i][j]);
      } else {  // W2[k][cc] = sum_r H1[r][k] D2[r][cc]
        const int u = t - t1, k0 = (u / (kW / 4)) * 4, c0 = (u % (kW / 4)) * 4;
        grad_tile(H1, kW, D2, kW, k0, c0, bn, g);
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) apply(o.W2 + (int64_t)(k0 + i) * kW + c0 + j, g[i][j]);
      }
    }
    MLP_MARK(5);
    // biases and W3 (rows in order)
    for (int i = tid; i < 3 * kW + 1; i += kMT2) {
      float g = 0.f;
      int64_t p;
      if (i < kW) {
        for (int r = 0; r < bn; ++r) g += D1[r * kW + i];
        p = o.b1 + i;
      } else if (i < 2 * kW) {
        for (int r = 0; r < bn; ++r) g += D2[r * kW + i - kW];
        p = o.b2 + i - kW;
      } else if (i < 3 * kW) {
        for (int r = 0; r < bn; ++r) g += H2[r * kW + i - 2 * kW] * dsc[r];
        p = o.W3 + i - 2 * kW;
      } else {
        for (int r = 0; r < bn; ++r) g += dsc[r];
        p = o.b3;
      }
      apply(p, g);
    }
    __syncthreads();
    MLP_MARK(6);
  }
  if (a.mode == TT_MODE_TRAIN)
    for (int64_t p = tid; p < o.total; p += kMT2) {
      a.prm[p] = P[p];
      a.m[p] = M[p];
      a.v[p] = V[p];
    }
}

inline size_t mlp_smem_bytes(int F) { return (size_t)mlp_smem_layout(F).total * sizeof(float); }

template <typename R>
static int mlp_predict(const R* prm, const R* X, int64_t n, int F, R* out, tt_stream_t st) {
  TT_REQUIRE(n >= 0 && F >= 1, "mlp predict: bad shape");
  if (n == 0) return TT_OK;
  const size_t smem = sizeof(MlpSmem<R>);
  auto kern = mlp_predict_kernel<R>;
  if (int rc = kernel_smem((const void*)kern, smem)) return rc;
  const int64_t tiles = (n + kTile - 1) / kTile;
  const int grid = (int)std::min<int64_t>(tiles, (int64_t)sm_count() * 2);
  kern<<<grid, kMT, smem, as_stream(st)>>>(prm, X, n, F, out);
  return check_launch("mlp predict");
}

template <typename R>
static size_t mlp_ws(int F, int B) {
  const MOff o = mlp_offsets(F);
  return align_up((size_t)(4 * kW + 3) * B * sizeof(R), 256) + align_up(o.total * sizeof(R), 256);
}

template <typename R>
static int mlp_train(R* prm, R* m, R* v, const R* X, const R* y, int F, const int32_t* order,
                     int64_t n_order, int B, int loss_kind, int mode, double lr, double b1,
                     double b2, double eps, const double* corr, R* step_loss, R* grad_out,
                     int32_t* status, void* ws, size_t ws_bytes, tt_stream_t st) {
  TT_REQUIRE(F >= 1 && B >= 1 && B <= 4096 && n_order >= 1, "mlp train: bad arguments");
  TT_REQUIRE(mode == TT_MODE_TRAIN || mode == TT_MODE_GRAD, "mlp train: bad mode");
  TT_REQUIRE(mode == TT_MODE_GRAD || corr != nullptr, "mlp train: corr required");
  if (mode == TT_MODE_GRAD) TT_REQUIRE(n_order <= B, "mlp grad: one minibatch only");
  TT_REQUIRE(ws_bytes >= mlp_ws<R>(F, B), "mlp train: workspace too small");
  MlpTrainArgs<R> a{};
  a.prm = prm;
  a.m = m;
  a.v = v;
  a.X = X;
  a.y = y;
  a.F = F;
  a.order = order;
  a.n_order = n_order;
  a.B = B;
  a.loss_kind = loss_kind;
  a.mode = mode;
  a.n_steps = (int)((n_order + B - 1) / B);
  a.hyp = AdamHyper{lr, b1, b2, eps};
  a.corr = corr;
  a.step_loss = step_loss;
  a.grad_out = grad_out;
  a.status = status;
  R* w = static_cast<R*>(ws);
  a.H1 = w;
  a.H2 = w + (size_t)kW * B;
  a.D1 = w + (size_t)2 * kW * B;
  a.D2 = w + (size_t)3 * kW * B;
  a.outs = w + (size_t)4 * kW * B;
  a.ys = a.outs + B;
  a.dsc = a.ys + B;
  a.grad = reinterpret_cast<R*>(static_cast<char*>(ws) +
                                align_up((size_t)(4 * kW + 3) * B * sizeof(R), 256));
  if constexpr (std::is_same<R, float>::value) {
    // shared-memory resident kernel when the minibatch and the parameters fit
    const size_t sm2 = mlp_smem_bytes(F);
    int dev = 0, optin = 0;
    TT_CUDA(cudaGetDevice(&dev));
    TT_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    if (B <= kMB && sm2 + 1024 <= (size_t)optin) {
      if (int rc = kernel_smem((const void*)mlp_train_smem_kernel, sm2)) return rc;
      mlp_train_smem_kernel<<<1, kMT2, sm2, as_stream(st)>>>(a);
      return check_launch("mlp train (smem)");
    }
  }
  const size_t smem = sizeof(MlpSmem<R>);
  auto kern = mlp_train_kernel<R>;
  if (int rc = kernel_smem((const void*)kern, smem)) return rc;
  kern<<<1, kMT, smem, as_stream(st)>>>(a);
  return check_launch("mlp train");
}

}  // namespace tt

using namespace tt;

extern "C" {

int64_t tt_mlp_param_count(int32_t F) { return F >= 1 ? mlp_offsets(F).total : -1; }

int tt_mlp_predict_f32(const float* prm, const float* X, int64_t n, int32_t F, float* out,
                       tt_stream_t st) {
  return mlp_predict<float>(prm, X, n, F, out, st);
}

int tt_mlp_predict_f64(const double* prm, const double* X, int64_t n, int32_t F, double* out,
                       tt_stream_t st) {
  return mlp_predict<double>(prm, X, n, F, out, st);
}

int tt_debug_mlp_phase_times(int64_t* h_out, int32_t n) {
  TT_REQUIRE(h_out != nullptr && n >= 0 && n <= 16, "debug: bad arguments");
  TT_CUDA(cudaMemcpyFromSymbol(h_out, g_mlp_prof, (size_t)n * sizeof(long long)));
  return TT_OK;
}

size_t tt_mlp_train_workspace_bytes(int32_t f64, int32_t F, int32_t B) {
  return f64 ? mlp_ws<double>(F, B) : mlp_ws<float>(F, B);
}

int tt_mlp_train_f32(float* prm, float* m, float* v, const float* X, const float* y, int32_t F,
                     const int32_t* order, int64_t n_order, int32_t B, int32_t loss_kind,
                     int32_t mode, double lr, double b1, double b2, double eps, const double* corr,
                     float* step_loss, float* grad_out, int32_t* status, void* ws, size_t ws_bytes,
                     tt_stream_t st) {
  return mlp_train<float>(prm, m, v, X, y, F, order, n_order, B, loss_kind, mode, lr, b1, b2, eps,
                          corr, step_loss, grad_out, status, ws, ws_bytes, st);
}

int tt_mlp_train_f64(double* prm, double* m, double* v, const double* X, const double* y,
                     int32_t F, const int32_t* order, int64_t n_order, int32_t B, int32_t loss_kind,
                     int32_t mode, double lr, double b1, double b2, double eps,
                     const double* corr, double* step_loss, double* grad_out, int32_t* status,
                     void* ws, size_t ws_bytes, tt_stream_t st) {
  return mlp_train<double>(prm, m, v, X, y, F, order, n_order, B, loss_kind, mode, lr, b1, b2, eps,
                           corr, step_loss, grad_out, status, ws, ws_bytes, st);
}

}  // extern "C"
