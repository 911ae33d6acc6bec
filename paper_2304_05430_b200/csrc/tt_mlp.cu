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

template <typename R>
static int mlp_predict(const R* prm, const R* X, int64_t n, int F, R* out, tt_stream_t st) {
  TT_REQUIRE(n >= 0 && F >= 1, "mlp predict: bad shape");
  if (n == 0) return TT_OK;
  const size_t smem = sizeof(MlpSmem<R>);
  auto kern = mlp_predict_kernel<R>;
  TT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
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
  const size_t smem = sizeof(MlpSmem<R>);
  auto kern = mlp_train_kernel<R>;
  TT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
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
