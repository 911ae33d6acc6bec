// Attention tuner: shared layout + forward building blocks.
//
// Reference: estimators/tuner.py
//   _LstmDirection.forward  :61-100   gates [i|f|g|o], masked steps hold state
//   stack                   :233-246  bw direction = forward over the reversed
//                                     padded sequence == reverse-within-segment
//                                     from zero state (padding is inert)
//   attention               :248-274  masked mean p0, K/V (no bias), U passes
//   head                    :276-279
//
// Execution model: a 256-thread CTA owns a tile of P programs.  Threads
// 0..127 run the forward direction, 128..255 the backward direction of the
// same layer concurrently (named barriers 1 and 2).  In the gate phase thread
// `c` owns gate column c: its Wh column (H values) and, for layers >= 1, its
// Wx column (2H values) live in registers for the whole layer, so the
// recurrent matvec streams only h (shared memory, broadcast) and the layer
// input row (L1, broadcast).  In the cell phase thread j owns hidden unit j of
// a subset of programs, keeping the cell state in registers.
#pragma once

#include "tt_ops.cuh"

namespace tt {

constexpr int kMaxLayers = 8;
constexpr int kHeadHidden = 64;  // tuner.py:24
constexpr int kThreads = 256;

struct TDims {
  int L, H, heads, U, d0, C, D, G, dh, Tmax;
  int64_t wx[kMaxLayers][2], wh[kMaxLayers][2], bb[kMaxLayers][2];
  int64_t Wq, Wk, Wv, Wo, bq, bo, W1, b1, W2, b2, total;
};

// Parameter offsets in the reference's dict order (tuner.py:194-210).
inline TDims make_dims(int L, int H, int heads, int U, int d0, int C, int Tmax) {
  TDims d{};
  d.L = L;
  d.H = H;
  d.heads = heads;
  d.U = U;
  d.d0 = d0;
  d.C = C;
  d.D = 2 * H;
  d.G = 4 * H;
  d.dh = heads > 0 ? d.D / heads : 0;
  d.Tmax = Tmax;
  int64_t o = 0;
  for (int l = 0; l < L && l < kMaxLayers; ++l) {
    const int din = l == 0 ? d0 : d.D;
    for (int s = 0; s < 2; ++s) {
      d.wx[l][s] = o;
      o += (int64_t)din * d.G;
      d.wh[l][s] = o;
      o += (int64_t)H * d.G;
      d.bb[l][s] = o;
      o += d.G;
    }
  }
  const int64_t DD = (int64_t)d.D * d.D;
  d.Wq = o;
  o += DD;
  d.Wk = o;
  o += DD;
  d.Wv = o;
  o += DD;
  d.Wo = o;
  o += DD;
  d.bq = o;
  o += d.D;
  d.bo = o;
  o += d.D;
  d.W1 = o;
  o += (int64_t)(d.D + C) * kHeadHidden;
  d.b1 = o;
  o += kHeadHidden;
  d.W2 = o;
  o += kHeadHidden;
  d.b2 = o;
  o += 1;
  d.total = o;
  return d;
}

// Weight loads: TRAIN kernels re-read parameters that other CTAs update
// (Adam) between grid barriers, so they use coherent ld.global (the barrier's
// ld.acquire.gpu invalidates L1); scoring kernels use the read-only path.
template <bool TRAIN, typename R>
__device__ __forceinline__ R ldw(const R* p) {
  if constexpr (TRAIN)
    return *p;
  else
    return __ldg(p);
}

// dot(x[0:N], w[0:N]) with 4 independent partial sums; x is an aligned row in
// global or shared memory (vectorised), w a register array.
template <int N>
__device__ __forceinline__ float dot_reg(const float* __restrict__ x, const float (&w)[N]) {
  float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
  if constexpr (N % 4 == 0) {
    const float4* x4 = reinterpret_cast<const float4*>(x);
#pragma unroll
    for (int k = 0; k < N / 4; ++k) {
      const float4 v = x4[k];
      a0 = fmaf(v.x, w[4 * k + 0], a0);
      a1 = fmaf(v.y, w[4 * k + 1], a1);
      a2 = fmaf(v.z, w[4 * k + 2], a2);
      a3 = fmaf(v.w, w[4 * k + 3], a3);
    }
  } else {
#pragma unroll
    for (int k = 0; k < N; ++k) a0 = fmaf(x[k], w[k], a0);
  }
  return (a0 + a1) + (a2 + a3);
}

template <int N>
__device__ __forceinline__ double dot_reg(const double* __restrict__ x, const double (&w)[N]) {
  double a0 = 0.0, a1 = 0.0;
  if constexpr (N % 2 == 0) {
    const double2* x2 = reinterpret_cast<const double2*>(x);
#pragma unroll
    for (int k = 0; k < N / 2; ++k) {
      const double2 v = x2[k];
      a0 = fma(v.x, w[2 * k + 0], a0);
      a1 = fma(v.y, w[2 * k + 1], a1);
    }
  } else {
#pragma unroll
    for (int k = 0; k < N; ++k) a0 = fma(x[k], w[k], a0);
  }
  return a0 + a1;
}

// Per-program pointers of a tile (shared memory).
template <typename R, int P>
struct TileInfo {
  int len[P];            // steps per program (0 = empty slot)
  const R* step0[P];     // first raw step row of the program
  const R* ctx[P];       // context row
  int64_t prog[P];       // program index (-1 = empty)
};

// ----------------------------------------------------------- LSTM layer --
// One bidirectional layer for P programs.  `in0[p]` + t*in_stride is the input
// row of program p at time t (raw steps for layer 0, previous layer output
// otherwise).  Output rows: out[(p*Tmax + t)*D + dir*H + j].
// TRAIN (P == 1): also records gates / cell state / tanh(cell) per step.
template <typename R, int H, int P, bool TRAIN>
__device__ void lstm_layer_fwd(const TDims& dm, const R* __restrict__ prm, int l,
                               const TileInfo<R, P>& ti, const R* const* in0, int in_stride,
                               R* __restrict__ out, R* sh_h, R* sh_g, R* cache_g, R* cache_c,
                               R* cache_tc) {
  constexpr int G = 4 * H, D = 2 * H, NR = 128 / G, NQ = 128 / H;
  const int dir = threadIdx.x >> 7, lt = threadIdx.x & 127;
  const int c = lt % G, r = lt / G;
  const int j = lt % H, q = lt / H;
  const int Tmax = dm.Tmax;
  const R* Wx = prm + dm.wx[l][dir];
  const R* Wh = prm + dm.wh[l][dir];
  R wh[H];
#pragma unroll
  for (int k = 0; k < H; ++k) wh[k] = ldw<TRAIN>(Wh + k * G + c);
  R wx[D];
  if (l > 0) {
#pragma unroll
    for (int k = 0; k < D; ++k) wx[k] = ldw<TRAIN>(Wx + k * G + c);
  }
  const R bc = ldw<TRAIN>(prm + dm.bb[l][dir] + c);
  const int d_in = l == 0 ? dm.d0 : D;
  constexpr int NC = (P + NQ - 1) / NQ;
  R creg[NC];
#pragma unroll
  for (int i = 0; i < NC; ++i) creg[i] = 0;
  R* hbase = sh_h + dir * P * H;
  R* gbase = sh_g + dir * P * G;
  for (int i = lt; i < P * H; i += 128) hbase[i] = 0;
  int Tt = 0;
#pragma unroll
  for (int p = 0; p < P; ++p) Tt = max(Tt, ti.len[p]);
  named_barrier(1 + dir, 128);
  for (int s = 0; s < Tt; ++s) {
    // gate phase: z = b + x_t Wx + h Wh ; activation by gate block
#pragma unroll
    for (int p = r; p < P; p += NR) {
      const int n = ti.len[p];
      if (s < n) {
        const int t = dir == 0 ? s : n - 1 - s;
        const R* x = in0[p] + (int64_t)t * in_stride;
        R z;
        if (l > 0) {
          z = dot_reg<D>(x, wx);
        } else {
          z = 0;
          for (int k = 0; k < d_in; ++k) z += x[k] * ldw<TRAIN>(Wx + k * G + c);
        }
        z += dot_reg<H>(hbase + p * H, wh) + bc;
        const int gate = c / H;
        const R a = gate == 2 ? Act<R>::tanh(z) : Act<R>::sigmoid(z);
        gbase[p * G + c] = a;
        if constexpr (TRAIN) cache_g[(dir * Tmax + t) * G + c] = a;
      }
    }
    named_barrier(1 + dir, 128);
    // cell phase: c = f c + i g ; h = o tanh(c)
#pragma unroll
    for (int ci = 0; ci < NC; ++ci) {
      const int p = q + ci * NQ;
      if (p < P) {
        const int n = ti.len[p];
        if (s < n) {
          const int t = dir == 0 ? s : n - 1 - s;
          const R* gp = gbase + p * G;
          const R gi = gp[j], gf = gp[H + j], gg = gp[2 * H + j], go = gp[3 * H + j];
          const R cn = gf * creg[ci] + gi * gg;
          const R tc = Act<R>::tanh(cn);
          const R hn = go * tc;
          creg[ci] = cn;
          hbase[p * H + j] = hn;
          out[((int64_t)p * Tmax + t) * D + dir * H + j] = hn;
          if constexpr (TRAIN) {
            cache_c[(dir * Tmax + t) * H + j] = cn;
            cache_tc[(dir * Tmax + t) * H + j] = tc;
          }
        }
      }
    }
    named_barrier(1 + dir, 128);
  }
}

// --------------------------------------------------- attention + head --
// Shared-memory scratch for a tile of P programs.
template <typename R, int P>
struct AttnSmem {
  R* pool;   // [P][D]
  R* q;      // [P][D]
  R* mix;    // [P][D]
  R* alpha;  // [P][heads][Tmax]
  R* z;      // [P][D + C]
  R* a1;     // [P][64]
};

// Training cache of one sample (P == 1).
template <typename R>
struct AttnCache {
  R* pin;    // [U][D]   pooled entering each pass
  R* q;      // [U][D]
  R* alpha;  // [U][heads][Tmax]
  R* mix;    // [U][D]
  R* z;      // [D + C]
  R* a1;     // [64]
  R* yhat;   // [1]
};

// S, K, V: [P][Tmax][D] (global scratch).  Writes yhat[p] to out_yhat[p] for
// occupied slots.  All 256 threads participate.
template <typename R, int H, int P, bool TRAIN>
__device__ void attention_head_fwd(const TDims& dm, const R* __restrict__ prm,
                                   const TileInfo<R, P>& ti, const R* __restrict__ S,
                                   R* __restrict__ Kb, R* __restrict__ Vb, const AttnSmem<R, P>& sm,
                                   const AttnCache<R>* cache, R* out_yhat) {
  constexpr int D = 2 * H;
  const int tid = threadIdx.x;
  const int Tmax = dm.Tmax, heads = dm.heads, dh = dm.dh, C = dm.C;
  const int warp = tid >> 5, lane = tid & 31;
  // p0 = masked mean (tuner.py:252-253)
  for (int i = tid; i < P * D; i += kThreads) {
    const int p = i / D, d = i % D;
    const int n = ti.len[p];
    R acc = 0;
    for (int t = 0; t < n; ++t) acc += S[((int64_t)p * Tmax + t) * D + d];
    sm.pool[i] = acc / (R)(n > 1 ? n : 1);
  }
  // K = S Wk, V = S Wv (no bias): thread column cc in [0, 2D)
  {
    constexpr int NCOL = 2 * D;
    constexpr int NGRP = kThreads / NCOL >= 1 ? kThreads / NCOL : 1;
    const int cc = tid % NCOL, grp = tid / NCOL;
    if (grp < NGRP) {
      const R* W = prm + (cc < D ? dm.Wk : dm.Wv);
      const int col = cc % D;
      R w[D];
#pragma unroll
      for (int k = 0; k < D; ++k) w[k] = ldw<TRAIN>(W + k * D + col);
      R* dst = cc < D ? Kb : Vb;
      for (int p = grp; p < P; p += NGRP) {
        const int n = ti.len[p];
        for (int t = 0; t < n; ++t) {
          const int64_t row = ((int64_t)p * Tmax + t) * D;
          dst[row + col] = dot_reg<D>(S + row, w);
        }
      }
    }
  }
  __syncthreads();
  const R inv_scale = (R)1 / sqrt((R)dh);
  (void)inv_scale;
  const R sq = sqrt((R)dh);
  for (int u = 0; u < dm.U; ++u) {
    // q = pooled Wq + bq
    for (int i = tid; i < P * D; i += kThreads) {
      const int p = i / D, c = i % D;
      const R* W = prm + dm.Wq + c;
      R acc = 0;
      for (int k = 0; k < D; ++k) acc += sm.pool[p * D + k] * ldw<TRAIN>(W + k * D);
      sm.q[i] = acc + ldw<TRAIN>(prm + dm.bq + c);
    }
    __syncthreads();
    if constexpr (TRAIN) {
      for (int i = tid; i < D; i += kThreads) {
        cache->pin[u * D + i] = sm.pool[i];
        cache->q[u * D + i] = sm.q[i];
      }
    }
    // per (program, head): logits over steps, softmax (warp-wide)
    for (int ph = warp; ph < P * heads; ph += kThreads / 32) {
      const int p = ph / heads, h = ph % heads;
      const int n = ti.len[p];
      const R* qh = sm.q + p * D + h * dh;
      R* al = sm.alpha + ((int64_t)p * heads + h) * Tmax;
      R mx = -INFINITY;
      for (int t = lane; t < n; t += 32) {
        const R* kr = Kb + ((int64_t)p * Tmax + t) * D + h * dh;
        R acc = 0;
        for (int d = 0; d < dh; ++d) acc += qh[d] * kr[d];
        acc = acc / sq;  // tuner.py:264 divides by sqrt(dh)
        al[t] = acc;
        mx = acc > mx ? acc : mx;
      }
      mx = warp_max(mx);
      R sum = 0;
      for (int t = lane; t < n; t += 32) {
        const R e = Act<R>::exp(al[t] - mx);
        al[t] = e;
        sum += e;
      }
      sum = warp_sum(sum);
      for (int t = lane; t < n; t += 32) al[t] = al[t] / sum;
    }
    __syncthreads();
    // mix = alpha V (per head block of columns)
    for (int i = tid; i < P * D; i += kThreads) {
      const int p = i / D, c = i % D, h = c / dh;
      const int n = ti.len[p];
      const R* al = sm.alpha + ((int64_t)p * heads + h) * Tmax;
      R acc = 0;
      for (int t = 0; t < n; ++t) acc += al[t] * Vb[((int64_t)p * Tmax + t) * D + c];
      sm.mix[i] = acc;
    }
    __syncthreads();
    if constexpr (TRAIN) {
      for (int i = tid; i < D; i += kThreads) cache->mix[u * D + i] = sm.mix[i];
      for (int i = tid; i < heads * Tmax; i += kThreads) cache->alpha[u * heads * Tmax + i] = sm.alpha[i];
    }
    // pooled = mix Wo + bo
    for (int i = tid; i < P * D; i += kThreads) {
      const int p = i / D, c = i % D;
      const R* W = prm + dm.Wo + c;
      R acc = 0;
      for (int k = 0; k < D; ++k) acc += sm.mix[p * D + k] * ldw<TRAIN>(W + k * D);
      sm.pool[i] = acc + ldw<TRAIN>(prm + dm.bo + c);
    }
    __syncthreads();
  }
  // head: z = [pooled | ctx] ; a1 = tanh(z W1 + b1) ; yhat = sigmoid(a1 W2 + b2)
  const int Z = D + C;
  for (int i = tid; i < P * Z; i += kThreads) {
    const int p = i / Z, k = i % Z;
    R v = 0;
    if (k < D)
      v = sm.pool[p * D + k];
    else if (ti.len[p] > 0)
      v = __ldg(ti.ctx[p] + (k - D));
    sm.z[i] = v;
  }
  __syncthreads();
  for (int i = tid; i < P * kHeadHidden; i += kThreads) {
    const int p = i / kHeadHidden, c = i % kHeadHidden;
    const R* W = prm + dm.W1 + c;
    const R* zp = sm.z + p * Z;
    R acc = 0;
    for (int k = 0; k < Z; ++k) acc += zp[k] * ldw<TRAIN>(W + k * kHeadHidden);
    sm.a1[i] = Act<R>::tanh(acc + ldw<TRAIN>(prm + dm.b1 + c));
  }
  __syncthreads();
  for (int p = warp; p < P; p += kThreads / 32) {
    R acc = 0;
    for (int c = lane; c < kHeadHidden; c += 32)
      acc += sm.a1[p * kHeadHidden + c] * ldw<TRAIN>(prm + dm.W2 + c);
    acc = warp_sum(acc);
    if (lane == 0 && ti.len[p] > 0) {
      const R yh = Act<R>::sigmoid(acc + ldw<TRAIN>(prm + dm.b2));
      out_yhat[p] = yh;
      if constexpr (TRAIN) cache->yhat[0] = yh;
    }
  }
  if constexpr (TRAIN) {
    for (int i = tid; i < Z; i += kThreads) cache->z[i] = sm.z[i];
    for (int i = tid; i < kHeadHidden; i += kThreads) cache->a1[i] = sm.a1[i];
  }
  __syncthreads();
}

}  // namespace tt
