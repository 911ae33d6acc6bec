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
//
// Attention/head weights (4 x 2Hx2H, 2H+C x 64, biases) are staged once into
// shared memory with a +1 padded row stride, so both column-owner (forward)
// and row-owner (backward, transposed) matvecs are bank-conflict free.
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

// Weight loads from global memory.  TRAIN kernels re-read parameters that
// other CTAs update (Adam) between grid barriers and keep their per-sample
// activation caches in L1, so weights are read L2-only (ld.global.cg: always
// coherent, never evicts the caches); scoring kernels use the read-only path.
template <bool TRAIN, typename R>
__device__ __forceinline__ R ldw(const R* p) {
  if constexpr (TRAIN)
    return __ldcg(p);
  else
    return __ldg(p);
}

// dot(x[0:N], w[0:N]) with independent partial sums; x is a 16-B aligned row
// in global or shared memory (vectorised), w a register array.
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

// ----------------------------------------------------- staged weights --
template <typename R>
struct AttnW {
  const R *Wq, *Wk, *Wv, *Wo;  // [D][ldd]
  const R *bq, *bo;            // [D]
  const R* W1;                 // [D+C][ld1]
  const R *b1, *W2;            // [64]
  R b2;
  int ldd, ld1;
};

__host__ __device__ inline int64_t attn_stage_elems(const TDims& d) {
  // [Wq|Wk|Wv|Wo|bq|bo] (4D+2 rows x D, ld D+1) then [W1|b1|W2] (D+C+2 rows x 64, ld 65)
  const int64_t n = (int64_t)(4 * d.D + 2) * (d.D + 1) + (int64_t)(d.D + d.C + 2) * (kHeadHidden + 1);
  return (n + 3) & ~int64_t(3);
}

template <typename R>
struct VecOf;
template <>
struct VecOf<float> {
  using T = float4;
  static constexpr int N = 4;
};
template <>
struct VecOf<double> {
  using T = double2;
  static constexpr int N = 2;
};

template <typename R>
__device__ __forceinline__ void store_vec(R* d, const float4& v) {
  d[0] = v.x;
  d[1] = v.y;
  d[2] = v.z;
  d[3] = v.w;
}
template <typename R>
__device__ __forceinline__ void store_vec(R* d, const double2& v) {
  d[0] = v.x;
  d[1] = v.y;
}

// Copy `rows` contiguous rows of COLS elements (16-B aligned source) into
// shared memory with row stride `ld` (padding breaks bank conflicts of the
// transposed accesses).  16-B vector loads, U in flight per thread, L2-only
// (the parameters change every step; L1 keeps the activation caches); the
// row/column split is a compile-time shift.
template <typename R, int COLS>
__device__ __forceinline__ void stage_rows(R* __restrict__ dst, int ld, const R* __restrict__ src,
                                           int rows) {
  using V = typename VecOf<R>::T;
  constexpr int VN = VecOf<R>::N;
  constexpr int VPR = COLS / VN;
  static_assert(COLS % VN == 0, "row width must be a multiple of the vector width");
  const int total = rows * VPR;
  const V* s = reinterpret_cast<const V*>(src);
  constexpr int U = 8;
  for (int i0 = threadIdx.x; i0 < total; i0 += U * kThreads) {
    V v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = i0 + u * kThreads;
      if (i < total) v[u] = __ldcg(s + i);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = i0 + u * kThreads;
      if (i < total) store_vec<R>(dst + (i / VPR) * ld + (i % VPR) * VN, v[u]);
    }
  }
}

// All threads; ends with __syncthreads.  The parameter layout keeps
// Wq,Wk,Wv,Wo,bq,bo and W1,b1,W2 contiguous, so two block copies suffice.
template <typename R, int D>
__device__ AttnW<R> stage_attn(const TDims& dm, const R* prm, R* dst) {
  AttnW<R> w;
  w.ldd = D + 1;
  w.ld1 = kHeadHidden + 1;
  R* d2 = dst + (int64_t)(4 * D + 2) * w.ldd;
  stage_rows<R, D>(dst, w.ldd, prm + dm.Wq, 4 * D + 2);
  stage_rows<R, kHeadHidden>(d2, w.ld1, prm + dm.W1, D + dm.C + 2);
  w.Wq = dst;
  w.Wk = dst + D * w.ldd;
  w.Wv = dst + 2 * D * w.ldd;
  w.Wo = dst + 3 * D * w.ldd;
  w.bq = dst + 4 * D * w.ldd;
  w.bo = dst + (4 * D + 1) * w.ldd;
  w.W1 = d2;
  w.b1 = d2 + (int64_t)(D + dm.C) * w.ld1;
  w.W2 = d2 + (int64_t)(D + dm.C + 1) * w.ld1;
  w.b2 = __ldcg(prm + dm.b2);
  __syncthreads();
  return w;
}

// Unstaged view (read-only kernels: the batched matvecs of a P-program tile
// read each weight once per tile with coalesced loads, so staging would only
// cost occupancy).
template <typename R>
__device__ AttnW<R> attn_global_view(const TDims& dm, const R* prm) {
  AttnW<R> w;
  w.ldd = dm.D;
  w.ld1 = kHeadHidden;
  w.Wq = prm + dm.Wq;
  w.Wk = prm + dm.Wk;
  w.Wv = prm + dm.Wv;
  w.Wo = prm + dm.Wo;
  w.bq = prm + dm.bq;
  w.bo = prm + dm.bo;
  w.W1 = prm + dm.W1;
  w.b1 = prm + dm.b1;
  w.W2 = prm + dm.W2;
  w.b2 = prm[dm.b2];
  return w;
}

// --------------------------------------------------------- block matvecs --
// out[c] = bias[c] + sum_{k<K} v[k] W[k*ld + c]   (c < NC, NC | 256)
// Thread (c = tid % NC, s = tid / NC) sums k = s (mod S); the S partials are
// combined in fixed order through `red` (deterministic).  Ends synced.
template <typename R>
__device__ void bmv_col(const R* v, const R* W, int ld, int K, int NC, const R* bias, R* out,
                        R* red) {
  const int S = kThreads / NC;
  const int c = threadIdx.x % NC, s = threadIdx.x / NC;
  R acc = 0;
  for (int k = s; k < K; k += S) acc += v[k] * W[k * ld + c];
  red[threadIdx.x] = acc;
  __syncthreads();
  if ((int)threadIdx.x < NC) {
    R t = 0;
    for (int q = 0; q < S; ++q) t += red[q * NC + threadIdx.x];
    out[threadIdx.x] = bias ? t + bias[threadIdx.x] : t;
  }
  __syncthreads();
}

// out[k] = sum_{c<NC} W[k*ld + c] v[c]   (k < NK, NK | 256).  Ends synced.
template <typename R>
__device__ void bmv_row(const R* W, int ld, const R* v, int NC, int NK, R* out, R* red) {
  const int S = kThreads / NK;
  const int k = threadIdx.x % NK, s = threadIdx.x / NK;
  R acc = 0;
  for (int c = s; c < NC; c += S) acc += W[k * ld + c] * v[c];
  red[threadIdx.x] = acc;
  __syncthreads();
  if ((int)threadIdx.x < NK) {
    R t = 0;
    for (int q = 0; q < S; ++q) t += red[q * NK + threadIdx.x];
    out[threadIdx.x] = t;
  }
  __syncthreads();
}

// Batched over P programs: out[p*ldo + c] = bias[c] + sum_k v[p*ldv + k] W[k*ld + c].
template <typename R, int P>
__device__ void bmv_col_batch(const R* v, int ldv, const R* W, int ld, int K, int NC,
                              const R* bias, R* out, int ldo) {
  const int NG = kThreads / NC;
  const int c = threadIdx.x % NC, g = threadIdx.x / NC;
  for (int p0 = g; p0 < P; p0 += 2 * NG) {
    const int p1 = p0 + NG;
    R a0 = 0, a1 = 0;
    const R* v0 = v + p0 * ldv;
    const R* v1 = v + (p1 < P ? p1 : p0) * ldv;
    for (int k = 0; k < K; ++k) {
      const R wk = W[k * ld + c];
      a0 = fma_rn(v0[k], wk, a0);
      a1 = fma_rn(v1[k], wk, a1);
    }
    const R b = bias ? bias[c] : (R)0;
    out[p0 * ldo + c] = a0 + b;
    if (p1 < P) out[p1 * ldo + c] = a1 + b;
  }
}

// ----------------------------------------------------------- LSTM layer --
// One bidirectional layer for P programs.  The input row of program p at time
// t is ti.step0[p] + t*d0 for layer 0 (raw steps) and inbuf + (p*Tmax+t)*D
// otherwise (previous layer output).  Output rows:
// out[(p*Tmax + t)*D + dir*H + j].
// TRAIN (P == 1): also records gates / cell state / tanh(cell) per step.
// Copy n16 16-byte chunks global -> shared with all threads of the CTA, four
// loads in flight per thread (a tile's layer rows; ends synced).
__device__ __forceinline__ void stage_rows_cta(const void* src_, void* dst_, int n16) {
  const int4* src = reinterpret_cast<const int4*>(src_);
  int4* dst = reinterpret_cast<int4*>(dst_);
  const int nt = blockDim.x;
  for (int i0 = threadIdx.x; i0 < n16; i0 += 4 * nt) {
    int4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (i0 + u * nt < n16) v[u] = src[i0 + u * nt];
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (i0 + u * nt < n16) dst[i0 + u * nt] = v[u];
  }
  __syncthreads();
}

template <typename R, int H, int P, bool TRAIN>
__device__ void lstm_layer_fwd(const TDims& dm, const R* __restrict__ prm, int l,
                               const TileInfo<R, P>& ti, const R* inbuf, R* __restrict__ out,
                               R* sh_h, R* sh_g, R* xzbuf, R* cache_g, R* cache_c, R* cache_tc,
                               R* xin_s = nullptr) {
  constexpr int G = 4 * H, D = 2 * H, NR = 128 / G, NQ = 128 / H;
  const int dir = threadIdx.x >> 7, lt = threadIdx.x & 127;
  const int c = lt % G, r = lt / G;
  const int j = lt % H, q = lt / H;
  const int Tmax = dm.Tmax;
  const R* Wx = prm + dm.wx[l][dir];
  const R* Wh = prm + dm.wh[l][dir];
  const R bc = ldw<TRAIN>(prm + dm.bb[l][dir] + c);
  const int d_in = l == 0 ? dm.d0 : D;
  // Input projection hoisted out of the recurrence (layers >= 1): for every
  // valid (p, t), xz = b + x_t Wx[:, c].  Each thread later reads back only
  // the entries it wrote, so no barrier is needed.  The Wx column is live
  // only here, leaving the recurrence with the Wh column alone.
  R* xz = xzbuf + (int64_t)dir * P * Tmax * G;
  if (l > 0 && xin_s != nullptr) {
    // (all threads of the CTA) the layer-input rows from the L2 scratch into
    // shared memory in one pass, so the projection below does not wait one
    // L2 round trip per row
    // whole tile block (rows past a program's end are copied but unused)
    stage_rows_cta(inbuf, xin_s, (int)(P * Tmax * D * sizeof(R) / 16));
  }
  if (l > 0) {
    R wx[D];
#pragma unroll
    for (int k = 0; k < D; ++k) wx[k] = ldw<TRAIN>(Wx + k * G + c);
    // (two copies of the loop so the staged one compiles to shared-memory loads)
    if (xin_s != nullptr) {
#pragma unroll 1
      for (int p = r; p < P; p += NR) {
        const int n = ti.len[p];
        for (int t = 0; t < n; ++t)
          xz[((int64_t)p * Tmax + t) * G + c] =
              dot_reg<D>(xin_s + ((int64_t)p * Tmax + t) * D, wx) + bc;
      }
    } else {
#pragma unroll 1
      for (int p = r; p < P; p += NR) {
        const int n = ti.len[p];
        for (int t = 0; t < n; ++t)
          xz[((int64_t)p * Tmax + t) * G + c] =
              dot_reg<D>(inbuf + ((int64_t)p * Tmax + t) * D, wx) + bc;
      }
    }
  }
  R wh[H];
#pragma unroll
  for (int k = 0; k < H; ++k) wh[k] = ldw<TRAIN>(Wh + k * G + c);
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
    // gate phase: z = b + x_t Wx + h Wh ; activation by gate block.  One
    // program at a time (not unrolled) keeps the register file for the
    // stationary weight columns.
#pragma unroll 2
    for (int p = r; p < P; p += NR) {
      const int n = ti.len[p];
      if (s < n) {
        const int t = dir == 0 ? s : n - 1 - s;
        R z;
        if (l > 0) {
          z = xz[((int64_t)p * Tmax + t) * G + c];
        } else {
          const R* x = ti.step0[p] + (int64_t)t * dm.d0;
          z = bc;
          for (int k = 0; k < d_in; ++k) z = fma_rn(x[k], ldw<TRAIN>(Wx + k * G + c), z);
        }
        z += dot_reg<H>(hbase + p * H, wh);
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
          const R cn = fma_rn(gf, creg[ci], gi * gg);
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
  R* red;    // [kThreads]
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
// occupied slots.  All 256 threads participate; weights come from `w`
// (shared memory).  The TRAIN instance (P == 1) uses latency-oriented sliced
// matvecs; scoring uses the same per-program summation order (sequential over
// K, bias last) for every tile size P, so a program's score does not depend on
// how many programs share its launch (search-time re-batching is bit-exact).
template <typename R, int H, int P, bool TRAIN>
__device__ void attention_head_fwd(const TDims& dm, const AttnW<R>& w, const TileInfo<R, P>& ti,
                                   const R* __restrict__ S, R* __restrict__ Kb,
                                   R* __restrict__ Vb, const AttnSmem<R, P>& sm,
                                   const AttnCache<R>* cache, R* out_yhat) {
  constexpr int D = 2 * H;
  const int tid = threadIdx.x;
  const int Tmax = dm.Tmax, heads = dm.heads, dh = dm.dh, C = dm.C;
  const int warp = tid >> 5, lane = tid & 31;
  const int Z = D + C;
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
      const int col = cc % D;
      const R* wp = (cc < D ? w.Wk : w.Wv) + col;
      const int ld = w.ldd;
      R wc[D];
#pragma unroll
      for (int k = 0; k < D; ++k) {
        wc[k] = *wp;
        wp += ld;
      }
      R* dst = cc < D ? Kb : Vb;
      for (int p = 0; p < P; ++p) {
        const int n = ti.len[p];
        for (int t = grp; t < n; t += NGRP) {
          const int64_t row = ((int64_t)p * Tmax + t) * D;
          dst[row + col] = dot_reg<D>(S + row, wc);
        }
      }
    }
  }
  __syncthreads();
  const R sq = sqrt((R)dh);
  for (int u = 0; u < dm.U; ++u) {
    // q = pooled Wq + bq
    if constexpr (P == 1 && TRAIN)
      bmv_col<R>(sm.pool, w.Wq, w.ldd, D, D, w.bq, sm.q, sm.red);
    else {
      bmv_col_batch<R, P>(sm.pool, D, w.Wq, w.ldd, D, D, w.bq, sm.q, D);
      __syncthreads();
    }
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
        for (int d = 0; d < dh; ++d) acc = fma_rn(qh[d], kr[d], acc);
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
      for (int t = 0; t < n; ++t) acc = fma_rn(al[t], Vb[((int64_t)p * Tmax + t) * D + c], acc);
      sm.mix[i] = acc;
    }
    __syncthreads();
    if constexpr (TRAIN) {
      for (int i = tid; i < D; i += kThreads) cache->mix[u * D + i] = sm.mix[i];
      for (int i = tid; i < heads * Tmax; i += kThreads) cache->alpha[u * heads * Tmax + i] = sm.alpha[i];
    }
    // pooled = mix Wo + bo
    if constexpr (P == 1 && TRAIN)
      bmv_col<R>(sm.mix, w.Wo, w.ldd, D, D, w.bo, sm.pool, sm.red);
    else {
      bmv_col_batch<R, P>(sm.mix, D, w.Wo, w.ldd, D, D, w.bo, sm.pool, D);
      __syncthreads();
    }
  }
  // head: z = [pooled | ctx] ; a1 = tanh(z W1 + b1) ; yhat = sigmoid(a1 W2 + b2)
  for (int i = tid; i < P * Z; i += kThreads) {
    const int p = i / Z, k = i % Z;
    R v = 0;
    if (k < D)
      v = sm.pool[p * D + k];
    else if (ti.prog[p] >= 0)  // a program without steps keeps its context (tuner.py:276)
      v = __ldg(ti.ctx[p] + (k - D));
    sm.z[i] = v;
  }
  __syncthreads();
  if constexpr (P == 1 && TRAIN)
    bmv_col<R>(sm.z, w.W1, w.ld1, Z, kHeadHidden, w.b1, sm.a1, sm.red);
  else {
    bmv_col_batch<R, P>(sm.z, Z, w.W1, w.ld1, Z, kHeadHidden, w.b1, sm.a1, kHeadHidden);
    __syncthreads();
  }
  for (int i = tid; i < P * kHeadHidden; i += kThreads) sm.a1[i] = Act<R>::tanh(sm.a1[i]);
  __syncthreads();
  for (int p = warp; p < P; p += kThreads / 32) {
    R acc = 0;
    for (int c = lane; c < kHeadHidden; c += 32) acc = fma_rn(sm.a1[p * kHeadHidden + c], w.W2[c], acc);
    acc = warp_sum(acc);
    if (lane == 0 && ti.prog[p] >= 0) {
      const R yh = Act<R>::sigmoid(acc + w.b2);
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

// Counting sort of n programs by length (longest first) into perm
// (tt_tuner_x3.cu); the tensor-core scorers fill their 128-program tiles in
// this order.
int sort_programs_by_length(const int64_t* rowoff, int64_t n, int Tmax, int32_t* perm, void* scratch,
                            cudaStream_t st);
size_t sort_scratch_bytes(int Tmax);

}  // namespace tt
