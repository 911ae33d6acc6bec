// Attention tuner: backward pass of one sample (tuner.py:287-360 and
// _LstmDirection.backward :102-151), accumulated into a per-CTA partial
// gradient vector laid out exactly like the parameter vector.
//
// Weights come from shared memory: the attention/head block staged by
// stage_attn (reused from the forward pass) and, per LSTM layer, both
// directions' Wx/Wh staged with a +1 padded row stride so the transposed
// products (dh = dz Wh^T, dX = dZ Wx^T) are bank-conflict free.
#pragma once

#include "tt_tuner.cuh"

namespace tt {

// Phase timestamps (clock64) of CTA 0 for one chosen minibatch: a debug aid
// exported as tt_debug_phase_times (off unless tt_debug_profile_step >= 0).
static __device__ long long g_phase[32];
static __device__ int g_prof_step = -1;
__device__ __forceinline__ void phase_mark(int step, int i) {
  if (blockIdx.x == 0 && threadIdx.x == 0 && step == g_prof_step) g_phase[i] = clock64();
}

// Element offsets of the per-sample training cache and the per-CTA backward
// scratch.  Every segment is padded to 4 elements so rows stay 16-B aligned.
struct TrainLayout {
  int64_t S, gates, cst, tcs, K, V, pin, q, mix, alpha, z, a1, yhat, sample_elems;
  int64_t dS, dK, dV, dZ, dX, xz, bwd_elems;
  int NH;  // dX partial groups
};

inline int64_t pad4(int64_t x) { return (x + 3) & ~int64_t(3); }

inline TrainLayout make_train_layout(const TDims& d) {
  TrainLayout t{};
  int64_t o = 0;
  auto seg = [&](int64_t n) {
    const int64_t at = o;
    o += pad4(n);
    return at;
  };
  const int64_t TD = (int64_t)d.Tmax * d.D;
  t.S = seg(d.L * TD);
  t.gates = seg((int64_t)d.L * 2 * d.Tmax * d.G);
  t.cst = seg((int64_t)d.L * 2 * d.Tmax * d.H);
  t.tcs = seg((int64_t)d.L * 2 * d.Tmax * d.H);
  t.K = seg(TD);
  t.V = seg(TD);
  t.pin = seg((int64_t)d.U * d.D);
  t.q = seg((int64_t)d.U * d.D);
  t.mix = seg((int64_t)d.U * d.D);
  t.alpha = seg((int64_t)d.U * d.heads * d.Tmax);
  t.z = seg(d.D + d.C);
  t.a1 = seg(kHeadHidden);
  t.yhat = seg(1);
  t.sample_elems = o;
  o = 0;
  t.NH = 128 / d.D > 0 ? 128 / d.D : 1;
  t.dS = seg(TD);
  t.dK = seg(TD);
  t.dV = seg(TD);
  t.dZ = seg((int64_t)2 * d.Tmax * d.G);
  t.dX = seg((int64_t)2 * t.NH * TD);
  t.xz = seg((int64_t)2 * d.Tmax * d.G);
  t.bwd_elems = o;
  return t;
}

// smem elements for one layer's staged LSTM weights (both directions)
__host__ __device__ inline int64_t lstm_stage_elems(const TDims& d) {
  // layers >= 1: 2 x [Wx | Wh | b] rows (D + H + 1); layer 0 stages Wh only
  const int64_t per_dir = (int64_t)(d.D + d.H + 1) * (d.G + 1);
  const int64_t l0 = (int64_t)d.H * (d.G + 1);
  const int64_t n = 2 * (per_dir > l0 ? per_dir : l0);
  return (n + 3) & ~int64_t(3);
}

template <typename R>
__device__ __forceinline__ void put(R* part, int64_t idx, R val, bool store) {
  if (store)
    part[idx] = val;
  else
    part[idx] += val;
}

// Backward shared memory (per CTA).
template <typename R>
struct BwdSmem {
  R* da1;   // [64]
  R* dpool; // [D]
  R* dmix;  // [D]
  R* dq;    // [D]
  R* dlog;  // [heads][Tmax]
  R* dz;    // [2][G]
  R* part;  // [2][NQ][H]
  R* red;   // [kThreads]
};

// -------------------------------------------------- LSTM layer backward --
// dS: in = d(loss)/d(layer output) [Tmax][D]; out (l > 0) = d/d(layer input).
// wst: shared memory for this layer's weights (lstm_stage_elems).
template <typename R, int H>
__device__ void lstm_layer_bwd(const TDims& dm, const TrainLayout& ly, const R* __restrict__ prm,
                               int l, int len, const R* xin, int in_stride, const R* smp,
                               R* bws, const BwdSmem<R>& sm, R* wst, R* part, bool fresh,
                               int step = -2) {
  const int pstep = l == 1 ? step : -2;  // fine-grained marks for the middle layer
  constexpr int G = 4 * H, D = 2 * H, NQ = 128 / H, NW = (G + NQ - 1) / NQ;
  const int dir = threadIdx.x >> 7, lt = threadIdx.x & 127;
  const int j = lt % H, q = lt / H;
  const int Tmax = dm.Tmax;
  const int ldg = G + 1;
  const int d_in = l == 0 ? dm.d0 : D;
  // ---- stage the layer's weights into shared memory.  In the parameter
  // layout a direction is [Wx | Wh | b] and the bw block follows the fw one,
  // so layers >= 1 are one contiguous block of 2*(D+H+1) rows; layer 0 only
  // needs Wh (its dX is discarded, dWx does not read Wx).
  int64_t per_dir;
  const R* Whs;
  const R* Wxs;
  if (l > 0) {
    per_dir = (int64_t)(D + H + 1) * ldg;
    stage_rows<R, G>(wst, ldg, prm + dm.wx[l][0], 2 * (D + H + 1));
    Wxs = wst + dir * per_dir;
    Whs = Wxs + (int64_t)D * ldg;
  } else {
    per_dir = (int64_t)H * ldg;
    stage_rows<R, G>(wst, ldg, prm + dm.wh[0][0], H);
    stage_rows<R, G>(wst + per_dir, ldg, prm + dm.wh[0][1], H);
    Whs = wst + dir * per_dir;
    Wxs = nullptr;
  }
  __syncthreads();
  phase_mark(pstep, 20);
  const R* gates = smp + ly.gates + (int64_t)l * 2 * Tmax * G;
  const R* cst = smp + ly.cst + (int64_t)l * 2 * Tmax * H;
  const R* tcs = smp + ly.tcs + (int64_t)l * 2 * Tmax * H;
  const R* Sout = smp + ly.S + (int64_t)l * Tmax * D;
  R* dS = bws + ly.dS;
  R* dZ = bws + ly.dZ + (int64_t)dir * Tmax * G;
  R* dzs = sm.dz + dir * G;
  R* parts = sm.part + dir * NQ * H;
  R whr[NW];
#pragma unroll
  for (int i = 0; i < NW; ++i) {
    const int c = q + i * NQ;
    whr[i] = c < G ? Whs[j * ldg + c] : (R)0;
  }
  R dwh[H];
#pragma unroll
  for (int k = 0; k < H; ++k) dwh[k] = 0;
  R dbc = 0, dc = 0;
  for (int i = lt; i < NQ * H; i += 128) parts[i] = 0;
  named_barrier(1 + dir, 128);
  for (int s = len - 1; s >= 0; --s) {
    const int t = dir == 0 ? s : len - 1 - s;
    const int tp = dir == 0 ? t - 1 : t + 1;
    if (lt < H) {
      R dh = 0;
#pragma unroll
      for (int qq = 0; qq < NQ; ++qq) dh += parts[qq * H + j];
      const R dh_tot = dS[t * D + dir * H + j] + dh;
      const R* gt = gates + ((int64_t)dir * Tmax + t) * G;
      const R gi = gt[j], gf = gt[H + j], gg = gt[2 * H + j], go = gt[3 * H + j];
      const R tc = tcs[((int64_t)dir * Tmax + t) * H + j];
      const R cp = s >= 1 ? cst[((int64_t)dir * Tmax + tp) * H + j] : (R)0;
      const R dO = dh_tot * tc;
      const R dcr = dc + dh_tot * go * ((R)1 - tc * tc);
      const R dzi = dcr * gg * gi * ((R)1 - gi);
      const R dzf = dcr * cp * gf * ((R)1 - gf);
      const R dzg = dcr * gi * ((R)1 - gg * gg);
      const R dzo = dO * go * ((R)1 - go);
      dc = dcr * gf;
      dzs[j] = dzi;
      dzs[H + j] = dzf;
      dzs[2 * H + j] = dzg;
      dzs[3 * H + j] = dzo;
      R* dzt = dZ + (int64_t)t * G;
      dzt[j] = dzi;
      dzt[H + j] = dzf;
      dzt[2 * H + j] = dzg;
      dzt[3 * H + j] = dzo;
    }
    named_barrier(1 + dir, 128);
    if (lt < G) {
      const R dz = dzs[lt];
      dbc += dz;
      if (s >= 1) {
        const R* hp = Sout + (int64_t)tp * D + dir * H;
#pragma unroll
        for (int k = 0; k < H; ++k) dwh[k] += hp[k] * dz;
      }
    }
    {
      R acc = 0;
#pragma unroll
      for (int i = 0; i < NW; ++i) {
        const int c = q + i * NQ;
        if (c < G) acc += whr[i] * dzs[c];
      }
      parts[q * H + j] = acc;
    }
    named_barrier(1 + dir, 128);
  }
  phase_mark(pstep, 21);
  if (lt < G) {
#pragma unroll
    for (int k = 0; k < H; ++k) put(part, dm.wh[l][dir] + (int64_t)k * G + lt, dwh[k], fresh);
    put(part, dm.bb[l][dir] + lt, dbc, fresh);
    // dWx[k][c] = sum_t x_t[k] dZ[t][c]
    if (l > 0) {
      R acc[D];
#pragma unroll
      for (int k = 0; k < D; ++k) acc[k] = 0;
      for (int t = 0; t < len; ++t) {
        const R dz = dZ[(int64_t)t * G + lt];
        const R* xr = xin + (int64_t)t * in_stride;
#pragma unroll
        for (int k = 0; k < D; ++k) acc[k] += xr[k] * dz;
      }
#pragma unroll
      for (int k = 0; k < D; ++k) put(part, dm.wx[l][dir] + (int64_t)k * G + lt, acc[k], fresh);
    } else {
      for (int k = 0; k < d_in; ++k) {
        R acc = 0;
        for (int t = 0; t < len; ++t) acc += xin[(int64_t)t * in_stride + k] * dZ[(int64_t)t * G + lt];
        put(part, dm.wx[l][dir] + (int64_t)k * G + lt, acc, fresh);
      }
    }
  }
  phase_mark(pstep, 22);
  if (l > 0) {
    // dX[t][k] = sum_c Wx[k][c] dZ[t][c]; thread (k, hq) owns the contiguous
    // column slice [hq*CW, (hq+1)*CW) of row k in registers and streams the
    // dZ rows as broadcast vector loads.
    constexpr int NHc = 128 / D;          // column groups (== ly.NH)
    constexpr int CW = G / NHc;           // columns per group
    const int k = lt % D, hq = lt / D;
    R wr[CW];
    const R* wrow = Wxs + (int64_t)k * ldg + hq * CW;
#pragma unroll
    for (int c = 0; c < CW; ++c) wr[c] = wrow[c];
    R* dX = bws + ly.dX + ((int64_t)(dir * NHc + hq) * Tmax) * D;
    for (int t = 0; t < len; ++t)
      dX[(int64_t)t * D + k] = dot_reg<CW>(dZ + (int64_t)t * G + hq * CW, wr);
  }
  __syncthreads();
  phase_mark(pstep, 23);
  if (l > 0) {
    const int NH = ly.NH;
    for (int i = threadIdx.x; i < len * D; i += kThreads) {
      R a = 0, b = 0;
      for (int hq = 0; hq < NH; ++hq) a += bws[ly.dX + (int64_t)hq * Tmax * D + i];
      for (int hq = 0; hq < NH; ++hq) b += bws[ly.dX + (int64_t)(NH + hq) * Tmax * D + i];
      dS[i] = a + b;  // dX_fw + dX_bw (tuner.py:359)
    }
  }
  __syncthreads();
}

// ------------------------------------------------------- sample backward --
// aw: attention/head weights staged in shared memory (stage_attn); wst: the
// LSTM staging region (may alias aw's storage -- aw is dead by then).
template <typename R, int H>
__device__ void backward_sample(const TDims& dm, const TrainLayout& ly, const R* __restrict__ prm,
                                const AttnW<R>& aw, int len, const R* step0, R dy, const R* smp,
                                R* bws, const BwdSmem<R>& sm, R* wst, R* part, bool fresh,
                                int step) {
  constexpr int D = 2 * H;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int Tmax = dm.Tmax, heads = dm.heads, dh = dm.dh, C = dm.C, U = dm.U;
  const int Z = D + C;
  const R sq = sqrt((R)dh);
  // ---- head (tuner.py:298-306)
  const R yh = smp[ly.yhat];
  const R dl = dy * yh * ((R)1 - yh);
  const R* a1 = smp + ly.a1;
  const R* z = smp + ly.z;
  if (tid < kHeadHidden) {
    const R av = a1[tid];
    put(part, dm.W2 + tid, av * dl, fresh);
    const R da = dl * aw.W2[tid] * ((R)1 - av * av);
    sm.da1[tid] = da;
    put(part, dm.b1 + tid, da, fresh);
  }
  if (tid == 0) put(part, dm.b2, dl, fresh);
  __syncthreads();
  for (int i = tid; i < Z * kHeadHidden; i += kThreads) {
    const int k = i / kHeadHidden, c = i % kHeadHidden;
    put(part, dm.W1 + i, z[k] * sm.da1[c], fresh);
  }
  bmv_row<R>(aw.W1, aw.ld1, sm.da1, kHeadHidden, D, sm.dpool, sm.red);
  // ---- attention passes in reverse (tuner.py:310-328)
  const R* Kb = smp + ly.K;
  const R* Vb = smp + ly.V;
  R* dK = bws + ly.dK;
  R* dV = bws + ly.dV;
  for (int u = U - 1; u >= 0; --u) {
    const bool st = fresh && (u == U - 1);
    const R* mix = smp + ly.mix + u * D;
    const R* pin = smp + ly.pin + u * D;
    const R* qv = smp + ly.q + u * D;
    const R* al = smp + ly.alpha + (int64_t)u * heads * Tmax;
    for (int i = tid; i < D * D; i += kThreads) put(part, dm.Wo + i, mix[i / D] * sm.dpool[i % D], st);
    for (int c = tid; c < D; c += kThreads) put(part, dm.bo + c, sm.dpool[c], st);
    bmv_row<R>(aw.Wo, aw.ldd, sm.dpool, D, D, sm.dmix, sm.red);
    for (int h = warp; h < heads; h += kThreads / 32) {
      R sacc = 0;
      for (int t = lane; t < len; t += 32) {
        R da = 0;
        for (int d = 0; d < dh; ++d) da += sm.dmix[h * dh + d] * Vb[(int64_t)t * D + h * dh + d];
        sm.dlog[h * Tmax + t] = da;
        sacc += da * al[h * Tmax + t];
      }
      sacc = warp_sum(sacc);
      for (int t = lane; t < len; t += 32) {
        const R da = sm.dlog[h * Tmax + t];
        sm.dlog[h * Tmax + t] = al[h * Tmax + t] * (da - sacc);
      }
    }
    __syncthreads();
    for (int i = tid; i < len * D; i += kThreads) {
      const int t = i / D, c = i % D, h = c / dh;
      const R dv = al[h * Tmax + t] * sm.dmix[c];
      const R dk = sm.dlog[h * Tmax + t] * qv[c] / sq;
      if (u == U - 1) {
        dV[i] = dv;
        dK[i] = dk;
      } else {
        dV[i] += dv;
        dK[i] += dk;
      }
    }
    for (int c = tid; c < D; c += kThreads) {
      const int h = c / dh;
      R acc = 0;
      for (int t = 0; t < len; ++t) acc += sm.dlog[h * Tmax + t] * Kb[(int64_t)t * D + c];
      sm.dq[c] = acc / sq;
    }
    __syncthreads();
    for (int i = tid; i < D * D; i += kThreads) put(part, dm.Wq + i, pin[i / D] * sm.dq[i % D], st);
    for (int c = tid; c < D; c += kThreads) put(part, dm.bq + c, sm.dq[c], st);
    bmv_row<R>(aw.Wq, aw.ldd, sm.dq, D, D, sm.dpool, sm.red);
  }
  phase_mark(step, 10);
  // ---- d S (tuner.py:331-338)
  const R* S = smp + ly.S + (int64_t)(dm.L - 1) * Tmax * D;
  // gWk / gWv: thread column cc in [0, 2D), accumulators over k in registers
  for (int cc = tid; cc < 2 * D; cc += kThreads) {
    const R* src = cc < D ? dK : dV;
    const int col = cc % D;
    const int64_t off = cc < D ? dm.Wk : dm.Wv;
    R acc[D];
#pragma unroll
    for (int k = 0; k < D; ++k) acc[k] = 0;
    for (int t = 0; t < len; ++t) {
      const R g = src[(int64_t)t * D + col];
      const R* sr = S + (int64_t)t * D;
#pragma unroll
      for (int k = 0; k < D; ++k) acc[k] += sr[k] * g;
    }
#pragma unroll
    for (int k = 0; k < D; ++k) put(part, off + (int64_t)k * D + col, acc[k], fresh);
  }
  R* dS = bws + ly.dS;
  const R denom = (R)(len > 1 ? len : 1);
  for (int i = tid; i < len * D; i += kThreads) {
    const int t = i / D, k = i % D;
    const R* wk = aw.Wk + k * aw.ldd;
    const R* wv = aw.Wv + k * aw.ldd;
    const R* dkr = dK + (int64_t)t * D;
    const R* dvr = dV + (int64_t)t * D;
    R a = 0, b = 0;
    for (int c = 0; c < D; ++c) {
      a += dkr[c] * wk[c];
      b += dvr[c] * wv[c];
    }
    dS[i] = (sm.dpool[k] / denom + a) + b;
  }
  __syncthreads();
  // ---- LSTM stack in reverse (tuner.py:340-359); the staging region
  //      overwrites the attention weights from here on.
  phase_mark(step, 11);
  for (int l = dm.L - 1; l >= 0; --l) {
    const R* xin = l == 0 ? step0 : smp + ly.S + (int64_t)(l - 1) * Tmax * D;
    const int stride = l == 0 ? dm.d0 : D;
    lstm_layer_bwd<R, H>(dm, ly, prm, l, len, xin, stride, smp, bws, sm, wst, part, fresh, step);
    phase_mark(step, 12 + (dm.L - 1 - l));
  }
}

}  // namespace tt
