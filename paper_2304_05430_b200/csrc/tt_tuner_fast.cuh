// Attention tuner training, latency path (v4): hidden 32, fp32, minibatch
// B <= #SMs with every per-sample cache in shared memory.
//
// Reference: estimators/tuner.py _train/_forward/_backward (:227-466),
// _LstmDirection (:55-151), ranking_grad (mlp.py:25-35), Adam (optim.py).
//
// One persistent cooperative launch runs a whole epoch.  Two CTA roles:
//
//  * sample CTAs (blockIdx < B): CTA k owns minibatch slot k.  It runs the
//    sample's forward (3 x biLSTM, attention passes, head), exchanges the
//    scores through L2, evaluates the minibatch loss (identical arithmetic in
//    every sample CTA), then runs the ACTIVATION backward only: the
//    per-direction recurrences (BPTT) run on one warp each, lane j owning
//    hidden unit j and its 4 gate columns / its Wh row in registers.  Every
//    operand a weight gradient needs (layer outputs, dZ, dK, dV, attention
//    pass vectors, head vectors) is published to an L2 exchange slot.
//  * gradient jobs (all CTAs, non-sample CTAs first): the parameter vector is
//    cut into column slices of every weight matrix; a job reduces
//    dW[:, slice] = sum_rows A^T B over the minibatch rows in a fixed order
//    (deterministic, no atomics on data) and applies the fused Adam update
//    (or writes the gradient in TT_MODE_GRAD).
//
// Phases are ordered by three monotone L2 counters instead of grid barriers:
// forward-done (score exchange), backward-done (jobs may start) and
// adam-done (next minibatch may read the parameters).  The weight gradient
// never materialises per sample: the traffic per step is the exchange slots
// (~45 KB/sample at T = 10) instead of B partial 330 KB gradient vectors.
#pragma once

#include "tt_tuner_train.cuh"

namespace tt {

constexpr int kFH = 32, kFD = 64, kFG = 128;  // hidden, 2H, 4H
constexpr int kLdA = 65;                       // staged attention weights row stride

// ------------------------------------------------------------ layouts --
struct FastSmem {  // float offsets in dynamic shared memory (sample role)
  int64_t S, gc, cs, xz, hb, K, V, alpha, pin, q, mix, pool, zb, a1, red, lb, dS, dS2, dZ, dK,
      dV, dlg, dmix, dq, dpool, da1, W, total;
};

struct FastXch {  // float offsets inside one exchange slot
  int64_t S, dZ, dK, dV, pin, mix, dpool, dq, z, a1, da1, dl, total;
};

inline FastSmem make_fast_smem(const TDims& d, int B) {
  FastSmem s{};
  int64_t o = 0;
  auto seg = [&](int64_t n) {
    const int64_t at = o;
    o += pad4(n);
    return at;
  };
  const int TM = d.Tmax;
  s.S = seg((int64_t)d.L * TM * kFD);
  s.gc = seg((int64_t)d.L * 2 * TM * kFG);
  s.cs = seg((int64_t)d.L * 2 * TM * kFH);
  s.xz = seg((int64_t)2 * TM * kFG);  // also the dX partials [4][TM][64]
  s.hb = seg(2 * 2 * kFH);
  s.K = seg((int64_t)TM * kFD);
  s.V = seg((int64_t)TM * kFD);
  s.alpha = seg((int64_t)d.U * d.heads * TM);
  s.pin = seg((int64_t)d.U * kFD);
  s.q = seg((int64_t)d.U * kFD);
  s.mix = seg((int64_t)d.U * kFD);
  s.pool = seg(kFD);
  s.zb = seg(kFD + d.C);
  s.a1 = seg(kHeadHidden);
  s.red = seg(kThreads);
  s.lb = seg((int64_t)3 * B);
  s.dS = seg((int64_t)TM * kFD);
  s.dS2 = seg((int64_t)TM * kFD);
  s.dZ = seg((int64_t)2 * TM * kFG);
  s.dK = seg((int64_t)TM * kFD);
  s.dV = seg((int64_t)TM * kFD);
  s.dlg = seg((int64_t)d.heads * TM);
  s.dmix = seg(kFD);
  s.dq = seg(kFD);
  s.dpool = seg(kFD);
  s.da1 = seg(kHeadHidden);
  // attention + head weights, row stride 65: [Wq|Wk|Wv|Wo|bq|bo] then [W1|b1|W2]
  s.W = seg((int64_t)(4 * kFD + 2) * kLdA + (int64_t)(kFD + d.C + 2) * kLdA);
  s.total = o;
  return s;
}

inline FastXch make_fast_xch(const TDims& d) {
  FastXch x{};
  int64_t o = 0;
  auto seg = [&](int64_t n) {
    const int64_t at = o;
    o += pad4(n);
    return at;
  };
  const int TM = d.Tmax;
  x.S = seg((int64_t)d.L * TM * kFD);
  x.dZ = seg((int64_t)d.L * 2 * TM * kFG);
  x.dK = seg((int64_t)TM * kFD);
  x.dV = seg((int64_t)TM * kFD);
  x.pin = seg((int64_t)d.U * kFD);
  x.mix = seg((int64_t)d.U * kFD);
  x.dpool = seg((int64_t)d.U * kFD);
  x.dq = seg((int64_t)d.U * kFD);
  x.z = seg(kFD + d.C);
  x.a1 = seg(kHeadHidden);
  x.da1 = seg(kHeadHidden);
  x.dl = seg(1);
  x.total = o;
  return x;
}

// ------------------------------------------------------ gradient jobs --
enum FastJobKind { FJ_LSTM = 0, FJ_WQ, FJ_WK, FJ_WV, FJ_WO, FJ_W1, FJ_W2 };
constexpr int kCwLstm = 8, kCwAttn = 16, kCwHead = 16;

struct FastJob {
  int kind, l, dir, c0, nb;  // nb = slice width (columns)
};

__host__ __device__ inline int fast_n_jobs(const TDims& d) {
  return d.L * 2 * (kFG / kCwLstm) + 4 * (kFD / kCwAttn) + kHeadHidden / kCwHead + 1;
}

__host__ __device__ inline FastJob fast_job(const TDims& d, int j) {
  const int nl = d.L * 2 * (kFG / kCwLstm);
  if (j < nl) {
    const int per = kFG / kCwLstm;
    const int ld = j / per;
    return FastJob{FJ_LSTM, ld / 2, ld % 2, (j % per) * kCwLstm, kCwLstm};
  }
  j -= nl;
  const int pa = kFD / kCwAttn;
  if (j < 4 * pa) return FastJob{FJ_WQ + j / pa, 0, 0, (j % pa) * kCwAttn, kCwAttn};
  j -= 4 * pa;
  if (j < kHeadHidden / kCwHead) return FastJob{FJ_W1, 0, 0, j * kCwHead, kCwHead};
  return FastJob{FJ_W2, 0, 0, 0, 1};
}

// A-operand width of a job (including the ones column when the slice has a bias)
__device__ inline int fast_job_ka(const TDims& d, const FastJob& jb, bool& has_bias) {
  switch (jb.kind) {
    case FJ_LSTM: has_bias = true; return (jb.l == 0 ? d.d0 : kFD) + kFH + 1;
    case FJ_WQ: case FJ_WO: has_bias = true; return kFD + 1;
    case FJ_WK: case FJ_WV: has_bias = false; return kFD;
    case FJ_W1: has_bias = true; return kFD + d.C + 1;
    default: has_bias = true; return kHeadHidden + 1;  // W2 | b2
  }
}

__host__ __device__ inline int round4(int x) { return (x + 3) & ~3; }

// smem floats a job needs for `rows` staged rows (plus the reduction area)
__host__ __device__ inline int64_t fast_job_smem(int kap, int nbp, int rows) {
  return (int64_t)rows * (kap + nbp) + (int64_t)kThreads * 16 + (int64_t)kap * nbp + 64;
}

// ------------------------------------------------------------- args --
struct FastArgs {
  TDims dm;
  FastSmem sl;
  FastXch xl;
  float* prm;
  float* m;
  float* v;
  const float* steps;
  const int64_t* rowoff;
  const float* ctx;
  const float* y;
  const int32_t* order;
  int64_t n_order;
  int B;
  int loss_kind;
  int mode;
  int n_steps;
  AdamHyper hyp;
  const double* corr;
  const uint8_t* trainable;
  float* step_loss;
  float* grad_out;
  int32_t* status;
  float* xch;          // [B][xl.total]
  int64_t* meta;       // [B][2]: row offset, steps
  float* yhat_buf;     // [B]
  unsigned int* ctr;   // [0] fwd, [1] bwd, [2] adam (monotone)
  int n_jobs;
  int64_t rch;         // job staging rows per chunk
};

// phase mark from any CTA (the first job CTA records the job timeline)
// (%globaltimer, ns: comparable across SMs, unlike clock64)
__device__ __forceinline__ void phase_mark_any(int step, int i) {
  if (threadIdx.x == 0 && step == g_prof_step) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_phase[i] = (long long)t;
  }
}

// ------------------------------------------------------------- sync --
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// All threads; thread 0 spins until *ctr >= target.
__device__ __forceinline__ void wait_counter(const unsigned* ctr, unsigned target, bool sleep) {
  if (threadIdx.x == 0) {
    while (ld_acquire(ctr) < target) {
      if (sleep) __nanosleep(64);
    }
  }
  __syncthreads();
}

__device__ __forceinline__ void signal_counter(unsigned* ctr, unsigned inc) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(ctr, inc);
  }
}

__device__ __forceinline__ void cp_async4(float* s, const float* g) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(s);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(sa), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_async16(float* s, const float* g) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(s);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_all;" ::: "memory");
}

// ------------------------------------------------------ recurrences --
// Forward recurrence of one direction on one warp.  Lane j: hidden unit j,
// gate columns {j, 32+j, 64+j, 96+j} of Wh in registers (128 floats).
// xz: [2][TM][128] input projections (bias included).  Writes the layer
// output rows S[t][dir*32 + j] (smem + exchange), gates and cell state.
__device__ __forceinline__ void fast_rec_fwd(int dir, int T, int TM, const float* __restrict__ Wh,
                                             const float* xz, float* S, float* Sg, float* gc,
                                             float* cs, float* hb) {
  const int j = threadIdx.x & 31;
  float w[4][kFH];
#pragma unroll
  for (int k = 0; k < kFH; ++k)
#pragma unroll
    for (int g = 0; g < 4; ++g) w[g][k] = __ldcg(Wh + k * kFG + g * kFH + j);
  float c = 0.f;
  float* h0 = hb + dir * 2 * kFH;
  h0[j] = 0.f;
  __syncwarp();
  int cur = 0;
  for (int s = 0; s < T; ++s) {
    const int t = dir == 0 ? s : T - 1 - s;
    const float* xr = xz + ((int64_t)dir * TM + t) * kFG;
    float a[4][2];
#pragma unroll
    for (int g = 0; g < 4; ++g) {
      a[g][0] = xr[g * kFH + j];
      a[g][1] = 0.f;
    }
    const float4* h4 = reinterpret_cast<const float4*>(h0 + cur * kFH);
#pragma unroll
    for (int m = 0; m < kFH / 4; ++m) {
      const float4 hv = h4[m];
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        a[g][m & 1] = fmaf(hv.x, w[g][4 * m + 0], a[g][m & 1]);
        a[g][m & 1] = fmaf(hv.y, w[g][4 * m + 1], a[g][m & 1]);
        a[g][m & 1] = fmaf(hv.z, w[g][4 * m + 2], a[g][m & 1]);
        a[g][m & 1] = fmaf(hv.w, w[g][4 * m + 3], a[g][m & 1]);
      }
    }
    const float gi = Act<float>::sigmoid(a[0][0] + a[0][1]);
    const float gf = Act<float>::sigmoid(a[1][0] + a[1][1]);
    const float gg = Act<float>::tanh(a[2][0] + a[2][1]);
    const float go = Act<float>::sigmoid(a[3][0] + a[3][1]);
    c = gf * c + gi * gg;
    const float h = go * Act<float>::tanh(c);
    h0[(cur ^ 1) * kFH + j] = h;
    S[(int64_t)t * kFD + dir * kFH + j] = h;
    Sg[(int64_t)t * kFD + dir * kFH + j] = h;
    float* gr = gc + ((int64_t)dir * TM + t) * kFG;
    gr[j] = gi;
    gr[kFH + j] = gf;
    gr[2 * kFH + j] = gg;
    gr[3 * kFH + j] = go;
    cs[((int64_t)dir * TM + t) * kFH + j] = c;
    __syncwarp();
    cur ^= 1;
  }
}

// BPTT of one direction on one warp (tuner.py:113-148 restricted to the
// valid steps).  Lane j owns row j of Wh (128 floats) for dh = dZ Wh^T.
// dS: [TM][64] upstream gradient of this layer's output.  Writes dZ rows
// (smem [2][TM][128] and the exchange slot).
__device__ __forceinline__ void fast_rec_bwd(int dir, int T, int TM, const float* __restrict__ Wh,
                                             const float* gc, const float* cs, const float* dS,
                                             float* dZ, float* dZg) {
  const int j = threadIdx.x & 31;
  float wr[kFG];
  const float4* w4 = reinterpret_cast<const float4*>(Wh + (int64_t)j * kFG);
#pragma unroll
  for (int m = 0; m < kFG / 4; ++m) {
    const float4 v = __ldcg(w4 + m);
    wr[4 * m + 0] = v.x;
    wr[4 * m + 1] = v.y;
    wr[4 * m + 2] = v.z;
    wr[4 * m + 3] = v.w;
  }
  float dh = 0.f, dc = 0.f;
  for (int s = 0; s < T; ++s) {
    // reverse of the direction's forward order
    const int t = dir == 0 ? T - 1 - s : s;
    const bool has_prev = s < T - 1;
    const int tp = dir == 0 ? t - 1 : t + 1;
    const float* gr = gc + ((int64_t)dir * TM + t) * kFG;
    const float gi = gr[j], gf = gr[kFH + j], gg = gr[2 * kFH + j], go = gr[3 * kFH + j];
    const float cn = cs[((int64_t)dir * TM + t) * kFH + j];
    const float tc = Act<float>::tanh(cn);
    const float cp = has_prev ? cs[((int64_t)dir * TM + tp) * kFH + j] : 0.f;
    const float dht = dS[(int64_t)t * kFD + dir * kFH + j] + dh;
    const float dO = dht * tc;
    const float dcr = dc + dht * go * (1.f - tc * tc);
    const float dzi = dcr * gg * gi * (1.f - gi);
    const float dzf = dcr * cp * gf * (1.f - gf);
    const float dzg = dcr * gi * (1.f - gg * gg);
    const float dzo = dO * go * (1.f - go);
    dc = dcr * gf;
    float* zr = dZ + ((int64_t)dir * TM + t) * kFG;
    float* zg = dZg + ((int64_t)dir * TM + t) * kFG;
    zr[j] = dzi;
    zr[kFH + j] = dzf;
    zr[2 * kFH + j] = dzg;
    zr[3 * kFH + j] = dzo;
    zg[j] = dzi;
    zg[kFH + j] = dzf;
    zg[2 * kFH + j] = dzg;
    zg[3 * kFH + j] = dzo;
    __syncwarp();
    if (has_prev) {
      const float4* z4 = reinterpret_cast<const float4*>(zr);
      float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
#pragma unroll
      for (int m = 0; m < kFG / 4; ++m) {
        const float4 zv = z4[m];
        a0 = fmaf(zv.x, wr[4 * m + 0], a0);
        a1 = fmaf(zv.y, wr[4 * m + 1], a1);
        a2 = fmaf(zv.z, wr[4 * m + 2], a2);
        a3 = fmaf(zv.w, wr[4 * m + 3], a3);
      }
      dh = (a0 + a1) + (a2 + a3);
    }
  }
}

// ------------------------------------------------- sample forward --
// All 256 threads.  Returns yhat (valid in every thread after the call).
__device__ float fast_sample_fwd(const FastArgs& a, float* sm, float* xs, int64_t r0, int T,
                                 int64_t idx, int step) {
  const TDims& dm = a.dm;
  const FastSmem& L = a.sl;
  const FastXch& X = a.xl;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int TM = dm.Tmax;
  float* S = sm + L.S;
  float* xz = sm + L.xz;
  float* W = sm + L.W;
  float* W1s = W + (4 * kFD + 2) * kLdA;
  for (int l = 0; l < dm.L; ++l) {
    // ---- input projection xz[dir][t][c] = b[c] + x_t Wx[:, c]
    {
      const int dir = tid >> 7, c = tid & 127;
      const float* Wx = a.prm + dm.wx[l][dir];
      const float bc = __ldcg(a.prm + dm.bb[l][dir] + c);
      float* xzr = xz + (int64_t)dir * TM * kFG + c;
      if (l == 0) {
        const float* x0 = a.steps + r0 * dm.d0;
        for (int t = 0; t < T; ++t) xzr[(int64_t)t * kFG] = bc;
        for (int k0 = 0; k0 < dm.d0; k0 += 8) {
          float wk[8];
#pragma unroll
          for (int kk = 0; kk < 8; ++kk)
            wk[kk] = k0 + kk < dm.d0 ? __ldcg(Wx + (int64_t)(k0 + kk) * kFG + c) : 0.f;
          for (int t = 0; t < T; ++t) {
            float acc = xzr[(int64_t)t * kFG];
#pragma unroll
            for (int kk = 0; kk < 8; ++kk)
              if (k0 + kk < dm.d0) acc = fmaf(__ldg(x0 + (int64_t)t * dm.d0 + k0 + kk), wk[kk], acc);
            xzr[(int64_t)t * kFG] = acc;
          }
        }
      } else {
        float wk[kFD];
#pragma unroll
        for (int k = 0; k < kFD; ++k) wk[k] = __ldcg(Wx + (int64_t)k * kFG + c);
        const float* xin = S + (int64_t)(l - 1) * TM * kFD;
        for (int t = 0; t < T; ++t) xzr[(int64_t)t * kFG] = dot_reg<kFD>(xin + (int64_t)t * kFD, wk) + bc;
      }
    }
    __syncthreads();
    if (warp < 2) {
      fast_rec_fwd(warp, T, TM, a.prm + dm.wh[l][warp], xz, S + (int64_t)l * TM * kFD,
                   xs + X.S + (int64_t)l * TM * kFD, sm + L.gc + (int64_t)l * 2 * TM * kFG,
                   sm + L.cs + (int64_t)l * 2 * TM * kFH, sm + L.hb);
      if (warp == 0) phase_mark(step, 2 + l);
    } else if (l == 0) {
      // idle warps stage the attention/head weights (changed by the last Adam step)
      const int t2 = tid - 64, n2 = kThreads - 64;
      const int rows1 = 4 * kFD + 2, rows2 = kFD + dm.C + 2;
      const float* src1 = a.prm + dm.Wq;
      const float* src2 = a.prm + dm.W1;
      const int tot1 = rows1 * (kFD / 4), tot2 = rows2 * (kHeadHidden / 4);
      for (int i0 = t2; i0 < tot1 + tot2; i0 += 4 * n2) {
        float4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int i = i0 + u * n2;
          if (i < tot1)
            v[u] = __ldcg(reinterpret_cast<const float4*>(src1) + i);
          else if (i < tot1 + tot2)
            v[u] = __ldcg(reinterpret_cast<const float4*>(src2) + (i - tot1));
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int i = i0 + u * n2;
          if (i < tot1) {
            float* d = W + (i >> 4) * kLdA + (i & 15) * 4;
            d[0] = v[u].x, d[1] = v[u].y, d[2] = v[u].z, d[3] = v[u].w;
          } else if (i < tot1 + tot2) {
            const int ii = i - tot1;
            float* d = W1s + (ii >> 4) * kLdA + (ii & 15) * 4;
            d[0] = v[u].x, d[1] = v[u].y, d[2] = v[u].z, d[3] = v[u].w;
          }
        }
      }
    }
    __syncthreads();
  }
  // ---- attention (tuner.py:248-274)
  const int heads = dm.heads, dh = dm.dh, U = dm.U;
  const float* Sl = S + (int64_t)(dm.L - 1) * TM * kFD;
  float* K = sm + L.K;
  float* V = sm + L.V;
  float* pool = sm + L.pool;
  float* red = sm + L.red;
  const float* Wq = W;
  const float* Wk = W + kFD * kLdA;
  const float* Wv = W + 2 * kFD * kLdA;
  const float* Wo = W + 3 * kFD * kLdA;
  const float* bq = W + 4 * kFD * kLdA;
  const float* bo = W + (4 * kFD + 1) * kLdA;
  const int Z = kFD + dm.C;
  const float* b1 = W1s + (int64_t)Z * kLdA;
  const float* W2 = W1s + (int64_t)(Z + 1) * kLdA;
  const float b2 = __ldcg(a.prm + dm.b2);
  if (tid < kFD) {
    float acc = 0.f;
    for (int t = 0; t < T; ++t) acc += Sl[(int64_t)t * kFD + tid];
    pool[tid] = acc / (float)(T > 1 ? T : 1);
  }
  {
    const int cc = tid & 127, grp = tid >> 7, col = cc & 63;
    const float* wp = (cc < kFD ? Wk : Wv) + col;
    float wc[kFD];
#pragma unroll
    for (int k = 0; k < kFD; ++k) wc[k] = wp[k * kLdA];
    float* dst = cc < kFD ? K : V;
    for (int t = grp; t < T; t += 2) dst[(int64_t)t * kFD + col] = dot_reg<kFD>(Sl + (int64_t)t * kFD, wc);
  }
  __syncthreads();
  const float sq = sqrtf((float)dh);
  float* xsg = xs;
  for (int u = 0; u < U; ++u) {
    float* q = sm + L.q + u * kFD;
    bmv_col<float>(pool, Wq, kLdA, kFD, kFD, bq, q, red);
    if (tid < kFD) {
      sm[L.pin + u * kFD + tid] = pool[tid];
      xsg[X.pin + u * kFD + tid] = pool[tid];
    }
    float* al = sm + L.alpha + (int64_t)u * heads * TM;
    for (int h = warp; h < heads; h += kThreads / 32) {
      const float* qh = q + h * dh;
      float* ar = al + (int64_t)h * TM;
      float mx = -INFINITY;
      for (int t = lane; t < T; t += 32) {
        const float* kr = K + (int64_t)t * kFD + h * dh;
        float acc = 0.f;
        for (int d = 0; d < dh; ++d) acc += qh[d] * kr[d];
        acc = acc / sq;
        ar[t] = acc;
        mx = fmaxf(mx, acc);
      }
      mx = warp_max(mx);
      float sum = 0.f;
      for (int t = lane; t < T; t += 32) {
        const float e = Act<float>::exp(ar[t] - mx);
        ar[t] = e;
        sum += e;
      }
      sum = warp_sum(sum);
      for (int t = lane; t < T; t += 32) ar[t] = ar[t] / sum;
    }
    __syncthreads();
    float* mix = sm + L.mix + u * kFD;
    if (tid < kFD) {
      const float* ar = al + (int64_t)(tid / dh) * TM;
      float acc = 0.f;
      for (int t = 0; t < T; ++t) acc += ar[t] * V[(int64_t)t * kFD + tid];
      mix[tid] = acc;
      xsg[X.mix + u * kFD + tid] = acc;
    }
    __syncthreads();
    bmv_col<float>(mix, Wo, kLdA, kFD, kFD, bo, pool, red);
  }
  float* zb = sm + L.zb;
  for (int i = tid; i < Z; i += kThreads) {
    const float vz = i < kFD ? pool[i] : __ldg(a.ctx + idx * dm.C + (i - kFD));
    zb[i] = vz;
    xsg[X.z + i] = vz;
  }
  __syncthreads();
  float* a1 = sm + L.a1;
  bmv_col<float>(zb, W1s, kLdA, Z, kHeadHidden, b1, a1, red);
  float yh = 0.f;
  if (warp == 0) {
    float acc = 0.f;
    for (int c = lane; c < kHeadHidden; c += 32) {
      const float av = Act<float>::tanh(a1[c]);
      a1[c] = av;
      xsg[X.a1 + c] = av;
      acc += av * W2[c];
    }
    acc = warp_sum(acc);
    if (lane == 0) red[0] = Act<float>::sigmoid(acc + b2);
  }
  __syncthreads();
  yh = red[0];
  __syncthreads();
  return yh;
}

// ------------------------------------------------ sample backward --
__device__ void fast_sample_bwd(const FastArgs& a, float* sm, float* xs, int T, float dy,
                                float yh, int step) {
  const TDims& dm = a.dm;
  const FastSmem& L = a.sl;
  const FastXch& X = a.xl;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int TM = dm.Tmax, heads = dm.heads, dh = dm.dh, U = dm.U;
  const float* W = sm + L.W;
  const float* Wq = W;
  const float* Wk = W + kFD * kLdA;
  const float* Wv = W + 2 * kFD * kLdA;
  const float* Wo = W + 3 * kFD * kLdA;
  const float* W1s = W + (4 * kFD + 2) * kLdA;
  const int Z = kFD + dm.C;
  const float* W2 = W1s + (int64_t)(Z + 1) * kLdA;
  float* red = sm + L.red;
  float* da1 = sm + L.da1;
  float* dpool = sm + L.dpool;
  float* dmix = sm + L.dmix;
  float* dq = sm + L.dq;
  float* dlg = sm + L.dlg;
  const float* K = sm + L.K;
  const float* V = sm + L.V;
  float* dK = sm + L.dK;
  float* dV = sm + L.dV;
  // ---- head (tuner.py:298-306)
  const float dl = dy * yh * (1.f - yh);
  if (tid < kHeadHidden) {
    const float av = sm[L.a1 + tid];
    const float d = dl * W2[tid] * (1.f - av * av);
    da1[tid] = d;
    xs[X.da1 + tid] = d;
  }
  if (tid == 0) xs[X.dl] = dl;
  __syncthreads();
  bmv_row<float>(W1s, kLdA, da1, kHeadHidden, kFD, dpool, red);
  // ---- attention passes in reverse (tuner.py:310-328)
  const float sq = sqrtf((float)dh);
  for (int u = U - 1; u >= 0; --u) {
    if (tid < kFD) xs[X.dpool + u * kFD + tid] = dpool[tid];
    bmv_row<float>(Wo, kLdA, dpool, kFD, kFD, dmix, red);
    const float* al = sm + L.alpha + (int64_t)u * heads * TM;
    const float* qv = sm + L.q + u * kFD;
    for (int h = warp; h < heads; h += kThreads / 32) {
      float sacc = 0.f;
      for (int t = lane; t < T; t += 32) {
        float da = 0.f;
        for (int d = 0; d < dh; ++d) da += dmix[h * dh + d] * V[(int64_t)t * kFD + h * dh + d];
        dlg[h * TM + t] = da;
        sacc += da * al[h * TM + t];
      }
      sacc = warp_sum(sacc);
      for (int t = lane; t < T; t += 32) dlg[h * TM + t] = al[h * TM + t] * (dlg[h * TM + t] - sacc);
    }
    __syncthreads();
    for (int i = tid; i < T * kFD; i += kThreads) {
      const int t = i / kFD, c = i % kFD, h = c / dh;
      const float dv = al[h * TM + t] * dmix[c];
      const float dk = dlg[h * TM + t] * qv[c] / sq;
      if (u == U - 1) {
        dV[i] = dv;
        dK[i] = dk;
      } else {
        dV[i] += dv;
        dK[i] += dk;
      }
    }
    if (tid < kFD) {
      const int h = tid / dh;
      float acc = 0.f;
      for (int t = 0; t < T; ++t) acc += dlg[h * TM + t] * K[(int64_t)t * kFD + tid];
      dq[tid] = acc / sq;
      xs[X.dq + u * kFD + tid] = acc / sq;
    }
    __syncthreads();
    bmv_row<float>(Wq, kLdA, dq, kFD, kFD, dpool, red);
  }
  // ---- dS = dpool/denom + dK Wk^T + dV Wv^T (tuner.py:331-338)
  float* dS = sm + L.dS;
  const float denom = (float)(T > 1 ? T : 1);
  for (int i = tid; i < T * kFD; i += kThreads) {
    const int t = i / kFD, k = i % kFD;
    const float* wk = Wk + k * kLdA;
    const float* wv = Wv + k * kLdA;
    const float* dkr = dK + (int64_t)t * kFD;
    const float* dvr = dV + (int64_t)t * kFD;
    float s0 = 0.f, s1 = 0.f;
    for (int c = 0; c < kFD; ++c) {
      s0 = fmaf(dkr[c], wk[c], s0);
      s1 = fmaf(dvr[c], wv[c], s1);
    }
    dS[i] = (dpool[k] / denom + s0) + s1;
    xs[X.dK + i] = dK[i];
    xs[X.dV + i] = dV[i];
  }
  __syncthreads();
  phase_mark(step, 10);
  // ---- LSTM stack in reverse (tuner.py:340-359)
  float* dSa = dS;
  float* dSb = sm + L.dS2;
  float* dZ = sm + L.dZ;
  float* part = sm + L.xz;  // [4][TM][64] dX partials (xz is dead)
  for (int l = dm.L - 1; l >= 0; --l) {
    if (warp < 2)
      fast_rec_bwd(warp, T, TM, a.prm + dm.wh[l][warp], sm + L.gc + (int64_t)l * 2 * TM * kFG,
                   sm + L.cs + (int64_t)l * 2 * TM * kFH, dSa, dZ,
                   xs + X.dZ + (int64_t)l * 2 * TM * kFG);
    if (warp == 0) phase_mark(step, 11 + (dm.L - 1 - l) * 2);
    if (l == 0) break;
    // dX partials need this layer's Wx rows: load them while the BPTT warps run
    const int pq = tid >> 6, kk = tid & 63, dir = pq >> 1, cb = (pq & 1) * 64;
    float wr[64];
    {
      const float4* w4 = reinterpret_cast<const float4*>(a.prm + dm.wx[l][dir] + (int64_t)kk * kFG + cb);
#pragma unroll
      for (int m = 0; m < 16; ++m) {
        const float4 v = __ldcg(w4 + m);
        wr[4 * m + 0] = v.x;
        wr[4 * m + 1] = v.y;
        wr[4 * m + 2] = v.z;
        wr[4 * m + 3] = v.w;
      }
    }
    __syncthreads();
    for (int t = 0; t < T; ++t)
      part[((int64_t)pq * TM + t) * kFD + kk] =
          dot_reg<64>(dZ + ((int64_t)dir * TM + t) * kFG + cb, wr);
    __syncthreads();
    for (int i = tid; i < T * kFD; i += kThreads) {
      const int t = i / kFD, k = i % kFD;
      const float p0 = part[((int64_t)0 * TM + t) * kFD + k], p1 = part[((int64_t)1 * TM + t) * kFD + k];
      const float p2 = part[((int64_t)2 * TM + t) * kFD + k], p3 = part[((int64_t)3 * TM + t) * kFD + k];
      dSb[i] = (p0 + p1) + (p2 + p3);  // dX_fw + dX_bw (tuner.py:359)
    }
    __syncthreads();
    phase_mark(step, 12 + (dm.L - 1 - l) * 2);
    float* tmp = dSa;
    dSa = dSb;
    dSb = tmp;
  }
  __syncthreads();
}

// ------------------------------------------------------ job runner --
// Stage the rows of job `jb` for minibatch slots [k0, k1) into smem:
// A rows [rows][kap] (ones column appended when the slice has a bias),
// B rows [rows][nbp].  Returns the number of staged rows.
__device__ int fast_job_stage(const FastArgs& a, const FastJob& jb, int k0, int k1, int ka,
                              bool has_bias, int kap, int nbp, float* As, float* Bs) {
  const TDims& dm = a.dm;
  const FastXch& X = a.xl;
  const int tid = threadIdx.x;
  const int TM = dm.Tmax;
  int rows = 0;
  for (int k = k0; k < k1; ++k) {
    const float* xs = a.xch + (int64_t)k * X.total;
    const int T = (int)__ldcg(a.meta + 2 * k + 1);
    int nr;
    switch (jb.kind) {
      case FJ_LSTM:
      case FJ_WK:
      case FJ_WV: nr = T; break;
      case FJ_WQ:
      case FJ_WO: nr = dm.U; break;
      default: nr = 1;
    }
    float* Ar = As + (int64_t)rows * kap;
    float* Br = Bs + (int64_t)rows * nbp;
    if (jb.kind == FJ_LSTM) {
      const int l = jb.l, dir = jb.dir;
      const int din = l == 0 ? dm.d0 : kFD;
      const float* Sl = xs + X.S + (int64_t)l * TM * kFD;
      const float* dZ = xs + X.dZ + ((int64_t)l * 2 + dir) * TM * kFG + jb.c0;
      if (l == 0) {
        const int64_t r0 = __ldcg(a.meta + 2 * k);
        const float* x0 = a.steps + r0 * dm.d0;
        for (int i = tid; i < T * din; i += kThreads) cp_async4(Ar + (i / din) * kap + (i % din), x0 + i);
      } else {
        const float* Sp = xs + X.S + (int64_t)(l - 1) * TM * kFD;
        for (int i = tid; i < T * 16; i += kThreads)
          cp_async16(Ar + (i >> 4) * kap + (i & 15) * 4, Sp + (int64_t)(i >> 4) * kFD + (i & 15) * 4);
      }
      // h_prev in the direction's order (zero state at its first step)
      for (int i = tid; i < T * 8; i += kThreads) {
        const int t = i >> 3, q = i & 7;
        const int tp = dir == 0 ? t - 1 : t + 1;
        float* d = Ar + t * kap + din + q * 4;
        if (tp >= 0 && tp < T) {
          const float* src = Sl + (int64_t)tp * kFD + dir * kFH + q * 4;
          if (din & 3) {
            cp_async4(d, src), cp_async4(d + 1, src + 1), cp_async4(d + 2, src + 2), cp_async4(d + 3, src + 3);
          } else {
            cp_async16(d, src);
          }
        } else
          d[0] = d[1] = d[2] = d[3] = 0.f;
      }
      for (int i = tid; i < T * (jb.nb / 4); i += kThreads) {
        const int t = i / (jb.nb / 4), q = i % (jb.nb / 4);
        cp_async16(Br + t * nbp + q * 4, dZ + (int64_t)t * kFG + q * 4);
      }
    } else if (jb.kind == FJ_WK || jb.kind == FJ_WV) {
      const float* Sl = xs + X.S + (int64_t)(dm.L - 1) * TM * kFD;
      const float* G = xs + (jb.kind == FJ_WK ? X.dK : X.dV) + jb.c0;
      for (int i = tid; i < T * 16; i += kThreads)
        cp_async16(Ar + (i >> 4) * kap + (i & 15) * 4, Sl + (int64_t)(i >> 4) * kFD + (i & 15) * 4);
      for (int i = tid; i < T * (jb.nb / 4); i += kThreads) {
        const int t = i / (jb.nb / 4), q = i % (jb.nb / 4);
        cp_async16(Br + t * nbp + q * 4, G + (int64_t)t * kFD + q * 4);
      }
    } else if (jb.kind == FJ_WQ || jb.kind == FJ_WO) {
      const float* Av = xs + (jb.kind == FJ_WQ ? X.pin : X.mix);
      const float* G = xs + (jb.kind == FJ_WQ ? X.dq : X.dpool) + jb.c0;
      for (int i = tid; i < dm.U * 16; i += kThreads)
        cp_async16(Ar + (i >> 4) * kap + (i & 15) * 4, Av + (int64_t)(i >> 4) * kFD + (i & 15) * 4);
      for (int i = tid; i < dm.U * (jb.nb / 4); i += kThreads) {
        const int u = i / (jb.nb / 4), q = i % (jb.nb / 4);
        cp_async16(Br + u * nbp + q * 4, G + (int64_t)u * kFD + q * 4);
      }
    } else if (jb.kind == FJ_W1) {
      const int Z = kFD + dm.C;
      for (int i = tid; i < Z; i += kThreads) cp_async4(Ar + i, xs + X.z + i);
      for (int i = tid; i < jb.nb / 4; i += kThreads) cp_async16(Br + i * 4, xs + X.da1 + jb.c0 + i * 4);
    } else {  // W2 | b2: A = a1, B = dl
      for (int i = tid; i < kHeadHidden / 4; i += kThreads) cp_async16(Ar + i * 4, xs + X.a1 + i * 4);
      if (tid == 0) {
        cp_async4(Br, xs + X.dl);
        Br[1] = Br[2] = Br[3] = 0.f;
      }
    }
    // ones column (bias) and zero padding of A; zero padding of B
    const int ka_w = has_bias ? ka - 1 : ka;
    for (int i = tid; i < nr * (kap - ka_w); i += kThreads) {
      const int r = i / (kap - ka_w), cix = ka_w + i % (kap - ka_w);
      Ar[r * kap + cix] = (has_bias && cix == ka_w) ? 1.f : 0.f;
    }
    if (jb.nb < nbp && jb.kind != FJ_W2)
      for (int i = tid; i < nr * (nbp - jb.nb); i += kThreads) {
        const int r = i / (nbp - jb.nb);
        Br[r * nbp + jb.nb + i % (nbp - jb.nb)] = 0.f;
      }
    rows += nr;
  }
  cp_async_wait_all();
  __syncthreads();
  return rows;
}

__device__ void fast_run_job(const FastArgs& a, const FastJob& jb, int bn, int step, float* sm) {
  const TDims& dm = a.dm;
  const int tid = threadIdx.x;
  bool has_bias = false;
  const int ka = fast_job_ka(dm, jb, has_bias);
  const int kap = round4(ka), nbp = round4(jb.nb);
  const int nkb = kap / 4, ncb = nbp / 4, nblk = nkb * ncb;
  const int RG = nblk >= kThreads ? 1 : kThreads / nblk;
  const int TM = dm.Tmax;
  int maxr;
  switch (jb.kind) {
    case FJ_LSTM: case FJ_WK: case FJ_WV: maxr = TM; break;
    case FJ_WQ: case FJ_WO: maxr = dm.U; break;
    default: maxr = 1;
  }
  const int per_chunk = (int)(a.rch / maxr > 1 ? a.rch / maxr : 1);  // samples per staging chunk
  float* As = sm;
  float* Bs = As + (int64_t)per_chunk * maxr * kap;
  float* redb = Bs + (int64_t)per_chunk * maxr * nbp;   // [RG][nblk][16]
  float* gout = redb + (int64_t)kThreads * 16;          // [kap][nbp]
  // thread -> (row group g, 4x4 output block blk); nblk <= 256 (fast_plan)
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int jj = 0; jj < 4; ++jj) acc[i][jj] = 0.f;
  const int g = tid / nblk, blk = tid % nblk;
  const bool active = tid < RG * nblk;
  const int kb = blk / ncb, cb = blk % ncb;
  for (int k0 = 0; k0 < bn; k0 += per_chunk) {
    const int k1 = min(bn, k0 + per_chunk);
    __syncthreads();
    const int R = fast_job_stage(a, jb, k0, k1, ka, has_bias, kap, nbp, As, Bs);
    if (active) {
      for (int rr = g; rr < R; rr += RG) {
        const float4 av = *reinterpret_cast<const float4*>(As + (int64_t)rr * kap + kb * 4);
        const float4 bv = *reinterpret_cast<const float4*>(Bs + (int64_t)rr * nbp + cb * 4);
        const float ax[4] = {av.x, av.y, av.z, av.w}, bx[4] = {bv.x, bv.y, bv.z, bv.w};
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int jj = 0; jj < 4; ++jj) acc[i][jj] = fmaf(ax[i], bx[jj], acc[i][jj]);
      }
    }
  }
  // fixed-order combination of the row groups -> gout[k][c]
  if (active)
#pragma unroll
    for (int e = 0; e < 16; ++e) redb[((int64_t)g * nblk + blk) * 16 + e] = acc[e >> 2][e & 3];
  __syncthreads();
  for (int i = tid; i < nblk * 16; i += kThreads) {
    const int b = i >> 4, e = i & 15;
    float s = 0.f;
    for (int gg = 0; gg < RG; ++gg) s += redb[((int64_t)gg * nblk + b) * 16 + e];
    gout[((b / ncb) * 4 + (e >> 2)) * nbp + (b % ncb) * 4 + (e & 3)] = s;
  }
  __syncthreads();
  // parameter addresses of the slice and the fused Adam update
  int64_t base, ldp, bias;
  switch (jb.kind) {
    case FJ_LSTM: base = dm.wx[jb.l][jb.dir]; ldp = kFG; bias = dm.bb[jb.l][jb.dir]; break;
    case FJ_WQ: base = dm.Wq; ldp = kFD; bias = dm.bq; break;
    case FJ_WK: base = dm.Wk; ldp = kFD; bias = -1; break;
    case FJ_WV: base = dm.Wv; ldp = kFD; bias = -1; break;
    case FJ_WO: base = dm.Wo; ldp = kFD; bias = dm.bo; break;
    case FJ_W1: base = dm.W1; ldp = kHeadHidden; bias = dm.b1; break;
    default: base = dm.W2; ldp = 1; bias = dm.b2; break;
  }
  const int ka_w = has_bias ? ka - 1 : ka;
  const double c1 = a.mode == TT_MODE_TRAIN ? a.corr[2 * step] : 1.0;
  const double c2 = a.mode == TT_MODE_TRAIN ? a.corr[2 * step + 1] : 1.0;
  for (int i = tid; i < ka * jb.nb; i += kThreads) {
    const int k = i / jb.nb, c = i % jb.nb;
    const int64_t p = k < ka_w ? base + (int64_t)k * ldp + jb.c0 + c : bias + jb.c0 + c;
    const float gv = gout[k * nbp + c];
    if (a.mode == TT_MODE_GRAD) {
      a.grad_out[p] = gv;
    } else if (!a.trainable || a.trainable[p]) {
      float pp = __ldcg(a.prm + p), mm = a.m[p], vv = a.v[p];
      adam_update<float>(pp, gv, mm, vv, a.hyp, c1, c2);
      a.prm[p] = pp;
      a.m[p] = mm;
      a.v[p] = vv;
    }
  }
}

// ------------------------------------------------------------ kernel --
__global__ void __launch_bounds__(kThreads, 1) tuner_train_fast_kernel(FastArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float* sm = reinterpret_cast<float*>(smem_raw);
  __shared__ int64_t s_meta[3];
  __shared__ int s_stop;
  const TDims& dm = a.dm;
  const int tid = threadIdx.x;
  const int G = gridDim.x, r = blockIdx.x;
  const bool sampler = r < a.B;
  const int first_job = (r - a.B + G) % G;
  int my_jobs = 0;
  for (int j = first_job; j < a.n_jobs; j += G) ++my_jobs;
  float* lb = sm + a.sl.lb;
  for (int step = 0; step < a.n_steps; ++step) {
    const int64_t b0 = (int64_t)step * a.B;
    const int bn = (int)(a.n_order - b0 < (int64_t)a.B ? a.n_order - b0 : (int64_t)a.B);
    const unsigned cum = (unsigned)(b0 + bn);
    if (sampler && r < bn) {
      phase_mark(step, 0);
      if (step > 0) wait_counter(a.ctr + 2, (unsigned)(step * a.n_jobs), false);
      phase_mark(step, 1);
      if (r == 0) phase_mark_any(step, 31);
      if (tid == 0) {
        const int64_t idx = a.order[b0 + r];
        const int64_t r0 = a.rowoff[idx];
        s_meta[0] = idx;
        s_meta[1] = r0;
        s_meta[2] = a.rowoff[idx + 1] - r0;
        a.meta[2 * r] = r0;
        a.meta[2 * r + 1] = s_meta[2];
      }
      for (int i = tid; i < bn; i += kThreads) lb[i] = a.y[a.order[b0 + i]];
      __syncthreads();
      const int64_t idx = s_meta[0], r0 = s_meta[1];
      const int T = (int)s_meta[2];
      float* xs = a.xch + (int64_t)r * a.xl.total;
      const float yh = fast_sample_fwd(a, sm, xs, r0, T, idx, step);
      phase_mark(step, 5);
      if (tid == 0) a.yhat_buf[r] = yh;
      signal_counter(a.ctr + 0, 1);
      wait_counter(a.ctr + 0, cum, false);
      phase_mark(step, 6);
      for (int i = tid; i < bn; i += kThreads) lb[bn + i] = __ldcg(a.yhat_buf + i);
      __syncthreads();
      const float loss = a.loss_kind == TT_LOSS_RANK
                             ? rank_loss_block<float>(lb, lb + bn, bn, lb + 2 * bn, sm + a.sl.red)
                             : mse_block<float>(lb, lb + bn, bn, lb + 2 * bn, sm + a.sl.red);
      if (tid == 0) {
        s_stop = !isfinite(loss);
        if (r == 0) {
          a.step_loss[step] = loss;
          if (s_stop) a.status[0] = step;
        }
      }
      __syncthreads();
      phase_mark(step, 7);
      if (!s_stop) fast_sample_bwd(a, sm, xs, T, lb[2 * bn + r], yh, step);
      phase_mark(step, 16);
      if (r == 0) phase_mark_any(step, 30);
      signal_counter(a.ctr + 1, 1);
      if (s_stop) break;
    }
    if (my_jobs == 0) {
      if (!sampler) break;  // idle CTA
      continue;
    }
    wait_counter(a.ctr + 1, cum, !sampler);
    if (r == a.B % G) phase_mark_any(step, 20);
    if (tid == 0) s_stop = __ldcg(a.status) >= 0;
    __syncthreads();
    if (s_stop) break;
    for (int j = first_job; j < a.n_jobs; j += G) fast_run_job(a, fast_job(dm, j), bn, step, sm);
    signal_counter(a.ctr + 2, (unsigned)my_jobs);
    if (r == a.B % G) phase_mark_any(step, 21);
  }
}

// --------------------------------------------------------- host side --
struct FastPlan {
  FastSmem sl;
  FastXch xl;
  size_t smem;
  int64_t rch;
  int n_jobs;
};

inline size_t fast_ws_bytes(const TDims& dm, int B) {
  const FastXch xl = make_fast_xch(dm);
  return align_up((size_t)B * xl.total * sizeof(float), 256) + align_up((size_t)B * 2 * 8, 256) +
         align_up((size_t)B * sizeof(float), 256) + 256;
}

// Eligible: fp32, hidden 32, one sample per CTA, every per-sample cache in
// shared memory.  Returns false (generic kernel) otherwise.
inline bool fast_plan(const TDims& dm, int B, int grid, FastPlan& p) {
  if (dm.H != kFH || B > grid || B < 1 || dm.Tmax > 32 || dm.heads < 1) return false;
  int dev = 0, optin = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return false;
  if (cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess)
    return false;
  p.sl = make_fast_smem(dm, B);
  p.xl = make_fast_xch(dm);
  p.n_jobs = fast_n_jobs(dm);
  const size_t static_smem = 64;
  const size_t budget = (size_t)optin - static_smem - 1024;
  size_t need = (size_t)p.sl.total * sizeof(float);
  if (need > budget) return false;
  // job staging: at least Tmax rows of the widest job
  const int kap_max = round4(std::max(dm.d0, kFD) + kFH + 1 > kFD + dm.C + 1
                                 ? std::max(dm.d0, kFD) + kFH + 1
                                 : kFD + dm.C + 1);
  const int nbp = 16;
  const int64_t job_fixed = fast_job_smem(kap_max, nbp, 0);
  const size_t avail = std::max(need, (size_t)budget);
  p.rch = (int64_t)((avail / sizeof(float) - job_fixed) / (kap_max + nbp));
  if (p.rch < dm.Tmax) return false;
  if ((kap_max / 4) * (nbp / 4) > kThreads) return false;  // one 4x4 block per thread at most
  const int64_t all_rows = (int64_t)B * dm.Tmax;
  if (p.rch > all_rows) p.rch = all_rows;
  need = std::max(need, (size_t)(job_fixed + p.rch * (kap_max + nbp)) * sizeof(float));
  p.smem = need;
  return true;
}

inline int fast_launch(FastArgs a, const FastPlan& p, void* ws, cudaStream_t st) {
  char* w = static_cast<char*>(ws);
  a.sl = p.sl;
  a.xl = p.xl;
  a.n_jobs = p.n_jobs;
  a.rch = p.rch;
  a.xch = reinterpret_cast<float*>(w);
  w += align_up((size_t)a.B * p.xl.total * sizeof(float), 256);
  a.meta = reinterpret_cast<int64_t*>(w);
  w += align_up((size_t)a.B * 2 * 8, 256);
  a.yhat_buf = reinterpret_cast<float*>(w);
  w += align_up((size_t)a.B * sizeof(float), 256);
  a.ctr = reinterpret_cast<unsigned int*>(w);
  TT_CUDA(cudaMemsetAsync(a.ctr, 0, 256, st));
  auto kern = tuner_train_fast_kernel;
  TT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem));
  int per_sm = 0;
  TT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads, p.smem));
  TT_REQUIRE(per_sm >= 1, "tuner train (fast): kernel cannot be resident (smem %zu)", p.smem);
  const int grid = sm_count();
  void* args[] = {&a};
  TT_CUDA(cudaLaunchCooperativeKernel((void*)kern, grid, kThreads, args, p.smem, st));
  return check_launch("tuner train (fast)");
}

}  // namespace tt
