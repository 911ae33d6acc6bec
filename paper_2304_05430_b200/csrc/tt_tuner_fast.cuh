// Attention tuner training, latency path: hidden 32, fp32, every per-sample
// cache in shared memory (longest program <= ~14 steps at the default widths).
//
// Reference: estimators/tuner.py _train/_forward/_backward (:227-466),
// _LstmDirection (:55-151), ranking_grad (mlp.py:25-35), Adam (optim.py).
//
// One persistent cooperative launch runs a whole epoch.  Two CTA roles:
//
//  * sample CTAs: CTA k owns minibatch slot k (B <= #SMs; larger minibatches
//    run several rounds per CTA, the forward caches of all but the last slot
//    parked in L2 by bulk copies).  A slot's forward (3 x biLSTM with a warp
//    PAIR per direction, attention passes, head), the score exchange through
//    L2, the minibatch loss (identical arithmetic in every sample CTA), then
//    the ACTIVATION backward only.  Every operand a weight gradient needs
//    (layer inputs, h_prev, dZ, dK, dV, attention pass vectors, head vectors)
//    is published to the L2 exchange, stacked by minibatch row.
//  * gradient jobs (all CTAs, non-sample CTAs first): the parameter vector is
//    cut into column slices of every weight matrix; a job reduces
//    dW[:, slice] = sum_rows A^T B over the minibatch rows in a fixed order
//    (deterministic, no atomics on data) and applies the fused Adam update
//    (or writes the gradient in TT_MODE_GRAD).  Data parallel (world > 1):
//    the reduced slice is first exchanged with the peer ranks through their
//    exchange buffers (fast_dp_exchange) and averaged in rank order.
//
// Phases are ordered by monotone L2 counters instead of grid barriers:
// forward-done (score exchange), backward-done per parameter group (jobs may
// start) and Adam-done per group (the next minibatch may read those
// parameters, layer by layer).  Heads-only mode (s_frozen): the recurrent
// stack is frozen, its last-layer outputs come from a cache, the steps run
// attention + head only.  The weight gradient never materialises per sample:
// the traffic per step is the exchange rows (~45 KB/sample at T = 10)
// instead of B partial 330 KB gradient vectors.
#pragma once

#include "tt_sm100.cuh"
#include "tt_tuner_train.cuh"

// 1: every LSTM layer >= 1 reads its weight block from shared memory and the
// attention/head block lands during the last layer's recurrence (A/B on the
// box: 55.05 -> 54.6 us per step, tools/ab_train.sh); 0: the round-1 layout
// (the last layer reads L2 directly, the attention block lands a layer earlier)
#ifndef TT_ATTN_LAST
#define TT_ATTN_LAST 1
#endif

namespace tt {

constexpr int kFH = 32, kFD = 64, kFG = 128;  // hidden, 2H, 4H
constexpr int kLdA = 68;  // staged attention weights row stride (16-B rows, see frow_mv)
constexpr int kMaxFastB = 160;   // minibatch limit of the latency path (one slot per CTA)
constexpr int kMaxRoundB = 2048; // minibatch limit of the multi-round mode
constexpr int kLdK = 65;        // K/V row stride in smem (odd: lanes over steps hit distinct banks)

__host__ __device__ inline int round4(int x) { return (x + 3) & ~3; }

// ------------------------------------------------------------ layouts --
struct FastSmem {  // float offsets in dynamic shared memory (sample role)
  int64_t x0, lbn, ctxs, S, gc, cs, xz, hb, gex, K, V, alpha, pin, q, mix, pool, zb, a1, red, lb, dS, dS2, dZ, dK,
      dV, dlg, dmix, dq, dpool, da1, ts, rsb, W, total;
};

struct FastXch {  // float offsets in the (stacked) exchange region
  int64_t Rmax;
  int w0, zw;
  int64_t x0, H, cst, S, dZ, dK, dV, pin, mix, dpool, dq, z, a1, da1, dl, total;
};

// attention + head weight image at the start of W (row stride kLdA):
// [Wq|Wk|Wv|Wo|bq|bo] then [W1|b1|W2|b2]
__host__ __device__ inline int64_t fast_attn_floats(const TDims& d) {
  return (int64_t)(4 * kFD + 2) * kLdA + (int64_t)(kFD + d.C + 3) * kLdA;
}

inline FastSmem make_fast_smem(const TDims& d, int B) {
  FastSmem s{};
  int64_t o = 0;
  auto seg = [&](int64_t n) {
    const int64_t at = o;
    o += pad4(n);
    return at;
  };
  const int TM = d.Tmax;
  s.x0 = seg((int64_t)TM * round4(d.d0));
  s.ctxs = seg(d.C);
  s.S = seg((int64_t)d.L * TM * kFD);
  s.gc = seg((int64_t)d.L * 2 * TM * kFG);
  s.cs = seg((int64_t)d.L * 2 * TM * kFH);
  s.xz = seg((int64_t)2 * TM * kFG);  // also the dX partials [4][TM][64]
  s.hb = seg(2 * 2 * 2 * kFH);   // [dir][warp copy][parity][32] hidden state
  s.gex = seg(2 * 2 * 2 * 2 * kFH);  // [dir][warp][parity][64] gate / dh exchange
  s.K = seg((int64_t)TM * kLdK);
  s.V = seg((int64_t)TM * kLdK);
  s.alpha = seg((int64_t)d.U * d.heads * TM);
  s.pin = seg((int64_t)d.U * kFD);
  s.q = seg((int64_t)d.U * kFD);
  s.mix = seg((int64_t)d.U * kFD);
  s.pool = seg(kFD);
  s.zb = seg(kFD + d.C);
  s.a1 = seg(kHeadHidden);
  s.red = seg(std::max(2 * kThreads, 2 * B));
  s.lb = seg((int64_t)3 * B);
  s.lbn = seg(B);
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
  s.ts = seg(B);   // int: step count of every minibatch slot
  s.rsb = seg(B);  // int: first stacked exchange row of every slot
  // attention + head weights, row stride 68: [Wq|Wk|Wv|Wo|bq|bo] then [W1|b1|W2]
  // attention/head weights (row stride 68, + b2 row) or one LSTM layer's two
  // direction blocks [Wx | Wh | b] (128 columns)
  s.W = seg(std::max<int64_t>(fast_attn_floats(d), (int64_t)2 * (kFD + kFH + 1) * kFG));
  s.total = o;
  return s;
}

// The exchange is STACKED by minibatch row: sample k's step rows occupy rows
// [rs_k, rs_k + T_k) of every per-step matrix (rs_k = sum of the earlier
// samples' step counts), its per-sample vectors row k (or k*U + u).  A
// gradient job then stages each operand with one flat copy loop.
inline FastXch make_fast_xch(const TDims& d, int B) {
  FastXch x{};
  int64_t o = 0;
  auto seg = [&](int64_t n) {
    const int64_t at = o;
    o += pad4(n);
    return at;
  };
  x.Rmax = (int64_t)B * d.Tmax;
  x.w0 = round4(d.d0);
  x.zw = round4(kFD + d.C);
  const int64_t R = x.Rmax;
  x.x0 = seg(R * x.w0);                       // raw step rows, zero padded
  x.S = seg((int64_t)d.L * R * kFD);          // layer outputs
  x.H = seg((int64_t)d.L * 2 * R * kFH);      // h_prev per direction (0 at its first step)
  x.dZ = seg((int64_t)d.L * 2 * R * kFG);     // gate pre-activation gradients
  x.dK = seg(R * kFD);
  x.dV = seg(R * kFD);
  x.pin = seg((int64_t)B * d.U * kFD);
  x.mix = seg((int64_t)B * d.U * kFD);
  x.dpool = seg((int64_t)B * d.U * kFD);
  x.dq = seg((int64_t)B * d.U * kFD);
  x.z = seg((int64_t)B * x.zw);               // [pooled | ctx], zero padded
  x.a1 = seg((int64_t)B * kHeadHidden);
  x.da1 = seg((int64_t)B * kHeadHidden);
  x.dl = seg((int64_t)B * 4);                 // [dl, 0, 0, 0]
  x.cst = seg(8);                             // [0 0 0 0 | 1 0 0 0]
  x.total = o;
  return x;
}

// ------------------------------------------------------ gradient jobs --
enum FastJobKind { FJ_LSTM = 0, FJ_WQ, FJ_WK, FJ_WV, FJ_WO, FJ_W1, FJ_W2 };
// Column-slice widths.  Layer 0's gradient jobs sit on the critical path
// into the next minibatch (its forward needs them first), so they are cut
// finest; the upper layers' jobs overlap that forward and are cut coarser
// (same total job count, fewer CTAs per non-critical group).
constexpr int kCwLstm0 = 4, kCwLstm = 16, kCwAttn = 16, kCwHead = 16;

__host__ __device__ inline int lstm_cw(int l, int L) {
  (void)L;
  return l == 0 ? kCwLstm0 : kCwLstm;
}
__host__ __device__ inline int lstm_jobs(int l, int L) { return 2 * (kFG / lstm_cw(l, L)); }
__host__ __device__ inline int attn_jobs() { return 4 * (kFD / kCwAttn) + kHeadHidden / kCwHead + 1; }

struct FastJob {
  int kind, l, dir, c0, nb;  // nb = slice width (columns)
};

__host__ __device__ inline int fast_n_jobs(const TDims& d) {
  int n = attn_jobs();
  for (int l = 0; l < d.L; ++l) n += lstm_jobs(l, d.L);
  return n;
}

__host__ __device__ inline FastJob fast_job(const TDims& d, int j) {
  for (int l = 0; l < d.L; ++l) {
    const int nl = lstm_jobs(l, d.L);
    if (j < nl) {
      const int cw = lstm_cw(l, d.L), per = kFG / cw;
      return FastJob{FJ_LSTM, l, j / per, (j % per) * cw, cw};
    }
    j -= nl;
  }
  const int pa = kFD / kCwAttn;
  if (j < 4 * pa) return FastJob{FJ_WQ + j / pa, 0, 0, (j % pa) * kCwAttn, kCwAttn};
  j -= 4 * pa;
  if (j < kHeadHidden / kCwHead) return FastJob{FJ_W1, 0, 0, j * kCwHead, kCwHead};
  return FastJob{FJ_W2, 0, 0, 0, 1};
}

// A-operand geometry of a job: segment 1 (n1 real columns padded to w1),
// optional segment 2 (n2 columns: the LSTM h_prev rows), then the ones column
// when the slice has a bias.  A column k maps to parameter row
//   k < n1 -> k ;  w1 <= k < w1 + n2 -> n1 + k - w1 ;  k == w1 + n2 -> bias
// (the LSTM block [Wx; Wh; b] is contiguous in the parameter layout).
struct JobGeo {
  int n1, w1, n2, ka, kap, nbp, maxr;
  bool bias;
  int64_t base, ldp, bptr;
};

__device__ inline JobGeo job_geo(const TDims& d, const FastJob& jb) {
  JobGeo g{};
  g.n2 = 0;
  g.bias = true;
  g.ldp = kFD;
  g.maxr = 1;
  switch (jb.kind) {
    case FJ_LSTM:
      g.n1 = jb.l == 0 ? d.d0 : kFD;
      g.n2 = kFH;
      g.base = d.wx[jb.l][jb.dir];
      g.ldp = kFG;
      g.bptr = d.bb[jb.l][jb.dir];
      g.maxr = d.Tmax;
      break;
    case FJ_WQ: g.n1 = kFD; g.base = d.Wq; g.bptr = d.bq; g.maxr = d.U; break;
    case FJ_WO: g.n1 = kFD; g.base = d.Wo; g.bptr = d.bo; g.maxr = d.U; break;
    case FJ_WK: g.n1 = kFD; g.base = d.Wk; g.bias = false; g.bptr = -1; g.maxr = d.Tmax; break;
    case FJ_WV: g.n1 = kFD; g.base = d.Wv; g.bias = false; g.bptr = -1; g.maxr = d.Tmax; break;
    case FJ_W1: g.n1 = kFD + d.C; g.base = d.W1; g.ldp = kHeadHidden; g.bptr = d.b1; break;
    default: g.n1 = kHeadHidden; g.base = d.W2; g.ldp = 1; g.bptr = d.b2; break;
  }
  g.w1 = round4(g.n1);
  g.ka = g.w1 + g.n2 + (g.bias ? 1 : 0);
  g.kap = round4(g.ka);
  g.nbp = round4(jb.nb);
  return g;
}

// smem floats a job needs for `rows` staged rows (plus the reduction area)
// (the last term: the persistent parameter/moment cache of a job CTA)
__host__ __device__ inline int64_t fast_job_smem(int kap, int nbp, int rows) {
  return (int64_t)rows * (kap + nbp) + (int64_t)kThreads * 16 + (int64_t)kap * nbp + 64 +
         (int64_t)4 * kap * nbp;
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
  float* xch;          // stacked exchange (FastXch)
  int64_t* meta;       // [B]: steps of each minibatch slot
  float* yhat_buf;     // [B]
  float* lossp;        // [B][2]: per-slot pair-loss partials (multi-round mode)
  const float* s_frozen;  // heads-only mode: frozen last-layer LSTM outputs [sum T][64] (else null)
  // data parallel (world > 1): every rank runs this kernel on its own shard;
  // each gradient job exchanges its slice with the peers through their
  // exchange buffers (xb[p], NVLink peer memory) before the Adam update
  int world, rank;
  int64_t gbase;        // global step index of this launch's first minibatch (monotone flags)
  int64_t dp_slice;     // floats per slice slot (>= kap * nbp of every job)
  void* const* xb;      // [world] exchange buffers (fast_dp_buffer_bytes each)
  long long dp_timeout_ns;  // bound on one wait for a peer's slice (status[1] = 1 past it)
  float* scache;       // [B][sl.red - sl.x0]: per-slot forward caches (multi-round mode)
  float* wcache;       // [grid][attn_floats]: attention/head weight image per CTA (multi-round)
  unsigned int* ctr;   // [0] fwd, [1 + g] bwd, [2 + L + g] adam, [kCtrLoss] loss (monotone)
  int n_jobs;
  int64_t rch;         // job staging rows per chunk
  int64_t pc_off;      // smem float offset of a job CTA's parameter cache [4][pc_n]
  int l0_smem;         // layer 0's weight blocks fit in W (bulk-copied at each step start)
  int pc_n;            // floats per cache array (kap_max * 16)
};

// Phase marks (debug, tt_debug_profile_step).  The profiled step is read
// from global memory ONCE per launch into shared memory: a global read per
// mark would cost an L2 round trip after every fence (they invalidate L1).
__shared__ int s_prof;
// Weight-prefetch barrier of a sample CTA (bulk copies into W) and its phase.
__shared__ __align__(8) uint64_t s_wbar;
__shared__ __align__(8) uint64_t s_cbar;  // multi-round cache restores
__shared__ uint32_t s_wph;

// CTA 0, clock64 (cycles)
__device__ __forceinline__ void fmark(int step, int i) {
  if (blockIdx.x == 0 && threadIdx.x == 0 && step == s_prof) g_phase[i] = clock64();
}
// any CTA, %globaltimer (ns: comparable across SMs, unlike clock64)
__device__ __forceinline__ void fmark_any(int step, int i) {
  if (threadIdx.x == 0 && step == s_prof) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_phase[i] = (long long)t;
  }
}

// ------------------------------------------------------------- sync --
// Counter layout (monotone within a launch):
//   ctr[0]             scores published (forward done), += 1 per sample
//   ctr[1 + g]         backward operands of parameter group g published
//   ctr[2 + L + g]     gradient jobs of group g done (parameters updated)
// Groups: g < L = LSTM layer g (both directions), g = L = attention + head.
// A gradient job waits only for its own group and the next minibatch's
// forward waits per layer, so the Adam updates of the upper layers overlap
// the next forward's first layers.
__device__ __forceinline__ int ctr_bwd(int g) { return 1 + g; }
constexpr int kCtrLoss = 63;  // last of the 64 counters (L <= 30)
__device__ __forceinline__ int ctr_adam(const TDims& d, int g) { return 2 + d.L + g; }
__device__ __forceinline__ int job_group(const TDims& d, int j) {
  for (int l = 0; l < d.L; ++l) {
    if (j < lstm_jobs(l, d.L)) return l;
    j -= lstm_jobs(l, d.L);
  }
  return d.L;
}
__device__ __forceinline__ int group_jobs(const TDims& d, int g) {
  return g < d.L ? lstm_jobs(g, d.L) : attn_jobs();
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// All threads; thread 0 spins until *ctr >= target.
__device__ __forceinline__ void wait_counter(const unsigned* ctr, unsigned target, bool sleep) {
  if (threadIdx.x == 0) {
    while (ld_acquire(ctr) < target) {
      if (sleep) __nanosleep(100);
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
#ifdef TT_SYNC_STAGE
  *reinterpret_cast<float4*>(s) = __ldcg(reinterpret_cast<const float4*>(g));
#else
  const unsigned sa = (unsigned)__cvta_generic_to_shared(s);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(g) : "memory");
#endif
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_all;" ::: "memory");
}

// Recurrence activations: the same MUFU ops as Act<float> (ex2.approx +
// rcp.approx) in their .ftz forms, which drop the denormal-range fix-up
// instructions from the per-step critical path (results differ only where
// exp underflows to a denormal).
__device__ __forceinline__ float fx_ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float fx_rcp(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float fsig(float x) { return fx_rcp(1.f + fx_ex2(-1.4426950408889634f * x)); }
__device__ __forceinline__ float ftanh(float x) {
  return 1.f - 2.f * fx_rcp(fx_ex2(2.8853900817779268f * x) + 1.f);
}

// ------------------------------------------------------ recurrences --
// Each direction's recurrence runs on a PAIR of warps (dir d: warps 2d and
// 2d+1, one per SM sub-partition); warp `sub` of the pair owns gate blocks
// {2 sub, 2 sub + 1} ([i|f] or [g|o]), i.e. 64 of the 128 columns, so a
// lane keeps 64 weights in registers.  One named barrier (id 2 + d, 64
// threads) per time step exchanges the gate values (forward) or the dh
// partial sums (backward); buffers alternate by step parity.
using WReg = float[64];

// Lane j of warp `sub`: Wh[k][(2 sub + q)*32 + j] -> w[q*32 + k].
__device__ __forceinline__ void load_wh_cols(WReg& w, const float* __restrict__ Wh, int sub) {
  const int j = threadIdx.x & 31;
#pragma unroll
  for (int k = 0; k < kFH; ++k)
#pragma unroll
    for (int q = 0; q < 2; ++q) w[q * kFH + k] = __ldcg(Wh + k * kFG + (2 * sub + q) * kFH + j);
}

// Lane j of warp `sub`: Wh[j][sub*64 + c] for c < 64 (half of row j).
__device__ __forceinline__ void load_wh_row(WReg& w, const float* __restrict__ Wh, int sub) {
  const int j = threadIdx.x & 31;
  const float4* w4 = reinterpret_cast<const float4*>(Wh + (int64_t)j * kFG + sub * 64);
#pragma unroll
  for (int m = 0; m < 16; ++m) {
    const float4 v = __ldcg(w4 + m);
    w[4 * m + 0] = v.x;
    w[4 * m + 1] = v.y;
    w[4 * m + 2] = v.z;
    w[4 * m + 3] = v.w;
  }
}

// Forward recurrence, warp `sub` of direction `dir`.  xz: [2][TM][128]
// input projections (bias included).  Both warps form c and h identically
// (each keeps its own copy of h for its next matvec); warp 0 of the pair
// writes the layer output row S[t][dir*32 + j] (smem + exchange) and the
// cell state, each warp its two gate blocks.
__device__ __forceinline__ void fast_rec_fwd(const WReg& w, int dir, int sub, int T, int TM,
                                             const float* xz, float* S, float* Sg, float* Hg,
                                             float* gc, float* cs, float* hb, float* gex) {
  const int j = threadIdx.x & 31;
  float c = 0.f;
  float* hm = hb + (dir * 2 + sub) * 2 * kFH;          // [parity][32]
  float* gx_me = gex + (dir * 2 + sub) * 2 * 2 * kFH;  // [parity][64]
  const float* gx_ot = gex + (dir * 2 + (sub ^ 1)) * 2 * 2 * kFH;
  hm[j] = 0.f;
  __syncwarp();
  for (int s = 0; s < T; ++s) {
    const int par = s & 1;
    const int t = dir == 0 ? s : T - 1 - s;
    const float* xr = xz + ((int64_t)dir * TM + t) * kFG + 2 * sub * kFH;
    float a00 = xr[j], a01 = 0.f, a10 = xr[kFH + j], a11 = 0.f;
    const float4* h4 = reinterpret_cast<const float4*>(hm + par * kFH);
#pragma unroll
    for (int m = 0; m < kFH / 4; m += 2) {
      const float4 u = h4[m], v = h4[m + 1];
      a00 = fmaf(u.x, w[4 * m + 0], a00);
      a10 = fmaf(u.x, w[kFH + 4 * m + 0], a10);
      a01 = fmaf(v.x, w[4 * m + 4], a01);
      a11 = fmaf(v.x, w[kFH + 4 * m + 4], a11);
      a00 = fmaf(u.y, w[4 * m + 1], a00);
      a10 = fmaf(u.y, w[kFH + 4 * m + 1], a10);
      a01 = fmaf(v.y, w[4 * m + 5], a01);
      a11 = fmaf(v.y, w[kFH + 4 * m + 5], a11);
      a00 = fmaf(u.z, w[4 * m + 2], a00);
      a10 = fmaf(u.z, w[kFH + 4 * m + 2], a10);
      a01 = fmaf(v.z, w[4 * m + 6], a01);
      a11 = fmaf(v.z, w[kFH + 4 * m + 6], a11);
      a00 = fmaf(u.w, w[4 * m + 3], a00);
      a10 = fmaf(u.w, w[kFH + 4 * m + 3], a10);
      a01 = fmaf(v.w, w[4 * m + 7], a01);
      a11 = fmaf(v.w, w[kFH + 4 * m + 7], a11);
    }
    const float z0 = a00 + a01, z1 = a10 + a11;
    // sub 0: (i, f) = sigmoid; sub 1: g = tanh, o = sigmoid
    const float v0 = sub == 0 ? fsig(z0) : ftanh(z0);
    const float v1 = fsig(z1);
    float* gr = gc + ((int64_t)dir * TM + t) * kFG + 2 * sub * kFH;
    gr[j] = v0;
    gr[kFH + j] = v1;
    gx_me[par * 2 * kFH + j] = v0;
    gx_me[par * 2 * kFH + kFH + j] = v1;
    named_barrier(2 + dir, 64);
    const float o0 = gx_ot[par * 2 * kFH + j], o1 = gx_ot[par * 2 * kFH + kFH + j];
    const float gi = sub == 0 ? v0 : o0, gf = sub == 0 ? v1 : o1;
    const float gg = sub == 0 ? o0 : v0, go = sub == 0 ? o1 : v1;
    c = gf * c + gi * gg;
    const float h = go * ftanh(c);
    hm[(par ^ 1) * kFH + j] = h;
    if (sub == 0) {
      S[(int64_t)t * kFD + dir * kFH + j] = h;
      Sg[(int64_t)t * kFD + dir * kFH + j] = h;
      cs[((int64_t)dir * TM + t) * kFH + j] = c;
    } else {
      // h_prev rows of the stacked exchange, in the direction's order
      if (s == 0) Hg[(int64_t)t * kFH + j] = 0.f;
      if (s + 1 < T) Hg[(int64_t)(dir == 0 ? t + 1 : t - 1) * kFH + j] = h;
    }
    __syncwarp();
  }
}

// BPTT (tuner.py:113-148 restricted to the valid steps), warp `sub` of
// direction `dir`: both warps form the elementwise gate gradients
// identically; warp `sub` publishes dZ for its gate blocks and the partial
// dh_j = sum_{c in its half} Wh[j][c] dz[c]; the two partials are summed in
// fixed order after the step's named barrier.  dS: [TM][64] upstream
// gradient of this layer's output.
__device__ __forceinline__ void fast_rec_bwd(const WReg& wr, int dir, int sub, int T, int TM,
                                             const float* gc, const float* cs, const float* dS,
                                             float* dZ, float* dZg, float* gex) {
  // dZg: this direction's stacked dZ rows of the sample (row t at t*128)
  const int j = threadIdx.x & 31;
  float* px = gex + dir * 2 * 2 * kFH;  // [warp][parity][32]
  float dh = 0.f, dc = 0.f;
  for (int s = 0; s < T; ++s) {
    const int par = s & 1;
    // reverse of the direction's forward order
    const int t = dir == 0 ? T - 1 - s : s;
    const bool has_prev = s < T - 1;
    const int tp = dir == 0 ? t - 1 : t + 1;
    const float* gr = gc + ((int64_t)dir * TM + t) * kFG;
    const float gi = gr[j], gf = gr[kFH + j], gg = gr[2 * kFH + j], go = gr[3 * kFH + j];
    const float cn = cs[((int64_t)dir * TM + t) * kFH + j];
    const float tc = ftanh(cn);
    const float cp = has_prev ? cs[((int64_t)dir * TM + tp) * kFH + j] : 0.f;
    const float dht = dS[(int64_t)t * kFD + dir * kFH + j] + dh;
    const float dO = dht * tc;
    const float dcr = dc + dht * go * (1.f - tc * tc);
    const float d0 = sub == 0 ? dcr * gg * gi * (1.f - gi) : dcr * gi * (1.f - gg * gg);
    const float d1 = sub == 0 ? dcr * cp * gf * (1.f - gf) : dO * go * (1.f - go);
    dc = dcr * gf;
    float* zr = dZ + ((int64_t)dir * TM + t) * kFG + 2 * sub * kFH;
    float* zg = dZg + (int64_t)t * kFG + 2 * sub * kFH;
    zr[j] = d0;
    zr[kFH + j] = d1;
    zg[j] = d0;
    zg[kFH + j] = d1;
    if (has_prev) {
      __syncwarp();
      const float4* z4 = reinterpret_cast<const float4*>(zr);
      float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
#pragma unroll
      for (int m = 0; m < 16; ++m) {
        const float4 zv = z4[m];
        a0 = fmaf(zv.x, wr[4 * m + 0], a0);
        a1 = fmaf(zv.y, wr[4 * m + 1], a1);
        a2 = fmaf(zv.z, wr[4 * m + 2], a2);
        a3 = fmaf(zv.w, wr[4 * m + 3], a3);
      }
      px[(sub * 2 + par) * kFH + j] = (a0 + a1) + (a2 + a3);
      named_barrier(2 + dir, 64);
      dh = px[(0 * 2 + par) * kFH + j] + px[(1 * 2 + par) * kFH + j];
    }
  }
}

// dot(x[0:64], w[OFF:OFF+64]) with x a 16-B aligned smem row
template <int OFF>
__device__ __forceinline__ float dot64(const float* __restrict__ x, const float (&w)[64 + OFF]) {
  const float4* x4 = reinterpret_cast<const float4*>(x);
  float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    const float4 v = x4[k];
    a0 = fmaf(v.x, w[OFF + 4 * k + 0], a0);
    a1 = fmaf(v.y, w[OFF + 4 * k + 1], a1);
    a2 = fmaf(v.z, w[OFF + 4 * k + 2], a2);
    a3 = fmaf(v.w, w[OFF + 4 * k + 3], a3);
  }
  return (a0 + a1) + (a2 + a3);
}

// out[k] = sum_{c < 64} W[k*kLdA + c] v[c] for k < 64 (v @ W^T), all threads:
// thread (k, part) reads its 16-column row segment as float4 (conflict-free
// at the 16-B row stride), partials combined in fixed order.  Ends synced.
__device__ __forceinline__ void frow_mv(const float* W, const float* v, float* out, float* red) {
  const int k = threadIdx.x & 63, part = threadIdx.x >> 6;
  const float4* w4 = reinterpret_cast<const float4*>(W + k * kLdA + part * 16);
  const float4* v4 = reinterpret_cast<const float4*>(v + part * 16);
  float acc = 0.f;
#pragma unroll
  for (int m = 0; m < 4; ++m) {
    const float4 w = w4[m], x = v4[m];
    acc = fmaf(w.x, x.x, acc);
    acc = fmaf(w.y, x.y, acc);
    acc = fmaf(w.z, x.z, acc);
    acc = fmaf(w.w, x.w, acc);
  }
  red[threadIdx.x] = acc;
  __syncthreads();
  if (threadIdx.x < 64) out[threadIdx.x] = (red[k] + red[64 + k]) + (red[128 + k] + red[192 + k]);
  __syncthreads();
}

// out[c] = bias[c] + sum_{k < K} v[k] W[k*kLdA + c] for c < 64, all threads:
// thread (c, part) sums rows k in [part*KQ, part*KQ + KQ) with four
// independent accumulators (latency-bound otherwise); the four partials are
// combined in fixed order.  Ends synced.
__device__ __forceinline__ void fcol_mv(const float* v, const float* W, int K, const float* bias,
                                        float* out, float* red) {
  const int c = threadIdx.x & 63, part = threadIdx.x >> 6;
  const int KQ = (K + 3) >> 2;
  const int k0 = part * KQ, k1 = min(K, k0 + KQ);
  const float* w = W + c;
  float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
  int k = k0;
  for (; k + 4 <= k1; k += 4) {
    a0 = fmaf(v[k], w[k * kLdA], a0);
    a1 = fmaf(v[k + 1], w[(k + 1) * kLdA], a1);
    a2 = fmaf(v[k + 2], w[(k + 2) * kLdA], a2);
    a3 = fmaf(v[k + 3], w[(k + 3) * kLdA], a3);
  }
  for (; k < k1; ++k) a0 = fmaf(v[k], w[k * kLdA], a0);
  red[threadIdx.x] = (a0 + a1) + (a2 + a3);
  __syncthreads();
  if (threadIdx.x < 64)
    out[c] = bias[c] + ((red[c] + red[64 + c]) + (red[128 + c] + red[192 + c]));
  __syncthreads();
}

// dot(a[0:n], b[0:n]) of two smem rows, four accumulators (n % 4 == 0)
__device__ __forceinline__ float fdot4(const float* a, const float* b, int n) {
  float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
  for (int d = 0; d < n; d += 4) {
    a0 = fmaf(a[d], b[d], a0);
    a1 = fmaf(a[d + 1], b[d + 1], a1);
    a2 = fmaf(a[d + 2], b[d + 2], a2);
    a3 = fmaf(a[d + 3], b[d + 3], a3);
  }
  return (a0 + a1) + (a2 + a3);
}

// out[c] = scale * sum_{t < T} w[h(c)][t] M[t*kLdK + c] for c < 64 (h(c) = c / dh,
// w rows of stride TM), all threads: thread (c, part) sums t = part, part+4,
// ...; partials combined in fixed order.  Optional copy to `out2`.  Ends synced.
__device__ __forceinline__ void fmix(const float* w, int TM, int dh, const float* M, int T,
                                     float scale, float* out, float* out2, float* red) {
  const int c = threadIdx.x & 63, part = threadIdx.x >> 6;
  const float* wr = w + (c / dh) * TM;
  float a0 = 0.f, a1 = 0.f;
  int t = part;
  for (; t + 4 < T; t += 8) {
    a0 = fmaf(wr[t], M[t * kLdK + c], a0);
    a1 = fmaf(wr[t + 4], M[(t + 4) * kLdK + c], a1);
  }
  if (t < T) a0 = fmaf(wr[t], M[t * kLdK + c], a0);
  red[threadIdx.x] = a0 + a1;
  __syncthreads();
  if (threadIdx.x < 64) {
    const float r = ((red[c] + red[64 + c]) + (red[128 + c] + red[192 + c])) * scale;
    out[c] = r;
    if (out2) out2[c] = r;
  }
  __syncthreads();
}

// ------------------------------------------------- sample forward --
// All 256 threads.  Returns yhat (valid in every thread after the call).
// rs: this sample's first row in the stacked exchange; slot: its minibatch slot.
__device__ float fast_sample_fwd(const FastArgs& a, float* sm, int64_t rs, int slot, int64_t r0,
                                 int T, int64_t idx, int step) {
  const TDims& dm = a.dm;
  const FastSmem& L = a.sl;
  const FastXch& X = a.xl;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int TM = dm.Tmax;
  float* S = sm + L.S;
  float* xz = sm + L.xz;
  float* W = sm + L.W;
  float* W1s = W + (4 * kFD + 2) * kLdA;
  // Weights of layer l >= 1 (per direction the contiguous parameter block
  // [Wx (64 rows) | Wh (32 rows) | b] of 128 columns) and finally the
  // attention/head block are copied into W by warps 4..7 with async 16-B
  // copies DURING the previous layer's recurrence, after that group's Adam
  // update of the previous minibatch is complete; layer 0 reads L2 directly
  // (its update was awaited at the step start).
  constexpr int kBlk = (kFD + kFH + 1) * kFG;  // floats per direction block
  // Layers 1..L-2 read their block from W; layer 0 and the last layer read
  // L2 directly, so the attention block can be prefetched during layer L-2
  // (two recurrences to land).
#if TT_ATTN_LAST
  // every layer >= 1 reads its block from W (bulk-copied during the previous
  // layer's recurrence); the attention/head block lands during the LAST
  // layer's recurrence
  const int att_l = dm.L - 1;
#else
  const int att_l = dm.L >= 2 ? dm.L - 2 : 0;  // layer during which attention is prefetched
#endif
  const int blk0 = (dm.d0 + kFH + 1) * kFG;     // layer-0 direction block (a.l0_smem)
  if (a.l0_smem && !a.s_frozen) {
    const uint32_t wph = s_wph;
    sm100::mbar_wait(&s_wbar, wph);
    __syncthreads();
    if (tid == 0) s_wph = wph ^ 1u;
  }
  // attention/head weights into 16-B rows of stride 68 (threads t0, t0 + stride, ..)
  auto copy_attn = [&](int t0, int stride) {
    const int rows1 = 4 * kFD + 2, rows2 = kFD + dm.C + 2;
    const float* src1 = a.prm + dm.Wq;
    const float* src2 = a.prm + dm.W1;
    const int tot = (rows1 + rows2) * 16 + 1;  // + the chunk holding b2
    for (int e = t0; e < tot; e += stride) {
      const int row = e >> 4, q = e & 15;
      if (row < rows1)
        cp_async16(W + row * kLdA + q * 4, src1 + e * 4);
      else if (e + 1 < tot)
        cp_async16(W1s + (row - rows1) * kLdA + q * 4, src2 + (e - rows1 * 16) * 4);
      else  // b2 is the last parameter: a 4-byte copy stays inside the buffer
        cp_async4(W1s + (int64_t)rows2 * kLdA, src2 + (int64_t)rows2 * 64);
    }
  };
  if (a.s_frozen) {
    // heads-only mode: the recurrent stack is frozen; its last-layer rows come
    // from the cache (to smem for the attention and to the exchange for the
    // Wk / Wv jobs) once the attention group's previous update is done
    if (step > 0) {
      if (tid == 0) {
        const unsigned target = (unsigned)(step * group_jobs(dm, dm.L));
        while (ld_acquire(a.ctr + ctr_adam(dm, dm.L)) < target) {
        }
      }
      __syncthreads();
    }
    copy_attn(tid, kThreads);
    float* Sl = S + (int64_t)(dm.L - 1) * TM * kFD;
    for (int i = tid; i < T * kFD / 4; i += kThreads) cp_async16(Sl + i * 4, a.s_frozen + r0 * kFD + i * 4);
    cp_async_wait_all();
    __syncthreads();
    float* xs = a.xch + X.S + ((int64_t)(dm.L - 1) * X.Rmax + rs) * kFD;
    for (int i = tid; i < T * kFD; i += kThreads) xs[i] = Sl[i];
  }
  for (int l = a.s_frozen ? dm.L : 0; l < dm.L; ++l) {
#if TT_ATTN_LAST
    const bool direct = l == 0;
#else
    const bool direct = l == 0 || l == dm.L - 1;  // (the last layer's update was
                                                  //  awaited during layer att_l)
#endif
    {
      // ---- input projection xz[dir][t][c] = b[c] + x_t Wx[:, c], thread = column
      const int dir = tid >> 7, c = tid & 127;
      float* xzr = xz + (int64_t)dir * TM * kFG + c;
      if (l == 0) {
        const float* Wx = a.l0_smem ? W + dir * blk0 + c : a.prm + dm.wx[0][dir] + c;
        const float bc = a.l0_smem ? Wx[(dm.d0 + kFH) * kFG] : __ldcg(a.prm + dm.bb[0][dir] + c);
        (void)direct;
        // raw rows staged in smem at the step start (zero padded to w0)
        const int w0 = round4(dm.d0);
        const float* x0 = sm + L.x0;
        for (int k0 = 0; k0 < w0; k0 += 8) {
          float wk[8];
#pragma unroll
          for (int kk = 0; kk < 8; ++kk)
            wk[kk] = k0 + kk < dm.d0 ? (a.l0_smem ? Wx[(k0 + kk) * kFG] : __ldcg(Wx + (int64_t)(k0 + kk) * kFG))
                                     : 0.f;
          for (int t = 0; t < T; ++t) {
            float acc = k0 == 0 ? bc : xzr[(int64_t)t * kFG];
#pragma unroll
            for (int kk = 0; kk < 8; ++kk)
              if (k0 + kk < w0) acc = fmaf(x0[t * w0 + k0 + kk], wk[kk], acc);
            xzr[(int64_t)t * kFG] = acc;
          }
        }
      } else {
        // prefetched block of this direction, or L2 for the last layer
        const float* Wb = direct ? a.prm + dm.wx[l][dir] + c : W + dir * kBlk + c;
        float wx[kFD];
        float bc;
        if (direct) {
#pragma unroll
          for (int k = 0; k < kFD; ++k) wx[k] = __ldcg(Wb + k * kFG);
          bc = __ldcg(Wb + (kFD + kFH) * kFG);
        } else {
#pragma unroll
          for (int k = 0; k < kFD; ++k) wx[k] = Wb[k * kFG];
          bc = Wb[(kFD + kFH) * kFG];
        }
        const float* xin = S + (int64_t)(l - 1) * TM * kFD;
        for (int t = 0; t < T; ++t) xzr[(int64_t)t * kFG] = dot64<0>(xin + (int64_t)t * kFD, wx) + bc;
      }
    }
    if (warp < 4) {
      WReg wh;
      const int dir = warp >> 1, sub = warp & 1;
      if (l == 0 && a.l0_smem) {
        const float* Wh = W + dir * blk0 + dm.d0 * kFG + lane;
#pragma unroll
        for (int k = 0; k < kFH; ++k)
#pragma unroll
          for (int q = 0; q < 2; ++q) wh[q * kFH + k] = Wh[k * kFG + (2 * sub + q) * kFH];
      } else if (direct) {
        load_wh_cols(wh, a.prm + dm.wh[l][dir], sub);
      } else {
        const float* Wh = W + dir * kBlk + kFD * kFG + lane;
#pragma unroll
        for (int k = 0; k < kFH; ++k)
#pragma unroll
          for (int q = 0; q < 2; ++q) wh[q * kFH + k] = Wh[k * kFG + (2 * sub + q) * kFH];
      }
      named_barrier(1, kThreads);  // projection done, W free
      if (warp == 0) fmark(step, 25 + l);
      fast_rec_fwd(wh, dir, sub, T, TM, xz, S + (int64_t)l * TM * kFD,
                   a.xch + X.S + ((int64_t)l * X.Rmax + rs) * kFD,
                   a.xch + X.H + (((int64_t)l * 2 + dir) * X.Rmax + rs) * kFH,
                   sm + L.gc + (int64_t)l * 2 * TM * kFG, sm + L.cs + (int64_t)l * 2 * TM * kFH,
                   sm + L.hb, sm + L.gex);
      if (warp == 0) fmark(step, 2 + l);
    } else {
      named_barrier(1, kThreads);
      // what this recurrence overlaps: layer l+1's block (if it reads W) or,
      // during layer att_l, the attention/head block
#if TT_ATTN_LAST
      const bool pf_lstm = l + 1 < dm.L;
#else
      const bool pf_lstm = l + 1 < dm.L - 1;
#endif
      const bool pf_attn = l == att_l;
      if (pf_lstm || pf_attn) {
        const int g = pf_lstm ? l + 1 : dm.L;
        if (step > 0) {  // that group's Adam update (previous minibatch) must be done
          if (tid == 128) {
            const unsigned target = (unsigned)(step * group_jobs(dm, g));
            while (ld_acquire(a.ctr + ctr_adam(dm, g)) < target) {
            }
          }
          named_barrier(5, kThreads - 128);  // ids 2, 3: recurrence warp pairs
        }
        if (pf_lstm) {
          // two contiguous direction blocks: bulk copies on the TMA engine
          if (warp == 4) {
            sm100::fence_proxy_async_smem();  // W's generic reads before the async writes
            if (lane == 0) sm100::mbar_expect_tx(&s_wbar, 2u * kBlk * 4u);
            __syncwarp();
            if (lane < 2) sm100::bulk_g2s(W + lane * kBlk, a.prm + dm.wx[l + 1][lane], kBlk * 4u, &s_wbar);
          }
        } else {
          // attention/head weights (per-thread async copies; they have this
          // and the last layer's recurrence to land)
          copy_attn(tid - 128, kThreads - 128);
          // the last layer reads L2 directly at its start: await its update
          // here, off the critical path
          if (!TT_ATTN_LAST && step > 0 && l + 1 == dm.L - 1) {
            if (tid == 128) {
              const unsigned target = (unsigned)(step * group_jobs(dm, dm.L - 1));
              while (ld_acquire(a.ctr + ctr_adam(dm, dm.L - 1)) < target) {
              }
            }
            named_barrier(5, kThreads - 128);
          }
        }
      }
      if (l == dm.L - 1) cp_async_wait_all();
    }
    __syncthreads();
    if (l + 1 < dm.L - (TT_ATTN_LAST ? 0 : 1)) {
      // the bulk copy issued during this layer's recurrence must have landed
      const uint32_t wph = s_wph;
      sm100::mbar_wait(&s_wbar, wph);
      __syncthreads();
      if (tid == 0) s_wph = wph ^ 1u;
    }
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
  const float b2 = W1s[(int64_t)(Z + 2) * kLdA];  // staged with the head block
  if (tid < kFD) {
    float a0 = 0.f, a1 = 0.f;
    int t = 0;
    for (; t + 1 < T; t += 2) {
      a0 += Sl[(int64_t)t * kFD + tid];
      a1 += Sl[(int64_t)(t + 1) * kFD + tid];
    }
    if (t < T) a0 += Sl[(int64_t)t * kFD + tid];
    pool[tid] = (a0 + a1) / (float)(T > 1 ? T : 1);
  }
  {
    const int cc = tid & 127, grp = tid >> 7, col = cc & 63;
    const float* wp = (cc < kFD ? Wk : Wv) + col;
    float wc[kFD];
#pragma unroll
    for (int k = 0; k < kFD; ++k) wc[k] = wp[k * kLdA];
    float* dst = cc < kFD ? K : V;
    for (int t = grp; t < T; t += 2) dst[(int64_t)t * kLdK + col] = dot_reg<kFD>(Sl + (int64_t)t * kFD, wc);
  }
  __syncthreads();
  fmark(step, 8);
  const float sq = sqrtf((float)dh);
  float* const xpin = a.xch + X.pin + (int64_t)slot * U * kFD;
  float* const xmix = a.xch + X.mix + (int64_t)slot * U * kFD;
  // Passes (tuner.py:259-274), warp-specialised: warp h owns head h end to
  // end -- its 32-column slice of q = pooled Wq + bq, the logits and softmax
  // over the program's steps, and its slice of mix -- with no block barrier;
  // one barrier before pooled = mix Wo + bo (threads 0..63) and one after.
  for (int u = 0; u < U; ++u) {
    float* q = sm + L.q + u * kFD;
    float* mix = sm + L.mix + u * kFD;
    float* al = sm + L.alpha + (int64_t)u * heads * TM;
    if (tid < kFD) {
      sm[L.pin + u * kFD + tid] = pool[tid];
      xpin[u * kFD + tid] = pool[tid];
    }
    for (int h = warp; h < heads; h += kThreads / 32) {
      for (int i = lane; i < dh; i += 32) {  // q_h
        const int c = h * dh + i;
        const float* wc = Wq + c;
        float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
#pragma unroll 4
        for (int k = 0; k < kFD; k += 4) {
          a0 = fmaf(pool[k], wc[k * kLdA], a0);
          a1 = fmaf(pool[k + 1], wc[(k + 1) * kLdA], a1);
          a2 = fmaf(pool[k + 2], wc[(k + 2) * kLdA], a2);
          a3 = fmaf(pool[k + 3], wc[(k + 3) * kLdA], a3);
        }
        q[c] = bq[c] + ((a0 + a1) + (a2 + a3));
      }
      __syncwarp();
      const float* qh = q + h * dh;
      float* ar = al + (int64_t)h * TM;
      float mx = -INFINITY;
      for (int t = lane; t < T; t += 32) {
        const float acc = fdot4(qh, K + (int64_t)t * kLdK + h * dh, dh) / sq;
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
      __syncwarp();
      for (int i = lane; i < dh; i += 32) {  // mix_h
        const int c = h * dh + i;
        float a0 = 0.f, a1 = 0.f;
        int t = 0;
        for (; t + 1 < T; t += 2) {
          a0 = fmaf(ar[t], V[(int64_t)t * kLdK + c], a0);
          a1 = fmaf(ar[t + 1], V[(int64_t)(t + 1) * kLdK + c], a1);
        }
        if (t < T) a0 = fmaf(ar[t], V[(int64_t)t * kLdK + c], a0);
        mix[c] = a0 + a1;
        xmix[u * kFD + c] = a0 + a1;
      }
    }
    __syncthreads();
    if (tid < kFD) {  // pooled = mix Wo + bo
      const float* wc = Wo + tid;
      float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
#pragma unroll 4
      for (int k = 0; k < kFD; k += 4) {
        a0 = fmaf(mix[k], wc[k * kLdA], a0);
        a1 = fmaf(mix[k + 1], wc[(k + 1) * kLdA], a1);
        a2 = fmaf(mix[k + 2], wc[(k + 2) * kLdA], a2);
        a3 = fmaf(mix[k + 3], wc[(k + 3) * kLdA], a3);
      }
      pool[tid] = bo[tid] + ((a0 + a1) + (a2 + a3));
    }
    __syncthreads();
    fmark(step, u == 0 ? 9 : 17);
  }
  float* zb = sm + L.zb;
  for (int i = tid; i < round4(Z); i += kThreads) {
    const float vz = i < kFD ? pool[i] : (i < Z ? sm[L.ctxs + (i - kFD)] : 0.f);
    if (i < Z) zb[i] = vz;
    a.xch[X.z + (int64_t)slot * X.zw + i] = vz;
  }
  __syncthreads();
  float* a1 = sm + L.a1;
  fcol_mv(zb, W1s, Z, b1, a1, red);
  float yh = 0.f;
  if (warp == 0) {
    float acc = 0.f;
    for (int c = lane; c < kHeadHidden; c += 32) {
      const float av = Act<float>::tanh(a1[c]);
      a1[c] = av;
      a.xch[X.a1 + (int64_t)slot * kHeadHidden + c] = av;
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

// Next-minibatch metadata of this CTA (kernel-wide shared state).
__shared__ int64_t s_nmeta[3];
__shared__ int s_pref;
__shared__ int s_Tn[kMaxFastB];

// Warp 7 during the first BPTT layer: fetch the next minibatch's step counts,
// labels and this CTA's slot metadata into shared memory (none depends on
// the parameters) and warm L2 with the next program's step rows and context,
// so the next forward does not start with dependent DRAM round trips.
__device__ __forceinline__ void prefetch_next_sample(const FastArgs& a, int step, float* lbn) {
  const int lane = threadIdx.x & 31;
  const int64_t nb0 = (int64_t)(step + 1) * a.B;
  if (step + 1 >= a.n_steps || nb0 + blockIdx.x >= a.n_order) return;
  const int bnn = (int)(a.n_order - nb0 < (int64_t)a.B ? a.n_order - nb0 : (int64_t)a.B);
  for (int i = lane; i < bnn; i += 32) {
    const int64_t idx = a.order[nb0 + i];
    const int64_t r0 = a.rowoff[idx], r1 = a.rowoff[idx + 1];
    lbn[i] = a.y[idx];
    s_Tn[i] = (int)(r1 - r0);
    if (i == (int)blockIdx.x) {
      s_nmeta[0] = idx;
      s_nmeta[1] = r0;
      s_nmeta[2] = r1 - r0;
      const char* p0 = reinterpret_cast<const char*>(a.steps + r0 * a.dm.d0);
      const char* p1 = reinterpret_cast<const char*>(a.steps + r1 * a.dm.d0);
      for (const char* p = p0; p < p1; p += 128) asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
      const char* c0 = reinterpret_cast<const char*>(a.ctx + idx * a.dm.C);
      for (int o = 0; o < a.dm.C * 4; o += 128) asm volatile("prefetch.global.L2 [%0];" ::"l"(c0 + o));
    }
  }
  __syncwarp();
  if (lane == 0) s_pref = step + 1;
}

// ------------------------------------------------ sample backward --
__device__ void fast_sample_bwd(const FastArgs& a, float* sm, int64_t rs, int slot, int T,
                                float dy, float yh, int step) {
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
    a.xch[X.da1 + (int64_t)slot * kHeadHidden + tid] = d;
  }
  if (tid < 4) a.xch[X.dl + (int64_t)slot * 4 + tid] = tid == 0 ? dl : 0.f;
  __syncthreads();
  frow_mv(W1s, da1, dpool, red);
  fmark(step, 18);
  // ---- attention passes in reverse (tuner.py:310-328)
  const float sq = sqrtf((float)dh);
  for (int u = U - 1; u >= 0; --u) {
    if (tid < kFD) a.xch[X.dpool + ((int64_t)slot * U + u) * kFD + tid] = dpool[tid];
    frow_mv(Wo, dpool, dmix, red);
    const float* al = sm + L.alpha + (int64_t)u * heads * TM;
    const float* qv = sm + L.q + u * kFD;
    for (int h = warp; h < heads; h += kThreads / 32) {
      float sacc = 0.f;
      for (int t = lane; t < T; t += 32) {
        const float da = fdot4(dmix + h * dh, V + (int64_t)t * kLdK + h * dh, dh);
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
    fmix(dlg, TM, dh, K, T, 1.f / sq, dq, a.xch + X.dq + ((int64_t)slot * U + u) * kFD, red);
    frow_mv(Wq, dq, dpool, red);
    fmark(step, u == U - 1 ? 19 : 24);
  }
  // ---- dS = dpool/denom + dK Wk^T + dV Wv^T (tuner.py:331-338)
  float* dS = sm + L.dS;
  const float denom = (float)(T > 1 ? T : 1);
  for (int i = tid; i < T * kFD; i += kThreads) {
    const int t = i / kFD, k = i % kFD;
    const float4* wk = reinterpret_cast<const float4*>(Wk + k * kLdA);
    const float4* wv = reinterpret_cast<const float4*>(Wv + k * kLdA);
    const float4* dkr = reinterpret_cast<const float4*>(dK + (int64_t)t * kFD);
    const float4* dvr = reinterpret_cast<const float4*>(dV + (int64_t)t * kFD);
    float s0 = 0.f, s1 = 0.f;
#pragma unroll 4
    for (int m = 0; m < kFD / 4; ++m) {
      const float4 a4 = dkr[m], b4 = wk[m], c4 = dvr[m], d4 = wv[m];
      s0 = fmaf(a4.x, b4.x, s0);
      s1 = fmaf(c4.x, d4.x, s1);
      s0 = fmaf(a4.y, b4.y, s0);
      s1 = fmaf(c4.y, d4.y, s1);
      s0 = fmaf(a4.z, b4.z, s0);
      s1 = fmaf(c4.z, d4.z, s1);
      s0 = fmaf(a4.w, b4.w, s0);
      s1 = fmaf(c4.w, d4.w, s1);
    }
    dS[i] = (dpool[k] / denom + s0) + s1;
    a.xch[X.dK + rs * kFD + i] = dK[i];
    a.xch[X.dV + rs * kFD + i] = dV[i];
  }
  __syncthreads();
  fmark(step, 10);
  signal_counter(a.ctr + ctr_bwd(dm.L), 1);  // attention/head operands published
  if (a.s_frozen) return;  // heads-only mode: the recurrent stack is frozen
  // ---- LSTM stack in reverse (tuner.py:340-359).  Warps 0..3 run the two
  //      BPTT recurrences (a warp pair per direction); every thread holds a
  //      64-column slice of one Wx row for dX, fetched before the BPTT so the
  //      load overlaps it.
  float* dSa = dS;
  float* dSb = sm + L.dS2;
  float* dZ = sm + L.dZ;
  float* part = sm + L.xz;  // [4][TM][64] dX partials (xz is dead)
  const int xk = tid & 63, xq = tid >> 6, xdir = xq >> 1, xhalf = xq & 1;
  // Wh rows of layer l-1 are prefetched into W (rows padded to 132 floats,
  // double-buffered by layer parity) by warps 4..7 during BPTT of layer l, so
  // only the first backward layer reads its Wh rows from L2.
  constexpr int kLdWh = 132;
  float* const Wm = sm + L.W;
  auto whs = [&](int ll) { return Wm + (ll & 1) * (2 * kFH * kLdWh); };
  for (int l = dm.L - 1; l >= 0; --l) {
    WReg whr;
    float wx[64];
    if (warp < 4) {
      if (l == dm.L - 1) {
        load_wh_row(whr, a.prm + dm.wh[l][warp >> 1], warp & 1);
      } else {
        const float4* w4 =
            reinterpret_cast<const float4*>(whs(l) + ((warp >> 1) * kFH + lane) * kLdWh + (warp & 1) * 64);
#pragma unroll
        for (int m = 0; m < 16; ++m) {
          const float4 v = w4[m];
          whr[4 * m + 0] = v.x;
          whr[4 * m + 1] = v.y;
          whr[4 * m + 2] = v.z;
          whr[4 * m + 3] = v.w;
        }
      }
    }
    auto load_wx = [&]() {
      const float4* w4 =
          reinterpret_cast<const float4*>(a.prm + dm.wx[l][xdir] + (int64_t)xk * kFG + xhalf * 64);
#pragma unroll
      for (int m = 0; m < 16; ++m) {
        const float4 v = __ldcg(w4 + m);
        wx[4 * m + 0] = v.x;
        wx[4 * m + 1] = v.y;
        wx[4 * m + 2] = v.z;
        wx[4 * m + 3] = v.w;
      }
    };
    // dX operands: warps 4..7 (direction 1) hold their Wx slice in registers
    // from L2; the recurrence warps must not have L2 loads outstanding during
    // the BPTT (they slow its per-step exchange), so warps 4..7 also stage
    // direction 0's Wx rows into the Wh buffer this layer no longer needs
    // (rows padded to 132 floats) and warps 0..3 read them after the BPTT
    if (l > 0 && l < dm.L - 1) __syncthreads();  // whr is out of whs(l)
    if (l > 0 && warp >= 4) {
      load_wx();
      float* dst = whs(l);
      for (int e = tid - 128; e < kFD * (kFG / 4); e += kThreads - 128) {
        const int row = e >> 5, q = e & 31;
        cp_async16(dst + row * kLdWh + q * 4, a.prm + dm.wx[l][0] + (int64_t)row * kFG + q * 4);
      }
    }
    if (warp < 4) {
      fast_rec_bwd(whr, warp >> 1, warp & 1, T, TM, sm + L.gc + (int64_t)l * 2 * TM * kFG,
                   sm + L.cs + (int64_t)l * 2 * TM * kFH, dSa, dZ,
                   a.xch + X.dZ + (((int64_t)l * 2 + (warp >> 1)) * X.Rmax + rs) * kFG,
                   sm + L.gex);
      if (warp == 0) fmark(step, 11 + (dm.L - 1 - l) * 2);
    } else {
      if (warp == 7 && l == dm.L - 1 && a.B <= (int)gridDim.x) prefetch_next_sample(a, step, sm + L.lbn);
      if (l > 0) {
        // next backward layer's Wh rows -> the other W buffer
        float* dst = whs(l - 1);
        for (int e = tid - 128; e < 2 * kFH * (kFG / 4); e += kThreads - 128) {
          const int row = e >> 5, q = e & 31;  // row = dir*32 + j
          cp_async16(dst + row * kLdWh + q * 4, a.prm + dm.wh[l - 1][row >> 5] + (row & 31) * kFG + q * 4);
        }
        cp_async_wait_all();
      }
    }
    __syncthreads();
    signal_counter(a.ctr + ctr_bwd(l), 1);  // this layer's dZ published
    if (l == 0) break;
    if (warp < 4) {
      const float4* w4 = reinterpret_cast<const float4*>(whs(l) + xk * kLdWh + xhalf * 64);
#pragma unroll
      for (int m = 0; m < 16; ++m) {
        const float4 v = w4[m];
        wx[4 * m + 0] = v.x;
        wx[4 * m + 1] = v.y;
        wx[4 * m + 2] = v.z;
        wx[4 * m + 3] = v.w;
      }
    }
    for (int t = 0; t < T; ++t)
      part[((int64_t)xq * TM + t) * kFD + xk] =
          dot64<0>(dZ + ((int64_t)xdir * TM + t) * kFG + xhalf * 64, wx);
    __syncthreads();
    for (int i = tid; i < T * kFD; i += kThreads) {
      const int64_t o = (int64_t)TM * kFD;
      dSb[i] = (part[i] + part[o + i]) + (part[2 * o + i] + part[3 * o + i]);  // dX_fw + dX_bw
    }
    __syncthreads();
    fmark(step, 12 + (dm.L - 1 - l) * 2);
    float* tmp = dSa;
    dSa = dSb;
    dSb = tmp;
  }
  __syncthreads();
}

// ------------------------------------------------------ job runner --
// Stage operand rows [r0, r1) of job `jb` into shared memory: A rows
// [n][kap] = [segment 1 (w1) | h_prev (32, LSTM) | ones/pad chunk], B rows
// [n][nbp] = the job's column slice.  The exchange is stacked by row, so
// every operand is one flat loop of 16-B cp.async.cg copies (L2 -> smem).
// what: 1 = A operand only (forward data: may be staged before the
// backward of the minibatch is done), 2 = B operand only, 3 = both.
__device__ void fast_job_stage(const FastArgs& a, const FastJob& jb, const JobGeo& g, int64_t r0,
                               int64_t r1, float* As, float* Bs, int what = 3) {
  const TDims& dm = a.dm;
  const FastXch& X = a.xl;
  const int tid = threadIdx.x;
  const int kap = g.kap, nbp = g.nbp, nq = jb.nb / 4 > 0 ? jb.nb / 4 : 1;
  const int q1 = g.w1 / 4;
  const int n = (int)(r1 - r0);
  const float* A1;
  const float* A2 = nullptr;
  const float* B1;
  int lda1, ldb1;
  const float* xc = a.xch;
  switch (jb.kind) {
    case FJ_LSTM:
      if (jb.l == 0) {
        A1 = xc + X.x0;
        lda1 = X.w0;
      } else {
        A1 = xc + X.S + (int64_t)(jb.l - 1) * X.Rmax * kFD;
        lda1 = kFD;
      }
      A2 = xc + X.H + ((int64_t)jb.l * 2 + jb.dir) * X.Rmax * kFH;
      B1 = xc + X.dZ + ((int64_t)jb.l * 2 + jb.dir) * X.Rmax * kFG + jb.c0;
      ldb1 = kFG;
      break;
    case FJ_WK:
    case FJ_WV:
      A1 = xc + X.S + (int64_t)(dm.L - 1) * X.Rmax * kFD;
      lda1 = kFD;
      B1 = xc + (jb.kind == FJ_WK ? X.dK : X.dV) + jb.c0;
      ldb1 = kFD;
      break;
    case FJ_WQ:
    case FJ_WO:
      A1 = xc + (jb.kind == FJ_WQ ? X.pin : X.mix);
      lda1 = kFD;
      B1 = xc + (jb.kind == FJ_WQ ? X.dq : X.dpool) + jb.c0;
      ldb1 = kFD;
      break;
    case FJ_W1:
      A1 = xc + X.z;
      lda1 = X.zw;
      B1 = xc + X.da1 + jb.c0;
      ldb1 = kHeadHidden;
      break;
    default:
      A1 = xc + X.a1;
      lda1 = kHeadHidden;
      B1 = xc + X.dl;
      ldb1 = 4;
  }
  A1 += r0 * lda1;
  B1 += r0 * ldb1;
  if (what & 1) {
  for (int e = tid; e < n * q1; e += kThreads) {
    const int r = e / q1, q = e - r * q1;
    cp_async16(As + r * kap + q * 4, A1 + (int64_t)r * lda1 + q * 4);
  }
  if (A2) {
    A2 += r0 * kFH;
    for (int e = tid; e < n * 8; e += kThreads) {
      const int r = e >> 3, q = e & 7;
      cp_async16(As + r * kap + g.w1 + q * 4, A2 + (int64_t)r * kFH + q * 4);
    }
  }
  const int c0 = g.w1 + g.n2;
  if (kap > c0) {  // ones column (bias) + zero padding, from the constant chunk
    const float* src = xc + X.cst + (g.bias ? 4 : 0);
    for (int r = tid; r < n; r += kThreads) cp_async16(As + r * kap + c0, src);
  }
  }
  if (what & 2)
    for (int e = tid; e < n * nq; e += kThreads) {
      const int r = e / nq, q = e - r * nq;
      cp_async16(Bs + r * nbp + q * 4, B1 + (int64_t)r * ldb1 + q * 4);
    }
  cp_async_wait_all();
  __syncthreads();
}

// Data-parallel exchange buffer of one rank (allocated by the host, shared
// with the peers by IPC): receive slots [parity][job][source rank][slice] of
// 8-byte words {value bits, flag} (the flag = global step + 1).
__host__ __device__ inline int64_t fast_dp_buffer_bytes(int n_jobs, int world, int64_t slice) {
  return 2 * (int64_t)n_jobs * world * slice * 8;
}

// The job's reduced slice gout[n] (this rank's microbatch) -> the mean over
// the world's microbatches (SURVEY §8e option A: pairs stay inside each
// rank's microbatch), identical on every rank.  Low-latency protocol: every
// value travels with its step flag in one 8-byte single-copy-atomic word,
// stored straight into each peer's receive slot; the receiver spins on its
// own words until the flags match and sums the ranks in fixed order -- no
// fences, no separate flag round trip.  Slots alternate by step parity: a
// rank can only reach the next use of a parity after every peer has read it
// (it needs their slices of the step in between).
// (out of line with scalar arguments: keeps the exchange out of the
// register allocation of the single-GPU kernel body)
// The spin on a peer's slot is bounded: every 256 polls it checks the
// launch's abort word (status[1]) and %globaltimer; past `timeout_ns` without
// the peer's word it raises status[1] = 1 and stops waiting (the slot reads as
// 0), and once the abort word is set every later exchange skips its waits, so
// a dead or diverged peer ends the epoch quickly with an error the host
// raises instead of hanging every rank.
__device__ __noinline__ void fast_dp_exchange(void* const* xb, int W, int me, int64_t gs,
                                              int64_t slice, int n_jobs, int j, float* gout, int n,
                                              int32_t* status, long long timeout_ns) {
  const int tid = threadIdx.x;
  const unsigned long long tag = (unsigned long long)(unsigned)(gs + 1) << 32;
  const int64_t base = ((gs & 1) * (int64_t)n_jobs + j) * W * slice;
  for (int i = tid; i < n; i += kThreads) {
    const unsigned long long w = tag | __float_as_uint(gout[i]);
    for (int p = 0; p < W; ++p)
      if (p != me) {
        unsigned long long* dst =
            reinterpret_cast<unsigned long long*>(xb[p]) + base + (int64_t)me * slice + i;
        asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(dst), "l"(w) : "memory");
      }
  }
  const unsigned long long* rx = reinterpret_cast<const unsigned long long*>(xb[me]) + base;
  const float inv = 1.f / (float)W;
  bool aborted = __ldcg(status + 1) != 0;
  for (int i = tid; i < n; i += kThreads) {
    float acc = 0.f;
    for (int p = 0; p < W; ++p) {
      float v;
      if (p == me) {
        v = gout[i];
      } else {
        unsigned long long w = 0;
        unsigned long long t0 = 0;
        for (unsigned spin = 0; !aborted; ++spin) {
          asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(w) : "l"(rx + (int64_t)p * slice + i) : "memory");
          if ((w & 0xffffffff00000000ull) == tag) break;
          if ((spin & 255) != 255) continue;
          unsigned long long now;
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
          if (t0 == 0) t0 = now;
          if (__ldcg(status + 1) != 0) {
            aborted = true;
          } else if ((long long)(now - t0) > timeout_ns) {
            atomicExch(status + 1, 1);
            aborted = true;
          }
        }
        v = aborted ? 0.f : __uint_as_float((unsigned)w);
      }
      acc += v;
    }
    gout[i] = acc * inv;
  }
  __syncthreads();
}

// R: stacked step rows of the minibatch; bn: samples.
// keep: this CTA owns the slice for the whole launch (not a sampler), so the
// parameters, Adam moments and trainable mask of the slice stay in shared
// memory across minibatches (loaded at the first step, moments written back
// at the last); otherwise they are read from and written to global memory.
__device__ __forceinline__ int64_t job_rows(const TDims& dm, const FastJob& jb, int bn, int64_t R) {
  return jb.kind == FJ_LSTM || jb.kind == FJ_WK || jb.kind == FJ_WV
             ? R
             : (jb.kind == FJ_WQ || jb.kind == FJ_WO ? (int64_t)bn * dm.U : bn);
}

// a_staged: the A operand of all rows was staged by the caller (single chunk).
__device__ void fast_run_job(const FastArgs& a, const FastJob& jb, int jidx, int bn, int64_t R,
                             int step, float* sm, bool keep, bool a_staged) {
  const TDims& dm = a.dm;
  const int tid = threadIdx.x;
  const JobGeo geo = job_geo(dm, jb);
  const int kap = geo.kap, nbp = geo.nbp, maxr = geo.maxr;
  const int nkb = kap / 4, ncb = nbp / 4, nblk = nkb * ncb;
  const int RG = nblk >= kThreads ? 1 : kThreads / nblk;
  (void)maxr;
  const int64_t nrows = job_rows(dm, jb, bn, R);
  const int64_t rch = a.rch;  // rows per staging chunk
  float* As = sm;
  float* Bs = As + rch * kap;
  float* redb = Bs + rch * nbp;                         // [RG][nblk][16]
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
  for (int64_t c0 = 0; c0 < nrows; c0 += rch) {
    const int64_t c1 = c0 + rch < nrows ? c0 + rch : nrows;
    __syncthreads();
    fast_job_stage(a, jb, geo, c0, c1, As, Bs, a_staged ? 2 : 3);
    if (blockIdx.x == (unsigned)(a.B % gridDim.x)) fmark_any(step, 22);
    const int n = (int)(c1 - c0);
    if (active) {
      for (int rr = g; rr < n; rr += RG) {
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
  if (blockIdx.x == (unsigned)(a.B % gridDim.x)) fmark_any(step, 23);
  if (a.world > 1 && a.mode == TT_MODE_TRAIN)
    fast_dp_exchange(a.xb, a.world, a.rank, a.gbase + step, a.dp_slice, a.n_jobs, jidx, gout, kap * nbp,
                     a.status, a.dp_timeout_ns);
  // parameter addresses of the slice and the fused Adam update
  const double c1 = a.mode == TT_MODE_TRAIN ? a.corr[2 * step] : 1.0;
  const double c2 = a.mode == TT_MODE_TRAIN ? a.corr[2 * step + 1] : 1.0;
  const int nb = jb.nb;
  for (int i = tid; i < geo.ka * nb; i += kThreads) {
    const int k = i / nb, c = i % nb;
    int64_t p;
    if (k < geo.n1)
      p = geo.base + (int64_t)k * geo.ldp + jb.c0 + c;
    else if (k < geo.w1)
      continue;  // zero padding column
    else if (k < geo.w1 + geo.n2)
      p = geo.base + (int64_t)(geo.n1 + k - geo.w1) * geo.ldp + jb.c0 + c;
    else
      p = geo.bptr + jb.c0 + c;
    const float gv = gout[k * nbp + c];
    if (a.mode == TT_MODE_GRAD) {
      a.grad_out[p] = gv;
    } else if (keep) {
      float* pc = sm + a.pc_off + k * nbp + c;
      float pp, mm, vv, tr;
      if (step == 0) {
        pp = __ldcg(a.prm + p);
        mm = a.m[p];
        vv = a.v[p];
        tr = (!a.trainable || a.trainable[p]) ? 1.f : 0.f;
        pc[3 * a.pc_n] = tr;
      } else {
        pp = pc[0];
        mm = pc[a.pc_n];
        vv = pc[2 * a.pc_n];
        tr = pc[3 * a.pc_n];
      }
      if (tr != 0.f) {
        adam_update<float>(pp, gv, mm, vv, a.hyp, c1, c2);
        a.prm[p] = pp;
        if (step == a.n_steps - 1) {
          a.m[p] = mm;
          a.v[p] = vv;
        }
      }
      pc[0] = pp;
      pc[a.pc_n] = mm;
      pc[2 * a.pc_n] = vv;
    } else if (!a.trainable || a.trainable[p]) {
      float pp = __ldcg(a.prm + p), mm = a.m[p], vv = a.v[p];
      adam_update<float>(pp, gv, mm, vv, a.hyp, c1, c2);
      a.prm[p] = pp;
      a.m[p] = mm;
      a.v[p] = vv;
    }
  }
}

// Pairwise logistic loss over the minibatch (mlp.py:25-35), all threads:
// warp w owns rows k = w, w+8, ..; lanes sweep j.  Same per-pair terms as
// rank_loss_block; per-row sums by warp shuffles, the row totals summed in
// fixed order.  red needs 2n floats.  Returns the loss in every thread.
__device__ float fast_rank_loss(const float* y, const float* s, int n, float* dscore, float* red) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int k = warp; k < n; k += kThreads / 32) {
    const float yk = y[k], sk = s[k];
    float d = 0.f, part = 0.f, pairs = 0.f;
    for (int j = lane; j < n; j += 32) {
      const float yj = y[j], sj = s[j];
      if (yj > yk) d += 1.f / (1.f + Act<float>::exp(sj - sk));
      if (yk > yj) {
        const float mg = sk - sj;
        d -= 1.f / (1.f + Act<float>::exp(mg));
        part += Act<float>::softplus(-mg);
        pairs += 1.f;
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
  __shared__ float s_tot[2];
  if (threadIdx.x == 0) {
    float tot = 0.f, np = 0.f;
    for (int k = 0; k < n; ++k) {
      tot += red[k];
      np += red[n + k];
    }
    s_tot[0] = tot;
    s_tot[1] = np;
  }
  __syncthreads();
  const float np = s_tot[1];
  for (int k = threadIdx.x; k < n; k += kThreads) dscore[k] = np == 0.f ? 0.f : dscore[k] / np;
  const float loss = np == 0.f ? 0.f : s_tot[0] / np;
  __syncthreads();
  return loss;
}

// Minibatches of <= 16: one pair (k, j) per thread (k = tid / 16, j =
// tid % 16), row sums by half-warp shuffles, the row totals by one warp --
// the same per-pair terms as fast_rank_loss in a fixed order.  red >= 48.
__device__ float fast_rank_loss16(const float* y, const float* s, int n, float* dscore, float* red) {
  const int tid = threadIdx.x, k = tid >> 4, j = tid & 15;
  float d = 0.f, part = 0.f, pairs = 0.f;
  if (k < n && j < n) {
    const float yk = y[k], sk = s[k], yj = y[j], sj = s[j];
    if (yj > yk) d = 1.f / (1.f + Act<float>::exp(sj - sk));
    if (yk > yj) {
      const float mg = sk - sj;
      d -= 1.f / (1.f + Act<float>::exp(mg));
      part = Act<float>::softplus(-mg);
      pairs = 1.f;
    }
  }
#pragma unroll
  for (int o = 8; o > 0; o >>= 1) {
    d += __shfl_xor_sync(0xffffffffu, d, o);
    part += __shfl_xor_sync(0xffffffffu, part, o);
    pairs += __shfl_xor_sync(0xffffffffu, pairs, o);
  }
  if (j == 0 && k < 16) {
    red[k] = d;
    red[16 + k] = part;
    red[32 + k] = pairs;
  }
  __syncthreads();
  __shared__ float s_l;
  if (tid < 32) {
    float tp = tid < n ? red[16 + tid] : 0.f, np = tid < n ? red[32 + tid] : 0.f;
    const float dk = tid < n ? red[tid] : 0.f;
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) {
      tp += __shfl_xor_sync(0xffffffffu, tp, o);
      np += __shfl_xor_sync(0xffffffffu, np, o);
    }
    if (tid < n) dscore[tid] = np == 0.f ? 0.f : dk / np;
    if (tid == 0) s_l = np == 0.f ? 0.f : tp / np;
  }
  __syncthreads();
  return s_l;
}

// Multi-round mode: the pair terms of this CTA's own slots only (rows
// k = r, r + G, ..; warp per row, lanes sweep j), unnormalised dscore into
// smem and the row's (loss part, pair count) into the global partials.
__device__ void fast_rank_rows(const float* y, const float* s, int n, int r, int G, float* dscore,
                               float* lossp) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int k = r + warp * G; k < n; k += (kThreads / 32) * G) {
    const float yk = y[k], sk = s[k];
    float d = 0.f, part = 0.f, pairs = 0.f;
    for (int j = lane; j < n; j += 32) {
      const float yj = y[j], sj = s[j];
      if (yj > yk) d += 1.f / (1.f + Act<float>::exp(sj - sk));
      if (yk > yj) {
        const float mg = sk - sj;
        d -= 1.f / (1.f + Act<float>::exp(mg));
        part += Act<float>::softplus(-mg);
        pairs += 1.f;
      }
    }
    d = warp_sum(d);
    part = warp_sum(part);
    pairs = warp_sum(pairs);
    if (lane == 0) {
      dscore[k] = d;
      lossp[2 * k] = part;
      lossp[2 * k + 1] = pairs;
    }
  }
}

// Fixed-order sum of the published partials (identical in every CTA).
__device__ void fast_sum_partials(const float* lossp, int n, float* red, float* out2) {
  const int tid = threadIdx.x;
  float a = 0.f, b = 0.f;
  for (int k = tid; k < n; k += kThreads) {
    a += __ldcg(lossp + 2 * k);
    b += __ldcg(lossp + 2 * k + 1);
  }
  red[tid] = a;
  red[kThreads + tid] = b;
  __syncthreads();
  if (tid == 0) {
    float ta = 0.f, tb = 0.f;
    for (int i = 0; i < kThreads; ++i) {
      ta += red[i];
      tb += red[kThreads + i];
    }
    out2[0] = ta;
    out2[1] = tb;
  }
  __syncthreads();
}

// ------------------------------------------------------------ kernel --
__global__ void __launch_bounds__(kThreads, 1) tuner_train_fast_kernel(FastArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float* sm = reinterpret_cast<float*>(smem_raw);
  __shared__ int64_t s_R;
  __shared__ int s_stop;
  const TDims& dm = a.dm;
  if (threadIdx.x == 0) {
    s_pref = -1;
    s_prof = g_prof_step;
    s_wph = 0;
    sm100::mbar_init(&s_wbar, 1);
    sm100::mbar_init(&s_cbar, 1);
    sm100::fence_barrier_init();
  }
  __syncthreads();
  if (blockIdx.x == 0 && threadIdx.x < 8)  // constant chunks [0 0 0 0 | 1 0 0 0] for job staging
    a.xch[a.xl.cst + threadIdx.x] = threadIdx.x == 4 ? 1.f : 0.f;
  const int tid = threadIdx.x;
  const int G = gridDim.x, r = blockIdx.x;
  const bool sampler = r < a.B;
  const int first_job = ((r - a.B) % G + G) % G;
  int my_jobs = 0, last_job = -1;
  for (int j = first_job; j < a.n_jobs; j += G) ++my_jobs, last_job = j;
  float* lb = sm + a.sl.lb;
  int* const sT = reinterpret_cast<int*>(sm + a.sl.ts);
  int* const sRs = reinterpret_cast<int*>(sm + a.sl.rsb);
  // layer 0's two direction blocks [Wx | Wh | b] into W (bulk copies by warp
  // 4; the attention weights there are dead), awaited inside the forward
  auto issue_l0 = [&]() {
    if (a.l0_smem && !a.s_frozen && (tid >> 5) == 4) {
      const uint32_t blk0 = (uint32_t)(dm.d0 + kFH + 1) * kFG;
      sm100::fence_proxy_async_smem();
      if ((tid & 31) == 0) sm100::mbar_expect_tx(&s_wbar, 2u * blk0 * 4u);
      __syncwarp();
      if ((tid & 31) < 2)
        sm100::bulk_g2s(sm + a.sl.W + (tid & 31) * blk0, a.prm + dm.wx[0][tid & 31], blk0 * 4u, &s_wbar);
    }
  };
  // raw step rows of slot k -> smem (layer-0 projection) and the stacked
  // exchange (layer-0 weight gradient), zero padded to 16 B rows; context row
  auto stage_rows = [&](int64_t rs, int64_t r0, int T, int64_t idx) {
    const int w0 = a.xl.w0;
    const float* x0 = a.steps + r0 * dm.d0;
    float* xg = a.xch + a.xl.x0 + rs * w0;
    for (int i = tid; i < (a.s_frozen ? 0 : T * w0); i += kThreads) {
      const int t = i / w0, k = i - t * w0;
      const float v = k < dm.d0 ? __ldg(x0 + (int64_t)t * dm.d0 + k) : 0.f;
      sm[a.sl.x0 + i] = v;
      xg[i] = v;
    }
    for (int i = tid; i < dm.C; i += kThreads) sm[a.sl.ctxs + i] = __ldg(a.ctx + idx * dm.C + i);
    __syncthreads();
  };
  // multi-round mode: a slot's forward caches ([x0, red) of the sample
  // layout) and the attention/head weight image in W go to L2 by bulk
  // stores after its forward and come back by bulk loads before its
  // backward (instead of recomputing the forward)
  const int64_t cfl = a.sl.red - a.sl.x0;
  const int64_t wfl = fast_attn_floats(dm);
  uint32_t cph = 0;
  auto save_slot = [&](int k, bool with_w) {
    __syncthreads();
    if (tid == 0) {
      sm100::fence_proxy_async_smem();
      sm100::bulk_s2g(a.scache + (int64_t)k * cfl, sm + a.sl.x0, (uint32_t)(cfl * 4));
      if (with_w) sm100::bulk_s2g(a.wcache + (int64_t)r * wfl, sm + a.sl.W, (uint32_t)(wfl * 4));
      sm100::bulk_commit();
      sm100::bulk_wait_read0();
    }
    __syncthreads();
  };
  auto restore_slot = [&](int k) {
    __syncthreads();
    if (tid == 0) {
      sm100::bulk_wait0();
      sm100::fence_proxy_async_smem();
      sm100::mbar_expect_tx(&s_cbar, (uint32_t)((cfl + wfl) * 4));
      sm100::bulk_g2s(sm + a.sl.x0, a.scache + (int64_t)k * cfl, (uint32_t)(cfl * 4), &s_cbar);
      sm100::bulk_g2s(sm + a.sl.W, a.wcache + (int64_t)r * wfl, (uint32_t)(wfl * 4), &s_cbar);
    }
    sm100::mbar_wait(&s_cbar, cph);
    cph ^= 1u;
  };
  for (int step = 0; step < a.n_steps; ++step) {
    const int64_t b0 = (int64_t)step * a.B;
    const int bn = (int)(a.n_order - b0 < (int64_t)a.B ? a.n_order - b0 : (int64_t)a.B);
    const unsigned cum = (unsigned)(b0 + bn);
    if (sampler && r < bn) {
      // slots k = r, r + G, ..: one per CTA on the latency path (B <= grid);
      // large minibatches run several rounds per CTA (forward of every slot,
      // loss, then per slot a recomputed forward -- the last slot's caches
      // are still resident -- and its backward)
      const int nmine = (bn - r + G - 1) / G;
      fmark(step, 0);
      if (step > 0 && !a.s_frozen)  // layer 0's update (the other groups are awaited where prefetched)
        wait_counter(a.ctr + ctr_adam(dm, 0), (unsigned)(step * group_jobs(dm, 0)), false);
      issue_l0();
      fmark(step, 1);
      if (r == 0) fmark_any(step, 31);
      // step counts, labels and slot metadata: prefetched into smem during the
      // previous step's backward (prefetch_next_sample), else loaded here
      if (s_pref != step) {
        for (int i = tid; i < bn; i += kThreads) {
          const int64_t idx = a.order[b0 + i];
          const int64_t r0 = a.rowoff[idx], r1 = a.rowoff[idx + 1];
          lb[i] = a.y[idx];
          sT[i] = (int)(r1 - r0);
          if (i == r) {
            s_nmeta[0] = idx;
            s_nmeta[1] = r0;
            s_nmeta[2] = r1 - r0;
          }
        }
      } else {
        for (int i = tid; i < bn; i += kThreads) {
          lb[i] = sm[a.sl.lbn + i];
          sT[i] = s_Tn[i];
        }
      }
      __syncthreads();
      if (a.B > G && tid < 32) {  // exclusive prefix of the step counts (stacked rows)
        int carry = 0;
        for (int base = 0; base < bn; base += 32) {
          const int i = base + tid;
          const int v = i < bn ? sT[i] : 0;
          int inc = v;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int u = __shfl_up_sync(0xffffffffu, inc, o);
            if (tid >= o) inc += u;
          }
          if (i < bn) sRs[i] = carry + inc - v;
          carry += __shfl_sync(0xffffffffu, inc, 31);
        }
      }
      if (a.B > G) __syncthreads();
      for (int m = 0; m < nmine; ++m) {
        const int k = r + m * G;
        int64_t idx, r0;
        int T;
        if (m == 0) {
          idx = s_nmeta[0];
          r0 = s_nmeta[1];
          T = (int)s_nmeta[2];
        } else {
          idx = a.order[b0 + k];
          r0 = a.rowoff[idx];
          T = sT[k];
          issue_l0();
        }
        if (tid == 0) a.meta[k] = T;
        int64_t rs;
        if (a.B <= G) {  // one slot: only its own first stacked row
          rs = 0;
          for (int i = 0; i < r; ++i) rs += sT[i];
          if (tid == 0) sRs[k] = (int)rs;  // for the backward (after stage_rows' barrier)
        } else {
          rs = sRs[k];
        }
        stage_rows(rs, r0, T, idx);
        const float yh = fast_sample_fwd(a, sm, rs, k, r0, T, idx, step);
        if (tid == 0) a.yhat_buf[k] = yh;
        signal_counter(a.ctr + 0, 1);
        if (m + 1 < nmine) save_slot(k, m == 0);
      }
      fmark(step, 5);
      wait_counter(a.ctr + 0, cum, false);
      fmark(step, 6);
      for (int i = tid; i < bn; i += kThreads) lb[bn + i] = __ldcg(a.yhat_buf + i);
      __syncthreads();
      float loss;
      if (a.loss_kind == TT_LOSS_RANK && a.B > G) {
        // O(B^2) pairs: each CTA evaluates its own rows, the loss total is
        // exchanged through L2 (one more counter)
        fast_rank_rows(lb, lb + bn, bn, r, G, lb + 2 * bn, a.lossp);
        signal_counter(a.ctr + kCtrLoss, (unsigned)nmine);
        wait_counter(a.ctr + kCtrLoss, cum, false);
        __shared__ float s_lt[2];
        fast_sum_partials(a.lossp, bn, sm + a.sl.red, s_lt);
        const float np = s_lt[1];
        for (int m = tid; m < nmine; m += kThreads) {
          const int k = r + m * G;
          lb[2 * bn + k] = np == 0.f ? 0.f : lb[2 * bn + k] / np;
        }
        loss = np == 0.f ? 0.f : s_lt[0] / np;
        __syncthreads();
      } else {
        loss = a.loss_kind == TT_LOSS_RANK
                   ? (bn <= 16 ? fast_rank_loss16(lb, lb + bn, bn, lb + 2 * bn, sm + a.sl.red)
                               : fast_rank_loss(lb, lb + bn, bn, lb + 2 * bn, sm + a.sl.red))
                   : mse_block<float>(lb, lb + bn, bn, lb + 2 * bn, sm + a.sl.red);
      }
      if (tid == 0) {
        // data parallel: a non-finite loss is recorded but the rank keeps
        // stepping (its peers wait for its slices); the host raises afterwards
        s_stop = !isfinite(loss) && a.world <= 1;
        if (r == 0) {
          a.step_loss[step] = loss;
          if (!isfinite(loss) && __ldcg(a.status) < 0) a.status[0] = step;
        }
      }
      __syncthreads();
      fmark(step, 7);
      if (!s_stop) {
        for (int m = nmine - 1; m >= 0; --m) {
          const int k = r + m * G;
          const int T = sT[k];
          if (m != nmine - 1) restore_slot(k);  // the last slot's caches are resident
          fast_sample_bwd(a, sm, sRs[k], k, T, lb[2 * bn + k], lb[bn + k], step);
        }
      } else {
        for (int g = 0; g <= dm.L; ++g) signal_counter(a.ctr + ctr_bwd(g), (unsigned)nmine);  // wake the jobs
      }
      fmark(step, 16);
      if (r == 0) fmark_any(step, 30);
      if (s_stop) break;
    }
    if (my_jobs == 0) {
      if (!sampler) break;  // idle CTA
      continue;
    }
    // minibatch row count: every sample CTA published its step count before
    // signalling the forward counter, so this read is off the critical path
    wait_counter(a.ctr + 0, cum, !sampler);
    if (tid == 0) {
      int64_t R = 0;
      for (int i = 0; i < bn; ++i) R += __ldcg(a.meta + i);
      s_R = R;
    }
    // this CTA's jobs, attention/head group first, then the LSTM layers top-down
    // (the order in which the samples publish their backward operands)
    const bool keep = !sampler && my_jobs == 1;
    bool a_staged = false;
    if (keep && !(a.s_frozen && job_group(dm, last_job) < dm.L)) {
      // single job: stage its A operand (forward data) while the samples run
      // their backward, so only the B operand waits for the backward counter
      __syncthreads();
      const FastJob jb = fast_job(dm, last_job);
      const int64_t nr = job_rows(dm, jb, bn, s_R);
      if (nr <= a.rch) {
        const JobGeo geo = job_geo(dm, jb);
        fast_job_stage(a, jb, geo, 0, nr, sm, sm + a.rch * geo.kap, 1);
        a_staged = true;
      }
    }
    for (int j = last_job; j >= 0; j -= G) {
      const int g = job_group(dm, j);
      if (a.s_frozen && g < dm.L) continue;  // heads-only: recurrent slices are frozen
      wait_counter(a.ctr + ctr_bwd(g), cum, !sampler);
      if (r == a.B % G) fmark_any(step, 20);
      if (tid == 0) s_stop = a.world <= 1 && __ldcg(a.status) >= 0;
      __syncthreads();
      if (s_stop) break;
      fast_run_job(a, fast_job(dm, j), j, bn, s_R, step, sm, keep, a_staged);
      signal_counter(a.ctr + ctr_adam(dm, g), 1);
      if (r == a.B % G) fmark_any(step, 21);
    }
    if (s_stop) break;
  }
}

// --------------------------------------------------------- host side --
// CTAs of the latency-path launch: every SM, unless a test splits the GPU
// between concurrently running "ranks" (tt_tuner_train_set_grid)
static int g_fast_grid = 0;
inline int fast_grid() { return g_fast_grid > 0 ? std::min(g_fast_grid, sm_count()) : sm_count(); }

struct FastPlan {
  FastSmem sl;
  FastXch xl;
  size_t smem;
  int64_t rch, pc_off;
  int pc_n, l0_smem;
  int n_jobs;
  int64_t dp_slice;  // floats per data-parallel slice slot
};

inline size_t fast_ws_bytes(const TDims& dm, int B) {
  const FastXch xl = make_fast_xch(dm, B);
  size_t b = align_up((size_t)xl.total * sizeof(float), 256) + align_up((size_t)B * 8, 256) +
             align_up((size_t)B * sizeof(float), 256) + align_up((size_t)B * 2 * sizeof(float), 256) + 256;
  if (B > fast_grid()) {  // multi-round: per-slot forward caches + per-CTA weight images
    const FastSmem sl = make_fast_smem(dm, B);
    b += align_up((size_t)B * (sl.red - sl.x0) * sizeof(float), 256) +
         align_up((size_t)fast_grid() * fast_attn_floats(dm) * sizeof(float), 256);
  }
  return b;
}

// Eligible: fp32, hidden 32, one sample per CTA, every per-sample cache in
// shared memory.  Returns false (generic kernel) otherwise.
inline bool fast_plan(const TDims& dm, int B, int grid, FastPlan& p) {
  // B <= grid: one slot per CTA (latency path, <= kMaxFastB for the metadata
  // prefetch); larger minibatches run ceil(B / grid) rounds per CTA
  if (dm.H != kFH || B < 1 || dm.Tmax > 32 || dm.heads < 1 || kFD % (4 * dm.heads) != 0)
    return false;
  if (B <= grid ? B > kMaxFastB : B > kMaxRoundB) return false;
  int dev = 0, optin = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return false;
  if (cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess)
    return false;
  p.sl = make_fast_smem(dm, B);
  p.xl = make_fast_xch(dm, B);
  p.n_jobs = fast_n_jobs(dm);
  cudaFuncAttributes fa{};
  if (cudaFuncGetAttributes(&fa, tuner_train_fast_kernel) != cudaSuccess) return false;
  const size_t budget = (size_t)optin - fa.sharedSizeBytes - 256;
  size_t need = (size_t)p.sl.total * sizeof(float);
  if (need > budget) return false;
  // job staging: at least Tmax rows of the widest job
  const int kap_max = std::max(round4(round4(std::max(dm.d0, kFD)) + kFH + 1),
                               round4(round4(kFD + dm.C) + 1));
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
  p.pc_n = kap_max * nbp;
  p.l0_smem = (int64_t)2 * (dm.d0 + kFH + 1) * kFG <= p.sl.total - p.sl.W ? 1 : 0;
  p.pc_off = (int64_t)(need / sizeof(float)) - 4 * (int64_t)p.pc_n;
  p.dp_slice = (int64_t)kap_max * nbp;
  return true;
}

inline int fast_launch(FastArgs a, const FastPlan& p, void* ws, cudaStream_t st) {
  char* w = static_cast<char*>(ws);
  a.sl = p.sl;
  a.xl = p.xl;
  a.n_jobs = p.n_jobs;
  a.dp_slice = p.dp_slice;
  a.rch = p.rch;
  a.pc_off = p.pc_off;
  a.l0_smem = p.l0_smem;
  a.pc_n = p.pc_n;
  a.xch = reinterpret_cast<float*>(w);
  w += align_up((size_t)p.xl.total * sizeof(float), 256);
  a.meta = reinterpret_cast<int64_t*>(w);
  w += align_up((size_t)a.B * 8, 256);
  a.yhat_buf = reinterpret_cast<float*>(w);
  w += align_up((size_t)a.B * sizeof(float), 256);
  a.lossp = reinterpret_cast<float*>(w);
  w += align_up((size_t)a.B * 2 * sizeof(float), 256);
  a.scache = a.wcache = nullptr;
  if (a.B > fast_grid()) {
    a.scache = reinterpret_cast<float*>(w);
    w += align_up((size_t)a.B * (p.sl.red - p.sl.x0) * sizeof(float), 256);
    a.wcache = reinterpret_cast<float*>(w);
    w += align_up((size_t)fast_grid() * fast_attn_floats(a.dm) * sizeof(float), 256);
  }
  a.ctr = reinterpret_cast<unsigned int*>(w);
  TT_CUDA(cudaMemsetAsync(a.ctr, 0, 256, st));
  auto kern = tuner_train_fast_kernel;
  int per_sm = 0;
  if (int rc = kernel_occupancy((const void*)kern, kThreads, p.smem, &per_sm)) return rc;
  TT_REQUIRE(per_sm >= 1, "tuner train (fast): kernel cannot be resident (smem %zu)", p.smem);
  const int grid = fast_grid();
  void* args[] = {&a};
  TT_CUDA(cudaLaunchCooperativeKernel((void*)kern, grid, kThreads, args, p.smem, st));
  return check_launch("tuner train (fast)");
}

}  // namespace tt
