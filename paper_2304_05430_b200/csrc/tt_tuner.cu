// Attention tuner kernels: bulk scoring (K5) and the fused training step
// (K5 cached forward + K7 loss + K6 backward + deterministic reduction + K8
// Adam) -- see tt_tuner.cuh / tt_tuner_train.cuh for the per-block code.
#include <cstring>
#include <type_traits>

#include "tt_tuner_fast.cuh"

namespace tt {

static int g_train_path = 0;  // 0 auto, 1 generic kernel only, 2 fast kernel only (tests)

#ifndef TT_SCORE_P32
#define TT_SCORE_P32 8
#endif
template <typename R>
struct ScoreP {
  static constexpr int value = sizeof(R) == 4 ? TT_SCORE_P32 : 4;  // programs per CTA tile
};

// ----------------------------------------------------------- scoring --
template <typename R, int P>
static size_t score_smem_bytes(const TDims& d) {
  const size_t n = (size_t)2 * P * d.H + (size_t)2 * P * d.G +
                   (size_t)3 * P * d.D + (size_t)P * d.heads * d.Tmax + (size_t)P * (d.D + d.C) +
                   (size_t)P * kHeadHidden + kThreads + P + 8 +
                   (size_t)P * d.Tmax * d.D + 4;  // + the staged layer-input rows
  return n * sizeof(R) + 64;
}

template <typename R, int H, int P>
// CTAs per SM the scorer is compiled for: 3 for fp32 (80 registers, a few
// hundred bytes of spills, but 24 warps per SM to hide the recurrence's
// latency: 11.9 -> 14.0 M programs/s on the box; 1, 2 and 4 CTAs and tiles
// of 4 / 16 programs measured slower), 2 for the fp64 parity build
#ifndef TT_PRED_MINB
#define TT_PRED_MINB (sizeof(R) == 4 ? 3 : 2)
#endif
__global__ void __launch_bounds__(kThreads, TT_PRED_MINB) tuner_predict_kernel(
    TDims dm, const R* __restrict__ prm, const R* __restrict__ steps,
    const int64_t* __restrict__ rowoff, const R* __restrict__ ctx, int64_t n,
    R* __restrict__ yhat, R* __restrict__ scratch, int64_t slot_elems, R* __restrict__ s_out) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ TileInfo<R, P> ti;
  constexpr int D = 2 * H, G = 4 * H;
  R* sp = reinterpret_cast<R*>(smem_raw);
  R* sh_h = sp;
  sp += 2 * P * H;
  R* sh_g = sp;
  sp += 2 * P * G;
  AttnSmem<R, P> am;
  am.pool = sp;
  sp += P * D;
  am.q = sp;
  sp += P * D;
  am.mix = sp;
  sp += P * D;
  am.alpha = sp;
  sp += (int64_t)P * dm.heads * dm.Tmax;
  am.z = sp;
  sp += P * (D + dm.C);
  am.a1 = sp;
  sp += P * kHeadHidden;
  am.red = sp;
  sp += kThreads;
  R* sh_y = sp;
  sp += P + 8;
  // layer-input rows of the tile, staged from the L2 scratch per layer (16-B aligned)
  R* xin_s = sp + ((16 - (reinterpret_cast<uintptr_t>(sp) & 15)) & 15) / sizeof(R);
  const AttnW<R> aw = attn_global_view<R>(dm, prm);
  const int64_t TD = (int64_t)dm.Tmax * D;
  R* buf[3];
  buf[0] = scratch + (int64_t)blockIdx.x * slot_elems;
  buf[1] = buf[0] + P * TD;
  buf[2] = buf[1] + P * TD;
  const int64_t n_tiles = (n + P - 1) / P;
  for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    if (threadIdx.x < P) {
      const int64_t p = tile * P + threadIdx.x;
      if (p < n) {
        const int64_t r0 = rowoff[p];
        ti.len[threadIdx.x] = (int)(rowoff[p + 1] - r0);
        ti.step0[threadIdx.x] = steps + r0 * dm.d0;
        ti.ctx[threadIdx.x] = ctx + p * dm.C;
        ti.prog[threadIdx.x] = p;
      } else {
        ti.len[threadIdx.x] = 0;
        ti.step0[threadIdx.x] = steps;
        ti.ctx[threadIdx.x] = ctx;
        ti.prog[threadIdx.x] = -1;
      }
    }
    __syncthreads();
    int cur = 0;
    for (int l = 0; l < dm.L; ++l) {
      lstm_layer_fwd<R, H, P, false>(dm, prm, l, ti, buf[cur ^ 1], buf[cur], sh_h, sh_g,
                                     buf[2] + P * TD, nullptr, nullptr, nullptr, xin_s);
      __syncthreads();
      cur ^= 1;
    }
    if (s_out) {  // last-layer outputs in the CSR row layout (heads-only training cache)
      const R* so = buf[cur ^ 1];
      for (int pp = 0; pp < P; ++pp) {
        const int64_t prog = ti.prog[pp];
        if (prog < 0) continue;
        const int64_t r0 = rowoff[prog];
        const int len = ti.len[pp];
        for (int i = threadIdx.x; i < len * D; i += kThreads)
          s_out[(r0 + i / D) * D + i % D] = so[((int64_t)pp * dm.Tmax + i / D) * D + i % D];
      }
    }
    // final layer output buf[cur ^ 1] -> shared memory (pooling and the K / V
    // projection read it); K -> buf[cur], V -> buf[2]
    stage_rows_cta(buf[cur ^ 1], xin_s, (int)(P * TD * sizeof(R) / 16));
    attention_head_fwd<R, H, P, false>(dm, aw, ti, xin_s, buf[cur], buf[2], am, nullptr, sh_y);
    if (threadIdx.x < P && ti.prog[threadIdx.x] >= 0) yhat[ti.prog[threadIdx.x]] = sh_y[threadIdx.x];
    __syncthreads();
  }
}

// ----------------------------------------------------------- training --
template <typename R>
struct TrainArgs {
  TDims dm;
  TrainLayout ly;
  R* prm;
  R* m;
  R* v;
  const R* steps;
  const int64_t* rowoff;
  const R* ctx;
  const R* y;
  const int32_t* order;
  int64_t n_order;
  int B;
  int loss_kind;
  int mode;
  int n_steps;
  AdamHyper hyp;
  const double* corr;
  const uint8_t* trainable;
  R* step_loss;
  R* grad_out;
  int32_t* status;
  R* partial;          // [nsample_ctas][NP]
  R* sample_scratch;   // [nsample_ctas][spc][sample_elems]
  int spc;
  R* bwd_scratch;      // [nsample_ctas][bwd_elems]
  R* batch_yhat;       // [B]
  R* lb;               // [3][B] loss staging (labels, scores, d/dscore) -- per CTA
  unsigned int* barrier;
  int cache_smem;      // per-sample caches + backward scratch live in shared memory
};

template <typename R>
static size_t train_smem_bytes(const TDims& d) {
  const int NQ = 128 / d.H;
  const int64_t wreg = std::max<int64_t>(attn_stage_elems(d), lstm_stage_elems(d));
  const size_t n = (size_t)wreg + 2 * d.H + 2 * d.G + 3 * d.D + d.heads * d.Tmax + d.D + d.C +
                   kHeadHidden + kThreads + 4 + kHeadHidden + 3 * d.D + d.heads * d.Tmax +
                   2 * d.G + 2 * NQ * d.H + 8;
  return n * sizeof(R) + 64;
}

template <typename R, int H>
__global__ void __launch_bounds__(kThreads, 1) tuner_train_kernel(TrainArgs<R> a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ TileInfo<R, 1> ti;
  __shared__ int s_stop;
  constexpr int D = 2 * H, G = 4 * H, NQ = 128 / H;
  const TDims& dm = a.dm;
  const TrainLayout& ly = a.ly;
  const int tid = threadIdx.x;
  // ---- shared memory carve-up
  R* sp = reinterpret_cast<R*>(smem_raw);
  R* wst = sp;  // staged weights (attention/head, then per-layer LSTM)
  sp += std::max<int64_t>(attn_stage_elems(dm), lstm_stage_elems(dm));
  R* sh_h = sp;
  sp += 2 * H;
  R* sh_g = sp;
  sp += 2 * G;
  R* red = sp;
  sp += kThreads;
  AttnSmem<R, 1> am;
  am.pool = sp;
  sp += D;
  am.q = sp;
  sp += D;
  am.mix = sp;
  sp += D;
  am.alpha = sp;
  sp += dm.heads * dm.Tmax;
  am.z = sp;
  sp += D + dm.C;
  am.a1 = sp;
  sp += kHeadHidden;
  am.red = red;
  R* sh_y = sp;
  sp += 4;
  BwdSmem<R> bm;
  bm.da1 = sp;
  sp += kHeadHidden;
  bm.dpool = sp;
  sp += D;
  bm.dmix = sp;
  sp += D;
  bm.dq = sp;
  sp += D;
  bm.dlog = sp;
  sp += dm.heads * dm.Tmax;
  bm.dz = sp;
  sp += 2 * G;
  bm.part = sp;
  sp += 2 * NQ * H;
  bm.red = red;
  // Per-sample forward caches and the backward scratch: shared memory when
  // they fit (the grid barrier's acquire invalidates L1, so global-memory
  // caches would come back from L2 on every dependent BPTT access).
  sp = reinterpret_cast<R*>((reinterpret_cast<uintptr_t>(sp) + 31) & ~uintptr_t(31));
  R* const cache_base = a.cache_smem ? sp
                                     : a.sample_scratch + (int64_t)blockIdx.x * a.spc * ly.sample_elems;

  const int64_t NP = dm.total;
  const bool sampler = blockIdx.x < (unsigned)min((int)gridDim.x, a.B);
  const int nsamp_ctas = min((int)gridDim.x, a.B);
  R* part = a.partial + (int64_t)blockIdx.x * NP;
  R* bws = a.cache_smem ? sp + (int64_t)a.spc * ly.sample_elems
                        : a.bwd_scratch + (int64_t)blockIdx.x * ly.bwd_elems;
  // minibatch loss staging: shared memory for the usual small batches
  constexpr int kLossSmem = 256;
  __shared__ R s_lb[3 * kLossSmem];
  R* lb_y = a.B <= kLossSmem ? s_lb : a.lb + (int64_t)blockIdx.x * 3 * a.B;
  R* lb_s = lb_y + a.B;
  R* lb_d = lb_s + a.B;
  unsigned int bar_target = 0;
  const int64_t TD = (int64_t)dm.Tmax * D;

  for (int step = 0; step < a.n_steps; ++step) {
    const int64_t b0 = (int64_t)step * a.B;
    const int bn = (int)(a.n_order - b0 < (int64_t)a.B ? a.n_order - b0 : (int64_t)a.B);
    AttnW<R> aw{};
    phase_mark(step, 0);
    if (sampler && (int)blockIdx.x < bn) {
      // labels of the whole minibatch, fetched early (used after the barrier)
      for (int k = tid; k < bn; k += kThreads) lb_y[k] = a.y[a.order[b0 + k]];
      aw = stage_attn<R, D>(dm, a.prm, wst);
    }
    phase_mark(step, 1);
    // ---- forward with caches for this CTA's samples
    int slot = 0;
    for (int k = blockIdx.x; k < bn; k += gridDim.x, ++slot) {
      const int64_t idx = a.order[b0 + k];
      R* smp = cache_base + (int64_t)slot * ly.sample_elems;
      if (tid == 0) {
        const int64_t r0 = a.rowoff[idx];
        ti.len[0] = (int)(a.rowoff[idx + 1] - r0);
        ti.step0[0] = a.steps + r0 * dm.d0;
        ti.ctx[0] = a.ctx + idx * dm.C;
        ti.prog[0] = idx;
      }
      __syncthreads();
      for (int l = 0; l < dm.L; ++l) {
        lstm_layer_fwd<R, H, 1, true>(dm, a.prm, l, ti, smp + ly.S + (int64_t)(l - 1) * TD,
                                      smp + ly.S + (int64_t)l * TD, sh_h, sh_g, bws + ly.xz,
                                      smp + ly.gates + (int64_t)l * 2 * dm.Tmax * G,
                                      smp + ly.cst + (int64_t)l * 2 * dm.Tmax * H,
                                      smp + ly.tcs + (int64_t)l * 2 * dm.Tmax * H);
        __syncthreads();
        phase_mark(step, 2 + l);
      }
      AttnCache<R> cache{smp + ly.pin, smp + ly.q,  smp + ly.alpha, smp + ly.mix,
                         smp + ly.z,   smp + ly.a1, smp + ly.yhat};
      attention_head_fwd<R, H, 1, true>(dm, aw, ti, smp + ly.S + (int64_t)(dm.L - 1) * TD,
                                        smp + ly.K, smp + ly.V, am, &cache, sh_y);
      if (tid == 0) a.batch_yhat[k] = sh_y[0];
      __syncthreads();
      phase_mark(step, 5);
    }
    grid_barrier(a.barrier, bar_target);
    phase_mark(step, 6);
    if (sampler && (int)blockIdx.x < bn) {
      // ---- loss over the whole minibatch (every sampling CTA, identical arithmetic)
      for (int k = tid; k < bn; k += kThreads) lb_s[k] = __ldcg(a.batch_yhat + k);
      __syncthreads();
      const R loss = a.loss_kind == TT_LOSS_RANK ? rank_loss_block<R>(lb_y, lb_s, bn, lb_d, red)
                                                 : mse_block<R>(lb_y, lb_s, bn, lb_d, red);
      if (tid == 0) {
        s_stop = !isfinite((double)loss);
        if (blockIdx.x == 0) {
          a.step_loss[step] = loss;
          if (s_stop) a.status[0] = step;
        }
      }
      __syncthreads();
      phase_mark(step, 7);
      // ---- backward for this CTA's samples into its partial gradient
      if (!s_stop) {
        slot = 0;
        for (int k = blockIdx.x; k < bn; k += gridDim.x, ++slot) {
          const int64_t idx = a.order[b0 + k];
          const R* smp = cache_base + (int64_t)slot * ly.sample_elems;
          const int64_t r0 = a.rowoff[idx];
          const int len = (int)(a.rowoff[idx + 1] - r0);
          if (slot > 0) aw = stage_attn<R, D>(dm, a.prm, wst);  // LSTM staging overwrote it
          backward_sample<R, H>(dm, ly, a.prm, aw, len, a.steps + r0 * dm.d0, lb_d[k], smp, bws,
                                bm, wst, part, slot == 0, step);
        }
      }
    }
    phase_mark(step, 16);
    grid_barrier(a.barrier, bar_target);
    phase_mark(step, 17);
    // every CTA reads the stop flag published by CTA 0 (status) -- uniform exit
    if (__ldcg(a.status) >= 0) break;
    // ---- deterministic fixed-order reduction + fused Adam (or gradient out), all CTAs
    const int nact = min(nsamp_ctas, bn);
    const double c1 = a.mode == TT_MODE_TRAIN ? a.corr[2 * step] : 1.0;
    const double c2 = a.mode == TT_MODE_TRAIN ? a.corr[2 * step + 1] : 1.0;
    for (int64_t p = (int64_t)blockIdx.x * kThreads + tid; p < NP; p += (int64_t)gridDim.x * kThreads) {
      R g = 0;
      for (int c = 0; c < nact; ++c) g += __ldcg(a.partial + (int64_t)c * NP + p);
      if (a.mode == TT_MODE_GRAD) {
        a.grad_out[p] = g;
      } else if (!a.trainable || a.trainable[p]) {
        R pp = __ldcg(a.prm + p), mm = a.m[p], vv = a.v[p];
        adam_update<R>(pp, g, mm, vv, a.hyp, c1, c2);
        a.prm[p] = pp;
        a.m[p] = mm;
        a.v[p] = vv;
      }
    }
    phase_mark(step, 18);
    grid_barrier(a.barrier, bar_target);
    phase_mark(step, 19);
  }
}

// ------------------------------------------------------------- dispatch --
// bound on one wait for a peer's gradient slice (tt_tuner_dp_set_timeout_ms)
static long long g_dp_timeout_ns = 30LL * 1000000000LL;

struct DpArgs {
  int world, rank;
  int64_t gbase;
  void* const* xb;
};

template <typename R>
struct Launch {
  // Small batches (search-time scoring: one candidate per annealing step,
  // <= 32 per evolution generation, search.py:319, :392-410) use one program
  // per CTA: a tile walks its programs one after another inside each time
  // step, so the latency grows with the programs per tile, while a small
  // batch cannot fill the GPU anyway.
  template <int H>
  static int predict_h(const TDims& dm, const R* prm, const R* steps, const int64_t* rowoff,
                       const R* ctx, int64_t n, R* yhat, void* ws, size_t ws_bytes,
                       cudaStream_t st, R* s_out) {
    if (n <= (int64_t)sm_count())
      return predict_hp<H, 1>(dm, prm, steps, rowoff, ctx, n, yhat, ws, ws_bytes, st, s_out);
    return predict_hp<H, ScoreP<R>::value>(dm, prm, steps, rowoff, ctx, n, yhat, ws, ws_bytes, st,
                                           s_out);
  }

  template <int H, int P>
  static int predict_hp(const TDims& dm, const R* prm, const R* steps, const int64_t* rowoff,
                        const R* ctx, int64_t n, R* yhat, void* ws, size_t ws_bytes,
                        cudaStream_t st, R* s_out) {
    const int64_t slot = (int64_t)3 * P * dm.Tmax * dm.D + (int64_t)2 * P * dm.Tmax * dm.G;
    const size_t smem = score_smem_bytes<R, P>(dm);
    auto kern = tuner_predict_kernel<R, H, P>;
    int per_sm = 0;
    if (int rc = kernel_occupancy((const void*)kern, kThreads, smem, &per_sm)) return rc;
    TT_REQUIRE(per_sm >= 1, "tuner predict: kernel cannot be resident (smem %zu)", smem);
    int grid = (int)std::min<int64_t>((n + P - 1) / P, (int64_t)sm_count() * per_sm);
    const size_t need = (size_t)grid * slot * sizeof(R);
    if (ws_bytes < need) {
      grid = (int)(ws_bytes / (slot * sizeof(R)));
      TT_REQUIRE(grid >= 1, "tuner predict: workspace too small");
    }
    kern<<<grid, kThreads, smem, st>>>(dm, prm, steps, rowoff, ctx, n, yhat,
                                       static_cast<R*>(ws), slot, s_out);
    return check_launch("tuner predict");
  }

  static int predict(const TDims& dm, const R* prm, const R* steps, const int64_t* rowoff,
                     const R* ctx, int64_t n, R* yhat, void* ws, size_t ws_bytes,
                     cudaStream_t st, R* s_out = nullptr) {
    switch (dm.H) {
      case 4: return predict_h<4>(dm, prm, steps, rowoff, ctx, n, yhat, ws, ws_bytes, st, s_out);
      case 8: return predict_h<8>(dm, prm, steps, rowoff, ctx, n, yhat, ws, ws_bytes, st, s_out);
      case 16: return predict_h<16>(dm, prm, steps, rowoff, ctx, n, yhat, ws, ws_bytes, st, s_out);
      case 32: return predict_h<32>(dm, prm, steps, rowoff, ctx, n, yhat, ws, ws_bytes, st, s_out);
    }
    set_error("tuner: hidden size %d unsupported (4, 8, 16, 32)", dm.H);
    return TT_EINVAL;
  }

  static int grid_for(int B) {
    (void)B;
    return sm_count();  // sampling CTAs = min(grid, B); all CTAs reduce + update
  }

  static size_t train_ws(const TDims& dm, int B) {
    const TrainLayout ly = make_train_layout(dm);
    const int grid = grid_for(B);
    const int ns = std::min(grid, B);
    const int spc = (B + ns - 1) / ns;
    size_t b = 0;
    b += align_up((size_t)ns * dm.total * sizeof(R), 256);
    b += align_up((size_t)ns * spc * ly.sample_elems * sizeof(R), 256);
    b += align_up((size_t)ns * ly.bwd_elems * sizeof(R), 256);
    b += align_up((size_t)B * sizeof(R), 256);
    b += align_up((size_t)grid * 3 * B * sizeof(R), 256);
    b += 256;
    return b;
  }

  template <int H>
  static int train_h(TrainArgs<R> a, void* ws, size_t ws_bytes, cudaStream_t st) {
    const int grid = grid_for(a.B);
    const int ns = std::min(grid, a.B);
    a.spc = (a.B + ns - 1) / ns;
    char* w = static_cast<char*>(ws);
    TT_REQUIRE(ws_bytes >= train_ws(a.dm, a.B), "tuner train: workspace %zu < %zu", ws_bytes,
               train_ws(a.dm, a.B));
    a.partial = reinterpret_cast<R*>(w);
    w += align_up((size_t)ns * a.dm.total * sizeof(R), 256);
    a.sample_scratch = reinterpret_cast<R*>(w);
    w += align_up((size_t)ns * a.spc * a.ly.sample_elems * sizeof(R), 256);
    a.bwd_scratch = reinterpret_cast<R*>(w);
    w += align_up((size_t)ns * a.ly.bwd_elems * sizeof(R), 256);
    a.batch_yhat = reinterpret_cast<R*>(w);
    w += align_up((size_t)a.B * sizeof(R), 256);
    a.lb = reinterpret_cast<R*>(w);
    w += align_up((size_t)grid * 3 * a.B * sizeof(R), 256);
    a.barrier = reinterpret_cast<unsigned int*>(w);
    TT_CUDA(cudaMemsetAsync(a.barrier, 0, 256, st));
    size_t smem = train_smem_bytes<R>(a.dm);
    {
      int dev = 0, optin = 0;
      TT_CUDA(cudaGetDevice(&dev));
      TT_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
      const size_t cache = ((size_t)a.spc * a.ly.sample_elems + a.ly.bwd_elems) * sizeof(R) + 64;
      const size_t static_smem = 3 * 256 * sizeof(R) + 1024;  // s_lb, TileInfo, flags
      a.cache_smem = smem + cache + static_smem <= (size_t)optin ? 1 : 0;
      if (a.cache_smem) smem += cache;
    }
    auto kern = tuner_train_kernel<R, H>;
    int per_sm = 0;
    if (int rc = kernel_occupancy((const void*)kern, kThreads, smem, &per_sm)) return rc;
    TT_REQUIRE(per_sm >= 1, "tuner train: kernel cannot be resident (smem %zu)", smem);
    void* args[] = {&a};
    TT_CUDA(cudaLaunchCooperativeKernel((void*)kern, grid, kThreads, args, smem, st));
    return check_launch("tuner train");
  }

  static int train(TrainArgs<R> a, void* ws, size_t ws_bytes, cudaStream_t st,
                   const R* scache = nullptr, const DpArgs* dp = nullptr) {
    if constexpr (std::is_same<R, float>::value) {
      // v4 latency path (tt_tuner_fast.cuh) when eligible, else the generic kernel
      FastPlan fp;
      const bool ok = g_train_path != 1 && fast_plan(a.dm, a.B, fast_grid(), fp) &&
                      ws_bytes >= fast_ws_bytes(a.dm, a.B);
      if (ok) {
        FastArgs f{};
        f.dm = a.dm;
        f.prm = a.prm;
        f.m = a.m;
        f.v = a.v;
        f.steps = a.steps;
        f.rowoff = a.rowoff;
        f.ctx = a.ctx;
        f.y = a.y;
        f.order = a.order;
        f.n_order = a.n_order;
        f.B = a.B;
        f.loss_kind = a.loss_kind;
        f.mode = a.mode;
        f.n_steps = a.n_steps;
        f.hyp = a.hyp;
        f.corr = a.corr;
        f.trainable = a.trainable;
        f.step_loss = a.step_loss;
        f.grad_out = a.grad_out;
        f.status = a.status;
        f.s_frozen = scache;
        f.world = 1;
        if (dp) {
          f.world = dp->world;
          f.rank = dp->rank;
          f.gbase = dp->gbase;
          f.xb = dp->xb;
          f.dp_timeout_ns = g_dp_timeout_ns;
        }
        return fast_launch(f, fp, ws, st);
      }
      TT_REQUIRE(dp == nullptr, "tuner train (data parallel): not eligible for the latency-path kernel");
      TT_REQUIRE(g_train_path != 2, "tuner train: fast path requested but not eligible");
      TT_REQUIRE(scache == nullptr, "tuner train (heads only): not eligible for the latency-path kernel");
    }
    switch (a.dm.H) {
      case 4: return train_h<4>(a, ws, ws_bytes, st);
      case 8: return train_h<8>(a, ws, ws_bytes, st);
      case 16: return train_h<16>(a, ws, ws_bytes, st);
      case 32: return train_h<32>(a, ws, ws_bytes, st);
    }
    set_error("tuner: hidden size %d unsupported (4, 8, 16, 32)", a.dm.H);
    return TT_EINVAL;
  }
};

static int check_dims(int L, int H, int heads, int U, int d0, int C, int Tmax) {
  TT_REQUIRE(L >= 1 && L <= kMaxLayers, "tuner: layers must be in [1, %d]", kMaxLayers);
  TT_REQUIRE(H == 4 || H == 8 || H == 16 || H == 32, "tuner: hidden must be 4, 8, 16 or 32");
  TT_REQUIRE(heads >= 1 && (2 * H) % heads == 0, "tuner: heads must divide 2*hidden");
  TT_REQUIRE(U >= 1, "tuner: unroll must be >= 1");
  TT_REQUIRE(d0 >= 1 && C >= 0, "tuner: bad step/context width");
  TT_REQUIRE(Tmax >= 1 && Tmax <= 4096, "tuner: max_steps out of range");
  return TT_OK;
}

template <typename R>
static int predict_entry(const R* prm, const R* steps, const int64_t* rowoff, const R* ctx,
                         int64_t n, int32_t L, int32_t H, int32_t heads, int32_t U, int32_t d0,
                         int32_t C, int32_t Tmax, R* yhat, void* ws, size_t ws_bytes,
                         tt_stream_t st, R* s_out = nullptr) {
  if (int rc = check_dims(L, H, heads, U, d0, C, Tmax)) return rc;
  TT_REQUIRE(n >= 0, "tuner predict: negative n");
  if (n == 0) return TT_OK;
  const TDims dm = make_dims(L, H, heads, U, d0, C, Tmax);
  return Launch<R>::predict(dm, prm, steps, rowoff, ctx, n, yhat, ws, ws_bytes, as_stream(st),
                            s_out);
}

template <typename R>
static int train_entry(R* prm, R* m, R* v, const R* steps, const int64_t* rowoff, const R* ctx,
                       const R* y, const int32_t* order, int64_t n_order, int32_t B,
                       int32_t loss_kind, int32_t mode, double lr, double b1, double b2,
                       double eps, const double* corr, const uint8_t* trainable, int32_t L,
                       int32_t H, int32_t heads, int32_t U, int32_t d0, int32_t C, int32_t Tmax,
                       R* step_loss, R* grad_out, int32_t* status, void* ws, size_t ws_bytes,
                       tt_stream_t st, const R* scache = nullptr, const DpArgs* dp = nullptr) {
  if (int rc = check_dims(L, H, heads, U, d0, C, Tmax)) return rc;
  TT_REQUIRE(B >= 1 && B <= 4096, "tuner train: batch size must be in [1, 4096]");
  TT_REQUIRE(n_order >= 1, "tuner train: empty order");
  TT_REQUIRE(mode == TT_MODE_TRAIN || mode == TT_MODE_GRAD, "tuner train: bad mode");
  TT_REQUIRE(loss_kind == TT_LOSS_MSE || loss_kind == TT_LOSS_RANK, "tuner train: bad loss");
  TT_REQUIRE(mode == TT_MODE_GRAD || corr != nullptr, "tuner train: corr required");
  TT_REQUIRE(status != nullptr, "tuner train: status required");
  if (mode == TT_MODE_GRAD) TT_REQUIRE(n_order <= B, "tuner grad: one minibatch only");
  TrainArgs<R> a{};
  a.dm = make_dims(L, H, heads, U, d0, C, Tmax);
  a.ly = make_train_layout(a.dm);
  a.prm = prm;
  a.m = m;
  a.v = v;
  a.steps = steps;
  a.rowoff = rowoff;
  a.ctx = ctx;
  a.y = y;
  a.order = order;
  a.n_order = n_order;
  a.B = B;
  a.loss_kind = loss_kind;
  a.mode = mode;
  a.n_steps = (int)((n_order + B - 1) / B);
  a.hyp = AdamHyper{lr, b1, b2, eps};
  a.corr = corr;
  a.trainable = trainable;
  a.step_loss = step_loss;
  a.grad_out = grad_out;
  a.status = status;
  return Launch<R>::train(a, ws, ws_bytes, as_stream(st), scache, dp);
}

}  // namespace tt

using namespace tt;

extern "C" {

int64_t tt_tuner_param_count(int32_t L, int32_t H, int32_t d0, int32_t C) {
  if (L < 1 || L > kMaxLayers) return -1;
  return make_dims(L, H, 1, 1, d0, C, 1).total;
}

size_t tt_tuner_predict_workspace_bytes(int32_t f64, int32_t L, int32_t H, int32_t Tmax) {
  (void)L;
  const size_t es = f64 ? 8 : 4;
  const int P = f64 ? ScoreP<double>::value : ScoreP<float>::value;
  const size_t slot = (size_t)3 * P * Tmax * 2 * H + (size_t)2 * P * Tmax * 4 * H;
  return (size_t)sm_count() * 3 * slot * es;
}

int tt_tuner_predict_f32(const float* prm, const float* steps, const int64_t* rowoff,
                         const float* ctx, int64_t n, int32_t L, int32_t H, int32_t heads,
                         int32_t U, int32_t d0, int32_t C, int32_t Tmax, float* yhat, void* ws,
                         size_t ws_bytes, tt_stream_t st) {
  return predict_entry<float>(prm, steps, rowoff, ctx, n, L, H, heads, U, d0, C, Tmax, yhat, ws,
                              ws_bytes, st);
}

int tt_tuner_predict_f64(const double* prm, const double* steps, const int64_t* rowoff,
                         const double* ctx, int64_t n, int32_t L, int32_t H, int32_t heads,
                         int32_t U, int32_t d0, int32_t C, int32_t Tmax, double* yhat, void* ws,
                         size_t ws_bytes, tt_stream_t st) {
  return predict_entry<double>(prm, steps, rowoff, ctx, n, L, H, heads, U, d0, C, Tmax, yhat, ws,
                               ws_bytes, st);
}

size_t tt_tuner_train_workspace_bytes(int32_t f64, int32_t L, int32_t H, int32_t d0, int32_t C,
                                      int32_t Tmax, int32_t B) {
  if (L < 1 || L > kMaxLayers || B < 1) return 0;
  TDims big = make_dims(L, H, 2, 2, d0, C, Tmax);
  // heads/unroll only size small cache segments; use generous upper bounds
  big.heads = 2 * H;
  big.U = 16;
  if (f64) return Launch<double>::train_ws(big, B);
  return std::max(Launch<float>::train_ws(big, B), fast_ws_bytes(big, B));
}

int tt_tuner_train_f32(float* prm, float* m, float* v, const float* steps, const int64_t* rowoff,
                       const float* ctx, const float* y, const int32_t* order, int64_t n_order,
                       int32_t B, int32_t loss_kind, int32_t mode, double lr, double b1,
                       double b2, double eps, const double* corr, const uint8_t* trainable,
                       int32_t L, int32_t H, int32_t heads, int32_t U, int32_t d0, int32_t C,
                       int32_t Tmax, float* step_loss, float* grad_out, int32_t* status, void* ws,
                       size_t ws_bytes, tt_stream_t st) {
  return train_entry<float>(prm, m, v, steps, rowoff, ctx, y, order, n_order, B, loss_kind, mode,
                            lr, b1, b2, eps, corr, trainable, L, H, heads, U, d0, C, Tmax,
                            step_loss, grad_out, status, ws, ws_bytes, st);
}

int tt_tuner_lstm_outputs_f32(const float* prm, const float* steps, const int64_t* rowoff,
                              const float* ctx, int64_t n, int32_t L, int32_t H, int32_t heads,
                              int32_t U, int32_t d0, int32_t C, int32_t Tmax, float* s_out,
                              float* yhat, void* ws, size_t ws_bytes, tt_stream_t st) {
  TT_REQUIRE(s_out != nullptr && yhat != nullptr, "tuner lstm outputs: null output");
  return predict_entry<float>(prm, steps, rowoff, ctx, n, L, H, heads, U, d0, C, Tmax, yhat, ws,
                              ws_bytes, st, s_out);
}

int tt_tuner_train_heads_f32(float* prm, float* m, float* v, const float* steps,
                             const int64_t* rowoff, const float* ctx, const float* y,
                             const int32_t* order, int64_t n_order, int32_t B, int32_t loss_kind,
                             double lr, double b1, double b2, double eps, const double* corr,
                             const uint8_t* trainable, int32_t L, int32_t H, int32_t heads,
                             int32_t U, int32_t d0, int32_t C, int32_t Tmax,
                             const float* s_cache, float* step_loss, int32_t* status, void* ws,
                             size_t ws_bytes, tt_stream_t st) {
  TT_REQUIRE(s_cache != nullptr, "tuner train (heads only): s_cache required");
  return train_entry<float>(prm, m, v, steps, rowoff, ctx, y, order, n_order, B, loss_kind,
                            TT_MODE_TRAIN, lr, b1, b2, eps, corr, trainable, L, H, heads, U, d0, C,
                            Tmax, step_loss, nullptr, status, ws, ws_bytes, st, s_cache);
}

size_t tt_tuner_dp_buffer_bytes(int32_t L, int32_t H, int32_t d0, int32_t C, int32_t world) {
  if (L < 1 || L > kMaxLayers || H != kFH || world < 1) return 0;
  const TDims dm = make_dims(L, H, 1, 1, d0, C, 1);
  const int kap_max = std::max(round4(round4(std::max(d0, kFD)) + kFH + 1), round4(round4(kFD + C) + 1));
  return (size_t)fast_dp_buffer_bytes(fast_n_jobs(dm), world, (int64_t)kap_max * 16);
}

int tt_tuner_train_dp_f32(float* prm, float* m, float* v, const float* steps, const int64_t* rowoff,
                          const float* ctx, const float* y, const int32_t* order, int64_t n_order,
                          int32_t B, int32_t loss_kind, double lr, double b1, double b2, double eps,
                          const double* corr, const uint8_t* trainable, int32_t L, int32_t H,
                          int32_t heads, int32_t U, int32_t d0, int32_t C, int32_t Tmax,
                          int32_t world, int32_t rank, int64_t gbase, void* const* d_xb,
                          float* step_loss, int32_t* status, void* ws, size_t ws_bytes,
                          tt_stream_t st) {
  TT_REQUIRE(world >= 1 && rank >= 0 && rank < world, "tuner train (dp): bad world/rank");
  TT_REQUIRE(world == 1 || d_xb != nullptr, "tuner train (dp): exchange buffers required");
  TT_REQUIRE(gbase >= 0, "tuner train (dp): bad step base");
  DpArgs dp{world, rank, gbase, d_xb};
  return train_entry<float>(prm, m, v, steps, rowoff, ctx, y, order, n_order, B, loss_kind,
                            TT_MODE_TRAIN, lr, b1, b2, eps, corr, trainable, L, H, heads, U, d0, C,
                            Tmax, step_loss, nullptr, status, ws, ws_bytes, st, nullptr,
                            world > 1 ? &dp : nullptr);
}

int tt_ipc_alloc(size_t bytes, void** d_ptr, uint8_t* h_handle) {
  TT_REQUIRE(d_ptr != nullptr && h_handle != nullptr && bytes > 0, "ipc alloc: bad arguments");
  void* p = nullptr;
  TT_CUDA(cudaMalloc(&p, bytes));
  TT_CUDA(cudaMemset(p, 0, bytes));
  cudaIpcMemHandle_t h;
  TT_CUDA(cudaIpcGetMemHandle(&h, p));
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
  memcpy(h_handle, &h, sizeof(h));
  *d_ptr = p;
  return TT_OK;
}

int tt_ipc_open(const uint8_t* h_handle, void** d_ptr) {
  TT_REQUIRE(d_ptr != nullptr && h_handle != nullptr, "ipc open: bad arguments");
  cudaIpcMemHandle_t h;
  memcpy(&h, h_handle, sizeof(h));
  TT_CUDA(cudaIpcOpenMemHandle(d_ptr, h, cudaIpcMemLazyEnablePeerAccess));
  return TT_OK;
}

int tt_ipc_close(void* d_ptr) {
  TT_CUDA(cudaIpcCloseMemHandle(d_ptr));
  return TT_OK;
}

int tt_dev_free(void* d_ptr) {
  TT_CUDA(cudaFree(d_ptr));
  return TT_OK;
}

int32_t tt_tuner_train_fast_eligible(int32_t L, int32_t H, int32_t heads, int32_t U, int32_t d0,
                                     int32_t C, int32_t Tmax, int32_t B) {
  if (check_dims(L, H, heads, U, d0, C, Tmax) != TT_OK) return 0;
  FastPlan fp;
  return fast_plan(make_dims(L, H, heads, U, d0, C, Tmax), B, fast_grid(), fp) ? 1 : 0;
}

int tt_tuner_dp_set_timeout_ms(int64_t ms) {
  TT_REQUIRE(ms >= 1, "dp timeout must be >= 1 ms");
  g_dp_timeout_ns = ms * 1000000LL;
  return TT_OK;
}

int tt_tuner_train_set_grid(int32_t grid) {
  TT_REQUIRE(grid >= 0, "grid must be >= 0");
  g_fast_grid = grid;
  return TT_OK;
}

int tt_tuner_train_set_path(int32_t path) {
  TT_REQUIRE(path >= 0 && path <= 2, "train path must be 0 (auto), 1 (generic) or 2 (fast)");
  g_train_path = path;
  return TT_OK;
}

int tt_debug_profile_step(int32_t step) {
  TT_CUDA(cudaMemcpyToSymbol(g_prof_step, &step, sizeof(int)));
  return TT_OK;
}

int tt_debug_phase_times(int64_t* out, int32_t n) {
  TT_REQUIRE(n >= 0 && n <= 32, "debug: n must be in [0, 32]");
  TT_CUDA(cudaMemcpyFromSymbol(out, g_phase, sizeof(long long) * n));
  return TT_OK;
}

int tt_tuner_train_f64(double* prm, double* m, double* v, const double* steps,
                       const int64_t* rowoff, const double* ctx, const double* y,
                       const int32_t* order, int64_t n_order, int32_t B, int32_t loss_kind,
                       int32_t mode, double lr, double b1, double b2, double eps,
                       const double* corr, const uint8_t* trainable, int32_t L, int32_t H,
                       int32_t heads, int32_t U, int32_t d0, int32_t C, int32_t Tmax,
                       double* step_loss, double* grad_out, int32_t* status, void* ws,
                       size_t ws_bytes, tt_stream_t st) {
  return train_entry<double>(prm, m, v, steps, rowoff, ctx, y, order, n_order, B, loss_kind, mode,
                             lr, b1, b2, eps, corr, trainable, L, H, heads, U, d0, C, Tmax,
                             step_loss, grad_out, status, ws, ws_bytes, st);
}

}  // extern "C"
