// K5 at fp32 accuracy on the 5th-generation tensor cores: attention-tuner
// scoring (tuner.py _forward :227-285, predict :468-476) with the biLSTM
// stack as split-precision tcgen05 GEMMs, then attention + head on the CUDA
// cores (tt_tuner.cu, the strict-fp32 code).
//
// kind::tf32 truncates fp32 operands to 10 mantissa bits
// (tools/tf32_rounding_probe.py), so every product is split
//   a.w = a_hi.w_hi + a_lo.w_hi + a_hi.w_lo   (+ a_lo.w_lo, ~2^-20 |a.w|, dropped)
// with x_hi = x & ~0x1fff and x_lo = x - x_hi (exact in fp32).  The weight
// side is pre-split into one stacked B image per (layer, direction):
//   B^T rows [0,128) = W_hi^T, rows [128,256) = W_lo^T   (K-major SWIZZLE_128B)
// so a time step is one N=256 MMA chain (A_hi . [W_hi | W_lo]) plus one
// N=128 chain (A_lo . W_hi) accumulating into the first half.
//
// One persistent CTA per SM, 288 threads, tiles of 128 programs:
//   warp 0        TMEM allocator (512 columns) and the single MMA-issuing lane
//   warps 1..8    two threads per program ("row threads"; TMEM lane = row),
//                 thread half hw owns hidden units [16 hw, 16 hw + 16)
// TMEM columns: G [0,256)  A_hi [256, 256+K)  A_lo [352, 352+K)  (K <= 96)
// The two directions of a layer run one after the other (one direction's
// G + A_hi + A_lo is 448 columns).  Per step the row threads read the gate
// pre-activations (G[0:128) + G[128:256) + bias), apply the Act<float>
// activations of the CUDA-core kernel, update c (registers) and h, write the
// layer output row (fp32) and the next step's A = [x_t | h] split into hi/lo.
// Programs shorter than the tile run past their end on zero inputs; those
// steps write nothing (the valid steps of both directions are a prefix).
//
// Layer outputs: the last layer lands in S = [n][Tmax][64] (fp32, padded
// per program), which the attention kernel reads; the layers before it
// alternate between the program's S rows and a per-CTA scratch tile.
#include "tt_sm100.cuh"
#include "tt_tuner.cuh"

namespace tt {

using namespace sm100;

namespace x3 {
constexpr int kRows = 128;
constexpr int kThreads = 288;
constexpr int kH = 32, kD = 64, kG = 128, kN = 256;  // kN: stacked [W_hi | W_lo]
constexpr uint32_t kColG = 0;     // G[s & 1] at 128 (s & 1)
constexpr uint32_t kColXh = 256;  // x_hi (kx <= 64 columns)
constexpr uint32_t kColXl = 320;  // x_lo
constexpr uint32_t kColHh = 384;  // h_hi (32)
constexpr uint32_t kColHl = 416;  // h_lo
// > half of the SM's shared memory: one CTA per SM (it allocates all of TMEM)
constexpr int kBBytes = 96 * 1024;
constexpr size_t kSmem = 1024 + kBBytes + 2 * kRows * 64 * sizeof(float);
constexpr int64_t kMaxChunkTilesPerSm = 4;  // programs per (LSTM, attention) launch pair / (148 x 128)
constexpr size_t kChunkBudget = 256u << 20;  // bytes of S per chunk (at least one tile)
}  // namespace x3

__host__ __device__ inline int x3_kx(int l) { return l == 0 ? 32 : 64; }
// one direction's stacked image: K/32 atoms of 256 rows x 128 B
__host__ __device__ inline uint32_t x3_image_bytes(int l) {
  return (uint32_t)((x3_kx(l) + 32) / 32) * (uint32_t)(x3::kN * 128);
}
__host__ __device__ inline int64_t x3_image_off(int l, int d) {
  int64_t o = 0;
  for (int i = 0; i < l; ++i) o += 2 * (int64_t)x3_image_bytes(i);
  return o + d * (int64_t)x3_image_bytes(l);
}

__device__ __forceinline__ float tf32_hi(float x) { return __uint_as_float(__float_as_uint(x) & 0xffffe000u); }

// [Wx ; Wh] of (layer, direction) = blockIdx.x / 2, % 2 -> stacked hi/lo B^T image.
__global__ void __launch_bounds__(256) tuner_x3_prepare_kernel(TDims dm, const float* __restrict__ prm,
                                                                unsigned char* img) {
  using namespace x3;
  const int l = blockIdx.x >> 1, d = blockIdx.x & 1;
  const int din = l == 0 ? dm.d0 : kD, kx = x3_kx(l), K = kx + kH;
  unsigned char* base = img + x3_image_off(l, d);
  const float* Wx = prm + dm.wx[l][d];
  const float* Wh = prm + dm.wh[l][d];
  for (int i = threadIdx.x; i < K * kN; i += blockDim.x) {
    const int n = i % kN, k = i / kN, c = n & (kG - 1);
    float w = 0.f;
    if (k < kx) {
      if (k < din) w = __ldg(Wx + (int64_t)k * kG + c);
    } else {
      w = __ldg(Wh + (int64_t)(k - kx) * kG + c);
    }
    const float hi = tf32_hi(w);
    *reinterpret_cast<float*>(base + (k >> 5) * (kN * 128) + sw128_offset(n, k & 31)) = n < kG ? hi : w - hi;
  }
}

struct X3Args {
  TDims dm;
  const float* prm;
  const float* steps;
  const int64_t* rowoff;
  int64_t n;
  float* S;        // [n][Tmax][64]
  float* scratch;  // per CTA [128][Tmax][64]
  const unsigned char* img;
};

struct __align__(8) X3Bars {
  uint64_t ax_full, ah_full, d_full, w_full;
  uint32_t tmem_base;
  int tmax;
};

__device__ __forceinline__ void cp_async16(float* s, const float* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(s)), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_async4(float* s, const float* g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(s)), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_async_commit_x() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait_x() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__device__ __forceinline__ void split16(const float* v, float (&hi)[16], float (&lo)[16]) {
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    hi[i] = tf32_hi(v[i]);
    lo[i] = v[i] - hi[i];
  }
}

__global__ void __launch_bounds__(x3::kThreads, 1) tuner_lstm_x3_kernel(X3Args a) {
  using namespace x3;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* Bs = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  float* xslots = reinterpret_cast<float*>(Bs + kBBytes);  // [256 row threads][2][32]
  __shared__ float sbias[kG];
  __shared__ X3Bars bars_s;
  X3Bars* bars = &bars_s;
  const TDims& dm = a.dm;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool rowt = warp >= 1;
  const int hw = (warp - 1) >> 2;            // which 16 hidden units
  const int row = ((warp & 3) << 5) | lane;  // TMEM lane quarter = warp % 4
  const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
  const int TM = dm.Tmax;
  const uint32_t bs_addr = smem_u32(Bs);

  if (threadIdx.x == 0) {
    mbar_init(&bars->ax_full, 2 * kRows);
    mbar_init(&bars->ah_full, 2 * kRows);
    mbar_init(&bars->d_full, 1);
    mbar_init(&bars->w_full, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<512>(&bars->tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bars->tmem_base;
  uint32_t pa = 0, pd = 0, pw = 0;
  float* xrow_cta = a.scratch + (int64_t)blockIdx.x * kRows * TM * kD + (int64_t)row * TM * kD;

  const int64_t n_tiles = (a.n + kRows - 1) / kRows;
  for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    const int64_t p = tile * kRows + row;
    const bool live = rowt && p < a.n;
    int64_t r0 = 0;
    int T = 0;
    if (live) {
      r0 = a.rowoff[p];
      T = (int)(a.rowoff[p + 1] - r0);
    }
    if (threadIdx.x == 0) bars->tmax = 0;
    __syncthreads();
    if (live && hw == 0) atomicMax(&bars->tmax, T);
    __syncthreads();
    const int Tt = bars->tmax;
    float* srow = a.S + (live ? p : 0) * TM * kD;

    for (int l = 0; l < dm.L; ++l) {
      const int kx = x3_kx(l);
      float* out = ((dm.L - 1 - l) & 1) == 0 ? srow : xrow_cta;
      const float* in = ((dm.L - l) & 1) == 0 ? srow : xrow_cta;  // layer l-1's output
      for (int d = 0; d < 2; ++d) {
        // ---- stacked image of (l, d) -> Bs (every MMA reading Bs has completed)
        __syncthreads();
        if (threadIdx.x == 0) {
          const uint32_t bytes = x3_image_bytes(l);
          const unsigned char* src = a.img + x3_image_off(l, d);
          mbar_expect_tx(&bars->w_full, bytes);
          for (uint32_t off = 0; off < bytes; off += 32768)
            bulk_g2s(Bs + off, src + off, bytes - off < 32768 ? bytes - off : 32768, &bars->w_full);
        }
        for (int i = threadIdx.x; i < kG; i += blockDim.x) sbias[i] = __ldg(a.prm + dm.bb[l][d] + i);
        mbar_wait(&bars->w_full, pw);
        pw ^= 1;
        __syncthreads();

        if (rowt) {
          const uint32_t Xh = tmem + lane_off + kColXh, Xl = tmem + lane_off + kColXl;
          const uint32_t Hh = tmem + lane_off + kColHh, Hl = tmem + lane_off + kColHl;
          const int xw = kx / 2;  // x columns per thread: 16 (layer 0) or 32
          // x row of step s (this thread's columns, zeros past the program's
          // end) -> shared slot s & 1 by async copies, two steps ahead
          float* slot0 = xslots + (threadIdx.x - 32) * 64;
          auto fetch_x = [&](int s) {
            float* dst = slot0 + (s & 1) * 32;
            const bool ok = live && s < T;
            const int t = d == 0 ? s : T - 1 - s;
            if (l == 0) {
              const float* xr = a.steps + (r0 + (ok ? t : 0)) * dm.d0;
              for (int i = 0; i < 16; ++i) {
                const int k = 16 * hw + i;
                float* e = dst + (((i >> 2) ^ (lane & 7)) << 2) + (i & 3);
                if (ok && k < dm.d0)
                  cp_async4(e, xr + k);
                else
                  *e = 0.f;
              }
            } else {
              const float* xr = in + (int64_t)(ok ? t : 0) * kD + 32 * hw;
#pragma unroll
              for (int q = 0; q < 8; ++q) {
                float* e = dst + ((q ^ (lane & 7)) << 2);
                if (ok)
                  cp_async16(e, xr + 4 * q);
                else
                  *reinterpret_cast<float4*>(e) = make_float4(0.f, 0.f, 0.f, 0.f);
              }
            }
            cp_async_commit_x();
          };
          auto put_x = [&](int s) {
            const float* src = slot0 + (s & 1) * 32;
#pragma unroll
            for (int j0 = 0; j0 < 32; j0 += 16) {
              if (j0 < xw) {
                float v[16], hi[16], lo[16];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                  const float4 f = *reinterpret_cast<const float4*>(src + ((((j0 >> 2) + q) ^ (lane & 7)) << 2));
                  v[4 * q] = f.x, v[4 * q + 1] = f.y, v[4 * q + 2] = f.z, v[4 * q + 3] = f.w;
                }
                split16(v, hi, lo);
                tmem_st16(Xh + xw * hw + j0, hi);
                tmem_st16(Xl + xw * hw + j0, lo);
              }
            }
          };
          auto put_h = [&](const float (&h)[16]) {
            float hi[16], lo[16];
            split16(h, hi, lo);
            tmem_st16(Hh + 16 * hw, hi);
            tmem_st16(Hl + 16 * hw, lo);
          };
          auto arrive = [&](uint64_t* bar) {
            tmem_wait_st();
            tc_fence_before();
            mbar_arrive(bar);
          };
          float c[16], h[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) c[i] = 0.f, h[i] = 0.f;
          if (Tt > 0) {
            fetch_x(0);
            if (Tt > 1) {
              fetch_x(1);
              cp_async_wait_x<1>();
            } else {
              cp_async_wait_x<0>();
            }
            put_x(0);
            arrive(&bars->ax_full);
            put_h(h);
            arrive(&bars->ah_full);
          }
          const float* bj = sbias + 16 * hw;
          for (int s = 0; s < Tt; ++s) {
            mbar_wait(&bars->d_full, pd);
            pd ^= 1;
            tc_fence_after();
            if (s + 1 < Tt) {
              // x part of step s+1: its MMAs run during this step's epilogue
              cp_async_wait_x<0>();
              put_x(s + 1);
              arrive(&bars->ax_full);
              if (s + 2 < Tt) fetch_x(s + 2);
            }
            const uint32_t Gt = tmem + lane_off + kColG + (uint32_t)(s & 1) * kG + 16 * hw;
            float zi[16], zf[16], zg[16], zo[16];
            tmem_ld16(Gt + 0 * kH, zi);
            tmem_ld16(Gt + 1 * kH, zf);
            tmem_ld16(Gt + 2 * kH, zg);
            tmem_ld16(Gt + 3 * kH, zo);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              const float gi = Act<float>::sigmoid(bj[i] + zi[i]), gf = Act<float>::sigmoid(bj[kH + i] + zf[i]);
              const float gg = Act<float>::tanh(bj[2 * kH + i] + zg[i]);
              const float go = Act<float>::sigmoid(bj[3 * kH + i] + zo[i]);
              c[i] = fma_rn(gf, c[i], gi * gg);
              h[i] = go * Act<float>::tanh(c[i]);
            }
            if (s + 1 < Tt) {
              put_h(h);
              arrive(&bars->ah_full);
            }
            if (live && s < T) {
              const int t = d == 0 ? s : T - 1 - s;
              float4* orow = reinterpret_cast<float4*>(out + (int64_t)t * kD + d * kH + 16 * hw);
#pragma unroll
              for (int q = 0; q < 4; ++q) orow[q] = make_float4(h[4 * q], h[4 * q + 1], h[4 * q + 2], h[4 * q + 3]);
            }
          }
        } else if (lane == 0) {
          // per step: x chains (as soon as x_s is in TMEM), then h chains;
          // G[s & 1] = X_hi W_hi + X_lo W_hi + X_hi W_lo + (same for h)
          const uint32_t id = idesc_tf32(kRows, kG);
          const int nx = kx / 8;
          for (int s = 0; s < Tt; ++s) {
            const uint32_t Gs = tmem + kColG + (uint32_t)(s & 1) * kG;
            mbar_wait(&bars->ax_full, pa);
            tc_fence_after();
            for (int part = 0; part < 3; ++part) {
              const uint32_t A = tmem + (part == 1 ? kColXl : kColXh);
              const uint32_t boff = part == 2 ? kG * 128 : 0;  // W_lo rows of the stacked image
              for (int kk = 0; kk < nx; ++kk) {
                const uint64_t bd = sw128_desc(bs_addr + (kk >> 2) * (kN * 128) + boff + (kk & 3) * 32);
                mma_tf32_ts(Gs, A + kk * 8, bd, id, part != 0 || kk != 0);
              }
            }
            mbar_wait(&bars->ah_full, pa);
            pa ^= 1;
            tc_fence_after();
            for (int part = 0; part < 3; ++part) {
              const uint32_t A = tmem + (part == 1 ? kColHl : kColHh);
              const uint32_t boff = part == 2 ? kG * 128 : 0;
              for (int kk = 0; kk < kH / 8; ++kk) {
                const uint64_t bd = sw128_desc(bs_addr + (kx >> 5) * (kN * 128) + boff + kk * 32);
                mma_tf32_ts(Gs, A + kk * 8, bd, id, 1);
              }
            }
            mma_commit(&bars->d_full);
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

// ---------------------------------------------------------------------------
// Attention + head from S (tuner.py:247-280), one program per thread, fp32
// FMAs.  K and V are never formed:
//   logit_{t,h} = q_h . (S_t Wk_h) = S_t . r_h,   r_h = Wk_h q_h
//   ctx_h = sum_t alpha_{t,h} (S_t Wv_h) = (sum_t alpha_{t,h} S_t) Wv_h
// (the same sums regrouped: ~2 x 4096 + 128 T multiply-adds per pass and
// head instead of 8192 T for K and V).  The softmax is online, one pass over
// the program's rows per (pass, head):
//   m_t = max(m_{t-1}, l_t), s_t = s_{t-1} e^{m_{t-1}-m_t} + e^{l_t-m_t},
//   u_t = u_{t-1} e^{m_{t-1}-m_t} + e^{l_t-m_t} S_t,   u_h = u_T / s_T.
// Weights sit in shared memory (all lanes read the same word: broadcast);
// a matvec's input vector is staged in the thread's private shared-memory
// column x[k][thread], so its k loop stays a loop (fully unrolled 64 x 64
// matvecs overflow the instruction cache).  Every scalar is accumulated in
// a fixed order inside one thread: a score does not depend on the launch.
namespace x3 {
constexpr int kAttnThreads = 256;
}

struct AttnRowsArgs {
  TDims dm;
  const float* prm;
  const int64_t* rowoff;
  const float* ctx;
  int64_t n;
  const float* S;
  float* yhat;
};

__host__ __device__ inline size_t x3_attn_smem_floats(const TDims& dm) {
  (void)dm;
  return 5 * 64 * 64 + 4 * 64 + 4 + (size_t)2 * 64 * x3::kAttnThreads;
}

// acc[0:W) += sum_{k0 <= k < k1} x[k] Wm[k][0:W)   (x: this thread's staged column)
template <int W>
__device__ __forceinline__ void mvs(const float* __restrict__ x, int k0, int k1, const float* __restrict__ Wm,
                                    float (&acc)[W]) {
#pragma unroll 2
  for (int k = k0; k < k1; ++k) {
    const float xk = x[k * x3::kAttnThreads];
    const float4* w4 = reinterpret_cast<const float4*>(Wm + k * 64);
#pragma unroll
    for (int j = 0; j < W / 4; ++j) {
      const float4 w = w4[j];
      acc[4 * j] = fma_rn(xk, w.x, acc[4 * j]);
      acc[4 * j + 1] = fma_rn(xk, w.y, acc[4 * j + 1]);
      acc[4 * j + 2] = fma_rn(xk, w.z, acc[4 * j + 2]);
      acc[4 * j + 3] = fma_rn(xk, w.w, acc[4 * j + 3]);
    }
  }
}

template <int W>
__device__ __forceinline__ void stage(float* __restrict__ x, const float (&v)[W], int k0 = 0) {
#pragma unroll
  for (int k = 0; k < W; ++k) x[(k0 + k) * x3::kAttnThreads] = v[k];
}

template <int HEADS>
__global__ void __launch_bounds__(x3::kAttnThreads, 1) tuner_attn_rows_kernel(AttnRowsArgs a) {
  using namespace x3;
  constexpr int DH = 64 / HEADS;
  extern __shared__ __align__(16) float sw[];
  const TDims& dm = a.dm;
  const int C = dm.C, TM = dm.Tmax, tid = threadIdx.x;
  float* Wq = sw;
  float* WkT = Wq + 4096;  // WkT[c][k] = Wk[k][c]
  float* Wv = WkT + 4096;
  float* Wo = Wv + 4096;
  float* W1 = Wo + 4096;  // rows [0, 64) of head_W1 (the pooled part)
  float* bq = W1 + 4096;
  float* bo = bq + 64;
  float* b1 = bo + 64;
  float* W2 = b1 + 64;
  float* b2 = W2 + 64;
  float* xq = b2 + 4 + tid;               // staged q, then ctx_flat
  float* xu = xq + 64 * kAttnThreads;     // staged pooled / u_h
  for (int i = tid; i < 4096; i += blockDim.x) {
    Wq[i] = __ldg(a.prm + dm.Wq + i);
    WkT[(i % 64) * 64 + i / 64] = __ldg(a.prm + dm.Wk + i);
    Wv[i] = __ldg(a.prm + dm.Wv + i);
    Wo[i] = __ldg(a.prm + dm.Wo + i);
    W1[i] = __ldg(a.prm + dm.W1 + i);
  }
  for (int i = tid; i < 64; i += blockDim.x) {
    bq[i] = __ldg(a.prm + dm.bq + i);
    bo[i] = __ldg(a.prm + dm.bo + i);
    b1[i] = __ldg(a.prm + dm.b1 + i);
    W2[i] = __ldg(a.prm + dm.W2 + i);
  }
  if (tid == 0) b2[0] = __ldg(a.prm + dm.b2);
  __syncthreads();
  const float sq = sqrtf((float)DH);
  const float* W1c = a.prm + dm.W1 + 64 * kHeadHidden;  // context rows (global, L1)
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + tid; p < a.n; p += (int64_t)gridDim.x * blockDim.x) {
    const int T = (int)(a.rowoff[p + 1] - a.rowoff[p]);
    const float4* Sp = reinterpret_cast<const float4*>(a.S + p * TM * 64);
    {
      float v[64];  // masked mean (tuner.py:252-253)
#pragma unroll
      for (int j = 0; j < 64; ++j) v[j] = 0.f;
      for (int t = 0; t < T; ++t)
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          const float4 f = Sp[t * 16 + q];
          v[4 * q] += f.x, v[4 * q + 1] += f.y, v[4 * q + 2] += f.z, v[4 * q + 3] += f.w;
        }
      const float den = (float)(T > 1 ? T : 1);
#pragma unroll
      for (int j = 0; j < 64; ++j) v[j] = v[j] / den;
      stage(xu, v);
    }
    for (int u = 0; u < dm.U; ++u) {
      {
        float q[64];  // q = pooled Wq + bq
#pragma unroll
        for (int j = 0; j < 64; ++j) q[j] = 0.f;
        mvs(xu, 0, 64, Wq, q);
#pragma unroll
        for (int j = 0; j < 64; ++j) q[j] += bq[j];
        stage(xq, q);
      }
#pragma unroll 1
      for (int h = 0; h < HEADS; ++h) {
        float r[64], uh[64];
#pragma unroll
        for (int k = 0; k < 64; ++k) r[k] = 0.f, uh[k] = 0.f;
        mvs(xq, h * DH, h * DH + DH, WkT, r);  // r_h = Wk[:, head h] q_h
        float mx = -INFINITY, sum = 0.f;
        for (int t = 0; t < T; ++t) {
          float a0 = 0.f, a1 = 0.f;
#pragma unroll
          for (int q = 0; q < 16; q += 2) {
            const float4 f = Sp[t * 16 + q], g = Sp[t * 16 + q + 1];
            a0 = fma_rn(f.x, r[4 * q], a0);
            a0 = fma_rn(f.y, r[4 * q + 1], a0);
            a0 = fma_rn(f.z, r[4 * q + 2], a0);
            a0 = fma_rn(f.w, r[4 * q + 3], a0);
            a1 = fma_rn(g.x, r[4 * q + 4], a1);
            a1 = fma_rn(g.y, r[4 * q + 5], a1);
            a1 = fma_rn(g.z, r[4 * q + 6], a1);
            a1 = fma_rn(g.w, r[4 * q + 7], a1);
          }
          const float l = (a0 + a1) / sq;  // tuner.py:264
          if (l > mx) {
            const float sc = Act<float>::exp(mx - l);  // 0 on the first step
            sum *= sc;
#pragma unroll
            for (int k = 0; k < 64; ++k) uh[k] *= sc;
            mx = l;
          }
          const float e = Act<float>::exp(l - mx);
          sum += e;
#pragma unroll
          for (int q = 0; q < 16; ++q) {
            const float4 f = Sp[t * 16 + q];  // L1 hit: the row was just read
            uh[4 * q] = fma_rn(e, f.x, uh[4 * q]);
            uh[4 * q + 1] = fma_rn(e, f.y, uh[4 * q + 1]);
            uh[4 * q + 2] = fma_rn(e, f.z, uh[4 * q + 2]);
            uh[4 * q + 3] = fma_rn(e, f.w, uh[4 * q + 3]);
          }
        }
        const float is = T > 0 ? 1.f / sum : 0.f;
#pragma unroll
        for (int k = 0; k < 64; ++k) uh[k] *= is;
        stage(xu, uh);
        float ch[DH];  // ctx_h = u_h Wv[:, head h] -> ctx_flat[head h] (over q_h)
#pragma unroll
        for (int c = 0; c < DH; ++c) ch[c] = 0.f;
        mvs(xu, 0, 64, Wv + h * DH, ch);
        stage(xq, ch, h * DH);
      }
      float v[64];  // pooled = ctx_flat Wo + bo
#pragma unroll
      for (int j = 0; j < 64; ++j) v[j] = 0.f;
      mvs(xq, 0, 64, Wo, v);
#pragma unroll
      for (int j = 0; j < 64; ++j) v[j] += bo[j];
      stage(xu, v);
    }
    // head: a1 = tanh([pooled | ctx] W1 + b1), y = sigmoid(a1 W2 + b2)
    float a1[64];
#pragma unroll
    for (int j = 0; j < 64; ++j) a1[j] = 0.f;
    mvs(xu, 0, 64, W1, a1);
    const float* cp = a.ctx + p * C;
#pragma unroll 1
    for (int k = 0; k < C; ++k) {
      const float xk = __ldg(cp + k);
      const float4* w4 = reinterpret_cast<const float4*>(W1c + k * 64);
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const float4 w = __ldg(w4 + j);
        a1[4 * j] = fma_rn(xk, w.x, a1[4 * j]);
        a1[4 * j + 1] = fma_rn(xk, w.y, a1[4 * j + 1]);
        a1[4 * j + 2] = fma_rn(xk, w.z, a1[4 * j + 2]);
        a1[4 * j + 3] = fma_rn(xk, w.w, a1[4 * j + 3]);
      }
    }
    float acc = 0.f;
#pragma unroll
    for (int j = 0; j < 64; ++j) acc = fma_rn(Act<float>::tanh(a1[j] + b1[j]), W2[j], acc);
    a.yhat[p] = Act<float>::sigmoid(acc + b2[0]);
  }
}

template <int HEADS>
static int launch_attn_rows(const AttnRowsArgs& a, cudaStream_t st) {
  const size_t smem = x3_attn_smem_floats(a.dm) * sizeof(float);
  auto kern = tuner_attn_rows_kernel<HEADS>;
  TT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 0;
  TT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, x3::kAttnThreads, smem));
  TT_REQUIRE(per_sm >= 1, "tuner attention: kernel cannot be resident (smem %zu)", smem);
  const int64_t blocks = (a.n + x3::kAttnThreads - 1) / x3::kAttnThreads;
  const int grid = (int)std::min<int64_t>(blocks, (int64_t)sm_count() * per_sm);
  kern<<<grid, x3::kAttnThreads, smem, st>>>(a);
  return check_launch("tuner attention rows");
}

static int attn_rows(const AttnRowsArgs& a, cudaStream_t st) {
  switch (a.dm.heads) {
    case 1: return launch_attn_rows<1>(a, st);
    case 2: return launch_attn_rows<2>(a, st);
    case 4: return launch_attn_rows<4>(a, st);
  }
  set_error("tuner fp32 tensor-core scoring: heads must be 1, 2 or 4");
  return TT_EINVAL;
}

// programs per (LSTM, attention) launch pair: up to 4 tiles per SM, fewer
// when the padded rows of a chunk would pass kChunkBudget (long programs)
static int64_t x3_chunk(int Tmax) {
  const size_t tile = (size_t)x3::kRows * Tmax * x3::kD * sizeof(float);
  const int64_t tiles = std::max<int64_t>(1, std::min<int64_t>(x3::kMaxChunkTilesPerSm * sm_count(),
                                                                 (int64_t)(x3::kChunkBudget / tile)));
  return tiles * x3::kRows;
}
static int x3_grid_max(int Tmax) { return (int)std::min<int64_t>(sm_count(), x3_chunk(Tmax) / x3::kRows); }

size_t tuner_predict_x3_ws(int L, int H, int Tmax) {
  (void)H;
  const size_t rowb = (size_t)Tmax * x3::kD * sizeof(float);
  size_t b = align_up((size_t)x3_chunk(Tmax) * rowb, 1024);              // S
  b += align_up((size_t)x3_grid_max(Tmax) * x3::kRows * rowb, 1024);     // layer scratch
  b += align_up((size_t)x3_image_off(L, 0), 1024);                      // B images
  return b;
}

int tuner_predict_x3(const float* prm, const float* steps, const int64_t* rowoff, const float* ctx,
                     int64_t n, int L, int H, int heads, int U, int d0, int C, int Tmax, float* yhat,
                     void* ws, size_t ws_bytes, cudaStream_t st) {
  TT_REQUIRE(H == 32, "tuner fp32 tensor-core scoring: hidden size must be 32");
  TT_REQUIRE(L >= 1 && L <= kMaxLayers, "tuner fp32 tensor-core scoring: bad layer count");
  TT_REQUIRE(heads == 1 || heads == 2 || heads == 4, "tuner fp32 tensor-core scoring: heads must be 1, 2 or 4");
  TT_REQUIRE(d0 >= 1 && d0 <= 32, "tuner fp32 tensor-core scoring: step width must be <= 32");
  TT_REQUIRE(C >= 0 && U >= 1, "tuner fp32 tensor-core scoring: bad context width / unroll");
  TT_REQUIRE(Tmax >= 1 && Tmax <= 4096, "tuner fp32 tensor-core scoring: bad max steps");
  TT_REQUIRE(n >= 0, "tuner fp32 tensor-core scoring: negative n");
  if (n == 0) return TT_OK;
  TT_REQUIRE(ws_bytes >= tuner_predict_x3_ws(L, H, Tmax), "tuner fp32 tensor-core scoring: workspace too small");
  const size_t rowb = (size_t)Tmax * x3::kD * sizeof(float);
  const int64_t chunk = x3_chunk(Tmax);
  unsigned char* w = static_cast<unsigned char*>(ws);
  X3Args a{};
  a.dm = make_dims(L, H, heads, U, d0, C, Tmax);
  a.prm = prm;
  a.steps = steps;
  a.S = reinterpret_cast<float*>(w);
  w += align_up((size_t)chunk * rowb, 1024);
  a.scratch = reinterpret_cast<float*>(w);
  w += align_up((size_t)x3_grid_max(Tmax) * x3::kRows * rowb, 1024);
  unsigned char* img = w;
  w += align_up((size_t)x3_image_off(L, 0), 1024);
  a.img = img;
  tuner_x3_prepare_kernel<<<2 * L, 256, 0, st>>>(a.dm, prm, img);
  TT_CUDA(cudaFuncSetAttribute(tuner_lstm_x3_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)x3::kSmem));
  for (int64_t p0 = 0; p0 < n; p0 += chunk) {
    const int64_t nc = std::min<int64_t>(chunk, n - p0);
    a.rowoff = rowoff + p0;
    a.n = nc;
    const int grid = (int)std::min<int64_t>((nc + x3::kRows - 1) / x3::kRows, x3_grid_max(Tmax));
    tuner_lstm_x3_kernel<<<grid, x3::kThreads, x3::kSmem, st>>>(a);
    if (int rc = check_launch("tuner lstm fp32 tensor-core")) return rc;
    AttnRowsArgs ar{a.dm, prm, rowoff + p0, ctx + p0 * C, nc, a.S, yhat + p0};
    if (int rc = attn_rows(ar, st)) return rc;
  }
  return TT_OK;
}

}  // namespace tt

extern "C" {

size_t tt_tuner_predict_f32tc_workspace_bytes(int32_t L, int32_t H, int32_t max_steps) {
  return tt::tuner_predict_x3_ws(L, H, max_steps);
}

int tt_tuner_f32tc_eligible(int32_t L, int32_t H, int32_t heads, int32_t d0, int32_t max_steps) {
  return H == 32 && L >= 1 && L <= tt::kMaxLayers && (heads == 1 || heads == 2 || heads == 4) &&
         d0 >= 1 && d0 <= 32 && max_steps >= 1 && max_steps <= 4096;
}

int tt_tuner_predict_f32tc(const float* prm, const float* steps, const int64_t* rowoff,
                           const float* ctx, int64_t n, int32_t L, int32_t H, int32_t heads,
                           int32_t U, int32_t d0, int32_t C, int32_t Tmax, float* yhat, void* ws,
                           size_t ws_bytes, tt_stream_t st) {
  return tt::tuner_predict_x3(prm, steps, rowoff, ctx, n, L, H, heads, U, d0, C, Tmax, yhat, ws,
                              ws_bytes, tt::as_stream(st));
}

}  // extern "C"
