// K5 at fp32 accuracy on the 5th-generation tensor cores: attention-tuner
// scoring (tuner.py _forward :227-285, predict :468-476) with the biLSTM
// stack as split-precision tcgen05 GEMMs (tuner_lstm_x3_kernel), then
// attention + head in fp32 on the CUDA cores (tuner_attn_rows_kernel /
// tuner_attn_warp_kernel, below).
//
// kind::tf32 truncates fp32 operands to 10 mantissa bits
// (tools/tf32_rounding_probe.py), so every product is split
//   a.w = a_hi.w_hi + a_lo.w_hi + a_hi.w_lo   (+ a_lo.w_lo, ~2^-20 |a.w|, dropped)
// with x_hi = x & ~0x1fff and x_lo = x - x_hi (exact in fp32).  The weight
// side is pre-split into one stacked B image per (layer, direction):
//   B^T rows [0,128) = W_hi^T, rows [128,256) = W_lo^T   (K-major SWIZZLE_128B)
// and each operand part (x, h) is three N = 128 chains into the step's gate
// buffer: A_hi W_hi, A_lo W_hi, A_hi W_lo.
//
// One persistent CTA per SM, 32 + 128 kParts threads, tiles of 128 programs:
//   warp 0        TMEM allocator (512 columns) and the single MMA-issuing lane
//   warps 1..16   4 threads per program ("row threads"; TMEM lane = row),
//                 part p owns hidden units 4p..4p+3 and 16+4p..16+4p+3
//                 (16 row warps, 4 per SM sub-partition, hide the MUFU
//                 latencies of the cell better than 8: 62.7 -> 65.8 M/s)
// TMEM columns: G[s & 1] [0,256)  x_hi [256,320)  x_lo [320,384)
//               h_hi [384,416)  h_lo [416,448)
// The two directions of a layer run one after the other (448 columns per
// direction).  Per step s the row threads load the gates G[s & 1] (+ bias),
// write x_{s+1} (prefetched two steps ahead by cp.async) so the MMA lane can
// issue the next step's x chains into G[(s+1) & 1] while they run the cell
// (5 ex2 + 3 rcp per unit: two sigmoid pairs share a reciprocal), then write
// h, whose three short chains close the step.  Programs are ordered by
// length per launch chunk (sort_programs_by_length) so a tile runs ~its own
// programs' steps; warps whose programs have ended skip their epilogue; a
// shorter program's steps past its end write nothing (the valid steps of
// both directions are a prefix).
//
// Layer outputs: the last layer lands in S = [n][Tmax][64] (fp32, padded
// per program), which the attention kernels read; the layers before it
// alternate between the program's S rows and a per-CTA scratch tile.
#include "tt_sm100.cuh"
#include "tt_tuner.cuh"

namespace tt {

using namespace sm100;

namespace x3 {
constexpr int kRows = 128;
constexpr int kParts = 4;                   // row threads per program
constexpr int kU = 32 / kParts;             // hidden units per row thread (two groups of 4)
constexpr int kRowThreads = kParts * 128;
constexpr int kThreads = 32 + kRowThreads;  // + the MMA warp
constexpr int kXq = 16 / kParts;            // 16-B x chunks per thread (layers >= 1)
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
  // blockIdx.y strides the elements: 16 CTAs per image keep this off the
  // latency of small scoring calls
  for (int i = blockIdx.y * blockDim.x + threadIdx.x; i < K * kN; i += gridDim.y * blockDim.x) {
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

// clock64 marks (debug aid, tt_debug_x3_phase_times): CTA 0, first tile;
// [18 + 2 (2l + d)] / [19 + ...]: (layer, direction) start / last MMA done;
// layer 1, forward direction, steps 2 and 3 (9 marks each): row thread 0
// [0] d_full [1] x_{s+1} arrived [2] gates loaded [3] activations done
// [4] h arrived; MMA lane [5] x ready [6] (unused) [7] h ready [8] committed
static __device__ long long g_x3_phase[32];
#define X3_MARK(cond, i) \
  do {                   \
    if (cond) g_x3_phase[i] = clock64(); \
  } while (0)

struct X3Args {
  TDims dm;
  const float* prm;
  const float* steps;
  const int64_t* rowoff;
  int64_t n;
  float* S;        // [n][Tmax][64]
  float* scratch;  // per CTA [128][Tmax][64]
  const unsigned char* img;
  const int32_t* perm;  // program of each tile slot (sort_programs_by_length), null: identity
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

__device__ __forceinline__ float rcp_approx(float x) {  // MUFU.RCP, <= 1 ulp
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ float ex2_approx(float x) {  // MUFU.EX2, flush-to-zero
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// LSTM cell from the gate pre-activations (tuner.py:86-96): 5 exponentials
// and 3 reciprocals (two of them shared by a pair: 1/a = b/(ab), 1/b = a/(ab);
// the clamps keep ab finite and move each activation by < 1e-18).
__device__ __forceinline__ void lstm_cell(float zi, float zf, float zg, float zo, float& c, float& h) {
  constexpr float kL = 43.f;       // e^43 squared < FLT_MAX
  constexpr float kLog2e = 1.4426950408889634f;
  const float ai = 1.f + ex2_approx(-kLog2e * fminf(fmaxf(zi, -kL), kL));
  const float af = 1.f + ex2_approx(-kLog2e * fminf(fmaxf(zf, -kL), kL));
  const float ag = 1.f + ex2_approx(2.f * kLog2e * fminf(fmaxf(zg, -0.5f * kL), 0.5f * kL));
  const float ao = 1.f + ex2_approx(-kLog2e * fminf(fmaxf(zo, -kL), kL));
  const float r1 = rcp_approx(ai * af);
  const float r2 = rcp_approx(ag * ao);
  const float gi = af * r1, gf = ai * r1;                // sigmoid(zi), sigmoid(zf)
  const float gg = fma_rn(-2.f, ao * r2, 1.f), go = ag * r2;  // tanh(zg), sigmoid(zo)
  c = fma_rn(gf, c, gi * gg);
  const float ac = 1.f + ex2_approx(2.f * kLog2e * fminf(fmaxf(c, -0.5f * kL), 0.5f * kL));
  h = go * fma_rn(-2.f, rcp_approx(ac), 1.f);  // tanh(c)
}

__global__ void __launch_bounds__(x3::kThreads, 1) tuner_lstm_x3_kernel(X3Args a) {
  using namespace x3;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* Bs = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  float* xslots = reinterpret_cast<float*>(Bs + kBBytes);  // [2 slots][kXq chunks][row threads] x 16 B
  __shared__ float sbias[kG];
  __shared__ X3Bars bars_s;
  X3Bars* bars = &bars_s;
  const TDims& dm = a.dm;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool rowt = warp >= 1;
  const int part = (warp - 1) >> 2;          // which kU hidden units
  const int row = ((warp & 3) << 5) | lane;  // TMEM lane quarter = warp % 4
  const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
  const int TM = dm.Tmax;
  const uint32_t bs_addr = smem_u32(Bs);

  if (threadIdx.x == 0) {
    mbar_init(&bars->ax_full, kRowThreads);
    mbar_init(&bars->ah_full, kRowThreads);
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

  auto issue_image = [&](int l, int d) {  // thread 0; Bs is not read by any MMA in flight
    const uint32_t bytes = x3_image_bytes(l);
    const unsigned char* src = a.img + x3_image_off(l, d);
    mbar_expect_tx(&bars->w_full, bytes);
    for (uint32_t off = 0; off < bytes; off += 32768)
      bulk_g2s(Bs + off, src + off, bytes - off < 32768 ? bytes - off : 32768, &bars->w_full);
  };
  bool img_issued = false;
  uint32_t pdm = 0;  // MMA lane: parity of the next d_full completion

  const int64_t n_tiles = (a.n + kRows - 1) / kRows;
  for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    // tiles are filled in order of program length (a.perm): a tile runs for
    // its longest program, so mixing lengths would waste steps
    const int64_t slot = tile * kRows + row;
    const int64_t p = slot < a.n ? (a.perm ? (int64_t)a.perm[slot] : slot) : a.n;
    const bool live = rowt && p < a.n;
    int64_t r0 = 0;
    int T = 0;
    if (live) {
      r0 = a.rowoff[p];
      T = (int)(a.rowoff[p + 1] - r0);
    }
    if (threadIdx.x == 0) bars->tmax = 0;
    __syncthreads();
    if (live && part == 0) atomicMax(&bars->tmax, T);
    __syncthreads();
    const int Tt = bars->tmax;
    const bool mk0 = blockIdx.x == 0 && tile == blockIdx.x && (threadIdx.x == 32 || threadIdx.x == 0);
    float* srow = a.S + (live ? p : 0) * TM * kD;

    for (int l = 0; l < dm.L; ++l) {
      const int kx = x3_kx(l);
      float* out = ((dm.L - 1 - l) & 1) == 0 ? srow : xrow_cta;
      const float* in = ((dm.L - l) & 1) == 0 ? srow : xrow_cta;  // layer l-1's output
      for (int d = 0; d < 2; ++d) {
        const bool mk = mk0 && l == 1 && d == 0;
        // ---- stacked image of (l, d) -> Bs: issued by the MMA lane as soon as
        // the previous (layer, direction)'s last MMA completed, else here
        __syncthreads();
        if (threadIdx.x == 0 && !img_issued) issue_image(l, d);
        img_issued = false;
        for (int i = threadIdx.x; i < kG; i += blockDim.x) sbias[i] = __ldg(a.prm + dm.bb[l][d] + i);
        mbar_wait(&bars->w_full, pw);
        pw ^= 1;
        __syncthreads();
        X3_MARK(mk0 && threadIdx.x == 32 && 2 * l + d < 6, 18 + 2 * (2 * l + d));  // (l, d) starts

        if (rowt) {
          const uint32_t Xh = tmem + lane_off + kColXh, Xl = tmem + lane_off + kColXl;
          const uint32_t Hh = tmem + lane_off + kColHh, Hl = tmem + lane_off + kColHl;
          const int xw = kx / kParts;  // x columns of this thread: kx / kParts
          // x row of step s (this thread's columns, zeros past the program's
          // end) -> shared slot s & 1 by async copies, two steps ahead; slots
          // are [slot][16-B chunk][row thread] so a warp's accesses are
          // consecutive
          const int rt = threadIdx.x - 32;
          auto xchunk = [&](int s, int q) { return xslots + ((size_t)((s & 1) * kXq + q) * kRowThreads + rt) * 4; };
          auto fetch_x = [&](int s) {
            const bool ok = live && s < T;
            const int t = d == 0 ? s : T - 1 - s;
            if (l == 0) {
              const float* xr = a.steps + (r0 + (ok ? t : 0)) * dm.d0;
              for (int i = 0; i < xw; ++i) {
                const int k = xw * part + i;
                float* e = xchunk(s, i >> 2) + (i & 3);
                if (ok && k < dm.d0)
                  cp_async4(e, xr + k);
                else
                  *e = 0.f;
              }
            } else {
              const float* xr = in + (int64_t)(ok ? t : 0) * kD + xw * part;
#pragma unroll
              for (int q = 0; q < kXq; ++q) {
                float* e = xchunk(s, q);
                if (ok)
                  cp_async16(e, xr + 4 * q);
                else
                  *reinterpret_cast<float4*>(e) = make_float4(0.f, 0.f, 0.f, 0.f);
              }
            }
            cp_async_commit_x();
          };
          auto put_x = [&](int s) {
#pragma unroll
            for (int j0 = 0; j0 < 4 * kXq; j0 += 8) {
              if (j0 < xw) {
                float hi[8], lo[8];
#pragma unroll
                for (int q = 0; q < 2; ++q) {
                  const float4 f = *reinterpret_cast<const float4*>(xchunk(s, j0 / 4 + q));
                  const float v[4] = {f.x, f.y, f.z, f.w};
#pragma unroll
                  for (int i = 0; i < 4; ++i) {
                    hi[4 * q + i] = tf32_hi(v[i]);
                    lo[4 * q + i] = v[i] - hi[4 * q + i];
                  }
                }
                tmem_st8(Xh + xw * part + j0, hi);
                tmem_st8(Xl + xw * part + j0, lo);
              }
            }
          };
          // hidden units of group g (4 each): columns cg[g] + 0..3
          const int cg[2] = {4 * part, 16 + 4 * part};
          auto put_h = [&](const float (&h)[kU], int g) {
            float hi[4], lo[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              hi[i] = tf32_hi(h[4 * g + i]);
              lo[i] = h[4 * g + i] - hi[i];
            }
            tmem_st4(Hh + cg[g], hi);
            tmem_st4(Hl + cg[g], lo);
          };
          auto arrive = [&](uint64_t* bar) {
            tmem_wait_st();
            tc_fence_before();
            mbar_arrive(bar);
          };
          float c[kU], h[kU];
#pragma unroll
          for (int i = 0; i < kU; ++i) c[i] = 0.f, h[i] = 0.f;
          // steps this warp's rows still need: past them (short or no
          // programs) the warp only keeps the barrier counts; its TMEM rows
          // then hold stale values, which only feed its own (unused) rows
          const int wT = __reduce_max_sync(0xffffffffu, live ? T : 0);
          if (Tt > 0) {
            if (wT > 0) {
              fetch_x(0);
              if (wT > 1) {
                fetch_x(1);
                cp_async_wait_x<1>();
              } else {
                cp_async_wait_x<0>();
              }
              put_x(0);
              put_h(h, 0);
              put_h(h, 1);
            }
            arrive(&bars->ax_full);
            arrive(&bars->ah_full);
          }
          for (int s = 0; s < Tt; ++s) {
            mbar_wait(&bars->d_full, pd);
            X3_MARK(mk && s >= 2 && s < 4, 9 * (s - 2) + 0);
            pd ^= 1;
            tc_fence_after();
            if (s >= wT) {  // this warp's programs have ended
              if (s + 1 < Tt) {
                arrive(&bars->ax_full);
                arrive(&bars->ah_full);
              }
              continue;
            }
            // gates first: once the next x MMAs run, TMEM loads queue behind them
            const uint32_t Gt = tmem + lane_off + kColG + (uint32_t)(s & 1) * kG;
            float zi[kU], zf[kU], zg[kU], zo[kU];
#pragma unroll
            for (int g = 0; g < 2; ++g) {
              tmem_ld4(Gt + 0 * kH + cg[g], zi + 4 * g);
              tmem_ld4(Gt + 1 * kH + cg[g], zf + 4 * g);
              tmem_ld4(Gt + 2 * kH + cg[g], zg + 4 * g);
              tmem_ld4(Gt + 3 * kH + cg[g], zo + 4 * g);
            }
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < kU; ++i) {  // bias now: shared-memory reads stall while the MMAs run
              const int j = cg[i >> 2] + (i & 3);
              zi[i] += sbias[j];
              zf[i] += sbias[kH + j];
              zg[i] += sbias[2 * kH + j];
              zo[i] += sbias[3 * kH + j];
            }
            X3_MARK(mk && s >= 2 && s < 4, 9 * (s - 2) + 2);
            if (s + 1 < Tt) {
              // x part of step s+1: its MMAs run during this step's activations
              if (s + 1 < wT) {
                cp_async_wait_x<0>();
                put_x(s + 1);
              }
              arrive(&bars->ax_full);
              X3_MARK(mk && s >= 2 && s < 4, 9 * (s - 2) + 1);
              if (s + 2 < wT) fetch_x(s + 2);
            }
#pragma unroll
            for (int i = 0; i < kU; ++i) lstm_cell(zi[i], zf[i], zg[i], zo[i], c[i], h[i]);
            if (s + 1 < Tt) {
              X3_MARK(mk && s >= 2 && s < 4, 9 * (s - 2) + 3);
              if (s + 1 < wT) {
                put_h(h, 0);
                put_h(h, 1);
              }
              arrive(&bars->ah_full);
              X3_MARK(mk && s >= 2 && s < 4, 9 * (s - 2) + 4);
            }
            if (live && s < T) {
              const int t = d == 0 ? s : T - 1 - s;
              float* orow = out + (int64_t)t * kD + d * kH;
#pragma unroll
              for (int g = 0; g < 2; ++g)
                *reinterpret_cast<float4*>(orow + cg[g]) =
                    make_float4(h[4 * g], h[4 * g + 1], h[4 * g + 2], h[4 * g + 3]);
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
            X3_MARK(mk && s >= 2 && s < 4, 9 * (s - 2) + 5);
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
            X3_MARK(mk && s >= 2 && s < 4, 9 * (s - 2) + 7);
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
            pdm ^= 1;
            X3_MARK(mk && s >= 2 && s < 4, 9 * (s - 2) + 8);
          }
          // next (layer, direction)'s weights while the row threads finish
          if (Tt > 0) mbar_wait(&bars->d_full, pdm ^ 1);
          X3_MARK(mk0 && 2 * l + d < 6, 19 + 2 * (2 * l + d));  // (l, d)'s last MMA done
          int nl = l, nd = d + 1;
          bool next = true;
          if (nd == 2) {
            nd = 0;
            if (++nl == dm.L) {
              nl = 0;
              next = tile + gridDim.x < n_tiles;
            }
          }
          if (next) {
            issue_image(nl, nd);
            img_issued = true;
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

// Counting sort of a chunk's programs by length, longest first, in two
// launches over kSortCtas CTAs: per-CTA bucket counts, then each CTA's
// offsets (longer buckets first, then lower CTAs) and a scatter.  Which tile
// a program lands in does not change its arithmetic (every row is
// independent), only how many padded steps its tile runs.
constexpr int kSortCtas = 64;

__global__ void __launch_bounds__(512) x3_sort_count_kernel(const int64_t* __restrict__ rowoff, int64_t n, int Tmax,
                                                            int* __restrict__ counts) {
  extern __shared__ int hist[];  // [Tmax + 1]
  for (int i = threadIdx.x; i <= Tmax; i += blockDim.x) hist[i] = 0;
  __syncthreads();
  const int64_t per = (n + gridDim.x - 1) / gridDim.x, lo = blockIdx.x * per, hi = min(n, lo + per);
  for (int64_t p = lo + threadIdx.x; p < hi; p += blockDim.x) atomicAdd(&hist[(int)(rowoff[p + 1] - rowoff[p])], 1);
  __syncthreads();
  for (int i = threadIdx.x; i <= Tmax; i += blockDim.x) counts[(int64_t)blockIdx.x * (Tmax + 1) + i] = hist[i];
}

__global__ void __launch_bounds__(512) x3_sort_scatter_kernel(const int64_t* __restrict__ rowoff, int64_t n,
                                                              int Tmax, const int* __restrict__ counts,
                                                              int32_t* __restrict__ perm) {
  extern __shared__ int cur[];  // [2 (Tmax + 1)]: bucket totals, then this CTA's cursors
  int* tot = cur + (Tmax + 1);
  for (int t = threadIdx.x; t <= Tmax; t += blockDim.x) {
    int all = 0, below = 0;
    for (int b = 0; b < (int)gridDim.x; ++b) {
      const int c = counts[(int64_t)b * (Tmax + 1) + t];
      all += c;
      if (b < (int)blockIdx.x) below += c;
    }
    tot[t] = all;
    cur[t] = below;
  }
  __syncthreads();
  if (threadIdx.x == 0) {  // exclusive offsets, longest bucket first
    int run = 0;
    for (int t = Tmax; t >= 0; --t) {
      cur[t] += run;
      run += tot[t];
    }
  }
  __syncthreads();
  const int64_t per = (n + gridDim.x - 1) / gridDim.x, lo = blockIdx.x * per, hi = min(n, lo + per);
  for (int64_t p = lo + threadIdx.x; p < hi; p += blockDim.x)
    perm[atomicAdd(&cur[(int)(rowoff[p + 1] - rowoff[p])], 1)] = (int32_t)p;
}

size_t sort_scratch_bytes(int Tmax) { return (size_t)kSortCtas * (Tmax + 1) * sizeof(int); }

int sort_programs_by_length(const int64_t* rowoff, int64_t n, int Tmax, int32_t* perm, void* scratch,
                            cudaStream_t st) {
  int* counts = static_cast<int*>(scratch);
  x3_sort_count_kernel<<<kSortCtas, 512, (size_t)(Tmax + 1) * sizeof(int), st>>>(rowoff, n, Tmax, counts);
  x3_sort_scatter_kernel<<<kSortCtas, 512, 2 * (size_t)(Tmax + 1) * sizeof(int), st>>>(rowoff, n, Tmax, counts,
                                                                                          perm);
  return check_launch("tuner length sort");
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

// Warp-per-program variant for small launches (search-time scoring): each
// scalar goes through the same operations in the same order as in
// tuner_attn_rows_kernel -- lane j owns outputs j and j + 32 of a matvec,
// lane t owns logit t, the online softmax's running max / sum are
// recomputed identically in every lane, lane 0 sums the head's 64-term dot
// product -- so both kernels give the same bits and a score does not depend
// on which one ran (tests/test_gpu_tuner_f32tc.py).
namespace x3 {
constexpr int kAttnWarps = 8;
constexpr int64_t kAttnWarpMax = 16384;  // programs per launch up to which the warp kernel runs
}

__host__ __device__ inline size_t x3_attn_warp_smem_floats(const TDims& dm) {
  return 5 * 64 * 64 + 4 * 64 + 4 + (size_t)x3::kAttnWarps * (128 + dm.Tmax);
}

template <int HEADS>
__global__ void __launch_bounds__(32 * x3::kAttnWarps) tuner_attn_warp_kernel(AttnRowsArgs a) {
  using namespace x3;
  constexpr int DH = 64 / HEADS;
  extern __shared__ __align__(16) float sw[];
  const TDims& dm = a.dm;
  const int C = dm.C, TM = dm.Tmax, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  float* Wq = sw;
  float* WkT = Wq + 4096;
  float* Wv = WkT + 4096;
  float* Wo = Wv + 4096;
  float* W1 = Wo + 4096;
  float* bq = W1 + 4096;
  float* bo = bq + 64;
  float* b1 = bo + 64;
  float* W2 = b1 + 64;
  float* b2 = W2 + 64;
  float* xs = b2 + 4 + warp * (128 + TM);  // per warp: x[64] y[64] logits[Tmax]
  float* ys = xs + 64;
  float* lg = ys + 64;
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
  const float* W1c = a.prm + dm.W1 + 64 * kHeadHidden;
  const int j0 = lane, j1 = lane + 32;
  for (int64_t p = (int64_t)blockIdx.x * kAttnWarps + warp; p < a.n; p += (int64_t)gridDim.x * kAttnWarps) {
    const int T = (int)(a.rowoff[p + 1] - a.rowoff[p]);
    const float* Sp = a.S + p * TM * 64;
    float v0 = 0.f, v1 = 0.f;
    for (int t = 0; t < T; ++t) {
      v0 += Sp[t * 64 + j0];
      v1 += Sp[t * 64 + j1];
    }
    const float den = (float)(T > 1 ? T : 1);
    __syncwarp();
    xs[j0] = v0 / den;
    xs[j1] = v1 / den;
    __syncwarp();
    for (int u = 0; u < dm.U; ++u) {
      float q0 = 0.f, q1 = 0.f;
      for (int k = 0; k < 64; ++k) {
        const float xk = xs[k];
        q0 = fma_rn(xk, Wq[k * 64 + j0], q0);
        q1 = fma_rn(xk, Wq[k * 64 + j1], q1);
      }
      ys[j0] = q0 + bq[j0];
      ys[j1] = q1 + bq[j1];
      __syncwarp();
#pragma unroll 1
      for (int h = 0; h < HEADS; ++h) {
        float r0 = 0.f, r1 = 0.f;
        for (int c = h * DH; c < h * DH + DH; ++c) {
          const float qc = ys[c];
          r0 = fma_rn(qc, WkT[c * 64 + j0], r0);
          r1 = fma_rn(qc, WkT[c * 64 + j1], r1);
        }
        __syncwarp();
        xs[j0] = r0;
        xs[j1] = r1;
        __syncwarp();
        for (int t = lane; t < T; t += 32) {
          const float4* Sr = reinterpret_cast<const float4*>(Sp + t * 64);
          float a0 = 0.f, a1 = 0.f;
#pragma unroll
          for (int q = 0; q < 16; q += 2) {
            const float4 f = Sr[q], g = Sr[q + 1];
            a0 = fma_rn(f.x, xs[4 * q], a0);
            a0 = fma_rn(f.y, xs[4 * q + 1], a0);
            a0 = fma_rn(f.z, xs[4 * q + 2], a0);
            a0 = fma_rn(f.w, xs[4 * q + 3], a0);
            a1 = fma_rn(g.x, xs[4 * q + 4], a1);
            a1 = fma_rn(g.y, xs[4 * q + 5], a1);
            a1 = fma_rn(g.z, xs[4 * q + 6], a1);
            a1 = fma_rn(g.w, xs[4 * q + 7], a1);
          }
          lg[t] = (a0 + a1) / sq;
        }
        __syncwarp();
        float mx = -INFINITY, sum = 0.f, u0 = 0.f, u1 = 0.f;
        for (int t = 0; t < T; ++t) {
          const float l = lg[t];
          if (l > mx) {
            const float sc = Act<float>::exp(mx - l);
            sum *= sc;
            u0 *= sc;
            u1 *= sc;
            mx = l;
          }
          const float e = Act<float>::exp(l - mx);
          sum += e;
          u0 = fma_rn(e, Sp[t * 64 + j0], u0);
          u1 = fma_rn(e, Sp[t * 64 + j1], u1);
        }
        const float is = T > 0 ? 1.f / sum : 0.f;
        __syncwarp();
        xs[j0] = u0 * is;
        xs[j1] = u1 * is;
        __syncwarp();
#pragma unroll
        for (int cc = 0; cc < 2; ++cc) {
          const int c = lane + 32 * cc;
          if (c < DH) {
            float ch = 0.f;
            for (int k = 0; k < 64; ++k) ch = fma_rn(xs[k], Wv[k * 64 + h * DH + c], ch);
            ys[h * DH + c] = ch;
          }
        }
        __syncwarp();
      }
      float p0 = 0.f, p1 = 0.f;
      for (int k = 0; k < 64; ++k) {
        const float ck = ys[k];
        p0 = fma_rn(ck, Wo[k * 64 + j0], p0);
        p1 = fma_rn(ck, Wo[k * 64 + j1], p1);
      }
      __syncwarp();
      xs[j0] = p0 + bo[j0];
      xs[j1] = p1 + bo[j1];
      __syncwarp();
    }
    float a0 = 0.f, a1 = 0.f;
    for (int k = 0; k < 64; ++k) {
      const float xk = xs[k];
      a0 = fma_rn(xk, W1[k * 64 + j0], a0);
      a1 = fma_rn(xk, W1[k * 64 + j1], a1);
    }
    const float* cp = a.ctx + p * C;
    for (int k = 0; k < C; ++k) {
      const float xk = __ldg(cp + k);
      a0 = fma_rn(xk, __ldg(W1c + k * 64 + j0), a0);
      a1 = fma_rn(xk, __ldg(W1c + k * 64 + j1), a1);
    }
    ys[j0] = Act<float>::tanh(a0 + b1[j0]);
    ys[j1] = Act<float>::tanh(a1 + b1[j1]);
    __syncwarp();
    if (lane == 0) {
      float acc = 0.f;
      for (int j = 0; j < 64; ++j) acc = fma_rn(ys[j], W2[j], acc);
      a.yhat[p] = Act<float>::sigmoid(acc + b2[0]);
    }
    __syncwarp();
  }
}

static int resident_blocks(const void* kern, int threads, size_t smem, int* per_sm) {
  return kernel_occupancy(kern, threads, smem, per_sm);
}

template <int HEADS>
static int launch_attn_warp(const AttnRowsArgs& a, cudaStream_t st) {
  const size_t smem = x3_attn_warp_smem_floats(a.dm) * sizeof(float);
  auto kern = tuner_attn_warp_kernel<HEADS>;
  int per_sm = 0;
  if (int rc = resident_blocks((const void*)kern, 32 * x3::kAttnWarps, smem, &per_sm)) return rc;
  TT_REQUIRE(per_sm >= 1, "tuner attention: kernel cannot be resident (smem %zu)", smem);
  const int64_t blocks = (a.n + x3::kAttnWarps - 1) / x3::kAttnWarps;
  const int grid = (int)std::min<int64_t>(blocks, (int64_t)sm_count() * per_sm);
  kern<<<grid, 32 * x3::kAttnWarps, smem, st>>>(a);
  return check_launch("tuner attention warp");
}

template <int HEADS>
static int launch_attn_rows(const AttnRowsArgs& a, cudaStream_t st) {
  const size_t smem = x3_attn_smem_floats(a.dm) * sizeof(float);
  auto kern = tuner_attn_rows_kernel<HEADS>;
  int per_sm = 0;
  if (int rc = resident_blocks((const void*)kern, x3::kAttnThreads, smem, &per_sm)) return rc;
  TT_REQUIRE(per_sm >= 1, "tuner attention: kernel cannot be resident (smem %zu)", smem);
  const int64_t blocks = (a.n + x3::kAttnThreads - 1) / x3::kAttnThreads;
  const int grid = (int)std::min<int64_t>(blocks, (int64_t)sm_count() * per_sm);
  kern<<<grid, x3::kAttnThreads, smem, st>>>(a);
  return check_launch("tuner attention rows");
}

static int attn_rows(const AttnRowsArgs& a, cudaStream_t st) {
  // both kernels give identical bits; the warp kernel wins while a launch
  // cannot fill the GPU with one program per thread
  static const int64_t warp_max = [] {
    const char* e = getenv("TT_X3_ATTN_WARP_MAX");
    return e ? (int64_t)atoll(e) : (int64_t)x3::kAttnWarpMax;
  }();
  const bool w = a.n <= warp_max;
  switch (a.dm.heads) {
    case 1: return w ? launch_attn_warp<1>(a, st) : launch_attn_rows<1>(a, st);
    case 2: return w ? launch_attn_warp<2>(a, st) : launch_attn_rows<2>(a, st);
    case 4: return w ? launch_attn_warp<4>(a, st) : launch_attn_rows<4>(a, st);
  }
  set_error("tuner fp32 tensor-core scoring: heads must be 1, 2 or 4");
  return TT_EINVAL;
}

// programs per (LSTM, attention) launch pair: up to 4 tiles per SM, fewer
// when the padded rows of a chunk would pass kChunkBudget (long programs)
static int64_t x3_chunk(int Tmax, int64_t n) {
  const size_t tile = (size_t)x3::kRows * Tmax * x3::kD * sizeof(float);
  const int64_t tiles = std::max<int64_t>(1, std::min<int64_t>(x3::kMaxChunkTilesPerSm * sm_count(),
                                                                 (int64_t)(x3::kChunkBudget / tile)));
  // small calls (search-time scoring) size everything by their own programs
  const int64_t need = std::max<int64_t>(1, (n + x3::kRows - 1) / x3::kRows);
  return std::min(tiles, need) * x3::kRows;
}
static int x3_grid_max(int Tmax, int64_t n) {
  return (int)std::min<int64_t>(sm_count(), x3_chunk(Tmax, n) / x3::kRows);
}

size_t tuner_predict_x3_ws(int L, int H, int Tmax, int64_t n) {
  (void)H;
  const size_t rowb = (size_t)Tmax * x3::kD * sizeof(float);
  size_t b = align_up((size_t)x3_chunk(Tmax, n) * rowb, 1024);           // S
  b += align_up((size_t)x3_grid_max(Tmax, n) * x3::kRows * rowb, 1024);  // layer scratch
  b += align_up((size_t)x3_image_off(L, 0), 1024);                      // B images
  b += align_up((size_t)x3_chunk(Tmax, n) * sizeof(int32_t), 1024);      // length order
  b += align_up(sort_scratch_bytes(Tmax), 1024);
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
  TT_REQUIRE(ws_bytes >= tuner_predict_x3_ws(L, H, Tmax, n), "tuner fp32 tensor-core scoring: workspace too small");
  const size_t rowb = (size_t)Tmax * x3::kD * sizeof(float);
  const int64_t chunk = x3_chunk(Tmax, n);
  unsigned char* w = static_cast<unsigned char*>(ws);
  X3Args a{};
  a.dm = make_dims(L, H, heads, U, d0, C, Tmax);
  a.prm = prm;
  a.steps = steps;
  a.S = reinterpret_cast<float*>(w);
  w += align_up((size_t)chunk * rowb, 1024);
  a.scratch = reinterpret_cast<float*>(w);
  w += align_up((size_t)x3_grid_max(Tmax, n) * x3::kRows * rowb, 1024);
  unsigned char* img = w;
  w += align_up((size_t)x3_image_off(L, 0), 1024);
  int32_t* perm = reinterpret_cast<int32_t*>(w);
  w += align_up((size_t)chunk * sizeof(int32_t), 1024);
  void* sort_scr = w;
  w += align_up(sort_scratch_bytes(Tmax), 1024);
  a.img = img;
  tuner_x3_prepare_kernel<<<dim3(2 * L, 16), 256, 0, st>>>(a.dm, prm, img);
  {
    int per_sm = 0;
    if (int rc = resident_blocks((const void*)tuner_lstm_x3_kernel, x3::kThreads, x3::kSmem, &per_sm)) return rc;
    TT_REQUIRE(per_sm == 1, "tuner lstm fp32 tensor-core: expected one CTA per SM, got %d", per_sm);
  }
  for (int64_t p0 = 0; p0 < n; p0 += chunk) {
    const int64_t nc = std::min<int64_t>(chunk, n - p0);
    a.rowoff = rowoff + p0;
    a.perm = nullptr;  // one tile: its order does not matter
    if (nc > x3::kRows) {
      if (int rc = sort_programs_by_length(a.rowoff, nc, Tmax, perm, sort_scr, st)) return rc;
      a.perm = perm;
    }
    a.n = nc;
    const int grid = (int)std::min<int64_t>((nc + x3::kRows - 1) / x3::kRows, x3_grid_max(Tmax, n));
    tuner_lstm_x3_kernel<<<grid, x3::kThreads, x3::kSmem, st>>>(a);
    if (int rc = check_launch("tuner lstm fp32 tensor-core")) return rc;
    AttnRowsArgs ar{a.dm, prm, rowoff + p0, ctx + p0 * C, nc, a.S, yhat + p0};
    if (int rc = attn_rows(ar, st)) return rc;
  }
  return TT_OK;
}

}  // namespace tt

extern "C" {

int tt_debug_x3_phase_times(int64_t* out, int32_t n) {
  TT_REQUIRE(n >= 0 && n <= 32, "debug: n must be in [0, 32]");
  TT_CUDA(cudaMemcpyFromSymbol(out, tt::g_x3_phase, sizeof(long long) * n));
  return TT_OK;
}

size_t tt_tuner_predict_f32tc_workspace_bytes(int32_t L, int32_t H, int32_t max_steps, int64_t n) {
  return tt::tuner_predict_x3_ws(L, H, max_steps, n);
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
