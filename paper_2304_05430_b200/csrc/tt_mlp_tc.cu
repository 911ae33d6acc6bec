// K3 on the 5th-generation tensor cores: CostMLP scoring (mlp.py:72-79) as a
// persistent, warp-specialised tcgen05 kernel (kind::tf32, fp32 accumulate).
//
//   warp 0      TMA producer: X tiles (128 rows x 32 fp32 boxes, SWIZZLE_128B,
//               out-of-bounds K columns zero-filled) into an NST-stage ring
//   warp 1      TMEM allocator + single-thread MMA issuer:
//                 GEMM1  acc1[128x64] = X[128xK] . W1          (A, B in smem)
//                 GEMM2  acc2[128x64] = tanh(acc1+b1) . W2     (A in TMEM)
//   warps 2..5  epilogue, one tile row per thread (TMEM lane): tanh(acc1+b1)
//               is written back to TMEM as GEMM2's A operand; tanh(acc2+b2)
//               . W3 + b3 is the score, stored coalesced.
// TMEM holds four tile buffers (acc1 -> h1 in place | acc2, 128 columns
// each) so GEMM1 runs up to three tiles ahead of the epilogue and the X ring
// drains as soon as stages land.
// Weights (W1^T zero-padded to K=ceil(F/32)*32, W2^T) are staged once per
// CTA in the K-major SW128 layout.
//
// Precision: tf32 operands (10-bit mantissa), fp32 accumulation, fp32
// activations -- the "tf32" precision mode with its own stated tolerance;
// the fp32 CUDA-core kernel (tt_mlp.cu) remains the strict-parity path.
#include "tt_ops.cuh"
#include "tt_sm100.cuh"

namespace tt {

using namespace sm100;

// tanh on the MUFU's native tanh.approx (one SFU op instead of ex2 + rcp):
// max abs error ~5e-4, inside the tf32 mode's stated 1e-2 / 1e-3 tolerance
__device__ __forceinline__ float tanh_ftz(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

constexpr int kTcRows = 128;   // rows per tile (M)
constexpr int kTcHid = 64;     // hidden width (N)
constexpr int kTcNst = 9;      // X pipeline stages (one 16 KB K-atom each; 1.5 tiles of F = 164 in flight)
constexpr int kTcThreads = 320;  // warp 0 TMA, warp 1 MMA, warps 2..9 epilogue (2 per lane quarter)
constexpr int kTcBufs = 4;       // TMEM tile buffers (128 columns each)
constexpr int kAtomBytesX = kTcRows * 128;  // 16 KB
constexpr int kAtomBytesW = kTcHid * 128;   // 8 KB

struct MlpTcParams {
  const float* prm;  // W1[F][64] b1 W2[64][64] b2 W3[64] b3
  float* out;
  int64_t n;
  int F;
  int kat;           // K atoms of 32 fp32 (ceil(F/32))
};

struct __align__(8) TcBars {
  uint64_t full[kTcNst], empty[kTcNst];
  uint64_t acc1_full[kTcBufs], h1_full[kTcBufs], acc2_full[kTcBufs], acc_free[kTcBufs];
  uint32_t tmem_base;
};

__global__ void __launch_bounds__(kTcThreads, 1)
    mlp_predict_tc_kernel(const __grid_constant__ CUtensorMap tmap_x, MlpTcParams p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // 1024-B aligned carve-up: [X stages][W1^T atoms][W2^T atoms][bars]
  unsigned char* base = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  unsigned char* xs = base;
  unsigned char* w1s = xs + kTcNst * kAtomBytesX;
  unsigned char* w2s = w1s + p.kat * kAtomBytesW;
  TcBars* bars = reinterpret_cast<TcBars*>(w2s + 2 * kAtomBytesW);
  __shared__ float s_b1[kTcHid], s_b2[kTcHid], s_w3[kTcHid];
  __shared__ float s_b3;
  __shared__ float s_part[kTcBufs][2][kTcRows];  // [buffer][column half][row] partial scores

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t n_tiles = (p.n + kTcRows - 1) / kTcRows;
  const int F = p.F;
  const int64_t oW1 = 0, ob1 = (int64_t)F * kTcHid, oW2 = ob1 + kTcHid, ob2 = oW2 + kTcHid * kTcHid,
                oW3 = ob2 + kTcHid, ob3 = oW3 + kTcHid;

  // ---- one-time setup
  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmap_x);
    for (int s = 0; s < kTcNst; ++s) {
      mbar_init(&bars->full[s], 1);
      mbar_init(&bars->empty[s], 1);
    }
    for (int b = 0; b < kTcBufs; ++b) {
      mbar_init(&bars->acc1_full[b], 1);
      mbar_init(&bars->h1_full[b], 256);
      mbar_init(&bars->acc2_full[b], 1);
      mbar_init(&bars->acc_free[b], 256);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(&bars->tmem_base);
  // stage W1^T (K-major, zero padded) and W2^T with the swizzle the MMA expects
  for (int i = threadIdx.x; i < p.kat * 32 * kTcHid; i += kTcThreads) {
    const int nrow = i % kTcHid, k = i / kTcHid;  // coalesced over n
    const float v = k < F ? p.prm[oW1 + (int64_t)k * kTcHid + nrow] : 0.0f;
    const int atom = k >> 5;
    *reinterpret_cast<float*>(w1s + atom * kAtomBytesW + sw128_offset(nrow, k & 31)) = v;
  }
  for (int i = threadIdx.x; i < kTcHid * kTcHid; i += kTcThreads) {
    const int nrow = i % kTcHid, k = i / kTcHid;
    const float v = p.prm[oW2 + (int64_t)k * kTcHid + nrow];
    *reinterpret_cast<float*>(w2s + (k >> 5) * kAtomBytesW + sw128_offset(nrow, k & 31)) = v;
  }
  for (int i = threadIdx.x; i < kTcHid; i += kTcThreads) {
    s_b1[i] = p.prm[ob1 + i];
    s_b2[i] = p.prm[ob2 + i];
    s_w3[i] = p.prm[oW3 + i];
  }
  if (threadIdx.x == 0) s_b3 = p.prm[ob3];
  fence_proxy_async_smem();  // generic-proxy writes -> visible to the tensor core
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bars->tmem_base;
  constexpr uint32_t kBufCols = 128;

  if (warp == 0) {
    // ================= TMA producer
    if (lane == 0) {
      uint32_t it = 0;
      for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
        for (int kc = 0; kc < p.kat; ++kc, ++it) {
          const uint32_t s = it % kTcNst, ph = (it / kTcNst) & 1;
          mbar_wait(&bars->empty[s], ph ^ 1);
          mbar_expect_tx(&bars->full[s], kAtomBytesX);
          tma_load_2d(xs + s * kAtomBytesX, &tmap_x, &bars->full[s], kc * 32,
                      (int)(tile * kTcRows));
        }
      }
    }
  } else if (warp == 1) {
    // ================= MMA issuer, software-pipelined by one tile: GEMM1 of
    // tile t+1 is issued before waiting for tile t's h1, so the tensor core
    // works on the next tile while the epilogue forms h1
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_tf32(kTcRows, kTcHid);
      uint32_t it = 0;
      const uint32_t w1a = smem_u32(w1s), w2a = smem_u32(w2s), xa = smem_u32(xs);
      auto gemm1 = [&](uint32_t t) {
        const uint32_t b = t % kTcBufs, bph = (t / kTcBufs) & 1;
        const uint32_t acc1 = tmem + b * kBufCols;
        mbar_wait(&bars->acc_free[b], bph ^ 1);
        tc_fence_after();
        for (int kc = 0; kc < p.kat; ++kc, ++it) {
          const uint32_t s = it % kTcNst, ph = (it / kTcNst) & 1;
          mbar_wait(&bars->full[s], ph);
          tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const uint64_t ad = sw128_desc(xa + s * kAtomBytesX + kk * 32);
            const uint64_t bd = sw128_desc(w1a + kc * kAtomBytesW + kk * 32);
            mma_tf32_ss(acc1, ad, bd, idesc, (kc | kk) != 0);
          }
          mma_commit(&bars->empty[s]);  // frees the X stage when these MMAs retire
        }
        mma_commit(&bars->acc1_full[b]);
      };
      const uint32_t my_tiles =
          (uint32_t)(n_tiles > blockIdx.x ? (n_tiles - 1 - blockIdx.x) / gridDim.x + 1 : 0);
      if (my_tiles > 0) gemm1(0);
      for (uint32_t t = 0; t < my_tiles; ++t) {
        if (t + 1 < my_tiles) gemm1(t + 1);
        const uint32_t b = t % kTcBufs, bph = (t / kTcBufs) & 1;
        const uint32_t h1 = tmem + b * kBufCols, acc2 = tmem + b * kBufCols + 64;
        mbar_wait(&bars->h1_full[b], bph);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint64_t bd = sw128_desc(w2a + (kk >> 2) * kAtomBytesW + (kk & 3) * 32);
          mma_tf32_ts(acc2, h1 + kk * 8, bd, idesc, kk != 0);
        }
        mma_commit(&bars->acc2_full[b]);
      }
    }
  } else {
    // ================= epilogue: warps 2..9, two warps per TMEM lane quarter;
    // warp half `hf` owns hidden columns [32 hf, 32 hf + 32) of the row
    const int quarter = warp & 3;  // TMEM lane quarter this warp may access
    const int hf = (warp - 2) >> 2;
    const int row = quarter * 32 + lane;
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    uint32_t t = 0;
    for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++t) {
      const uint32_t b = t % kTcBufs, bph = (t / kTcBufs) & 1;
      const uint32_t acc1 = tmem + lane_off + b * kBufCols, h1 = acc1, acc2 = acc1 + 64;
      mbar_wait(&bars->acc1_full[b], bph);
      tc_fence_after();
#pragma unroll
      for (int c0 = hf * 32; c0 < hf * 32 + 32; c0 += 16) {
        float v[16];
        tmem_ld16(acc1 + c0, v);
        tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = tanh_ftz(v[i] + s_b1[c0 + i]);
        tmem_st16(h1 + c0, v);
      }
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(&bars->h1_full[b]);
      mbar_wait(&bars->acc2_full[b], bph);
      tc_fence_after();
      float acc = 0.f;
#pragma unroll
      for (int c0 = hf * 32; c0 < hf * 32 + 32; c0 += 16) {
        float v[16];
        tmem_ld16(acc2 + c0, v);
        tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 16; ++i) acc += tanh_ftz(v[i] + s_b2[c0 + i]) * s_w3[c0 + i];
      }
      tc_fence_before();
      mbar_arrive(&bars->acc_free[b]);
      // combine the two column halves of the row in fixed order
      s_part[b][hf][row] = acc;
      named_barrier(1, 256);
      const int64_t r = tile * kTcRows + row;
      if (hf == 0 && r < p.n) p.out[r] = (s_part[b][0][row] + s_part[b][1][row]) + s_b3;
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

// ---------------------------------------------------- split precision --
// The same scorer at fp32 accuracy ("fp32" precision, the default): every
// operand is split into a tf32 head and a tf32 tail, v = hi + lo with
// hi = round_tf32(v) and lo = v - hi (exact in fp32), and each dense layer
// runs as three tensor-core products accumulated in fp32,
//     A.B ~= Ahi.Bhi + Ahi.Blo + Alo.Bhi      (Alo.Blo ~ 2^-22 |A.B| dropped)
// so the layer error is ~2^-21 relative instead of tf32's 2^-11.
//
//   warp 0      TMA producer: raw fp32 X atoms into an NST-stage ring
//   warp 1      TMEM allocator + MMA issuer (3 MMAs per K step)
//   warps 2..5  converters: one TMEM lane (tile row) per thread -- read the
//               row's 32 values of an X atom from shared memory, split, and
//               store hi | lo (32 + 32 columns) into a TMEM operand slot
//               (GEMM1's A operands come from TMEM); the X stage is released
//               as soon as it is read
//   warps 6..13 epilogue: h1 = tanh(acc1 + b1) split into hi | lo in TMEM
//               (GEMM2's A), then tanh(acc2 + b2) . W3 + b3 -> score.
// Activations use the accurate exp-based tanh of the fp32 CUDA-core kernel
// (Act<float>::tanh), not tanh.approx.
// TMEM: 2 operand slots x 64 columns + 2 tile buffers x 192 columns
// (acc1 -> h1hi | h1lo | acc2) = 512.
constexpr int kX3Nst = 5;
constexpr int kX3Slots = 2;
constexpr int kX3Bufs = 2;
constexpr int kX3Threads = 448;

__device__ __forceinline__ void split_tf32(float v, float& hi, float& lo) {
  // round to the nearest tf32 (10 explicit mantissa bits), ties away from zero
  const uint32_t u = __float_as_uint(v);
  hi = __uint_as_float((u + 0x1000u) & 0xffffe000u);
  lo = v - hi;
}

struct __align__(8) X3Bars {
  uint64_t full[kX3Nst], empty[kX3Nst];
  uint64_t op_full[kX3Slots], op_free[kX3Slots];
  uint64_t acc1_full[kX3Bufs], h1_full[kX3Bufs], acc2_full[kX3Bufs], acc_free[kX3Bufs];
  uint32_t tmem_base;
};

__global__ void __launch_bounds__(kX3Threads, 1)
    mlp_predict_x3_kernel(const __grid_constant__ CUtensorMap tmap_x, MlpTcParams p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* base = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  unsigned char* xs = base;                                  // [NST] X atoms
  unsigned char* w1h = xs + kX3Nst * kAtomBytesX;            // [kat] W1 hi atoms
  unsigned char* w1l = w1h + p.kat * kAtomBytesW;            // [kat] W1 lo atoms
  unsigned char* w2h = w1l + p.kat * kAtomBytesW;            // [2]
  unsigned char* w2l = w2h + 2 * kAtomBytesW;                // [2]
  X3Bars* bars = reinterpret_cast<X3Bars*>(w2l + 2 * kAtomBytesW);
  __shared__ float s_b1[kTcHid], s_b2[kTcHid], s_w3[kTcHid];
  __shared__ float s_b3;
  __shared__ float s_part[kX3Bufs][2][kTcRows];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t n_tiles = (p.n + kTcRows - 1) / kTcRows;
  const int F = p.F;
  const int64_t ob1 = (int64_t)F * kTcHid, oW2 = ob1 + kTcHid, ob2 = oW2 + kTcHid * kTcHid,
                oW3 = ob2 + kTcHid, ob3 = oW3 + kTcHid;

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmap_x);
    for (int s = 0; s < kX3Nst; ++s) {
      mbar_init(&bars->full[s], 1);
      mbar_init(&bars->empty[s], 128);
    }
    for (int s = 0; s < kX3Slots; ++s) {
      mbar_init(&bars->op_full[s], 128);
      mbar_init(&bars->op_free[s], 1);
    }
    for (int b = 0; b < kX3Bufs; ++b) {
      mbar_init(&bars->acc1_full[b], 1);
      mbar_init(&bars->h1_full[b], 256);
      mbar_init(&bars->acc2_full[b], 1);
      mbar_init(&bars->acc_free[b], 256);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(&bars->tmem_base);
  // weights: hi / lo halves, K-major SW128 (W^T rows = hidden unit n)
  for (int i = threadIdx.x; i < p.kat * 32 * kTcHid; i += kX3Threads) {
    const int nrow = i % kTcHid, k = i / kTcHid;
    const float v = k < F ? p.prm[(int64_t)k * kTcHid + nrow] : 0.0f;
    float hi, lo;
    split_tf32(v, hi, lo);
    const uint32_t off = (k >> 5) * kAtomBytesW + sw128_offset(nrow, k & 31);
    *reinterpret_cast<float*>(w1h + off) = hi;
    *reinterpret_cast<float*>(w1l + off) = lo;
  }
  for (int i = threadIdx.x; i < kTcHid * kTcHid; i += kX3Threads) {
    const int nrow = i % kTcHid, k = i / kTcHid;
    float hi, lo;
    split_tf32(p.prm[oW2 + (int64_t)k * kTcHid + nrow], hi, lo);
    const uint32_t off = (k >> 5) * kAtomBytesW + sw128_offset(nrow, k & 31);
    *reinterpret_cast<float*>(w2h + off) = hi;
    *reinterpret_cast<float*>(w2l + off) = lo;
  }
  for (int i = threadIdx.x; i < kTcHid; i += kX3Threads) {
    s_b1[i] = p.prm[ob1 + i];
    s_b2[i] = p.prm[ob2 + i];
    s_w3[i] = p.prm[oW3 + i];
  }
  if (threadIdx.x == 0) s_b3 = p.prm[ob3];
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bars->tmem_base;
  // column map: operand slot s at [64 s, 64 s + 64) (hi | lo);
  // tile buffer b at 128 + 192 b: acc1/h1hi [0,64) h1lo [64,128) acc2 [128,192)
  constexpr uint32_t kOpCols = 64, kBufBase = kX3Slots * kOpCols, kBufCols = 192;
  const uint32_t my_tiles =
      (uint32_t)(n_tiles > blockIdx.x ? (n_tiles - 1 - blockIdx.x) / gridDim.x + 1 : 0);

  if (warp == 0) {
    if (lane == 0) {
      uint32_t it = 0;
      for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
        for (int kc = 0; kc < p.kat; ++kc, ++it) {
          const uint32_t s = it % kX3Nst, ph = (it / kX3Nst) & 1;
          mbar_wait(&bars->empty[s], ph ^ 1);
          mbar_expect_tx(&bars->full[s], kAtomBytesX);
          tma_load_2d(xs + s * kAtomBytesX, &tmap_x, &bars->full[s], kc * 32, (int)(tile * kTcRows));
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_tf32(kTcRows, kTcHid);
      const uint32_t w1ha = smem_u32(w1h), w1la = smem_u32(w1l), w2ha = smem_u32(w2h),
                     w2la = smem_u32(w2l);
      uint32_t it = 0;
      auto gemm1 = [&](uint32_t t) {
        const uint32_t b = t % kX3Bufs, bph = (t / kX3Bufs) & 1;
        const uint32_t acc1 = tmem + kBufBase + b * kBufCols;
        mbar_wait(&bars->acc_free[b], bph ^ 1);
        tc_fence_after();
        for (int kc = 0; kc < p.kat; ++kc, ++it) {
          const uint32_t s = it % kX3Slots, ph = (it / kX3Slots) & 1;
          mbar_wait(&bars->op_full[s], ph);
          tc_fence_after();
          const uint32_t ahi = tmem + s * kOpCols, alo = ahi + 32;
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const uint64_t bh = sw128_desc(w1ha + kc * kAtomBytesW + kk * 32);
            const uint64_t bl = sw128_desc(w1la + kc * kAtomBytesW + kk * 32);
            mma_tf32_ts(acc1, ahi + kk * 8, bh, idesc, (kc | kk) != 0);
            mma_tf32_ts(acc1, ahi + kk * 8, bl, idesc, 1);
            mma_tf32_ts(acc1, alo + kk * 8, bh, idesc, 1);
          }
          mma_commit(&bars->op_free[s]);
        }
        mma_commit(&bars->acc1_full[b]);
      };
      if (my_tiles > 0) gemm1(0);
      for (uint32_t t = 0; t < my_tiles; ++t) {
        if (t + 1 < my_tiles) gemm1(t + 1);
        const uint32_t b = t % kX3Bufs, bph = (t / kX3Bufs) & 1;
        const uint32_t hhi = tmem + kBufBase + b * kBufCols, hlo = hhi + 64, acc2 = hhi + 128;
        mbar_wait(&bars->h1_full[b], bph);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t woff = (kk >> 2) * kAtomBytesW + (kk & 3) * 32;
          const uint64_t bh = sw128_desc(w2ha + woff), bl = sw128_desc(w2la + woff);
          mma_tf32_ts(acc2, hhi + kk * 8, bh, idesc, kk != 0);
          mma_tf32_ts(acc2, hhi + kk * 8, bl, idesc, 1);
          mma_tf32_ts(acc2, hlo + kk * 8, bh, idesc, 1);
        }
        mma_commit(&bars->acc2_full[b]);
      }
    }
  } else if (warp < 6) {
    // converters: thread = tile row (TMEM lane); 32 values per X atom
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    uint32_t it = 0;
    for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
      for (int kc = 0; kc < p.kat; ++kc, ++it) {
        const uint32_t s = it % kX3Nst, ph = (it / kX3Nst) & 1;
        const uint32_t os = it % kX3Slots, oph = (it / kX3Slots) & 1;
        mbar_wait(&bars->full[s], ph);
        const unsigned char* atom = xs + s * kAtomBytesX;
        float hv[32], lv[32];
#pragma unroll
        for (int c4 = 0; c4 < 8; ++c4) {
          const float4 v = *reinterpret_cast<const float4*>(atom + sw128_offset(row, c4 * 4));
          split_tf32(v.x, hv[4 * c4 + 0], lv[4 * c4 + 0]);
          split_tf32(v.y, hv[4 * c4 + 1], lv[4 * c4 + 1]);
          split_tf32(v.z, hv[4 * c4 + 2], lv[4 * c4 + 2]);
          split_tf32(v.w, hv[4 * c4 + 3], lv[4 * c4 + 3]);
        }
        mbar_arrive(&bars->empty[s]);  // the X stage is free for the next TMA
        mbar_wait(&bars->op_free[os], oph ^ 1);
        tc_fence_after();
        const uint32_t dst = tmem + lane_off + os * kOpCols;
        tmem_st16(dst, *reinterpret_cast<const float(*)[16]>(hv));
        tmem_st16(dst + 16, *reinterpret_cast<const float(*)[16]>(hv + 16));
        tmem_st16(dst + 32, *reinterpret_cast<const float(*)[16]>(lv));
        tmem_st16(dst + 48, *reinterpret_cast<const float(*)[16]>(lv + 16));
        tmem_wait_st();
        tc_fence_before();
        mbar_arrive(&bars->op_full[os]);
      }
    }
  } else {
    // epilogue: warps 6..13, two per lane quarter, column half hf
    const int quarter = warp & 3;
    const int hf = (warp - 6) >> 2;
    const int row = quarter * 32 + lane;
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    uint32_t t = 0;
    for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++t) {
      const uint32_t b = t % kX3Bufs, bph = (t / kX3Bufs) & 1;
      const uint32_t acc1 = tmem + lane_off + kBufBase + b * kBufCols;
      const uint32_t hlo = acc1 + 64, acc2 = acc1 + 128;
      mbar_wait(&bars->acc1_full[b], bph);
      tc_fence_after();
#pragma unroll
      for (int c0 = hf * 32; c0 < hf * 32 + 32; c0 += 16) {
        float v[16], lo[16];
        tmem_ld16(acc1 + c0, v);
        tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const float h = Act<float>::tanh(v[i] + s_b1[c0 + i]);
          split_tf32(h, v[i], lo[i]);
        }
        tmem_st16(acc1 + c0, v);
        tmem_st16(hlo + c0, lo);
      }
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(&bars->h1_full[b]);
      mbar_wait(&bars->acc2_full[b], bph);
      tc_fence_after();
      float acc = 0.f;
#pragma unroll
      for (int c0 = hf * 32; c0 < hf * 32 + 32; c0 += 16) {
        float v[16];
        tmem_ld16(acc2 + c0, v);
        tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 16; ++i) acc = fmaf(Act<float>::tanh(v[i] + s_b2[c0 + i]), s_w3[c0 + i], acc);
      }
      tc_fence_before();
      mbar_arrive(&bars->acc_free[b]);
      s_part[b][hf][row] = acc;
      named_barrier(1, 256);
      const int64_t r = tile * kTcRows + row;
      if (hf == 0 && r < p.n) p.out[r] = (s_part[b][0][row] + s_part[b][1][row]) + s_b3;
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

// ---------------------------------------------------------------- host --
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(ptr);
  }
  return fn;
}

static size_t tc_smem_bytes(int kat) {
  return 1024 + (size_t)kTcNst * kAtomBytesX + (size_t)(kat + 2) * kAtomBytesW + sizeof(TcBars) + 64;
}

static int make_x_map(const float* X, int64_t n, int F, CUtensorMap* map) {
  EncodeTiledFn enc = encode_fn();
  TT_REQUIRE(enc != nullptr, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {(cuuint64_t)F, (cuuint64_t)n};
  cuuint64_t strides[1] = {(cuuint64_t)F * 4};
  cuuint32_t box[2] = {32, kTcRows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(X), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  TT_REQUIRE(r == CUDA_SUCCESS, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return TT_OK;
}

int mlp_predict_tc(const float* prm, const float* X, int64_t n, int F, float* out,
                   cudaStream_t st) {
  TT_REQUIRE(F >= 1 && (F * 4) % 16 == 0, "mlp tf32 path: F*4 must be a multiple of 16");
  TT_REQUIRE(((uintptr_t)X & 15) == 0, "mlp tf32 path: X must be 16-B aligned");
  TT_REQUIRE(n >= 1 && n <= (int64_t)0x7fffffff, "mlp tf32 path: bad n");
  const int kat = (F + 31) / 32;
  const size_t smem = tc_smem_bytes(kat);
  TT_REQUIRE(smem <= 227 * 1024, "mlp tf32 path: F=%d too wide for shared memory", F);
  CUtensorMap map;
  if (int rc = make_x_map(X, n, F, &map)) return rc;
  MlpTcParams p{prm, out, n, F, kat};
  TT_CUDA(cudaFuncSetAttribute(mlp_predict_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)smem));
  const int64_t tiles = (n + kTcRows - 1) / kTcRows;
  const int grid = (int)std::min<int64_t>(tiles, sm_count());
  mlp_predict_tc_kernel<<<grid, kTcThreads, smem, st>>>(map, p);
  return check_launch("mlp predict tf32");
}

static size_t x3_smem_bytes(int kat) {
  return 1024 + (size_t)kX3Nst * kAtomBytesX + (size_t)(2 * kat + 4) * kAtomBytesW + sizeof(X3Bars) + 64;
}

// 1 if the split-precision tensor-core scorer covers this shape
int mlp_x3_eligible(int F, const float* X) {
  const int kat = (F + 31) / 32;
  return F >= 1 && (F * 4) % 16 == 0 && ((uintptr_t)X & 15) == 0 && x3_smem_bytes(kat) <= 227 * 1024;
}

int mlp_predict_x3(const float* prm, const float* X, int64_t n, int F, float* out, cudaStream_t st) {
  TT_REQUIRE(mlp_x3_eligible(F, X), "mlp fp32 tensor-core path: F=%d not eligible", F);
  TT_REQUIRE(n >= 1 && n <= (int64_t)0x7fffffff, "mlp fp32 tensor-core path: bad n");
  const int kat = (F + 31) / 32;
  const size_t smem = x3_smem_bytes(kat);
  CUtensorMap map;
  if (int rc = make_x_map(X, n, F, &map)) return rc;
  MlpTcParams p{prm, out, n, F, kat};
  TT_CUDA(cudaFuncSetAttribute(mlp_predict_x3_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)smem));
  const int64_t tiles = (n + kTcRows - 1) / kTcRows;
  const int grid = (int)std::min<int64_t>(tiles, sm_count());
  mlp_predict_x3_kernel<<<grid, kX3Threads, smem, st>>>(map, p);
  return check_launch("mlp predict fp32 (split tf32)");
}

}  // namespace tt

extern "C" int tt_mlp_predict_tf32(const float* prm, const float* X, int64_t n, int32_t F,
                                   float* out, tt_stream_t st) {
  if (n == 0) return TT_OK;
  return tt::mlp_predict_tc(prm, X, n, F, out, tt::as_stream(st));
}

extern "C" int tt_mlp_predict_f32tc(const float* prm, const float* X, int64_t n, int32_t F,
                                    float* out, tt_stream_t st) {
  if (n == 0) return TT_OK;
  return tt::mlp_predict_x3(prm, X, n, F, out, tt::as_stream(st));
}

extern "C" int32_t tt_mlp_f32tc_eligible(int32_t F, const float* X) { return tt::mlp_x3_eligible(F, X); }
