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
// accurate tanh (see the split-precision kernel below): limits exact at +-inf
__device__ __forceinline__ float tanh_acc(float x) {
  float e, r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(2.8853900817779268f * x));
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(e + 1.f));
  return fmaf(-2.f, r, 1.f);
}

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
// operand is split into a tf32 head and a tf32 tail, v = hi + lo, and each
// dense layer runs as three tensor-core products accumulated in fp32,
//     A.B ~= Ahi.Bhi + Ahi.Blo + Alo.Bhi      (Alo.Blo ~ 2^-20 |A.B| dropped)
// so the layer error is ~2^-19 relative instead of tf32's 2^-10.
// kind::tf32 TRUNCATES its fp32 operands to tf32 (measured,
// tools/tf32_rounding_probe.py), so the raw fp32 X tile in shared memory IS
// Xhi = trunc(X) for the MMA, and only Xlo = X - trunc(X) (exact in fp32) has
// to be formed: by the converter warps, into TMEM operand slots.
//
//   warp 0       TMA producer: raw fp32 X atoms into an NST-stage ring
//   warp 1       TMEM allocator + GEMM1 issuer: per K step
//                  [acc1a | acc1b] += X.[W1hi | W1lo]   (one N = 128 MMA,
//                                                     A = X atom in smem)
//                  acc1a += Xlo.W1hi                     (A = Xlo in TMEM)
//                the epilogue adds the two halves
//   warp 2       GEMM2 issuer: [acc2a | acc2b] = h1hi.[W2hi | W2lo] (N = 128),
//                acc2a += h1lo.W2hi
//                (its own warp, so a ready tile's GEMM2 does not queue behind
//                the issue of the next tiles' GEMM1)
//   warps 3..10  converters: two per TMEM lane quarter, thread = tile row,
//                16 columns of the atom each: Xlo -> TMEM slot
//   warps 11..18 epilogue: h1 = tanh(acc1 + b1) -> (h1hi | h1lo) in place,
//                then tanh(acc2 + b2) . W3 + b3 -> score.
// Activations use the accurate exp-based tanh, 1 - 2 / (e^{2x} + 1), of the
// fp32 CUDA-core kernel (Act<float>::tanh) -- not tanh.approx -- with the
// flush-to-zero MUFU forms (ex2.approx.ftz, rcp.approx.ftz): the same two
// SFU ops without the denormal-range fix-ups (e^{2x} + 1 >= 1 never needs
// them), a third fewer instructions in the epilogue.
// TMEM (512 columns): 4 Xlo slots x 32 | 2 tile buffers x 128 (acc1a |
// acc1b -> h1hi | h1lo in place) | 1 acc2a | acc2b x 128 (read out right
// away by the epilogue).
constexpr int kX3Nst = 5;
constexpr int kX3Slots = 4;
constexpr int kX3Bufs = 2;
constexpr int kX3Threads = 608;
constexpr int kX3Conv = 256;  // converter threads

__device__ __forceinline__ float trunc_tf32(float v) {
  return __uint_as_float(__float_as_uint(v) & 0xffffe000u);
}

struct __align__(8) X3Bars {
  uint64_t full[kX3Nst], empty[kX3Nst];
  uint64_t op_full[kX3Slots], op_free[kX3Slots];
  uint64_t acc1_full[kX3Bufs], h1_full[kX3Bufs], buf_free[kX3Bufs];
  uint64_t acc2_full, acc2_free;
  uint32_t tmem_base;
};

__global__ void __launch_bounds__(kX3Threads, 1)
    mlp_predict_x3_kernel(const __grid_constant__ CUtensorMap tmap_x, MlpTcParams p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* base = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  unsigned char* xs = base;                                  // [NST] X atoms
  unsigned char* w1s = xs + kX3Nst * kAtomBytesX;            // [kat] [W1hi | W1lo]^T atoms (128 rows)
  unsigned char* w2s = w1s + p.kat * 2 * kAtomBytesW;        // [2] [W2hi | W2lo]^T atoms (128 rows)
  X3Bars* bars = reinterpret_cast<X3Bars*>(w2s + 4 * kAtomBytesW);
  __shared__ float s_b1[kTcHid], s_b2[kTcHid], s_w3[kTcHid];
  __shared__ float s_b3;
  __shared__ float s_part[2][2][kTcRows];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t n_tiles = (p.n + kTcRows - 1) / kTcRows;
  const int F = p.F;
  const int64_t ob1 = (int64_t)F * kTcHid, oW2 = ob1 + kTcHid, ob2 = oW2 + kTcHid * kTcHid,
                oW3 = ob2 + kTcHid, ob3 = oW3 + kTcHid;

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmap_x);
    for (int s = 0; s < kX3Nst; ++s) {
      mbar_init(&bars->full[s], 1);
      mbar_init(&bars->empty[s], kX3Conv + 1);  // converters read it + the MMAs retire
    }
    for (int s = 0; s < kX3Slots; ++s) {
      mbar_init(&bars->op_full[s], kX3Conv);
      mbar_init(&bars->op_free[s], 1);
    }
    for (int b = 0; b < kX3Bufs; ++b) {
      mbar_init(&bars->acc1_full[b], 1);
      mbar_init(&bars->h1_full[b], 256);
      mbar_init(&bars->buf_free[b], 1);
    }
    mbar_init(&bars->acc2_full, 1);
    mbar_init(&bars->acc2_free, 256);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(&bars->tmem_base);
  // weights: hi = trunc_tf32(w) (what the MMA sees of w anyway), lo = w - hi
  for (int i = threadIdx.x; i < p.kat * 32 * kTcHid; i += kX3Threads) {
    const int nrow = i % kTcHid, k = i / kTcHid;
    const float v = k < F ? p.prm[(int64_t)k * kTcHid + nrow] : 0.0f;
    const float hi = trunc_tf32(v);
    unsigned char* atom = w1s + (k >> 5) * 2 * kAtomBytesW;
    *reinterpret_cast<float*>(atom + sw128_offset(nrow, k & 31)) = hi;
    *reinterpret_cast<float*>(atom + sw128_offset(nrow + kTcHid, k & 31)) = v - hi;
  }
  for (int i = threadIdx.x; i < kTcHid * kTcHid; i += kX3Threads) {
    const int nrow = i % kTcHid, k = i / kTcHid;
    const float v = p.prm[oW2 + (int64_t)k * kTcHid + nrow];
    const float hi = trunc_tf32(v);
    unsigned char* atom = w2s + (k >> 5) * 2 * kAtomBytesW;
    *reinterpret_cast<float*>(atom + sw128_offset(nrow, k & 31)) = hi;
    *reinterpret_cast<float*>(atom + sw128_offset(nrow + kTcHid, k & 31)) = v - hi;
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
  constexpr uint32_t kOpCols = 32, kBufBase = kX3Slots * kOpCols, kBufCols = 128;
  constexpr uint32_t kAcc2 = kBufBase + kX3Bufs * kBufCols;  // 384
  const uint32_t my_tiles =
      (uint32_t)(n_tiles > blockIdx.x ? (n_tiles - 1 - blockIdx.x) / gridDim.x + 1 : 0);
  constexpr uint32_t idesc = idesc_tf32(kTcRows, kTcHid);

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
      constexpr uint32_t idesc2 = idesc_tf32(kTcRows, 2 * kTcHid);
      const uint32_t xa = smem_u32(xs), w1a = smem_u32(w1s);
      uint32_t it = 0;
      for (uint32_t t = 0; t < my_tiles; ++t) {
        const uint32_t b = t % kX3Bufs, bph = (t / kX3Bufs) & 1;
        const uint32_t acc1 = tmem + kBufBase + b * kBufCols;
        mbar_wait(&bars->buf_free[b], bph ^ 1);
        tc_fence_after();
        for (int kc = 0; kc < p.kat; ++kc, ++it) {
          const uint32_t s = it % kX3Nst, ph = (it / kX3Nst) & 1;
          const uint32_t os = it % kX3Slots, oph = (it / kX3Slots) & 1;
          mbar_wait(&bars->full[s], ph);
          mbar_wait(&bars->op_full[os], oph);
          tc_fence_after();
          const uint32_t alo = tmem + os * kOpCols;
          // K steps of 8 that hold real columns (the last atom of F = 164
          // has 4: one step instead of four)
          const int ksteps = min(4, (F - kc * 32 + 7) >> 3);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            if (kk >= ksteps) break;
            const uint64_t ad = sw128_desc(xa + s * kAtomBytesX + kk * 32);
            const uint64_t bd = sw128_desc(w1a + kc * 2 * kAtomBytesW + kk * 32);
            mma_tf32_ss(acc1, ad, bd, idesc2, (kc | kk) != 0);     // rows 0-63: W1hi, 64-127: W1lo
            mma_tf32_ts(acc1, alo + kk * 8, bd, idesc, 1);          // first 64 rows = W1hi
          }
          mma_commit(&bars->empty[s]);
          mma_commit(&bars->op_free[os]);
        }
        mma_commit(&bars->acc1_full[b]);
      }
    }
  } else if (warp == 2) {
    if (lane == 0) {
      constexpr uint32_t idesc2 = idesc_tf32(kTcRows, 2 * kTcHid);
      const uint32_t w2a = smem_u32(w2s);
      const uint32_t acc2 = tmem + kAcc2;
      for (uint32_t t = 0; t < my_tiles; ++t) {
        const uint32_t b = t % kX3Bufs, bph = (t / kX3Bufs) & 1;
        const uint32_t hhi = tmem + kBufBase + b * kBufCols, hlo = hhi + 64;
        mbar_wait(&bars->h1_full[b], bph);
        mbar_wait(&bars->acc2_free, (t & 1) ^ 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint64_t bd = sw128_desc(w2a + (kk >> 2) * 2 * kAtomBytesW + (kk & 3) * 32);
          mma_tf32_ts(acc2, hhi + kk * 8, bd, idesc2, kk != 0);  // [W2hi | W2lo]
          mma_tf32_ts(acc2, hlo + kk * 8, bd, idesc, 1);         // W2hi rows
        }
        mma_commit(&bars->acc2_full);
        mma_commit(&bars->buf_free[b]);  // h1 consumed: the buffer may take a new acc1
      }
    }
  } else if (warp < 11) {
    // converters: two warps per lane quarter, 16 columns of the atom each
    const int quarter = warp & 3;
    const int hc = (warp - 3) >> 2;
    const int row = quarter * 32 + lane;
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    uint32_t it = 0;
    for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
      for (int kc = 0; kc < p.kat; ++kc, ++it) {
        const uint32_t s = it % kX3Nst, ph = (it / kX3Nst) & 1;
        const uint32_t os = it % kX3Slots, oph = (it / kX3Slots) & 1;
        mbar_wait(&bars->full[s], ph);
        const unsigned char* atom = xs + s * kAtomBytesX;
        float lv[16];
#pragma unroll
        for (int c4 = 0; c4 < 4; ++c4) {
          const float4 v = *reinterpret_cast<const float4*>(atom + sw128_offset(row, hc * 16 + c4 * 4));
          lv[4 * c4 + 0] = v.x - trunc_tf32(v.x);
          lv[4 * c4 + 1] = v.y - trunc_tf32(v.y);
          lv[4 * c4 + 2] = v.z - trunc_tf32(v.z);
          lv[4 * c4 + 3] = v.w - trunc_tf32(v.w);
        }
        mbar_arrive(&bars->empty[s]);
        mbar_wait(&bars->op_free[os], oph ^ 1);
        tc_fence_after();
        tmem_st16(tmem + lane_off + os * kOpCols + hc * 16, lv);
        tmem_wait_st();
        tc_fence_before();
        mbar_arrive(&bars->op_full[os]);
      }
    }
  } else {
    // epilogue: warps 11..18, two per lane quarter, column half hf
    const int quarter = warp & 3;
    const int hf = (warp - 11) >> 2;
    const int row = quarter * 32 + lane;
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    const uint32_t acc2 = tmem + lane_off + kAcc2;
    uint32_t t = 0;
    for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++t) {
      const uint32_t b = t % kX3Bufs, bph = (t / kX3Bufs) & 1;
      const uint32_t acc1 = tmem + lane_off + kBufBase + b * kBufCols;
      const uint32_t hlo = acc1 + 64;
      mbar_wait(&bars->acc1_full[b], bph);
      tc_fence_after();
#pragma unroll
      for (int c0 = hf * 32; c0 < hf * 32 + 32; c0 += 16) {
        float v[16], lo[16];
        tmem_ld16(acc1 + c0, v);
        tmem_ld16(hlo + c0, lo);   // acc1b = X.W1lo
        tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const float h = tanh_acc((v[i] + lo[i]) + s_b1[c0 + i]);
          v[i] = trunc_tf32(h);
          lo[i] = h - v[i];
        }
        tmem_st16(acc1 + c0, v);
        tmem_st16(hlo + c0, lo);
      }
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(&bars->h1_full[b]);
      mbar_wait(&bars->acc2_full, t & 1);
      tc_fence_after();
      float a2[32], b2[32];
      tmem_ld16(acc2 + hf * 32, *reinterpret_cast<float(*)[16]>(a2));
      tmem_ld16(acc2 + hf * 32 + 16, *reinterpret_cast<float(*)[16]>(a2 + 16));
      tmem_ld16(acc2 + 64 + hf * 32, *reinterpret_cast<float(*)[16]>(b2));
      tmem_ld16(acc2 + 64 + hf * 32 + 16, *reinterpret_cast<float(*)[16]>(b2 + 16));
      tmem_wait_ld();
      tc_fence_before();
      mbar_arrive(&bars->acc2_free);  // acc2 read out: the next tile's GEMM2 may write it
      float acc = 0.f;
#pragma unroll
      for (int i = 0; i < 32; ++i)
        acc = fmaf(tanh_acc((a2[i] + b2[i]) + s_b2[hf * 32 + i]), s_w3[hf * 32 + i], acc);
      const int pb = t & 1;
      s_part[pb][hf][row] = acc;
      named_barrier(1, 256);
      const int64_t r = tile * kTcRows + row;
      if (hf == 0 && r < p.n) p.out[r] = (s_part[pb][0][row] + s_part[pb][1][row]) + s_b3;
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
  if (int rc = kernel_smem((const void*)mlp_predict_tc_kernel, smem)) return rc;
  const int64_t tiles = (n + kTcRows - 1) / kTcRows;
  const int grid = (int)std::min<int64_t>(tiles, sm_count());
  mlp_predict_tc_kernel<<<grid, kTcThreads, smem, st>>>(map, p);
  return check_launch("mlp predict tf32");
}

static size_t x3_smem_bytes(int kat) {
  return 1024 + (size_t)kX3Nst * kAtomBytesX + (size_t)(2 * kat + 4) * kAtomBytesW + sizeof(X3Bars) + 64;
}  // W1: kat atoms of 128 rows (= 2 kat 64-row atoms); W2 hi + lo: 4 atoms

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
  if (int rc = kernel_smem((const void*)mlp_predict_x3_kernel, smem)) return rc;
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
