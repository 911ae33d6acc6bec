// K5 on the 5th-generation tensor cores: attention-tuner scoring (tuner.py
// _forward :227-285, predict :468-476) with every dense layer as a tcgen05
// GEMM tile of 128 programs (kind::tf32, fp32 accumulate in TMEM).
//
// One persistent CTA per SM, 160 threads:
//   warp 0        TMEM allocator (512 columns) and the single MMA-issuing lane
//   warps 1..4    one program per thread ("row thread"; TMEM lane = row)
//
// LSTM layer l, time step s of a tile (tile length = longest program):
//   row threads   write A_d = [x_t | h] for both directions into TMEM
//                 (tcgen05.st; x_t is the previous layer's output row, the
//                 backward direction reads t = T_p - 1 - s), arrive on bar_a
//   MMA lane      G_d[128 x 128] = A_d . [Wx_d ; Wh_d]   (A from TMEM, B =
//                 both directions' weights, K-major SWIZZLE_128B in smem),
//                 commit -> bar_d
//   row threads   tcgen05.ld the row's 128 gate pre-activations per
//                 direction, + bias, sigmoid/tanh, cell update (c in
//                 registers), h -> TMEM (next step's A) and the layer output
//                 (L2 scratch); programs shorter than the tile hold state
//                 (tuner.py:97-98 masked hold).
// Attention per pass (tuner.py:259-274) without materialising K and V:
//   q = pooled Wq + bq ; r_h = Wk[:, h] q_h          (two GEMMs)
//   logit_{t,h} = S_t . r_h / sqrt(dh), softmax over the program's steps,
//   u_h = sum_t alpha_{t,h} S_t                      (row thread, fp32 FMA)
//   mix = [u_h] . blockdiag(Wv_h) ; pooled = mix Wo + bo  (two GEMMs)
// Head: a1 = tanh([pooled | ctx] W1 + b1) (GEMM), y = sigmoid(a1 . W2 + b2).
//
// Precision: tf32 GEMM operands, fp32 everything else -- the "tf32" scoring
// mode with its own stated tolerance (tests/test_gpu_tuner_tc.py); the
// CUDA-core kernel (tt_tuner.cu) is the strict fp32 path.
#include "tt_sm100.cuh"
#include "tt_tuner.cuh"

namespace tt {

using namespace sm100;

namespace sc {
constexpr int kRows = 128;
constexpr int kThreads = 160;
constexpr int kH = 32, kD = 64, kG = 128;
constexpr uint32_t kColG = 0;    // G_fw [0,128) G_bw [128,256) ; attention D [0,128)
constexpr uint32_t kColA = 256;  // A_fw [256,256+K) A_bw [256+K,256+2K) ; attention A [256,384)
constexpr int kBBytes = 128 * 1024;
constexpr int kMaxHeads = 2;
}  // namespace sc

struct ScArgs {
  TDims dm;
  const float* prm;
  const float* steps;
  const int64_t* rowoff;
  const float* ctx;
  int64_t n;
  float* yhat;
  float* scratch;       // per CTA: [2][128][Tmax][64] layer outputs (ping-pong)
  int64_t scr_per_cta;  // floats
};

struct __align__(8) ScBars {
  uint64_t a_full, d_full;
  uint32_t tmem_base;
  int tmax;
};

// W[k][n] (row stride ld, rows [0, Kr) valid, zero for Kr <= k < Kcnt) ->
// K-major SW128 B^T tiles of N rows, at K offset kbase.  All threads.
__device__ void sc_stage(unsigned char* dst, int N, int kbase, int Kcnt, const float* __restrict__ src,
                         int ld, int Kr) {
  for (int i = threadIdx.x; i < Kcnt * N; i += blockDim.x) {
    const int n = i % N, k = i / N;
    const float v = k < Kr ? __ldg(src + (int64_t)k * ld + n) : 0.f;
    const int kk = kbase + k;
    *reinterpret_cast<float*>(dst + (kk >> 5) * (N * 128) + sw128_offset(n, kk & 31)) = v;
  }
}

// D[tmem] = A[tmem](128 x K) . B (N rows K-major SW128 at b_smem); one lane.
__device__ __forceinline__ void sc_issue(uint32_t d, uint32_t a, uint32_t b_smem, int N, int K) {
  const uint32_t idesc = idesc_tf32(sc::kRows, N);
  for (int kk = 0; kk < K / 8; ++kk) {
    const uint64_t bd = sw128_desc(b_smem + (kk >> 2) * (N * 128) + (kk & 3) * 32);
    mma_tf32_ts(d, a + kk * 8, bd, idesc, kk != 0);
  }
}

__global__ void __launch_bounds__(sc::kThreads, 1) tuner_predict_tc_kernel(ScArgs a) {
  using namespace sc;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* base = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  unsigned char* Bs = base;                                         // B operands (128 KB)
  float* sbias = reinterpret_cast<float*>(base + kBBytes);          // 512 floats
  float* slog = sbias + 512;                                        // [128][Tmax*heads] logits
  ScBars* bars = reinterpret_cast<ScBars*>(slog + (int64_t)kRows * a.dm.Tmax * kMaxHeads);
  const TDims& dm = a.dm;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool rowt = warp >= 1;
  const int row = ((warp & 3) << 5) | lane;  // TMEM lane quarter = warp % 4
  const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
  const int TM = dm.Tmax, heads = dm.heads, dh = dm.dh, C = dm.C;
  const int Z = kD + C, Zp = (Z + 31) & ~31;
  const uint32_t bs_addr = smem_u32(Bs);

  if (threadIdx.x == 0) {
    mbar_init(&bars->a_full, kRows);
    mbar_init(&bars->d_full, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<512>(&bars->tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bars->tmem_base;
  uint32_t ph = 0;
  float* scr0 = a.scratch + (int64_t)blockIdx.x * a.scr_per_cta;

  // one GEMM hand-off: row threads have written A; the MMA lane issues.
  auto gemm = [&](uint32_t d, uint32_t aa, uint32_t b_smem, int N, int K) {
    if (rowt) {
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(&bars->a_full);
    } else if (lane == 0) {
      mbar_wait(&bars->a_full, ph);
      tc_fence_after();
      sc_issue(d, aa, b_smem, N, K);
      mma_commit(&bars->d_full);
    }
    if (rowt) {
      mbar_wait(&bars->d_full, ph);
      tc_fence_after();
    }
    ph ^= 1;
  };

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
    if (live) atomicMax(&bars->tmax, T);
    __syncthreads();
    const int Tt = bars->tmax;

    // ================================================================ LSTM
    float c_fw[kH], c_bw[kH];
    for (int l = 0; l < dm.L; ++l) {
      const int din = l == 0 ? dm.d0 : kD;
      const int kx = l == 0 ? 32 : kD;
      const int K = kx + kH;
      const int nat = K / 32;
      // ---- stage [Wx_d ; Wh_d]^T for both directions (+ biases)
      __syncthreads();  // previous users of Bs are done
      for (int d = 0; d < 2; ++d) {
        unsigned char* bd = Bs + d * nat * (kG * 128);
        sc_stage(bd, kG, 0, kx, a.prm + dm.wx[l][d], kG, din);
        sc_stage(bd, kG, kx, kH, a.prm + dm.wh[l][d], kG, kH);
        for (int i = threadIdx.x; i < kG; i += blockDim.x) sbias[d * kG + i] = __ldg(a.prm + dm.bb[l][d] + i);
      }
      fence_proxy_async_smem();
      __syncthreads();
      const float* xin = scr0 + (int64_t)((l - 1) & 1) * kRows * TM * kD + (int64_t)row * TM * kD;
      float* xout = scr0 + (int64_t)(l & 1) * kRows * TM * kD + (int64_t)row * TM * kD;
#pragma unroll
      for (int j = 0; j < kH; ++j) c_fw[j] = c_bw[j] = 0.f;
      const uint32_t Af = tmem + lane_off + kColA, Ab = Af + K;
      const uint32_t Gf = tmem + lane_off + kColG, Gb = Gf + kG;
      for (int s = 0; s < Tt; ++s) {
        // tcgen05.ld/st are warp-collective: every row thread executes them;
        // rows past their program's end compute on stale inputs (their state
        // is dead for the rest of the layer) and never write the output.
        const bool valid = live && s < T;
        if (rowt) {
          // A_d = [x_t | h] ; h is already in place from the previous step
#pragma unroll
          for (int d = 0; d < 2; ++d) {
            const uint32_t Ad = d == 0 ? Af : Ab;
            if (s == 0) {
              float z[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
              for (int j0 = 0; j0 < kH; j0 += 8) tmem_st8(Ad + kx + j0, z);
            }
            const int t = d == 0 ? s : T - 1 - s;
            if (l == 0) {
              const float* xr = a.steps + (r0 + (valid ? t : 0)) * dm.d0;
              for (int j0 = 0; j0 < kx; j0 += 8) {
                float v[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) v[i] = (valid && j0 + i < din) ? __ldg(xr + j0 + i) : 0.f;
                tmem_st8(Ad + j0, v);
              }
            } else {
              const float4* xr = reinterpret_cast<const float4*>(xin + (int64_t)(valid ? t : 0) * kD);
#pragma unroll
              for (int j0 = 0; j0 < kD; j0 += 16) {
                float v[16];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                  const float4 f = valid ? __ldcg(xr + j0 / 4 + q) : make_float4(0.f, 0.f, 0.f, 0.f);
                  v[4 * q] = f.x, v[4 * q + 1] = f.y, v[4 * q + 2] = f.z, v[4 * q + 3] = f.w;
                }
                tmem_st16(Ad + j0, v);
              }
            }
          }
        }
        // both directions' gates: one hand-off, two GEMMs
        if (rowt) {
          tmem_wait_st();
          tc_fence_before();
          mbar_arrive(&bars->a_full);
        } else if (lane == 0) {
          mbar_wait(&bars->a_full, ph);
          tc_fence_after();
          sc_issue(tmem + kColG, tmem + kColA, bs_addr, kG, K);
          sc_issue(tmem + kColG + kG, tmem + kColA + K, bs_addr + nat * (kG * 128), kG, K);
          mma_commit(&bars->d_full);
        }
        if (rowt) {
          mbar_wait(&bars->d_full, ph);
          tc_fence_after();
#pragma unroll
          for (int d = 0; d < 2; ++d) {
            const uint32_t Gd = d == 0 ? Gf : Gb;
            const uint32_t Ad = d == 0 ? Af : Ab;
            const float* bd = sbias + d * kG;
            const int t = d == 0 ? s : T - 1 - s;
            float* orow = xout + (int64_t)t * kD + d * kH;
#pragma unroll
            for (int j0 = 0; j0 < kH; j0 += 8) {
              float gi[8], gf[8], gg[8], go[8], h[8];
              tmem_ld8(Gd + j0, gi);
              tmem_ld8(Gd + kH + j0, gf);
              tmem_ld8(Gd + 2 * kH + j0, gg);
              tmem_ld8(Gd + 3 * kH + j0, go);
              tmem_wait_ld();
#pragma unroll
              for (int i = 0; i < 8; ++i) {
                const int j = j0 + i;
                const float ig = Act<float>::sigmoid(gi[i] + bd[j]);
                const float fg = Act<float>::sigmoid(gf[i] + bd[kH + j]);
                const float cg = Act<float>::tanh(gg[i] + bd[2 * kH + j]);
                const float og = Act<float>::sigmoid(go[i] + bd[3 * kH + j]);
                float& cc = d == 0 ? c_fw[j] : c_bw[j];
                cc = fg * cc + ig * cg;
                h[i] = og * Act<float>::tanh(cc);
              }
              tmem_st8(Ad + kx + j0, h);
              if (valid) {
                reinterpret_cast<float4*>(orow + j0)[0] = make_float4(h[0], h[1], h[2], h[3]);
                reinterpret_cast<float4*>(orow + j0)[1] = make_float4(h[4], h[5], h[6], h[7]);
              }
            }
          }
        }
        ph ^= 1;
      }
    }

    // =========================================================== attention
    __syncthreads();
    const int L1 = (dm.L - 1) & 1;
    const float* Srow = scr0 + (int64_t)L1 * kRows * TM * kD + (int64_t)row * TM * kD;
    // B layout: Wq^T | Bk^T | Bv^T | Wo^T | W1^T
    const int NK = heads * kD;  // r width and u width
    unsigned char* bq_t = Bs;
    unsigned char* bk_t = bq_t + 2 * (kD * 128);
    unsigned char* bv_t = bk_t + 2 * (NK * 128);
    unsigned char* bo_t = bv_t + (NK / 32) * (kD * 128);
    unsigned char* b1_t = bo_t + 2 * (kD * 128);
    sc_stage(bq_t, kD, 0, kD, a.prm + dm.Wq, kD, kD);
    sc_stage(bo_t, kD, 0, kD, a.prm + dm.Wo, kD, kD);
    sc_stage(b1_t, kD, 0, Zp, a.prm + dm.W1, kHeadHidden, Z);
    // Bk^T[h*64 + k][c] = Wk[k][c] for c in head h ; Bv^T[c][h*64 + k] = Wv[k][c] for c in head h
    for (int i = threadIdx.x; i < NK * kD; i += blockDim.x) {
      const int nrow = i % NK, c = i / NK;  // Bk^T row nrow, K index c
      const int h = nrow / kD, k = nrow % kD;
      const float v = (c / dh == h) ? __ldg(a.prm + dm.Wk + (int64_t)k * kD + c) : 0.f;
      *reinterpret_cast<float*>(bk_t + (c >> 5) * (NK * 128) + sw128_offset(nrow, c & 31)) = v;
    }
    for (int i = threadIdx.x; i < kD * NK; i += blockDim.x) {
      const int c = i % kD, kk = i / kD;  // Bv^T row c, K index kk = h*64 + k
      const int h = kk / kD, k = kk % kD;
      const float v = (c / dh == h) ? __ldg(a.prm + dm.Wv + (int64_t)k * kD + c) : 0.f;
      *reinterpret_cast<float*>(bv_t + (kk >> 5) * (kD * 128) + sw128_offset(c, kk & 31)) = v;
    }
    for (int i = threadIdx.x; i < kD; i += blockDim.x) {
      sbias[i] = __ldg(a.prm + dm.bq + i);
      sbias[kD + i] = __ldg(a.prm + dm.bo + i);
    }
    for (int i = threadIdx.x; i < kHeadHidden; i += blockDim.x) {
      sbias[2 * kD + i] = __ldg(a.prm + dm.b1 + i);
      sbias[2 * kD + kHeadHidden + i] = __ldg(a.prm + dm.W2 + i);
    }
    if (threadIdx.x == 0) sbias[2 * kD + 2 * kHeadHidden] = __ldg(a.prm + dm.b2);
    fence_proxy_async_smem();
    __syncthreads();
    const uint32_t A0 = tmem + lane_off + kColA, D0 = tmem + lane_off + kColG;
    float pool[kD];
    if (live) {
#pragma unroll
      for (int k = 0; k < kD; ++k) pool[k] = 0.f;
      for (int t = 0; t < T; ++t) {
        const float4* sr = reinterpret_cast<const float4*>(Srow + (int64_t)t * kD);
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          const float4 f = __ldcg(sr + q);
          pool[4 * q] += f.x, pool[4 * q + 1] += f.y, pool[4 * q + 2] += f.z, pool[4 * q + 3] += f.w;
        }
      }
      const float inv = (float)(T > 1 ? T : 1);
#pragma unroll
      for (int k = 0; k < kD; ++k) pool[k] = pool[k] / inv;
    }
    const float sq = sqrtf((float)dh);
    float* lg = slog + (int64_t)row * TM * kMaxHeads;
    for (int u = 0; u < dm.U; ++u) {
      // q = pooled Wq + bq
      if (rowt) {
#pragma unroll
        for (int j0 = 0; j0 < kD; j0 += 16) {
          float v[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] = live ? pool[j0 + i] : 0.f;
          tmem_st16(A0 + j0, v);
        }
      }
      gemm(tmem + kColG, tmem + kColA, smem_u32(bq_t), kD, kD);
      if (rowt) {  // q -> A (r = q Bk)
#pragma unroll
        for (int j0 = 0; j0 < kD; j0 += 16) {
          float v[16];
          tmem_ld16(D0 + j0, v);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] += sbias[j0 + i];
          tmem_st16(A0 + j0, v);
        }
      }
      gemm(tmem + kColG, tmem + kColA, smem_u32(bk_t), NK, kD);
      float uvec[kMaxHeads * kD];
      if (rowt) {
        float r[kMaxHeads * kD];
#pragma unroll
        for (int j0 = 0; j0 < kMaxHeads * kD; j0 += 16) {
          if (j0 < NK) {
            float v[16];
            tmem_ld16(D0 + j0, v);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 16; ++i) r[j0 + i] = v[i];
          } else {
#pragma unroll
            for (int i = 0; i < 16; ++i) r[j0 + i] = 0.f;
          }
        }
        float mx[kMaxHeads], sum[kMaxHeads];
#pragma unroll
        for (int h = 0; h < kMaxHeads; ++h) mx[h] = -INFINITY, sum[h] = 0.f;
        if (live) {
          for (int t = 0; t < T; ++t) {
            const float4* sr = reinterpret_cast<const float4*>(Srow + (int64_t)t * kD);
            float acc[kMaxHeads];
#pragma unroll
            for (int h = 0; h < kMaxHeads; ++h) acc[h] = 0.f;
#pragma unroll
            for (int q = 0; q < 16; ++q) {
              const float4 f = __ldcg(sr + q);
#pragma unroll
              for (int h = 0; h < kMaxHeads; ++h) {
                acc[h] = fmaf(f.x, r[h * kD + 4 * q], acc[h]);
                acc[h] = fmaf(f.y, r[h * kD + 4 * q + 1], acc[h]);
                acc[h] = fmaf(f.z, r[h * kD + 4 * q + 2], acc[h]);
                acc[h] = fmaf(f.w, r[h * kD + 4 * q + 3], acc[h]);
              }
            }
#pragma unroll
            for (int h = 0; h < kMaxHeads; ++h) {
              const float v = acc[h] / sq;
              lg[t * kMaxHeads + h] = v;
              mx[h] = fmaxf(mx[h], v);
            }
          }
          for (int t = 0; t < T; ++t)
#pragma unroll
            for (int h = 0; h < kMaxHeads; ++h) {
              const float e = Act<float>::exp(lg[t * kMaxHeads + h] - mx[h]);
              lg[t * kMaxHeads + h] = e;
              sum[h] += e;
            }
        }
#pragma unroll
        for (int k = 0; k < kMaxHeads * kD; ++k) uvec[k] = 0.f;
        if (live) {
          for (int t = 0; t < T; ++t) {
            float al[kMaxHeads];
#pragma unroll
            for (int h = 0; h < kMaxHeads; ++h) al[h] = lg[t * kMaxHeads + h] / sum[h];
            const float4* sr = reinterpret_cast<const float4*>(Srow + (int64_t)t * kD);
#pragma unroll
            for (int q = 0; q < 16; ++q) {
              const float4 f = __ldcg(sr + q);
#pragma unroll
              for (int h = 0; h < kMaxHeads; ++h) {
                uvec[h * kD + 4 * q] = fmaf(al[h], f.x, uvec[h * kD + 4 * q]);
                uvec[h * kD + 4 * q + 1] = fmaf(al[h], f.y, uvec[h * kD + 4 * q + 1]);
                uvec[h * kD + 4 * q + 2] = fmaf(al[h], f.z, uvec[h * kD + 4 * q + 2]);
                uvec[h * kD + 4 * q + 3] = fmaf(al[h], f.w, uvec[h * kD + 4 * q + 3]);
              }
            }
          }
        }
#pragma unroll
        for (int j0 = 0; j0 < kMaxHeads * kD; j0 += 16) {
          if (j0 < NK) {
            float v[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) v[i] = uvec[j0 + i];
            tmem_st16(A0 + j0, v);
          }
        }
      }
      gemm(tmem + kColG, tmem + kColA, smem_u32(bv_t), kD, NK);  // mix = u . blockdiag(Wv)
      if (rowt) {
#pragma unroll
        for (int j0 = 0; j0 < kD; j0 += 16) {
          float v[16];
          tmem_ld16(D0 + j0, v);
          tmem_wait_ld();
          tmem_st16(A0 + j0, v);
        }
      }
      gemm(tmem + kColG, tmem + kColA, smem_u32(bo_t), kD, kD);  // pooled = mix Wo + bo
      if (rowt) {
#pragma unroll
        for (int j0 = 0; j0 < kD; j0 += 16) {
          float v[16];
          tmem_ld16(D0 + j0, v);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 16; ++i) pool[j0 + i] = v[i] + sbias[kD + j0 + i];
        }
      }
    }
    // ================================================================ head
    if (rowt) {
#pragma unroll
      for (int j0 = 0; j0 < kD; j0 += 16) {
        float v[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = pool[j0 + i];
        tmem_st16(A0 + j0, v);
      }
      for (int j0 = kD; j0 < Zp; j0 += 8) {
        float v[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = (live && j0 + i < Z) ? __ldg(a.ctx + p * C + (j0 + i - kD)) : 0.f;
        tmem_st8(A0 + j0, v);
      }
    }
    gemm(tmem + kColG, tmem + kColA, smem_u32(b1_t), kHeadHidden, Zp);
    if (rowt) {
      float acc = 0.f;
#pragma unroll
      for (int j0 = 0; j0 < kHeadHidden; j0 += 16) {
        float v[16];
        tmem_ld16(D0 + j0, v);
        tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 16; ++i)
          acc = fmaf(Act<float>::tanh(v[i] + sbias[2 * kD + j0 + i]),
                     sbias[2 * kD + kHeadHidden + j0 + i], acc);
      }
      if (live) a.yhat[p] = Act<float>::sigmoid(acc + sbias[2 * kD + 2 * kHeadHidden]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

static size_t sc_smem_bytes(int Tmax) {
  return 1024 + sc::kBBytes + 512 * 4 + (size_t)sc::kRows * Tmax * sc::kMaxHeads * 4 +
         sizeof(ScBars) + 64;
}

size_t tuner_predict_tc_ws(int Tmax) {
  return (size_t)sm_count() * 2 * sc::kRows * Tmax * sc::kD * sizeof(float);
}

int tuner_predict_tc(const float* prm, const float* steps, const int64_t* rowoff, const float* ctx,
                     int64_t n, int L, int H, int heads, int U, int d0, int C, int Tmax, float* yhat,
                     void* ws, size_t ws_bytes, cudaStream_t st) {
  TT_REQUIRE(H == 32, "tuner tf32 scoring: hidden size must be 32");
  TT_REQUIRE(L >= 1 && L <= kMaxLayers, "tuner tf32 scoring: bad layer count");
  TT_REQUIRE(heads >= 1 && heads <= sc::kMaxHeads && 64 % heads == 0,
             "tuner tf32 scoring: heads must be 1 or 2");
  TT_REQUIRE(d0 >= 1 && d0 <= 32, "tuner tf32 scoring: step width must be <= 32");
  TT_REQUIRE(C >= 0 && 64 + C <= 128, "tuner tf32 scoring: context width must be <= 64");
  TT_REQUIRE(U >= 1 && Tmax >= 1 && Tmax <= 4096, "tuner tf32 scoring: bad unroll / max steps");
  if (n == 0) return TT_OK;
  TT_REQUIRE(ws_bytes >= tuner_predict_tc_ws(Tmax), "tuner tf32 scoring: workspace too small");
  const size_t smem = sc_smem_bytes(Tmax);
  TT_REQUIRE(smem <= 227 * 1024, "tuner tf32 scoring: max steps %d too long for shared memory", Tmax);
  ScArgs a{};
  a.dm = make_dims(L, H, heads, U, d0, C, Tmax);
  a.prm = prm;
  a.steps = steps;
  a.rowoff = rowoff;
  a.ctx = ctx;
  a.n = n;
  a.yhat = yhat;
  a.scratch = static_cast<float*>(ws);
  a.scr_per_cta = (int64_t)2 * sc::kRows * Tmax * sc::kD;
  TT_CUDA(cudaFuncSetAttribute(tuner_predict_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)smem));
  const int64_t tiles = (n + sc::kRows - 1) / sc::kRows;
  const int grid = (int)std::min<int64_t>(tiles, sm_count());
  tuner_predict_tc_kernel<<<grid, sc::kThreads, smem, st>>>(a);
  return check_launch("tuner predict tf32");
}

}  // namespace tt

extern "C" {

size_t tt_tuner_predict_tf32_workspace_bytes(int32_t max_steps) {
  return tt::tuner_predict_tc_ws(max_steps);
}

int tt_tuner_predict_tf32(const float* prm, const float* steps, const int64_t* rowoff,
                          const float* ctx, int64_t n, int32_t L, int32_t H, int32_t heads,
                          int32_t U, int32_t d0, int32_t C, int32_t Tmax, float* yhat, void* ws,
                          size_t ws_bytes, tt_stream_t st) {
  return tt::tuner_predict_tc(prm, steps, rowoff, ctx, n, L, H, heads, U, d0, C, Tmax, yhat, ws,
                              ws_bytes, tt::as_stream(st));
}

}  // extern "C"
