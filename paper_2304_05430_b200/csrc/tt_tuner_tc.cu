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
//                 (L2 scratch, fp16: the tf32 MMA keeps 10 mantissa bits of
//                 it anyway; 48 MB for 148 tiles of 128 x 10 steps instead of
//                 97 MB, so it stays in L2 instead of being written back to
//                 HBM); programs shorter than the tile hold state
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
#define TT_TC_TANH_APPROX 1
#include <cuda_fp16.h>

#include "tt_sm100.cuh"
#include "tt_tuner.cuh"

namespace tt {

using namespace sm100;

// clock64 marks of CTA 0 / row thread 0 on its first tile (debug aid,
// tt_debug_tc_phase_times): 0 tile start, 1+l after LSTM layer l, 20 after
// attention, 21 end; layer 1 step 1: 22 before A, 23 A arrived, 24 gates
// ready, 25 epilogue done.
static __device__ long long g_tc_phase[32];
#define TC_MARK(cond, i) \
  do {                   \
    if (cond) g_tc_phase[i] = clock64(); \
  } while (0)

// Activations for the tf32 scoring mode: ex2.approx.ftz / rcp.approx.ftz
// (same MUFU ops as Act<float>, without the denormal-range fix-ups).
__device__ __forceinline__ float ex2f(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float rcpf(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
#ifdef TT_TC_TANH_APPROX
// one SFU op per activation (MUFU.TANH): sigmoid(x) = 0.5 tanh(x/2) + 0.5
__device__ __forceinline__ float tanh_f(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float sig_f(float x) { return fmaf(0.5f, tanh_f(0.5f * x), 0.5f); }
#else
__device__ __forceinline__ float sig_f(float x) { return rcpf(1.f + ex2f(-1.4426950408889634f * x)); }
__device__ __forceinline__ float tanh_f(float x) {
  return 1.f - 2.f * rcpf(ex2f(2.8853900817779268f * x) + 1.f);
}
#endif

namespace sc {
constexpr int kRows = 128;
constexpr int kThreads = 288;  // warp 0: MMA; warps 1..4 and 5..8: two row groups
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
  __half* scratch;      // per CTA: [2][128][Tmax][64] layer outputs (ping-pong, fp16)
  const unsigned char* img;  // prepared B^T images (tuner_tc_prepare_kernel)
  int64_t scr_per_cta;  // halves
  const int32_t* perm;  // program of each tile slot, longest first (sort_programs_by_length)
};

struct __align__(8) ScBars {
  uint64_t a_full, d_full;
  uint64_t a_dir[2], d_dir[2];  // LSTM hand-offs per direction
  uint64_t w_full;              // weight image landed
  uint32_t tmem_base;
  int tmax;
};

// W[k][n] (row stride ld, rows [0, Kr) valid, zero for Kr <= k < Kcnt) ->
// K-major SW128 B^T tiles of N rows, at K offset kbase.  All threads.
__device__ void sc_stage(unsigned char* dst, int N, int kbase, int Kcnt, const float* __restrict__ src,
                         int ld, int Kr) {
  for (int i = blockIdx.y * blockDim.x + threadIdx.x; i < Kcnt * N; i += gridDim.y * blockDim.x) {
    const int n = i % N, k = i / N;
    const float v = k < Kr ? __ldg(src + (int64_t)k * ld + n) : 0.f;
    const int kk = kbase + k;
    *reinterpret_cast<float*>(dst + (kk >> 5) * (N * 128) + sw128_offset(n, kk & 31)) = v;
  }
}

__host__ __device__ inline int sc_slot_floats(int Tmax) {
  return 2 * sc::kD > Tmax * sc::kMaxHeads ? 2 * sc::kD : Tmax * sc::kMaxHeads;
}

__device__ __forceinline__ void cp_async16_cg(float* s, const float* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(s)), "l"(g) : "memory");
}
// L2 evict_last cache-policy loads/stores for the layer-output scratch, so
// the rows the next layer and the attention passes re-read stay in L2
// instead of streaming out with the input programs.
__device__ __forceinline__ uint64_t l2_keep_policy() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void st_keep(float* g, float4 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(g), "f"(v.x),
               "f"(v.y), "f"(v.z), "f"(v.w), "l"(pol)
               : "memory");
}
__device__ __forceinline__ float4 ld_keep(const float* g, uint64_t pol) {
  float4 v;
  asm volatile("ld.global.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(g), "l"(pol));
  return v;
}
__device__ __forceinline__ void st_keep_u4(void* g, uint4 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v4.u32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(g), "r"(v.x), "r"(v.y),
               "r"(v.z), "r"(v.w), "l"(pol)
               : "memory");
}
__device__ __forceinline__ uint4 ld_keep_u4(const void* g, uint64_t pol) {
  uint4 v;
  asm volatile("ld.global.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4], %5;"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(g), "l"(pol));
  return v;
}
__device__ __forceinline__ uint32_t pack_h2(float a, float b) {
  const __half2 h = __floats2half2_rn(a, b);
  return *reinterpret_cast<const uint32_t*>(&h);
}
__device__ __forceinline__ float2 unpack_h2(uint32_t u) {
  return __half22float2(*reinterpret_cast<const __half2*>(&u));
}
// 8 fp16 layer-output values (16 B) -> fp32
__device__ __forceinline__ void h8_to_f(uint4 u, float* f) {
  const float2 a = unpack_h2(u.x), b = unpack_h2(u.y), c = unpack_h2(u.z), d = unpack_h2(u.w);
  f[0] = a.x, f[1] = a.y, f[2] = b.x, f[3] = b.y, f[4] = c.x, f[5] = c.y, f[6] = d.x, f[7] = d.y;
}
// the next step's 128-B layer-output row into L1 ahead of its loads (the
// per-row attention loops otherwise wait one L2 round trip per step)
constexpr int kPf = 1;  // rows prefetched ahead (deeper measured no better)
__device__ __forceinline__ void prefetch_row_l1(const __half* g) {
  asm volatile("prefetch.global.L1 [%0];" ::"l"(g));
}
__device__ __forceinline__ void cp_async16_keep(float* s, const float* g, uint64_t pol) {
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(smem_u32(s)),
               "l"(g), "l"(pol)
               : "memory");
}

__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait0() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// Byte sizes / offsets of the per-layer LSTM images ([Wx_d ; Wh_d]^T for
// d = fw, bw) and of the attention/head image, all in the shared-memory
// byte layout (1024-B aligned atoms, so the swizzle is position independent).
__host__ __device__ inline uint32_t sc_lstm_image_bytes(int l) {
  return 2u * (uint32_t)(((l == 0 ? 32 : 64) + 32) / 32) * (128u * 128u);
}
__host__ __device__ inline int64_t sc_lstm_image_off(int l) {
  int64_t o = 0;
  for (int i = 0; i < l; ++i) o += sc_lstm_image_bytes(i);
  return o;
}
__host__ __device__ inline uint32_t sc_attn_image_bytes(const TDims& dm) {
  const int NK = dm.heads * 64, Zp = (64 + dm.C + 31) & ~31;
  return (uint32_t)(2 * 64 * 128 + 2 * NK * 128 + (NK / 32) * 64 * 128 + 2 * 64 * 128 +
                    (Zp / 32) * 64 * 128);
}
__host__ __device__ inline int64_t sc_attn_image_off(const TDims& dm) { return sc_lstm_image_off(dm.L); }

// D[tmem] = A[tmem](128 x K) . B (N rows K-major SW128 at b_smem); one lane.
__device__ __forceinline__ void sc_issue(uint32_t d, uint32_t a, uint32_t b_smem, int N, int K) {
  const uint32_t idesc = idesc_tf32(sc::kRows, N);
  for (int kk = 0; kk < K / 8; ++kk) {
    const uint64_t bd = sw128_desc(b_smem + (kk >> 2) * (N * 128) + (kk & 3) * 32);
    mma_tf32_ts(d, a + kk * 8, bd, idesc, kk != 0);
  }
}

// Attention/head B^T image at `base` (smem or global).  All threads.
__device__ void sc_stage_attn(unsigned char* base, const TDims& dm, const float* __restrict__ prm) {
  using namespace sc;
  const int heads = dm.heads, dh = dm.dh, C = dm.C;
  const int Z = kD + C, Zp = (Z + 31) & ~31;
  const int NK = heads * kD;
  unsigned char* bq_t = base;
  unsigned char* bk_t = bq_t + 2 * (kD * 128);
  unsigned char* bv_t = bk_t + 2 * (NK * 128);
  unsigned char* bo_t = bv_t + (NK / 32) * (kD * 128);
  unsigned char* b1_t = bo_t + 2 * (kD * 128);
  sc_stage(bq_t, kD, 0, kD, prm + dm.Wq, kD, kD);
  sc_stage(bo_t, kD, 0, kD, prm + dm.Wo, kD, kD);
  sc_stage(b1_t, kD, 0, Zp, prm + dm.W1, kHeadHidden, Z);
  // Bk^T[h*64 + k][c] = Wk[k][c] for c in head h ; Bv^T[c][h*64 + k] = Wv[k][c] for c in head h
  for (int i = blockIdx.y * blockDim.x + threadIdx.x; i < NK * kD; i += gridDim.y * blockDim.x) {
    const int nrow = i % NK, c = i / NK;
    const int h = nrow / kD, k = nrow % kD;
    const float v = (c / dh == h) ? __ldg(prm + dm.Wk + (int64_t)k * kD + c) : 0.f;
    *reinterpret_cast<float*>(bk_t + (c >> 5) * (NK * 128) + sw128_offset(nrow, c & 31)) = v;
  }
  for (int i = blockIdx.y * blockDim.x + threadIdx.x; i < kD * NK; i += gridDim.y * blockDim.x) {
    const int c = i % kD, kk = i / kD;
    const int h = kk / kD, k = kk % kD;
    const float v = (c / dh == h) ? __ldg(prm + dm.Wv + (int64_t)k * kD + c) : 0.f;
    *reinterpret_cast<float*>(bv_t + (kk >> 5) * (kD * 128) + sw128_offset(c, kk & 31)) = v;
  }
}

// Builds the B^T images of every LSTM layer (block l < L) and of the
// attention/head block (block L) in global memory, once per scoring call.
__global__ void __launch_bounds__(256) tuner_tc_prepare_kernel(TDims dm, const float* __restrict__ prm,
                                                                unsigned char* img) {
  using namespace sc;
  const int l = blockIdx.x;
  if (l < dm.L) {
    const int din = l == 0 ? dm.d0 : kD, kx = l == 0 ? 32 : kD, nat = (kx + kH) / 32;
    unsigned char* base = img + sc_lstm_image_off(l);
    for (int d = 0; d < 2; ++d) {
      unsigned char* bd = base + d * nat * (kG * 128);
      sc_stage(bd, kG, 0, kx, prm + dm.wx[l][d], kG, din);
      sc_stage(bd, kG, kx, kH, prm + dm.wh[l][d], kG, kH);
    }
  } else {
    sc_stage_attn(img + sc_attn_image_off(dm), dm, prm);
  }
}

__global__ void __launch_bounds__(sc::kThreads, 1) tuner_predict_tc_kernel(ScArgs a) {
  using namespace sc;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* base = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  unsigned char* Bs = base;                                         // B operands (128 KB)
  __shared__ float sbias[512];  // biases / head vectors (static: LDS, not generic loads)
  // LSTM: per-row x slots [128][2][64]; attention: per-row logits [128][Tmax][2] (aliased)
  float* sxs = reinterpret_cast<float*>(base + kBBytes);
  float* slog = sxs;
  ScBars* bars = reinterpret_cast<ScBars*>(sxs + (int64_t)kRows * sc_slot_floats(a.dm.Tmax));
  const TDims& dm = a.dm;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool rowt = warp >= 1;
  const int grp = (warp - 1) >> 2;           // row group (LSTM direction)
  const bool att = rowt && grp == 0;         // attention/head row threads
  const int row = ((warp & 3) << 5) | lane;  // TMEM lane quarter = warp % 4
  const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
  const int TM = dm.Tmax, heads = dm.heads, dh = dm.dh, C = dm.C;
  const int Z = kD + C, Zp = (Z + 31) & ~31;
  const uint32_t bs_addr = smem_u32(Bs);

  if (threadIdx.x == 0) {
    mbar_init(&bars->a_full, 2 * kRows);  // both row groups arrive
    mbar_init(&bars->d_full, 1);
    for (int d = 0; d < 2; ++d) {
      mbar_init(&bars->a_dir[d], kRows);
      mbar_init(&bars->d_dir[d], 1);
    }
    mbar_init(&bars->w_full, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<512>(&bars->tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bars->tmem_base;
  uint32_t ph = 0;
  uint32_t pd[2] = {0, 0};  // phase bits of the per-direction LSTM hand-offs
  const uint64_t pol_keep = l2_keep_policy();
  __half* scr0 = a.scratch + (int64_t)blockIdx.x * a.scr_per_cta;

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

  // bulk-copy a prepared B^T image into Bs (all threads; previous readers done)
  uint32_t pw = 0;
  auto load_image = [&](const unsigned char* src, uint32_t bytes) {
    __syncthreads();
    if (threadIdx.x == 0) {
      mbar_expect_tx(&bars->w_full, bytes);
      for (uint32_t off = 0; off < bytes; off += 32768)
        bulk_g2s(Bs + off, src + off, bytes - off < 32768 ? bytes - off : 32768, &bars->w_full);
    }
    mbar_wait(&bars->w_full, pw);
    pw ^= 1;
  };

  const int64_t n_tiles = (a.n + kRows - 1) / kRows;
  for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    const int64_t slot = tile * kRows + row;
    const int64_t p = slot < a.n ? (int64_t)a.perm[slot] : a.n;  // length-ordered tiles
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
    const bool pm = blockIdx.x == 0 && threadIdx.x == 32 && tile == blockIdx.x;
    TC_MARK(pm, 0);

    // ================================================================ LSTM
    // Per direction d its own hand-off pair (a_full[d] / d_full[d], phase
    // bit ph_d): the MMA of one direction runs while the row threads do the
    // other direction's epilogue, and the next step's x rows are loaded at
    // the start of an epilogue so their L2 latency hides behind it.
    // cell state lives in TMEM columns [448, 512) (c_fw | c_bw), not registers
    const uint32_t Cst = tmem + lane_off + 448;
    for (int l = 0; l < dm.L; ++l) {
      const int din = l == 0 ? dm.d0 : kD;
      const int kx = l == 0 ? 32 : kD;
      const int K = kx + kH;
      const int nat = K / 32;
      // ---- [Wx_d ; Wh_d]^T of both directions: one bulk copy of the image
      load_image(a.img + sc_lstm_image_off(l), sc_lstm_image_bytes(l));
      for (int d = 0; d < 2; ++d)
        for (int i = threadIdx.x; i < kG; i += blockDim.x) sbias[d * kG + i] = __ldg(a.prm + dm.bb[l][d] + i);
      __syncthreads();
      const __half* xin = scr0 + (int64_t)((l - 1) & 1) * kRows * TM * kD + (int64_t)row * TM * kD;
      __half* xout = scr0 + (int64_t)(l & 1) * kRows * TM * kD + (int64_t)row * TM * kD;
      // x row of direction d at step s (zeros past the program's end):
      // layer 0 reads the raw step row into registers; layers >= 1 copy the
      // previous layer's output row into this thread's shared-memory slot
      // with async 16-B copies (issued one half-step ahead, no registers).
      float* xslot = sxs + (int64_t)row * 2 * kD;  // per direction 64 fp16 (128 B) used
      auto fetch_x = [&](int d, int s) {
        if (l == 0) return;
        const bool ok = live && s < T;
        float* dst = xslot + d * kD;
        if (ok) {
          const __half* src = xin + (int64_t)(d == 0 ? s : T - 1 - s) * kD;
#pragma unroll
          for (int q = 0; q < 8; ++q)
            cp_async16_keep(dst + 4 * q, reinterpret_cast<const float*>(src + 8 * q), pol_keep);
        } else {
#pragma unroll
          for (int q = 0; q < 8; ++q) reinterpret_cast<uint4*>(dst)[q] = make_uint4(0u, 0u, 0u, 0u);
        }
        cp_async_commit();
      };
      auto put_x = [&](int d, int s, uint32_t Ad) {
        if (l == 0) {
          const bool ok = live && s < T;
          const float* xr = a.steps + (r0 + (ok ? (d == 0 ? s : T - 1 - s) : 0)) * dm.d0;
#pragma unroll
          for (int j0 = 0; j0 < 32; j0 += 16) {
            float v[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) v[i] = (ok && j0 + i < din) ? __ldg(xr + j0 + i) : 0.f;
            tmem_st16(Ad + j0, v);
          }
        } else {
          cp_async_wait0();
          const uint4* x8 = reinterpret_cast<const uint4*>(xslot + d * kD);
#pragma unroll
          for (int j0 = 0; j0 < kD; j0 += 16) {
            float v[16];
            h8_to_f(x8[j0 / 8], v);
            h8_to_f(x8[j0 / 8 + 1], v + 8);
            tmem_st16(Ad + j0, v);
          }
        }
      };
      if (rowt) {
        // row group `grp` runs direction d = grp: two independent recurrences,
        // two warps per SM sub-partition, so one direction's activation math
        // hides the other's latencies
        const int d = grp;
        const uint32_t Ad = tmem + lane_off + kColA + d * K;
        const uint32_t Gd = tmem + lane_off + kColG + d * kG;
        const uint32_t Cd = Cst + d * kH;
        const float* bd = sbias + d * kG;
        if (Tt > 0) {  // a tile of programs without steps issues no MMAs: no hand-off either
          float z[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
          for (int j0 = 0; j0 < kH; j0 += 8) {
            tmem_st8(Ad + kx + j0, z);
            tmem_st8(Cd + j0, z);
          }
          fetch_x(d, 0);
          put_x(d, 0, Ad);
          tmem_wait_st();
          tc_fence_before();
          mbar_arrive(&bars->a_dir[d]);
        }
        for (int s = 0; s < Tt; ++s) {
          const bool valid = live && s < T;
          const bool pms = pm && l == 1 && s == 1;
          TC_MARK(pms, 22);
          if (s + 1 < Tt) fetch_x(d, s + 1);  // in flight during the epilogue
          mbar_wait(&bars->d_dir[d], pd[d]);
          tc_fence_after();
          TC_MARK(pms, 24);
          const int t = d == 0 ? s : T - 1 - s;
          __half* orow = xout + (int64_t)t * kD + d * kH;
#pragma unroll
          for (int j0 = 0; j0 < kH; j0 += 16) {
            float gi[16], gf[16], gg[16], go[16], cc[16], h[16];
            tmem_ld16(Gd + j0, gi);
            tmem_ld16(Gd + kH + j0, gf);
            tmem_ld16(Gd + 2 * kH + j0, gg);
            tmem_ld16(Gd + 3 * kH + j0, go);
            tmem_ld16(Cd + j0, cc);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              const int j = j0 + i;
              const float ig = sig_f(gi[i] + bd[j]);
              const float fg = sig_f(gf[i] + bd[kH + j]);
              const float cg = tanh_f(gg[i] + bd[2 * kH + j]);
              const float og = sig_f(go[i] + bd[3 * kH + j]);
              cc[i] = fg * cc[i] + ig * cg;
              h[i] = og * tanh_f(cc[i]);
            }
            tmem_st16(Cd + j0, cc);
            tmem_st16(Ad + kx + j0, h);
            if (valid) {
#pragma unroll
              for (int q = 0; q < 2; ++q)
                st_keep_u4(orow + j0 + 8 * q,
                           make_uint4(pack_h2(h[8 * q], h[8 * q + 1]), pack_h2(h[8 * q + 2], h[8 * q + 3]),
                                      pack_h2(h[8 * q + 4], h[8 * q + 5]), pack_h2(h[8 * q + 6], h[8 * q + 7])),
                           pol_keep);
            }
          }
          if (s + 1 < Tt) {
            put_x(d, s + 1, Ad);
            tmem_wait_st();
            tc_fence_before();
            mbar_arrive(&bars->a_dir[d]);
          }
          pd[d] ^= 1;
          TC_MARK(pms, 25);
        }
      } else if (lane == 0) {
        // MMA lane: both directions, step by step
        for (int s = 0; s < Tt; ++s)
          for (int d = 0; d < 2; ++d) {
            mbar_wait(&bars->a_dir[d], pd[d]);
            tc_fence_after();
            sc_issue(tmem + kColG + d * kG, tmem + kColA + d * K, bs_addr + d * nat * (kG * 128), kG, K);
            mma_commit(&bars->d_dir[d]);
            pd[d] ^= 1;
          }
      }
      TC_MARK(pm, 1 + l);
    }

    // =========================================================== attention
    __syncthreads();
    const int L1 = (dm.L - 1) & 1;
    const __half* Srow = scr0 + (int64_t)L1 * kRows * TM * kD + (int64_t)row * TM * kD;
    // B layout: Wq^T | Bk^T | Bv^T | Wo^T | W1^T (image built by the prepare kernel)
    const int NK = heads * kD;  // r width and u width
    unsigned char* bq_t = Bs;
    unsigned char* bk_t = bq_t + 2 * (kD * 128);
    unsigned char* bv_t = bk_t + 2 * (NK * 128);
    unsigned char* bo_t = bv_t + (NK / 32) * (kD * 128);
    unsigned char* b1_t = bo_t + 2 * (kD * 128);
    load_image(a.img + sc_attn_image_off(dm), sc_attn_image_bytes(dm));
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
    TC_MARK(pm, 26);
    const uint32_t A0 = tmem + lane_off + kColA, D0 = tmem + lane_off + kColG;
    // Row group g owns head g for the per-step work (logits, softmax, u_h);
    // group 0 writes the other GEMM operands.  pooled never lives in
    // registers: it is written straight into the next GEMM's A columns.
    const bool hg = rowt && grp < heads;  // this thread owns head grp
    if (att) {
      float pool[kD];
#pragma unroll
      for (int k = 0; k < kD; ++k) pool[k] = 0.f;
      if (live) {
        for (int t = 0; t < kPf && t < T; ++t) prefetch_row_l1(Srow + (int64_t)t * kD);
        for (int t = 0; t < T; ++t) {
          const __half* sr = Srow + (int64_t)t * kD;
          if (t + kPf < T) prefetch_row_l1(Srow + (int64_t)(t + kPf) * kD);
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            float f[8];
            h8_to_f(ld_keep_u4(sr + 8 * q, pol_keep), f);
#pragma unroll
            for (int i = 0; i < 8; ++i) pool[8 * q + i] += f[i];
          }
        }
      }
      const float inv = (float)(T > 1 ? T : 1);
#pragma unroll
      for (int j0 = 0; j0 < kD; j0 += 16) {
        float v[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = pool[j0 + i] / inv;
        tmem_st16(A0 + j0, v);
      }
    }
    TC_MARK(pm, 27);
    const float sq = sqrtf((float)dh);
    // logits as [t][head][row]: lanes (rows) hit consecutive banks
    float* lg = slog + row;
    for (int u = 0; u < dm.U; ++u) {
      gemm(tmem + kColG, tmem + kColA, smem_u32(bq_t), kD, kD);  // q = pooled Wq
      if (att) {  // q + bq -> A (r = q Bk)
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
      gemm(tmem + kColG, tmem + kColA, smem_u32(bk_t), NK, kD);  // r_h = Wk[:, h] q_h
      TC_MARK(pm && u == 0, 28);
      if (rowt) {
        float r[kD], uvec[kD];
        if (hg) {
#pragma unroll
          for (int j0 = 0; j0 < kD; j0 += 16) {
            float v[16];
            tmem_ld16(D0 + grp * kD + j0, v);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 16; ++i) r[j0 + i] = v[i];
          }
        }
        if (hg && live) {
          float mx = -INFINITY, sum = 0.f;
          for (int t = 0; t < kPf && t < T; ++t) prefetch_row_l1(Srow + (int64_t)t * kD);
          for (int t = 0; t < T; ++t) {
            const __half* sr = Srow + (int64_t)t * kD;
            if (t + kPf < T) prefetch_row_l1(Srow + (int64_t)(t + kPf) * kD);
            float a0 = 0.f, a1 = 0.f;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              float f[8];
              h8_to_f(ld_keep_u4(sr + 8 * q, pol_keep), f);
#pragma unroll
              for (int i = 0; i < 8; i += 2) {
                a0 = fmaf(f[i], r[8 * q + i], a0);
                a1 = fmaf(f[i + 1], r[8 * q + i + 1], a1);
              }
            }
            const float v = (a0 + a1) / sq;
            lg[(t * kMaxHeads + grp) * kRows] = v;
            mx = fmaxf(mx, v);
          }
          for (int t = 0; t < T; ++t) {
            const float e = Act<float>::exp(lg[(t * kMaxHeads + grp) * kRows] - mx);
            lg[(t * kMaxHeads + grp) * kRows] = e;
            sum += e;
          }
#pragma unroll
          for (int k = 0; k < kD; ++k) uvec[k] = 0.f;
          for (int t = 0; t < kPf && t < T; ++t) prefetch_row_l1(Srow + (int64_t)t * kD);
          for (int t = 0; t < T; ++t) {
            const float al = lg[(t * kMaxHeads + grp) * kRows] / sum;
            const __half* sr = Srow + (int64_t)t * kD;
            if (t + kPf < T) prefetch_row_l1(Srow + (int64_t)(t + kPf) * kD);
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              float f[8];
              h8_to_f(ld_keep_u4(sr + 8 * q, pol_keep), f);
#pragma unroll
              for (int i = 0; i < 8; ++i) uvec[8 * q + i] = fmaf(al, f[i], uvec[8 * q + i]);
            }
          }
        }
        if (hg) {
          const bool ok = live;
#pragma unroll
          for (int j0 = 0; j0 < kD; j0 += 16) {
            float v[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) v[i] = ok ? uvec[j0 + i] : 0.f;
            tmem_st16(A0 + grp * kD + j0, v);
          }
        }
      }
      TC_MARK(pm && u == 0, 29);
      gemm(tmem + kColG, tmem + kColA, smem_u32(bv_t), kD, NK);  // mix = [u_h] blockdiag(Wv)
      if (att) {
#pragma unroll
        for (int j0 = 0; j0 < kD; j0 += 16) {
          float v[16];
          tmem_ld16(D0 + j0, v);
          tmem_wait_ld();
          tmem_st16(A0 + j0, v);
        }
      }
      gemm(tmem + kColG, tmem + kColA, smem_u32(bo_t), kD, kD);  // pooled = mix Wo + bo
      if (att) {
#pragma unroll
        for (int j0 = 0; j0 < kD; j0 += 16) {
          float v[16];
          tmem_ld16(D0 + j0, v);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] += sbias[kD + j0 + i];
          tmem_st16(A0 + j0, v);  // next pass's query input / the head's z[0:64]
        }
      }
    }
    TC_MARK(pm, 20);
    // ================================================================ head
    if (att) {
      for (int j0 = kD; j0 < Zp; j0 += 8) {
        float v[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = (live && j0 + i < Z) ? __ldg(a.ctx + p * C + (j0 + i - kD)) : 0.f;
        tmem_st8(A0 + j0, v);
      }
    }
    gemm(tmem + kColG, tmem + kColA, smem_u32(b1_t), kHeadHidden, Zp);
    if (att) {
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
    TC_MARK(pm, 21);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

static size_t sc_smem_bytes(int Tmax) {
  return 1024 + sc::kBBytes + (size_t)sc::kRows * sc_slot_floats(Tmax) * 4 +
         sizeof(ScBars) + 64;
}

constexpr size_t kScImageBytes = 1u << 20;  // >= every LSTM image (L <= 8) + the attention image

static int64_t tc_chunk() { return 4 * (int64_t)sm_count() * sc::kRows; }

size_t tuner_predict_tc_ws(int Tmax) {
  return align_up((size_t)sm_count() * 2 * sc::kRows * Tmax * sc::kD * sizeof(__half), 1024) + kScImageBytes +
         align_up((size_t)tc_chunk() * sizeof(int32_t), 1024) + align_up(sort_scratch_bytes(Tmax), 1024);
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
  a.scratch = static_cast<__half*>(ws);
  a.scr_per_cta = (int64_t)2 * sc::kRows * Tmax * sc::kD;
  unsigned char* img = static_cast<unsigned char*>(ws) +
                       align_up((size_t)sm_count() * a.scr_per_cta * sizeof(__half), 1024);
  TT_REQUIRE(sc_attn_image_off(a.dm) + sc_attn_image_bytes(a.dm) <= (int64_t)kScImageBytes - 1024,
             "tuner tf32 scoring: weight images exceed the workspace");
  a.img = img;
  tuner_tc_prepare_kernel<<<dim3(L + 1, 16), 256, 0, st>>>(a.dm, prm, img);
  if (int rc = kernel_smem((const void*)tuner_predict_tc_kernel, smem)) return rc;
  // chunks of 4 tiles per SM, each ordered by program length so a tile runs
  // for about its own programs' length (the result of a row does not depend
  // on its tile)
  int32_t* perm = reinterpret_cast<int32_t*>(img + kScImageBytes);
  void* sort_scr = reinterpret_cast<unsigned char*>(perm) + align_up((size_t)tc_chunk() * sizeof(int32_t), 1024);
  const int64_t chunk = tc_chunk();
  for (int64_t p0 = 0; p0 < n; p0 += chunk) {
    const int64_t nc = std::min<int64_t>(chunk, n - p0);
    if (int rc = sort_programs_by_length(rowoff + p0, nc, Tmax, perm, sort_scr, st)) return rc;
    a.rowoff = rowoff + p0;
    a.ctx = ctx + p0 * C;
    a.yhat = yhat + p0;
    a.n = nc;
    a.perm = perm;
    const int grid = (int)std::min<int64_t>((nc + sc::kRows - 1) / sc::kRows, sm_count());
    tuner_predict_tc_kernel<<<grid, sc::kThreads, smem, st>>>(a);
    if (int rc = check_launch("tuner predict tf32")) return rc;
  }
  return TT_OK;
}

}  // namespace tt

extern "C" {

int tt_debug_tc_phase_times(int64_t* out, int32_t n) {
  TT_REQUIRE(n >= 0 && n <= 32, "debug: n must be in [0, 32]");
  TT_CUDA(cudaMemcpyFromSymbol(out, tt::g_tc_phase, sizeof(long long) * n));
  return TT_OK;
}

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
