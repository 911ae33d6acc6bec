// K1 segmented pairwise-comparison-accuracy counter and K10 segmented top-k.
//
// Reference: metrics.py:46-58 (PCA over i<j, a tie agrees only with a tie),
//            metrics.py:61-75 (stable argsort(-score)[:k]).
//
// PCA design (exact integers, ALU-bound):
//   1. rank: per (task, vector) dense ranks of y and s as float32.  Ranking
//      preserves every pairwise sign (ties -> equal ranks, -0.0 == +0.0), so
//      the count is unchanged; ranks < 2^24 are exact in fp32.  Tasks up to
//      8192 entries: bitonic sort in shared memory + block scan; larger
//      tasks: competition ranks by counting (also order-preserving).
//   2. count: the upper triangle of each task's pair matrix is tiled into
//      1024x1024 blocks; a 256-thread CTA holds 4 rows per thread in
//      registers and streams the column block from shared memory.  Per pair:
//        d1 = ry_i - ry_j, d2 = rs_i - rs_j          (exact small integers)
//        conc += sat(d1*d2)      1 iff both orders strictly agree
//        nt   += sat(|d1|+|d2|)  1 iff the pair is not tied on both sides
//      agree = conc + (1 - nt).  Padding slots hold NaN, which .sat maps to 0,
//      so ragged edges need no predicates.  Diagonal blocks count the full
//      square and fold it: (S - n)/2.  Per-tile integer totals are combined
//      with 64-bit integer atomics (order-independent => deterministic).
#include <vector>

#include "tt_common.cuh"

namespace tt {

constexpr int kSortMax = 8192;  // in-smem bitonic sort bound (keys 8 B + idx 4 B)
constexpr int kBlk = 1024;      // pair tile edge
constexpr int kThr = 256;
constexpr int kRows = kBlk / kThr;  // rows per thread

struct PairTile {
  int32_t task;
  int32_t i0, j0;   // element offsets inside the task
  int32_t ni, nj;   // valid rows / columns
  int32_t diag;
  int64_t base;     // global element offset of the task
};

// ---------------------------------------------------------------- ranking --
__global__ void __launch_bounds__(512) rank_sort_kernel(const double* __restrict__ y,
                                                        const double* __restrict__ s,
                                                        const int64_t* __restrict__ off,
                                                        const int32_t* __restrict__ task_ids,
                                                        float2* __restrict__ ranks) {
  extern __shared__ unsigned char smem_raw[];
  const int task = task_ids[blockIdx.x];
  const int which = blockIdx.y;  // 0: labels, 1: scores
  const int64_t a = off[task];
  const int n = (int)(off[task + 1] - a);
  int np2 = 1;
  while (np2 < n) np2 <<= 1;
  double* key = reinterpret_cast<double*>(smem_raw);
  int* idx = reinterpret_cast<int*>(key + np2);
  int* scan = idx + np2;  // np2 ints
  const double* src = which == 0 ? y : s;
  for (int k = threadIdx.x; k < np2; k += blockDim.x) {
    if (k < n) {
      double v = src[a + k];
      key[k] = v == 0.0 ? 0.0 : v;  // canonical zero
      idx[k] = k;
    } else {
      key[k] = INFINITY;
      idx[k] = -1;
    }
  }
  __syncthreads();
  // bitonic sort ascending (ties: any order -- equal keys get equal ranks)
  for (int size = 2; size <= np2; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int k = threadIdx.x; k < np2 / 2; k += blockDim.x) {
        const int lo = 2 * k - (k & (stride - 1));
        const int hi = lo + stride;
        const bool up = (lo & size) == 0;
        const double kl = key[lo], kh = key[hi];
        if ((kl > kh) == up) {
          key[lo] = kh;
          key[hi] = kl;
          const int t = idx[lo];
          idx[lo] = idx[hi];
          idx[hi] = t;
        }
      }
      __syncthreads();
    }
  }
  // dense rank = inclusive prefix count of "new value" flags, minus one
  for (int k = threadIdx.x; k < np2; k += blockDim.x)
    scan[k] = (k < n && (k == 0 || key[k] != key[k - 1])) ? 1 : 0;
  __syncthreads();
  for (int d = 1; d < np2; d <<= 1) {  // Hillis-Steele, in place with two phases
    int add[kSortMax / 512];
    int c = 0;
    for (int k = threadIdx.x; k < np2; k += blockDim.x) add[c++] = k >= d ? scan[k - d] : 0;
    __syncthreads();
    c = 0;
    for (int k = threadIdx.x; k < np2; k += blockDim.x) scan[k] += add[c++];
    __syncthreads();
  }
  for (int k = threadIdx.x; k < n; k += blockDim.x) {
    float* dst = reinterpret_cast<float*>(&ranks[a + idx[k]]);
    dst[which] = (float)(scan[k] - 1);
  }
}

// competition rank (#strictly smaller) for tasks too large for the smem sort
__global__ void __launch_bounds__(256) rank_count_kernel(const double* __restrict__ y,
                                                         const double* __restrict__ s,
                                                         int64_t a, int n,
                                                         float2* __restrict__ ranks) {
  __shared__ double ty[256], ts[256];
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const double vy = i < n ? y[a + i] : 0.0, vs = i < n ? s[a + i] : 0.0;
  int cy = 0, cs = 0;
  for (int j0 = 0; j0 < n; j0 += 256) {
    __syncthreads();
    if (j0 + (int)threadIdx.x < n) {
      ty[threadIdx.x] = y[a + j0 + threadIdx.x];
      ts[threadIdx.x] = s[a + j0 + threadIdx.x];
    }
    __syncthreads();
    const int m = min(256, n - j0);
    for (int j = 0; j < m; ++j) {
      cy += ty[j] < vy;
      cs += ts[j] < vs;
    }
  }
  if (i < n) ranks[a + i] = make_float2((float)cy, (float)cs);
}

// ---------------------------------------------------------------- counting --
__global__ void __launch_bounds__(kThr) pca_tile_kernel(const float2* __restrict__ ranks,
                                                        const PairTile* __restrict__ tiles,
                                                        unsigned long long* __restrict__ correct) {
  __shared__ float4 col[kBlk / 2];
  __shared__ long long red[kThr / 32];
  const PairTile tl = tiles[blockIdx.x];
  const float NaN = __int_as_float(0x7fc00000);
  // stage the column block (pairs of elements per float4), NaN padded
  for (int k = threadIdx.x; k < kBlk / 2; k += kThr) {
    const int j = 2 * k;
    float2 e0 = j < tl.nj ? ranks[tl.base + tl.j0 + j] : make_float2(NaN, NaN);
    float2 e1 = j + 1 < tl.nj ? ranks[tl.base + tl.j0 + j + 1] : make_float2(NaN, NaN);
    col[k] = make_float4(e0.x, e0.y, e1.x, e1.y);
  }
  float ry[kRows], rs[kRows];
#pragma unroll
  for (int r = 0; r < kRows; ++r) {
    const int i = threadIdx.x + r * kThr;
    float2 e = i < tl.ni ? ranks[tl.base + tl.i0 + i] : make_float2(NaN, NaN);
    ry[r] = e.x;
    rs[r] = e.y;
  }
  __syncthreads();
  float conc[kRows], nt[kRows];
#pragma unroll
  for (int r = 0; r < kRows; ++r) conc[r] = nt[r] = 0.f;
#pragma unroll 4
  for (int k = 0; k < kBlk / 2; ++k) {
    const float4 q = col[k];
#pragma unroll
    for (int r = 0; r < kRows; ++r) {
      float d1 = ry[r] - q.x, d2 = rs[r] - q.y;
      conc[r] += __saturatef(d1 * d2);
      nt[r] += __saturatef(fabsf(d1) + fabsf(d2));
      d1 = ry[r] - q.z;
      d2 = rs[r] - q.w;
      conc[r] += __saturatef(d1 * d2);
      nt[r] += __saturatef(fabsf(d1) + fabsf(d2));
    }
  }
  // every accumulator <= 1024: exact in fp32
  long long v = 0;
#pragma unroll
  for (int r = 0; r < kRows; ++r) v += (long long)conc[r] - (long long)nt[r];
  v = warp_sum(v);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    long long tot = 0;
    for (int w = 0; w < kThr / 32; ++w) tot += red[w];
    long long agree;
    if (tl.diag) {
      const long long sq = tot + (long long)tl.ni * tl.ni;  // full square incl. diagonal
      agree = (sq - tl.ni) / 2;
    } else {
      agree = tot + (long long)tl.ni * tl.nj;
    }
    atomicAdd(&correct[tl.task], (unsigned long long)agree);
  }
}

// ------------------------------------------------------------------- top-k --
// One warp per task.  Order: score descending, then index ascending (numpy's
// stable argsort of -score; -0.0 == +0.0).
__global__ void topk_kernel(const double* __restrict__ y, const double* __restrict__ s,
                            const int64_t* __restrict__ off, int n_tasks, int k,
                            double* __restrict__ pick, double* __restrict__ best) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= n_tasks) return;
  const int64_t a = off[warp];
  const int n = (int)(off[warp + 1] - a);
  double ymax = -INFINITY;
  for (int i = lane; i < n; i += 32) ymax = fmax(ymax, y[a + i]);
  ymax = warp_max(ymax);
  const int kk = min(k, n);
  double last_s = INFINITY;
  int last_i = -1;
  double pmax = -INFINITY;
  for (int r = 0; r < kk; ++r) {
    double bs = -INFINITY;
    int bi = 0x7fffffff;
    for (int i = lane; i < n; i += 32) {
      const double v = s[a + i];
      const bool eligible = r == 0 || v < last_s || (v == last_s && i > last_i);
      if (eligible && (v > bs || (v == bs && i < bi))) {
        bs = v;
        bi = i;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double os = __shfl_xor_sync(0xffffffffu, bs, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (os > bs || (os == bs && oi < bi)) {
        bs = os;
        bi = oi;
      }
    }
    last_s = bs;
    last_i = bi;
    pmax = fmax(pmax, y[a + bi]);
  }
  if (lane == 0) {
    pick[warp] = pmax;
    best[warp] = ymax;
  }
}

static void plan(const int64_t* h_off, int32_t n_tasks, std::vector<PairTile>* tiles,
                 std::vector<int32_t>* sort_tasks, std::vector<int32_t>* big_tasks,
                 int64_t* total) {
  *total = n_tasks > 0 ? h_off[n_tasks] - h_off[0] : 0;
  for (int t = 0; t < n_tasks; ++t) {
    const int64_t n = h_off[t + 1] - h_off[t];
    if (n < 2) continue;
    if (n <= kSortMax)
      sort_tasks->push_back(t);
    else
      big_tasks->push_back(t);
    const int nb = (int)((n + kBlk - 1) / kBlk);
    for (int I = 0; I < nb; ++I)
      for (int J = I; J < nb; ++J) {
        PairTile p;
        p.task = t;
        p.i0 = I * kBlk;
        p.j0 = J * kBlk;
        p.ni = (int)std::min<int64_t>(kBlk, n - p.i0);
        p.nj = (int)std::min<int64_t>(kBlk, n - p.j0);
        p.diag = I == J;
        p.base = h_off[t];
        tiles->push_back(p);
      }
  }
}

}  // namespace tt

using namespace tt;

extern "C" {

size_t tt_pca_workspace_bytes(const int64_t* h_off, int32_t n_tasks) {
  std::vector<PairTile> tiles;
  std::vector<int32_t> st, bt;
  int64_t total = 0;
  plan(h_off, n_tasks, &tiles, &st, &bt, &total);
  return align_up((size_t)total * sizeof(float2), 256) +
         align_up(tiles.size() * sizeof(PairTile), 256) + align_up(st.size() * 4 + 4, 256) +
         align_up(sizeof(int64_t) * (n_tasks + 1), 256);
}

int tt_pca_counts(const double* d_y, const double* d_s, const int64_t* h_off, int32_t n_tasks,
                  int64_t* d_correct, void* d_ws, size_t ws_bytes, tt_stream_t stream) {
  TT_REQUIRE(n_tasks >= 0, "pca: negative task count");
  if (n_tasks == 0) return TT_OK;
  cudaStream_t st = as_stream(stream);
  std::vector<PairTile> tiles;
  std::vector<int32_t> sort_tasks, big_tasks;
  int64_t total = 0;
  plan(h_off, n_tasks, &tiles, &sort_tasks, &big_tasks, &total);
  const size_t need = tt_pca_workspace_bytes(h_off, n_tasks);
  TT_REQUIRE(ws_bytes >= need, "pca: workspace %zu < %zu", ws_bytes, need);
  char* ws = static_cast<char*>(d_ws);
  float2* ranks = reinterpret_cast<float2*>(ws);
  ws += align_up((size_t)total * sizeof(float2), 256);
  PairTile* d_tiles = reinterpret_cast<PairTile*>(ws);
  ws += align_up(tiles.size() * sizeof(PairTile), 256);
  int32_t* d_sort = reinterpret_cast<int32_t*>(ws);
  ws += align_up(sort_tasks.size() * 4 + 4, 256);
  int64_t* d_off = reinterpret_cast<int64_t*>(ws);
  // ranks are addressed with the task's absolute offset, so shift the base
  ranks -= h_off[0];
  TT_CUDA(cudaMemsetAsync(d_correct, 0, sizeof(int64_t) * n_tasks, st));
  if (tiles.empty()) return TT_OK;
  TT_CUDA(cudaMemcpyAsync(d_tiles, tiles.data(), tiles.size() * sizeof(PairTile),
                          cudaMemcpyHostToDevice, st));
  if (!sort_tasks.empty()) {
    TT_CUDA(cudaMemcpyAsync(d_sort, sort_tasks.data(), sort_tasks.size() * 4,
                            cudaMemcpyHostToDevice, st));
    int maxn = 0;
    for (int t : sort_tasks) maxn = std::max<int>(maxn, (int)(h_off[t + 1] - h_off[t]));
    int np2 = 1;
    while (np2 < maxn) np2 <<= 1;
    const size_t smem = (size_t)np2 * (8 + 4 + 4);
    TT_CUDA(cudaMemcpyAsync(d_off, h_off, sizeof(int64_t) * (n_tasks + 1), cudaMemcpyHostToDevice,
                            st));
    if (int rc = kernel_smem((const void*)rank_sort_kernel, smem)) return rc;
    dim3 grid((unsigned)sort_tasks.size(), 2);
    rank_sort_kernel<<<grid, 512, smem, st>>>(d_y, d_s, d_off, d_sort, ranks);
    if (int rc = check_launch("pca rank_sort")) return rc;
  }
  for (int t : big_tasks) {
    const int n = (int)(h_off[t + 1] - h_off[t]);
    rank_count_kernel<<<(n + 255) / 256, 256, 0, st>>>(d_y, d_s, h_off[t], n, ranks);
    if (int rc = check_launch("pca rank_count")) return rc;
  }
  pca_tile_kernel<<<(unsigned)tiles.size(), kThr, 0, st>>>(
      ranks, d_tiles, reinterpret_cast<unsigned long long*>(d_correct));
  if (int rc = check_launch("pca tiles")) return rc;
  return TT_OK;
}

int tt_topk(const double* d_y, const double* d_s, const int64_t* d_off, int32_t n_tasks, int32_t k,
            double* d_pick, double* d_best, tt_stream_t stream) {
  TT_REQUIRE(n_tasks >= 0 && k >= 1, "topk: bad arguments");
  if (n_tasks == 0) return TT_OK;
  const int threads = 256;
  const int blocks = (n_tasks * 32 + threads - 1) / threads;
  topk_kernel<<<blocks, threads, 0, as_stream(stream)>>>(d_y, d_s, d_off, n_tasks, k, d_pick,
                                                          d_best);
  return check_launch("topk");
}

}  // extern "C"
