// GBDT: squared-error boosting with exact greedy splits,
// bit-exact against estimators/gbdt.py:51-265 in float64.
//
// A tree grows level by level.  The F x n matrix `ord` holds, for every
// feature, the row indices sorted by that feature (the host's stable
// argsort, gbdt.py:109); every node of a level owns the same column range
// [start, start + m) in all F rows.  Per level:
//
//   node_total   one thread per node: G = 0.0 + pairwise_sum(g[ord0 seg]) --
//                numpy's pairwise summation (8 accumulators per block of
//                <= 128, halves split at multiples of 8) reproduced exactly,
//                so G equals the reference's g[samples].sum();
//   split_scan   one thread per (node, feature): the SEQUENTIAL prefix sum
//                of g over the feature-sorted rows (np.cumsum's order), the
//                score c^2/nl + (G-c)^2/nr with explicit round-to-nearest
//                operations (no FMA contraction), eligibility x[i] < x[i+1]
//                and min_leaf on both sides, first maximum kept (np.argmax);
//   decide       one CTA: per node the first feature with the largest gain
//                (strict >), leaf value G/m or the split; children get
//                level-order ids from a block scan (deterministic);
//   flag         one CTA per node: split nodes mark rows x <= cut, leaves
//                write the increment G/m to their rows;
//   partition    one warp per (split node, feature): stable ballot-scan
//                compaction of the segment into the other ord buffer (left
//                rows first, both halves keep their sorted order).
//
// The host renumbers the level-order ids into the reference's stack order
// (oracle/gbdt.py dfs_renumber).  Prediction walks each tree per row and
// accumulates out = out + lr * leaf in tree order, like gbdt.py:234-244.
#include "tt_common.cuh"

namespace tt {

// numpy pairwise_sum for float64 (numpy/_core/src/umath/loops_utils.h.src)
// over v(i), i in [o, o + len): < 8 terms sequentially from 0.0; <= 128 terms
// in 8 strided accumulators combined ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7))
// plus the tail; longer ranges split at n2 = len/2 rounded down to a
// multiple of 8.  np.add.reduce adds the result to the identity 0.0.
template <typename Get>
__device__ double np_pairwise(const Get& v, int64_t o, int64_t len) {
  if (len < 8) {
    double s = 0.0;
    for (int64_t i = 0; i < len; ++i) s = __dadd_rn(s, v(o + i));
    return s;
  }
  if (len <= 128) {
    double r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = v(o + j);
    int64_t i = 8;
    for (; i < len - (len % 8); i += 8) {
#pragma unroll
      for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], v(o + i + j));
    }
    double s = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                         __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (; i < len; ++i) s = __dadd_rn(s, v(o + i));
    return s;
  }
  int64_t n2 = len / 2;
  n2 -= n2 % 8;
  const double a = np_pairwise(v, o, n2);
  const double b = np_pairwise(v, o + n2, len - n2);
  return __dadd_rn(a, b);
}

template <typename Get>
__device__ double np_sum(const Get& v, int64_t n) {
  return __dadd_rn(0.0, np_pairwise(v, 0, n));
}

struct GbdtWs {
  int32_t* ord[2];      // [F][n] row indices, double buffered
  int32_t* list[2];     // node ids of the current / next level
  int32_t* cnt;         // [0], [1]: level sizes by parity; [2]: node count
  int32_t* nstart;      // [2n] segment start per node
  int32_t* nlen;        // [2n] segment length
  double* gtot;         // [2n]
  int8_t* found;        // [cap * F] per (level slot, feature)
  double* gain;
  double* cutv;
  uint8_t* flag;        // [n] row goes left
};

__global__ void gbdt_init_kernel(int32_t* cnt, int32_t* list0, int32_t* nstart, int32_t* nlen, int n,
                                 int32_t* feat, int32_t* left, int32_t* right) {
  cnt[0] = 1;  // level 0: the root
  cnt[1] = 0;
  cnt[2] = 1;  // node count
  list0[0] = 0;
  nstart[0] = 0;
  nlen[0] = n;
  feat[0] = -1;
  left[0] = -1;
  right[0] = -1;
}

// The same sum with the leaves (the <= 128-term blocks of the pairwise
// recursion) computed by the 32 lanes of a warp, then combined by lane 0 in
// the recursion's order: the same additions in the same order, one warp per
// node instead of one thread (the root's 16 k indirect loads no longer sit on
// one thread).  Nodes of <= 128 rows or more than kMaxLeaves leaves: lane 0
// alone, as before.
constexpr int kMaxLeaves = 2048;

__device__ double np_combine(const double* leaf, int64_t len, int& idx) {
  if (len <= 128) return leaf[idx++];
  int64_t n2 = len / 2;
  n2 -= n2 % 8;
  const double a = np_combine(leaf, n2, idx);
  const double b = np_combine(leaf, len - n2, idx);
  return __dadd_rn(a, b);
}

__global__ void __launch_bounds__(32) gbdt_node_total_warp_kernel(const double* __restrict__ g,
                                                                  const int32_t* __restrict__ ord0,
                                                                  const int32_t* list, const int32_t* cnt,
                                                                  int par, const int32_t* nstart,
                                                                  const int32_t* nlen, double* gtot) {
  __shared__ int32_t leaf_lo[kMaxLeaves];
  __shared__ int16_t leaf_len[kMaxLeaves];
  __shared__ double leaf_sum[kMaxLeaves];
  __shared__ int32_t st_lo[32], st_len[32];
  __shared__ int n_leaves;
  const int k = blockIdx.x, lane = threadIdx.x;
  if (k >= cnt[par]) return;
  const int node = list[k];
  const int32_t* o = ord0 + nstart[node];
  const int64_t n = nlen[node];
  auto v = [&](int64_t i) { return g[o[i]]; };
  if (n <= 128 || n > (int64_t)kMaxLeaves * 64) {
    if (lane == 0) gtot[node] = np_sum(v, n);
    return;
  }
  if (lane == 0) {  // leaves in order: depth-first, left first (stack in shared memory:
                    // the recursions below need the thread's small call stack)
    int sp = 0, nl = 0;
    st_lo[sp] = 0, st_len[sp] = (int32_t)n, ++sp;
    while (sp > 0) {
      --sp;
      const int32_t a = st_lo[sp], l = st_len[sp];
      if (l <= 128) {
        leaf_lo[nl] = (int32_t)a;
        leaf_len[nl] = (int16_t)l;
        ++nl;
        continue;
      }
      int32_t n2 = l / 2;
      n2 -= n2 % 8;
      st_lo[sp] = a + n2, st_len[sp] = l - n2, ++sp;  // right, popped second
      st_lo[sp] = a, st_len[sp] = n2, ++sp;
    }
    n_leaves = nl;
  }
  __syncwarp();
  for (int i = lane; i < n_leaves; i += 32) leaf_sum[i] = np_pairwise(v, leaf_lo[i], leaf_len[i]);
  __syncwarp();
  if (lane == 0) {
    int idx = 0;
    gtot[node] = __dadd_rn(0.0, np_combine(leaf_sum, n, idx));
  }
}

// The split search of one (node, feature) by a warp, 32 positions at a time:
// every lane folds the chunk's 32 gradient terms in order onto the running
// prefix (the same sequential additions as np.cumsum; lane j keeps the
// prefix at its position), then the lanes score their positions in parallel
// (the two divisions per position were the single thread's bottleneck) and
// a warp reduction keeps the first maximum (larger score, then smaller
// position; across chunks only a strictly larger score replaces the best).
// The same results as one thread scanning the positions in order.
__global__ void __launch_bounds__(128) gbdt_split_scan_warp_kernel(
    const double* __restrict__ Xc, const double* __restrict__ g, const int32_t* __restrict__ ord, int64_t n, int F,
    const int32_t* __restrict__ list, const int32_t* __restrict__ cnt, int par, const int32_t* nstart,
    const int32_t* nlen, const double* gtot, int depth, int max_depth, int min_leaf, int8_t* found, double* gain,
    double* cutv) {
  __shared__ double sg[4][32];
  const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t t = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;  // (slot, feature) pair
  const int slot = (int)(t / F), j = (int)(t % F);
  if (slot >= cnt[par]) return;  // warp-uniform
  const int node = list[slot];
  const int m = nlen[node];
  if (lane == 0) found[t] = 0;
  if (depth >= max_depth || m < 2 * min_leaf) return;
  const int32_t* o = ord + (int64_t)j * n + nstart[node];
  const double* x = Xc + (int64_t)j * n;
  const double G = gtot[node];
  const double md = (double)m;
  double c = g[o[0]];        // prefix through position i0 (all lanes)
  double xprev = x[o[0]];    // x at position i0 (for lane 0's xa)
  double best = -INFINITY, bxa = 0.0, bxb = 0.0;
  int bpos = -1;
  for (int i0 = 0; i0 < m - 1; i0 += 32) {
    const int i = i0 + lane;  // this lane's boundary: rows [0, i] left of it
    const bool in = i < m - 1;
    double xb = 0.0, gb = 0.0;
    if (in) {
      const int r1 = o[i + 1];
      xb = x[r1];
      gb = g[r1];
    }
    double xa = __shfl_up_sync(0xffffffffu, xb, 1);
    if (lane == 0) xa = xprev;
    sg[wib][lane] = gb;
    __syncwarp();
    // sequential fold: my prefix (before adding my own gb) and the chunk total
    double mine = c, run = c;
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      if (k == lane) mine = run;
      run = __dadd_rn(run, sg[wib][k]);
    }
    __syncwarp();
    const int nl = i + 1;
    double sc = -INFINITY;
    bool ok = in && xa < xb && nl >= min_leaf && m - nl >= min_leaf;
    if (ok) {
      const double nld = (double)nl;
      const double nrd = __dsub_rn(md, nld);
      const double rc = __dsub_rn(G, mine);
      sc = __dadd_rn(__ddiv_rn(__dmul_rn(mine, mine), nld), __ddiv_rn(__dmul_rn(rc, rc), nrd));
    }
    // first maximum of the chunk: larger score, then smaller position
    double rsc = sc;
    int rpos = ok ? i : 0x7fffffff;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const double osc = __shfl_xor_sync(0xffffffffu, rsc, off);
      const int opos = __shfl_xor_sync(0xffffffffu, rpos, off);
      if (opos != 0x7fffffff && (rpos == 0x7fffffff || osc > rsc || (osc == rsc && opos < rpos))) {
        rsc = osc;
        rpos = opos;
      }
    }
    if (rpos != 0x7fffffff && (bpos < 0 || rsc > best)) {
      best = rsc;
      bpos = rpos;
      const int src = rpos - i0;
      bxa = __shfl_sync(0xffffffffu, xa, src);
      bxb = __shfl_sync(0xffffffffu, xb, src);
    }
    c = run;
    xprev = __shfl_sync(0xffffffffu, xb, 31);
  }
  if (lane != 0 || bpos < 0) return;
  found[t] = 1;
  gain[t] = best;
  cutv[t] = __ddiv_rn(__dadd_rn(bxa, bxb), 2.0);
}

// one CTA (1024 threads): decisions + level-order child ids
__global__ void __launch_bounds__(1024) gbdt_decide_kernel(
    int F, const int32_t* __restrict__ list, int32_t* __restrict__ next_list, int32_t* cnt, int par,
    int32_t* nstart, int32_t* nlen, const double* gtot, const int8_t* found, const double* gain,
    const double* cutv, int32_t* feat, double* thr, int32_t* left, int32_t* right, double* val,
    int node_cap) {
  __shared__ int warp_tot[32];
  __shared__ int base_s;
  const int count = cnt[par];
  const int tid = threadIdx.x;
  if (tid == 0) base_s = 0;
  __syncthreads();
  for (int c0 = 0; c0 < count; c0 += blockDim.x) {
    const int slot = c0 + tid;
    int split = 0, bj = -1;
    double bg = 0.0;
    int node = -1;
    if (slot < count) {
      node = list[slot];
      for (int j = 0; j < F; ++j) {
        const int64_t t = (int64_t)slot * F + j;
        if (found[t] && (bj < 0 || gain[t] > bg)) {
          bg = gain[t];
          bj = j;
        }
      }
      split = bj >= 0;
    }
    // block exclusive scan of `split` (order = slot order)
    const int lane = tid & 31, w = tid >> 5;
    const unsigned bal = __ballot_sync(0xffffffffu, split);
    const int before = __popc(bal & ((1u << lane) - 1));
    if (lane == 0) warp_tot[w] = __popc(bal);
    __syncthreads();
    int woff = 0;
    for (int i = 0; i < w; ++i) woff += warp_tot[i];
    int total = 0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) total += warp_tot[i];
    const int rank = base_s + woff + before;
    if (slot < count) {
      if (split) {
        const int lid = cnt[2] + 2 * rank, rid = lid + 1;
        if (rid < node_cap) {
          feat[node] = bj;
          thr[node] = cutv[(int64_t)slot * F + bj];
          val[node] = 0.0;
          left[node] = lid;
          right[node] = rid;
          for (int c = 0; c < 2; ++c) {
            const int id = lid + c;
            feat[id] = -1;
            thr[id] = 0.0;
            left[id] = -1;
            right[id] = -1;
            val[id] = 0.0;
            nstart[id] = nstart[node];  // right child's start fixed by partition
            nlen[id] = 0;
          }
          next_list[2 * rank] = lid;
          next_list[2 * rank + 1] = rid;
        }
      } else {
        feat[node] = -1;
        thr[node] = 0.0;
        left[node] = -1;
        right[node] = -1;
        val[node] = __ddiv_rn(gtot[node], (double)nlen[node]);
      }
    }
    __syncthreads();
    if (tid == 0) base_s += total;
    __syncthreads();
  }
  if (tid == 0) {
    cnt[par ^ 1] = 2 * base_s;
    cnt[2] += 2 * base_s;
  }
}

// one CTA per level slot: split nodes flag their rows, leaves write increments
__global__ void gbdt_flag_kernel(const double* __restrict__ Xc, int64_t n, const int32_t* __restrict__ ord,
                                 const int32_t* __restrict__ list, const int32_t* cnt, int par,
                                 const int32_t* nstart, const int32_t* nlen, const int32_t* feat,
                                 const double* thr, const double* val, uint8_t* flag, double* incr) {
  const int slot = blockIdx.x;
  if (slot >= cnt[par]) return;
  const int node = list[slot];
  const int s = nstart[node], m = nlen[node];
  const int j = feat[node];
  if (j >= 0) {
    const int32_t* o = ord + (int64_t)j * n + s;
    const double* x = Xc + (int64_t)j * n;
    const double cut = thr[node];
    for (int i = threadIdx.x; i < m; i += blockDim.x) {
      const int r = o[i];
      flag[r] = x[r] <= cut;
    }
  } else {
    const int32_t* o = ord + s;
    const double v = val[node];
    for (int i = threadIdx.x; i < m; i += blockDim.x) incr[o[i]] = v;
  }
}

// one warp per (level slot, feature) of split nodes: stable partition
__global__ void gbdt_partition_kernel(const int32_t* __restrict__ src, int32_t* __restrict__ dst, int64_t n,
                                      int F, const int32_t* __restrict__ list, const int32_t* cnt, int par,
                                      int32_t* nstart, int32_t* nlen, const int32_t* feat,
                                      const int32_t* left, const int32_t* right,
                                      const uint8_t* __restrict__ flag) {
  const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int slot = (int)(wid / F), f = (int)(wid % F);
  if (slot >= cnt[par]) return;
  const int node = list[slot];
  if (feat[node] < 0) return;
  const int s = nstart[node], m = nlen[node];
  const int32_t* in = src + (int64_t)f * n + s;
  int32_t* out = dst + (int64_t)f * n + s;
  // pass 1: left count
  int nl = 0;
  for (int i0 = 0; i0 < m; i0 += 32) {
    const int i = i0 + lane;
    const int fl = i < m ? flag[in[i]] : 0;
    nl += __popc(__ballot_sync(0xffffffffu, fl));
  }
  int lo = 0, ro = nl;
  for (int i0 = 0; i0 < m; i0 += 32) {
    const int i = i0 + lane;
    int r = 0, fl = 0;
    if (i < m) {
      r = in[i];
      fl = flag[r];
    }
    const unsigned bl = __ballot_sync(0xffffffffu, fl && i < m);
    const unsigned br = __ballot_sync(0xffffffffu, !fl && i < m);
    const unsigned below = (1u << lane) - 1;
    if (i < m) {
      if (fl)
        out[lo + __popc(bl & below)] = r;
      else
        out[ro + __popc(br & below)] = r;
    }
    lo += __popc(bl);
    ro += __popc(br);
  }
  if (f == 0 && lane == 0) {
    const int l = left[node], rr = right[node];
    nstart[l] = s;
    nlen[l] = nl;
    nstart[rr] = s + nl;
    nlen[rr] = m - nl;
  }
}

__global__ void gbdt_update_kernel(double* pred, const double* incr, const double* y, double* g, double lr,
                                   int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double p = __dadd_rn(pred[i], __dmul_rn(lr, incr[i]));
    pred[i] = p;
    g[i] = __dsub_rn(y[i], p);
  }
}

__global__ void gbdt_residual_kernel(const double* pred, const double* y, double* g, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    g[i] = __dsub_rn(y[i], pred[i]);
}

// out[r] = (acc ? out[r] : base) then + lr * leaf(tree t, row r) for t in [0, n_trees)
__global__ void gbdt_predict_kernel(const int32_t* __restrict__ feat, const double* __restrict__ thr,
                                    const int32_t* __restrict__ left, const int32_t* __restrict__ right,
                                    const double* __restrict__ val, const int64_t* __restrict__ toff,
                                    int n_trees, double base, double lr, const double* __restrict__ X,
                                    int64_t n, int F, int64_t rstride, int64_t cstride, double* out,
                                    int acc) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
    double o = acc ? out[r] : base;
    const double* xr = X + r * rstride;
    for (int t = 0; t < n_trees; ++t) {
      const int64_t b = toff[t];
      int64_t node = b;
      for (int guard = 0; guard < 1 << 20; ++guard) {
        const int f = feat[node];
        if (f < 0) break;
        node = b + (xr[(int64_t)f * cstride] <= thr[node] ? left[node] : right[node]);
      }
      o = __dadd_rn(o, __dmul_rn(lr, val[node]));
    }
    out[r] = o;
  }
}

static GbdtWs carve(void* ws, int64_t n, int F, int64_t cap) {
  char* p = static_cast<char*>(ws);
  GbdtWs w{};
  auto take = [&](size_t bytes) {
    void* q = p;
    p += align_up(bytes, 256);
    return q;
  };
  w.ord[0] = (int32_t*)take((size_t)F * n * 4);
  w.ord[1] = (int32_t*)take((size_t)F * n * 4);
  w.list[0] = (int32_t*)take((size_t)(n + 1) * 4);
  w.list[1] = (int32_t*)take((size_t)(n + 1) * 4);
  w.cnt = (int32_t*)take(16);
  w.nstart = (int32_t*)take((size_t)(2 * n + 1) * 4);
  w.nlen = (int32_t*)take((size_t)(2 * n + 1) * 4);
  w.gtot = (double*)take((size_t)(2 * n + 1) * 8);
  w.found = (int8_t*)take((size_t)cap * F);
  w.gain = (double*)take((size_t)cap * F * 8);
  w.cutv = (double*)take((size_t)cap * F * 8);
  w.flag = (uint8_t*)take((size_t)n);
  (void)take(0);
  return w;
}

static int64_t level_cap(int64_t n, int max_depth) {
  // widest level: <= 2^max_depth nodes and <= n nodes (each holds >= 1 row)
  int64_t c = 1;
  for (int d = 0; d < max_depth && c < n; ++d) c *= 2;
  return c < n ? c : n;
}

}  // namespace tt

using namespace tt;

extern "C" {

size_t tt_gbdt_workspace_bytes(int64_t n, int32_t F, int32_t max_depth) {
  if (n < 1 || F < 1 || max_depth < 0) return 0;
  const int64_t cap = level_cap(n, max_depth);
  size_t b = 0;
  b += 2 * align_up((size_t)F * n * 4, 256);
  b += 2 * align_up((size_t)(n + 1) * 4, 256);
  b += align_up(16, 256);
  b += 2 * align_up((size_t)(2 * n + 1) * 4, 256);
  b += align_up((size_t)(2 * n + 1) * 8, 256);
  b += align_up((size_t)cap * F, 256) + 2 * align_up((size_t)cap * F * 8, 256);
  b += align_up((size_t)n, 256);
  return b;
}

int tt_gbdt_grow(const double* Xc, const double* g, const int32_t* root_order, int64_t n, int32_t F,
                 int32_t max_depth, int32_t min_leaf, int32_t* feat, double* thr, int32_t* left,
                 int32_t* right, double* val, int32_t* node_count, double* incr, void* ws,
                 size_t ws_bytes, tt_stream_t st) {
  TT_REQUIRE(n >= 1 && n < (1LL << 30), "gbdt: n must be in [1, 2^30)");
  TT_REQUIRE(F >= 1 && max_depth >= 0 && min_leaf >= 1, "gbdt: bad F / max_depth / min_leaf");
  TT_REQUIRE(ws_bytes >= tt_gbdt_workspace_bytes(n, F, max_depth), "gbdt: workspace too small");
  cudaStream_t s = as_stream(st);
  const int64_t cap = level_cap(n, max_depth);
  GbdtWs w = carve(ws, n, F, cap);
  TT_CUDA(cudaMemcpyAsync(w.ord[0], root_order, (size_t)F * n * 4, cudaMemcpyDeviceToDevice, s));
  gbdt_init_kernel<<<1, 1, 0, s>>>(w.cnt, w.list[0], w.nstart, w.nlen, (int)n, feat, left, right);
  const int node_cap = (int)(2 * n + 1);
  int cur = 0;
  int64_t width = 1;
  for (int d = 0; d <= max_depth; ++d) {
    const int par = d & 1;
    const int64_t pairs = width * F;
    gbdt_node_total_warp_kernel<<<(unsigned)width, 32, 0, s>>>(g, w.ord[cur], w.list[par], w.cnt, par, w.nstart,
                                                                w.nlen, w.gtot);
    gbdt_split_scan_warp_kernel<<<(unsigned)((pairs + 3) / 4), 128, 0, s>>>(
        Xc, g, w.ord[cur], n, F, w.list[par], w.cnt, par, w.nstart, w.nlen, w.gtot, d, max_depth, min_leaf,
        w.found, w.gain, w.cutv);
    gbdt_decide_kernel<<<1, 1024, 0, s>>>(F, w.list[par], w.list[par ^ 1], w.cnt, par, w.nstart, w.nlen,
                                          w.gtot, w.found, w.gain, w.cutv, feat, thr, left, right, val,
                                          node_cap);
    gbdt_flag_kernel<<<(unsigned)width, 256, 0, s>>>(Xc, n, w.ord[cur], w.list[par], w.cnt, par, w.nstart,
                                                     w.nlen, feat, thr, val, w.flag, incr);
    if (d < max_depth) {
      const int64_t threads = pairs * 32;
      gbdt_partition_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, s>>>(
          w.ord[cur], w.ord[cur ^ 1], n, F, w.list[par], w.cnt, par, w.nstart, w.nlen, feat, left, right,
          w.flag);
      cur ^= 1;
    }
    width = std::min<int64_t>(2 * width, std::min<int64_t>(cap, n));
  }
  TT_CUDA(cudaMemcpyAsync(node_count, w.cnt + 2, 4, cudaMemcpyDeviceToDevice, s));
  return check_launch("gbdt grow");
}

int tt_gbdt_update(double* pred, const double* incr, const double* y, double* g, double lr, int64_t n,
                   tt_stream_t st) {
  TT_REQUIRE(n >= 0, "gbdt update: negative n");
  if (n == 0) return TT_OK;
  const int grid = (int)std::min<int64_t>((n + 255) / 256, 8 * sm_count());
  if (incr == nullptr)
    gbdt_residual_kernel<<<grid, 256, 0, as_stream(st)>>>(pred, y, g, n);
  else
    gbdt_update_kernel<<<grid, 256, 0, as_stream(st)>>>(pred, incr, y, g, lr, n);
  return check_launch("gbdt update");
}

int tt_gbdt_predict(const int32_t* feat, const double* thr, const int32_t* left, const int32_t* right,
                    const double* val, const int64_t* tree_offsets, int32_t n_trees, double base, double lr,
                    const double* X, int64_t n, int32_t F, int32_t col_major, double* out, int32_t accumulate,
                    tt_stream_t st) {
  TT_REQUIRE(n >= 0 && F >= 1 && n_trees >= 0, "gbdt predict: bad sizes");
  if (n == 0) return TT_OK;
  const int grid = (int)std::min<int64_t>((n + 127) / 128, 16 * sm_count());
  const int64_t rs = col_major ? 1 : F, cs = col_major ? n : 1;
  gbdt_predict_kernel<<<grid, 128, 0, as_stream(st)>>>(feat, thr, left, right, val, tree_offsets, n_trees, base,
                                                      lr, X, n, F, rs, cs, out, accumulate);
  return check_launch("gbdt predict");
}

}  // extern "C"
