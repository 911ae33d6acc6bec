// ABI plumbing + standalone Adam (optim.py:33-46) and segmented pairwise
// logistic loss (mlp.py:25-35).
#include <stdarg.h>

#include <mutex>
#include <vector>

#include "tt_ops.cuh"

namespace tt {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s: launch failed: %s", what, cudaGetErrorString(e));
    return TT_ECUDA;
  }
  return TT_OK;
}

namespace {
struct KernelEntry {
  int dev;
  const void* f;
  int threads;  // -1: the shared-memory limit entry
  size_t smem;  // limit entry: the largest value set so far
  int per_sm;
};
std::mutex g_kernel_mu;
std::vector<KernelEntry> g_kernels;
}  // namespace

int kernel_smem(const void* kern, size_t smem) {
  if (smem <= 48 * 1024) return TT_OK;  // below the default limit
  int dev = 0;
  TT_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> g(g_kernel_mu);
  for (KernelEntry& e : g_kernels)
    if (e.dev == dev && e.f == kern && e.threads == -1) {
      if (e.smem < smem) {
        TT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        e.smem = smem;
      }
      return TT_OK;
    }
  TT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  g_kernels.push_back(KernelEntry{dev, kern, -1, smem, 0});
  return TT_OK;
}

int kernel_occupancy(const void* kern, int threads, size_t smem, int* per_sm) {
  if (int rc = kernel_smem(kern, smem)) return rc;
  int dev = 0;
  TT_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> g(g_kernel_mu);
  for (const KernelEntry& e : g_kernels)
    if (e.dev == dev && e.f == kern && e.threads == threads && e.smem == smem) {
      *per_sm = e.per_sm;
      return TT_OK;
    }
  TT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(per_sm, kern, threads, smem));
  g_kernels.push_back(KernelEntry{dev, kern, threads, smem, *per_sm});
  return TT_OK;
}

int sm_count() {
  int dev = 0, n = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 148;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 148;
  return n > 0 ? n : 148;
}

template <typename R>
__global__ void __launch_bounds__(256) adam_kernel(R* __restrict__ p, const R* __restrict__ g,
                                                   R* __restrict__ m, R* __restrict__ v, int64_t n,
                                                   const uint8_t* __restrict__ mask, AdamHyper h,
                                                   double c1, double c2) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (mask && !mask[i]) continue;
    R pi = p[i], mi = m[i], vi = v[i];
    adam_update<R>(pi, g[i], mi, vi, h, c1, c2);
    p[i] = pi;
    m[i] = mi;
    v[i] = vi;
  }
}

template <typename R>
__global__ void __launch_bounds__(256) rank_loss_kernel(const R* __restrict__ y,
                                                        const R* __restrict__ s,
                                                        const int64_t* __restrict__ off,
                                                        R* __restrict__ loss, R* __restrict__ grad) {
  extern __shared__ unsigned char smem_raw[];
  const int seg = blockIdx.x;
  const int64_t a = off[seg];
  const int n = (int)(off[seg + 1] - a);
  R* ys = reinterpret_cast<R*>(smem_raw);
  R* ss = ys + n;
  R* ds = ss + n;
  R* red = ds + n;
  for (int k = threadIdx.x; k < n; k += blockDim.x) {
    ys[k] = y[a + k];
    ss[k] = s[a + k];
  }
  __syncthreads();
  R l = rank_loss_block<R>(ys, ss, n, ds, red);
  for (int k = threadIdx.x; k < n; k += blockDim.x) grad[a + k] = ds[k];
  if (threadIdx.x == 0) loss[seg] = l;
}

template <typename R>
static int adam_launch(R* p, const R* g, R* m, R* v, int64_t n, const uint8_t* mask, double lr,
                       double b1, double b2, double eps, double c1, double c2, tt_stream_t st) {
  TT_REQUIRE(n >= 0, "adam: negative size");
  if (n == 0) return TT_OK;
  AdamHyper h{lr, b1, b2, eps};
  int grid = (int)((n + 255) / 256);
  if (grid > 4 * sm_count()) grid = 4 * sm_count();
  adam_kernel<R><<<grid, 256, 0, as_stream(st)>>>(p, g, m, v, n, mask, h, c1, c2);
  return check_launch("adam");
}

template <typename R>
static int rank_launch(const R* y, const R* s, const int64_t* off, int32_t n_segs, R* loss,
                       R* grad, tt_stream_t st, int64_t max_seg) {
  TT_REQUIRE(n_segs >= 0, "rank_loss: negative segment count");
  if (n_segs == 0) return TT_OK;
  size_t smem = (3 * (size_t)max_seg + 256) * sizeof(R);
  TT_REQUIRE(smem <= 200 * 1024, "rank_loss: segment too large (%lld)", (long long)max_seg);
  if (int rc = kernel_smem((const void*)rank_loss_kernel<R>, smem)) return rc;
  rank_loss_kernel<R><<<n_segs, 256, smem, as_stream(st)>>>(y, s, off, loss, grad);
  return check_launch("rank_loss");
}

}  // namespace tt

using namespace tt;

extern "C" {

int tt_abi_version(void) { return 1; }

const char* tt_last_error(void) { return tt::g_err; }

int tt_adam_step_f32(float* p, const float* g, float* m, float* v, int64_t n, const uint8_t* mask,
                     double lr, double b1, double b2, double eps, double c1, double c2,
                     tt_stream_t st) {
  return adam_launch<float>(p, g, m, v, n, mask, lr, b1, b2, eps, c1, c2, st);
}

int tt_adam_step_f64(double* p, const double* g, double* m, double* v, int64_t n,
                     const uint8_t* mask, double lr, double b1, double b2, double eps, double c1,
                     double c2, tt_stream_t st) {
  return adam_launch<double>(p, g, m, v, n, mask, lr, b1, b2, eps, c1, c2, st);
}

int tt_rank_loss_f32(const float* y, const float* s, const int64_t* off, int32_t n_segs,
                     int32_t max_seg, float* loss, float* grad, tt_stream_t st) {
  return rank_launch<float>(y, s, off, n_segs, loss, grad, st, max_seg);
}

int tt_rank_loss_f64(const double* y, const double* s, const int64_t* off, int32_t n_segs,
                     int32_t max_seg, double* loss, double* grad, tt_stream_t st) {
  return rank_launch<double>(y, s, off, n_segs, loss, grad, st, max_seg);
}

}  // extern "C"
