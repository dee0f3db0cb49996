// Small-n path (n <= 8): dispatch to the per-n instantiations
// (ks_small_n<n>.cu); the kernels themselves are in ks_small_impl.cuh.
#include <cuda_runtime.h>

#include <mutex>
#include <set>
#include <utility>

#include "ks_internal.cuh"

namespace ks {
namespace smalld {
template <int N> cudaError_t factor_n(const SmallFactorArgs &, cudaStream_t);
template <int N> cudaError_t backward_n(const SmallBackwardArgs &, cudaStream_t);
template <int N> cudaError_t whiten_n(const SmallWhitenArgs &, cudaStream_t, int *);
template <int N> cudaError_t factor_tail_n(const SmallTailArgs &, cudaStream_t);
template <int N> int tail_cols_n();
template <int N> cudaError_t backward_tail_n(const SmallBwdTailArgs &, cudaStream_t);
}  // namespace smalld

using namespace smalld;

size_t small_entry_doubles(int n) { return (size_t)entry_doubles(n); }
int64_t small_rrec_doubles(int n) { return 2ll * n * n + n + (int64_t)n * (n + 1) / 2; }

#ifdef KS_SMALL_ONLY6   // register-allocation experiments: instantiate n = 6 only
#define KS_SMALL_DISPATCH(fn, n, ...)            \
  switch (n) {                                  \
    case 6: return fn<6>(__VA_ARGS__);          \
    default: return cudaErrorInvalidValue;      \
  }
#else
#define KS_SMALL_DISPATCH(fn, n, ...)            \
  switch (n) {                                  \
    case 1: return fn<1>(__VA_ARGS__);          \
    case 2: return fn<2>(__VA_ARGS__);          \
    case 3: return fn<3>(__VA_ARGS__);          \
    case 4: return fn<4>(__VA_ARGS__);          \
    case 5: return fn<5>(__VA_ARGS__);          \
    case 6: return fn<6>(__VA_ARGS__);          \
    case 7: return fn<7>(__VA_ARGS__);          \
    case 8: return fn<8>(__VA_ARGS__);          \
    default: return cudaErrorInvalidValue;      \
  }
#endif

cudaError_t launch_small_factor(const SmallFactorArgs &a, int n, cudaStream_t s) {
  KS_SMALL_DISPATCH(factor_n, n, a, s)
}
cudaError_t launch_small_backward(const SmallBackwardArgs &a, int n, cudaStream_t s) {
  KS_SMALL_DISPATCH(backward_n, n, a, s)
}
cudaError_t launch_small_factor_tail(const SmallTailArgs &t, int n, cudaStream_t s) {
  KS_SMALL_DISPATCH(factor_tail_n, n, t, s)
}
cudaError_t launch_small_backward_tail(const SmallBwdTailArgs &t, int n, cudaStream_t s) {
  KS_SMALL_DISPATCH(backward_tail_n, n, t, s)
}
int small_tail_max_cols(int n) {
#define KS_TAIL_COLS(k) \
  if (n == k) return tail_cols_n<k>();
#ifdef KS_SMALL_ONLY6
  KS_TAIL_COLS(6)
#else
  KS_TAIL_COLS(1) KS_TAIL_COLS(2) KS_TAIL_COLS(3) KS_TAIL_COLS(4) KS_TAIL_COLS(5) KS_TAIL_COLS(6) KS_TAIL_COLS(7)
  KS_TAIL_COLS(8)
#endif
#undef KS_TAIL_COLS
  return 0;
}
cudaError_t launch_small_whiten(const SmallWhitenArgs &a, cudaStream_t s, int *nlaunch) {
  KS_SMALL_DISPATCH(whiten_n, a.n, a, s, nlaunch)
}

// Gathered AoS boundary entries (rank r at recv + r E) -> pair-interleaved
// tiles: element e of column t at (t >> 6) 64E + (t & 1) 32E + 32 e + ((t >> 1) & 31).
__global__ void boundary_ptile_kernel(const double *__restrict__ recv, double *__restrict__ out, int P, int E) {
  const int64_t total = (int64_t)P * E;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = idx / E, e = idx - t * E;
    out[(t >> 6) * 64 * E + (t & 1) * 32 * E + 32 * e + ((t >> 1) & 31)] = recv[idx];
  }
}
cudaError_t launch_boundary_ptile(const double *recv, double *out, int P, int n, cudaStream_t s) {
  const int E = (int)entry_doubles(n);
  const int64_t total = (int64_t)P * E;
  boundary_ptile_kernel<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(recv, out, P, E);
  return cudaGetLastError();
}

__global__ void update_y_kernel(const double *__restrict__ M, int64_t sM, const double *__restrict__ o, int64_t so,
                                const int32_t *__restrict__ m, int mx, int rc, int64_t N, double *__restrict__ y,
                                int ptiled) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  const double *Mi = M + i * sM, *oi = o + i * so;
  const int mi = m ? m[i] : mx;
  // element r of step i (the output doubles as the substitution's scratch)
  auto at = [&](int r) -> double & {
    return ptiled ? y[(i >> 6) * 64 * rc + (i & 1) * 32 * rc + 32 * r + ((i >> 1) & 31)] : y[i * rc + r];
  };
  for (int r = 0; r < mx; ++r) {
    double v = 0.0;
    if (r < mi) {
      v = oi[r];
      for (int k = 0; k < r; ++k) v = fma(-Mi[r * mx + k], at(k), v);
      v = v / Mi[r * mx + r];
    }
    at(r) = v;
  }
}
cudaError_t launch_update_y(const double *M, int64_t sM, const double *o, int64_t so, const int32_t *m, int mx,
                            int rc, int64_t N, double *y, int ptiled, cudaStream_t s) {
  update_y_kernel<<<(unsigned)((N + 127) / 128), 128, 0, s>>>(M, sM, o, so, m, mx, rc, N, y, ptiled);
  return cudaGetLastError();
}

cudaError_t set_carveout_max(const void *func) {
  static std::mutex mu;
  static std::set<std::pair<const void *, int>> done;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> g(mu);
  if (done.count({func, dev})) return cudaSuccess;
  e = cudaFuncSetAttribute(func, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
  if (e == cudaSuccess) done.insert({func, dev});
  return e;
}

cudaError_t set_smem_attr(const void *func, int bytes) {
  static std::mutex mu;
  static std::set<std::pair<const void *, int>> done;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> g(mu);
  if (done.count({func, dev})) return cudaSuccess;
  e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) done.insert({func, dev});
  return e;
}

}  // namespace ks
