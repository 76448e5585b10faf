// Shared device helpers for libgemcore (sm_100a).
//
// Everything that decides a score is fp64 with explicit round-to-nearest
// intrinsics (the library is also built with --fmad=false) so the arithmetic
// is the reference's operation for operation:
//   /root/reference/pkg/src/gemap/_kernels.pyx:18-55   (_eval_one)
//   /root/reference/pkg/src/gemap/_util.py:8-18        (ordered_sum: serial fp64)
#pragma once

#include <cstdint>
#include <cstddef>
#include <cuda_runtime.h>

#include "../../include/gemcore.h"

namespace gem {

// ---------------------------------------------------------------------------
// error plumbing: every entry point returns an int status; the message of the
// last failure is kept per host thread and exposed through gem_last_error().

void set_error(const char* fmt, ...);
int fail_cuda(cudaError_t err, const char* what);

#define GEM_CHECK_CUDA(expr)                                   \
  do {                                                         \
    cudaError_t _e = (expr);                                   \
    if (_e != cudaSuccess) return ::gem::fail_cuda(_e, #expr); \
  } while (0)

#define GEM_CHECK_LAUNCH(name)                                  \
  do {                                                          \
    cudaError_t _e = cudaGetLastError();                        \
    if (_e != cudaSuccess) return ::gem::fail_cuda(_e, name);   \
  } while (0)

#define GEM_REQUIRE(cond, ...)                                  \
  do {                                                          \
    if (!(cond)) {                                              \
      ::gem::set_error(__VA_ARGS__);                            \
      return GEM_ERR_INVALID;                                   \
    }                                                           \
  } while (0)

__host__ __device__ __forceinline__ int64_t imin64(int64_t a, int64_t b) { return a < b ? a : b; }
__host__ __device__ __forceinline__ int64_t imax64(int64_t a, int64_t b) { return a > b ? a : b; }

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

int num_sms();
void keep_pool();

// ---------------------------------------------------------------------------
// Curve evaluation: C_g(n) for one GPU's sampled curve.
// Branch structure and expression order follow _kernels.pyx:18-55 exactly:
//   n<=0 -> 0; exact sample hit; dense staircase (ceiling sample);
//   interpolate (from the origin below the first sample);
//   extrapolate from the last two samples (from the origin if only one).
__host__ __device__ __forceinline__ double eval_one(const int64_t* xs, const double* ys,
                                                    int64_t size, int64_t dense_limit,
                                                    int64_t n) {
  if (n <= 0) return 0.0;
  int64_t lo = 0, hi = size;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (xs[mid] < n) lo = mid + 1; else hi = mid;
  }
  const int64_t idx = lo;
  if (idx < size && xs[idx] == n) return ys[idx];
  if (n <= dense_limit) return ys[idx];
  int64_t x0, x1;
  double y0, y1;
  if (idx == size) {
    if (size == 1) { x0 = 0; y0 = 0.0; }
    else { x0 = xs[size - 2]; y0 = ys[size - 2]; }
    x1 = xs[size - 1];
    y1 = ys[size - 1];
  } else if (idx == 0) {
    x0 = 0; y0 = 0.0; x1 = xs[0]; y1 = ys[0];
  } else {
    x0 = xs[idx - 1]; y0 = ys[idx - 1]; x1 = xs[idx]; y1 = ys[idx];
  }
#ifdef __CUDA_ARCH__
  // y0 + (y1 - y0) * (double)(n - x0) / (double)(x1 - x0), left to right
  const double num = __dmul_rn(__dsub_rn(y1, y0), (double)(n - x0));
  return __dadd_rn(y0, __ddiv_rn(num, (double)(x1 - x0)));
#else
  volatile double num = (y1 - y0) * (double)(n - x0);
  volatile double q = num / (double)(x1 - x0);
  return y0 + q;
#endif
}

// Serial fp64 accumulate (one dependency chain; never reassociated).
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
// max over non-negative, non-NaN latencies (value-exact, like np.maximum)
__device__ __forceinline__ double dmax(double a, double b) { return a > b ? a : b; }

// ---------------------------------------------------------------------------
// Philox4x32-10 counter-based RNG (Salmon et al., SC'11). Integer-only, so the
// CPU restatement in oracle/ reproduces every draw bit for bit.
struct u32x4 { uint32_t x, y, z, w; };

__host__ __device__ __forceinline__ void mulhilo(uint32_t a, uint32_t b, uint32_t& hi, uint32_t& lo) {
  const uint64_t p = (uint64_t)a * (uint64_t)b;
  hi = (uint32_t)(p >> 32);
  lo = (uint32_t)p;
}

__host__ __device__ __forceinline__ u32x4 philox4x32_10(u32x4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    uint32_t hi0, lo0, hi1, lo1;
    mulhilo(0xD2511F53u, c.x, hi0, lo0);
    mulhilo(0xCD9E8D57u, c.z, hi1, lo1);
    u32x4 n;
    n.x = hi1 ^ c.y ^ k0;
    n.y = lo1;
    n.z = hi0 ^ c.w ^ k1;
    n.w = lo0;
    c = n;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return c;
}

}  // namespace gem
