// Error reporting, version and device queries for libgemcore.
#include <cstdarg>
#include <cstdio>

#include "gem_common.cuh"

namespace gem {

static thread_local char g_last_error[1024] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_last_error, sizeof(g_last_error), fmt, ap);
  va_end(ap);
}

int fail_cuda(cudaError_t err, const char* what) {
  set_error("%s: %s (%s)", what, cudaGetErrorName(err), cudaGetErrorString(err));
  return GEM_ERR_CUDA;
}

// Stream-ordered scratch (cudaMallocAsync) must not be returned to the OS at
// every synchronisation: keep the current device's default pool warm.
void keep_pool() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) != cudaSuccess) return;
  uint64_t thr = ~0ull;
  cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
}

int num_sms() {
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess)
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms > 0 ? sms : 148;
}

}  // namespace gem

extern "C" const char* gem_version(void) { return "gemcore 0.1.0 (sm_100a)"; }

extern "C" const char* gem_last_error(void) { return gem::g_last_error; }

extern "C" int gem_device_info(int* sm_count, int* cc_major, int* cc_minor) {
  int dev = 0;
  GEM_CHECK_CUDA(cudaGetDevice(&dev));
  cudaDeviceProp prop;
  GEM_CHECK_CUDA(cudaGetDeviceProperties(&prop, dev));
  if (sm_count) *sm_count = prop.multiProcessorCount;
  if (cc_major) *cc_major = prop.major;
  if (cc_minor) *cc_minor = prop.minor;
  return GEM_OK;
}
