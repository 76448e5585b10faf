// Scale study (scale.py:100-129): per Monte-Carlo sample, the relative gap
// (fastest - slowest) / fastest over the first n GPUs of the sample's draws,
// for every fleet size n. One thread per sample walks its row once, keeping the
// running max/min (exact, order-free) and emitting a gap at each size; the
// fp64 subtraction and division are the reference's (no FMA: --fmad=false),
// so every gap is bit-identical and the host's mean over samples is too.
#include "gem_common.cuh"

namespace gem {

__global__ void scale_gaps_kernel(const double* __restrict__ draws, int64_t S, int64_t nmax,
                                  const int64_t* __restrict__ sizes, int K, double* __restrict__ gaps) {
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < S; s += (int64_t)gridDim.x * blockDim.x) {
    const double* row = draws + s * nmax;
    double hi = row[0], lo = row[0];
    int64_t j = 1;
    for (int k = 0; k < K; ++k) {
      const int64_t n = sizes[k];
      for (; j < n; ++j) {
        const double v = row[j];
        hi = v > hi ? v : hi;
        lo = v < lo ? v : lo;
      }
      gaps[(int64_t)k * S + s] = __ddiv_rn(__dsub_rn(hi, lo), hi);
    }
  }
}

}  // namespace gem

using namespace gem;

extern "C" int gem_scale_gaps(const double* draws, int64_t S, int64_t nmax, const int64_t* sizes, int32_t K,
                              double* gaps, void* stream) {
  GEM_REQUIRE(draws && sizes && gaps && S >= 1 && nmax >= 1 && K >= 1, "gem_scale_gaps: bad arguments");
  const unsigned blocks = (unsigned)imin64((S + 255) / 256, 16 * num_sms());
  scale_gaps_kernel<<<blocks, 256, 0, as_stream(stream)>>>(draws, S, nmax, sizes, K, gaps);
  GEM_CHECK_LAUNCH("scale_gaps_kernel");
  return GEM_OK;
}
