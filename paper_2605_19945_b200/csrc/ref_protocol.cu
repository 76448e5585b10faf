// Tier 1 of the C ABI: the reference's kernel-backend protocol
// (/root/reference/pkg/src/gemap/kernels.py:22-47) on the GPU.
//
// Callers hand over HOST arrays exactly as the Cython module receives them
// (_kernels.pyx:58-160); each call stages them on the device on the calling
// thread's per-thread default stream, runs, and returns the host result.
// Loads and latencies are taken as given (the protocol passes them in), and
// curve lookups use the binary-search eval_one, so arbitrary int64 counts
// behave exactly as in the reference.
#include <vector>

#include "gem_common.cuh"

namespace gem {

struct Curves {
  const int64_t* xs;
  const double* ys;
  const int64_t* off;
  const int64_t* dl;
  __device__ __forceinline__ double eval(int g, int64_t n) const {
    const int64_t o = off[g];
    return eval_one(xs + o, ys + o, off[g + 1] - o, dl[g], n);
  }
};

// step costs of one swap candidate (i,j); serial sum done by one thread after
__global__ void swap_step_cost_kernel(const int64_t* __restrict__ tokens, int64_t T, int64_t E,
                                      const int64_t* __restrict__ assignment, const int64_t* __restrict__ loads,
                                      const double* __restrict__ lat, int G, Curves cv, int64_t i, int64_t j,
                                      double* __restrict__ cost) {
  const int a = (int)assignment[i], b = (int)assignment[j];
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < T; t += (int64_t)gridDim.x * blockDim.x) {
    const double la = cv.eval(a, loads[t * G + a] - tokens[t * E + i] + tokens[t * E + j]);
    const double lb = cv.eval(b, loads[t * G + b] - tokens[t * E + j] + tokens[t * E + i]);
    double m = __longlong_as_double(0xfff0000000000000LL);
    for (int g = 0; g < G; ++g)
      if (g != a && g != b && lat[t * G + g] > m) m = lat[t * G + g];
    if (la > m) m = la;
    if (lb > m) m = lb;
    cost[t] = m;
  }
}

__global__ void serial_sum_kernel(const double* __restrict__ v, int64_t n, double* __restrict__ out) {
  double s = 0.0;
  for (int64_t t = 0; t < n; ++t) s = dadd(s, v[t]);
  *out = s;
}

// one thread per cross-GPU pair (i<j); candidates in flat i*E+j order
__global__ void protocol_pairs_kernel(const int64_t* __restrict__ tokens, int64_t T, int64_t E,
                                      const int64_t* __restrict__ assignment, const int64_t* __restrict__ loads,
                                      const double* __restrict__ lat, int G, Curves cv, double* __restrict__ cand) {
  const int64_t total = E * E;
  for (int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; f < total; f += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = f / E, j = f % E;
    const int a = (int)assignment[i], b = (int)assignment[j];
    if (j <= i || a == b) { cand[f] = __longlong_as_double(0x7ff0000000000000LL); continue; }
    double s = 0.0;
    for (int64_t t = 0; t < T; ++t) {
      const double la = cv.eval(a, loads[t * G + a] - tokens[t * E + i] + tokens[t * E + j]);
      const double lb = cv.eval(b, loads[t * G + b] - tokens[t * E + j] + tokens[t * E + i]);
      double m = __longlong_as_double(0xfff0000000000000LL);
      for (int g = 0; g < G; ++g)
        if (g != a && g != b && lat[t * G + g] > m) m = lat[t * G + g];
      if (la > m) m = la;
      if (lb > m) m = lb;
      s = dadd(s, m);
    }
    cand[f] = s;
  }
}

// first strict minimum in flat order (= lexicographic (i,j), _kernels.pyx:154)
__global__ void argmin_first_kernel(const double* __restrict__ cand, const int64_t* __restrict__ assignment, int64_t E,
                                    int64_t* __restrict__ out_flat, double* __restrict__ out_val) {
  __shared__ double sv[256];
  __shared__ int64_t sf[256];
  double bv = __longlong_as_double(0x7ff0000000000000LL);
  int64_t bf = -1;
  for (int64_t f = threadIdx.x; f < E * E; f += blockDim.x) {
    const int64_t i = f / E, j = f % E;
    if (j <= i || assignment[i] == assignment[j]) continue;
    const double v = cand[f];
    if (bf < 0 || v < bv || (v == bv && f < bf)) { bv = v; bf = f; }
  }
  sv[threadIdx.x] = bv;
  sf[threadIdx.x] = bf;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < (int)blockDim.x; ++k) {
      if (sf[k] < 0) continue;
      if (bf < 0 || sv[k] < bv || (sv[k] == bv && sf[k] < bf)) { bv = sv[k]; bf = sf[k]; }
    }
    *out_flat = bf;
    *out_val = bv;
  }
}

// RAII device buffers on one stream
struct DevArena {
  cudaStream_t st;
  std::vector<void*> ptrs;
  explicit DevArena(cudaStream_t s) : st(s) {}
  ~DevArena() {
    for (void* p : ptrs) cudaFreeAsync(p, st);
    cudaStreamSynchronize(st);
  }
  template <typename T>
  T* alloc(size_t n, cudaError_t* err) {
    void* p = nullptr;
    *err = cudaMallocAsync(&p, n * sizeof(T) + 16, st);
    if (*err == cudaSuccess) ptrs.push_back(p);
    return static_cast<T*>(p);
  }
  template <typename T>
  T* upload(const T* h, size_t n, cudaError_t* err) {
    T* d = alloc<T>(n, err);
    if (*err != cudaSuccess) return nullptr;
    if (n) *err = cudaMemcpyAsync(d, h, n * sizeof(T), cudaMemcpyHostToDevice, st);
    return d;
  }
};

#define GEM_ARENA_CHECK(err, what) \
  do {                             \
    if ((err) != cudaSuccess) return ::gem::fail_cuda((err), what); \
  } while (0)

static int upload_curves(DevArena& ar, const int64_t* xs_flat, const double* ys_flat, const int64_t* offsets,
                         const int64_t* dense_limits, int64_t G, Curves* cv) {
  cudaError_t err = cudaSuccess;
  const int64_t total = offsets[G];
  cv->xs = ar.upload(xs_flat, (size_t)total, &err);
  GEM_ARENA_CHECK(err, "upload xs_flat");
  cv->ys = ar.upload(ys_flat, (size_t)total, &err);
  GEM_ARENA_CHECK(err, "upload ys_flat");
  cv->off = ar.upload(offsets, (size_t)G + 1, &err);
  GEM_ARENA_CHECK(err, "upload offsets");
  cv->dl = ar.upload(dense_limits, (size_t)G, &err);
  GEM_ARENA_CHECK(err, "upload dense_limits");
  return GEM_OK;
}

}  // namespace gem

using namespace gem;

extern "C" int gem_ref_eval_curve_packed(const int64_t* xs_flat, const double* ys_flat, const int64_t* offsets,
                                         const int64_t* dense_limits, int64_t num_gpus, int64_t gpu,
                                         const int64_t* counts, int64_t n, double* out) {
  GEM_REQUIRE(xs_flat && ys_flat && offsets && dense_limits && num_gpus >= 1 && gpu >= 0 && gpu < num_gpus,
              "gem_ref_eval_curve_packed: bad arguments (gpu=%lld of %lld)", (long long)gpu, (long long)num_gpus);
  if (n <= 0) return GEM_OK;
  GEM_REQUIRE(counts && out, "gem_ref_eval_curve_packed: null counts/out");
  const int64_t o0 = offsets[gpu], o1 = offsets[gpu + 1];
  GEM_REQUIRE(o1 > o0, "gem_ref_eval_curve_packed: empty curve");
  cudaStream_t st = cudaStreamPerThread;
  DevArena ar(st);
  cudaError_t err = cudaSuccess;
  const int64_t* dxs = ar.upload(xs_flat + o0, (size_t)(o1 - o0), &err);
  GEM_ARENA_CHECK(err, "upload xs");
  const double* dys = ar.upload(ys_flat + o0, (size_t)(o1 - o0), &err);
  GEM_ARENA_CHECK(err, "upload ys");
  const int64_t* dcounts = ar.upload(counts, (size_t)n, &err);
  GEM_ARENA_CHECK(err, "upload counts");
  double* dout = ar.alloc<double>((size_t)n, &err);
  GEM_ARENA_CHECK(err, "alloc out");
  // reuse the K4 kernel through its device-pointer entry (same code path as the package)
  std::vector<int64_t> off2 = {0, o1 - o0};
  int64_t* doff = ar.upload(off2.data(), 2, &err);
  GEM_ARENA_CHECK(err, "upload offsets");
  int64_t* ddl = ar.upload(dense_limits + gpu, 1, &err);
  GEM_ARENA_CHECK(err, "upload dense_limit");
  int rc = gem_eval_curve(dxs, dys, doff, ddl, 0, dcounts, n, dout, nullptr, (void*)st);
  if (rc) return rc;
  GEM_CHECK_CUDA(cudaMemcpyAsync(out, dout, (size_t)n * sizeof(double), cudaMemcpyDeviceToHost, st));
  GEM_CHECK_CUDA(cudaStreamSynchronize(st));
  return GEM_OK;
}

extern "C" int gem_ref_swap_candidate_score(const int64_t* tokens, int64_t steps, int64_t experts,
                                            const int64_t* assignment, const int64_t* loads, const double* lat,
                                            int64_t num_gpus, const int64_t* xs_flat, const double* ys_flat,
                                            const int64_t* offsets, const int64_t* dense_limits, int64_t i, int64_t j,
                                            double* out) {
  GEM_REQUIRE(tokens && assignment && loads && lat && xs_flat && ys_flat && offsets && dense_limits && out &&
                  steps >= 0 && experts >= 1 && num_gpus >= 1,
              "gem_ref_swap_candidate_score: bad arguments");
  GEM_REQUIRE(i >= 0 && i < experts && j >= 0 && j < experts, "gem_ref_swap_candidate_score: expert out of range");
  GEM_REQUIRE(assignment[i] >= 0 && assignment[i] < num_gpus && assignment[j] >= 0 && assignment[j] < num_gpus,
              "gem_ref_swap_candidate_score: assignment out of range");
  if (steps == 0) { *out = 0.0; return GEM_OK; }
  cudaStream_t st = cudaStreamPerThread;
  DevArena ar(st);
  cudaError_t err = cudaSuccess;
  Curves cv;
  int rc = upload_curves(ar, xs_flat, ys_flat, offsets, dense_limits, num_gpus, &cv);
  if (rc) return rc;
  const int64_t* dtok = ar.upload(tokens, (size_t)(steps * experts), &err);
  GEM_ARENA_CHECK(err, "upload tokens");
  const int64_t* dasg = ar.upload(assignment, (size_t)experts, &err);
  GEM_ARENA_CHECK(err, "upload assignment");
  const int64_t* dld = ar.upload(loads, (size_t)(steps * num_gpus), &err);
  GEM_ARENA_CHECK(err, "upload loads");
  const double* dlat = ar.upload(lat, (size_t)(steps * num_gpus), &err);
  GEM_ARENA_CHECK(err, "upload lat");
  double* dcost = ar.alloc<double>((size_t)steps, &err);
  GEM_ARENA_CHECK(err, "alloc cost");
  double* dsum = ar.alloc<double>(1, &err);
  GEM_ARENA_CHECK(err, "alloc sum");
  int64_t blocks = (steps + 255) / 256;
  if (blocks > 4096) blocks = 4096;
  swap_step_cost_kernel<<<(unsigned)blocks, 256, 0, st>>>(dtok, steps, experts, dasg, dld, dlat, (int)num_gpus, cv, i,
                                                         j, dcost);
  GEM_CHECK_LAUNCH("swap_step_cost_kernel");
  serial_sum_kernel<<<1, 1, 0, st>>>(dcost, steps, dsum);
  GEM_CHECK_LAUNCH("serial_sum_kernel");
  GEM_CHECK_CUDA(cudaMemcpyAsync(out, dsum, sizeof(double), cudaMemcpyDeviceToHost, st));
  GEM_CHECK_CUDA(cudaStreamSynchronize(st));
  return GEM_OK;
}

extern "C" int gem_ref_best_swap(const int64_t* tokens, int64_t steps, int64_t experts, const int64_t* assignment,
                                 const int64_t* loads, const double* lat, int64_t num_gpus, const int64_t* xs_flat,
                                 const double* ys_flat, const int64_t* offsets, const int64_t* dense_limits,
                                 int32_t* found, int64_t* best_i, int64_t* best_j, double* best_cand) {
  GEM_REQUIRE(tokens && assignment && loads && lat && xs_flat && ys_flat && offsets && dense_limits && found &&
                  best_i && best_j && best_cand && steps >= 0 && experts >= 1 && num_gpus >= 1,
              "gem_ref_best_swap: bad arguments");
  for (int64_t e = 0; e < experts; ++e)
    GEM_REQUIRE(assignment[e] >= 0 && assignment[e] < num_gpus, "gem_ref_best_swap: assignment out of range");
  cudaStream_t st = cudaStreamPerThread;
  DevArena ar(st);
  cudaError_t err = cudaSuccess;
  Curves cv;
  int rc = upload_curves(ar, xs_flat, ys_flat, offsets, dense_limits, num_gpus, &cv);
  if (rc) return rc;
  const int64_t* dtok = ar.upload(tokens, (size_t)(steps * experts), &err);
  GEM_ARENA_CHECK(err, "upload tokens");
  const int64_t* dasg = ar.upload(assignment, (size_t)experts, &err);
  GEM_ARENA_CHECK(err, "upload assignment");
  const int64_t* dld = ar.upload(loads, (size_t)(steps * num_gpus), &err);
  GEM_ARENA_CHECK(err, "upload loads");
  const double* dlat = ar.upload(lat, (size_t)(steps * num_gpus), &err);
  GEM_ARENA_CHECK(err, "upload lat");
  double* dcand = ar.alloc<double>((size_t)(experts * experts), &err);
  GEM_ARENA_CHECK(err, "alloc cand");
  int64_t* dflat = ar.alloc<int64_t>(1, &err);
  GEM_ARENA_CHECK(err, "alloc flat");
  double* dval = ar.alloc<double>(1, &err);
  GEM_ARENA_CHECK(err, "alloc val");
  int64_t blocks = (experts * experts + 127) / 128;
  if (blocks > 8192) blocks = 8192;
  protocol_pairs_kernel<<<(unsigned)blocks, 128, 0, st>>>(dtok, steps, experts, dasg, dld, dlat, (int)num_gpus, cv,
                                                         dcand);
  GEM_CHECK_LAUNCH("protocol_pairs_kernel");
  argmin_first_kernel<<<1, 256, 0, st>>>(dcand, dasg, experts, dflat, dval);
  GEM_CHECK_LAUNCH("argmin_first_kernel");
  int64_t flat = -1;
  double val = 0.0;
  GEM_CHECK_CUDA(cudaMemcpyAsync(&flat, dflat, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  GEM_CHECK_CUDA(cudaMemcpyAsync(&val, dval, sizeof(double), cudaMemcpyDeviceToHost, st));
  GEM_CHECK_CUDA(cudaStreamSynchronize(st));
  if (flat < 0) {
    *found = 0;
    *best_i = -1;
    *best_j = -1;
    *best_cand = __builtin_inf();
  } else {
    *found = 1;
    *best_i = flat / experts;
    *best_j = flat % experts;
    *best_cand = val;
  }
  return GEM_OK;
}
