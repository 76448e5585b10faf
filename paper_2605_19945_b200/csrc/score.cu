// Curve evaluation, LUT build, candidate scoring and replay (sm_100a).
//
//  K4 gem_eval_curve / gem_curve_lut   profiles.py:106-190, _kernels.pyx:18-73
//  K5 gem_score_batch                  mapping.py:146-166 (+ cli.py:427 layer sum)
//     gem_replay                       mapping.py:169-198
//
// Scores are the reference's Eq. 1: S(M) = sum_t max_g C_g(n_g(M,t)), the
// t-sum strictly serial in fp64 (_util.py:8-18). All parallelism is across
// candidates and layers; a candidate's chain is never split.
#include "gem_common.cuh"

namespace gem {

// one GPU's curve; its bounds are read on the device (no host round trip).
// An empty curve sets err_flag (GEM_ERR_INVALID) and leaves out untouched.
__global__ void eval_curve_kernel(const int64_t* __restrict__ xs_flat, const double* __restrict__ ys_flat,
                                  const int64_t* __restrict__ offsets, const int64_t* __restrict__ dense_limits,
                                  int gpu, const int64_t* __restrict__ counts, int64_t n, double* __restrict__ out,
                                  int32_t* __restrict__ err_flag) {
  const int64_t o0 = offsets[gpu], o1 = offsets[gpu + 1], dl = dense_limits[gpu];
  if (o1 <= o0) {
    if (err_flag && blockIdx.x == 0 && threadIdx.x == 0) atomicCAS(err_flag, 0, (int32_t)GEM_ERR_INVALID);
    return;
  }
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = eval_one(xs_flat + o0, ys_flat + o0, o1 - o0, dl, counts[i]);
}

// equal_latency_load (profiles.py:308-333) on one thread: the largest n_b
// with C_b(n_b) <= C_a(n_a), by doubling then bisection on the monotone
// curve, saturating at max_search. Same probes in the same order as the
// reference, each one eval_one, so the answer is the reference's.
__global__ void equal_latency_kernel(const int64_t* __restrict__ xs_flat, const double* __restrict__ ys_flat,
                                     const int64_t* __restrict__ offsets, const int64_t* __restrict__ dense_limits,
                                     int ga, int gb, int64_t n_a, int64_t max_search, int64_t* __restrict__ out) {
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  const int64_t a0 = offsets[ga], a1 = offsets[ga + 1], b0 = offsets[gb], b1 = offsets[gb + 1];
  auto cb = [&](int64_t n) { return eval_one(xs_flat + b0, ys_flat + b0, b1 - b0, dense_limits[gb], n); };
  const double target = eval_one(xs_flat + a0, ys_flat + a0, a1 - a0, dense_limits[ga], n_a);
  if (cb(1) > target) {
    *out = 0;
    return;
  }
  int64_t lo = 1, hi = 2;
  while (hi < max_search && cb(hi) <= target) {
    lo = hi;
    hi *= 2;
  }
  if (hi >= max_search) {
    *out = lo;
    return;
  }
  while (lo + 1 < hi) {
    const int64_t mid = (lo + hi) / 2;
    if (cb(mid) <= target) lo = mid; else hi = mid;
  }
  *out = lo;
}

__global__ void curve_lut_kernel(const int64_t* __restrict__ xs_flat, const double* __restrict__ ys_flat,
                                 const int64_t* __restrict__ offsets, const int64_t* __restrict__ dense_limits,
                                 int G, int64_t nmax, double* __restrict__ lut) {
  const int64_t width = nmax + 1;
  const int64_t total = width * G;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int g = (int)(i / width);
    const int64_t n = i % width;
    const int64_t off = offsets[g];
    lut[i] = eval_one(xs_flat + off, ys_flat + off, offsets[g + 1] - off, dense_limits[g], n);
  }
}

// ---------------------------------------------------------------------------
// K5 (CUDA-core version): one thread = one candidate, one CTA = 128 candidates
// of one layer. Each thread keeps its experts sorted by GPU (counting sort)
// in shared memory; histogram rows are staged in shared memory per t-chunk.
constexpr int kScoreThreads = 128;
constexpr int kScoreTChunk = 16;

__global__ void __launch_bounds__(kScoreThreads)
score_layers_kernel(const int32_t* __restrict__ hist, int64_t T, int E, int G, const int8_t* __restrict__ cand,
                    int64_t C, int64_t L, const double* __restrict__ lut, int64_t nmax,
                    double* __restrict__ layer_scores, int32_t* __restrict__ err) {
  extern __shared__ unsigned char smem_raw[];
  int32_t* hs = reinterpret_cast<int32_t*>(smem_raw);                 // [kScoreTChunk][E]
  uint8_t* perm = reinterpret_cast<uint8_t*>(hs + kScoreTChunk * E);   // [E][kScoreThreads]
  int16_t* offs = reinterpret_cast<int16_t*>(perm + (size_t)E * kScoreThreads);  // [G+1][kScoreThreads]
  const int tid = threadIdx.x;
  const int64_t l = blockIdx.y;
  const int64_t c = (int64_t)blockIdx.x * kScoreThreads + tid;
  const bool live = c < C;
  // counting sort of this candidate's experts by GPU
  if (live) {
    const int8_t* m = cand + (c * L + l) * E;
    for (int g = 0; g <= G; ++g) offs[g * kScoreThreads + tid] = 0;
    for (int e = 0; e < E; ++e) offs[(m[e] + 1) * kScoreThreads + tid] += 1;
    for (int g = 0; g < G; ++g) offs[(g + 1) * kScoreThreads + tid] += offs[g * kScoreThreads + tid];
    // place (use a running cursor per GPU held in a second pass)
    for (int g = 0; g < G; ++g) {
      int pos = offs[g * kScoreThreads + tid];
      for (int e = 0; e < E; ++e)
        if (m[e] == g) perm[(pos++) * kScoreThreads + tid] = (uint8_t)e;
    }
  }
  double total = 0.0;
  const int64_t width = nmax + 1;
  bool range_err = false;
  for (int64_t t0 = 0; t0 < T; t0 += kScoreTChunk) {
    const int tn = (int)imin64(kScoreTChunk, T - t0);
    __syncthreads();
    for (int i = tid; i < tn * E; i += kScoreThreads) hs[i] = hist[(l * T + t0) * E + i];
    __syncthreads();
    if (live) {
      for (int tt = 0; tt < tn; ++tt) {
        const int32_t* row = hs + tt * E;
        double m = 0.0;
        bool first = true;
        for (int g = 0; g < G; ++g) {
          const int b0 = offs[g * kScoreThreads + tid], b1 = offs[(g + 1) * kScoreThreads + tid];
          int64_t s = 0;
          for (int i = b0; i < b1; ++i) s += row[perm[i * kScoreThreads + tid]];
          if (s > nmax) { range_err = true; s = nmax; }
          const double v = __ldg(lut + g * width + s);
          if (first || v > m) { m = v; first = false; }
        }
        total = dadd(total, m);
      }
    }
  }
  if (live) layer_scores[c * L + l] = total;
  if (range_err) atomicExch(err, 1);
}

__global__ void layer_sum_kernel(const double* __restrict__ layer_scores, int64_t C, int64_t L,
                                 double* __restrict__ total) {
  for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < C; c += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;  // cli.py:427 aggregate = aggregate + best_score, ascending layer order
    for (int64_t l = 0; l < L; ++l) s = dadd(s, layer_scores[c * L + l]);
    total[c] = s;
  }
}

// ---------------------------------------------------------------------------
// replay: per-step loads / latencies / straggler, then serial sums
__global__ void replay_steps_kernel(const int32_t* __restrict__ hist, int64_t T, int E, int G,
                                    const int8_t* __restrict__ assign, const double* __restrict__ lut, int64_t nmax,
                                    int64_t* __restrict__ loads, double* __restrict__ lat,
                                    double* __restrict__ step_max, int32_t* __restrict__ straggler,
                                    int32_t* __restrict__ err) {
  extern __shared__ int8_t s_assign[];
  for (int e = threadIdx.x; e < E; e += blockDim.x) s_assign[e] = assign[e];
  __syncthreads();
  const int64_t width = nmax + 1;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < T; t += (int64_t)gridDim.x * blockDim.x) {
    const int32_t* row = hist + t * E;
    double best = 0.0;
    int arg = 0;
    for (int g = 0; g < G; ++g) {
      int64_t s = 0;
      for (int e = 0; e < E; ++e) s += (s_assign[e] == g) ? (int64_t)row[e] : 0;
      if (s > nmax) { atomicExch(err, 1); s = nmax; }
      const double v = lut[g * width + s];
      loads[t * G + g] = s;
      lat[t * G + g] = v;
      if (g == 0 || v > best) { best = v; arg = g; }  // argmax: lowest index on ties
    }
    step_max[t] = best;
    straggler[t] = arg;
  }
}

__global__ void replay_sums_kernel(const int64_t* __restrict__ loads, const double* __restrict__ lat,
                                   const double* __restrict__ step_max, int64_t T, int G, double* __restrict__ total,
                                   double* __restrict__ busy, int64_t* __restrict__ gpu_tokens) {
  const int w = threadIdx.x;  // w < G: GPU chain; w == G: total chain
  if (w < G) {
    double s = 0.0;
    int64_t n = 0;
    for (int64_t t = 0; t < T; ++t) {
      s = dadd(s, lat[t * G + w]);
      n += loads[t * G + w];
    }
    busy[w] = s;
    gpu_tokens[w] = n;
  } else if (w == G) {
    double s = 0.0;
    for (int64_t t = 0; t < T; ++t) s = dadd(s, step_max[t]);
    *total = s;
  }
}

}  // namespace gem

using namespace gem;

static unsigned grid_for(int64_t n, int threads, int cap = 65535) {
  int64_t b = (n + threads - 1) / threads;
  if (b > cap) b = cap;
  if (b < 1) b = 1;
  return (unsigned)b;
}

extern "C" int gem_eval_curve(const int64_t* xs_flat, const double* ys_flat, const int64_t* offsets,
                              const int64_t* dense_limits, int32_t gpu, const int64_t* counts, int64_t n, double* out,
                              int32_t* err_flag, void* stream) {
  GEM_REQUIRE(xs_flat && ys_flat && offsets && dense_limits && gpu >= 0, "gem_eval_curve: bad arguments");
  if (n <= 0) return GEM_OK;
  GEM_REQUIRE(counts && out, "gem_eval_curve: null counts/out");
  // asynchronous: the curve's bounds are device data, read by the kernel
  eval_curve_kernel<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(xs_flat, ys_flat, offsets, dense_limits, gpu,
                                                                     counts, n, out, err_flag);
  GEM_CHECK_LAUNCH("eval_curve_kernel");
  return GEM_OK;
}

extern "C" int gem_equal_latency_load(const int64_t* xs_flat, const double* ys_flat, const int64_t* offsets,
                                      const int64_t* dense_limits, int32_t gpu_a, int32_t gpu_b, int64_t n_a,
                                      int64_t max_search, int64_t* out, void* stream) {
  GEM_REQUIRE(xs_flat && ys_flat && offsets && dense_limits && out && gpu_a >= 0 && gpu_b >= 0 && n_a >= 1 &&
                  max_search >= 2,
              "gem_equal_latency_load: bad arguments");
  equal_latency_kernel<<<1, 32, 0, as_stream(stream)>>>(xs_flat, ys_flat, offsets, dense_limits, gpu_a, gpu_b, n_a,
                                                        max_search, out);
  GEM_CHECK_LAUNCH("equal_latency_kernel");
  return GEM_OK;
}

extern "C" int gem_curve_lut(const int64_t* xs_flat, const double* ys_flat, const int64_t* offsets,
                             const int64_t* dense_limits, int32_t G, int64_t nmax, double* lut, void* stream) {
  GEM_REQUIRE(xs_flat && ys_flat && offsets && dense_limits && lut && G >= 1 && nmax >= 0,
              "gem_curve_lut: bad arguments");
  curve_lut_kernel<<<grid_for((nmax + 1) * G, 256, 8192), 256, 0, as_stream(stream)>>>(xs_flat, ys_flat, offsets,
                                                                                       dense_limits, G, nmax, lut);
  GEM_CHECK_LAUNCH("curve_lut_kernel");
  return GEM_OK;
}

extern "C" int gem_score_batch_v1(const int32_t* hist, int64_t L, int64_t T, int32_t E, int32_t G,
                                  const int8_t* cand, int64_t C, const double* lut, int64_t nmax,
                                  double* layer_scores, int32_t* err_flag, void* stream) {
  GEM_REQUIRE(hist && cand && lut && err_flag && layer_scores && L >= 1 && L <= 65535 && T >= 1 && E >= 1 &&
                  E <= 256 && G >= 1 && G <= 127 && C >= 1,
              "gem_score_batch_v1: bad arguments");
  cudaStream_t st = as_stream(stream);
  const size_t smem = (size_t)kScoreTChunk * E * 4 + (size_t)E * kScoreThreads + (size_t)(G + 1) * kScoreThreads * 2;
  GEM_CHECK_CUDA(cudaFuncSetAttribute(score_layers_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  dim3 grid((unsigned)((C + kScoreThreads - 1) / kScoreThreads), (unsigned)L);
  score_layers_kernel<<<grid, kScoreThreads, smem, st>>>(hist, T, E, G, cand, C, L, lut, nmax, layer_scores,
                                                         err_flag);
  GEM_CHECK_LAUNCH("score_layers_kernel");
  return GEM_OK;
}

extern "C" int gem_score_batch(const int32_t* hist, int64_t L, int64_t T, int32_t E, int32_t G, const int8_t* cand,
                               int64_t C, const double* lut, int64_t nmax, double* layer_scores, double* total,
                               int32_t* err_flag, void* stream) {
  GEM_REQUIRE(hist && cand && lut && err_flag && L >= 1 && T >= 1 && E >= 1 && E <= 256 && G >= 1 && G <= 127 &&
                  C >= 1,
              "gem_score_batch: bad arguments (E <= 256, G <= 127)");
  GEM_REQUIRE(L <= 65535, "gem_score_batch: L too large");
  GEM_REQUIRE(layer_scores, "gem_score_batch: layer_scores workspace is required");
  cudaStream_t st = as_stream(stream);
  // tensor-core loads + screened exact maximum (score_tc.cu) when its preconditions hold
  const int rc = gem_score_batch_tc(hist, L, T, E, G, cand, C, lut, nmax, layer_scores, err_flag, stream);
  if (rc < 0) return rc;
  if (rc == 1) {
    const size_t smem =
        (size_t)kScoreTChunk * E * 4 + (size_t)E * kScoreThreads + (size_t)(G + 1) * kScoreThreads * 2;
    GEM_CHECK_CUDA(cudaFuncSetAttribute(score_layers_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    dim3 grid((unsigned)((C + kScoreThreads - 1) / kScoreThreads), (unsigned)L);
    score_layers_kernel<<<grid, kScoreThreads, smem, st>>>(hist, T, E, G, cand, C, L, lut, nmax, layer_scores,
                                                           err_flag);
    GEM_CHECK_LAUNCH("score_layers_kernel");
  }
  if (total) {
    layer_sum_kernel<<<grid_for(C, 256), 256, 0, st>>>(layer_scores, C, L, total);
    GEM_CHECK_LAUNCH("layer_sum_kernel");
  }
  return GEM_OK;
}

extern "C" int gem_layer_sum(const double* layer_scores, int64_t C, int64_t L, double* total, void* stream) {
  GEM_REQUIRE(layer_scores && total && C >= 0 && L >= 1, "gem_layer_sum: bad arguments");
  if (C == 0) return GEM_OK;
  layer_sum_kernel<<<grid_for(C, 256), 256, 0, as_stream(stream)>>>(layer_scores, C, L, total);
  GEM_CHECK_LAUNCH("layer_sum_kernel");
  return GEM_OK;
}

extern "C" int gem_replay(const int32_t* hist, int64_t T, int32_t E, int32_t G, const int8_t* assign,
                          const double* lut, int64_t nmax, int64_t* loads, double* lat, double* step_max,
                          int32_t* straggler, double* total, double* busy, int64_t* gpu_tokens, int32_t* err_flag,
                          void* stream) {
  GEM_REQUIRE(hist && assign && lut && loads && lat && step_max && straggler && total && busy && gpu_tokens &&
                  err_flag && T >= 1 && E >= 1 && G >= 1 && G <= 1023,
              "gem_replay: bad arguments");
  cudaStream_t st = as_stream(stream);
  replay_steps_kernel<<<grid_for(T, 128), 128, E, st>>>(hist, T, E, G, assign, lut, nmax, loads, lat, step_max,
                                                        straggler, err_flag);
  GEM_CHECK_LAUNCH("replay_steps_kernel");
  replay_sums_kernel<<<1, ((G + 1 + 31) / 32) * 32, 0, st>>>(loads, lat, step_max, T, G, total, busy, gpu_tokens);
  GEM_CHECK_LAUNCH("replay_sums_kernel");
  return GEM_OK;
}
