// GEM-Place search on sm_100a: greedy init, best-swap scan, refinement.
//
//  K7 greedy_kernel      search.py:134-164   (_greedy_assignment)
//  K6 best_swap_kernel   _kernels.pyx:120-160 (best_swap) via per-GPU-pair tiles
//  K8 apply_swap_kernel  search.py:209-239   (_refine_assignment loop body)
//     gem_search_runs    host driver: all runs of all layers advance together,
//                        one scan + one apply launch per refinement round
//
// Bit-exactness rules kept from the reference:
//  * every score is ONE serial fp64 chain over t (never split across threads);
//  * greedy picks the lowest GPU on ties (strict <, search.py:156);
//  * the swap scan returns the first (i,j) in lexicographic order among equal
//    minima (_kernels.pyx:154) -> reduce (cand, i*E+j) lexicographically;
//  * latencies are recomputed from integer loads through the LUT, which holds
//    exactly eval_one(g, n), so lat == C_g(loads) as in latency_matrix();
//  * convergence: stop unless found && cand < score && 1-cand/score >= thr,
//    then the full rescore must equal cand bit for bit (search.py:236).
#include <vector>

#include "gem_common.cuh"

namespace gem {

constexpr int kSearchThreads = 256;
constexpr int kGreedyTChunk = 256;
constexpr int kSwapTChunk = 64;
constexpr int kSwapPairsPerThread = 4;

struct SearchWs {
  int32_t* loads;      // [R][T][G]
  double* pair_cand;   // [R][NP]
  int32_t* pair_flat;  // [R][NP]
  double* run_score;   // [R]
  double* run_cand;    // [R]
  int32_t* run_found;  // [R]
  int32_t* run_i;      // [R]
  int32_t* run_j;      // [R]
  int32_t* run_active; // [R]
  int32_t* counters;   // [4]: active count, mismatch, range
};

static size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

static size_t carve(SearchWs* ws, void* base, int64_t R, int64_t T, int G) {
  const int64_t NP = (int64_t)G * (G - 1) / 2 > 0 ? (int64_t)G * (G - 1) / 2 : 1;
  size_t off = 0;
  char* b = static_cast<char*>(base);
  auto take = [&](size_t bytes) { char* p = b ? b + off : nullptr; off += align_up(bytes); return p; };
  SearchWs w;
  w.loads = (int32_t*)take((size_t)R * T * G * 4);
  w.pair_cand = (double*)take((size_t)R * NP * 8);
  w.pair_flat = (int32_t*)take((size_t)R * NP * 4);
  w.run_score = (double*)take((size_t)R * 8);
  w.run_cand = (double*)take((size_t)R * 8);
  w.run_found = (int32_t*)take((size_t)R * 4);
  w.run_i = (int32_t*)take((size_t)R * 4);
  w.run_j = (int32_t*)take((size_t)R * 4);
  w.run_active = (int32_t*)take((size_t)R * 4);
  w.counters = (int32_t*)take(16);
  if (ws) *ws = w;
  return off;
}

// lat = C_g(n) from the LUT
__device__ __forceinline__ double lut_at(const double* __restrict__ lut, int64_t width, int g, int64_t n) {
  return __ldg(lut + g * width + n);
}

// ---------------------------------------------------------------------------
// K7: greedy placement, one CTA per run
__global__ void __launch_bounds__(kSearchThreads)
greedy_kernel(const int32_t* __restrict__ hist, int64_t T, int E, int G, const double* __restrict__ lut,
              int64_t nmax, const int32_t* __restrict__ run_layer, const uint8_t* __restrict__ needs_greedy,
              const int16_t* __restrict__ order, int8_t* __restrict__ assign, int32_t* __restrict__ loads_ws) {
  extern __shared__ double gsm[];
  double* cost = gsm;  // [G][kGreedyTChunk]
  __shared__ int counts[32];
  __shared__ int s_best;
  const int64_t r = blockIdx.x;
  if (!needs_greedy[r]) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t width = nmax + 1;
  const int32_t* h = hist + (int64_t)run_layer[r] * T * E;
  int32_t* ld = loads_ws + r * T * G;
  for (int64_t i = tid; i < T * G; i += blockDim.x) ld[i] = 0;
  if (tid < 32) counts[tid] = 0;
  const int cap = E / G;
  __syncthreads();
  for (int idx = 0; idx < E; ++idx) {
    const int e = order[r * E + idx];
    double sum = 0.0;  // lane g of warp 0 owns GPU g's chain
    for (int64_t t0 = 0; t0 < T; t0 += kGreedyTChunk) {
      const int tn = (int)imin64(kGreedyTChunk, T - t0);
      for (int tt = tid; tt < tn; tt += blockDim.x) {
        const int64_t t = t0 + tt;
        const int32_t* lrow = ld + t * G;
        double m1 = -1.0, m2 = -1.0;
        int i1 = -1;
        for (int g = 0; g < G; ++g) {
          const double v = lut_at(lut, width, g, lrow[g]);
          if (v > m1) { m2 = m1; m1 = v; i1 = g; }
          else if (v > m2) { m2 = v; }
        }
        const int32_t hv = h[t * E + e];
        for (int g = 0; g < G; ++g) {
          if (counts[g] == cap) continue;
          const double cl = lut_at(lut, width, g, (int64_t)lrow[g] + hv);
          double sc;
          if (G > 1) {
            const double others = (i1 == g) ? m2 : m1;  // max over the other GPUs' lat
            sc = others > cl ? others : cl;
          } else {
            sc = cl;
          }
          cost[g * kGreedyTChunk + tt] = sc;
        }
      }
      __syncthreads();
      if (warp == 0 && lane < G && counts[lane] < cap) {
        const double* cg = cost + lane * kGreedyTChunk;
        for (int tt = 0; tt < tn; ++tt) sum = dadd(sum, cg[tt]);
      }
      __syncthreads();
    }
    if (warp == 0) {
      // strict < in ascending GPU order among GPUs with capacity
      double best = 0.0;
      int bg = -1;
      for (int g = 0; g < G; ++g) {
        const double s = __shfl_sync(0xffffffffu, sum, g);
        if (counts[g] == cap) continue;
        if (bg < 0 || s < best) { best = s; bg = g; }
      }
      if (lane == 0) { s_best = bg; counts[bg] += 1; }
    }
    __syncthreads();
    const int bg = s_best;
    for (int64_t t = tid; t < T; t += blockDim.x) ld[t * G + bg] += h[t * E + e];
    if (tid == 0) assign[r * E + e] = (int8_t)bg;
    __syncthreads();
  }
}

// loads for seeded runs (or all runs when all_runs)
__global__ void init_loads_kernel(const int32_t* __restrict__ hist, int64_t T, int E, int G,
                                  const int32_t* __restrict__ run_layer, const uint8_t* __restrict__ needs_greedy,
                                  const int8_t* __restrict__ assign, int32_t* __restrict__ loads_ws) {
  extern __shared__ int8_t s_as[];
  const int64_t r = blockIdx.y;
  if (needs_greedy && needs_greedy[r]) return;
  for (int e = threadIdx.x; e < E; e += blockDim.x) s_as[e] = assign[r * E + e];
  __syncthreads();
  const int32_t* h = hist + (int64_t)run_layer[r] * T * E;
  int32_t* ld = loads_ws + r * T * G;
  const int64_t total = T * G;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = i / G;
    const int g = (int)(i % G);
    int32_t s = 0;
    for (int e = 0; e < E; ++e) s += (s_as[e] == g) ? h[t * E + e] : 0;
    ld[i] = s;
  }
}

// full score of a run from its loads: serial over t of max_g lat (block-level)
__device__ double block_score(const int32_t* __restrict__ ld, int64_t T, int G, const double* __restrict__ lut,
                              int64_t width, double* buf /*[kGreedyTChunk]*/) {
  double sum = 0.0;
  for (int64_t t0 = 0; t0 < T; t0 += kGreedyTChunk) {
    const int tn = (int)imin64(kGreedyTChunk, T - t0);
    for (int tt = threadIdx.x; tt < tn; tt += blockDim.x) {
      const int32_t* lrow = ld + (t0 + tt) * G;
      double m = lut_at(lut, width, 0, lrow[0]);
      for (int g = 1; g < G; ++g) {
        const double v = lut_at(lut, width, g, lrow[g]);
        m = v > m ? v : m;
      }
      buf[tt] = m;
    }
    __syncthreads();
    if (threadIdx.x == 0)
      for (int tt = 0; tt < tn; ++tt) sum = dadd(sum, buf[tt]);
    __syncthreads();
  }
  return sum;  // valid in thread 0
}

__global__ void __launch_bounds__(kSearchThreads)
init_score_kernel(int64_t T, int G, const double* __restrict__ lut, int64_t nmax, SearchWs ws, int64_t traj_cap,
                  double* __restrict__ trajectory, int32_t* __restrict__ swaps) {
  __shared__ double buf[kGreedyTChunk];
  const int64_t r = blockIdx.x;
  const double s = block_score(ws.loads + r * T * G, T, G, lut, nmax + 1, buf);
  if (threadIdx.x == 0) {
    ws.run_score[r] = s;
    ws.run_active[r] = 1;
    swaps[r] = 0;
    if (traj_cap > 0) trajectory[r * traj_cap] = s;
  }
}

// ---------------------------------------------------------------------------
// K6: best-swap scan. CTA = (run, GPU pair a<b). Each thread owns up to
// kSwapPairsPerThread expert pairs (x on a, y on b), each a serial chain
// over t: cand = sum_t max(pother_ab, C_a(l_a - h_x + h_y), C_b(l_b - h_y + h_x)).
__global__ void __launch_bounds__(kSearchThreads)
best_swap_kernel(const int32_t* __restrict__ hist, int64_t T, int E, int G, const double* __restrict__ lut,
                 int64_t nmax, const int32_t* __restrict__ run_layer, const int8_t* __restrict__ assign,
                 SearchWs ws) {
  extern __shared__ unsigned char bsm[];
  const int64_t r = blockIdx.x;
  if (!ws.run_active[r]) return;
  const int NP = G * (G - 1) / 2;
  // pair index -> (a, b), a < b
  int p = blockIdx.y, a = 0;
  while (p >= G - 1 - a) { p -= G - 1 - a; ++a; }
  const int b = a + 1 + p;
  int16_t* list_a = reinterpret_cast<int16_t*>(bsm);
  int16_t* list_b = list_a + E;
  __shared__ int s_na, s_nb;
  if (threadIdx.x == 0) {
    int na = 0, nb = 0;
    for (int e = 0; e < E; ++e) {
      const int g = assign[r * E + e];
      if (g == a) list_a[na++] = (int16_t)e;
      else if (g == b) list_b[nb++] = (int16_t)e;
    }
    s_na = na;
    s_nb = nb;
  }
  __syncthreads();
  const int na = s_na, nb = s_nb;
  const int P = na * nb;
  // staging after the two lists (8-byte aligned)
  size_t off = ((size_t)2 * E * sizeof(int16_t) + 15) & ~size_t(15);
  double* po = reinterpret_cast<double*>(bsm + off);                 // [kSwapTChunk]
  int32_t* la = reinterpret_cast<int32_t*>(po + kSwapTChunk);        // [kSwapTChunk]
  int32_t* lb = la + kSwapTChunk;                                    // [kSwapTChunk]
  int32_t* ha = lb + kSwapTChunk;                                    // [kSwapTChunk][na]
  int32_t* hb = ha + kSwapTChunk * na;                               // [kSwapTChunk][nb]
  const int64_t width = nmax + 1;
  const int32_t* h = hist + (int64_t)run_layer[r] * T * E;
  const int32_t* ld = ws.loads + r * T * G;
  const double* lut_a = lut + a * width;
  const double* lut_b = lut + b * width;

  double best_c = __longlong_as_double(0x7ff0000000000000LL);  // +inf
  int best_f = 0x7fffffff;
  const int per_pass = blockDim.x * kSwapPairsPerThread;
  for (int pass0 = 0; pass0 < P; pass0 += per_pass) {
    double acc[kSwapPairsPerThread];
    int px[kSwapPairsPerThread], py[kSwapPairsPerThread];
#pragma unroll
    for (int q = 0; q < kSwapPairsPerThread; ++q) {
      acc[q] = 0.0;
      const int pp = pass0 + q * blockDim.x + threadIdx.x;
      px[q] = pp < P ? pp / nb : -1;
      py[q] = pp < P ? pp % nb : -1;
    }
    for (int64_t t0 = 0; t0 < T; t0 += kSwapTChunk) {
      const int tn = (int)imin64(kSwapTChunk, T - t0);
      __syncthreads();
      for (int tt = threadIdx.x; tt < tn; tt += blockDim.x) {
        const int32_t* lrow = ld + (t0 + tt) * G;
        double m = __longlong_as_double(0xfff0000000000000LL);  // -inf when G == 2
        for (int g = 0; g < G; ++g) {
          if (g == a || g == b) continue;
          const double v = lut_at(lut, width, g, lrow[g]);
          m = v > m ? v : m;
        }
        po[tt] = m;
        la[tt] = lrow[a];
        lb[tt] = lrow[b];
      }
      for (int i = threadIdx.x; i < tn * na; i += blockDim.x)
        ha[i] = h[(t0 + i / na) * E + list_a[i % na]];
      for (int i = threadIdx.x; i < tn * nb; i += blockDim.x)
        hb[i] = h[(t0 + i / nb) * E + list_b[i % nb]];
      __syncthreads();
#pragma unroll
      for (int q = 0; q < kSwapPairsPerThread; ++q) {
        if (px[q] < 0) continue;
        double s = acc[q];
        for (int tt = 0; tt < tn; ++tt) {
          const int32_t hx = ha[tt * na + px[q]], hy = hb[tt * nb + py[q]];
          const double va = __ldg(lut_a + (la[tt] - hx + hy));
          const double vb = __ldg(lut_b + (lb[tt] - hy + hx));
          double m = po[tt];
          m = va > m ? va : m;
          m = vb > m ? vb : m;
          s = dadd(s, m);
        }
        acc[q] = s;
      }
    }
#pragma unroll
    for (int q = 0; q < kSwapPairsPerThread; ++q) {
      if (px[q] < 0) continue;
      const int x = list_a[px[q]], y = list_b[py[q]];
      const int f = x < y ? x * E + y : y * E + x;
      if (acc[q] < best_c || (acc[q] == best_c && f < best_f)) { best_c = acc[q]; best_f = f; }
    }
  }
  // block reduce (cand, flat) lexicographically
  __shared__ double rc[kSearchThreads / 32];
  __shared__ int rf[kSearchThreads / 32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double oc = __shfl_xor_sync(0xffffffffu, best_c, o);
    const int of = __shfl_xor_sync(0xffffffffu, best_f, o);
    if (oc < best_c || (oc == best_c && of < best_f)) { best_c = oc; best_f = of; }
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) { rc[warp] = best_c; rf[warp] = best_f; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
      if (rc[w] < best_c || (rc[w] == best_c && rf[w] < best_f)) { best_c = rc[w]; best_f = rf[w]; }
    ws.pair_cand[r * NP + blockIdx.y] = best_c;
    ws.pair_flat[r * NP + blockIdx.y] = best_f;
  }
}

__global__ void reduce_pairs_kernel(int64_t R, int G, int E, SearchWs ws) {
  const int NP = G * (G - 1) / 2;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < R; r += (int64_t)gridDim.x * blockDim.x) {
    if (!ws.run_active[r]) continue;
    double bc = __longlong_as_double(0x7ff0000000000000LL);
    int bf = 0x7fffffff;
    for (int p = 0; p < NP; ++p) {
      const double c = ws.pair_cand[r * NP + p];
      const int f = ws.pair_flat[r * NP + p];
      if (c < bc || (c == bc && f < bf)) { bc = c; bf = f; }
    }
    const bool found = bf != 0x7fffffff;
    ws.run_found[r] = found;
    ws.run_i[r] = found ? bf / E : -1;
    ws.run_j[r] = found ? bf % E : -1;
    ws.run_cand[r] = bc;
  }
}

// K8: apply the accepted swap and re-score (one CTA per run)
__global__ void __launch_bounds__(kSearchThreads)
apply_swap_kernel(const int32_t* __restrict__ hist, int64_t T, int E, int G, const double* __restrict__ lut,
                  int64_t nmax, const int32_t* __restrict__ run_layer, int8_t* __restrict__ assign, SearchWs ws,
                  double threshold, int64_t swap_cap, int64_t traj_cap, double* __restrict__ trajectory,
                  int32_t* __restrict__ swaps) {
  __shared__ double buf[kGreedyTChunk];
  __shared__ int s_go;
  const int64_t r = blockIdx.x;
  if (!ws.run_active[r]) return;
  if (threadIdx.x == 0) {
    const double score = ws.run_score[r], cand = ws.run_cand[r];
    int go = ws.run_found[r] && (cand < score);
    // convergence is judged on the best candidate before applying it (search.py:224-227)
    if (go && __dsub_rn(1.0, __ddiv_rn(cand, score)) < threshold) go = 0;
    s_go = go;
    if (!go) ws.run_active[r] = 0;
  }
  __syncthreads();
  if (!s_go) return;
  const int i = ws.run_i[r], j = ws.run_j[r];
  const int a = assign[r * E + i], b = assign[r * E + j];
  const int32_t* h = hist + (int64_t)run_layer[r] * T * E;
  int32_t* ld = ws.loads + r * T * G;
  for (int64_t t = threadIdx.x; t < T; t += blockDim.x) {
    const int32_t d = h[t * E + j] - h[t * E + i];
    ld[t * G + a] += d;
    ld[t * G + b] -= d;
  }
  __syncthreads();
  const double s = block_score(ld, T, G, lut, nmax + 1, buf);
  if (threadIdx.x == 0) {
    assign[r * E + i] = (int8_t)b;
    assign[r * E + j] = (int8_t)a;
    if (s != ws.run_cand[r]) atomicExch(&ws.counters[1], 1);  // search.py:236 assert
    ws.run_score[r] = s;
    const int n = swaps[r] + 1;
    swaps[r] = n;
    if (n < traj_cap) trajectory[r * traj_cap + n] = s;
    if (n >= swap_cap) ws.run_active[r] = 0;
    else atomicAdd(&ws.counters[0], 1);
  }
}

__global__ void final_copy_kernel(int64_t R, SearchWs ws, double* __restrict__ final_score) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < R; r += (int64_t)gridDim.x * blockDim.x)
    final_score[r] = ws.run_score[r];
}

static size_t swap_smem(int E) {
  const size_t lists = ((size_t)2 * E * sizeof(int16_t) + 15) & ~size_t(15);
  return lists + kSwapTChunk * 8 + 2 * kSwapTChunk * 4 + (size_t)kSwapTChunk * E * 4;
}

}  // namespace gem

using namespace gem;

extern "C" size_t gem_search_workspace_bytes(int64_t R, int64_t T, int32_t E, int32_t G) {
  (void)E;
  return carve(nullptr, nullptr, R, T, G);
}

static int check_search_args(const int32_t* hist, int64_t L, int64_t T, int32_t E, int32_t G, const double* lut,
                             int64_t nmax, int64_t R, const int32_t* run_layer, size_t ws_bytes, void* workspace) {
  GEM_REQUIRE(hist && lut && run_layer && workspace && L >= 1 && T >= 1 && E >= 1 && G >= 1 && R >= 1,
              "gem_search: bad arguments");
  GEM_REQUIRE(G <= 32 && E <= 127 * 32 && E <= 32767, "gem_search: G <= 32 required (got G=%d)", G);
  GEM_REQUIRE(E % G == 0, "gem_search: %d experts cannot be split evenly across %d GPUs", E, G);
  GEM_REQUIRE(E <= 2048, "gem_search: E <= 2048 required");
  GEM_REQUIRE(nmax >= 0 && nmax < (1LL << 31), "gem_search: nmax out of range");
  GEM_REQUIRE(ws_bytes >= gem_search_workspace_bytes(R, T, E, G), "gem_search: workspace too small");
  GEM_REQUIRE(R <= (1LL << 31) - 1, "gem_search: too many runs");
  return GEM_OK;
}

static int launch_scan(const int32_t* hist, int64_t T, int32_t E, int32_t G, const double* lut, int64_t nmax,
                       int64_t R, const int32_t* run_layer, const int8_t* assign, const SearchWs& ws,
                       cudaStream_t st) {
  const int NP = G * (G - 1) / 2;
  if (NP == 0) return GEM_OK;
  const size_t smem = swap_smem(E);
  GEM_CHECK_CUDA(cudaFuncSetAttribute(best_swap_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  dim3 grid((unsigned)R, (unsigned)NP);
  best_swap_kernel<<<grid, kSearchThreads, smem, st>>>(hist, T, E, G, lut, nmax, run_layer, assign, ws);
  GEM_CHECK_LAUNCH("best_swap_kernel");
  reduce_pairs_kernel<<<(unsigned)((R + 255) / 256), 256, 0, st>>>(R, G, E, ws);
  GEM_CHECK_LAUNCH("reduce_pairs_kernel");
  return GEM_OK;
}

extern "C" int gem_search_runs(const int32_t* hist, int64_t L, int64_t T, int32_t E, int32_t G, const double* lut,
                               int64_t nmax, int64_t R, const int32_t* run_layer, const uint8_t* needs_greedy,
                               const int16_t* order, int8_t* assign, double threshold, int64_t swap_cap,
                               int64_t traj_cap, double* trajectory, int32_t* swaps, double* final_score,
                               void* workspace, size_t workspace_bytes, void* stream) {
  int rc = check_search_args(hist, L, T, E, G, lut, nmax, R, run_layer, workspace_bytes, workspace);
  if (rc) return rc;
  GEM_REQUIRE(needs_greedy && order && assign && swaps && final_score && trajectory && traj_cap >= 1 && swap_cap >= 0,
              "gem_search_runs: bad arguments");
  cudaStream_t st = as_stream(stream);
  SearchWs ws;
  carve(&ws, workspace, R, T, G);
  GEM_CHECK_CUDA(cudaMemsetAsync(ws.counters, 0, 16, st));
  const size_t gsmem = (size_t)G * kGreedyTChunk * sizeof(double);
  GEM_CHECK_CUDA(cudaFuncSetAttribute(greedy_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gsmem));
  greedy_kernel<<<(unsigned)R, kSearchThreads, gsmem, st>>>(hist, T, E, G, lut, nmax, run_layer, needs_greedy, order,
                                                            assign, ws.loads);
  GEM_CHECK_LAUNCH("greedy_kernel");
  {
    int64_t bx = (T * G + 255) / 256;
    if (bx > 64) bx = 64;
    dim3 grid((unsigned)bx, (unsigned)R);
    init_loads_kernel<<<grid, 256, E, st>>>(hist, T, E, G, run_layer, needs_greedy, assign, ws.loads);
    GEM_CHECK_LAUNCH("init_loads_kernel");
  }
  init_score_kernel<<<(unsigned)R, kSearchThreads, 0, st>>>(T, G, lut, nmax, ws, traj_cap, trajectory, swaps);
  GEM_CHECK_LAUNCH("init_score_kernel");
  for (int64_t it = 0; it < swap_cap; ++it) {
    rc = launch_scan(hist, T, E, G, lut, nmax, R, run_layer, assign, ws, st);
    if (rc) return rc;
    if (G < 2) break;  // no cross-GPU pair exists: found == false for every run
    GEM_CHECK_CUDA(cudaMemsetAsync(ws.counters, 0, 4, st));
    apply_swap_kernel<<<(unsigned)R, kSearchThreads, 0, st>>>(hist, T, E, G, lut, nmax, run_layer, assign, ws,
                                                              threshold, swap_cap, traj_cap, trajectory, swaps);
    GEM_CHECK_LAUNCH("apply_swap_kernel");
    int32_t active = 0;
    GEM_CHECK_CUDA(cudaMemcpyAsync(&active, ws.counters, 4, cudaMemcpyDeviceToHost, st));
    GEM_CHECK_CUDA(cudaStreamSynchronize(st));
    if (active == 0) break;
  }
  final_copy_kernel<<<(unsigned)((R + 255) / 256), 256, 0, st>>>(R, ws, final_score);
  GEM_CHECK_LAUNCH("final_copy_kernel");
  int32_t mismatch = 0;
  GEM_CHECK_CUDA(cudaMemcpyAsync(&mismatch, ws.counters + 1, 4, cudaMemcpyDeviceToHost, st));
  GEM_CHECK_CUDA(cudaStreamSynchronize(st));
  if (mismatch) {
    set_error("gem_search_runs: incremental swap score differs from the full rescore");
    return GEM_ERR_MISMATCH;
  }
  return GEM_OK;
}

extern "C" int gem_best_swap_runs(const int32_t* hist, int64_t L, int64_t T, int32_t E, int32_t G, const double* lut,
                                  int64_t nmax, int64_t R, const int32_t* run_layer, const int8_t* assign,
                                  int32_t* found, int32_t* best_i, int32_t* best_j, double* best_cand,
                                  void* workspace, size_t workspace_bytes, void* stream) {
  int rc = check_search_args(hist, L, T, E, G, lut, nmax, R, run_layer, workspace_bytes, workspace);
  if (rc) return rc;
  GEM_REQUIRE(assign && found && best_i && best_j && best_cand, "gem_best_swap_runs: null output");
  cudaStream_t st = as_stream(stream);
  SearchWs ws;
  carve(&ws, workspace, R, T, G);
  int64_t bx = (T * G + 255) / 256;
  if (bx > 64) bx = 64;
  init_loads_kernel<<<dim3((unsigned)bx, (unsigned)R), 256, E, st>>>(hist, T, E, G, run_layer, nullptr, assign,
                                                                     ws.loads);
  GEM_CHECK_LAUNCH("init_loads_kernel");
  std::vector<int32_t> ones(R, 1);
  GEM_CHECK_CUDA(cudaMemcpyAsync(ws.run_active, ones.data(), R * 4, cudaMemcpyHostToDevice, st));
  if (G >= 2) {
    rc = launch_scan(hist, T, E, G, lut, nmax, R, run_layer, assign, ws, st);
    if (rc) return rc;
    GEM_CHECK_CUDA(cudaMemcpyAsync(found, ws.run_found, R * 4, cudaMemcpyDeviceToDevice, st));
    GEM_CHECK_CUDA(cudaMemcpyAsync(best_i, ws.run_i, R * 4, cudaMemcpyDeviceToDevice, st));
    GEM_CHECK_CUDA(cudaMemcpyAsync(best_j, ws.run_j, R * 4, cudaMemcpyDeviceToDevice, st));
    GEM_CHECK_CUDA(cudaMemcpyAsync(best_cand, ws.run_cand, R * 8, cudaMemcpyDeviceToDevice, st));
  } else {
    GEM_CHECK_CUDA(cudaMemsetAsync(found, 0, R * 4, st));
    GEM_CHECK_CUDA(cudaMemsetAsync(best_i, 0xff, R * 4, st));
    GEM_CHECK_CUDA(cudaMemsetAsync(best_j, 0xff, R * 4, st));
    std::vector<double> inf(R, __builtin_inf());
    GEM_CHECK_CUDA(cudaMemcpyAsync(best_cand, inf.data(), R * 8, cudaMemcpyHostToDevice, st));
  }
  GEM_CHECK_CUDA(cudaStreamSynchronize(st));
  return GEM_OK;
}
