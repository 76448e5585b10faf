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
#include <cstdio>
#include <cstdlib>
#include <type_traits>
#include <vector>

#include "gem_common.cuh"

namespace gem {

constexpr int kSearchThreads = 256;
constexpr int kGreedyTChunk = 256;
#ifndef GEM_GREEDY_REFINE
#define GEM_GREEDY_REFINE 1
#endif
constexpr bool kGreedyRefine = GEM_GREEDY_REFINE;         // fp64 parallel screen before the exact chains
constexpr double kRefineWindow = 1.0 + 1.0 / 68719476736.0;  // 1 + 2^-36
constexpr int kSwapTChunk = 64;
constexpr int kSwapPairsPerThread = 4;
// screening window: exact winners satisfy approx <= min(approx) * (1 + 2^-20) (see K6 v3 / K7 v2)
constexpr double kWindow = 1.0 + 1.0 / 1048576.0;
constexpr int kBuckets = 1024;  // value buckets of the clamp-point search (K6 v5)
// window of the fp32-chunk-sum screen (K6 v5): error < 2^-18.9 relative, so the
// exact winner is within (1 + 2^-18.9) / (1 - 2^-18.9) < 1 + 2^-17.8 of the minimum
constexpr double kWindow5 = 1.0 + 1.0 / 131072.0;

__device__ __forceinline__ float lds_f32(uint32_t addr) {  // 32-bit shared-window address
  float v;
  asm("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr));
  return v;
}

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
  int32_t* run_list;   // [R] compacted indices of the active runs
  int32_t* counters;   // [4]: active count, mismatch, range, list length
  // screened scan (K6 v3)
  double* loc_min;     // [R][NP] approximate minimum of each (run, GPU pair) tile
  int32_t* loc_cnt;    // [R][NP] pairs inside the tile's window (may exceed kLocK)
  double* loc_cand;    // [R][NP][kLocK]
  int32_t* loc_flat;   // [R][NP][kLocK]
  int32_t* cand_flat;  // [R][kCandK] pairs to evaluate exactly
  int32_t* cand_n;     // [R]
  int32_t* need_exact; // [R] kNeedExact: window overflow -> exact full scan of the run;
                       // kPreAccept / kPreReject: the window alone decides (search only)
  double* cand_exact;  // [R][kCandK]
  float* latT;         // [R][G][Tp] fp32 latencies of the current loads (screened scan)
  uint16_t* loadT;     // [R][G][Tp] current loads (screened scan)
  uint32_t* top3;      // [R][4][Tp] per step: the three largest fp32 latencies (bits) and their GPUs (packed)
  double* split_acc;   // [R][NP][n][n] step-range-split scans: partial approximate sums of every pair
  int64_t Tp;          // T rounded up to 32 (whole 16-byte pieces for every chunk of the transposed arrays)
  const float* lut32;  // [G][nmax+1] fp32 rounding of the latency table (set by the driver)
  const uint16_t* ht16;  // [L][E][Tp] transposed counts (set by the driver when every count < 65536)
  const uint16_t* ht16s; // [L][E][Tp] the same counts times 4 (byte offsets into fp32 rows; 4U < 65536)
  int32_t lut_monotone;  // every fp32 table row is nondecreasing (set by the driver)
  int32_t lut_monotone64;  // every fp64 table row is nondecreasing (set by the driver)
  int32_t win;           // loads never exceed win - 1 (= min(U, nmax)): table window of the screened scan
  const uint16_t* first;  // [G][kBuckets + 2] first n whose value bucket is >= b (clamp-point search hints)
  const float* bscale;    // [G] buckets per unit latency: bucket(v) = min(kBuckets, (int)(v * bscale[g]))
};

#ifndef GEM_LOCK
#define GEM_LOCK 64
#endif
#ifndef GEM_CANDK
#define GEM_CANDK 256
#endif
constexpr int kLocK = GEM_LOCK;
constexpr int kCandK = GEM_CANDK;
constexpr int32_t kNeedExact = 1, kPreAccept = 2, kPreReject = 3;

static size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

static size_t carve(SearchWs* ws, void* base, int64_t R, int64_t T, int E, int G) {
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
  w.run_list = (int32_t*)take((size_t)R * 4);
  w.counters = (int32_t*)take(16);
  w.loc_min = (double*)take((size_t)R * NP * 8);
  w.loc_cnt = (int32_t*)take((size_t)R * NP * 4);
  w.loc_cand = (double*)take((size_t)R * NP * kLocK * 8);
  w.loc_flat = (int32_t*)take((size_t)R * NP * kLocK * 4);
  w.cand_flat = (int32_t*)take((size_t)R * kCandK * 4);
  w.cand_n = (int32_t*)take((size_t)R * 4);
  w.need_exact = (int32_t*)take((size_t)R * 4);
  w.cand_exact = (double*)take((size_t)R * kCandK * 8);
  w.Tp = (T + 31) / 32 * 32;
  w.latT = (float*)take((size_t)R * G * w.Tp * 4);
  w.loadT = (uint16_t*)take((size_t)R * G * w.Tp * 2);
  w.top3 = (uint32_t*)take((size_t)R * 4 * w.Tp * 4);
  w.split_acc = (double*)take((size_t)R * NP * (G > 0 ? (size_t)(E / G) * (E / G) : 1) * 8);
  w.lut32 = nullptr;
  w.ht16 = nullptr;
  w.ht16s = nullptr;
  w.lut_monotone = 0;
  w.lut_monotone64 = 0;
  w.win = 0;
  w.first = nullptr;
  w.bscale = nullptr;
  if (ws) *ws = w;
  return off;
}

// lat = C_g(n) from the LUT
__device__ __forceinline__ double lut_at(const double* __restrict__ lut, int64_t width, int g, int64_t n) {
  return __ldg(lut + g * width + n);
}

// max over g < G, g != xa, g != xb of C_g(lrow[g]) (-inf when empty): the
// loads, then the gathers, 8 GPUs per batch in flight (a runtime loop of
// load -> dependent gather costs two L2 round trips per GPU)
__device__ __forceinline__ double max_lat_excl(const int32_t* __restrict__ lrow, int G, const double* __restrict__ lut,
                                               int64_t width, int xa, int xb) {
  double m = __longlong_as_double(0xfff0000000000000LL);
  for (int g0 = 0; g0 < G; g0 += 8) {
    int32_t n[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) n[q] = g0 + q < G ? lrow[g0 + q] : 0;
    double v[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int g = g0 + q;
      v[q] = (g < G && g != xa && g != xb) ? lut_at(lut, width, g, n[q]) : __longlong_as_double(0xfff0000000000000LL);
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) m = v[q] > m ? v[q] : m;
  }
  return m;
}

// ---------------------------------------------------------------------------
// K7: greedy placement, one CTA per run (the exact v1 kernel: any G up to
// kMaxGpus; the screened K7 v3 below handles G <= 32). Per chunk of tchunk
// steps every thread fills the exact terms of every GPU with capacity, then
// thread g extends GPU g's serial chain in t order; the strict-< lowest-index
// rule (search.py:156) picks the GPU.
constexpr int kMaxGpus = 127;  // assignments are int8
__global__ void __launch_bounds__(kSearchThreads)
greedy_kernel(const int32_t* __restrict__ hist, int64_t T, int E, int G, const double* __restrict__ lut,
              int64_t nmax, const int32_t* __restrict__ run_layer, const uint8_t* __restrict__ needs_greedy,
              const int16_t* __restrict__ order, int8_t* __restrict__ assign, int32_t* __restrict__ loads_ws,
              int tchunk) {
  extern __shared__ double gsm[];
  double* cost = gsm;  // [G][tchunk]
  __shared__ int counts[kMaxGpus + 1];
  __shared__ double sums[kMaxGpus + 1];
  __shared__ int s_best;
  const int64_t r = blockIdx.x;
  if (!needs_greedy[r]) return;
  const int tid = threadIdx.x;
  const int64_t width = nmax + 1;
  const int32_t* h = hist + (int64_t)run_layer[r] * T * E;
  int32_t* ld = loads_ws + r * T * G;
  for (int64_t i = tid; i < T * G; i += blockDim.x) ld[i] = 0;
  for (int g = tid; g <= kMaxGpus; g += blockDim.x) counts[g] = 0;
  const int cap = E / G;
  __syncthreads();
  for (int idx = 0; idx < E; ++idx) {
    const int e = order[r * E + idx];
    double sum = 0.0;  // thread g owns GPU g's chain
    for (int64_t t0 = 0; t0 < T; t0 += tchunk) {
      const int tn = (int)imin64(tchunk, T - t0);
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
          cost[g * tchunk + tt] = sc;
        }
      }
      __syncthreads();
      if (tid < G && counts[tid] < cap) {
        const double* cg = cost + tid * tchunk;
        for (int tt = 0; tt < tn; ++tt) sum = dadd(sum, cg[tt]);
      }
      __syncthreads();
    }
    if (tid < G) sums[tid] = sum;
    __syncthreads();
    if (tid == 0) {  // strict < in ascending GPU order among GPUs with capacity
      double best = 0.0;
      int bg = -1;
      for (int g = 0; g < G; ++g) {
        if (counts[g] == cap) continue;
        if (bg < 0 || sums[g] < best) { best = sums[g]; bg = g; }
      }
      s_best = bg;
      counts[bg] += 1;
    }
    __syncthreads();
    const int bg = s_best;
    for (int64_t t = tid; t < T; t += blockDim.x) ld[t * G + bg] += h[t * E + e];
    if (tid == 0) assign[r * E + e] = (int8_t)bg;
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// K7 v2: screened greedy placement.
//
// Greedy (search.py:142-163) places the experts of a run one at a time on the
// GPU with the smallest exact serial-fp64 score sum_t max(others, C_g(l_g+h)),
// lowest GPU on ties. v1 pays two L1 table gathers per (t, GPU) and a serial
// chain per GPU. v2 keeps the fp32 rounding of the table window [0, U] in
// shared memory (U = max over steps of the sum of the n = E/G largest counts:
// no GPU load, before or after a placement, can exceed it) and scores every
// candidate GPU approximately: terms fl32(max(..)) summed in fp64 in ANY
// order (per-thread partials + tree), so |S' - S| <= (2^-24 + T 2^-52) S and
// the exact winner lies inside S' <= min' (1 + 2^-20). One GPU in the window
// decides; otherwise the window's GPUs are scored exactly (v1's serial chain
// in t order) and the strict-< / lowest-index rule picks among them.
constexpr int kG2Threads = 512;
// 32-GPU slots: 256 threads, so the per-thread GPU arrays get 255 registers
__host__ __device__ constexpr int g2_threads(int GM) { return GM >= 32 ? 256 : kG2Threads; }
#ifndef GEM_GREEDY_UNROLL
#define GEM_GREEDY_UNROLL 4
#endif
constexpr int kGreedyUnroll = GEM_GREEDY_UNROLL;

// U[l] = max_t (sum of the n largest counts of step t): one warp per step row
// (n_dev, when given, replaces n with max(*n_dev, 1): the caller's bound stays on the device)
__global__ void topn_bound_kernel(const int32_t* __restrict__ hist, int64_t L, int64_t T, int E, int n,
                                  const int32_t* __restrict__ n_dev, int32_t* __restrict__ bound,
                                  int32_t* __restrict__ top1, int32_t* __restrict__ rowmin) {
  extern __shared__ int32_t tb_rows[];  // [warps][E]
  if (n_dev != nullptr) n = min(max(*n_dev, 1), E);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int32_t* row = tb_rows + (size_t)w * E;
  const int64_t rows = L * T;
  for (int64_t rr = (int64_t)blockIdx.x * nw + w; rr < rows; rr += (int64_t)gridDim.x * nw) {
    const int32_t* h = hist + rr * E;
    int64_t rs = 0;  // the step's total (rowmin: smallest over all steps)
    for (int e = lane; e < E; e += 32) {
      row[e] = h[e];
      rs += h[e];
    }
    if (rowmin != nullptr) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) rs += __shfl_xor_sync(0xffffffffu, rs, o);
      if (lane == 0) atomicMin(rowmin, (int32_t)(rs < 0x7fffffff ? rs : 0x7fffffff));
    }
    __syncwarp();
    int64_t sum = 0;
    for (int k = 0; k < n; ++k) {
      int best = -1, bi = -1;
      for (int e = lane; e < E; e += 32)
        if (row[e] > best) { best = row[e]; bi = e; }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const int ob = __shfl_xor_sync(0xffffffffu, best, o), oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
      }
      sum += best;
      if (k == 0 && top1 != nullptr && lane == 0) atomicMax(&top1[rr / T], best);
      if (lane == 0) row[bi] = -1;
      __syncwarp();
    }
    if (lane == 0) atomicMax(&bound[rr / T], (int32_t)(sum < 0x7fffffff ? sum : 0x7fffffff));
    __syncwarp();
  }
}

// transposed uint16 copy of the histogram: ht[l][e][t] = hist[l][t][e] for
// t < T, 0 for T <= t < Tp (every count <= U < 65536 on this path)
__global__ void hist_t16_kernel(const int32_t* __restrict__ hist, int64_t T, int64_t Tp, int E, int shift,
                                uint16_t* __restrict__ ht) {
  __shared__ uint16_t tile[32][33];
  const int64_t l = blockIdx.z;
  const int64_t t0 = (int64_t)blockIdx.x * 32;
  const int e0 = blockIdx.y * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
  for (int k = ty; k < 32; k += 8) {
    const int64_t t = t0 + k;
    const int e = e0 + tx;
    tile[k][tx] = (t < T && e < E) ? (uint16_t)(hist[(l * T + t) * E + e] << shift) : (uint16_t)0;
  }
  __syncthreads();
  for (int k = ty; k < 32; k += 8) {
    const int e = e0 + k;
    const int64_t t = t0 + tx;
    if (t < Tp && e < E) ht[(l * E + e) * Tp + t] = tile[tx][k];
  }
}

// Piecewise-linear fp32 rows for K7's approximate pass when the fp32 table is
// off-chip (G = 32 with a wide window): bucket j >= 1 covers the loads
// (64(j-1), 64j] -- the profiles' tile staircase and the sparse interpolation
// segments above the dense limit are linear on them -- and bucket 0 the load
// 0: C'(n) = a_j + b_j (n - n0_j), n0_j = 64(j-1)+1, with (a_j, b_j) =
// (fl32 C(n0_j), fl32 of the bucket's slope). pw_check_kernel flags any row
// where some n in [0, W) misses C(n) by more than 2^-22 C(n); the greedy then
// keeps the global fp32 table. 64 B of shared memory per 64 loads per GPU
// instead of 256 B in L1/L2.
constexpr int kPwShift = 6;
__host__ __device__ constexpr int pw_buckets(int W) { return ((W - 1 + (1 << kPwShift) - 1) >> kPwShift) + 1; }
__device__ __forceinline__ int pw_bucket(uint32_t n) { return (int)((n + (1u << kPwShift) - 1u) >> kPwShift); }
__device__ __forceinline__ float pw_eval(float2 ab, uint32_t n, int j) {
  return fmaf(ab.y, (float)((int)n - (((j - 1) << kPwShift) + 1)), ab.x);
}
__global__ void pw_table_kernel(const double* __restrict__ lut, int64_t width, int G, int W, float2* __restrict__ pw) {
  const int K = pw_buckets(W);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < G * K; i += gridDim.x * blockDim.x) {
    const int g = i / K, j = i - g * K;
    const double* row = lut + (int64_t)g * width;
    if (j == 0) {
      pw[i] = make_float2((float)row[0], 0.0f);
      continue;
    }
    const int n0 = ((j - 1) << kPwShift) + 1, n1 = min(j << kPwShift, W - 1);
    const double c0 = row[n0];
    const float b = n1 > n0 ? (float)((row[n1] - c0) / (double)(n1 - n0)) : 0.0f;
    pw[i] = make_float2((float)c0, b);
  }
}
__global__ void pw_check_kernel(const double* __restrict__ lut, int64_t width, int G, int W,
                                const float2* __restrict__ pw, int32_t* __restrict__ bad) {
  const int K = pw_buckets(W);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < (int64_t)G * W;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int g = (int)(i / W), n = (int)(i - (int64_t)g * W);
    const int j = pw_bucket((uint32_t)n);
    const double c = lut[(int64_t)g * width + n];
    const double a = (double)pw_eval(pw[g * K + j], (uint32_t)n, j);
    if (!(c >= 0.0) || !(fabs(a - c) <= c * 0x1p-22)) atomicOr(bad, 1);
  }
}

// FULL: G == GM (no padded GPU columns: the per-GPU guards vanish at compile time)
// SL: the fp32 table window [G][W] sits in shared memory; otherwise (G = 32
// with a wide window) the gathers read ws.lut32 through L1/L2
// TOP2 (monotone fp64 table rows): every step's exact top-2 of the current
// latencies is kept in global memory and updated after each placement (only
// the chosen GPU's latency changes, and it can only grow), so the max over
// the OTHER GPUs of GPU g is (g == arg ? D2 : D1) -- no per-placement
// re-gather of all G current latencies in the approximate pass (fp32: the
// rounding of D1/D2, rounding being monotone) nor in the exact re-scores.
template <int GM, bool FULL, bool SL, bool TOP2>
__global__ void __launch_bounds__(g2_threads(GM), 1)
greedy2_kernel(const int32_t* __restrict__ hist, int64_t T, int E, int G_,
               const double* __restrict__ lut, int64_t nmax, int W, const int32_t* __restrict__ run_layer,
               const uint8_t* __restrict__ needs_greedy, const int16_t* __restrict__ order,
               int8_t* __restrict__ assign, uint16_t* __restrict__ loads16, SearchWs ws,
               float2* __restrict__ top_p, double2* __restrict__ top_d, uint8_t* __restrict__ top_a,
               const float2* __restrict__ pw, const int32_t* __restrict__ pw_bad) {
  const int G = FULL ? GM : G_;
  extern __shared__ __align__(16) unsigned char g2s[];
  float* s_lut = reinterpret_cast<float*>(g2s);                                        // [G][W] (SL)
  const uint32_t lut_base = (uint32_t)__cvta_generic_to_shared(s_lut);
  double* red = reinterpret_cast<double*>(g2s + (SL ? (((size_t)G * W * 4 + 15) & ~size_t(15)) : 0));  // [warps][GM]
  double* buf = red + (g2_threads(GM) / 32) * GM;                                          // [kGreedyTChunk]
  float2* s_pw = reinterpret_cast<float2*>(buf + kGreedyTChunk * GM);                       // [G][K] (!SL, pw)
  __shared__ int counts[GM];
  __shared__ int s_best, s_ncand;
  __shared__ int s_cand[GM];
  __shared__ unsigned s_exc;  // GPUs whose candidate latency may reach the others' maximum at some step
  const int64_t r = blockIdx.x;
  if (!needs_greedy[r]) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  const int64_t width = nmax + 1;
  const int64_t layer = run_layer[r];
  const int32_t* h = hist + layer * T * E;
  const uint16_t* hl = ws.ht16 + layer * E * ws.Tp;
  uint16_t* ld = loads16 + r * T * GM;  // row stride GM (padded), unused GPUs stay 0
  auto LDI = [&](int64_t t, int g) -> int64_t { return t * GM + g; };
  if (SL)
    for (int i = tid; i < G * W; i += blockDim.x) {
      const int g = i / W, nn = i - g * W;
      s_lut[i] = ws.lut32[(int64_t)g * width + nn];
    }
  // table value of GPU slot g (rows of padded slots g >= G read row G - 1)
  auto tab = [&](const uint32_t* row_addr, int g, uint32_t nn) -> float {
    if (SL) return lds_f32(row_addr[g] + 4u * nn);
    return __ldg(ws.lut32 + (int64_t)(g < G ? g : G - 1) * width + nn);
  };
  // !SL: the piecewise rows in shared memory when they reproduce the table (pw_check_kernel)
  const bool usepw = !SL && pw != nullptr && *pw_bad == 0;
  const int pwK = pw_buckets(W);
  if (usepw)
    for (int i = tid; i < G * pwK; i += blockDim.x) s_pw[i] = pw[i];
  if (tid < GM) counts[tid] = 0;
  if (tid == 0) s_exc = 0u;
  for (int64_t i = tid; i < T * GM; i += blockDim.x) ld[i] = 0;
  float2* tp = nullptr;
  double2* td = nullptr;
  uint8_t* ta = nullptr;
  if (TOP2) {  // no load yet: every latency is C_g(0) = 0; one GPU has no "others" (-inf)
    tp = top_p + r * T;
    td = top_d + r * T;
    ta = top_a + r * T;
    const float ninf = __int_as_float(0xff800000);
    for (int64_t t = tid; t < T; t += blockDim.x) {
      tp[t] = make_float2(0.0f, G > 1 ? 0.0f : ninf);
      td[t] = make_double2(0.0, G > 1 ? 0.0 : (double)ninf);
      ta[t] = 0;
    }
  }
  const int cap = E / G;
  __syncthreads();
  for (int idx = 0; idx < E; ++idx) {
    const int e = order[r * E + idx];
    const uint16_t* hcol = hl + (int64_t)e * ws.Tp;
    unsigned avail = 0;
    for (int g = 0; g < G; ++g)
      if (counts[g] < cap) avail |= 1u << g;
    // ---- approximate scores of every GPU (any summation order; GPUs without
    // capacity are computed too and ignored by the selection). Per step: the
    // current fp32 latencies of all GPUs (8 gathers), the max over the others
    // of each GPU from prefix/suffix maxima (branch-free), the candidate
    // latency C'_g(l_g + h) (one gather per GPU); every fp32 term is added to
    // an fp64 partial sum (any order: relative error <= 2^-24 + T 2^-53, the
    // kWindow screen -- a wider window would send more near-ties of cold
    // experts to the exact re-score).
    double acc[GM];
    uint32_t row_addr[GM];
    unsigned exc = 0u;
    const uint32_t wlast = (uint32_t)W - 1u;
#pragma unroll
    for (int g = 0; g < GM; ++g) {
      acc[g] = 0.0;
      row_addr[g] = lut_base + 4u * (uint32_t)(g < G ? g : G - 1) * (uint32_t)W;
    }
    auto approx_pass = [&](auto pw_tag) {
      constexpr bool PW = decltype(pw_tag)::value;
#pragma unroll kGreedyUnroll
    for (int64_t t = tid; t < T; t += blockDim.x) {
      const uint32_t hv = (uint32_t)hcol[t];
      float2 p12;
      int parg = 0;
      if (TOP2) {
        p12 = tp[t];
        parg = ta[t];
      }
      uint32_t lrow[GM];
      // the step's GM u16 loads: GM/8 16-byte loads (rows are 16-byte aligned)
#pragma unroll
      for (int qv = 0; qv < GM / 8; ++qv) {
        const uint4 v = reinterpret_cast<const uint4*>(ld + t * GM)[qv];
        const uint32_t w4[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          lrow[8 * qv + 2 * q] = w4[q] & 0xffffu;
          lrow[8 * qv + 2 * q + 1] = w4[q] >> 16;
        }
      }
      // rows of GPUs g >= G (GM padding) read row G-1 and are masked by select: no branches
      float pre[GM + 1], suf[GM + 1];
      if (!TOP2) {
        float cur[GM];
#pragma unroll
        for (int g = 0; g < GM; ++g) {
          const float v = tab(row_addr, g, lrow[g]);
          cur[g] = g < G ? v : __int_as_float(0xff800000);
        }
        pre[0] = __int_as_float(0xff800000);
        suf[GM] = __int_as_float(0xff800000);
#pragma unroll
        for (int g = 0; g < GM; ++g) pre[g + 1] = fmaxf(pre[g], cur[g]);
#pragma unroll
        for (int g = GM - 1; g >= 0; --g) suf[g] = fmaxf(suf[g + 1], cur[g]);
      }
#pragma unroll
      for (int g = 0; g < GM; ++g) {
        // a GPU with free capacity never exceeds the window (l + h <= U); a
        // full one (ignored by the selection) is clamped to stay inside it
        float cl;
        if constexpr (PW) {  // within 2^-22 of C: the exc test below keeps a 2^-20 margin
          const uint32_t nn = min(lrow[g] + hv, wlast);
          const int j = pw_bucket(nn);
          cl = pw_eval(s_pw[(g < G ? g : G - 1) * pwK + j], nn, j);
        } else {
          cl = tab(row_addr, g, min(lrow[g] + hv, wlast));
        }
        const float pm = TOP2 ? (g == parg ? p12.y : p12.x) : fmaxf(pre[g], suf[g + 1]);
        acc[g] += (double)fmaxf(pm, cl);  // g >= G: ignored by the selection
        // hv == 0: the term is the step maximum exactly; PW: cl may sit 2^-22
        // below C, so only cl (1 + 2^-20) < pm proves C < the others' maximum
        if (hv != 0u && (PW ? cl * (1.0f + 0x1p-20f) >= pm : cl >= pm)) exc |= 1u << g;
      }
    }
    };
    if constexpr (!SL) {
      if (usepw) approx_pass(std::true_type{});
      else approx_pass(std::false_type{});
    } else {
      approx_pass(std::false_type{});
    }
#pragma unroll
    for (int g = 0; g < GM; ++g) {
      double v = acc[g];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0) red[warp * GM + g] = v;
    }
    exc = __reduce_or_sync(0xffffffffu, exc);
    if (lane == 0 && exc) atomicOr(&s_exc, exc);
    __syncthreads();
    if (tid == 0) {
      double mn = __longlong_as_double(0x7ff0000000000000LL);
      for (int g = 0; g < G; ++g) {
        double v = 0.0;
        for (int w = 0; w < nwarps; ++w) v += red[w * GM + g];
        red[g] = v;  // warp 0's slots are no longer needed
        if (avail >> g & 1u) mn = fmin(mn, v);
      }
      const double lim = mn * kWindow;
      // Monotone tables: no placement scores below S_M = the serial sum of the
      // current step maxima. A GPU scores exactly S_M if at every step either
      // the expert adds nothing (h = 0: the same table entry) or its fp32
      // candidate latency is strictly below the fp32 maximum of the others
      // (then so is the exact one -- rounding is monotone -- and the GPU is
      // not the step's unique maximum, so the others' maximum is the step's).
      // The lowest such GPU g* wins unless a window GPU of lower index ties
      // it; only those need the exact chains.
      const unsigned nx = ws.lut_monotone64 ? (avail & ~s_exc) : 0u;
      const int gstar = nx ? __ffs(nx) - 1 : G;
      s_exc = 0u;
      int nc = 0;
      for (int g = 0; g < gstar; ++g)
        if ((avail >> g & 1u) && red[g] <= lim) s_cand[nc++] = g;
      if (gstar < G) s_cand[nc++] = gstar;
      s_ncand = nc;
      s_best = s_cand[0];
    }
    __syncthreads();
    if (s_ncand > 1 && kGreedyRefine) {
      // ---- fp64 screen of the window's GPUs: the exact terms (v1 arithmetic)
      // summed in parallel (per thread, then a warp tree, then warps in order:
      // <= T/threads + 5 + warps adds per term), so every score is within
      // 2^-38.9 of its serial chain (which is within T 2^-53 of the real sum);
      // GPUs above min * kRefineWindow cannot hold the strict-< minimum. A
      // single survivor is the winner; ties and near-ties go to the chains.
      const int nc = s_ncand;
      double a64[GM];
#pragma unroll
      for (int c = 0; c < GM; ++c) a64[c] = 0.0;
      for (int64_t t = tid; t < T; t += blockDim.x) {
        double m1 = -1.0, m2 = -1.0;
        int i1 = -1;
        if (TOP2) {
          const double2 d = td[t];
          m1 = d.x;
          m2 = d.y;
          i1 = ta[t];
        } else {
          for (int q = 0; q < G; ++q) {
            const double v = __ldg(lut + q * width + ld[LDI(t, q)]);
            if (v > m1) { m2 = m1; m1 = v; i1 = q; }
            else if (v > m2) { m2 = v; }
          }
        }
        const int hv = hcol[t];
#pragma unroll
        for (int c = 0; c < GM; ++c) {
          if (c >= nc) break;
          const int g = s_cand[c];
          const double cl = __ldg(lut + g * width + (int64_t)ld[LDI(t, g)] + hv);
          double scv = cl;
          if (G > 1) {
            const double others = (i1 == g) ? m2 : m1;
            scv = others > cl ? others : cl;
          }
          a64[c] += scv;
        }
      }
#pragma unroll
      for (int c = 0; c < GM; ++c) {
        if (c >= nc) break;
        double v = a64[c];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) red[warp * GM + c] = v;
      }
      __syncthreads();
      if (tid == 0) {
        double mn = __longlong_as_double(0x7ff0000000000000LL);
        for (int c = 0; c < nc; ++c) {
          double v = 0.0;
          for (int w = 0; w < nwarps; ++w) v += red[w * GM + c];
          red[c] = v;  // warp 0's slots are consumed in order
          mn = fmin(mn, v);
        }
        const double lim = mn * kRefineWindow;
        int k = 0;
        for (int c = 0; c < nc; ++c)
          if (red[c] <= lim) s_cand[k++] = s_cand[c];  // ascending GPU order is kept
        s_ncand = k;
        s_best = s_cand[0];
      }
      __syncthreads();
    }
    if (s_ncand > 1) {
      if (tid == 0) atomicAdd(&ws.counters[2], 1);  // statistics: exact re-scores
      // ---- exact serial scores of the window's GPUs (v1 arithmetic, t order):
      // per chunk all threads fill the exact terms of every window GPU (one
      // exact top-2 per step), then thread c extends candidate c's serial chain
      const int nc = s_ncand;
      double chain = 0.0;
      for (int64_t t0 = 0; t0 < T; t0 += kGreedyTChunk) {
        const int tn = (int)imin64(kGreedyTChunk, T - t0);
        for (int tt = tid; tt < tn; tt += blockDim.x) {
          const int64_t t = t0 + tt;
          double m1 = -1.0, m2 = -1.0;
          int i1 = -1;
          if (TOP2) {
            const double2 d = td[t];
            m1 = d.x;
            m2 = d.y;
            i1 = ta[t];
          } else {
            for (int q = 0; q < G; ++q) {
              const double v = __ldg(lut + q * width + ld[LDI(t, q)]);
              if (v > m1) { m2 = m1; m1 = v; i1 = q; }
              else if (v > m2) { m2 = v; }
            }
          }
          const int hv = h[t * E + e];
          for (int c = 0; c < nc; ++c) {
            const int g = s_cand[c];
            const double cl = __ldg(lut + g * width + (int64_t)ld[LDI(t, g)] + hv);
            double scv = cl;
            if (G > 1) {
              const double others = (i1 == g) ? m2 : m1;
              scv = others > cl ? others : cl;
            }
            buf[c * kGreedyTChunk + tt] = scv;
          }
        }
        __syncthreads();
        if (tid < nc) {
          const double* bc = buf + tid * kGreedyTChunk;
          for (int tt = 0; tt < tn; ++tt) chain = dadd(chain, bc[tt]);
        }
        __syncthreads();
      }
      if (tid < nc) red[tid] = chain;  // red[] is free again (the approximate scores are consumed)
      __syncthreads();
      if (tid == 0) {  // strict < in ascending GPU order (search.py:156)
        double best = red[0];
        int bg = s_cand[0];
        for (int c = 1; c < nc; ++c)
          if (red[c] < best) { best = red[c]; bg = s_cand[c]; }
        s_best = bg;
      }
      __syncthreads();
    }
    const int bg = s_best;
    // add the expert's counts to the chosen GPU's loads: all loads of a batch
    // first, then the stores (the compiler cannot move a load of hcol above a
    // store to ld, so the naive loop pays one L2 round trip per step)
    constexpr int kUpd = 8;
    for (int64_t t0 = tid; t0 < T; t0 += (int64_t)kUpd * blockDim.x) {
      uint32_t hv[kUpd], lv[kUpd];
#pragma unroll
      for (int u = 0; u < kUpd; ++u) {
        const int64_t t = t0 + (int64_t)u * blockDim.x;
        hv[u] = t < T ? hcol[t] : 0u;
        lv[u] = t < T ? ld[LDI(t, bg)] : 0u;
      }
#pragma unroll
      for (int u = 0; u < kUpd; ++u) {
        const int64_t t = t0 + (int64_t)u * blockDim.x;
        if (t < T) ld[LDI(t, bg)] = (uint16_t)(lv[u] + hv[u]);
      }
      if (TOP2) {  // the chosen GPU's latency grew where the expert has tokens
        double nl[kUpd];
        double2 d[kUpd];
        int a[kUpd];
#pragma unroll
        for (int u = 0; u < kUpd; ++u) {
          const int64_t t = t0 + (int64_t)u * blockDim.x;
          const bool on = t < T && hv[u] != 0u;
          nl[u] = on ? __ldg(lut + (int64_t)bg * width + lv[u] + hv[u]) : 0.0;
          d[u] = on ? td[t] : make_double2(0.0, 0.0);
          a[u] = on ? ta[t] : 0;
        }
#pragma unroll
        for (int u = 0; u < kUpd; ++u) {
          const int64_t t = t0 + (int64_t)u * blockDim.x;
          if (!(t < T && hv[u] != 0u)) continue;
          double d1 = d[u].x, d2 = d[u].y;
          int ar = a[u];
          if (ar == bg) {
            d1 = nl[u];  // the maximum grew (it was bg's); the runner-up is unchanged
          } else if (nl[u] > d1) {
            d2 = d1;
            d1 = nl[u];
            ar = bg;
          } else if (nl[u] > d2) {
            d2 = nl[u];
          }
          td[t] = make_double2(d1, d2);
          tp[t] = make_float2((float)d1, (float)d2);
          ta[t] = (uint8_t)ar;
        }
      }
    }
    if (tid == 0) {
      assign[r * E + e] = (int8_t)bg;
      counts[bg] += 1;
    }
    __syncthreads();
  }
  // hand the loads to the refinement in the int32 [T][G] layout
  int32_t* out = ws.loads + r * T * G;
  for (int64_t i = tid; i < T * G; i += blockDim.x) out[i] = ld[LDI(i / G, (int)(i % G))];
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
// Serial score of one run (sum over t in order of max_g lat). Thread 0 extends
// the chain over chunk c while warps 1.. fill chunk c+1 (double buffer), so
// the chain -- the latency floor -- is not serialised with the table gathers.
constexpr int kScoreChunk = 1024;  // steps per block_score buffer (several gathers in flight per producer)
// One serial fp64 chain over T terms per CTA: warps 1.. fill chunk k+1 of
// term(t) into shared memory while thread 0 folds chunk k in t order.
template <int CHUNK = kScoreChunk, typename Term>
__device__ double block_chain(int64_t T, double* buf /*[2][CHUNK]*/, Term term) {
  const int nw = blockDim.x >> 5;
  const int ptid = nw > 1 ? (int)threadIdx.x - 32 : (int)threadIdx.x;  // producer index (warps 1..)
  const int np = nw > 1 ? (int)blockDim.x - 32 : (int)blockDim.x;
  auto fill = [&](int64_t t0, double* b) {
    const int tn = (int)imin64(CHUNK, T - t0);
#pragma unroll 4
    for (int tt = ptid; tt < tn; tt += np) b[tt] = term(t0 + tt);
  };
  double sum = 0.0;
  if (ptid >= 0) fill(0, buf);
  __syncthreads();
  int k = 0;
  for (int64_t t0 = 0; t0 < T; t0 += CHUNK, k ^= 1) {
    const int tn = (int)imin64(CHUNK, T - t0);
    if (nw == 1) {
      if (threadIdx.x == 0)
        for (int tt = 0; tt < tn; ++tt) sum = dadd(sum, buf[k * CHUNK + tt]);
      __syncthreads();
      if (t0 + CHUNK < T) fill(t0 + CHUNK, buf + (k ^ 1) * CHUNK);
    } else if (threadIdx.x == 0) {
      const double* b = buf + k * CHUNK;
#pragma unroll 8
      for (int tt = 0; tt < tn; ++tt) sum = dadd(sum, b[tt]);
    } else if (ptid >= 0 && t0 + CHUNK < T) {
      fill(t0 + CHUNK, buf + (k ^ 1) * CHUNK);
    }
    __syncthreads();
  }
  return sum;  // valid in thread 0
}

__device__ double block_score(const int32_t* __restrict__ ld, int64_t T, int G, const double* __restrict__ lut,
                              int64_t width, double* buf /*[2][kScoreChunk]*/) {
  return block_chain(T, buf, [&](int64_t t) { return max_lat_excl(ld + t * G, G, lut, width, -1, -1); });
}

__global__ void __launch_bounds__(kSearchThreads)
init_score_kernel(int64_t T, int G, const double* __restrict__ lut, int64_t nmax, SearchWs ws, int64_t traj_cap,
                  double* __restrict__ trajectory, int32_t* __restrict__ swaps) {
  __shared__ double buf[2 * kScoreChunk];
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
                 SearchWs ws, const int32_t* __restrict__ filter, const int32_t* __restrict__ rlist) {
  extern __shared__ unsigned char bsm[];
  const int64_t r = rlist ? rlist[blockIdx.x] : blockIdx.x;  // rlist: the compacted active runs
  if (!ws.run_active[r] || (filter && filter[r] != kNeedExact)) return;
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


// ---------------------------------------------------------------------------
// K6 v3: screened best-swap scan.
//
// The reference picks the pair with the smallest EXACT serial-fp64 candidate
// score (lowest i*E+j on ties). Evaluating every pair exactly is bound by the
// two latency-table gathers per pair-step; the fp64 table rows of two GPUs do
// not fit shared memory next to the staging buffers, and from L1 a random
// gather costs a wavefront per line. So the scan runs in two passes:
//
//  1. approximate pass (this kernel): the fp32 rounding of the table rows a
//     and b lives in shared memory (2 x (nmax+1) x 4 B); each pair-step is
//     m' = max(po', C'_a, C'_b) in fp32 (rounding is monotone, so m' is
//     exactly fl32(m)) accumulated serially in fp64. Then
//     |cand' - cand| <= 2^-24 cand + 2 T 2^-53 cand < 2^-22 cand, and the
//     exact winner satisfies cand'(win) <= min' * (1+2^-22)/(1-2^-22)
//     < min' * (1 + 2^-20) =: window. Every CTA keeps the pairs inside ITS
//     window (a superset of the ones inside the run's window);
//  2. the pairs inside the run's window (usually one or two) are evaluated
//     exactly, exactly as v1 does, and the lexicographic (cand, flat) minimum
//     is taken. A run whose window holds more than kCandK pairs (or a tile
//     that overflowed kLocK) falls back to the exact v1 scan.
// The selected pair and its score are therefore the reference's, bit for bit.
//
// CTA = (GPU pair a<b, RPC active runs). Every run places exactly n = E/G
// experts on each GPU, so a (run, pair) tile has n*n expert pairs; a thread
// owns one x (on a) and kSwapY consecutive y (on b): kSwapY independent
// chains. Per t-chunk the CTA copies, with 16-byte cp.async into a double
// buffer, for each of its runs: the count rows of the a- and b-experts
// (transposed uint16 histogram, one contiguous 64-byte run per expert), the
// run's l_a / l_b rows and the fp32 latency rows of every GPU (transposed
// per-run state kept current across swaps), then derives pother'.
#ifndef GEM_SWAP_Y
#define GEM_SWAP_Y 4
#endif
constexpr int kSwapY = GEM_SWAP_Y;
#ifndef GEM_SCAN_THREADS
#define GEM_SCAN_THREADS 256
#endif
constexpr int kSwap3Threads = GEM_SCAN_THREADS;
constexpr int kSwap3TChunk = 32;

struct Swap3Geom {
  int n, ng, nb_pad, units_per_run, rpc;
};

__host__ __device__ inline Swap3Geom swap3_geom(int E, int G, int Y = kSwapY) {
  Swap3Geom g;
  g.n = E / G;
  g.ng = (g.n + Y - 1) / Y;
  g.nb_pad = g.ng * Y;
  g.units_per_run = g.n * g.ng;
  g.rpc = kSwap3Threads / g.units_per_run;
  if (g.rpc < 1) g.rpc = 1;
  if (g.rpc > 16) g.rpc = 16;
  return g;
}

// one staging buffer: per run, [n + nb_pad] count rows + l_a + l_b (uint16),
// [G] latency rows + pother' (fp32); every row is kSwap3TChunk long
__host__ __device__ inline size_t swap3_buf_bytes(const Swap3Geom& g, int G) {
  return (size_t)g.rpc * kSwap3TChunk * (2 * ((size_t)g.n + g.nb_pad + 2) + 4 * ((size_t)G + 1));
}

__host__ __device__ inline size_t swap3_smem(int E, int G, int64_t nmax) {
  const Swap3Geom g = swap3_geom(E, G);
  const size_t lut = ((size_t)2 * (size_t)(nmax + 1) * 4 + 15) & ~size_t(15);
  const size_t fixed = (size_t)g.rpc * (8 + 8 + 8 + 8 + 2 * g.n * 2) + 64;
  return lut + 2 * swap3_buf_bytes(g, G) + fixed;
}

__device__ __forceinline__ unsigned long long ord_bits(double v) {  // monotone for v >= 0 (and +inf)
  return (unsigned long long)__double_as_longlong(v);
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(smem)),
               "l"(gmem)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait_n() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__global__ void __launch_bounds__(kSwap3Threads, 2)
approx_scan_kernel(int64_t T, int E, int G, int64_t nmax, const int32_t* __restrict__ run_layer,
                   const int8_t* __restrict__ assign, int32_t n_active, SearchWs ws) {
  extern __shared__ __align__(16) unsigned char s3[];
  const Swap3Geom geo = swap3_geom(E, G);
  const int n = geo.n, ng = geo.ng, RPC = geo.rpc, nb_pad = geo.nb_pad;
  const int NP = G * (G - 1) / 2;
  const int slot0 = blockIdx.y * RPC;
  if (slot0 >= n_active) return;
  const int nruns = min(RPC, n_active - slot0);
  int p = blockIdx.x, a = 0;
  while (p >= G - 1 - a) { p -= G - 1 - a; ++a; }
  const int b = a + 1 + p;
  const int64_t width = nmax + 1;
  const int64_t Tp = ws.Tp;
  constexpr int TC = kSwap3TChunk;
  constexpr int V = TC * 2 / 16;  // 16-byte pieces per uint16 row of a chunk
  constexpr int VF = TC * 4 / 16; // 16-byte pieces per fp32 row of a chunk
  const int hrows = n + nb_pad;   // a-expert rows, then b-expert rows (zero padded)

  float* lut_a = reinterpret_cast<float*>(s3);
  float* lut_b = lut_a + width;
  unsigned char* cur = s3 + (((size_t)2 * width * 4 + 15) & ~size_t(15));
  const size_t buf_bytes = swap3_buf_bytes(geo, G);
  unsigned char* bufs = cur;
  cur += 2 * buf_bytes;
  unsigned long long* smin = reinterpret_cast<unsigned long long*>(cur);  cur += (size_t)RPC * 8;
  const uint16_t** hsrc = reinterpret_cast<const uint16_t**>(cur);       cur += (size_t)RPC * 8;  // ht16 + layer*E*Tp
  const uint16_t** lsrc = reinterpret_cast<const uint16_t**>(cur);       cur += (size_t)RPC * 8;  // loadT + r*G*Tp
  const float** fsrc = reinterpret_cast<const float**>(cur);             cur += (size_t)RPC * 8;  // latT + r*G*Tp
  int16_t* lists = reinterpret_cast<int16_t*>(cur);                       // [RPC][2][n]
  struct Buf {
    uint16_t* h;   // [RPC][hrows][TC]
    uint16_t* l;   // [RPC][2][TC]   l_a, l_b
    float* lat;    // [RPC][G][TC]
    float* po;     // [RPC][TC]
  };
  auto buf_at = [&](int k) {
    unsigned char* c = bufs + k * buf_bytes;
    Buf B;
    B.h = reinterpret_cast<uint16_t*>(c);  c += (size_t)RPC * hrows * TC * 2;
    B.l = reinterpret_cast<uint16_t*>(c);  c += (size_t)RPC * 2 * TC * 2;
    B.lat = reinterpret_cast<float*>(c);   c += (size_t)RPC * G * TC * 4;
    B.po = reinterpret_cast<float*>(c);
    return B;
  };

  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
  {
    const float* la32 = ws.lut32 + (int64_t)a * width;
    const float* lb32 = ws.lut32 + (int64_t)b * width;
    for (int64_t i = tid; i < width; i += blockDim.x) {
      lut_a[i] = __ldg(la32 + i);
      lut_b[i] = __ldg(lb32 + i);
    }
  }
  if (tid < RPC) smin[tid] = ord_bits(__longlong_as_double(0x7ff0000000000000LL));
  if (tid < nruns) {
    const int r = ws.run_list[slot0 + tid];
    hsrc[tid] = ws.ht16 + (int64_t)run_layer[r] * E * Tp;
    lsrc[tid] = ws.loadT + (int64_t)r * G * Tp;
    fsrc[tid] = ws.latT + (int64_t)r * G * Tp;
  }
  // expert lists of the CTA's runs (ascending expert index on each GPU)
  for (int w = wid; w < nruns; w += nw) {
    const int r = ws.run_list[slot0 + w];
    const int8_t* as = assign + (int64_t)r * E;
    int base_a = 0, base_b = 0;
    for (int e0 = 0; e0 < E; e0 += 32) {
      const int e = e0 + lane;
      const int g = e < E ? as[e] : -1;
      const unsigned ma = __ballot_sync(0xffffffffu, g == a), mb = __ballot_sync(0xffffffffu, g == b);
      const unsigned below = (1u << lane) - 1u;
      if (g == a) lists[(w * 2 + 0) * n + base_a + __popc(ma & below)] = (int16_t)e;
      if (g == b) lists[(w * 2 + 1) * n + base_b + __popc(mb & below)] = (int16_t)e;
      base_a += __popc(ma);
      base_b += __popc(mb);
    }
  }
  // padded b-rows (y >= n) stay zero in both buffers
  for (int k = 0; k < 2; ++k) {
    const Buf B = buf_at(k);
    for (int i = tid; i < RPC * hrows * TC; i += blockDim.x) B.h[i] = 0;
  }
  __syncthreads();

  // 16-byte cp.async pieces of one chunk: per run, (n + n) count rows, 2 load
  // rows, G latency rows
  const int pieces_h = 2 * n * V, pieces_l = 2 * V, pieces_f = G * VF;
  const int pieces_run = pieces_h + pieces_l + pieces_f;
  auto issue = [&](int64_t t0, int k) {
    const Buf B = buf_at(k);
    for (int i = tid; i < nruns * pieces_run; i += blockDim.x) {
      const int ss = i / pieces_run;
      int q = i - ss * pieces_run;
      if (q < pieces_h) {
        const int row = q / V, v = q - row * V;  // row < n: a-expert row, else b-expert row - n
        const int e = row < n ? lists[(ss * 2 + 0) * n + row] : lists[(ss * 2 + 1) * n + row - n];
        const int drow = row < n ? row : row - n + n;  // b rows start at n (padding after them)
        cp_async16(B.h + ((size_t)ss * hrows + drow) * TC + v * 8, hsrc[ss] + (int64_t)e * Tp + t0 + v * 8);
      } else if ((q -= pieces_h) < pieces_l) {
        const int which = q / V, v = q - which * V;
        cp_async16(B.l + ((size_t)ss * 2 + which) * TC + v * 8,
                   lsrc[ss] + (int64_t)(which ? b : a) * Tp + t0 + v * 8);
      } else {
        q -= pieces_l;
        const int g = q / VF, v = q - g * VF;
        cp_async16(B.lat + ((size_t)ss * G + g) * TC + v * 4, fsrc[ss] + (int64_t)g * Tp + t0 + v * 4);
      }
    }
  };

  const int units_total = nruns * geo.units_per_run;
  for (int pass0 = 0; pass0 < units_total; pass0 += blockDim.x) {
    const int u = pass0 + tid;
    const bool live = u < units_total;
    const int s = live ? u / geo.units_per_run : 0;
    const int ur = live ? u % geo.units_per_run : 0;
    const int x = ur / ng, yg = ur % ng;
    double acc[kSwapY];
#pragma unroll
    for (int q = 0; q < kSwapY; ++q) acc[q] = 0.0;

    issue(0, 0);
    cp_async_commit();
    int k = 0;
    for (int64_t t0 = 0; t0 < T; t0 += TC, k ^= 1) {
      const int tn = (int)imin64(TC, T - t0);
      if (t0 + TC < T) issue(t0 + TC, k ^ 1);
      cp_async_commit();  // (possibly empty) group of the next chunk
      cp_async_wait1();   // this chunk's group has landed
      __syncthreads();
      const Buf B = buf_at(k);
      for (int rr = tid; rr < nruns * TC; rr += blockDim.x) {
        const int ss = rr / TC, tt = rr % TC;
        const float* lat = B.lat + (size_t)ss * G * TC + tt;
        float m = __int_as_float(0xff800000);  // -inf when G == 2
        for (int g = 0; g < G; ++g)
          if (g != a && g != b) m = fmaxf(m, lat[g * TC]);
        B.po[ss * TC + tt] = m;
      }
      __syncthreads();
      if (live) {
        const float* pos = B.po + s * TC;
        const uint16_t* las = B.l + (size_t)s * 2 * TC;
        const uint16_t* lbs = las + TC;
        const uint16_t* hAs = B.h + ((size_t)s * hrows + x) * TC;
        const uint16_t* hBs = B.h + ((size_t)s * hrows + n + yg * kSwapY) * TC;
#pragma unroll 4
        for (int tt = 0; tt < tn; ++tt) {
          const int32_t hx = hAs[tt];
          const int32_t ra = (int32_t)las[tt] - hx, rb = (int32_t)lbs[tt] + hx;
          const float pm = pos[tt];
#pragma unroll
          for (int q = 0; q < kSwapY; ++q) {
            const int32_t hy = hBs[q * TC + tt];
            const float m = fmaxf(fmaxf(pm, lut_a[ra + hy]), lut_b[rb - hy]);
            acc[q] = dadd(acc[q], (double)m);
          }
        }
      }
      __syncthreads();  // buffer k is rewritten by the issue of the chunk after next
    }
    // tile minimum, then every pair inside the tile's window is recorded
    if (live) {
      double mn = acc[0];
#pragma unroll
      for (int q = 1; q < kSwapY; ++q)
        if (yg * kSwapY + q < n) mn = fmin(mn, acc[q]);
      atomicMin(&smin[s], ord_bits(mn));
    }
    __syncthreads();
    if (live) {
      const int r = ws.run_list[slot0 + s];
      const int64_t tile = (int64_t)r * NP + blockIdx.x;
      const double lim = __longlong_as_double((long long)smin[s]) * kWindow;
      const int xe = lists[(s * 2 + 0) * n + x];
#pragma unroll
      for (int q = 0; q < kSwapY; ++q) {
        const int yi = yg * kSwapY + q;
        if (yi >= n || !(acc[q] <= lim)) continue;
        const int ye = lists[(s * 2 + 1) * n + yi];
        const int f = xe < ye ? xe * E + ye : ye * E + xe;
        const int kk = atomicAdd(&ws.loc_cnt[tile], 1);
        if (kk < kLocK) {
          ws.loc_cand[tile * kLocK + kk] = acc[q];
          ws.loc_flat[tile * kLocK + kk] = f;
        }
      }
    }
  }
  __syncthreads();
  if (tid < nruns) {
    const int r = ws.run_list[slot0 + tid];
    ws.loc_min[(int64_t)r * NP + blockIdx.x] = __longlong_as_double((long long)smin[tid]);
  }
}

// ---------------------------------------------------------------------------
// K6 v5: the screened scan with fp32 chunk sums and conflict-free staging.
//
// ncu on v4: shared-memory wavefronts at 95% of peak, 8.1 wavefronts per warp
// pair-step, of which the two table gathers are 5.4 (random rows: ~2.7-way
// bank conflicts) and the count-row loads 2.2 (64-byte row stride puts the
// rows of one warp on the same banks); 15.5 instructions per pair-step
// (address arithmetic, u16 unpacking, F2F + DADD per term).
//
// v5 keeps v4's CTA layout and the exact second pass, and changes the inner loop:
//  * count rows are staged with an 80-byte stride and a thread's y experts are
//    interleaved (y = yg + q*ng), so the 8 x rows and the 4 y rows a warp reads
//    at one step sit on distinct banks; 4 steps per 64-bit load;
//  * counts are pre-scaled by 4 (byte offsets: ht16s), so a gather address is
//    ONE add: (table base + 4 l_a - 4 h_x) + 4 h_y;
//  * each term m' = fl32(m) (exact rounding of the exact maximum, as in v4) is
//    summed in fp32 over a 32-step chunk and the chunk sum is added to an
//    fp64 chain: |cand' - cand| <= (32 * 2^-24 + (T/32) 2^-53) cand < 2^-18.9
//    cand for nonnegative tables, so the exact winner lies inside
//    cand' <= min' * (1 + 2^-17) (kWindow5). Steps past T are zero rows and
//    add exactly 0 (C_g(0) = 0, pother' = 0).
#ifndef GEM_SCAN_TC
#define GEM_SCAN_TC 32
#endif
#ifndef GEM_SCAN_MINB
#define GEM_SCAN_MINB 2
#endif
constexpr int kSwap5TChunk = GEM_SCAN_TC;
#ifndef GEM_SCAN_STAGES
#define GEM_SCAN_STAGES 3
#endif
constexpr int kSwap5Stages = GEM_SCAN_STAGES;  // cp.async staging buffers
static_assert(kSwap5Stages >= 3, "the scan issues chunk c+S-1 after chunk c-1's slot is free");
constexpr int kSwap5RowU16 = kSwap5TChunk + 8;  // staged count row: the chunk's steps + 16-byte pad

__host__ __device__ inline size_t swap5_buf_bytes(const Swap3Geom& g, int G) {
  (void)G;
  return (size_t)g.rpc * ((size_t)(g.n + g.nb_pad) * kSwap5RowU16 * 2 + 2 * (size_t)kSwap5TChunk * 2 +
                          4 * ((size_t)4 + 3) * kSwap5TChunk);  // top-3 rows (4), pother', 2 clamp rows
}

// W = table window (loads never exceed W - 1)
__host__ __device__ inline size_t swap5_smem(int E, int G, int64_t W, int Y) {
  const Swap3Geom g = swap3_geom(E, G, Y);
  const size_t lut = ((size_t)2 * (size_t)W * 4 + 15) & ~size_t(15);
  const size_t fixed = (size_t)g.rpc * (8 + 8 + 8 + 8) + ((((size_t)g.rpc * 2 * g.n * 2) + 15) & ~size_t(15)) +
                       2 * (kBuckets + 2) * 2 + 64;
  return lut + kSwap5Stages * swap5_buf_bytes(g, G) + fixed;
}


// GT > 0: instantiated for exactly GT GPUs (the pother pass unrolls); 0: any G.
// Y: y experts per thread (4; 2 when a GPU holds <= 8 experts, so a CTA's
// per-run staging halves and two CTAs fit an SM -- the DeepSeek-V3 shape)
template <int GT, int Y>
__global__ void __launch_bounds__(kSwap3Threads, GEM_SCAN_MINB)
approx_scan5_kernel(int E, int G_, int64_t nmax, int W, int monotone, const int32_t* __restrict__ run_layer,
                    const int8_t* __restrict__ assign, int32_t n_active, SearchWs ws, int64_t tseg,
                    const uint8_t* __restrict__ prune) {
  extern __shared__ __align__(16) unsigned char s5[];
  const int G = GT > 0 ? GT : G_;
  const Swap3Geom geo = swap3_geom(E, G, Y);
  const int n = geo.n, ng = geo.ng, RPC = geo.rpc, nb_pad = geo.nb_pad;
  const int NP = G * (G - 1) / 2;
  const int slot0 = blockIdx.y * RPC;
  if (slot0 >= n_active) return;
  const int nslots = min(RPC, n_active - slot0);
  // the CTA's runs whose tile survives the bound (tile_bound_kernel; all when
  // prune == nullptr), compacted: unit s works on active slot slot0 + s_live[s]
  __shared__ int s_live[16], s_nlive;
  int p = blockIdx.x, a = 0;
  while (p >= G - 1 - a) { p -= G - 1 - a; ++a; }
  const int b = a + 1 + p;
  const int64_t width = nmax + 1;
  // step range of this CTA: all of [0, Tp), or (split scans, tseg > 0) the
  // blockIdx.z-th segment of tseg steps; split CTAs add their partial sums to
  // ws.split_acc and split_window_kernel finishes the tiles
  const bool split = tseg > 0;
  if (threadIdx.x == 0) {
    int c = 0;
    for (int w = 0; w < nslots; ++w) {
      if (prune != nullptr && prune[(int64_t)(slot0 + w) * NP + blockIdx.x] != 0) {
        // no pair of this tile can be accepted: it takes no part in the minimum
        ws.loc_min[(int64_t)ws.run_list[slot0 + w] * NP + blockIdx.x] = __longlong_as_double(0x7ff0000000000000LL);
      } else {
        s_live[c++] = w;
      }
    }
    s_nlive = c;
  }
  __syncthreads();
  const int nruns = s_nlive;
  if (nruns == 0) return;
  const int64_t Tp = ws.Tp;  // row stride of the transposed arrays
  const int64_t tb = split ? (int64_t)blockIdx.z * tseg : 0;
  const int64_t te = split ? imin64(Tp, tb + tseg) : Tp;  // this CTA's steps: [tb, te)
  if (tb >= te) return;
  constexpr int TC = kSwap5TChunk;
  constexpr int RS = kSwap5RowU16;
  constexpr int V = TC * 2 / 16;  // 16-byte pieces per uint16 row of a chunk
  constexpr int VF = TC * 4 / 16; // 16-byte pieces per fp32 row of a chunk
  const int hrows = n + nb_pad;   // a-expert rows, then b-expert rows (zero padded)

  float* lut_a = reinterpret_cast<float*>(s5);
  float* lut_b = lut_a + W;
  unsigned char* cur = s5 + (((size_t)2 * W * 4 + 15) & ~size_t(15));
  const size_t buf_bytes = swap5_buf_bytes(geo, G);
  unsigned char* bufs = cur;
  cur += kSwap5Stages * buf_bytes;
  unsigned long long* smin = reinterpret_cast<unsigned long long*>(cur);  cur += (size_t)RPC * 8;
  const uint16_t** hsrc = reinterpret_cast<const uint16_t**>(cur);       cur += (size_t)RPC * 8;
  const uint16_t** lsrc = reinterpret_cast<const uint16_t**>(cur);       cur += (size_t)RPC * 8;
  const float** fsrc = reinterpret_cast<const float**>(cur);             cur += (size_t)RPC * 8;
  int16_t* lists = reinterpret_cast<int16_t*>(cur);                       // [RPC][2][n]
  cur += (((size_t)RPC * 2 * n * 2) + 15) & ~size_t(15);
  uint16_t* first_a = reinterpret_cast<uint16_t*>(cur);                   // [kBuckets + 2] x 2
  uint16_t* first_b = first_a + (kBuckets + 2);
  struct Buf {
    uint16_t* h;   // [RPC][hrows][RS]  4 * count
    uint16_t* l;   // [RPC][2][TC]      l_a, l_b
    float* lat;    // [RPC][G][TC]
    float* po;     // [RPC][TC]
    uint32_t* th;  // [RPC][2][TC]  clamp addresses into the a and b rows
  };
  auto buf_at = [&](int k) {
    unsigned char* c = bufs + k * buf_bytes;
    Buf B;
    B.h = reinterpret_cast<uint16_t*>(c);  c += (size_t)RPC * hrows * RS * 2;
    B.l = reinterpret_cast<uint16_t*>(c);  c += (size_t)RPC * 2 * TC * 2;
    B.lat = reinterpret_cast<float*>(c);   c += (size_t)RPC * 4 * TC * 4;  // top-3 values + packed GPUs
    B.po = reinterpret_cast<float*>(c);    c += (size_t)RPC * TC * 4;
    B.th = reinterpret_cast<uint32_t*>(c);
    return B;
  };

  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
  {
    const float* la32 = ws.lut32 + (int64_t)a * width;
    const float* lb32 = ws.lut32 + (int64_t)b * width;
    for (int i = tid; i < W; i += blockDim.x) {
      lut_a[i] = __ldg(la32 + i);
      lut_b[i] = __ldg(lb32 + i);
    }
    for (int i = tid; i < kBuckets + 2; i += blockDim.x) {
      first_a[i] = ws.first[a * (kBuckets + 2) + i];
      first_b[i] = ws.first[b * (kBuckets + 2) + i];
    }
  }
  if (tid < RPC) smin[tid] = ord_bits(__longlong_as_double(0x7ff0000000000000LL));
  if (tid < nruns) {
    const int r = ws.run_list[slot0 + s_live[tid]];
    hsrc[tid] = ws.ht16s + (int64_t)run_layer[r] * E * Tp;
    lsrc[tid] = ws.loadT + (int64_t)r * G * Tp;
    fsrc[tid] = reinterpret_cast<const float*>(ws.top3) + (int64_t)r * 4 * Tp;
  }
  for (int w = wid; w < nruns; w += nw) {
    const int r = ws.run_list[slot0 + s_live[w]];
    const int8_t* as = assign + (int64_t)r * E;
    int base_a = 0, base_b = 0;
    for (int e0 = 0; e0 < E; e0 += 32) {
      const int e = e0 + lane;
      const int g = e < E ? as[e] : -1;
      const unsigned ma = __ballot_sync(0xffffffffu, g == a), mb = __ballot_sync(0xffffffffu, g == b);
      const unsigned below = (1u << lane) - 1u;
      if (g == a) lists[(w * 2 + 0) * n + base_a + __popc(ma & below)] = (int16_t)e;
      if (g == b) lists[(w * 2 + 1) * n + base_b + __popc(mb & below)] = (int16_t)e;
      base_a += __popc(ma);
      base_b += __popc(mb);
    }
  }
  for (int k = 0; k < kSwap5Stages; ++k) {
    const Buf B = buf_at(k);
    for (int i = tid; i < RPC * hrows * RS; i += blockDim.x) B.h[i] = 0;
  }
  __syncthreads();

  const int pieces_h = 2 * n * V, pieces_l = 2 * V, pieces_f = 4 * VF;
  const int pieces_run = pieces_h + pieces_l + pieces_f;
  // this thread's 16-byte cp.async pieces of a chunk (source at t0 = 0, byte
  // offset in a staging buffer); a chunk at t0 adds t0 * element size
  constexpr int kMaxPieces = 4;
  const bool fixed_pieces = nruns * pieces_run <= kMaxPieces * (int)blockDim.x;
  const char* psrc[kMaxPieces];
  uint32_t pdst[kMaxPieces], pshift[kMaxPieces];
  int npieces = 0;
  auto piece = [&](int i, const char*& src, uint32_t& dst, uint32_t& sh) {
    const int ss = i / pieces_run;
    int q = i - ss * pieces_run;
    const Buf B0 = buf_at(0);
    const unsigned char* base0 = bufs;
    if (q < pieces_h) {
      const int row = q / V, v = q - row * V;  // rows [0, n): a experts; [n, 2n): b experts
      const int e = row < n ? lists[(ss * 2 + 0) * n + row] : lists[(ss * 2 + 1) * n + row - n];
      dst = (uint32_t)(reinterpret_cast<unsigned char*>(B0.h + ((size_t)ss * hrows + row) * RS + v * 8) - base0);
      src = reinterpret_cast<const char*>(hsrc[ss] + (int64_t)e * Tp + v * 8);
      sh = 1;
    } else if ((q -= pieces_h) < pieces_l) {
      const int which = q / V, v = q - which * V;
      dst = (uint32_t)(reinterpret_cast<unsigned char*>(B0.l + ((size_t)ss * 2 + which) * TC + v * 8) - base0);
      src = reinterpret_cast<const char*>(lsrc[ss] + (int64_t)(which ? b : a) * Tp + v * 8);
      sh = 1;
    } else {
      q -= pieces_l;
      const int g = q / VF, v = q - g * VF;
      dst = (uint32_t)(reinterpret_cast<unsigned char*>(B0.lat + ((size_t)ss * 4 + g) * TC + v * 4) - base0);
      src = reinterpret_cast<const char*>(fsrc[ss] + (int64_t)g * Tp + v * 4);
      sh = 2;
    }
  };
  if (fixed_pieces) {
#pragma unroll
    for (int j = 0; j < kMaxPieces; ++j) {
      const int i = tid + j * (int)blockDim.x;
      psrc[j] = nullptr;
      pdst[j] = 0;
      pshift[j] = 0;
      if (i < nruns * pieces_run) {
        piece(i, psrc[j], pdst[j], pshift[j]);
        npieces = j + 1;
      }
    }
  }
  auto issue = [&](int64_t t0, int k) {
    unsigned char* bk = bufs + k * buf_bytes;
    if (fixed_pieces) {
#pragma unroll
      for (int j = 0; j < kMaxPieces; ++j)
        if (j < npieces) cp_async16(bk + pdst[j], psrc[j] + (t0 << pshift[j]));
      return;
    }
    for (int i = tid; i < nruns * pieces_run; i += blockDim.x) {
      const char* src;
      uint32_t dst, sh;
      piece(i, src, dst, sh);
      cp_async16(bk + dst, src + (t0 << sh));
    }
  };

  const float bscale_a = ws.bscale[a], bscale_b = ws.bscale[b];
  const uint32_t base_a = (uint32_t)__cvta_generic_to_shared(lut_a);
  const uint32_t base_b = (uint32_t)__cvta_generic_to_shared(lut_b);
  const int units_total = nruns * geo.units_per_run;
  for (int pass0 = 0; pass0 < units_total; pass0 += blockDim.x) {
    const int u = pass0 + tid;
    const bool live = u < units_total;
    const int s = live ? u / geo.units_per_run : 0;
    const int ur = live ? u % geo.units_per_run : 0;
    const int x = ur / ng, yg = ur % ng;  // y experts of this thread: yg + q*ng
    double acc[Y];
#pragma unroll
    for (int q = 0; q < Y; ++q) acc[q] = 0.0;

    // kSwap5Stages-deep cp.async ring: chunks c+1 .. c+S-1 in flight while c is scanned
#pragma unroll
    for (int c = 0; c < kSwap5Stages - 1; ++c) {
      if (tb + (int64_t)c * TC < te) issue(tb + (int64_t)c * TC, c);
      cp_async_commit();
    }
    int k = 0;
    for (int64_t t0 = tb; t0 < te; t0 += TC, k = (k + 1 == kSwap5Stages) ? 0 : k + 1) {
      cp_async_wait_n<kSwap5Stages - 2>();  // chunk c has landed (c+1 .. may be in flight)
      __syncthreads();                      // ... for every thread; and chunk c-1 is scanned by all
      const int kn = (k + kSwap5Stages - 1) % kSwap5Stages;  // the slot freed by chunk c-1
      if (t0 + (kSwap5Stages - 1) * TC < te) issue(t0 + (kSwap5Stages - 1) * TC, kn);
      cp_async_commit();
      const Buf B = buf_at(k);
      // pother' and, per side, the clamp point: the largest n whose table
      // value (monotone rows) is <= pother'. Indices below it read the clamp
      // point instead -- a value <= pother', so every term is unchanged -- and
      // all such lanes of a warp hit one address (broadcast, no conflict).
      for (int rr = tid; rr < 2 * nruns * TC; rr += blockDim.x) {
        const int side = rr >= nruns * TC;
        const int r2 = side ? rr - nruns * TC : rr;
        const int ss = r2 / TC, tt = r2 % TC;
        const float* lat = B.lat + (size_t)ss * 4 * TC + tt;
        const uint32_t ix = __float_as_uint(lat[3 * TC]);
        const uint32_t j1 = ix & 0xffu, j2 = (ix >> 8) & 0xffu;
        // pother' = the first of the top-3 on neither a nor b (-inf when G == 2)
        const float m = (j1 != (uint32_t)a && j1 != (uint32_t)b) ? lat[0]
                        : ((j2 != (uint32_t)a && j2 != (uint32_t)b) ? lat[TC] : lat[2 * TC]);
        if (!side) B.po[ss * TC + tt] = m;
        const float* tab = side ? lut_b : lut_a;
        int lo = 0;
        if (monotone && tab[0] <= m) {
          // the clamp point lies in [first[q] - 1, first[q+1] - 1], q = bucket(m):
          // values in lower buckets are < m, values in higher buckets are > m
          const uint16_t* fb = side ? first_b : first_a;
          const float sc = side ? bscale_b : bscale_a;
          const int q = min(kBuckets, (int)(m * sc));
          lo = max((int)fb[q] - 1, 0);
          int hi = max((int)fb[q + 1] - 1, lo);
          while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (tab[mid] <= m) lo = mid; else hi = mid - 1;
          }
        }
        B.th[(ss * 2 + side) * TC + tt] = (side ? base_b : base_a) + 4u * (uint32_t)lo;
      }
      __syncthreads();
      if (live) {
        const float* pos = B.po + s * TC;
        const uint32_t* tha = B.th + s * 2 * TC;
        const uint32_t* thb = tha + TC;
        const uint16_t* las = B.l + (size_t)s * 2 * TC;
        const uint16_t* lbs = las + TC;
        const uint16_t* hAs = B.h + ((size_t)s * hrows + x) * RS;
        const uint16_t* hBs = B.h + ((size_t)s * hrows + n + yg) * RS;
        float c[Y];
#pragma unroll
        for (int q = 0; q < Y; ++q) c[q] = 0.0f;
#pragma unroll 2
        for (int tt = 0; tt < TC; tt += 4) {
          const uint2 hx2 = *reinterpret_cast<const uint2*>(hAs + tt);
          const uint2 la2 = *reinterpret_cast<const uint2*>(las + tt);
          const uint2 lb2 = *reinterpret_cast<const uint2*>(lbs + tt);
          const float4 p4 = *reinterpret_cast<const float4*>(pos + tt);
          const uint4 ta4 = *reinterpret_cast<const uint4*>(tha + tt);
          const uint4 tb4 = *reinterpret_cast<const uint4*>(thb + tt);
          const uint32_t taj[4] = {ta4.x, ta4.y, ta4.z, ta4.w}, tbj[4] = {tb4.x, tb4.y, tb4.z, tb4.w};
          uint2 hy2[Y];
#pragma unroll
          for (int q = 0; q < Y; ++q) hy2[q] = *reinterpret_cast<const uint2*>(hBs + (size_t)q * ng * RS + tt);
          const float pj[4] = {p4.x, p4.y, p4.z, p4.w};
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const uint32_t wx = (j < 2) ? hx2.x : hx2.y, wa = (j < 2) ? la2.x : la2.y, wb = (j < 2) ? lb2.x : lb2.y;
            const uint32_t hx = (j & 1) ? (wx >> 16) : (wx & 0xffffu);
            const uint32_t la = (j & 1) ? (wa >> 16) : (wa & 0xffffu);
            const uint32_t lb = (j & 1) ? (wb >> 16) : (wb & 0xffffu);
            const uint32_t ra = base_a + la * 4u - hx, rb = base_b + lb * 4u + hx;
#pragma unroll
            for (int q = 0; q < Y; ++q) {
              const uint32_t wy = (j < 2) ? hy2[q].x : hy2[q].y;
              const uint32_t hy = (j & 1) ? (wy >> 16) : (wy & 0xffffu);
              c[q] += fmaxf(fmaxf(pj[j], lds_f32(max(ra + hy, taj[j]))), lds_f32(max(rb - hy, tbj[j])));
            }
          }
        }
#pragma unroll
        for (int q = 0; q < Y; ++q) acc[q] = dadd(acc[q], (double)c[q]);
      }
    }
    if (split) {  // partial sums of this step range (fp64 adds in any order: within the screen's bound)
      if (live) {
        const int r = ws.run_list[slot0 + s_live[s]];
        double* pa = ws.split_acc + (((int64_t)r * NP + blockIdx.x) * n + x) * n;
#pragma unroll
        for (int q = 0; q < Y; ++q)
          if (yg + q * ng < n) atomicAdd(pa + yg + q * ng, acc[q]);
      }
      continue;
    }
    if (live) {
      double mn = acc[0];
#pragma unroll
      for (int q = 1; q < Y; ++q)
        if (yg + q * ng < n) mn = fmin(mn, acc[q]);
      atomicMin(&smin[s], ord_bits(mn));
    }
    __syncthreads();
    if (live) {
      const int r = ws.run_list[slot0 + s_live[s]];
      const int64_t tile = (int64_t)r * NP + blockIdx.x;
      const double lim = __longlong_as_double((long long)smin[s]) * kWindow5;
      const int xe = lists[(s * 2 + 0) * n + x];
#pragma unroll
      for (int q = 0; q < Y; ++q) {
        const int yi = yg + q * ng;
        if (yi >= n || !(acc[q] <= lim)) continue;
        const int ye = lists[(s * 2 + 1) * n + yi];
        const int f = xe < ye ? xe * E + ye : ye * E + xe;
        const int kk = atomicAdd(&ws.loc_cnt[tile], 1);
        if (kk < kLocK) {
          ws.loc_cand[tile * kLocK + kk] = acc[q];
          ws.loc_flat[tile * kLocK + kk] = f;
        }
      }
    }
  }
  if (split) return;
  __syncthreads();
  if (tid < nruns) {
    const int r = ws.run_list[slot0 + s_live[tid]];
    ws.loc_min[(int64_t)r * NP + blockIdx.x] = __longlong_as_double((long long)smin[tid]);
  }
}

// split scans: per (GPU-pair tile, active run) the tile minimum of the summed
// partial scores and the pairs inside the tile's window (as approx_scan5 does)
__global__ void split_window_kernel(int E, int G, const int8_t* __restrict__ assign, int32_t n_active,
                                    SearchWs ws) {
  __shared__ unsigned long long s_min;
  __shared__ int16_t s_list[2][2048 / 2];
  const int slot = blockIdx.y;
  if (slot >= n_active) return;
  const int r = ws.run_list[slot];
  const int NP = G * (G - 1) / 2, n = E / G;
  int p = blockIdx.x, a = 0;
  while (p >= G - 1 - a) { p -= G - 1 - a; ++a; }
  const int b = a + 1 + p;
  const int64_t tile = (int64_t)r * NP + blockIdx.x;
  const double* pa = ws.split_acc + tile * n * n;
  const int tid = threadIdx.x, lane = tid & 31;
  if (tid == 0) s_min = ord_bits(__longlong_as_double(0x7ff0000000000000LL));
  if (tid < 32) {  // ascending expert lists of GPUs a and b
    const int8_t* as = assign + (int64_t)r * E;
    int ba = 0, bb = 0;
    for (int e0 = 0; e0 < E; e0 += 32) {
      const int e = e0 + lane;
      const int g = e < E ? as[e] : -1;
      const unsigned ma = __ballot_sync(0xffffffffu, g == a), mb = __ballot_sync(0xffffffffu, g == b);
      const unsigned below = (1u << lane) - 1u;
      if (g == a) s_list[0][ba + __popc(ma & below)] = (int16_t)e;
      if (g == b) s_list[1][bb + __popc(mb & below)] = (int16_t)e;
      ba += __popc(ma);
      bb += __popc(mb);
    }
  }
  __syncthreads();
  for (int k = tid; k < n * n; k += blockDim.x) atomicMin(&s_min, ord_bits(pa[k]));
  __syncthreads();
  const double mn = __longlong_as_double((long long)s_min);
  const double lim = mn * kWindow5;
  for (int k = tid; k < n * n; k += blockDim.x) {
    const double v = pa[k];
    if (!(v <= lim)) continue;
    const int xe = s_list[0][k / n], ye = s_list[1][k % n];
    const int kk = atomicAdd(&ws.loc_cnt[tile], 1);
    if (kk < kLocK) {
      ws.loc_cand[tile * kLocK + kk] = v;
      ws.loc_flat[tile * kLocK + kk] = xe < ye ? xe * E + ye : ye * E + xe;
    }
  }
  if (tid == 0) ws.loc_min[tile] = mn;
}

// per active run: the run's window over all GPU-pair tiles -> exact-candidate list.
// thr >= 0 (the search's convergence threshold; the refinement only needs the
// winner when it is accepted, search.py:222-227): the acceptance test is
// monotone in the candidate score, so with bounds lo <= exact min <= hi from
// the approximate minimum (|cand' - cand| < 2^-18.9 cand) a run whose lo is
// rejected stops without exact scores, and a run with ONE pair in its window
// (necessarily the exact winner) whose hi is accepted swaps without one (the
// apply kernel's full re-score is the exact candidate, search.py:236).
__global__ void window_kernel(int32_t n_active, int G, double window, double thr, SearchWs ws) {
  const int NP = G * (G - 1) / 2;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n_active; i += gridDim.x * blockDim.x) {
    const int r = ws.run_list[i];
    double gmin = __longlong_as_double(0x7ff0000000000000LL);
    for (int p = 0; p < NP; ++p) gmin = fmin(gmin, ws.loc_min[(int64_t)r * NP + p]);
    const double lim = gmin * window;
    int cnt = 0, overflow = 0;
    for (int p = 0; p < NP; ++p) {
      const int64_t tile = (int64_t)r * NP + p;
      if (!(ws.loc_min[tile] <= lim)) continue;
      const int c = ws.loc_cnt[tile];
      if (c > kLocK) { overflow = 1; continue; }
      for (int k = 0; k < c; ++k) {
        if (!(ws.loc_cand[tile * kLocK + k] <= lim)) continue;
        if (cnt < kCandK) ws.cand_flat[(int64_t)r * kCandK + cnt] = ws.loc_flat[tile * kLocK + k];
        ++cnt;
      }
    }
    if (cnt > kCandK) overflow = 1;
    ws.cand_n[r] = overflow ? 0 : cnt;
    int32_t mode = overflow ? kNeedExact : 0;
    if (thr >= 0.0) {
      const double s = ws.run_score[r];
      const double lo = gmin * (1.0 - 0x1p-17), hi = gmin * (1.0 + 0x1p-17);
      if (!(lo < s) || __dsub_rn(1.0, __ddiv_rn(lo, s)) < thr) mode = kPreReject;
      else if (!overflow && cnt == 1 && hi < s && !(__dsub_rn(1.0, __ddiv_rn(hi, s)) < thr)) mode = kPreAccept;
    }
    ws.need_exact[r] = mode;
  }
}

// exact candidate score of one (run, expert pair) per CTA iteration (grid-
// strided over the n_active x kCandK slots): warps 1.. evaluate v1's terms,
// thread 0 extends the serial fp64 chain in t order (block_chain)
// exact candidate score of one (run, expert pair) per warp (many active runs):
// lanes fill 256 terms per chunk, lane 0 extends the serial fp64 chain from
// shared memory
__global__ void exact_pairs_warp_kernel(const int32_t* __restrict__ hist, int64_t T, int E, int G,
                                        const double* __restrict__ lut, int64_t nmax,
                                        const int32_t* __restrict__ run_layer, const int8_t* __restrict__ assign,
                                        int32_t n_active, SearchWs ws) {
  const int warp_global = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int slot = warp_global / kCandK, k = warp_global % kCandK;
  if (slot >= n_active) return;
  const int r = ws.run_list[slot];
  if (ws.need_exact[r] || k >= ws.cand_n[r]) return;
  const int f = ws.cand_flat[(int64_t)r * kCandK + k];
  const int i = f / E, j = f % E;
  const int a = assign[(int64_t)r * E + i], b = assign[(int64_t)r * E + j];
  const int64_t width = nmax + 1;
  const int32_t* h = hist + (int64_t)run_layer[r] * T * E;
  const int32_t* ld = ws.loads + (int64_t)r * T * G;
  __shared__ double xbuf[8][256];  // blockDim.x == 256: one row per warp
  double* xb = xbuf[(threadIdx.x >> 5) & 7];
  double sum = 0.0;
  for (int64_t t0 = 0; t0 < T; t0 += 256) {
    const int tn = (int)imin64(256, T - t0);
#pragma unroll 2
    for (int q = lane; q < tn; q += 32) {
      const int64_t t = t0 + q;
      const int32_t* lrow = ld + t * G;
      const int32_t hi = h[t * E + i], hj = h[t * E + j], la = lrow[a], lb = lrow[b];
      const double va = __ldg(lut + a * width + (la - hi + hj));
      const double vb = __ldg(lut + b * width + (lb - hj + hi));
      double m = max_lat_excl(lrow, G, lut, width, a, b);
      m = va > m ? va : m;
      m = vb > m ? vb : m;
      xb[q] = m;
    }
    __syncwarp();
    if (lane == 0)
      for (int q = 0; q < tn; ++q) sum = dadd(sum, xb[q]);
    __syncwarp();
  }
  if (lane == 0) ws.cand_exact[(int64_t)r * kCandK + k] = sum;
}

constexpr int kPairThreads = 128;  // exact_pairs: three producer warps + the chain thread's warp
constexpr int kPairChunk = 512;
#ifndef GEM_PAIR_CTA_RUNS
#define GEM_PAIR_CTA_RUNS 320
#endif
constexpr int kPairCtaRuns = GEM_PAIR_CTA_RUNS;  // exact_pairs: CTA per pair at <= this many active runs
__global__ void __launch_bounds__(kPairThreads)
exact_pairs_kernel(const int32_t* __restrict__ hist, int64_t T, int E, int G, const double* __restrict__ lut,
                   int64_t nmax, const int32_t* __restrict__ run_layer, const int8_t* __restrict__ assign,
                   int32_t n_active, SearchWs ws) {
  __shared__ double buf[2 * kPairChunk];
  const int64_t width = nmax + 1;
  for (int64_t idx = blockIdx.x; idx < (int64_t)n_active * kCandK; idx += gridDim.x) {
    const int slot = (int)(idx / kCandK), k = (int)(idx % kCandK);
    const int r = ws.run_list[slot];
    if (ws.need_exact[r] || k >= ws.cand_n[r]) continue;  // uniform over the CTA
    const int f = ws.cand_flat[(int64_t)r * kCandK + k];
    const int i = f / E, j = f % E;
    const int a = assign[(int64_t)r * E + i], b = assign[(int64_t)r * E + j];
    const int32_t* h = hist + (int64_t)run_layer[r] * T * E;
    const int32_t* ld = ws.loads + (int64_t)r * T * G;
    const double sum = block_chain<kPairChunk>(T, buf, [&](int64_t t) {
      const int32_t* lrow = ld + t * G;
      const int32_t hi = h[t * E + i], hj = h[t * E + j], la = lrow[a], lb = lrow[b];
      const double va = __ldg(lut + a * width + (la - hi + hj));
      const double vb = __ldg(lut + b * width + (lb - hj + hi));
      double m = max_lat_excl(lrow, G, lut, width, a, b);
      m = va > m ? va : m;
      m = vb > m ? vb : m;
      return m;
    });
    if (threadIdx.x == 0) ws.cand_exact[(int64_t)r * kCandK + k] = sum;
    __syncthreads();  // buf is reused by the next slot
  }
}

// per active run without overflow: lexicographic (exact cand, flat) minimum
__global__ void select_pairs_kernel(int32_t n_active, int E, SearchWs ws) {
  for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < n_active; s += gridDim.x * blockDim.x) {
    const int r = ws.run_list[s];
    const int32_t mode = ws.need_exact[r];
    if (mode == kNeedExact) continue;
    if (mode == kPreAccept || mode == kPreReject) {
      const int f = ws.cand_flat[(int64_t)r * kCandK];
      ws.run_found[r] = mode == kPreAccept;
      ws.run_i[r] = mode == kPreAccept ? f / E : -1;
      ws.run_j[r] = mode == kPreAccept ? f % E : -1;
      ws.run_cand[r] = __longlong_as_double(0x7ff8000000000000LL);  // exact value: the apply's re-score
      continue;
    }
    double bc = __longlong_as_double(0x7ff0000000000000LL);
    int bf = 0x7fffffff;
    for (int k = 0; k < ws.cand_n[r]; ++k) {
      const double c = ws.cand_exact[(int64_t)r * kCandK + k];
      const int f = ws.cand_flat[(int64_t)r * kCandK + k];
      if (c < bc || (c == bc && f < bf)) { bc = c; bf = f; }
    }
    const bool found = bf != 0x7fffffff;
    ws.run_found[r] = found;
    ws.run_i[r] = found ? bf / E : -1;
    ws.run_j[r] = found ? bf % E : -1;
    ws.run_cand[r] = bc;
  }
}

// transposed per-run state for the screened scan: loadT[r][g][t], latT[r][g][t]
// (zero past T)
__global__ void state_t_kernel(int64_t R, int64_t T, int G, int64_t width, SearchWs ws) {
  const int64_t Tp = ws.Tp;
  const int64_t n = R * G * Tp;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = i % Tp, rg = i / Tp;
    const int g = (int)(rg % G);
    const int64_t r = rg / G;
    int32_t l = 0;
    float v = 0.0f;
    if (t < T) {
      l = ws.loads[(r * T + t) * G + g];
      v = ws.lut32[(int64_t)g * width + l];
    }
    ws.loadT[i] = (uint16_t)l;
    ws.latT[i] = v;
  }
}

// clamp-point search hints (K6 v5): bscale[g] = kBuckets / (largest value of
// row g inside the window), bucket(v) = min(kBuckets, (int)(v * bscale[g]))
__global__ void bucket_scale_kernel(const float* __restrict__ lut32, int G, int64_t width, int W,
                                    float* __restrict__ bscale) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= G) return;
  const float vmax = lut32[(int64_t)g * width + W - 1];
  bscale[g] = vmax > 0.0f ? (float)kBuckets / vmax : 0.0f;
}

// first[g][b] = smallest n in [0, W) with bucket(lut32[g][n]) >= b (W if none),
// b in [0, kBuckets + 1]; rows are nondecreasing, so n writes the buckets in
// (bucket(n-1), bucket(n)] and the last n also those above its bucket
__global__ void bucket_first_kernel(const float* __restrict__ lut32, int G, int64_t width, int W,
                                    const float* __restrict__ bscale, uint16_t* __restrict__ first) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < (int64_t)G * W;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int g = (int)(i / W), nn = (int)(i - (int64_t)g * W);
    const float sc = bscale[g];
    auto bk = [&](int n) { return min(kBuckets, (int)(lut32[(int64_t)g * width + n] * sc)); };
    const int lo = nn == 0 ? -1 : bk(nn - 1), hi = bk(nn);
    uint16_t* f = first + (int64_t)g * (kBuckets + 2);
    for (int b = lo + 1; b <= hi; ++b) f[b] = (uint16_t)nn;
    if (nn == W - 1)
      for (int b = hi + 1; b <= kBuckets + 1; ++b) f[b] = (uint16_t)W;
  }
}

// flag[0] = 1 when some fp32 table row decreases somewhere
// flag bit 0: some fp32 row decreases; bit 1: some fp64 row decreases
__global__ void lut_monotone_kernel(const float* __restrict__ lut32, const double* __restrict__ lut, int G,
                                    int64_t width, int32_t* __restrict__ flag) {
  const int64_t n = (int64_t)G * width;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = i % width;
    if (k + 1 < width && !(lut32[i] <= lut32[i + 1])) atomicOr(flag, 1);
    if (k + 1 < width && !(lut[i] <= lut[i + 1])) atomicOr(flag, 2);
  }
}

// per active run and step: the three largest fp32 latencies and their GPUs
// (-inf / 255 past G). pother of a GPU pair (a, b) is the first of them on
// neither a nor b, so a scan tile stages 4 rows instead of G.
__global__ void top3_kernel(int32_t n_active, int64_t Tp, int G, SearchWs ws) {
  const int64_t total = (int64_t)n_active * Tp;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = i % Tp;
    const int r = ws.run_list[i / Tp];
    const float* lat = ws.latT + (int64_t)r * G * Tp + t;
    float v1 = __int_as_float(0xff800000), v2 = v1, v3 = v1;
    uint32_t i1 = 255, i2 = 255, i3 = 255;
    for (int g = 0; g < G; ++g) {
      const float v = lat[(int64_t)g * Tp];
      if (v > v1) { v3 = v2; i3 = i2; v2 = v1; i2 = i1; v1 = v; i1 = g; }
      else if (v > v2) { v3 = v2; i3 = i2; v2 = v; i2 = g; }
      else if (v > v3) { v3 = v; i3 = g; }
    }
    uint32_t* out = ws.top3 + (int64_t)r * 4 * Tp + t;
    out[0] = __float_as_uint(v1);
    out[Tp] = __float_as_uint(v2);
    out[2 * Tp] = __float_as_uint(v3);
    out[3 * Tp] = i1 | (i2 << 8) | (i3 << 16);
  }
}

// fp64 latency table -> its fp32 rounding (round to nearest: monotone)
// Search-only tile pruning (K6). For a swap on GPUs (a, b) every step's term
// is max(pother_ab, C_a, C_b) >= pother_ab = the maximum over the OTHER GPUs,
// so every pair of the tile scores at least LB_ab = sum_t pother_ab(t) (the
// serial fp64 sum is monotone in its terms). With M, m2, m3 the step's three
// largest latencies and g1, g2 the GPUs of the first two:
//   sum_t (M - pother_ab) = X_a + X_b + Y_ab,
//   X_g = sum_{t: g1 = g} (M - m2),  Y_ab = sum_{t: {g1,g2} = {a,b}} (m2 - m3).
// If LB_ab already fails the acceptance test (search.py:222-227), no pair of
// the tile can be accepted: the run either takes a pair of another tile (the
// exact minimum cannot be in this one) or stops -- the same outcome, so the
// scan skips the tile. Sums from the fp32 top-3 in any order; the margin
// 2^-21 * score covers their rounding (<= 2^-23 score) and every summation
// error. One CTA per active run; prune[slot][p] = 1 for skipped tiles.
__global__ void tile_bound_kernel(int32_t n_active, int64_t Tp, int G, double thr, SearchWs ws,
                                  uint8_t* __restrict__ prune) {
  __shared__ double X[32], Y[32 * 32];
  const int slot = blockIdx.x;
  if (slot >= n_active) return;
  const int r = ws.run_list[slot];
  for (int i = threadIdx.x; i < 32; i += blockDim.x) X[i] = 0.0;
  for (int i = threadIdx.x; i < 32 * 32; i += blockDim.x) Y[i] = 0.0;
  __syncthreads();
  const uint32_t* tb = ws.top3 + (int64_t)r * 4 * Tp;
  for (int64_t t = threadIdx.x; t < Tp; t += blockDim.x) {
    const float v1 = __uint_as_float(tb[t]), v2 = __uint_as_float(tb[Tp + t]), v3 = __uint_as_float(tb[2 * Tp + t]);
    const uint32_t pk = tb[3 * Tp + t];
    const uint32_t g1 = pk & 255u, g2 = (pk >> 8) & 255u;
    if (g1 < 32u && v1 > v2) atomicAdd(&X[g1], (double)v1 - (double)v2);
    if (g1 < 32u && g2 < 32u && v2 > v3) atomicAdd(&Y[min(g1, g2) * 32 + max(g1, g2)], (double)v2 - (double)v3);
  }
  __syncthreads();
  const double score = ws.run_score[r];
  const int NP = G * (G - 1) / 2;
  for (int p = threadIdx.x; p < NP; p += blockDim.x) {
    int q = p, a = 0;
    while (q >= G - 1 - a) { q -= G - 1 - a; ++a; }
    const int b = a + 1 + q;
    const double lb = score - (X[a] + X[b] + Y[a * 32 + b]) - score * 0x1p-21;
    const bool reject = !(lb < score) || __dsub_rn(1.0, __ddiv_rn(lb, score)) < thr;
    prune[(int64_t)slot * NP + p] = (G >= 3 && reject) ? 1 : 0;  // G = 2: no other GPU bounds the pair
  }
}

__global__ void lut_to_f32_kernel(const double* __restrict__ lut, int64_t n, float* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = __double2float_rn(lut[i]);
}

// compact the indices of active runs (order is irrelevant: runs are independent)
__global__ void compact_runs_kernel(int64_t R, SearchWs ws) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < R; r += (int64_t)gridDim.x * blockDim.x)
    if (ws.run_active[r]) ws.run_list[atomicAdd(&ws.counters[3], 1)] = (int32_t)r;
}

__global__ void reduce_pairs_kernel(int64_t R, int G, int E, SearchWs ws, const int32_t* __restrict__ filter) {
  const int NP = G * (G - 1) / 2;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < R; r += (int64_t)gridDim.x * blockDim.x) {
    if (!ws.run_active[r] || (filter && filter[r] != kNeedExact)) continue;
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
  __shared__ double buf[2 * kScoreChunk];
  __shared__ int s_go;
  const int64_t r = blockIdx.x;
  if (!ws.run_active[r]) return;
  if (threadIdx.x == 0) {
    const double score = ws.run_score[r], cand = ws.run_cand[r];
    int go = ws.run_found[r] && (cand < score);
    // convergence is judged on the best candidate before applying it (search.py:224-227)
    if (go && __dsub_rn(1.0, __ddiv_rn(cand, score)) < threshold) go = 0;
    if (ws.need_exact[r] == kPreAccept) go = 1;  // accepted by the window bound (window_kernel)
    s_go = go;
    if (!go) ws.run_active[r] = 0;
  }
  __syncthreads();
  if (!s_go) return;
  const int i = ws.run_i[r], j = ws.run_j[r];
  const int a = assign[r * E + i], b = assign[r * E + j];
  const int32_t* h = hist + (int64_t)run_layer[r] * T * E;
  int32_t* ld = ws.loads + r * T * G;
  const bool screened = ws.ht16 != nullptr;
  const int64_t width = nmax + 1;
  const int64_t Tp = ws.Tp;
#pragma unroll 4
  for (int64_t t = threadIdx.x; t < T; t += blockDim.x) {
    const int32_t d = h[t * E + j] - h[t * E + i];
    const int32_t na = ld[t * G + a] + d, nb = ld[t * G + b] - d;
    ld[t * G + a] = na;
    ld[t * G + b] = nb;
    if (screened) {
      ws.loadT[(r * G + a) * Tp + t] = (uint16_t)na;
      ws.loadT[(r * G + b) * Tp + t] = (uint16_t)nb;
      ws.latT[(r * G + a) * Tp + t] = ws.lut32[a * width + na];
      ws.latT[(r * G + b) * Tp + t] = ws.lut32[b * width + nb];
    }
  }
  __syncthreads();
  const double s = block_score(ld, T, G, lut, nmax + 1, buf);
  if (threadIdx.x == 0) {
    assign[r * E + i] = (int8_t)b;
    assign[r * E + j] = (int8_t)a;
    if (ws.need_exact[r] != kPreAccept && s != ws.run_cand[r]) atomicExch(&ws.counters[1], 1);  // search.py:236
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

// restart orders: one CTA per run; expert e goes to position
// #{e' : key[e'] > key[e]} + #{e' < e : key[e'] == key[e]} (a stable sort by
// descending key; -0.0 == 0.0 as in numpy's comparison)
__global__ void restart_order_kernel(const double* __restrict__ keys, int E, int16_t* __restrict__ order) {
  extern __shared__ double s_key[];
  const int64_t r = blockIdx.x;
  for (int e = threadIdx.x; e < E; e += blockDim.x) s_key[e] = keys[r * E + e];
  __syncthreads();
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    const double v = s_key[e];
    int pos = 0;
    for (int q = 0; q < E; ++q) {
      const double w = s_key[q];
      pos += (w > v) || (w == v && q < e);
    }
    order[r * E + pos] = (int16_t)e;
  }
}

extern "C" int gem_restart_order(const double* keys, int64_t R, int32_t E, int16_t* order, void* stream) {
  GEM_REQUIRE(keys && order && R >= 1 && E >= 1 && E <= 6144, "gem_restart_order: bad arguments (E <= 6144)");
  restart_order_kernel<<<(unsigned)R, 128, (size_t)E * sizeof(double), as_stream(stream)>>>(keys, E, order);
  GEM_CHECK_LAUNCH("restart_order_kernel");
  return GEM_OK;
}

extern "C" size_t gem_search_workspace_bytes(int64_t R, int64_t T, int32_t E, int32_t G) {
  return carve(nullptr, nullptr, R, T, E, G);
}

static int check_search_args(const int32_t* hist, int64_t L, int64_t T, int32_t E, int32_t G, const double* lut,
                             int64_t nmax, int64_t R, const int32_t* run_layer, size_t ws_bytes, void* workspace) {
  GEM_REQUIRE(hist && lut && run_layer && workspace && L >= 1 && T >= 1 && E >= 1 && G >= 1 && R >= 1,
              "gem_search: bad arguments");
  GEM_REQUIRE(G <= kMaxGpus && E <= 32767, "gem_search: G <= %d required (got G=%d)", kMaxGpus, G);
  GEM_REQUIRE(E % G == 0, "gem_search: %d experts cannot be split evenly across %d GPUs", E, G);
  GEM_REQUIRE(E <= 2048, "gem_search: E <= 2048 required");
  GEM_REQUIRE(nmax >= 0 && nmax < (1LL << 31), "gem_search: nmax out of range");
  GEM_REQUIRE(ws_bytes >= gem_search_workspace_bytes(R, T, E, G), "gem_search: workspace too small");
  GEM_REQUIRE(R <= (1LL << 31) - 1, "gem_search: too many runs");
  return GEM_OK;
}

// n_listed > 0: only the n_listed runs of ws.run_list (the active ones) are candidates
static int launch_exact_scan(const int32_t* hist, int64_t T, int32_t E, int32_t G, const double* lut, int64_t nmax,
                             int64_t R, const int32_t* run_layer, const int8_t* assign, const SearchWs& ws,
                             const int32_t* filter, cudaStream_t st, int64_t n_listed = 0) {
  const size_t smem = swap_smem(E);
  GEM_CHECK_CUDA(cudaFuncSetAttribute(best_swap_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  dim3 grid((unsigned)(n_listed > 0 ? n_listed : R), (unsigned)(G * (G - 1) / 2));
  best_swap_kernel<<<grid, kSearchThreads, smem, st>>>(hist, T, E, G, lut, nmax, run_layer, assign, ws, filter,
                                                       n_listed > 0 ? ws.run_list : nullptr);
  GEM_CHECK_LAUNCH("best_swap_kernel");
  reduce_pairs_kernel<<<(unsigned)((R + 255) / 256), 256, 0, st>>>(R, G, E, ws, filter);
  GEM_CHECK_LAUNCH("reduce_pairs_kernel");
  return GEM_OK;
}

// One best-swap scan over the active runs: screened (v3) when the two fp32
// table rows fit shared memory, else the exact v1 scan for every active run.
// thr >= 0: the search's convergence threshold (window-bound accept / reject,
// see window_kernel); < 0: every active run gets its exact best pair
static int launch_scan(const int32_t* hist, int64_t T, int32_t E, int32_t G, const double* lut, int64_t nmax,
                       int64_t R, int64_t n_active, const int32_t* run_layer, const int8_t* assign,
                       const SearchWs& ws, cudaStream_t st, double thr = -1.0) {
  const int NP = G * (G - 1) / 2;
  if (NP == 0 || n_active <= 0) return GEM_OK;
  const size_t smem3 = swap3_smem(E, G, nmax);
  int dev = 0, optin = 0;
  GEM_CHECK_CUDA(cudaGetDevice(&dev));
  GEM_CHECK_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  // v5 needs only the two tables of its GPU pair in shared memory (v4 stages
  // every GPU's latencies: too large at G = 32)
  const int W5 = ws.win > 0 ? ws.win : (int)(nmax + 1);
  const int y5 = E / G <= 8 ? 2 : kSwapY;
  const size_t smem5 = swap5_smem(E, G, W5, y5);
  const bool v5 = ws.ht16s != nullptr && ws.first != nullptr && smem5 <= (size_t)optin && !std::getenv("GEM_SCAN_V4");
  if (ws.lut32 == nullptr || ws.ht16 == nullptr || (!v5 && smem3 > (size_t)optin)) {
    return launch_exact_scan(hist, T, E, G, lut, nmax, R, run_layer, assign, ws, nullptr, st);
  }
  GEM_CHECK_CUDA(cudaMemsetAsync(ws.counters + 3, 0, 4, st));
  compact_runs_kernel<<<(unsigned)((R + 255) / 256), 256, 0, st>>>(R, ws);
  GEM_CHECK_LAUNCH("compact_runs_kernel");
  GEM_CHECK_CUDA(cudaMemsetAsync(ws.loc_cnt, 0, (size_t)R * NP * 4, st));
  const Swap3Geom g = swap3_geom(E, G, v5 ? y5 : kSwapY);
  dim3 grid((unsigned)NP, (unsigned)((n_active + g.rpc - 1) / g.rpc));
  double window = kWindow;
  if (v5) {
    top3_kernel<<<(unsigned)imin64((n_active * ws.Tp + 255) / 256, 16 * num_sms()), 256, 0, st>>>(
        (int32_t)n_active, ws.Tp, G, ws);
    GEM_CHECK_LAUNCH("top3_kernel");
    const int clamp = ws.lut_monotone && !std::getenv("GEM_SCAN_NOCLAMP");
    // few active runs (the late refinement rounds): split every run-scan's
    // steps over several CTAs so the grid still fills two CTAs per SM
    const int64_t ctas = (int64_t)grid.x * grid.y;
    int64_t tseg = 0;
    const int n = E / G;
    if (ctas < 2 * (int64_t)num_sms() && E / G * (E / G) <= 2048 && !std::getenv("GEM_SCAN_NOSPLIT")) {
      const int64_t want = (2 * (int64_t)num_sms() + ctas - 1) / ctas;
      const int64_t minseg = 16 * (int64_t)kSwap5TChunk;  // >= 16 chunks per segment
      const int64_t nseg = imin64(want, ws.Tp / minseg);
      if (nseg > 1) tseg = ((ws.Tp + nseg - 1) / nseg + kSwap5TChunk - 1) / kSwap5TChunk * kSwap5TChunk;
    }
    dim3 g5 = grid;
    if (tseg > 0) {
      g5.z = (unsigned)((ws.Tp + tseg - 1) / tseg);
      GEM_CHECK_CUDA(cudaMemsetAsync(ws.split_acc, 0, (size_t)R * NP * n * n * 8, st));
    }
    // search mode (thr >= 0), unsplit scans: skip the tiles whose pother bound rejects every pair
    uint8_t* prune = nullptr;
    // (G >= 16: with few GPUs every pair touches a step maximum often enough that no tile is
    // provably rejected -- none at the Qwen3-235B shape -- and the bound pass only costs)
    if (thr >= 0.0 && tseg == 0 && G >= 16 && G <= 32 && !std::getenv("GEM_SCAN_NOPRUNE")) {
      GEM_CHECK_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&prune), (size_t)n_active * NP, st));
      tile_bound_kernel<<<(unsigned)n_active, 256, 0, st>>>((int32_t)n_active, ws.Tp, G, thr, ws, prune);
      GEM_CHECK_LAUNCH("tile_bound_kernel");
    }
    struct FreePrune {
      uint8_t* p;
      cudaStream_t s;
      ~FreePrune() {
        if (p) cudaFreeAsync(p, s);
      }
    } free_prune{prune, st};
    auto go5 = [&](auto kern) -> int {
      GEM_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem5));
      kern<<<g5, kSwap3Threads, smem5, st>>>(E, G, nmax, W5, clamp, run_layer, assign, (int32_t)n_active, ws, tseg,
                                             prune);
      GEM_CHECK_LAUNCH("approx_scan5_kernel");
      if (tseg > 0) {
        split_window_kernel<<<dim3((unsigned)NP, (unsigned)n_active), 256, 0, st>>>(E, G, assign, (int32_t)n_active,
                                                                                   ws);
        GEM_CHECK_LAUNCH("split_window_kernel");
      }
      return GEM_OK;
    };
    const int rc5 =
        y5 == 2 ? (G == 8 ? go5(approx_scan5_kernel<8, 2>) : (G == 4 ? go5(approx_scan5_kernel<4, 2>)
                                                                      : go5(approx_scan5_kernel<0, 2>)))
                : (G == 8 ? go5(approx_scan5_kernel<8, kSwapY>) : (G == 4 ? go5(approx_scan5_kernel<4, kSwapY>)
                                                                           : go5(approx_scan5_kernel<0, kSwapY>)));
    if (rc5) return rc5;
    window = kWindow5;
  } else {
    GEM_CHECK_CUDA(cudaFuncSetAttribute(approx_scan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem3));
    approx_scan_kernel<<<grid, kSwap3Threads, smem3, st>>>(T, E, G, nmax, run_layer, assign, (int32_t)n_active, ws);
    GEM_CHECK_LAUNCH("approx_scan_kernel");
  }
  window_kernel<<<(unsigned)((n_active + 127) / 128), 128, 0, st>>>((int32_t)n_active, G, window, thr, ws);
  GEM_CHECK_LAUNCH("window_kernel");
  const int64_t slots = n_active * kCandK;
  if (n_active > kPairCtaRuns)  // many runs: a warp per pair keeps more chains in flight
    exact_pairs_warp_kernel<<<(unsigned)((slots * 32 + 255) / 256), 256, 0, st>>>(
        hist, T, E, G, lut, nmax, run_layer, assign, (int32_t)n_active, ws);
  else  // few runs: a CTA per pair, its chain fed by three producer warps
    exact_pairs_kernel<<<(unsigned)imin64(slots, 16 * num_sms()), kPairThreads, 0, st>>>(
        hist, T, E, G, lut, nmax, run_layer, assign, (int32_t)n_active, ws);
  GEM_CHECK_LAUNCH("exact_pairs_kernel");
  select_pairs_kernel<<<(unsigned)((n_active + 127) / 128), 128, 0, st>>>((int32_t)n_active, E, ws);
  GEM_CHECK_LAUNCH("select_pairs_kernel");
  // runs whose window overflowed: the exact scan (CTAs of other active runs exit at once)
  return launch_exact_scan(hist, T, E, G, lut, nmax, R, run_layer, assign, ws, ws.need_exact, st, n_active);
}

static int launch_greedy(const int32_t* hist, int64_t T, int32_t E, int32_t G, const double* lut, int64_t nmax,
                         int64_t U, int64_t R, const int32_t* run_layer, const uint8_t* needs_greedy,
                         const int16_t* order, int8_t* assign, const SearchWs& ws, cudaStream_t st) {
  int dev = 0, optin = 0;
  GEM_CHECK_CUDA(cudaGetDevice(&dev));
  GEM_CHECK_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  if (ws.ht16 && G <= 32) {
    const int W = (int)imin64(U, nmax) + 1;
    const int GM = G <= 8 ? 8 : (G <= 16 ? 16 : 32);
    const size_t rest = (size_t)(g2_threads(GM) / 32) * GM * 8 + (size_t)GM * kGreedyTChunk * 8;
    size_t smem = (((size_t)G * W * 4 + 15) & ~size_t(15)) + rest;
    const bool sl = smem <= (size_t)optin;  // else the table stays in global memory (L1/L2 gathers)
    if (!sl) smem = rest;
    if (smem <= (size_t)optin) {
      uint16_t* l16 = nullptr;  // uint16 per-run loads, stream-ordered scratch
      GEM_CHECK_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&l16), (size_t)R * T * GM * 2, st));
      // per-step exact top-2 state (monotone fp64 rows only; GEM_GREEDY_NOTOP2=1 disables it)
      // (only for the off-chip table: with the table in shared memory the 8
      // re-gathers per step are cheaper than the state traffic, 74 vs 102 ms at C4)
      const bool top2 = ws.lut_monotone64 && !sl && G <= 255 && !std::getenv("GEM_GREEDY_NOTOP2");
      float2* tp = nullptr;
      double2* td = nullptr;
      uint8_t* ta = nullptr;
      if (top2) {
        GEM_CHECK_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&tp), (size_t)R * T * sizeof(float2), st));
        GEM_CHECK_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&td), (size_t)R * T * sizeof(double2), st));
        GEM_CHECK_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&ta), (size_t)R * T, st));
      }
      // off-chip table: piecewise rows in shared memory when they reproduce it (GEM_GREEDY_NOPW=1 disables)
      float2* pw = nullptr;
      int32_t* pw_bad = nullptr;
      const size_t pw_bytes = (size_t)G * pw_buckets(W) * sizeof(float2);
      if (!sl && !std::getenv("GEM_GREEDY_NOPW") && smem + pw_bytes <= (size_t)optin) {
        GEM_CHECK_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&pw), pw_bytes + 16, st));
        pw_bad = reinterpret_cast<int32_t*>(reinterpret_cast<char*>(pw) + pw_bytes);
        GEM_CHECK_CUDA(cudaMemsetAsync(pw_bad, 0, 4, st));
        pw_table_kernel<<<(unsigned)((G * pw_buckets(W) + 255) / 256), 256, 0, st>>>(lut, nmax + 1, G, W, pw);
        GEM_CHECK_LAUNCH("pw_table_kernel");
        pw_check_kernel<<<(unsigned)imin64(((int64_t)G * W + 255) / 256, 4 * num_sms()), 256, 0, st>>>(
            lut, nmax + 1, G, W, pw, pw_bad);
        GEM_CHECK_LAUNCH("pw_check_kernel");
        smem += pw_bytes;
      }
      auto go = [&](auto kern) -> cudaError_t {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        kern<<<(unsigned)R, g2_threads(GM), smem, st>>>(hist, T, E, G, lut, nmax, W, run_layer, needs_greedy, order,
                                                    assign, l16, ws, tp, td, ta, pw, pw_bad);
        return cudaGetLastError();
      };
      auto pick = [&](auto tag) -> cudaError_t {
        constexpr bool T2 = decltype(tag)::value;
        return sl ? (GM == G ? (GM == 8 ? go(greedy2_kernel<8, true, true, T2>)
                                        : (GM == 16 ? go(greedy2_kernel<16, true, true, T2>)
                                                    : go(greedy2_kernel<32, true, true, T2>)))
                             : (GM == 8 ? go(greedy2_kernel<8, false, true, T2>)
                                        : (GM == 16 ? go(greedy2_kernel<16, false, true, T2>)
                                                    : go(greedy2_kernel<32, false, true, T2>))))
                  : (GM == G ? (GM == 8 ? go(greedy2_kernel<8, true, false, T2>)
                                        : (GM == 16 ? go(greedy2_kernel<16, true, false, T2>)
                                                    : go(greedy2_kernel<32, true, false, T2>)))
                             : (GM == 8 ? go(greedy2_kernel<8, false, false, T2>)
                                        : (GM == 16 ? go(greedy2_kernel<16, false, false, T2>)
                                                    : go(greedy2_kernel<32, false, false, T2>))));
      };
      const cudaError_t ek = top2 ? pick(std::true_type{}) : pick(std::false_type{});
      cudaFreeAsync(l16, st);
      if (pw) cudaFreeAsync(pw, st);
      if (top2) {
        cudaFreeAsync(tp, st);
        cudaFreeAsync(td, st);
        cudaFreeAsync(ta, st);
      }
      if (ek != cudaSuccess) return fail_cuda(ek, "greedy2_kernel");
      return GEM_OK;
    }
  }
  // per-GPU cost chunks in shared memory: 256 steps, fewer when G is large
  int tchunk = kGreedyTChunk;
  while (tchunk > 32 && (size_t)G * tchunk * sizeof(double) > (size_t)optin - 4096) tchunk /= 2;
  const size_t gsmem = (size_t)G * tchunk * sizeof(double);
  GEM_CHECK_CUDA(cudaFuncSetAttribute(greedy_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gsmem));
  greedy_kernel<<<(unsigned)R, kSearchThreads, gsmem, st>>>(hist, T, E, G, lut, nmax, run_layer, needs_greedy, order,
                                                            assign, ws.loads, tchunk);
  GEM_CHECK_LAUNCH("greedy_kernel");
  return GEM_OK;
}

// Screening scratch (K6 v3+, K7 v2): the fp32 table, the transposed uint16
// histogram and the load bound U; stream-ordered allocations freed on every
// exit path. Without a transposed histogram (some count >= 65536) the search
// runs the exact v1 kernels.
struct Screen {
  float* lut32 = nullptr;
  uint16_t* ht16 = nullptr;
  uint16_t* ht16s = nullptr;
  uint16_t* first = nullptr;
  float* bscale = nullptr;
  int64_t U = 0;
  cudaStream_t st = nullptr;
  ~Screen() {
    if (first) cudaFreeAsync(first, st);
    if (bscale) cudaFreeAsync(bscale, st);
    if (lut32) cudaFreeAsync(lut32, st);
    if (ht16) cudaFreeAsync(ht16, st);
    if (ht16s) cudaFreeAsync(ht16s, st);
  }
};

static int prepare_screen(const int32_t* hist, int64_t L, int64_t T, int32_t E, int32_t G, const double* lut,
                          int64_t nmax, Screen& sc, SearchWs& ws, cudaStream_t st) {
  sc.st = st;
  keep_pool();
  // G > 32: the screened kernels keep GPU sets in 32-bit masks -- the exact
  // v1 kernels (any G) run instead
  if (G < 2 || G > 32 || T > (1LL << 24)) return GEM_OK;
  const int64_t n = (int64_t)G * (nmax + 1);
  GEM_CHECK_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&sc.lut32), (size_t)n * sizeof(float), st));
  lut_to_f32_kernel<<<(unsigned)imin64((n + 255) / 256, 4096), 256, 0, st>>>(lut, n, sc.lut32);
  GEM_CHECK_LAUNCH("lut_to_f32_kernel");
  ws.lut32 = sc.lut32;
  // U = max over layers and steps of the sum of the E/G largest counts
  int32_t* bound = nullptr;
  GEM_CHECK_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&bound), (size_t)(L + 1) * 4, st));
  GEM_CHECK_CUDA(cudaMemsetAsync(bound, 0, (size_t)(L + 1) * 4, st));
  lut_monotone_kernel<<<(unsigned)imin64((n + 255) / 256, 4096), 256, 0, st>>>(sc.lut32, lut, G, nmax + 1,
                                                                               bound + L);
  GEM_CHECK_LAUNCH("lut_monotone_kernel");
  const int warps = 8;
  topn_bound_kernel<<<(unsigned)imin64((L * T + warps - 1) / warps, 16 * num_sms()), warps * 32,
                      (size_t)warps * E * 4, st>>>(hist, L, T, E, E / G, nullptr, bound, nullptr, nullptr);
  std::vector<int32_t> ub((size_t)L + 1);
  cudaError_t e1 = cudaGetLastError();
  cudaError_t e2 = cudaMemcpyAsync(ub.data(), bound, (size_t)(L + 1) * 4, cudaMemcpyDeviceToHost, st);
  cudaError_t e3 = cudaStreamSynchronize(st);
  cudaFreeAsync(bound, st);
  if (e1 != cudaSuccess) return fail_cuda(e1, "topn_bound_kernel");
  if (e2 != cudaSuccess) return fail_cuda(e2, "topn bound copy");
  if (e3 != cudaSuccess) return fail_cuda(e3, "topn bound sync");
  for (int64_t l = 0; l < L; ++l) sc.U = imax64(sc.U, ub[l]);
  ws.lut_monotone = (ub[L] & 1) == 0;
  ws.lut_monotone64 = (ub[L] & 2) == 0;
  ws.win = (int32_t)imin64(sc.U, nmax) + 1;
  if (ws.win <= 65535) {  // u16 search hints
    GEM_CHECK_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&sc.bscale), (size_t)G * 4, st));
    GEM_CHECK_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&sc.first), (size_t)G * (kBuckets + 2) * 2, st));
    bucket_scale_kernel<<<1, 32 * ((G + 31) / 32), 0, st>>>(sc.lut32, G, nmax + 1, ws.win, sc.bscale);
    GEM_CHECK_LAUNCH("bucket_scale_kernel");
    bucket_first_kernel<<<(unsigned)imin64(((int64_t)G * ws.win + 255) / 256, 4096), 256, 0, st>>>(
        sc.lut32, G, nmax + 1, ws.win, sc.bscale, sc.first);
    GEM_CHECK_LAUNCH("bucket_first_kernel");
    ws.first = sc.first;
    ws.bscale = sc.bscale;
  }
  if (sc.U >= 65536) return GEM_OK;
  GEM_CHECK_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&sc.ht16), (size_t)L * E * ws.Tp * 2, st));
  dim3 tg((unsigned)(ws.Tp / 32), (unsigned)((E + 31) / 32), (unsigned)L);
  hist_t16_kernel<<<tg, dim3(32, 8), 0, st>>>(hist, T, ws.Tp, E, 0, sc.ht16);
  GEM_CHECK_LAUNCH("hist_t16_kernel");
  ws.ht16 = sc.ht16;
  if (4 * sc.U < 65536) {  // K6 v5: counts as byte offsets into fp32 rows
    GEM_CHECK_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&sc.ht16s), (size_t)L * E * ws.Tp * 2, st));
    hist_t16_kernel<<<tg, dim3(32, 8), 0, st>>>(hist, T, ws.Tp, E, 2, sc.ht16s);
    GEM_CHECK_LAUNCH("hist_t16_kernel");
    ws.ht16s = sc.ht16s;
  }
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
  carve(&ws, workspace, R, T, E, G);
  Screen screen;
  if ((rc = prepare_screen(hist, L, T, E, G, lut, nmax, screen, ws, st))) return rc;
  GEM_CHECK_CUDA(cudaMemsetAsync(ws.counters, 0, 16, st));
  GEM_CHECK_CUDA(cudaMemsetAsync(ws.need_exact, 0, (size_t)R * 4, st));  // the apply reads the window's verdict
  cudaEvent_t g0 = nullptr, g1 = nullptr;
  if (std::getenv("GEM_SEARCH_TRACE")) {
    GEM_CHECK_CUDA(cudaEventCreate(&g0));
    GEM_CHECK_CUDA(cudaEventCreate(&g1));
    GEM_CHECK_CUDA(cudaEventRecord(g0, st));
  }
  rc = launch_greedy(hist, T, E, G, lut, nmax, screen.U, R, run_layer, needs_greedy, order, assign, ws, st);
  if (rc) return rc;
  {
    int64_t bx = (T * G + 255) / 256;
    if (bx > 64) bx = 64;
    dim3 grid((unsigned)bx, (unsigned)R);
    init_loads_kernel<<<grid, 256, E, st>>>(hist, T, E, G, run_layer, needs_greedy, assign, ws.loads);
    GEM_CHECK_LAUNCH("init_loads_kernel");
  }
  init_score_kernel<<<(unsigned)R, kSearchThreads, 0, st>>>(T, G, lut, nmax, ws, traj_cap, trajectory, swaps);
  GEM_CHECK_LAUNCH("init_score_kernel");
  if (ws.ht16) {
    state_t_kernel<<<4 * num_sms(), 256, 0, st>>>(R, T, G, nmax + 1, ws);
    GEM_CHECK_LAUNCH("state_t_kernel");
  }
  if (g0) {
    GEM_CHECK_CUDA(cudaEventRecord(g1, st));
    GEM_CHECK_CUDA(cudaEventSynchronize(g1));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, g0, g1);
    int32_t nex = 0;
    cudaMemcpy(&nex, ws.counters + 2, 4, cudaMemcpyDeviceToHost);
    std::fprintf(stderr, "gem_search greedy+init (%lld runs): %.3f ms, exact greedy re-scores %d\n", (long long)R, ms,
                 nex);
    cudaEventDestroy(g0);
    cudaEventDestroy(g1);
  }
  // GEM_SEARCH_TRACE=1: per-round timing (CUDA events) and active-run counts on stderr
  const bool trace = std::getenv("GEM_SEARCH_TRACE") != nullptr;
  cudaEvent_t ev[3] = {nullptr, nullptr, nullptr};
  if (trace) {
    for (auto& e : ev) GEM_CHECK_CUDA(cudaEventCreate(&e));
  }
  int64_t n_active = R;  // every run is active before its first scan
  for (int64_t it = 0; it < swap_cap; ++it) {
    if (trace) GEM_CHECK_CUDA(cudaEventRecord(ev[0], st));
    rc = launch_scan(hist, T, E, G, lut, nmax, R, n_active, run_layer, assign, ws, st, threshold);
    if (rc) return rc;
    if (trace) GEM_CHECK_CUDA(cudaEventRecord(ev[1], st));
    if (G < 2) break;  // no cross-GPU pair exists: found == false for every run
    GEM_CHECK_CUDA(cudaMemsetAsync(ws.counters, 0, 4, st));
    apply_swap_kernel<<<(unsigned)R, kSearchThreads, 0, st>>>(hist, T, E, G, lut, nmax, run_layer, assign, ws,
                                                              threshold, swap_cap, traj_cap, trajectory, swaps);
    GEM_CHECK_LAUNCH("apply_swap_kernel");
    int32_t active = 0;
    GEM_CHECK_CUDA(cudaMemcpyAsync(&active, ws.counters, 4, cudaMemcpyDeviceToHost, st));
    GEM_CHECK_CUDA(cudaStreamSynchronize(st));
    if (trace) {
      GEM_CHECK_CUDA(cudaEventRecord(ev[2], st));
      GEM_CHECK_CUDA(cudaEventSynchronize(ev[2]));
      float ms_scan = 0.f, ms_all = 0.f;
      cudaEventElapsedTime(&ms_scan, ev[0], ev[1]);
      cudaEventElapsedTime(&ms_all, ev[0], ev[2]);
      std::fprintf(stderr, "gem_search round %lld: active %lld scan %.3f ms apply %.3f ms\n", (long long)it,
                   (long long)n_active, ms_scan, ms_all - ms_scan);
    }
    if (active == 0) break;
    n_active = active;
  }
  if (trace) {
    for (auto& e : ev) cudaEventDestroy(e);
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
  carve(&ws, workspace, R, T, E, G);
  Screen screen;
  if ((rc = prepare_screen(hist, L, T, E, G, lut, nmax, screen, ws, st))) return rc;
  int64_t bx = (T * G + 255) / 256;
  if (bx > 64) bx = 64;
  init_loads_kernel<<<dim3((unsigned)bx, (unsigned)R), 256, E, st>>>(hist, T, E, G, run_layer, nullptr, assign,
                                                                     ws.loads);
  GEM_CHECK_LAUNCH("init_loads_kernel");
  if (ws.ht16) {
    state_t_kernel<<<4 * num_sms(), 256, 0, st>>>(R, T, G, nmax + 1, ws);
    GEM_CHECK_LAUNCH("state_t_kernel");
  }
  std::vector<int32_t> ones(R, 1);
  GEM_CHECK_CUDA(cudaMemcpyAsync(ws.run_active, ones.data(), R * 4, cudaMemcpyHostToDevice, st));
  if (G >= 2) {
    rc = launch_scan(hist, T, E, G, lut, nmax, R, R, run_layer, assign, ws, st);
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
