// Trace ingestion and statistics on sm_100a.
//
//  K9 gem_gen_topk      synthetic router ids (Philox, integer-only)
//  (K1 gem_topk_hist lives in hist.cu)
//     gem_hist_colstats counts -> per-expert totals (ExpertTrace input)
//  K2 gem_step_gram     step-level co-activation Gram (Pearson statistics)
//  K3 gem_stats_finalize / gem_classify
//
// The reference takes the histogram as input (trace.py:24-45)
// and derives statistics with numpy (trace.py:87-114). K1 is the missing
// ingestion step; its bytes dominate the whole statistics phase, so it is the
// kernel sized against HBM: ids are streamed with 128-bit loads and counted
// into per-lane private sub-histograms (u16x2 words laid out bin-pair-major,
// lane-minor, so lane L always hits bank L: no conflicts, no atomics
// contention), reduced once per step with a bank-rotated transpose.
#include <cstdio>
#include <cstdlib>

#include "gem_common.cuh"

namespace gem {

// ---------------------------------------------------------------------------
// K9: synthetic top-k ids
// ---------------------------------------------------------------------------
constexpr uint32_t kTagConsistent = 0x80000000u;
constexpr uint32_t kTagGroup = 0xC0000000u;
constexpr int kGenMaxK = 32;
constexpr int kGenAttempts = 32;

__device__ __forceinline__ uint32_t draw_u32(uint64_t seed, uint32_t c0, uint32_t c1,
                                             uint32_t c2, uint32_t c3) {
  u32x4 c{c0, c1, c2, c3};
  return philox4x32_10(c, (uint32_t)seed, (uint32_t)(seed >> 32)).x;
}

template <typename IdT>
__global__ void gen_topk_kernel(int64_t N, int k, int B, int E, const uint32_t* __restrict__ weight,
                                const int8_t* __restrict__ role, uint32_t p_cons, uint32_t p_burst,
                                uint32_t burst_mult, uint64_t seed, int64_t token_offset,
                                int64_t first_step, IdT* __restrict__ ids) {
  extern __shared__ unsigned char smem_raw[];
  uint64_t* cdf = reinterpret_cast<uint64_t*>(smem_raw);  // [E] inclusive prefix
  uint64_t* wts = cdf + E;                                // [E] gated weights
  const int l = blockIdx.y;
  const int64_t step = first_step + blockIdx.x;
  const uint32_t s_lo = (uint32_t)step, s_hi = (uint32_t)(step >> 32);

  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    const int r = role[(int64_t)l * E + e];
    uint64_t w = weight[(int64_t)l * E + e];
    if (r == 1) {
      if (draw_u32(seed, s_lo, s_hi, (uint32_t)l, kTagConsistent | (uint32_t)e) >= p_cons) w = 0;
    } else if (r >= 2) {
      const uint32_t g = (uint32_t)(r - 2);
      if (draw_u32(seed, s_lo, s_hi, (uint32_t)l, kTagGroup | g) < p_burst) w *= burst_mult;
      else w = 0;
    }
    wts[e] = w;
  }
  __syncthreads();
  if (threadIdx.x == 0) {  // E <= 1024: a serial prefix is cheap next to the token draws
    uint64_t run = 0;
    for (int e = 0; e < E; ++e) { run += wts[e]; cdf[e] = run; }
  }
  __syncthreads();
  const uint64_t total = cdf[E - 1];

  // local token range of this step
  const int64_t g0 = step * (int64_t)B, g1 = g0 + B;
  const int64_t n0 = imax64(g0 - token_offset, 0);
  const int64_t n1 = imin64(g1 - token_offset, N);
  IdT* out = ids + (int64_t)l * N * k;
  for (int64_t n = n0 + threadIdx.x; n < n1; n += blockDim.x) {
    const int64_t gtok = token_offset + n;
    const uint32_t t_lo = (uint32_t)gtok, t_hi = (uint32_t)(gtok >> 32);
    int chosen[kGenMaxK];
    for (int s = 0; s < k; ++s) {
      int pick = -1;
      if (total > 0) {
        for (int a = 0; a < kGenAttempts && pick < 0; ++a) {
          const uint32_t u = draw_u32(seed, t_lo, t_hi, (uint32_t)l, (uint32_t)(s * 64 + a));
          const uint64_t r = ((uint64_t)u * total) >> 32;  // [0, total)
          int lo = 0, hi = E - 1;                            // first e with cdf[e] > r
          while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (cdf[mid] > r) hi = mid; else lo = mid + 1;
          }
          bool dup = false;
          for (int q = 0; q < s; ++q) dup |= (chosen[q] == lo);
          if (!dup) pick = lo;
        }
      }
      if (pick < 0) {  // deterministic fallback: lowest unchosen positive weight, then lowest unchosen
        for (int pass = 0; pass < 2 && pick < 0; ++pass) {
          for (int e = 0; e < E && pick < 0; ++e) {
            if (pass == 0 && wts[e] == 0) continue;
            bool dup = false;
            for (int q = 0; q < s; ++q) dup |= (chosen[q] == e);
            if (!dup) pick = e;
          }
        }
      }
      chosen[s] = pick;
      out[n * k + s] = (IdT)pick;
    }
  }
}

// counts -> colsum / active / heavy (ExpertTrace path). heavy counts the
// steps in which the expert got at least its fair share, h*E >= row total
// (the same predicate K1 applies while it builds the rows).
constexpr int kColstatsChunk = 256;

__global__ void __launch_bounds__(256)
hist_colstats_kernel(const int32_t* __restrict__ hist, int64_t T, int E, int64_t* __restrict__ colsum,
                     int32_t* __restrict__ active, int32_t* __restrict__ heavy) {
  __shared__ int64_t rtot[kColstatsChunk];
  const int64_t l = blockIdx.y;
  const int64_t t0 = (int64_t)blockIdx.x * kColstatsChunk, t1 = imin64(t0 + kColstatsChunk, T);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int64_t t = t0 + warp; t < t1; t += blockDim.x >> 5) {
    int64_t s = 0;
    for (int e = lane; e < E; e += 32) s += hist[(l * T + t) * E + e];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) rtot[t - t0] = s;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    int64_t s = 0;
    int32_t a = 0, hv = 0;
    for (int64_t t = t0; t < t1; ++t) {
      const int32_t h = hist[(l * T + t) * E + e];
      s += h;
      a += (h > 0);
      hv += (h > 0 && (int64_t)h * E >= rtot[t - t0]);
    }
    if (s) atomicAdd((unsigned long long*)&colsum[l * E + e], (unsigned long long)s);
    if (a) atomicAdd(&active[l * E + e], a);
    if (hv) atomicAdd(&heavy[l * E + e], hv);
  }
}

// ---------------------------------------------------------------------------
// K2: step-level Gram, CUDA-core version (64x64 tile, 4x4 per thread, T split)
// ---------------------------------------------------------------------------
constexpr int kGramTile = 64;
constexpr int kGramTChunk = 32;

__global__ void __launch_bounds__(256)
step_gram_kernel(const int32_t* __restrict__ hist, int64_t T, int E, int64_t t_per_block,
                 int64_t* __restrict__ gram) {
  __shared__ int32_t sa[kGramTChunk][kGramTile];
  __shared__ int32_t sb[kGramTChunk][kGramTile];
  const int64_t l = blockIdx.z;
  const int tiles = (E + kGramTile - 1) / kGramTile;
  const int ta = blockIdx.y / tiles, tb = blockIdx.y % tiles;
  if (tb < ta) return;  // upper triangle of tiles; finalize mirrors
  const int a0 = ta * kGramTile, b0 = tb * kGramTile;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  int64_t acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0;
  const int64_t tb0 = (int64_t)blockIdx.x * t_per_block;
  const int64_t tb1 = imin64(tb0 + t_per_block, T);
  for (int64_t t0 = tb0; t0 < tb1; t0 += kGramTChunk) {
    for (int i = threadIdx.x; i < kGramTChunk * kGramTile; i += 256) {
      const int r = i / kGramTile, c = i % kGramTile;
      const int64_t t = t0 + r;
      const bool tv = t < tb1;
      sa[r][c] = (tv && a0 + c < E) ? hist[(l * T + t) * E + a0 + c] : 0;
      sb[r][c] = (tv && b0 + c < E) ? hist[(l * T + t) * E + b0 + c] : 0;
    }
    __syncthreads();
#pragma unroll 4
    for (int r = 0; r < kGramTChunk; ++r) {
      int32_t va[4], vb[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) { va[i] = sa[r][ty * 4 + i]; vb[i] = sb[r][tx * 4 + i]; }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] += (int64_t)va[i] * (int64_t)vb[j];
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int a = a0 + ty * 4 + i, b = b0 + tx * 4 + j;
      if (a < E && b < E && acc[i][j])
        atomicAdd((unsigned long long*)&gram[(l * E + a) * E + b], (unsigned long long)acc[i][j]);
    }
}

// ---------------------------------------------------------------------------
// K3: finalize statistics + classification
// ---------------------------------------------------------------------------
__device__ __forceinline__ double i128_to_double(__int128 v) {
  const bool neg = v < 0;
  unsigned __int128 u = neg ? (unsigned __int128)(-v) : (unsigned __int128)v;
  const double d = (double)(uint64_t)(u >> 64) * 18446744073709551616.0 + (double)(uint64_t)u;
  return neg ? -d : d;
}

__device__ __forceinline__ int64_t gram_at(const int64_t* g, int E, int a, int b) {
  return a <= b ? g[(int64_t)a * E + b] : g[(int64_t)b * E + a];
}

__global__ void stats_finalize_kernel(const int64_t* __restrict__ colsum, const int32_t* __restrict__ active,
                                      const int64_t* __restrict__ gram, int64_t T, int E,
                                      double* __restrict__ mean_util, double* __restrict__ active_frac,
                                      double* __restrict__ corr) {
  const int64_t l = blockIdx.y;
  const int64_t* cs = colsum + l * E;
  __shared__ unsigned long long s_total;
  if (threadIdx.x == 0) s_total = 0;
  __syncthreads();
  if (blockIdx.x == 0) {
    unsigned long long part = 0;
    for (int e = threadIdx.x; e < E; e += blockDim.x) part += (unsigned long long)cs[e];
    atomicAdd(&s_total, part);
  }
  __syncthreads();
  if (blockIdx.x == 0) {
    const double total = (double)(int64_t)s_total;
    for (int e = threadIdx.x; e < E; e += blockDim.x) {
      if (mean_util) mean_util[l * E + e] = __ddiv_rn((double)cs[e], total);
      if (active_frac) active_frac[l * E + e] = __ddiv_rn((double)active[l * E + e], (double)T);
    }
  }
  if (!corr || !gram) return;
  const int64_t* g = gram + l * (int64_t)E * E;
  double* cr = corr + l * (int64_t)E * E;
  const int64_t pairs = (int64_t)E * E;
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < pairs; p += (int64_t)gridDim.x * blockDim.x) {
    const int a = (int)(p / E), b = (int)(p % E);
    double v;
    if (a == b) {
      v = 1.0;
    } else {
      const int lo = a < b ? a : b, hi = a < b ? b : a;  // compute from (lo,hi): exact symmetry
      const __int128 sa = cs[lo], sb = cs[hi];
      const __int128 va = (__int128)T * gram_at(g, E, lo, lo) - sa * sa;
      const __int128 vb = (__int128)T * gram_at(g, E, hi, hi) - sb * sb;
      if (va == 0 || vb == 0) {
        v = 0.0;
      } else {
        const __int128 num = (__int128)T * gram_at(g, E, lo, hi) - sa * sb;
        v = i128_to_double(num) / (sqrt(i128_to_double(va)) * sqrt(i128_to_double(vb)));
        v = fmin(1.0, fmax(-1.0, v));
      }
    }
    cr[p] = v;
  }
}

__global__ void classify_kernel(const int64_t* __restrict__ colsum, const int32_t* __restrict__ heavy,
                                const int64_t* __restrict__ gram, int64_t T, int E, int64_t cons_num,
                                int64_t cons_den, int64_t corr_num, int64_t corr_den,
                                int8_t* __restrict__ cls, int16_t* __restrict__ group,
                                int32_t* __restrict__ err) {
  extern __shared__ uint32_t csm[];
  const int words = (E + 31) / 32;
  uint32_t* adj = csm;                                   // [E][words]
  int32_t* label = reinterpret_cast<int32_t*>(adj + (size_t)E * words);
  int8_t* scls = reinterpret_cast<int8_t*>(label + E);
  __shared__ int changed;
  const int64_t l = blockIdx.x;
  const int64_t* cs = colsum + l * E;
  const int64_t* g = gram + l * (int64_t)E * E;
  // consistent: heavy (>= fair share) in at least cons_num/cons_den of the
  // steps; candidates for temporal: heavy in some step but not consistent
  // (kClassBurst marks them until the correlation pass confirms them)
  constexpr int8_t kClassBurst = 3;
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    const int64_t hv = heavy[l * E + e];
    scls[e] = ((__int128)hv * cons_den >= (__int128)cons_num * T) ? GEM_CLASS_CONSISTENT
              : hv > 0                                           ? kClassBurst
                                                                 : GEM_CLASS_OTHER;
  }
  for (int i = threadIdx.x; i < E * words; i += blockDim.x) adj[i] = 0;
  __syncthreads();
  const __int128 lim = (__int128)1 << 60;
  for (int64_t p = threadIdx.x; p < (int64_t)E * E; p += blockDim.x) {
    const int a = (int)(p / E), b = (int)(p % E);
    if (b <= a || scls[a] != kClassBurst || scls[b] != kClassBurst) continue;
    const __int128 sa = cs[a], sb = cs[b];
    const __int128 va = (__int128)T * gram_at(g, E, a, a) - sa * sa;
    const __int128 vb = (__int128)T * gram_at(g, E, b, b) - sb * sb;
    if (va == 0 || vb == 0) continue;
    const __int128 num = (__int128)T * gram_at(g, E, a, b) - sa * sb;
    if (num <= 0) continue;
    if (num >= lim || va >= lim || vb >= lim) { atomicExch(err, 1); continue; }
    // r >= corr_num/corr_den  <=>  den^2 num^2 >= n^2 va vb   (num > 0)
    const __int128 lhs = (__int128)(corr_den * corr_den) * (num * num);
    const __int128 rhs = (__int128)(corr_num * corr_num) * (va * vb);
    if (lhs >= rhs) {
      atomicOr(&adj[(size_t)a * words + b / 32], 1u << (b % 32));
      atomicOr(&adj[(size_t)b * words + a / 32], 1u << (a % 32));
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    bool any = false;
    for (int w = 0; w < words; ++w) any |= adj[(size_t)e * words + w] != 0;
    if (scls[e] == kClassBurst) scls[e] = any ? GEM_CLASS_TEMPORAL : GEM_CLASS_OTHER;
    label[e] = scls[e] == GEM_CLASS_TEMPORAL ? e : -1;
  }
  __syncthreads();
  // min-label propagation over the temporal correlation graph
  for (int it = 0; it < E; ++it) {
    if (threadIdx.x == 0) changed = 0;
    __syncthreads();
    for (int e = threadIdx.x; e < E; e += blockDim.x) {
      if (label[e] < 0) continue;
      int best = label[e];
      for (int w = 0; w < words; ++w) {
        uint32_t m = adj[(size_t)e * words + w];
        while (m) {
          const int f = w * 32 + __ffs(m) - 1;
          m &= m - 1;
          const int lf = label[f];
          if (lf >= 0 && lf < best) best = lf;
        }
      }
      if (best < label[e]) { atomicMin(&label[e], best); changed = 1; }
    }
    __syncthreads();
    if (!changed) break;
    __syncthreads();
  }
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    cls[l * E + e] = scls[e];
    group[l * E + e] = (int16_t)label[e];
  }
}

}  // namespace gem

using namespace gem;

extern "C" int gem_gen_topk(int64_t L, int64_t N, int32_t k, int32_t B, int32_t E, const uint32_t* weight,
                            const int8_t* role, uint32_t p_consistent, uint32_t p_burst, uint32_t burst_mult,
                            uint64_t seed, int64_t token_offset, int32_t id_bytes, void* ids, void* stream) {
  GEM_REQUIRE(L >= 1 && N >= 1 && k >= 1 && k <= kGenMaxK && B >= 1 && E >= 1 && E <= 1024,
              "gem_gen_topk: bad shape L=%lld N=%lld k=%d B=%d E=%d", (long long)L, (long long)N, k, B, E);
  GEM_REQUIRE(k <= E, "gem_gen_topk: k=%d exceeds E=%d", k, E);
  GEM_REQUIRE(id_bytes == 2 || id_bytes == 4, "gem_gen_topk: id_bytes must be 2 or 4");
  GEM_REQUIRE(token_offset >= 0, "gem_gen_topk: negative token_offset");
  GEM_REQUIRE(weight && role && ids, "gem_gen_topk: null pointer");
  const int64_t first_step = token_offset / B;
  const int64_t last_step = (token_offset + N - 1) / B;
  const int64_t steps = last_step - first_step + 1;
  GEM_REQUIRE(L <= 65535, "gem_gen_topk: L too large");
  dim3 grid((unsigned)steps, (unsigned)L);
  const size_t smem = (size_t)E * 16;
  if (id_bytes == 2)
    gen_topk_kernel<int16_t><<<grid, 256, smem, as_stream(stream)>>>(N, k, B, E, weight, role, p_consistent, p_burst,
                                                                    burst_mult, seed, token_offset, first_step,
                                                                    (int16_t*)ids);
  else
    gen_topk_kernel<int32_t><<<grid, 256, smem, as_stream(stream)>>>(N, k, B, E, weight, role, p_consistent, p_burst,
                                                                    burst_mult, seed, token_offset, first_step,
                                                                    (int32_t*)ids);
  GEM_CHECK_LAUNCH("gen_topk_kernel");
  return GEM_OK;
}

extern "C" int gem_hist_colstats(const int32_t* hist, int64_t L, int64_t T, int32_t E, int64_t* colsum,
                                 int32_t* active, int32_t* heavy, void* stream) {
  GEM_REQUIRE(L >= 1 && T >= 1 && E >= 1 && hist && colsum && active && heavy, "gem_hist_colstats: bad arguments");
  GEM_REQUIRE(L <= 65535, "gem_hist_colstats: L too large");
  dim3 grid((unsigned)((T + kColstatsChunk - 1) / kColstatsChunk), (unsigned)L);
  hist_colstats_kernel<<<grid, 256, 0, as_stream(stream)>>>(hist, T, E, colsum, active, heavy);
  GEM_CHECK_LAUNCH("hist_colstats_kernel");
  return GEM_OK;
}

extern "C" int gem_step_gram_cc(const int32_t* hist, int64_t L, int64_t T, int32_t E, int64_t* gram, void* stream) {
  GEM_REQUIRE(L >= 1 && T >= 1 && E >= 1 && hist && gram, "gem_step_gram: bad arguments");
  GEM_REQUIRE(L <= 65535, "gem_step_gram: L too large");
  const int tiles = (E + kGramTile - 1) / kGramTile;
  // split T so the grid covers the machine a few times over
  const int64_t tile_blocks = (int64_t)tiles * (tiles + 1) / 2 * L;
  int64_t splits = (4LL * num_sms() + tile_blocks - 1) / tile_blocks;
  if (splits < 1) splits = 1;
  int64_t t_per = (T + splits - 1) / splits;
  t_per = ((t_per + kGramTChunk - 1) / kGramTChunk) * kGramTChunk;
  splits = (T + t_per - 1) / t_per;
  dim3 grid((unsigned)splits, (unsigned)(tiles * tiles), (unsigned)L);
  step_gram_kernel<<<grid, 256, 0, as_stream(stream)>>>(hist, T, E, t_per, gram);
  GEM_CHECK_LAUNCH("step_gram_kernel");
  return GEM_OK;
}

// K2 dispatcher: the tcgen05 kernel (gram_tc.cu) whenever its preconditions
// hold (E a multiple of 128 up to 512; every count in [0, 65535], which the
// caller vouches for through max_count), the CUDA-core kernel otherwise.
extern "C" int gem_step_gram_path(int32_t E, int64_t max_count) {
  return (E >= 128 && E <= 512 && E % 128 == 0 && max_count >= 0 && max_count <= 65535) ? 1 : 0;
}

extern "C" int gem_step_gram(const int32_t* hist, int64_t L, int64_t T, int32_t E, int64_t max_count, int64_t* gram,
                             void* stream) {
  if (gem_step_gram_path(E, max_count) == 1) return gem_step_gram_tc(hist, L, T, E, gram, stream);
  return gem_step_gram_cc(hist, L, T, E, gram, stream);
}

extern "C" int gem_stats_finalize(const int64_t* colsum, const int32_t* active, const int64_t* gram, int64_t L,
                                  int64_t T, int32_t E, double* mean_util, double* active_frac, double* corr,
                                  void* stream) {
  GEM_REQUIRE(L >= 1 && T >= 1 && E >= 1 && colsum && active, "gem_stats_finalize: bad arguments");
  GEM_REQUIRE(!corr || gram, "gem_stats_finalize: corr requires gram");
  const int64_t pairs = (int64_t)E * E;
  int bx = (int)((pairs + 255) / 256);
  if (bx > 64) bx = 64;
  if (bx < 1) bx = 1;
  dim3 grid((unsigned)bx, (unsigned)L);
  stats_finalize_kernel<<<grid, 256, 0, as_stream(stream)>>>(colsum, active, gram, T, E, mean_util, active_frac,
                                                            corr);
  GEM_CHECK_LAUNCH("stats_finalize_kernel");
  return GEM_OK;
}

extern "C" int gem_classify(const int64_t* colsum, const int32_t* heavy, const int64_t* gram, int64_t L, int64_t T,
                            int32_t E, int64_t cons_num, int64_t cons_den, int64_t corr_num, int64_t corr_den,
                            int8_t* cls, int16_t* group, int32_t* err_flag, void* stream) {
  GEM_REQUIRE(L >= 1 && T >= 1 && E >= 1 && E <= 1024 && colsum && heavy && gram && cls && group && err_flag,
              "gem_classify: bad arguments");
  GEM_REQUIRE(cons_den > 0 && cons_num >= 0 && corr_den > 0 && corr_num > 0 && corr_num <= corr_den &&
                  corr_den <= (1 << 20),
              "gem_classify: thresholds must be rationals with small positive denominators");
  cudaStream_t st = as_stream(stream);
  const int words = (E + 31) / 32;
  const size_t smem = (size_t)E * words * 4 + (size_t)E * 4 + (size_t)E;
  GEM_CHECK_CUDA(cudaFuncSetAttribute(classify_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  classify_kernel<<<(unsigned)L, 256, smem, st>>>(colsum, heavy, gram, T, E, cons_num, cons_den, corr_num, corr_den,
                                                  cls, group, err_flag);
  GEM_CHECK_LAUNCH("classify_kernel");
  return GEM_OK;
}
