// K5 v4: straggler scoring of thousands of candidate mappings on B200.
//
//   score[c][l] = sum_t (serial fp64)  max_g C_g( n_g(c,l,t) ),
//   n_g(c,l,t)  = sum_{e : cand[c][l][e] == g} h[l][t][e]        (mapping.py:146-166)
//
// Order keys. Every latency the scorer can meet is a table value lut[g][n]
// with n in [s_g, U] (U = max over steps of the sum of the `maxcnt` largest
// counts, maxcnt = the most experts any candidate puts on one GPU: no load can
// exceed it; s_g = the gather clamp, below which a load may read the key at
// s_g without changing any step maximum). The distinct values of those rows,
// sorted, give each (n, g) a key = the rank of lut[g][n] (u16, or u32 past
// 65,536 distinct values): keys compare exactly like the fp64 values (equal
// values share a key), so the per-step maximum is an integer max over G keys
// and its exact value is vals[key].
//
//  pass 1 (maxkey_tc_kernel, tcgen05 kind::i8): the per-GPU loads of every
//    candidate are a one-hot GEMM D[t][(c,g)] = sum_e H[t][e] * O[e][(c,g)]
//    with H split into u8 limbs [lo | 16*hi] along K and O as [O | 16*O], so
//    the s32 accumulator in TMEM is the load itself. M = 128 steps, N = 256
//    (candidate, GPU) columns, K = 2E bytes (E = 256: two K parts through one
//    A buffer). The epilogue drains TMEM (tcgen05.ld: one step per lane),
//    looks every load up in the key rows (shared memory; rows too long for it
//    split with a global table) and writes the step's maximum key per
//    candidate: [layer][t][c] -- 1/G of the bytes of the loads themselves.
//  pass 2 (keysum_kernel): one thread per 4 candidates of a layer walks t in
//    order and adds vals[key] to each fp64 chain exactly as the reference
//    sums (_util.py:8-18); the low end of vals sits in shared memory.
//
// Bit-exact with score_layers_kernel and the oracle by construction.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_select.cuh>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "gem_common.cuh"
#include "tc.cuh"

namespace gem {

__global__ void topn_bound_kernel(const int32_t* __restrict__ hist, int64_t L, int64_t T, int E, int n,
                                  const int32_t* __restrict__ n_dev, int32_t* __restrict__ bound,
                                  int32_t* __restrict__ top1, int32_t* __restrict__ rowmin);  // search.cu

#ifndef GEM_LT_WARPS
#define GEM_LT_WARPS 8
#endif
#ifndef GEM_LT_WARPS_SKIP
#define GEM_LT_WARPS_SKIP 16
#endif
constexpr int kLtWarps = GEM_LT_WARPS;  // maxkey CTA: 8 or 16 warps (4 per TMEM lane quarter per column group)
// with step floors (G >= 16): the skipped columns free registers (122 at
// DeepSeek-V3 shapes), and 16 warps hide the gathers' latency better
constexpr int kLtWarpsSkip = GEM_LT_WARPS_SKIP;
constexpr int kLtN = 256;        // MMA N (candidate x GPU columns per CTA)
constexpr int kMaxKeys = 65536;  // u16 keys
constexpr int kSumThreads = 256;
#ifndef GEM_SUM_VALS
#define GEM_SUM_VALS 8192
#endif
constexpr int kSumSmemVals = GEM_SUM_VALS;  // vals[base, base + 8192) in shared memory (64 KB)
constexpr int kSumCtasPerSm = (227 * 1024) / (kSumSmemVals * 8 + 1024);  // shared-memory limited

struct LoadsTcShared {
  uint64_t mma_bar;
  uint32_t tmem_base;
};

// max number of experts any candidate places on one GPU, and a flag for
// entries outside [0, G): out[0] = maxcnt, out[1] = invalid
__global__ void cand_stats_kernel(const int8_t* __restrict__ cand, int64_t rows, int E, int G,
                                  int32_t* __restrict__ out) {
  extern __shared__ int32_t cs_cnt[];  // [warps][G]
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int32_t* cnt = cs_cnt + (size_t)w * G;
  for (int64_t r = (int64_t)blockIdx.x * nw + w; r < rows; r += (int64_t)gridDim.x * nw) {
    for (int g = lane; g < G; g += 32) cnt[g] = 0;
    __syncwarp();
    const int8_t* m = cand + r * E;
    for (int e = lane; e < E; e += 32) {
      const int g = m[e];
      if (g < 0 || g >= G) atomicExch(&out[1], 1);
      else atomicAdd(&cnt[g], 1);
    }
    __syncwarp();
    int mx = 0;
    for (int g = lane; g < G; g += 32) mx = max(mx, cnt[g]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (lane == 0) atomicMax(&out[0], mx);
    __syncwarp();
  }
}


// bad: bit 0 if any table entry is negative, NaN or infinite (checked over the
// whole [G][width] table so the decision is known at the one host sync)
// (bit 0), and bit 1 if a row decreases anywhere (the gather clamp needs
// nondecreasing rows; CostCurve guarantees them, the flag only guards)
__global__ void lut_bad_kernel(const double* __restrict__ lut, int G, int64_t width, int32_t* __restrict__ bad) {
  const int64_t count = (int64_t)G * width;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
    const double v = lut[i];
    if ((unsigned long long)__double_as_longlong(v) >= 0x7ff0000000000000ull) atomicOr(bad, 1);
    if (i % width != 0 && v < lut[i - 1]) atomicOr(bad, 2);
  }
}

// Gather clamp, on the values (before any sort): v* = the smallest table value
// such that sum_g cap_g(v*) >= bmin, cap_g(v) = #{n : lut[g][n] <= v}. No
// step with >= bmin ids can have every GPU strictly below v* (its loads would
// sum to < bmin), so every step maximum is >= v*, and a load n <= thr_g =
// cap_g(v*) - 1 may read the latency at thr_g (<= v* <= the maximum) instead:
// thr[g] = that index (0: no clamp for rows that are bad or decreasing).
// One warp, lane = GPU (G <= 32); bisection on the fp64 bit patterns, which
// order like the values for finite v >= 0.
__global__ void value_clamp_kernel(const double* __restrict__ lut, int G, int64_t width,
                                   const int32_t* __restrict__ bmin, const int32_t* __restrict__ bad,
                                   int32_t* __restrict__ thr) {
  const int g = threadIdx.x;
  if (*bad) {
    if (g < G) thr[g] = 0;
    return;
  }
  const double* row = lut + (int64_t)(g < G ? g : 0) * width;
  auto cap = [&](unsigned long long vb) -> int64_t {  // #{n : lut[g][n] <= v}, 0 for lanes >= G
    if (g >= G) return 0;
    const double v = __longlong_as_double((long long)vb);
    int64_t lo = 0, hi = width;  // first n with row[n] > v
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (row[mid] <= v) lo = mid + 1; else hi = mid;
    }
    return lo;
  };
  auto total = [&](unsigned long long vb) {
    int64_t c = cap(vb);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    return c;
  };
  const int64_t need = *bmin > 0 ? *bmin : 0;
  unsigned long long hi = 0;
  for (int gg = 0; gg < G; ++gg) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(lut[(int64_t)gg * width + width - 1]);
    hi = b > hi ? b : hi;
  }
  unsigned long long lo = 0;  // smallest bit pattern with total >= need (hi always qualifies)
  while (lo < hi) {
    const unsigned long long mid = lo + ((hi - lo) >> 1);
    if (total(mid) >= need) hi = mid; else lo = mid + 1;
  }
  const int64_t c = cap(lo);
  if (g < G) thr[g] = (int32_t)(c > 0 ? c - 1 : 0);
}

// packed key rows of K5 v4: keys[rb_g + n - s_g] = rank of lut[g][n] for n in
// [s_g, U] (rowinfo: [g] = s_g, [G+g] = rb_g, [2G] = total entries)
template <typename KT>
__global__ void key_rows_kernel(const double* __restrict__ lut, int64_t width, int G, int W,
                                const int32_t* __restrict__ rowinfo, const unsigned long long* __restrict__ uniq,
                                const int32_t* __restrict__ nuniq, KT* __restrict__ keys) {
  const int K = *nuniq;
  const int total = rowinfo[2 * G];
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    int g = 0;
    while (g + 1 < G && rowinfo[G + g + 1] <= i) ++g;
    const int n = rowinfo[g] + (i - rowinfo[G + g]);
    if (n >= W) continue;  // row padding of the [G][WG] layout (never read: loads <= U = W - 1)
    const unsigned long long b = (unsigned long long)__double_as_longlong(lut[(int64_t)g * width + n]);
    int lo = 0, hi = K - 1;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (uniq[mid] < b) lo = mid + 1; else hi = mid;
    }
    keys[i] = (KT)lo;
  }
}

// Per-GPU key-row constants of K5 (byte offsets; see maxkey_tc_kernel)
struct KeyRowConsts {
  int32_t koff[32];
  int32_t kbase[32];
  int32_t kend[32];
  int32_t goff[32];
};

// Step floor (K5 at G >= 16). Every expert sits on some GPU, so a step whose
// largest expert count is h has a GPU with load >= h, and with nondecreasing
// rows its maximum is >= v(h) = min_g lut[g][h]. A GPU whose load n is <= the
// step's skip level s(h) = min_g (last n' with lut[g][n'] <= v(h)) has latency
// <= v(h), so it cannot raise the maximum above the floor: the epilogue starts
// each step's maximum at the floor's key and gathers only the GPUs above s(h)
// (skipped with a warp-uniform branch when all 32 steps of a warp are at or
// below it -- at DeepSeek-V3 shapes only the GPUs that hold the step's heavy
// experts). The floor key is the clamped key of (argmin g, h) -- the same entry
// the gather itself would read, which is <= the key of the maximum (h >= s_g:
// it is v(h) itself; h < s_g: the gather-clamp value, <= every maximum).
// Rows that decrease anywhere (bad bit 1) disable the skip: level -1, key 0.
// table[h] = {s(h), key}, h in [0, W)
template <typename KT>
__global__ void floor_table_kernel(const double* __restrict__ lut, int64_t width, int G, int W,
                                   const int32_t* __restrict__ bad, const KT* __restrict__ gkeys,
                                   const __grid_constant__ KeyRowConsts kr, int2* __restrict__ table) {
  const int h = blockIdx.x * blockDim.x + threadIdx.x;
  if (h >= W) return;
  if (*bad & 2) {
    table[h] = make_int2(-1, 0);
    return;
  }
  double v = lut[h];
  int gp = 0;
  for (int g = 1; g < G; ++g) {
    const double x = lut[(int64_t)g * width + h];
    if (x < v) v = x, gp = g;
  }
  int smin = INT32_MAX;
  for (int g = 0; g < G; ++g) {  // first n with row[n] > v, minus one (>= h for g = gp)
    const double* row = lut + (int64_t)g * width;
    int lo = 0, hi = W;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (row[mid] <= v) lo = mid + 1; else hi = mid;
    }
    smin = min(smin, lo - 1);
  }
  const int32_t rel = max((int32_t)sizeof(KT) * h + kr.koff[gp], kr.kbase[gp]);
  const KT key = *reinterpret_cast<const KT*>(reinterpret_cast<const char*>(gkeys) + rel + kr.goff[gp]);
  table[h] = make_int2(smin, (int)key);
}

// per step of every layer: {skip level, floor key} of its largest expert count
// (kmin: the smallest floor key -- no step maximum ranks below it; keysum
// stages the values from there)
__global__ void step_floor_kernel(const int32_t* __restrict__ hist, int64_t rows, int E, int W,
                                  const int2* __restrict__ table, int2* __restrict__ floor_out,
                                  int32_t* __restrict__ kmin) {
  const int lane = threadIdx.x & 31;
  int32_t kl = INT32_MAX;
  const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = w0; r < rows; r += nw) {
    const int32_t* row = hist + r * E;
    int32_t m = 0;
    for (int e = lane; e < E; e += 32) m = max(m, row[e]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane == 0) {
      const int2 f = table[min(m, W - 1)];  // m <= U = W - 1 (the load bound)
      floor_out[r] = f;
      kl = min(kl, f.y);
    }
  }
  if (lane == 0 && kl != INT32_MAX) atomicMin(kmin, kl);
}

// bits[i] = the fp64 pattern of lut[g][n] over the packed rows n in [s_g, U]
// (rowinfo as in key_rows_kernel): only these values can be gathered
__global__ void row_bits_kernel(const double* __restrict__ lut, int64_t width, int G,
                                const int32_t* __restrict__ rowinfo, unsigned long long* __restrict__ bits) {
  const int total = rowinfo[2 * G];
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    int g = 0;
    while (g + 1 < G && rowinfo[G + g + 1] <= i) ++g;
    const int n = rowinfo[g] + (i - rowinfo[G + g]);
    bits[i] = (unsigned long long)__double_as_longlong(lut[(int64_t)g * width + n]);
  }
}

// ---------------------------------------------------------------------------
// pass 1 (v4): CTA = (candidate tile of CT = N/G candidates, layer of the
// batch); walks every 128-step tile of the layer in order.
//
// Loads on tcgen05 kind::i8 with exact integer accumulators: a count h < 4096
// is split into u8 limbs lo = h & 255 and hi16 = 16*(h >> 8) (<= 240); the A
// tile holds [lo | hi16] along K (K = 2E bytes per step row) and the one-hot
// B holds [O | 16*O], so D = sum lo*O + sum 16hi*16O is the load n itself in
// s32 (v3 used fp16 values and fp32 sums: one FADD per load to recover n).
// The epilogue maps n straight to the shared-memory address of its order key:
// GPU g's key row only covers [s_g, U] (s_g = the gather clamp: a load below
// it reads the key at s_g, which never exceeds the step maximum), so
// addr = max(2n + koff_g, base_g) -- LEA + max, one LDS.U16, one max per GPU
// -- and the compressed rows free shared memory for longer load windows.
// KH: the A tile holds E/KH experts (one K part: [lo | hi16] of those
// experts); KH = 2 for E = 256 stages the two halves through the same A
// buffer (two MMA batches into one accumulator), so the B one-hot (K = 2E
// bytes per column) and the key rows fit beside it.
// SPLIT: the key rows do not fit shared memory (G = 32 with wide load
// windows): shared memory holds the first WS keys of every row (uniform
// stride, loads [s_g, s_g + WS)), the full rows [s_g, U] stay in a global
// [G][WG] table (L2) for the rest; each gather is one predicated LDS or LDG.
// Per-GPU key-row constants, passed by value: the unrolled GPU loop reads them
// as constant-bank operands (no registers; at G = 32 two register arrays of
// 32 spilled). Byte offsets relative to the shared key rows:
//   rel = max(KBY*n + koff[g], kbase[g])  -- the clamped key's offset;
//   SPLIT: rel < kend[g] reads shared memory, else the global table at byte
//   offset rel + goff[g].  (KeyRowConsts above.)

// KT: u16 keys, or u32 when the window holds more than 65,536 distinct latencies.
// K5 A operand, once per layer batch: counts h < 4096 as u8 limbs [lo | 16*hi]
// per K part of EH = E/KH experts, rows padded with zeros to a multiple of 128
// steps (limbs[(lb*Tpad + t)*2E + p*2EH + {0, EH} + e - p*EH]); every candidate tile
// of a layer then moves 16-byte chunks instead of converting counts
__global__ void limbs_kernel(const int32_t* __restrict__ hist, int64_t L, int64_t T, int64_t Tpad, int E, int EH,
                             uint8_t* __restrict__ limbs) {
  const int E4 = E / 4;
  const int64_t n = L * Tpad * E4;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / E4;
    const int e = (int)(i - r * E4) * 4;
    const int64_t l = r / Tpad, t = r - l * Tpad;
    int4 h = make_int4(0, 0, 0, 0);
    if (t < T) h = __ldg(reinterpret_cast<const int4*>(hist + (l * T + t) * E + e));
    const uint32_t lo = (uint32_t)(h.x & 255) | ((uint32_t)(h.y & 255) << 8) | ((uint32_t)(h.z & 255) << 16) |
                        ((uint32_t)(h.w & 255) << 24);
    const uint32_t hi = (uint32_t)((h.x >> 8) << 4) | ((uint32_t)((h.y >> 8) << 4) << 8) |
                        ((uint32_t)((h.z >> 8) << 4) << 16) | ((uint32_t)((h.w >> 8) << 4) << 24);
    const int p = e / EH, eo = e - p * EH;
    uint8_t* row = limbs + r * (2 * E) + p * 2 * EH;
    *reinterpret_cast<uint32_t*>(row + eo) = lo;
    *reinterpret_cast<uint32_t*>(row + EH + eo) = hi;
  }
}

// key gathers: volatile under SKIP so they stay inside their warp-uniform
// branch (not speculated above it); free to schedule otherwise
#define GEM_KEY_LD(...)                 \
  do {                                  \
    if constexpr (SKIP)                 \
      asm volatile(__VA_ARGS__);        \
    else                                \
      asm(__VA_ARGS__);                 \
  } while (0)

// SKIP: step floors (floor_tab [L][T] = {skip level, floor key}, see
// floor_table_kernel): a GPU column is gathered only when one of the warp's 32
// steps has its load above the step's skip level.
template <int E, int G, int KH, bool SPLIT, typename KT, int NW, bool SKIP>
__global__ void __launch_bounds__(NW * 32, 1)
maxkey_tc_kernel(const uint8_t* __restrict__ limbs, int64_t T, const int8_t* __restrict__ cand, int64_t C,
                 int64_t L, int64_t layer0, int64_t Cp, const KT* __restrict__ gkeys, int keys_total,
                 const __grid_constant__ KeyRowConsts kr, int WS, int WG, const int2* __restrict__ floor_tab,
                 KT* __restrict__ out_keys) {
  constexpr int KBY = (int)sizeof(KT);       // bytes per key
  constexpr int EH = E / KH;                 // experts per K part
  constexpr int KBH = 2 * EH;                // K bytes per step row per part: [lo | hi16]
  constexpr int KCH = KBH / 16;              // 16-byte K chunks per part
  constexpr uint32_t LBO_A = 128 * 16 + 16;  // A: [KCH][128 rows][16 B], K slices padded by 16 B (bank spread)
  constexpr uint32_t LBO_B = kLtN * 16;      // B: [KH][KCH][N rows][16 B]
  constexpr int A_BYTES = (int)LBO_A * KCH;
  constexpr int B_BYTES = kLtN * KBH * KH;
  constexpr int CT = kLtN / G;               // candidates per CTA
  constexpr int NQ = NW / 4;                 // column groups (warps per TMEM lane quarter)
  constexpr int NT = NW * 32;                // threads
  constexpr int KPT = CT / NQ;               // keys per thread per tile (one column group)
  constexpr int CPL = 32 / G;                // candidates per 32-column TMEM load
  constexpr int STG_ROW = KPT * KBY + 16;    // staging row: the thread's keys + 16 B pad
  constexpr int STG_BYTES = NW * 32 * STG_ROW;
  static_assert(STG_BYTES <= A_BYTES, "key staging size (the host reserves it after the key rows)");
  static_assert(G >= 4 && G <= 32 && (kLtN % G) == 0, "G in {4, 8, 16, 32}");
  static_assert(EH == 64 || EH == 128, "K parts of 64 or 128 experts");
  constexpr int KPP = 16 / KBY;              // keys per 16-byte piece
  extern __shared__ __align__(1024) unsigned char lt_smem[];
  unsigned char* sa = lt_smem;
  unsigned char* sb = lt_smem + A_BYTES;
  LoadsTcShared* sh = reinterpret_cast<LoadsTcShared*>(sb + B_BYTES);
  KT* skeys = reinterpret_cast<KT*>(sb + B_BYTES + 64 + 256);  // packed key rows (SPLIT: [G][WS])
  // key staging: the bytes after the key rows (the next tile's MMAs use the A tile)
  unsigned char* stg = reinterpret_cast<unsigned char*>(skeys) +
                       (SPLIT ? (size_t)G * WS * KBY : (((size_t)keys_total * KBY + 15) & ~size_t(15)));

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t c0 = (int64_t)blockIdx.x * CT;
  const int64_t lb = blockIdx.y;  // layer within the batch
  const int64_t l = layer0 + lb;
  const int64_t Tpad = (T + 127) / 128 * 128;
  const uint8_t* al = limbs + lb * Tpad * (2 * E);  // this layer's A rows (limbs of the batch)
  KT* out = out_keys + lb * T * Cp;

  if (tid == 0) {
    tc::mbar_init(&sh->mma_bar, 1);
    tc::fence_mbar_init();
  }
  if (warp == 0) tc::tmem_alloc<2 * kLtN>(&sh->tmem_base);  // two accumulators (MMA/epilogue overlap)
  if (!SPLIT) {  // key rows -> shared memory (16-byte pieces; the global copy is padded to 16 bytes)
    const int pieces = (keys_total * KBY + 15) / 16;
    for (int i = tid; i < pieces; i += NT)
      reinterpret_cast<uint4*>(skeys)[i] = __ldg(reinterpret_cast<const uint4*>(gkeys) + i);
  } else {  // the first WS keys of every [G][WG] row (WS, WG multiples of 8)
    const int pr = WS / KPP;
    for (int i = tid; i < G * pr; i += NT) {
      const int g = i / pr, q = i - g * pr;
      reinterpret_cast<uint4*>(skeys)[i] = __ldg(reinterpret_cast<const uint4*>(gkeys + (int64_t)g * WG) + q);
    }
  }
  // one-hot B: row r = j*G + g (candidate j of the tile, GPU g); in K part p,
  // chunk q < EH/16 holds experts p*EH + 16q.. as 1, chunk q >= EH/16 the
  // same experts as 16
  for (int i = tid; i < kLtN * KCH * KH; i += NT) {
    const int r = i / (KCH * KH), qq = i % (KCH * KH);
    const int part = qq / KCH, q = qq % KCH;
    uint32_t w[4] = {0u, 0u, 0u, 0u};
    const int j = r / G, g = r % G;
    const bool hiq = q >= EH / 16;
    const int e0 = part * EH + (hiq ? q - EH / 16 : q) * 16;
    const uint32_t one = hiq ? 16u : 1u;
    if (c0 + j < C) {
      const int8_t* m = cand + ((c0 + j) * L + l) * E + e0;
#pragma unroll
      for (int x = 0; x < 16; ++x)
        if (m[x] == g) w[x >> 2] |= one << ((x & 3) * 8);
    }
    *reinterpret_cast<uint4*>(sb + (size_t)qq * LBO_B + (size_t)r * 16) = make_uint4(w[0], w[1], w[2], w[3]);
  }
  tc::fence_async_smem();
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = sh->tmem_base;
  const uint32_t sa_addr = tc::smem_u32(sa), sb_addr = tc::smem_u32(sb);
  const uint32_t idesc = tc::instr_desc(/*S32*/ 2, /*u8*/ 0, /*u8*/ 0, 128, kLtN);
  const int ntiles = (int)((T + 127) / 128);
  const int lg = warp & 3, cg = warp >> 2;
  const uint32_t sk_addr = tc::smem_u32(skeys);
  const char* gk_bytes = reinterpret_cast<const char*>(gkeys);

  // A rows of one K part come precomputed as u8 limbs (limbs_kernel: [batch layers][Tpad][2E],
  // part p = bytes [p*KBH, (p+1)*KBH) of a row, zero rows past T): each lane
  // moves 16-byte K chunks (coalesced rows in, conflict-free padded K slices
  // out); the next part's rows are in flight during the current part's MMA
  // (and epilogue)
  constexpr int RPW = 128 / NW;                  // rows per warp
  constexpr int LPR = KCH;                       // lanes per row (one 16-byte K chunk each)
  constexpr int RPI = 32 / LPR;                  // rows per warp instruction
  constexpr int NX = RPW / RPI;
  static_assert(RPW % RPI == 0, "rows per warp");
  int4 x[NX];
  auto load_rows = [&](int i, int part) {
#pragma unroll
    for (int v = 0; v < NX; ++v) {
      const int row = warp * RPW + v * RPI + lane / LPR;
      x[v] = __ldg(reinterpret_cast<const int4*>(al + ((int64_t)i * 128 + row) * (2 * E) + part * KBH) +
                   (lane % LPR));
    }
  };
  auto write_a = [&]() {
#pragma unroll
    for (int v = 0; v < NX; ++v) {
      const int row = warp * RPW + v * RPI + lane / LPR;
      *reinterpret_cast<int4*>(sa + (size_t)(lane % LPR) * LBO_A + (size_t)row * 16) = x[v];
    }
    tc::fence_async_smem();
  };
  auto issue_mma = [&](int part, uint32_t col) {
    if (tid == 0) {
      tc::tc_fence_after();
#pragma unroll
      for (int k = 0; k < KBH / 32; ++k) {
        const uint64_t ad = tc::smem_desc(sa_addr + k * 2 * LBO_A, LBO_A, 128);
        const uint64_t bd = tc::smem_desc(sb_addr + (part * KCH + k * 2) * LBO_B, LBO_B, 128);
        tc::mma_i8(tmem + col, ad, bd, idesc, (part > 0 || k > 0) ? 1u : 0u);
      }
      tc::mma_commit(&sh->mma_bar);
    }
  };
  uint32_t mma_phase = 0;
  load_rows(0, 0);
  const int2* fl_l = SKIP ? floor_tab + l * T : nullptr;
  auto step_floor = [&](int i) {  // this lane's step (TMEM lane): {skip level, floor key}
    int2 fl = make_int2(INT32_MAX, 0);
    if constexpr (SKIP) {
      const int64_t ts = (int64_t)i * 128 + lg * 32 + lane;
      if (ts < T) fl = __ldg(fl_l + ts);
    }
    return fl;
  };
  auto mma_wait = [&]() {
    tc::mbar_wait(&sh->mma_bar, mma_phase);
    mma_phase ^= 1u;
    tc::tc_fence_after();
  };
  // ---- epilogue of tile i from TMEM columns [tcol, tcol + kLtN): warp w drains
  // TMEM lanes 32(w%4).. (one step per lane) and column group w/4 in 32-column
  // chunks; load n of GPU g -> key; the maximum over a candidate's G columns is
  // its step key. mid() runs after the first chunk.
  auto epilogue = [&](int i, uint32_t tcol, const int2 fl, auto&& mid) {
      {
        const uint32_t trow = tmem + tcol + ((uint32_t)(lg * 32) << 16);
        uint32_t kk[KPT];
  #pragma unroll
        for (int ch = 0; ch < kLtN / NQ / 32; ++ch) {
          uint32_t v[32];
          tc::tmem_ld32(trow + cg * (kLtN / NQ) + ch * 32, v);
          tc::tmem_ld_wait();
  #pragma unroll
          for (int j = 0; j < CPL; ++j) {
            auto gather = [&](int g) -> uint32_t {
              uint32_t key;
              const int32_t rel = max((int32_t)v[j * G + g] * KBY + kr.koff[g], kr.kbase[g]);
              const uint32_t sak = sk_addr + (uint32_t)rel;
              if (!SPLIT && SKIP) {  // lanes at or below their step's skip level load nothing (key 0)
                const uint32_t need = (int32_t)v[j * G + g] > fl.x ? 1u : 0u;
                if constexpr (KBY == 2) {
                  uint16_t k16;
                  GEM_KEY_LD("{\n\t.reg .pred pn;\n\tsetp.ne.u32 pn, %2, 0;\n\tmov.u16 %0, 0;\n\t"
                             "@pn ld.shared.u16 %0, [%1];\n\t}" : "=h"(k16) : "r"(sak), "r"(need));
                  key = k16;
                } else {
                  GEM_KEY_LD("{\n\t.reg .pred pn;\n\tsetp.ne.u32 pn, %2, 0;\n\tmov.u32 %0, 0;\n\t"
                             "@pn ld.shared.u32 %0, [%1];\n\t}" : "=r"(key) : "r"(sak), "r"(need));
                }
              } else if (!SPLIT) {
                if constexpr (KBY == 2) {
                  uint16_t k16;
                  GEM_KEY_LD("ld.shared.u16 %0, [%1];" : "=h"(k16) : "r"(sak));
                  key = k16;
                } else {
                  GEM_KEY_LD("ld.shared.u32 %0, [%1];" : "=r"(key) : "r"(sak));
                }
              } else if constexpr (SKIP) {
                // a lane whose own load is at or below its step's skip level
                // cannot raise the maximum and loads nothing (key 0): most lanes
                // of a gathered column, whose load would often miss the shared
                // rows and go to L2
                const char* ga = gk_bytes + (rel + kr.goff[g]);
                const uint32_t need = (int32_t)v[j * G + g] > fl.x ? 1u : 0u;
                if constexpr (KBY == 2) {
                  uint16_t k16;
                  GEM_KEY_LD("{\n\t.reg .pred pw, pn, ps, pg;\n\tsetp.lt.s32 pw, %1, %2;\n\t"
                      "setp.ne.u32 pn, %5, 0;\n\tand.pred ps, pw, pn;\n\tand.pred pg, !pw, pn;\n\t"
                      "mov.u16 %0, 0;\n\t@ps ld.shared.u16 %0, [%3];\n\t@pg ld.global.nc.u16 %0, [%4];\n\t}"
                      : "=h"(k16)
                      : "r"(rel), "r"(kr.kend[g]), "r"(sak), "l"(ga), "r"(need));
                  key = k16;
                } else {
                  GEM_KEY_LD("{\n\t.reg .pred pw, pn, ps, pg;\n\tsetp.lt.s32 pw, %1, %2;\n\t"
                      "setp.ne.u32 pn, %5, 0;\n\tand.pred ps, pw, pn;\n\tand.pred pg, !pw, pn;\n\t"
                      "mov.u32 %0, 0;\n\t@ps ld.shared.u32 %0, [%3];\n\t@pg ld.global.nc.u32 %0, [%4];\n\t}"
                      : "=r"(key)
                      : "r"(rel), "r"(kr.kend[g]), "r"(sak), "l"(ga), "r"(need));
                }
              } else {
                const char* ga = gk_bytes + (rel + kr.goff[g]);
                if constexpr (KBY == 2) {
                  uint16_t k16;
                  GEM_KEY_LD("{\n\t.reg .pred p;\n\tsetp.lt.s32 p, %1, %2;\n\t"
                      "@p ld.shared.u16 %0, [%3];\n\t@!p ld.global.nc.u16 %0, [%4];\n\t}"
                      : "=h"(k16)
                      : "r"(rel), "r"(kr.kend[g]), "r"(sak), "l"(ga));
                  key = k16;
                } else {
                  GEM_KEY_LD("{\n\t.reg .pred p;\n\tsetp.lt.s32 p, %1, %2;\n\t"
                      "@p ld.shared.u32 %0, [%3];\n\t@!p ld.global.nc.u32 %0, [%4];\n\t}"
                      : "=r"(key)
                      : "r"(rel), "r"(kr.kend[g]), "r"(sak), "l"(ga));
                }
              }
              return key;
            };
            uint32_t m = 0u;
            if constexpr (SKIP) {
              // warp-uniform set of the GPU columns with a load above the skip
              // level in any of the warp's 32 steps; their gathers are issued
              // back to back (the maximum is taken after the last one)
              uint32_t kx[G];
  #pragma unroll
              for (int g = 0; g < G; ++g)
                kx[g] = __any_sync(0xffffffffu, (int32_t)v[j * G + g] > fl.x) ? gather(g) : 0u;
              m = (uint32_t)fl.y;
  #pragma unroll
              for (int g = 0; g < G; ++g) m = max(m, kx[g]);
            } else {
  #pragma unroll
              for (int g = 0; g < G; ++g) m = max(m, gather(g));
            }
            kk[ch * CPL + j] = m;
          }
          if (ch == 0) mid();
        }
        // stage the keys (the A tile's space once its MMAs completed; a separate
        // buffer when the next tile's MMAs run under this epilogue), then store rows
        // of KPT keys per step, 16-byte pieces
        unsigned char* wst = stg + warp * 32 * STG_ROW;
        __syncwarp();  // the warp's reads of its staging rows (previous tile) are done
        if constexpr (KBY == 2) {
  #pragma unroll
          for (int x8 = 0; x8 < KPT / 8; ++x8)
            *reinterpret_cast<uint4*>(wst + lane * STG_ROW + x8 * 16) =
                make_uint4(kk[8 * x8] | (kk[8 * x8 + 1] << 16), kk[8 * x8 + 2] | (kk[8 * x8 + 3] << 16),
                           kk[8 * x8 + 4] | (kk[8 * x8 + 5] << 16), kk[8 * x8 + 6] | (kk[8 * x8 + 7] << 16));
          if (KPT % 8 == 4)
            *reinterpret_cast<uint2*>(wst + lane * STG_ROW + (KPT / 8) * 16) =
                make_uint2(kk[KPT - 4] | (kk[KPT - 3] << 16), kk[KPT - 2] | (kk[KPT - 1] << 16));
          if (KPT == 2) *reinterpret_cast<uint32_t*>(wst + lane * STG_ROW) = kk[0] | (kk[1] << 16);
        } else {
  #pragma unroll
          for (int x4 = 0; x4 < KPT / 4; ++x4)
            *reinterpret_cast<uint4*>(wst + lane * STG_ROW + x4 * 16) =
                make_uint4(kk[4 * x4], kk[4 * x4 + 1], kk[4 * x4 + 2], kk[4 * x4 + 3]);
          if (KPT == 2) *reinterpret_cast<uint2*>(wst + lane * STG_ROW) = make_uint2(kk[0], kk[1]);
        }
        __syncwarp();
        const int64_t tbase = (int64_t)i * 128 + lg * 32;
        const int64_t cbase = c0 + cg * KPT;
        if constexpr (KPT >= KPP) {
          constexpr int PPR = KPT / KPP;  // 16-byte pieces per row
          for (int q = lane; q < 32 * PPR; q += 32) {
            const int r = q / PPR, piece = q % PPR;
            const int64_t t = tbase + r;
            if (t < T)
              *reinterpret_cast<uint4*>(out + t * Cp + cbase + piece * KPP) =
                  *reinterpret_cast<const uint4*>(wst + r * STG_ROW + piece * 16);
          }
        } else if constexpr (KPT * KBY == 8) {  // one 8-byte piece per row
          const int64_t t = tbase + lane;
          if (t < T)
            *reinterpret_cast<uint2*>(out + t * Cp + cbase) = *reinterpret_cast<const uint2*>(wst + lane * STG_ROW);
        } else {  // u16, KPT == 2: one 4-byte piece per row
          static_assert(KPT * KBY == 4, "key row pieces of 4, 8 or 16k bytes");
          const int64_t t = tbase + lane;
          if (t < T)
            *reinterpret_cast<uint32_t*>(out + t * Cp + cbase) = *reinterpret_cast<const uint32_t*>(wst + lane * STG_ROW);
        }
      }
  };
  // tile i+1's MMAs run under tile i's epilogue (the epilogue's gathers are the
  // long part): TMEM double-buffered (2 x kLtN columns), part 0 issued before
  // it, part 1 (E = 256) after its first chunk; keys staged in a buffer of their
  // own (the A tile is busy)
  {
#pragma unroll
    for (int part = 0; part < KH; ++part) {  // tile 0 into columns [0, kLtN)
      write_a();
      __syncthreads();
      issue_mma(part, 0);
      if (part + 1 < KH) load_rows(0, part + 1);
      else if (ntiles > 1) load_rows(1, 0);
      mma_wait();
      if (part + 1 < KH) {
        tc::tc_fence_before();
        __syncthreads();
      }
    }
    for (int i = 0; i < ntiles; ++i) {
      const int2 fl = step_floor(i);
      const uint32_t cur = (uint32_t)(i & 1) * kLtN, nxt = cur ^ (uint32_t)kLtN;
      const bool more = i + 1 < ntiles;
      if (more) {
        write_a();  // rows (i+1, part 0); the A buffer's last MMA completed
        __syncthreads();
        issue_mma(0, nxt);
        if (KH == 2) load_rows(i + 1, 1);
        else if (i + 2 < ntiles) load_rows(i + 2, 0);
      }
      epilogue(i, cur, fl, [&] {
        if (KH == 2 && more) {
          mma_wait();  // part 0 of tile i+1: the A buffer is free
          tc::tc_fence_before();
          write_a();
          __syncthreads();
          issue_mma(1, nxt);
          if (i + 2 < ntiles) load_rows(i + 2, 0);
        }
      });
      if (more) mma_wait();  // the last part of tile i+1
      // no barrier here: the next iteration's first __syncthreads (before tile
      // i+2's MMA into columns cur) follows every warp's reads of them, and each
      // warp's key staging area is its own
      tc::tc_fence_before();
    }
  }
  __syncthreads();  // every warp's last TMEM reads precede the dealloc
  tc::tc_fence_after();
  if (warp == 0) tc::tmem_dealloc<2 * kLtN>(tmem);
}

// ---------------------------------------------------------------------------
// pass 2: thread = (4 consecutive candidates, layer of the batch), four
// serial chains over t; one 8-byte load carries the 4 step keys (Cp is a
// multiple of 8: candidate tiles are 256/G >= 8 wide). vals[0, kSumSmemVals)
// sits in shared memory (99.9% of step maxima at C4 rank below 8,192); a
// miss goes to L2 on the chain's critical path.
// four 4-key groups of a step: u16 keys in 8 bytes, u32 keys in 16
template <typename KT> struct Key4;
template <> struct Key4<uint16_t> {
  using V = uint2;
  __device__ static uint32_t get(const V& v, int j) {
    const uint32_t w = j < 2 ? v.x : v.y;
    return (j & 1) ? (w >> 16) : (w & 0xffffu);
  }
  __device__ static V zero() { return make_uint2(0u, 0u); }
};
template <> struct Key4<uint32_t> {
  using V = uint4;
  __device__ static uint32_t get(const V& v, int j) { return j == 0 ? v.x : j == 1 ? v.y : j == 2 ? v.z : v.w; }
  __device__ static V zero() { return make_uint4(0u, 0u, 0u, 0u); }
};

template <typename KT>
__global__ void __launch_bounds__(kSumThreads, kSumCtasPerSm)
keysum_kernel(const KT* __restrict__ keys, int64_t T, int64_t C, int64_t Cp, int64_t L, int64_t layer0,
              const double* __restrict__ vals, const int32_t* __restrict__ nvals, const int32_t* __restrict__ vbase,
              double* __restrict__ layer_scores) {
  using K4 = Key4<KT>;
  using V = typename K4::V;
  extern __shared__ double s_vals[];  // [kSumSmemVals]
  // vals[base, base + K) in shared memory: base = the smallest step-floor key
  // when the floors ran (G >= 16: the keys a maximum can take start there), else 0
  const int base = vbase ? *vbase : 0;
  const int K = max(0, min(*nvals - base, kSumSmemVals));
  for (int i = threadIdx.x; i < K; i += blockDim.x) s_vals[i] = vals[base + i];
  __syncthreads();
  const int64_t c0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4;
  const int64_t lb = blockIdx.y;
  if (c0 >= C) return;
  const V* p = reinterpret_cast<const V*>(keys + lb * T * Cp + c0);
  const int64_t stride = Cp / 4;  // V per step
  auto val = [&](uint32_t k) -> double {
    const uint32_t r = k - (uint32_t)base;
    return r < (uint32_t)K ? s_vals[r] : __ldg(vals + k);
  };
  // keys 64 bytes ahead of the serial fp64 chains (which stay in t order):
  // 8 steps of u16 keys, 4 of u32 (8 x 16 bytes spilled under 3 CTAs/SM)
  constexpr int D = sizeof(KT) == 2 ? 8 : 4;
  V q[D];
#pragma unroll
  for (int d = 0; d < D; ++d) q[d] = d < T ? __ldcs(p + (int64_t)d * stride) : K4::zero();
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  int64_t t = 0;
  for (; t + D <= T; t += D) {
#pragma unroll
    for (int d = 0; d < D; ++d) {
      const V k = q[d];
      q[d] = t + D + d < T ? __ldcs(p + (t + D + d) * stride) : K4::zero();
      s0 = dadd(s0, val(K4::get(k, 0)));
      s1 = dadd(s1, val(K4::get(k, 1)));
      s2 = dadd(s2, val(K4::get(k, 2)));
      s3 = dadd(s3, val(K4::get(k, 3)));
    }
  }
  for (int d = 0; t < T; ++t, ++d) {
    const V k = q[d];
    s0 = dadd(s0, val(K4::get(k, 0)));
    s1 = dadd(s1, val(K4::get(k, 1)));
    s2 = dadd(s2, val(K4::get(k, 2)));
    s3 = dadd(s3, val(K4::get(k, 3)));
  }
  const double sv[4] = {s0, s1, s2, s3};
#pragma unroll
  for (int j = 0; j < 4; ++j)
    if (c0 + j < C) layer_scores[(c0 + j) * L + layer0 + lb] = sv[j];
}

// the key staging of one tile (8 warps x 32 steps x KPT keys + pad) must fit the A tile
template <int E, int G, typename KT, int NW>
constexpr bool maxkey_fits() {
  constexpr int KH = E == 256 ? 2 : 1;
  return NW * 32 * ((kLtN / G / (NW / 4)) * (int)sizeof(KT) + 16) <= (128 * 16 + 16) * (2 * (E / KH) / 16);
}

template <int E, typename KT>
static int launch_maxkey(int G, bool split, bool skip, dim3 grid, size_t smem, cudaStream_t st, const uint8_t* limbs,
                         int64_t T, const int8_t* cand, int64_t C, int64_t L, int64_t l0, int64_t Cp,
                         const KT* keys, int keys_total, const KeyRowConsts& kr, int WS, int WG, const int2* fl,
                         KT* out) {
  constexpr int KH = E == 256 ? 2 : 1;
  constexpr int NW = kLtWarps, NWS = kLtWarpsSkip;
  auto pick = [&](auto kern) -> int {
    GEM_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<grid, (skip ? NWS : NW) * 32, smem, st>>>(limbs, T, cand, C, L, l0, Cp, keys, keys_total, kr, WS, WG, fl,
                                                     out);
    GEM_CHECK_LAUNCH("maxkey_tc_kernel");
    return GEM_OK;
  };
  auto pick2 = [&](auto k_full, auto k_split) -> int { return split ? pick(k_split) : pick(k_full); };
  // step floors only where a GPU holds few experts (G >= 16): most GPU columns
  // of a warp's 32 steps then sit below the floor and are skipped
  auto pick4 = [&](auto k_full, auto k_split, auto k_full_skip, auto k_split_skip) -> int {
    return skip ? pick2(k_full_skip, k_split_skip) : pick2(k_full, k_split);
  };
  switch (G) {
    case 4:
      if constexpr (maxkey_fits<E, 4, KT, NW>())
        return pick2(maxkey_tc_kernel<E, 4, KH, false, KT, NW, false>, maxkey_tc_kernel<E, 4, KH, true, KT, NW, false>);
      else return 1;
    case 8:
      if constexpr (maxkey_fits<E, 8, KT, NW>())
        return pick2(maxkey_tc_kernel<E, 8, KH, false, KT, NW, false>, maxkey_tc_kernel<E, 8, KH, true, KT, NW, false>);
      else return 1;
    case 16:
      if constexpr (maxkey_fits<E, 16, KT, NW>() && maxkey_fits<E, 16, KT, NWS>())
        return pick4(maxkey_tc_kernel<E, 16, KH, false, KT, NW, false>, maxkey_tc_kernel<E, 16, KH, true, KT, NW, false>,
                     maxkey_tc_kernel<E, 16, KH, false, KT, NWS, true>, maxkey_tc_kernel<E, 16, KH, true, KT, NWS, true>);
      else return 1;
    default:
      if constexpr (maxkey_fits<E, 32, KT, NW>() && maxkey_fits<E, 32, KT, NWS>())
        return pick4(maxkey_tc_kernel<E, 32, KH, false, KT, NW, false>, maxkey_tc_kernel<E, 32, KH, true, KT, NW, false>,
                     maxkey_tc_kernel<E, 32, KH, false, KT, NWS, true>, maxkey_tc_kernel<E, 32, KH, true, KT, NWS, true>);
      else return 1;
  }
}

}  // namespace gem

using namespace gem;

// The tensor-core scorer. Returns GEM_OK when it ran, 1 when its preconditions
// do not hold (the caller then runs the CUDA-core scorer), <0 on error.
extern "C" int gem_score_batch_tc(const int32_t* hist, int64_t L, int64_t T, int32_t E, int32_t G, const int8_t* cand,
                                  int64_t C, const double* lut, int64_t nmax, double* layer_scores,
                                  int32_t* err_flag, void* stream) {
  (void)err_flag;
  if (!(E == 64 || E == 128 || E == 256) || !(G == 4 || G == 8 || G == 16 || G == 32) || (E == 64 && G == 4))
    return 1;
  if (T < 1 || C < 1 || nmax < 0 || L > 65535) return 1;
  cudaStream_t st = as_stream(stream);
  keep_pool();
  int dev = 0, optin = 0;
  GEM_CHECK_CUDA(cudaGetDevice(&dev));
  GEM_CHECK_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  // stream-ordered scratch, freed on every exit path
  std::vector<void*> scratch;
  struct Free {
    std::vector<void*>& v;
    cudaStream_t s;
    ~Free() {
      for (void* p : v) cudaFreeAsync(p, s);
    }
  } free_all{scratch, st};
  auto alloc = [&](size_t bytes) -> void* {
    void* p = nullptr;
    if (cudaMallocAsync(&p, bytes, st) != cudaSuccess) return nullptr;
    scratch.push_back(p);
    return p;
  };
  // ---- bounds, all on the device, then ONE host sync for the launch geometry:
  // [0] experts per GPU (maxcnt), [1] invalid entry, [2, 2+L) top-maxcnt load bound U[l],
  // [2+L, 2+2L) largest count, [2+2L] smallest step total, [3+2L] bad table flags,
  // [4+2L, 4+2L+G) gather clamp thr_g (value level)
  const int64_t NB = 4 + 2 * L + G;
  int32_t* bnd_d = static_cast<int32_t*>(alloc((size_t)NB * 4));
  if (!bnd_d) return fail_cuda(cudaErrorMemoryAllocation, "gem_score_batch_tc scratch");
  GEM_CHECK_CUDA(cudaMemsetAsync(bnd_d, 0, (size_t)NB * 4, st));
  GEM_CHECK_CUDA(cudaMemsetAsync(bnd_d + 2 + 2 * L, 0x7f, 4, st));  // rowmin starts at 0x7f7f7f7f
  cand_stats_kernel<<<(unsigned)imin64((C * L + 7) / 8, 16 * num_sms()), 256, (size_t)8 * G * 4, st>>>(
      cand, C * L, E, G, bnd_d);
  GEM_CHECK_LAUNCH("cand_stats_kernel");
  const int warps = 8;
  const unsigned tb_grid = (unsigned)imin64((L * T + warps - 1) / warps, 16 * num_sms());
  topn_bound_kernel<<<tb_grid, warps * 32, (size_t)warps * E * 4, st>>>(hist, L, T, E, 1, bnd_d, bnd_d + 2,
                                                                        bnd_d + 2 + L, bnd_d + 2 + 2 * L);
  GEM_CHECK_LAUNCH("topn_bound_kernel");
  lut_bad_kernel<<<(unsigned)imin64(((int64_t)G * (nmax + 1) + 255) / 256, 4096), 256, 0, st>>>(
      lut, G, nmax + 1, bnd_d + 3 + 2 * L);
  GEM_CHECK_LAUNCH("lut_bad_kernel");
  value_clamp_kernel<<<1, 32, 0, st>>>(lut, G, nmax + 1, bnd_d + 2 + 2 * L, bnd_d + 3 + 2 * L, bnd_d + 4 + 2 * L);
  GEM_CHECK_LAUNCH("value_clamp_kernel");
  std::vector<int32_t> bnd((size_t)NB);
  GEM_CHECK_CUDA(cudaMemcpyAsync(bnd.data(), bnd_d, (size_t)NB * 4, cudaMemcpyDeviceToHost, st));
  GEM_CHECK_CUDA(cudaStreamSynchronize(st));  // the only sync when the window has <= 65,536 entries
  if (bnd[1] || (bnd[3 + 2 * L] & 1)) return 1;  // invalid entries / bad table values: the CUDA-core scorer reports them
  int64_t U = 0, hmax = 0;
  for (int64_t l = 0; l < L; ++l) {
    U = imax64(U, bnd[2 + l]);
    hmax = imax64(hmax, bnd[2 + L + l]);
  }
  if (U > nmax || U >= (1 << 20)) return 1;  // table range
  const int W = (int)U + 1;
  if (hmax > 4095) return 1;  // u8 limbs (h < 4096)
  // key rows [s_g, U], s_g = min(thr_g, U): rowinfo [g] = s_g, [G+g] = row offset, [2G] = total
  std::vector<int32_t> packed((size_t)2 * G + 1);
  int npacked = 0, wmax = 0;
  const bool noclamp = std::getenv("GEM_SCORE_NOCLAMP") != nullptr;
  for (int g = 0; g < G; ++g) {
    const int sg = noclamp ? 0 : (int)imin64(imax64(bnd[4 + 2 * L + g], 0), U);
    packed[g] = sg;
    packed[G + g] = npacked;
    npacked += W - sg;
    wmax = wmax > W - sg ? wmax : W - sg;
  }
  packed[2 * G] = npacked;

  // ---- order keys: sort the distinct fp64 values of the rows (only those can be gathered)
  auto* bits = static_cast<unsigned long long*>(alloc((size_t)npacked * 8));
  auto* sorted = static_cast<unsigned long long*>(alloc((size_t)npacked * 8));
  auto* uniq = static_cast<unsigned long long*>(alloc((size_t)npacked * 8));
  auto* nu = static_cast<int32_t*>(alloc(8));  // [0] distinct count
  int32_t* packed_d = static_cast<int32_t*>(alloc(packed.size() * 4));
  if (!bits || !sorted || !uniq || !nu || !packed_d) return fail_cuda(cudaErrorMemoryAllocation, "gem_score_batch_tc keys");
  GEM_CHECK_CUDA(cudaMemsetAsync(nu, 0, 8, st));
  GEM_CHECK_CUDA(cudaMemcpyAsync(packed_d, packed.data(), packed.size() * 4, cudaMemcpyHostToDevice, st));
  row_bits_kernel<<<(unsigned)imin64((npacked + 255) / 256, 4096), 256, 0, st>>>(lut, nmax + 1, G, packed_d, bits);
  GEM_CHECK_LAUNCH("row_bits_kernel");
  size_t t1 = 0, t2 = 0;
  GEM_CHECK_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, t1, bits, sorted, npacked, 0, 64, st));
  GEM_CHECK_CUDA(cub::DeviceSelect::Unique(nullptr, t2, sorted, uniq, nu, npacked, st));
  void* tmp = alloc(t1 > t2 ? t1 : t2);
  if (!tmp) return fail_cuda(cudaErrorMemoryAllocation, "gem_score_batch_tc cub");
  GEM_CHECK_CUDA(cub::DeviceRadixSort::SortKeys(tmp, t1, bits, sorted, npacked, 0, 64, st));
  GEM_CHECK_CUDA(cub::DeviceSelect::Unique(tmp, t2, sorted, uniq, nu, npacked, st));
  bool wide = std::getenv("GEM_SCORE_KEY32") != nullptr;  // tests: force u32 keys
  if (npacked > kMaxKeys) {  // only then can the distinct count exceed the u16 key range (second sync)
    int32_t nk = 0;
    GEM_CHECK_CUDA(cudaMemcpyAsync(&nk, nu, 4, cudaMemcpyDeviceToHost, st));
    GEM_CHECK_CUDA(cudaStreamSynchronize(st));
    if (nk < 1) return 1;
    wide = wide || nk > kMaxKeys;
  }
  if (wide && (G == 4 || (G == 8 && E == 64))) return 1;  // the u32 key staging does not fit the A tile
  const int KBY = wide ? 4 : 2;

  // ---- shared memory: A (one K part of E/KH experts), B (K = 2E), barriers, row info, key rows
  const int KH = E == 256 ? 2 : 1;
  // step floors (G >= 16; GEM_SCORE_NOSKIP turns them off); the kernels stage
  // the step keys in a buffer of their own (the next tile's MMAs use the A tile)
  const bool skip = G >= 16 && !std::getenv("GEM_SCORE_NOSKIP");
  const int nw_launch = skip ? kLtWarpsSkip : kLtWarps;
  const size_t stg_bytes = (size_t)nw_launch * 32 * ((kLtN / G) / (nw_launch / 4) * KBY + 16);
  const size_t fixed =
      (size_t)(128 * 16 + 16) * (2 * (E / KH) / 16) + (size_t)kLtN * 2 * E + 64 + 256 + stg_bytes;
  std::vector<int32_t> rowinfo = packed;
  int keys_total = npacked;
  size_t key_smem = (((size_t)keys_total * KBY) + 15) & ~size_t(15);
  bool split = false;
  int WS = 0, WG = 0;
  if (fixed + key_smem > (size_t)optin || std::getenv("GEM_SCORE_SPLIT")) {
    // rows too long for shared memory: the first WS keys of each row there, all of it in a global [G][WG] table
    split = true;
    WG = (wmax + 7) & ~7;
    const int64_t room = ((int64_t)optin - (int64_t)fixed) / ((int64_t)KBY * G);
    WS = (int)imin64(room & ~int64_t(7), WG);
    if (std::getenv("GEM_SCORE_SPLIT")) WS = (int)imin64(WS, imax64(8, (WG / 4) & ~7));  // tests: force misses
    if (WS < 8) return 1;
    for (int g = 0; g < G; ++g) rowinfo[G + g] = g * WG;
    rowinfo[2 * G] = keys_total = G * WG;
    key_smem = (size_t)G * WS * KBY;
  }
  const size_t lt_smem = fixed + key_smem;
  if (std::getenv("GEM_SCORE_DEBUG")) {  // geometry of the launch, for tools/kbench.py experiments
    fprintf(stderr, "score_tc: U=%lld W=%d npacked=%d wide=%d split=%d WS=%d WG=%d smem=%zu s_g:", (long long)U, W,
            npacked, (int)wide, (int)split, WS, WG, lt_smem);
    for (int g = 0; g < G; ++g) fprintf(stderr, " %d", packed[g]);
    fprintf(stderr, "\n");
  }
  if (lt_smem > (size_t)optin) return 1;
  KeyRowConsts kr{};
  for (int g = 0; g < G; ++g) {
    const int sg = rowinfo[g];
    const int srow = split ? g * WS : rowinfo[G + g];  // row start in shared memory (entries)
    kr.koff[g] = KBY * (srow - sg);                    // KBY*n + koff = offset of key[g][n]
    kr.kbase[g] = KBY * srow;                          // offset of key[g][s_g]
    kr.kend[g] = split ? KBY * (srow + WS) : INT32_MAX;
    kr.goff[g] = split ? KBY * (g * WG) - kr.kbase[g] : 0;  // shared offset -> global byte offset
  }
  void* keys = alloc((((size_t)keys_total * KBY) + 15) & ~size_t(15));
  int32_t* rowinfo_d = static_cast<int32_t*>(alloc(rowinfo.size() * 4));
  if (!keys || !rowinfo_d) return fail_cuda(cudaErrorMemoryAllocation, "gem_score_batch_tc key rows");
  GEM_CHECK_CUDA(cudaMemcpyAsync(rowinfo_d, rowinfo.data(), rowinfo.size() * 4, cudaMemcpyHostToDevice, st));
  // row padding and the tail of the last 16-byte piece are copied to shared memory, never read
  GEM_CHECK_CUDA(cudaMemsetAsync(keys, 0, (((size_t)keys_total * KBY) + 15) & ~size_t(15), st));
  const unsigned kr_grid = (unsigned)imin64((keys_total + 255) / 256, 4096);
  if (wide)
    key_rows_kernel<uint32_t><<<kr_grid, 256, 0, st>>>(lut, nmax + 1, G, W, rowinfo_d, uniq, nu,
                                                        static_cast<uint32_t*>(keys));
  else
    key_rows_kernel<uint16_t><<<kr_grid, 256, 0, st>>>(lut, nmax + 1, G, W, rowinfo_d, uniq, nu,
                                                        static_cast<uint16_t*>(keys));
  GEM_CHECK_LAUNCH("key_rows_kernel");
  const double* vals = reinterpret_cast<const double*>(uniq);  // the bit patterns are the values

  // ---- layer batches: P layers of step keys [P][T][Cp] in flight (<= ~32 GB)
  const int CT = kLtN / G;
  const int64_t ntile = (C + CT - 1) / CT;
  const int64_t Cp = ntile * CT;
  const size_t per_layer = (size_t)T * Cp * KBY;
  int64_t P = imin64((int64_t)(32ull << 30) / (int64_t)per_layer, L);
  if (P < 1) return 1;
  void* kbuf = alloc(per_layer * P);
  if (!kbuf) return fail_cuda(cudaErrorMemoryAllocation, "gem_score_batch_tc key buffer");
  // A rows as u8 limbs, per layer batch (half the batch's histogram bytes),
  // once for all candidate tiles
  const int64_t Tpad = (T + 127) / 128 * 128;
  uint8_t* limbs = static_cast<uint8_t*>(alloc((size_t)P * Tpad * 2 * E));
  if (!limbs) return fail_cuda(cudaErrorMemoryAllocation, "gem_score_batch_tc limbs");
  // step floors: {skip level, floor key} per load level h in [0, W), then per
  // step of every layer
  int2* floors = nullptr;
  int32_t* kmin = nullptr;
  if (skip) {
    int2* ftab = static_cast<int2*>(alloc((size_t)W * 8));
    floors = static_cast<int2*>(alloc((size_t)L * T * 8));
    kmin = static_cast<int32_t*>(alloc(4));
    if (!ftab || !floors || !kmin) return fail_cuda(cudaErrorMemoryAllocation, "gem_score_batch_tc step floors");
    GEM_CHECK_CUDA(cudaMemsetAsync(kmin, 0x7f, 4, st));
    if (wide)
      floor_table_kernel<uint32_t><<<(W + 127) / 128, 128, 0, st>>>(lut, nmax + 1, G, W, bnd_d + 3 + 2 * L,
                                                                   static_cast<const uint32_t*>(keys), kr, ftab);
    else
      floor_table_kernel<uint16_t><<<(W + 127) / 128, 128, 0, st>>>(lut, nmax + 1, G, W, bnd_d + 3 + 2 * L,
                                                                   static_cast<const uint16_t*>(keys), kr, ftab);
    GEM_CHECK_LAUNCH("floor_table_kernel");
    step_floor_kernel<<<(unsigned)imin64((L * T + 7) / 8, 32 * num_sms()), 256, 0, st>>>(hist, L * T, E, W, ftab,
                                                                                         floors, kmin);
    GEM_CHECK_LAUNCH("step_floor_kernel");
  }
  auto run = [&](auto kt) -> int {
    using KT = decltype(kt);
    auto ks = keysum_kernel<KT>;
    GEM_CHECK_CUDA(cudaFuncSetAttribute(ks, cudaFuncAttributeMaxDynamicSharedMemorySize, kSumSmemVals * 8));
    GEM_CHECK_CUDA(cudaFuncSetAttribute(ks, cudaFuncAttributePreferredSharedMemoryCarveout,
                                        cudaSharedmemCarveoutMaxShared));  // 3 CTAs x 64 KB per SM
    const KT* kt_keys = static_cast<const KT*>(keys);
    KT* kt_buf = static_cast<KT*>(kbuf);
    for (int64_t l0 = 0; l0 < L; l0 += P) {
      const int64_t nb = imin64(P, L - l0);
      const dim3 g1((unsigned)ntile, (unsigned)nb);
      limbs_kernel<<<(unsigned)imin64((nb * Tpad * (E / 4) + 255) / 256, 32 * num_sms()), 256, 0, st>>>(
          hist + l0 * T * E, nb, T, Tpad, E, E == 256 ? 128 : E, limbs);
      GEM_CHECK_LAUNCH("limbs_kernel");
      const int rc =
          E == 256 ? launch_maxkey<256, KT>(G, split, skip, g1, lt_smem, st, limbs, T, cand, C, L, l0, Cp, kt_keys,
                                            keys_total, kr, WS, WG, floors, kt_buf)
          : E == 128 ? launch_maxkey<128, KT>(G, split, skip, g1, lt_smem, st, limbs, T, cand, C, L, l0, Cp, kt_keys,
                                              keys_total, kr, WS, WG, floors, kt_buf)
                     : launch_maxkey<64, KT>(G, split, skip, g1, lt_smem, st, limbs, T, cand, C, L, l0, Cp, kt_keys,
                                             keys_total, kr, WS, WG, floors, kt_buf);
      if (rc) return rc;
      // CTA size with the fullest last wave (3 CTAs per SM, shared-memory
      // limited): at C4 940 CTAs of 256 = 2.12 waves, 1316 of 192 = 2.96
      int bs = kSumThreads;
      double best = -1.0;
      for (int cand_bs = kSumThreads; cand_bs >= 128; cand_bs -= 64) {
        const double waves = (double)(((C + 4 * cand_bs - 1) / (4 * cand_bs)) * nb) / ((double)kSumCtasPerSm * num_sms());
        const double eff = waves / std::ceil(waves);
        if (eff > best + 0.02) best = eff, bs = cand_bs;
      }
      ks<<<dim3((unsigned)((C + 4 * bs - 1) / (4 * bs)), (unsigned)nb), bs, (size_t)kSumSmemVals * 8, st>>>(
          kt_buf, T, C, Cp, L, l0, vals, nu, kmin, layer_scores);
      GEM_CHECK_LAUNCH("keysum_kernel");
    }
    return GEM_OK;
  };
  const int rc = wide ? run(uint32_t{}) : run(uint16_t{});
  if (rc) return rc;
  return GEM_OK;
}
