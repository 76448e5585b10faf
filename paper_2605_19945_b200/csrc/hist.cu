// K1: router top-k ids -> per-step expert histograms (sm_100a).
//
// The reference starts from counts (trace.py:24-45); this is the ingestion
// step that produces them. Bytes dominate: every id is read once (int16/int32,
// 128-bit streaming loads) and every histogram cell is written once, so the
// kernel is sized against HBM bandwidth.
//
// Counting: each warp owns a work unit of up to kHistStepsPerUnit consecutive
// steps of one layer and keeps 32 lane-private sub-histograms in shared
// memory, laid out bin-major / lane-minor (word = bin*32 + lane), so lane L
// always touches bank L: increments never conflict and never contend, and a
// shared atomic without return carries no dependency chain. Both int16 ids of
// a 32-bit word are clamped with one __vminu2 to an overflow row (which counts
// ids outside [0,E)), so the inner loop is branch-free: ~3.5 instructions per
// id. Once per step the rows are reduced with conflict-free 128-bit reads and
// written coalesced; per-expert totals and active-step counts accumulate in
// registers and are flushed with one atomic per expert per unit. E > 160 uses
// u16x2 counters (two bins per word) to halve shared memory.
#include <cstdlib>

#include "gem_common.cuh"
#include "tc.cuh"

namespace gem {

constexpr int kHistWarps = 4;

// "heavy" step of an expert: it received at least its fair share of the
// step's routed ids, h * E >= row total (exact integers; h > 0 so an empty
// step counts for nobody). Feeds the consistent-expert predicate of K3b.
__device__ __forceinline__ uint32_t is_heavy(uint32_t h, uint32_t E, uint32_t row_total) {
  return (h > 0 && (uint64_t)h * E >= (uint64_t)row_total) ? 1u : 0u;
}
constexpr int kHistStepsPerUnit = 32;
constexpr int kHistUnroll = 8;  // 128-bit loads in flight per lane (x2 with double buffering)

// ---- wide layout (E <= kWideMaxE): one u32 counter per (bin, lane),
//      word = bin*32 + lane; row E is the overflow row for ids >= E.
constexpr int kWideMaxE = 160;

// count the ids held in one 16-byte vector (int16: 8 ids, int32: 4 ids)
template <typename IdT>
__device__ __forceinline__ void count_vec_wide(uint32_t* cnt_lane, const uint4& v, uint32_t E, uint32_t Epair) {
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
  // int16: shared-window byte address of (bin, lane) = lane base + bin*128.
  // The high id of a word m = hi<<16 | lo gives hi*128 = m >> 9 directly
  // (lo <= E < 512 after the clamp, so its bits shift out): 2 instructions
  // for the pair's addresses besides the clamp, one reduction each.
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(cnt_lane);
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    if (sizeof(IdT) == 2) {
      const uint32_t m = __vminu2(w[c], Epair);  // clamp both halves to the overflow row E
      const uint32_t a_lo = base + (__byte_perm(m, 0u, 0x4410) << 7);  // PRMT + LEA
      const uint32_t a_hi = base + (m >> 9);
      asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(a_lo) : "memory");
      asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(a_hi) : "memory");
    } else {
      atomicAdd(cnt_lane + (min(w[c], E) << 5), 1u);
    }
  }
}

// ---- packed layout (any E): two u16 counters per word,
//      word = (bin>>1)*32 + lane; bin E (rounded to its pair) is the overflow bin.
template <typename IdT>
__device__ __forceinline__ void count_vec_packed(uint32_t* cnt_lane, const uint4& v, uint32_t E, uint32_t Epair) {
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    if (sizeof(IdT) == 2) {
      const uint32_t m = __vminu2(w[c], Epair);
      const uint32_t lo = m & 0xffffu, hi = m >> 16;
      atomicAdd(cnt_lane + ((lo >> 1) << 5), 1u << ((lo & 1) << 4));
      atomicAdd(cnt_lane + ((hi >> 1) << 5), 1u << ((hi & 1) << 4));
    } else {
      const uint32_t b = min(w[c], E);
      atomicAdd(cnt_lane + ((b >> 1) << 5), 1u << ((b & 1) << 4));
    }
  }
}

template <typename IdT, bool WIDE>
__device__ __forceinline__ void count_vec(uint32_t* cnt_lane, const uint4& v, uint32_t E, uint32_t Epair) {
  if (WIDE) count_vec_wide<IdT>(cnt_lane, v, E, Epair);
  else count_vec_packed<IdT>(cnt_lane, v, E, Epair);
}

template <bool WIDE>
__device__ __forceinline__ void count_scalar(uint32_t* cnt_lane, uint32_t id, uint32_t E) {
  const uint32_t b = min(id, E);
  if (WIDE) atomicAdd(cnt_lane + (b << 5), 1u);
  else atomicAdd(cnt_lane + ((b >> 1) << 5), 1u << ((b & 1) << 4));
}

// One warp = one work unit = up to kHistStepsPerUnit consecutive steps of one
// layer. MAXR = histogram rows owned per lane in the reduction (rows/32).
template <typename IdT, bool WIDE, int MAXR>
__global__ void __launch_bounds__(kHistWarps * 32, WIDE ? 3 : 2)
topk_hist_kernel(const IdT* __restrict__ ids, int64_t L, int64_t N, int k, int B, int E, int64_t T, int64_t HT,
                 int32_t* __restrict__ hist, int64_t* __restrict__ colsum, int32_t* __restrict__ active,
                 int32_t* __restrict__ heavy, int64_t* __restrict__ dropped_out) {
  extern __shared__ __align__(16) uint32_t hsm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // counter rows: WIDE: E bins + 1 overflow row; packed: ceil((E+1)/2) pair rows
  const int rows = WIDE ? E + 1 : (E + 2) / 2;
  uint32_t* cnt = hsm + (size_t)warp * rows * 32;
  uint32_t* cnt_lane = cnt + lane;
  for (int w = lane; w < rows * 32; w += 32) cnt[w] = 0;
  __syncwarp();
  const uint32_t uE = (uint32_t)E;
  const uint32_t Epair = uE | (uE << 16);
  const int hrows = WIDE ? E : E / 2;  // reduced rows that hold real bins (packed: full pairs)

  const int64_t units_per_layer = (T + kHistStepsPerUnit - 1) / kHistStepsPerUnit;
  const int64_t total_units = L * units_per_layer;
  const int64_t gwarp = (int64_t)blockIdx.x * kHistWarps + warp;
  const int64_t nwarps = (int64_t)gridDim.x * kHistWarps;
  constexpr int BINS = WIDE ? 1 : 2;

  for (int64_t unit = gwarp; unit < total_units; unit += nwarps) {
    const int64_t l = unit / units_per_layer;
    const int64_t t_begin = (unit % units_per_layer) * kHistStepsPerUnit;
    const int64_t t_end = imin64(t_begin + kHistStepsPerUnit, T);
    uint32_t csum[MAXR * BINS], act[MAXR * BINS], hvy[MAXR * BINS];
#pragma unroll
    for (int q = 0; q < MAXR * BINS; ++q) { csum[q] = 0; act[q] = 0; hvy[q] = 0; }
    uint32_t dropped = 0;
    bool t_end_done = false;

    // ---- fast path (wide layout): the unit's ids are one contiguous block, so
    // stream it in 4 KB warp batches with the next batch always in flight
    // (also across step boundaries) and keep CUMULATIVE lane counters: the
    // per-step reduction only reads, and hist = row sum - previous row sum.
    const int64_t step_bytes = (int64_t)B * k * (int64_t)sizeof(IdT);
    const IdT* ubase = ids + (l * N + t_begin * B) * k;
    if (WIDE && step_bytes % (kHistUnroll * 32 * 16) == 0 && t_end * B <= N &&
        (reinterpret_cast<uintptr_t>(ubase) & 15) == 0) {
      const int bps = (int)(step_bytes / (kHistUnroll * 32 * 16));  // batches per step
      const int64_t nb = (t_end - t_begin) * bps;
      const uint4* pv = reinterpret_cast<const uint4*>(ubase) + lane;
      uint32_t prev[MAXR];
#pragma unroll
      for (int q = 0; q < MAXR; ++q) prev[q] = 0;
      uint4 cur[kHistUnroll], nxt[kHistUnroll];
#pragma unroll
      for (int u = 0; u < kHistUnroll; ++u) cur[u] = __ldcs(pv + u * 32);
      int in_step = 0;
      int64_t t = t_begin;
      for (int64_t bt = 0; bt < nb; ++bt) {
        if (bt + 1 < nb) {
          const uint4* q = pv + (bt + 1) * (kHistUnroll * 32);
#pragma unroll
          for (int u = 0; u < kHistUnroll; ++u) nxt[u] = __ldcs(q + u * 32);
        }
#pragma unroll
        for (int u = 0; u < kHistUnroll; ++u) count_vec<IdT, WIDE>(cnt_lane, cur[u], uE, Epair);
        if (++in_step == bps) {
          in_step = 0;
          __syncwarp();
          int32_t* hrow = hist + (l * HT + t) * E;
          uint32_t hq[MAXR], part = 0;
#pragma unroll
          for (int q = 0; q < MAXR; ++q) {
            const int row = lane + q * 32;
            hq[q] = 0;
            if (row < hrows) {
              const uint4* rp = reinterpret_cast<const uint4*>(cnt + row * 32);
              uint32_t sum = 0;
#pragma unroll
              for (int c = 0; c < 8; ++c) {
                const uint4 v = rp[(c + lane) & 7];
                sum += (v.x + v.y) + (v.z + v.w);
              }
              const uint32_t h = sum - prev[q];
              prev[q] = sum;
              hrow[row] = (int32_t)h;
              act[q] += (h > 0);
              hq[q] = h;
              part += h;
            }
          }
          const uint32_t stot = __reduce_add_sync(0xffffffffu, part);
#pragma unroll
          for (int q = 0; q < MAXR; ++q) hvy[q] += is_heavy(hq[q], uE, stot);
          __syncwarp();
          ++t;
        }
#pragma unroll
        for (int u = 0; u < kHistUnroll; ++u) cur[u] = nxt[u];
      }
#pragma unroll
      for (int q = 0; q < MAXR; ++q) csum[q] = prev[q];
      // dropped ids of the whole unit sit in the overflow row; reset all counters
      dropped += cnt[E * 32 + lane];
      __syncwarp();
      for (int w = lane; w < rows * 32; w += 32) cnt[w] = 0;
      __syncwarp();
      t_end_done = true;
    }
    if (!t_end_done)
    for (int64_t t = t_begin; t < t_end; ++t) {
      const int64_t tok0 = t * B;
      const int64_t tok1 = imin64(tok0 + B, N);
      const IdT* p = ids + (l * N + tok0) * k;
      const int64_t cntn = (tok1 - tok0) * k;  // ids in this step
      constexpr int per_vec = 16 / sizeof(IdT);
      int64_t done = 0;
      if ((reinterpret_cast<uintptr_t>(p) & 15) == 0) {
        const int64_t nvec = cntn / per_vec;
        const uint4* pv = reinterpret_cast<const uint4*>(p);
        const int64_t nfull = nvec / (kHistUnroll * 32);  // full batches for the whole warp
        if (nfull > 0) {
          uint4 cur[kHistUnroll], nxt[kHistUnroll];
#pragma unroll
          for (int u = 0; u < kHistUnroll; ++u) cur[u] = __ldcs(pv + lane + u * 32);
          for (int64_t bt = 0; bt < nfull; ++bt) {
            const bool more = bt + 1 < nfull;
            if (more) {
              const uint4* q = pv + (bt + 1) * (kHistUnroll * 32) + lane;
#pragma unroll
              for (int u = 0; u < kHistUnroll; ++u) nxt[u] = __ldcs(q + u * 32);
            }
#pragma unroll
            for (int u = 0; u < kHistUnroll; ++u) count_vec<IdT, WIDE>(cnt_lane, cur[u], uE, Epair);
            if (more) {
#pragma unroll
              for (int u = 0; u < kHistUnroll; ++u) cur[u] = nxt[u];
            }
          }
        }
        for (int64_t v = nfull * (kHistUnroll * 32) + lane; v < nvec; v += 32)
          count_vec<IdT, WIDE>(cnt_lane, __ldcs(pv + v), uE, Epair);
        done = nvec * per_vec;
      }
      for (int64_t i = done + lane; i < cntn; i += 32) {
        const uint32_t id = (sizeof(IdT) == 2) ? (uint32_t)(uint16_t)p[i] : (uint32_t)p[i];
        count_scalar<WIDE>(cnt_lane, id, uE);
      }
      __syncwarp();
      // Reduce the 32 lane-private columns of every row. Lane owns rows
      // lane + 32q and reads them as 8 x 128-bit chunks, chunk (c+lane)&7 in
      // iteration c (4 wavefronts per LDS.128: conflict-free), zeroing as it goes.
      int32_t* hrow = hist + (l * HT + t) * E;
      uint32_t hq[MAXR * BINS], part = 0;
#pragma unroll
      for (int q = 0; q < MAXR * BINS; ++q) hq[q] = 0;
#pragma unroll
      for (int q = 0; q < MAXR; ++q) {
        const int row = lane + q * 32;
        if (row < hrows) {
          uint4* rp = reinterpret_cast<uint4*>(cnt + row * 32);
          uint32_t s = 0;
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const int j = (c + lane) & 7;
            const uint4 v = rp[j];
            s += (v.x + v.y) + (v.z + v.w);
            rp[j] = make_uint4(0u, 0u, 0u, 0u);
          }
          if (WIDE) {
            hrow[row] = (int32_t)s;
            csum[q] += s;
            act[q] += (s > 0);
            hq[q] = s;
            part += s;
          } else {
            const uint32_t lo = s & 0xffffu, hi = s >> 16;
            hrow[2 * row] = (int32_t)lo;  // two stores: with odd E the pair is not 8-byte aligned
            hrow[2 * row + 1] = (int32_t)hi;
            csum[2 * q] += lo;
            csum[2 * q + 1] += hi;
            act[2 * q] += (lo > 0);
            act[2 * q + 1] += (hi > 0);
            hq[2 * q] = lo;
            hq[2 * q + 1] = hi;
            part += lo + hi;
          }
        }
      }
      // overflow: WIDE row E; packed: pair row E/2 (holds bin E-1 in its low
      // half when E is odd, overflow in the high half; overflow alone when E is even)
      {
        const int orow = WIDE ? E : E / 2;
        const uint32_t ov = cnt[orow * 32 + lane];
        cnt[orow * 32 + lane] = 0;
        uint32_t odd = 0;  // packed layout, odd E: bin E-1 sits alone in the overflow pair row
        if (WIDE || (E & 1) == 0) {
          dropped += ov;
        } else {
          dropped += ov >> 16;
          odd = __reduce_add_sync(0xffffffffu, ov & 0xffffu);
        }
        const uint32_t stot = __reduce_add_sync(0xffffffffu, part) + odd;
#pragma unroll
        for (int q = 0; q < MAXR * BINS; ++q) hvy[q] += is_heavy(hq[q], uE, stot);
        if (!WIDE && (E & 1) && lane == 0) {
          hrow[E - 1] = (int32_t)odd;
          if (odd) {
            atomicAdd((unsigned long long*)&colsum[l * E + E - 1], (unsigned long long)odd);
            atomicAdd(&active[l * E + E - 1], 1);
            if (is_heavy(odd, uE, stot)) atomicAdd(&heavy[l * E + E - 1], 1);
          }
        }
      }
      __syncwarp();
    }
    // flush this unit's per-expert totals
#pragma unroll
    for (int q = 0; q < MAXR; ++q) {
      const int row = lane + q * 32;
      if (row >= hrows) continue;
#pragma unroll
      for (int bb = 0; bb < BINS; ++bb) {
        const int bin = row * BINS + bb;
        const uint32_t cs = csum[q * BINS + bb], ac = act[q * BINS + bb], hv = hvy[q * BINS + bb];
        if (cs) atomicAdd((unsigned long long*)&colsum[l * E + bin], (unsigned long long)cs);
        if (ac) atomicAdd(&active[l * E + bin], (int)ac);
        if (hv) atomicAdd(&heavy[l * E + bin], (int)hv);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) dropped += __shfl_xor_sync(0xffffffffu, dropped, o);
    if (lane == 0 && dropped) atomicAdd((unsigned long long*)&dropped_out[l], (unsigned long long)dropped);
  }
}

// ---------------------------------------------------------------------------
// K1 ring variant (int16 ids, wide counters, whole-unit fast path only): one
// warp per CTA, the unit's 4 KB batches staged by cp.async into a
// kRingStages-deep shared-memory ring, so kRingStages-1 batches (12 KB) are in
// flight per warp while it counts -- the register double buffer of the main
// kernel holds one, and its stream stalls on the counting. Every lane counts
// exactly the 16-byte pieces it copied itself, so cp.async.wait_group alone
// orders the ring (no barrier); counting, reduction and flush are the main
// kernel's.
#ifndef GEM_HIST_RING
#define GEM_HIST_RING 5
#endif
#ifndef GEM_RING_UNROLL
#define GEM_RING_UNROLL 4
#endif
constexpr int kRingStages = GEM_HIST_RING;
constexpr int kRingUnroll = GEM_RING_UNROLL;  // 16-byte pieces per lane per batch

__device__ __forceinline__ void ring_cp16(uint32_t saddr, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(saddr), "l"(gmem) : "memory");
}
__device__ __forceinline__ void ring_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void ring_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// ---------------------------------------------------------------------------
// Heavy-step counts from written histogram rows: heavy[l][e] += #steps t with
// h > 0 and h*E >= the step's row total (is_heavy, exact). The ring kernel
// leaves them out of its hot loop (an extra per-bin predicate there cost more
// than this whole pass); this pass re-reads the L*T*E*4 histogram bytes once.
// One warp per row: lane-strided loads (16-byte when E % 4 == 0), a 64-bit
// warp sum, per-lane counters over the CTA's rows, one shared-memory merge and
// one global atomic per expert per CTA.
constexpr int kHeavyRows = 256;   // rows (steps) per CTA
constexpr int kHeavyWarps = 8;

// NJ: 128-expert column blocks (VEC: one int4 per lane per block) or
// 32-expert scalar columns / 4 (!VEC); RU rows in flight per warp.
template <bool VEC, int NJ>
__global__ void __launch_bounds__(kHeavyWarps * 32)
hist_heavy_rows_kernel(const int32_t* __restrict__ hist, int64_t T, int64_t HT, int E, int32_t* __restrict__ heavy) {
  constexpr int RU = 4;
  constexpr int PER = 4 * NJ;  // counters per lane
  extern __shared__ int32_t hsum[];  // [E]
  const int64_t l = blockIdx.y;
  const int64_t t0 = (int64_t)blockIdx.x * kHeavyRows, t1 = imin64(t0 + kHeavyRows, T);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int e = threadIdx.x; e < E; e += blockDim.x) hsum[e] = 0;
  __syncthreads();
  auto col = [&](int j, int i) { return VEC ? (j * 32 + lane) * 4 + i : (4 * j + i) * 32 + lane; };
  uint32_t cnt[PER];
#pragma unroll
  for (int i = 0; i < PER; ++i) cnt[i] = 0;
  for (int64_t tb = t0 + warp * RU; tb < t1; tb += kHeavyWarps * RU) {
    uint32_t h[RU][PER];
#pragma unroll
    for (int r = 0; r < RU; ++r) {
      const int64_t t = tb + r;
      const int32_t* row = hist + (l * HT + t) * E;
#pragma unroll
      for (int j = 0; j < NJ; ++j) {
        if (VEC) {
          const int e = col(j, 0);
          const int4 v = (t < t1 && e < E) ? __ldg(reinterpret_cast<const int4*>(row + e)) : make_int4(0, 0, 0, 0);
          h[r][4 * j] = (uint32_t)v.x; h[r][4 * j + 1] = (uint32_t)v.y;
          h[r][4 * j + 2] = (uint32_t)v.z; h[r][4 * j + 3] = (uint32_t)v.w;
        } else {
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int e = col(j, i);
            h[r][4 * j + i] = (t < t1 && e < E) ? (uint32_t)__ldg(row + e) : 0u;
          }
        }
      }
    }
#pragma unroll
    for (int r = 0; r < RU; ++r) {
      uint64_t part = 0;
#pragma unroll
      for (int i = 0; i < PER; ++i) part += h[r][i];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
#pragma unroll
      for (int i = 0; i < PER; ++i) cnt[i] += (h[r][i] > 0u && (uint64_t)h[r][i] * (uint64_t)E >= part) ? 1u : 0u;
    }
  }
#pragma unroll
  for (int j = 0; j < NJ; ++j)
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int e = col(j, i);
      if (e < E && cnt[4 * j + i]) atomicAdd(&hsum[e], (int)cnt[4 * j + i]);
    }
  __syncthreads();
  for (int e = threadIdx.x; e < E; e += blockDim.x)
    if (hsum[e]) atomicAdd(&heavy[l * E + e], hsum[e]);
}

template <bool VEC, int NJ>
static void heavy_rows_t(dim3 grid, size_t smem, cudaStream_t st, const int32_t* hist, int64_t T, int64_t HT, int E,
                         int32_t* heavy) {
  hist_heavy_rows_kernel<VEC, NJ><<<grid, kHeavyWarps * 32, smem, st>>>(hist, T, HT, E, heavy);
}

static int launch_heavy_rows(const int32_t* hist, int64_t L, int64_t T, int64_t HT, int E, int32_t* heavy,
                             cudaStream_t st) {
  if (L > 65535) {
    set_error("heavy-step counts: more than 65535 layers");
    return GEM_ERR_INVALID;
  }
  const dim3 grid((unsigned)((T + kHeavyRows - 1) / kHeavyRows), (unsigned)L);
  const size_t smem = (size_t)E * sizeof(int32_t);
  if (E % 4 == 0) {
    const int nj = (E + 127) / 128;
    if (nj == 1) heavy_rows_t<true, 1>(grid, smem, st, hist, T, HT, E, heavy);
    else if (nj == 2) heavy_rows_t<true, 2>(grid, smem, st, hist, T, HT, E, heavy);
    else heavy_rows_t<true, 4>(grid, smem, st, hist, T, HT, E, heavy);
  } else {
    const int nj = (E + 127) / 128;
    if (nj == 1) heavy_rows_t<false, 1>(grid, smem, st, hist, T, HT, E, heavy);
    else heavy_rows_t<false, 4>(grid, smem, st, hist, T, HT, E, heavy);
  }
  GEM_CHECK_LAUNCH("hist_heavy_rows_kernel");
  return GEM_OK;
}

// counter rows of the ring kernel: E (+1 overflow) wide rows or E/2 (+1) pair
// rows, padded to the 32*MAXR rows the per-step reduction reads unguarded
template <bool WIDE, int MAXR>
__host__ __device__ constexpr int ring_rows(int E) {
  return (WIDE ? E + 1 : E / 2 + 1) > 32 * MAXR ? (WIDE ? E + 1 : E / 2 + 1) : 32 * MAXR;
}

// WIDE: u32 counters, rows E + 1; packed (even E only): u16x2 counters, pair
// rows E/2 + 1 (row E/2 low half = overflow), halves summed separately in the
// cumulative reduction (a lane's half counts at most B*k <= 65535 per unit).
// HV: count heavy steps in the per-step reduction (row total = warp sum of
// the row differences) instead of a separate pass over the written rows
template <bool WIDE, int MAXR, bool HV>
__global__ void __launch_bounds__(32)
topk_hist_ring_kernel(const int16_t* __restrict__ ids, int64_t L, int64_t N, int k, int B, int E, int64_t T,
                      int64_t HT, int32_t* __restrict__ hist, int64_t* __restrict__ colsum,
                      int32_t* __restrict__ active, int32_t* __restrict__ heavy, int64_t* __restrict__ dropped_out) {
  extern __shared__ __align__(16) uint4 rsm[];
  constexpr int BATCH = kRingUnroll * 32;  // uint4 per warp batch (4 KB)
  const int lane = threadIdx.x;
  uint4* ring = rsm;                                                  // [kRingStages][kRingUnroll][32]
  uint32_t* cnt = reinterpret_cast<uint32_t*>(rsm + kRingStages * BATCH);  // [E + 1][32]
  uint32_t* cnt_lane = cnt + lane;
  const int rows = ring_rows<WIDE, MAXR>(E);  // padded to 32*MAXR
  const int hrows = WIDE ? E : E / 2;  // reduced rows holding real bins
  constexpr int BINS = WIDE ? 1 : 2;
  for (int w = lane; w < rows * 32; w += 32) cnt[w] = 0;
  __syncwarp();
  const uint32_t uE = (uint32_t)E, Epair = uE | (uE << 16);
  const uint32_t ring_base = (uint32_t)__cvta_generic_to_shared(ring) + 16u * (uint32_t)lane;
  const int64_t units_per_layer = (T + kHistStepsPerUnit - 1) / kHistStepsPerUnit;
  const int64_t total_units = L * units_per_layer;
  const int bps = (int)((int64_t)B * k * 2 / (BATCH * 16));  // batches per step (caller checked divisibility)

  for (int64_t unit = blockIdx.x; unit < total_units; unit += gridDim.x) {
    const int64_t l = unit / units_per_layer;
    const int64_t t_begin = (unit % units_per_layer) * kHistStepsPerUnit;
    const int64_t t_end = imin64(t_begin + kHistStepsPerUnit, T);
    const int64_t nb = (t_end - t_begin) * bps;
    const uint4* pv = reinterpret_cast<const uint4*>(ids + (l * N + t_begin * B) * k) + lane;
    auto issue = [&](int64_t b) {
      const uint32_t dst = ring_base + (uint32_t)((b % kRingStages) * BATCH * 16);
#pragma unroll
      for (int u = 0; u < kRingUnroll; ++u) ring_cp16(dst + u * 32 * 16, pv + b * BATCH + u * 32);
    };
#pragma unroll
    for (int sidx = 0; sidx < kRingStages - 1; ++sidx) {
      if (sidx < nb) issue(sidx);
      ring_commit();
    }
    uint32_t prev[MAXR * BINS], act[MAXR * BINS], hvy[MAXR * BINS];
#pragma unroll
    for (int q = 0; q < MAXR * BINS; ++q) { prev[q] = 0; act[q] = 0; hvy[q] = 0; }
    int in_step = 0;
    int64_t t = t_begin;
    for (int64_t bt = 0; bt < nb; ++bt) {
      ring_wait<kRingStages - 2>();  // this lane's copies of batch bt have landed
      // the slot of batch bt-1 (consumed by this lane) takes batch bt+S-1
      if (bt + kRingStages - 1 < nb) issue(bt + kRingStages - 1);
      ring_commit();
      const uint4* cur = ring + (bt % kRingStages) * BATCH + lane;
#pragma unroll
      for (int u = 0; u < kRingUnroll; ++u) count_vec<int16_t, WIDE>(cnt_lane, cur[u * 32], uE, Epair);
      if (++in_step == bps) {
        in_step = 0;
        __syncwarp();
        int32_t* hrow = hist + (l * HT + t) * E;
        // all row sums first (the counter block is padded to 32*MAXR rows, so
        // the loads need no guard and can all be in flight), then the updates
        uint32_t sa[MAXR], sb[MAXR];
#pragma unroll
        for (int q = 0; q < MAXR; ++q) {
          const uint4* rp = reinterpret_cast<const uint4*>(cnt + (lane + q * 32) * 32);
          uint32_t a = 0, b = 0;
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const uint4 v = rp[(c + lane) & 7];
            if (WIDE) {
              a += (v.x + v.y) + (v.z + v.w);
            } else {
              a += ((v.x & 0xffffu) + (v.y & 0xffffu)) + ((v.z & 0xffffu) + (v.w & 0xffffu));
              b += ((v.x >> 16) + (v.y >> 16)) + ((v.z >> 16) + (v.w >> 16));
            }
          }
          sa[q] = a;
          sb[q] = b;
        }
        if (HV && WIDE) {  // the step's row total (the overflow row E holds dropped ids: not counted)
          uint32_t part = 0;
#pragma unroll
          for (int q = 0; q < MAXR; ++q)
            if (lane + q * 32 < hrows) part += sa[q] - prev[q];
          const uint32_t stot = __reduce_add_sync(0xffffffffu, part);
#pragma unroll
          for (int q = 0; q < MAXR; ++q) hvy[q] += is_heavy(sa[q] - prev[q], uE, stot);
        }
#pragma unroll
        for (int q = 0; q < MAXR; ++q) {
          const int row = lane + q * 32;
          if (row < hrows) {
            if (WIDE) {
              const uint32_t h = sa[q] - prev[q];
              prev[q] = sa[q];
              hrow[row] = (int32_t)h;
              act[q] += (h > 0);
            } else {
              const uint32_t hl = sa[q] - prev[2 * q], hh = sb[q] - prev[2 * q + 1];
              prev[2 * q] = sa[q];
              prev[2 * q + 1] = sb[q];
              *reinterpret_cast<int2*>(hrow + 2 * row) = make_int2((int)hl, (int)hh);
              act[2 * q] += (hl > 0);
              act[2 * q + 1] += (hh > 0);
            }
          }
        }
        __syncwarp();
        ++t;
      }
    }
    ring_wait<0>();
    // overflow row: WIDE row E; packed (even E) the low half of pair row E/2
    uint32_t dropped = WIDE ? cnt[E * 32 + lane] : (cnt[(E / 2) * 32 + lane] & 0xffffu);
    __syncwarp();
    for (int w = lane; w < rows * 32; w += 32) cnt[w] = 0;
    dropped = __reduce_add_sync(0xffffffffu, dropped);
    __syncwarp();
#pragma unroll
    for (int q = 0; q < MAXR; ++q) {
      const int row = lane + q * 32;
      if (row >= hrows) continue;
#pragma unroll
      for (int bb = 0; bb < BINS; ++bb) {
        const int bin = row * BINS + bb;
        const uint32_t cs = prev[q * BINS + bb], ac = act[q * BINS + bb];
        if (cs) atomicAdd((unsigned long long*)&colsum[l * E + bin], (unsigned long long)cs);
        if (ac) atomicAdd(&active[l * E + bin], (int)ac);
        if (HV && hvy[q * BINS + bb]) atomicAdd(&heavy[l * E + bin], (int)hvy[q * BINS + bb]);
      }
    }
    if (lane == 0 && dropped) atomicAdd((unsigned long long*)&dropped_out[l], (unsigned long long)dropped);
  }
}

template <bool WIDE, int MAXR>
static int launch_hist_ring(const void* ids, int64_t L, int64_t N, int k, int B, int E, int64_t T, int64_t HT,
                            int32_t* hist, int64_t* colsum, int32_t* active, int32_t* heavy, int64_t* dropped, cudaStream_t st) {
  const int rows = ring_rows<WIDE, MAXR>(E);
  const size_t smem = (size_t)kRingStages * kRingUnroll * 32 * 16 + (size_t)rows * 32 * 4;
  const bool hv = WIDE && !std::getenv("GEM_HIST_HEAVY_PASS");  // heavy steps counted in the ring's reduction
  auto kern = hv ? topk_hist_ring_kernel<WIDE, MAXR, WIDE> : topk_hist_ring_kernel<WIDE, MAXR, false>;
  GEM_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  GEM_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                                      cudaSharedmemCarveoutMaxShared));
  int per_sm = 0;
  GEM_CHECK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32, smem));
  if (per_sm < 1) per_sm = 1;
  const int64_t units = L * ((T + kHistStepsPerUnit - 1) / kHistStepsPerUnit);
  int64_t blocks = (int64_t)num_sms() * per_sm;
  if (blocks > units) blocks = units;
  kern<<<(unsigned)blocks, 32, smem, st>>>((const int16_t*)ids, L, N, k, B, E, T, HT, hist, colsum, active, heavy,
                                           dropped);
  GEM_CHECK_LAUNCH("topk_hist_ring_kernel");
  return hv ? GEM_OK : launch_heavy_rows(hist, L, T, HT, E, heavy, st);
}

// ---------------------------------------------------------------------------
// K1 CTA variant for large E (int16 ids, u32 lane-private counters SHARED by
// the CTA's W warps). At E = 256 the per-step reduction of E x 32 lane
// counters costs as much as the counting, and 32 KB of u32 counters per warp
// (or the u16x2 packing that halves them at ~2x the instructions per id) caps
// a one-warp-per-CTA design at 8 warps per SM. Here W warps count into ONE
// set of lane-private counters -- lane L of every warp always hits bank L, so
// the reductions never conflict, and warps never conflict with each other --
// each warp takes bps/W of a step's 2 KB batches, a named barrier closes the
// step, every warp reduces its 32*R rows (cumulative counters: the reduction
// only reads, hist = row sum - previous row sum) and a second barrier reopens
// the counters. No shared-memory staging of the ids: each lane loads its
// 16-byte pieces straight into registers NB steps ahead (buf rotates with a
// compile-time index: the step loop is unrolled by NB), so W*NB 2 KB batches
// per CTA are in flight through the barriers. (A TMA-bulk-copy ring in
// shared memory was tried first: its copies in and reads out are shared
// wavefronts the counting needs; 4.86 ms vs 3.26 ms at DeepSeek-V3 shape.)
constexpr int kCtaBatch = 2048;  // bytes of one warp's slice of a step (1024 int16 ids)

template <int W, int R, int G, int NB, int BPW, int MINB>
__global__ void __launch_bounds__(W * 32, MINB)
topk_hist_creg_kernel(const int16_t* __restrict__ ids, int64_t L, int64_t N, int k, int B, int E, int64_t T,
                      int64_t HT, int32_t* __restrict__ hist, int64_t* __restrict__ colsum,
                      int32_t* __restrict__ active, int64_t* __restrict__ dropped_out) {
  extern __shared__ __align__(128) uint32_t crs[];
  constexpr int PER = BPW * (kCtaBatch / 16 / 32);  // uint4 per lane per step
  constexpr int D = G * NB;                          // step slots in registers
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rows = (E + 1) > 32 * R * W ? E + 1 : 32 * R * W;
  const int set_words = rows * 32;
  for (int i = threadIdx.x; i < G * set_words; i += W * 32) crs[i] = 0;
  __syncthreads();
  const uint32_t uE = (uint32_t)E, Epair = uE | (uE << 16);
  const int64_t upl = (T + kHistStepsPerUnit - 1) / kHistStepsPerUnit;
  const int64_t total_units = L * upl;
  const int64_t step_vec = (int64_t)B * k / 8;  // uint4 per step
  const int64_t lane_off = (int64_t)warp * BPW * (kCtaBatch / 16) + lane;

  // producer: slots of (unit, step), G per group; slots past the unit's end are empty
  int64_t p_unit = blockIdx.x;
  int p_left = 0, p_j = 0;
  const uint4* p_ptr = nullptr;
  auto p_open = [&]() {
    if (p_unit < total_units) {
      const int64_t l = p_unit / upl, tb = (p_unit % upl) * kHistStepsPerUnit;
      p_left = (int)(imin64(tb + kHistStepsPerUnit, T) - tb);
      p_ptr = reinterpret_cast<const uint4*>(ids + (l * N + tb * B) * k) + lane_off;
    }
  };
  p_open();
  uint4 buf[D][PER];
  auto load_next = [&](uint4 (&b)[PER]) {
    if (p_unit >= total_units) return;
    if (p_left > 0) {
#pragma unroll
      for (int u = 0; u < PER; ++u) b[u] = __ldcs(p_ptr + u * 32);
      p_ptr += step_vec;
      --p_left;
    }
    if (++p_j == G) {
      p_j = 0;
      if (p_left == 0) {
        p_unit += gridDim.x;
        p_open();
      }
    }
  };
#pragma unroll
  for (int d = 0; d < D; ++d) load_next(buf[d]);

  // consumer
  int64_t c_unit = blockIdx.x;
  int64_t c_l = 0, c_t = 0, c_tend = 0;
  auto c_open = [&]() {
    if (c_unit < total_units) {
      c_l = c_unit / upl;
      c_t = (c_unit % upl) * kHistStepsPerUnit;
      c_tend = imin64(c_t + kHistStepsPerUnit, T);
    }
  };
  c_open();
  uint32_t prev[G][R], act[R];
#pragma unroll
  for (int q = 0; q < R; ++q) {
    act[q] = 0;
#pragma unroll
    for (int j = 0; j < G; ++j) prev[j][q] = 0;
  }
  while (c_unit < total_units) {
#pragma unroll
    for (int g = 0; g < NB; ++g) {
      if (c_unit < total_units) {
        const int nvalid = (int)imin64(G, c_tend - c_t);
#pragma unroll
        for (int j = 0; j < G; ++j) {
          if (j < nvalid) {
            uint32_t* cnt_lane = crs + j * set_words + lane;
#pragma unroll
            for (int u = 0; u < PER; ++u) count_vec_wide<int16_t>(cnt_lane, buf[g * G + j][u], uE, Epair);
          }
          load_next(buf[g * G + j]);
        }
        asm volatile("bar.sync 1, %0;" ::"n"(W * 32) : "memory");  // the group's steps counted by every warp
#pragma unroll
        for (int j = 0; j < G; ++j) {
          if (j < nvalid) {
            int32_t* hrow = hist + (c_l * HT + c_t + j) * E;
            uint32_t sa[R];
#pragma unroll
            for (int q = 0; q < R; ++q) {
              const uint4* rp =
                  reinterpret_cast<const uint4*>(crs + j * set_words + ((warp * R + q) * 32 + lane) * 32);
              uint32_t a = 0;
#pragma unroll
              for (int c = 0; c < 8; ++c) {
                const uint4 x = rp[(c + lane) & 7];
                a += (x.x + x.y) + (x.z + x.w);
              }
              sa[q] = a;
            }
#pragma unroll
            for (int q = 0; q < R; ++q) {
              const int row = (warp * R + q) * 32 + lane;
              const uint32_t h = sa[q] - prev[j][q];
              prev[j][q] = sa[q];
              if (row < E) {
                hrow[row] = (int32_t)h;
                act[q] += (h > 0);
              }
            }
          }
        }
        c_t += nvalid;
        if (c_t == c_tend) {  // unit end: dropped ids, per-expert totals, counters reset
          if (warp == 0) {
            uint32_t dd = 0;
#pragma unroll
            for (int j = 0; j < G; ++j) dd += crs[j * set_words + E * 32 + lane];
            dd = __reduce_add_sync(0xffffffffu, dd);
            if (lane == 0 && dd) atomicAdd((unsigned long long*)&dropped_out[c_l], (unsigned long long)dd);
          }
#pragma unroll
          for (int q = 0; q < R; ++q) {
            const int row = (warp * R + q) * 32 + lane;
            uint32_t cs = 0;
#pragma unroll
            for (int j = 0; j < G; ++j) {
              cs += prev[j][q];
              prev[j][q] = 0;
            }
            if (row < E) {
              if (cs) atomicAdd((unsigned long long*)&colsum[c_l * E + row], (unsigned long long)cs);
              if (act[q]) atomicAdd(&active[c_l * E + row], (int)act[q]);
            }
            act[q] = 0;
          }
          asm volatile("bar.sync 1, %0;" ::"n"(W * 32) : "memory");
          for (int i = threadIdx.x; i < G * set_words; i += W * 32) crs[i] = 0;
          c_unit += gridDim.x;
          c_open();
        }
        asm volatile("bar.sync 1, %0;" ::"n"(W * 32) : "memory");  // reads (and resets) done
      }
    }
  }
}

template <int W, int R, int G, int NB, int BPW, int MINB>
static int launch_hist_creg(const void* ids, int64_t L, int64_t N, int k, int B, int E, int64_t T, int64_t HT,
                            int32_t* hist, int64_t* colsum, int32_t* active, int32_t* heavy, int64_t* dropped,
                            cudaStream_t st) {
  const int rows = (E + 1) > 32 * R * W ? E + 1 : 32 * R * W;
  const size_t smem = (size_t)G * rows * 32 * 4;
  auto kern = topk_hist_creg_kernel<W, R, G, NB, BPW, MINB>;
  GEM_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 0;
  GEM_CHECK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, W * 32, smem));
  if (per_sm < 1) per_sm = 1;
  const int64_t units = L * ((T + kHistStepsPerUnit - 1) / kHistStepsPerUnit);
  int64_t blocks = (int64_t)num_sms() * per_sm;
  if (blocks > units) blocks = units;
  kern<<<(unsigned)blocks, W * 32, smem, st>>>((const int16_t*)ids, L, N, k, B, E, T, HT, hist, colsum, active,
                                               dropped);
  GEM_CHECK_LAUNCH("topk_hist_creg_kernel");
  return launch_heavy_rows(hist, L, T, HT, E, heavy, st);
}

template <typename IdT, bool WIDE, int MAXR>
static int launch_hist_t(const void* ids, int64_t L, int64_t N, int k, int B, int E, int64_t T, int64_t HT,
                         int32_t* hist,
                         int64_t* colsum, int32_t* active, int32_t* heavy, int64_t* dropped, cudaStream_t st) {
  const int rows = WIDE ? E + 1 : (E + 2) / 2;
  const size_t smem = (size_t)kHistWarps * rows * 32 * sizeof(uint32_t);
  auto kern = topk_hist_kernel<IdT, WIDE, MAXR>;
  GEM_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 0;
  GEM_CHECK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kHistWarps * 32, smem));
  if (per_sm < 1) per_sm = 1;
  const int64_t units = L * ((T + kHistStepsPerUnit - 1) / kHistStepsPerUnit);
  int64_t blocks = (int64_t)num_sms() * per_sm;
  const int64_t need = (units + kHistWarps - 1) / kHistWarps;
  if (blocks > need) blocks = need;
  if (blocks < 1) blocks = 1;
  kern<<<(unsigned)blocks, kHistWarps * 32, smem, st>>>((const IdT*)ids, L, N, k, B, E, T, HT, hist, colsum, active,
                                                         heavy, dropped);
  GEM_CHECK_LAUNCH("topk_hist_kernel");
  return GEM_OK;
}

template <typename IdT>
static int dispatch_hist(const void* ids, int64_t L, int64_t N, int k, int B, int E, int64_t T, int64_t HT,
                         int32_t* hist,
                         int64_t* colsum, int32_t* active, int32_t* heavy, int64_t* dropped, cudaStream_t st) {
  // ring variant: int16 ids, every unit one whole-batch block (steps of whole
  // 2 KB batches, N a multiple of B, 16-byte aligned ids); wide counters up to
  // 160 experts, packed ones for even E up to 512
  const int64_t step_bytes = (int64_t)B * k * (int64_t)sizeof(IdT);
  if (sizeof(IdT) == 2 && N % B == 0 && step_bytes % (kRingUnroll * 32 * 16) == 0 &&
      (reinterpret_cast<uintptr_t>(ids) & 15) == 0 && (E <= kWideMaxE || E % 2 == 0) &&
      !std::getenv("GEM_HIST_NORING")) {
    // E in (160, 256]: the CTA-shared-counter kernel (GEM_HIST_CTA=0 disables it,
    // =1 also takes it for smaller E); other shapes: the one-warp ring kernels
    const char* cta_env = std::getenv("GEM_HIST_CTA");
    const int cta_mode = cta_env ? std::atoi(cta_env) : -1;
    const int bps = (int)(step_bytes / kCtaBatch);
    if (cta_mode != 0 && E <= 256 && (E > kWideMaxE || cta_mode == 1)) {
      if (bps == 8)
        return launch_hist_creg<8, 1, 1, 3, 1, 2>(ids, L, N, k, B, E, T, HT, hist, colsum, active, heavy, dropped, st);
      if (bps == 4)
        return launch_hist_creg<4, 2, 1, 3, 1, 2>(ids, L, N, k, B, E, T, HT, hist, colsum, active, heavy, dropped, st);
      if (bps == 2 && E <= 128)
        return launch_hist_creg<2, 2, 1, 3, 1, 4>(ids, L, N, k, B, E, T, HT, hist, colsum, active, heavy, dropped, st);
    }
    if (E <= 64) return launch_hist_ring<true, 2>(ids, L, N, k, B, E, T, HT, hist, colsum, active, heavy, dropped, st);
    if (E <= 128) return launch_hist_ring<true, 4>(ids, L, N, k, B, E, T, HT, hist, colsum, active, heavy, dropped, st);
    if (E <= kWideMaxE) return launch_hist_ring<true, 5>(ids, L, N, k, B, E, T, HT, hist, colsum, active, heavy, dropped, st);
    if (E <= 256) return launch_hist_ring<false, 4>(ids, L, N, k, B, E, T, HT, hist, colsum, active, heavy, dropped, st);
    return launch_hist_ring<false, 8>(ids, L, N, k, B, E, T, HT, hist, colsum, active, heavy, dropped, st);
  }
  if (E <= 64) return launch_hist_t<IdT, true, 2>(ids, L, N, k, B, E, T, HT, hist, colsum, active, heavy, dropped, st);
  if (E <= 128) return launch_hist_t<IdT, true, 4>(ids, L, N, k, B, E, T, HT, hist, colsum, active, heavy, dropped, st);
  if (E <= kWideMaxE) return launch_hist_t<IdT, true, 5>(ids, L, N, k, B, E, T, HT, hist, colsum, active, heavy, dropped, st);
  if (E <= 256) return launch_hist_t<IdT, false, 4>(ids, L, N, k, B, E, T, HT, hist, colsum, active, heavy, dropped, st);
  return launch_hist_t<IdT, false, 8>(ids, L, N, k, B, E, T, HT, hist, colsum, active, heavy, dropped, st);
}

}  // namespace gem

using namespace gem;

static int topk_hist_rows(const char* who, const void* ids, int32_t id_bytes, int64_t L, int64_t N, int32_t k,
                          int32_t B, int32_t E, int32_t* hist, int64_t hist_rows, int64_t* colsum, int32_t* active,
                          int32_t* heavy, int64_t* dropped, void* stream) {
  GEM_REQUIRE(id_bytes == 2 || id_bytes == 4, "%s: id_bytes must be 2 or 4", who);
  GEM_REQUIRE(L >= 1 && N >= 1 && k >= 1 && B >= 1 && E >= 1 && E <= 512,
              "%s: bad shape L=%lld N=%lld k=%d B=%d E=%d (E <= 512)", who, (long long)L, (long long)N, k, B, E);
  GEM_REQUIRE(ids && hist && colsum && active && heavy && dropped, "%s: null pointer", who);
  // a lane's u32 (wide) or u16 (packed) counter must not wrap within one step
  GEM_REQUIRE(E <= kWideMaxE || (int64_t)B * k <= 65535, "%s: E > %d needs at most 65535 ids per step", who,
              kWideMaxE);
  const int64_t T = (N + B - 1) / B;
  GEM_REQUIRE(hist_rows >= T, "%s: %lld histogram rows per layer cannot hold %lld steps", who, (long long)hist_rows,
              (long long)T);
  cudaStream_t st = as_stream(stream);
  if (id_bytes == 2) return dispatch_hist<int16_t>(ids, L, N, k, B, E, T, hist_rows, hist, colsum, active, heavy, dropped, st);
  return dispatch_hist<int32_t>(ids, L, N, k, B, E, T, hist_rows, hist, colsum, active, heavy, dropped, st);
}

extern "C" int gem_topk_hist(const void* ids, int32_t id_bytes, int64_t L, int64_t N, int32_t k, int32_t B,
                             int32_t E, int32_t* hist, int64_t* colsum, int32_t* active, int32_t* heavy,
                             int64_t* dropped, void* stream) {
  return topk_hist_rows("gem_topk_hist", ids, id_bytes, L, N, k, B, E, hist, (N + B - 1) / B, colsum, active,
                        heavy, dropped, stream);
}

extern "C" int gem_topk_hist_rows(const void* ids, int32_t id_bytes, int64_t L, int64_t N, int32_t k, int32_t B,
                                  int32_t E, int32_t* hist, int64_t hist_rows, int64_t* colsum, int32_t* active,
                                  int32_t* heavy, int64_t* dropped, void* stream) {
  return topk_hist_rows("gem_topk_hist_rows", ids, id_bytes, L, N, k, B, E, hist, hist_rows, colsum, active,
                        heavy, dropped, stream);
}
