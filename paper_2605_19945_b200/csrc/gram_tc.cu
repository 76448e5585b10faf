// K2 on the 5th-generation tensor cores: step-level co-activation Gram
//     gram[l][a][b] += sum_t h[l][t][a] * h[l][t][b]        (int64, exact)
// as an int8 X^T X contraction (tcgen05.mma kind::i8, s32 accumulators in TMEM).
//
// Exactness. Every count 0 <= h <= 65535 is split into two u8 limbs,
// h = 256*hi + lo. One CTA accumulates, for a 128-expert block pair (A, B),
//     LL = sum lo_a lo_b, LH = sum lo_a hi_b, HL = sum hi_a lo_b, HH = sum hi_a hi_b
// in s32 over at most kSegSteps = 16384 steps (16384 * 255^2 < 2^31, so no
// accumulator can wrap), then combines them in int64,
//     G = LL + 256 (LH + HL) + 65536 HH,
// and adds the segment into gram with 64-bit atomics. Integer arithmetic only,
// so the result is bit-identical to the CUDA-core kernel and to the oracle.
//
// Data flow per CTA (persistent: one contiguous range of the flattened
// (layer, step) space, split at layer boundaries and every kSegSteps steps):
//   * all 8 warps stream int32 histogram rows with 128-bit loads (the next
//     chunk's loads are issued before the current chunk is converted), split
//     them into limbs, transpose 4 steps x 4 experts in registers with byte
//     permutes and store the u8 operand tile K-major (K = steps) into a
//     4-stage shared-memory ring with bank-conflict-free 32-bit stores;
//   * thread 0 issues, per 32-step K slice, two 128x256x32 MMAs
//     (A = lo rows / hi rows of block A, B = [lo; hi] rows of block B) into
//     TMEM columns [0,256) and [256,512), and commits each stage to an mbarrier
//     that frees the ring slot;
//   * at a segment end the 4 limb products are read back with tcgen05.ld and
//     flushed.
// Bound: HBM (each histogram byte is read once); the MMAs need ~1/8 of the
// tensor pipe at that rate.
#include "gem_common.cuh"
#include "tc.cuh"

namespace gem {

#ifndef GEM_GTC_WARPS
#define GEM_GTC_WARPS 16
#endif
constexpr int kGtcWarps = GEM_GTC_WARPS;   // producer warps (all of them also drain TMEM)
constexpr int kGtcThreads = 32 * kGtcWarps;
constexpr int kGtcTasksPerWarp = 32 / kGtcWarps;  // (16 steps x 32 experts) tasks per warp and stage
constexpr int kGtcStages = 4;
constexpr int64_t kSegSteps = 16384;
constexpr int kGtcStageBytes = 32768;
constexpr uint32_t kGtcIdesc = tc::instr_desc(/*S32*/ 2, /*u8*/ 0, /*u8*/ 0, 128, 256);

struct GramPairs {  // 128-expert block pairs (a <= b), by value
  int2 p[10];
};

struct GramTcShared {
  uint64_t stage_bar[kGtcStages];
  uint64_t acc_bar;
  uint32_t tmem_base;
};

// NB = number of 128-expert blocks staged: 1 (diagonal block pair, A == B) or
// 2 (off-diagonal pair). KT = steps per stage so that a stage is 32 KB.
template <int NB>
__global__ void __launch_bounds__(kGtcThreads, 1)
gram_tc_kernel(const int32_t* __restrict__ hist, int64_t T, int E, int64_t total_steps, int64_t range,
               const GramPairs pairs, int64_t* __restrict__ gram) {
  constexpr int KT = 128 / NB;        // steps per stage
  constexpr int ROWS = 256 * NB;      // operand rows per stage: [lo_A; hi_A] (+ [lo_B; hi_B])
  constexpr uint32_t LBO = ROWS * 16; // bytes per 16-step K slice
  constexpr int TG = KT / 16;         // 16-step groups per stage
  constexpr int TASKS = TG * 4 * NB;  // (16 steps x 32 experts) tasks per stage
  static_assert(TASKS == 32 && TASKS == kGtcWarps * kGtcTasksPerWarp, "32 tasks per stage");
  static_assert(TG * LBO == kGtcStageBytes, "stage size");

  extern __shared__ __align__(1024) unsigned char gtc_smem[];
  unsigned char* ring = gtc_smem;
  GramTcShared* sh = reinterpret_cast<GramTcShared*>(gtc_smem + kGtcStages * kGtcStageBytes);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t s0 = (int64_t)blockIdx.x * range;
  const int64_t s1 = imin64(s0 + range, total_steps);
  if (s0 >= s1) return;
  const int2 pr = pairs.p[blockIdx.y];
  const int blkA = pr.x * 128, blkB = pr.y * 128;

  if (tid == 0) {
    for (int s = 0; s < kGtcStages; ++s) tc::mbar_init(&sh->stage_bar[s], 1);
    tc::mbar_init(&sh->acc_bar, 1);
    tc::fence_mbar_init();
  }
  if (warp == 0) tc::tmem_alloc<512>(&sh->tmem_base);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = sh->tmem_base;
  const uint32_t ring_addr = tc::smem_u32(ring);

  // lane geometry inside a (16 steps x 32 experts) task
  const int t4 = lane >> 3, e4 = lane & 7;
  const int rot = e4 >> 1;  // store rotation -> 32 distinct banks

  int64_t chunk = 0;  // global chunk counter (ring slot + phase)
  int seg_no = 0;
  int64_t p = s0;
  while (p < s1) {
    const int64_t l = p / T;
    const int64_t t_begin = p % T;
    const int64_t seg_len = imin64(imin64(s1 - p, T - t_begin), kSegSteps);
    const int64_t t_end = t_begin + seg_len;
    const int32_t* hl = hist + l * T * E;
    const int nchunks = (int)((seg_len + KT - 1) / KT);

    int4 cur[kGtcTasksPerWarp][4], nxt[kGtcTasksPerWarp][4];
    auto load_chunk = [&](int c, int4 (&buf)[kGtcTasksPerWarp][4]) {
      const int64_t tc0 = t_begin + (int64_t)c * KT;
#pragma unroll
      for (int q = 0; q < kGtcTasksPerWarp; ++q) {
        const int task = warp * kGtcTasksPerWarp + q;
        const int blk = task / (TG * 4);
        const int rem = task % (TG * 4);
        const int tg = rem >> 2, eg = rem & 3;
        const int e = (blk ? blkB : blkA) + eg * 32 + e4 * 4;
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const int64_t t = tc0 + tg * 16 + t4 * 4 + r;
          buf[q][r] = t < t_end ? __ldg(reinterpret_cast<const int4*>(hl + t * E + e)) : make_int4(0, 0, 0, 0);
        }
      }
    };
    load_chunk(0, cur);
    for (int c = 0; c < nchunks; ++c) {
      if (c + 1 < nchunks) load_chunk(c + 1, nxt);
      const int slot = (int)(chunk % kGtcStages);
      if (chunk >= kGtcStages) tc::mbar_wait(&sh->stage_bar[slot], (uint32_t)((chunk / kGtcStages - 1) & 1));
      unsigned char* st = ring + slot * kGtcStageBytes;
#pragma unroll
      for (int q = 0; q < kGtcTasksPerWarp; ++q) {
        const int task = warp * kGtcTasksPerWarp + q;
        const int blk = task / (TG * 4);
        const int rem = task % (TG * 4);
        const int tg = rem >> 2, eg = rem & 3;
        // 4 steps x 4 experts -> per expert one lo word and one hi word (byte i = step i)
        uint32_t lo[4], hi[4];
        const uint32_t v[4][4] = {
            {(uint32_t)cur[q][0].x, (uint32_t)cur[q][0].y, (uint32_t)cur[q][0].z, (uint32_t)cur[q][0].w},
            {(uint32_t)cur[q][1].x, (uint32_t)cur[q][1].y, (uint32_t)cur[q][1].z, (uint32_t)cur[q][1].w},
            {(uint32_t)cur[q][2].x, (uint32_t)cur[q][2].y, (uint32_t)cur[q][2].z, (uint32_t)cur[q][2].w},
            {(uint32_t)cur[q][3].x, (uint32_t)cur[q][3].y, (uint32_t)cur[q][3].z, (uint32_t)cur[q][3].w}};
#pragma unroll
        for (int x = 0; x < 4; ++x) {
          const uint32_t p01 = __byte_perm(v[0][x], v[1][x], 0x5140);  // s0.b0 s1.b0 s0.b1 s1.b1
          const uint32_t p23 = __byte_perm(v[2][x], v[3][x], 0x5140);
          lo[x] = __byte_perm(p01, p23, 0x5410);
          hi[x] = __byte_perm(p01, p23, 0x7632);
        }
        const int row0 = blk * 256 + eg * 32 + e4 * 4;  // lo row of expert x is row0 + x, hi row is +128
        unsigned char* kslice = st + tg * LBO + t4 * 4;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int x = (i + rot) & 3;
          const uint32_t wl = x == 0 ? lo[0] : x == 1 ? lo[1] : x == 2 ? lo[2] : lo[3];
          const uint32_t wh = x == 0 ? hi[0] : x == 1 ? hi[1] : x == 2 ? hi[2] : hi[3];
          *reinterpret_cast<uint32_t*>(kslice + (row0 + x) * 16) = wl;
          *reinterpret_cast<uint32_t*>(kslice + (row0 + 128 + x) * 16) = wh;
        }
      }
      tc::fence_async_smem();
      __syncthreads();
      if (tid == 0) {
        tc::tc_fence_after();
        const uint32_t sbase = ring_addr + slot * kGtcStageBytes;
        const uint32_t b_off = NB == 2 ? 256 * 16 : 0;
#pragma unroll
        for (int ks = 0; ks < KT / 32; ++ks) {
          const uint32_t kb = sbase + ks * 2 * LBO;
          const uint64_t a_lo = tc::smem_desc(kb, LBO, 128);
          const uint64_t a_hi = tc::smem_desc(kb + 128 * 16, LBO, 128);
          const uint64_t bd = tc::smem_desc(kb + b_off, LBO, 128);
          const uint32_t acc = (c > 0 || ks > 0) ? 1u : 0u;
          tc::mma_i8(tmem, a_lo, bd, kGtcIdesc, acc);
          tc::mma_i8(tmem + 256, a_hi, bd, kGtcIdesc, acc);
        }
        tc::mma_commit(&sh->stage_bar[slot]);
        if (c + 1 == nchunks) tc::mma_commit(&sh->acc_bar);
      }
      ++chunk;
#pragma unroll
      for (int q = 0; q < kGtcTasksPerWarp; ++q)
#pragma unroll
        for (int r = 0; r < 4; ++r) cur[q][r] = nxt[q][r];
    }

    // ---- segment epilogue: TMEM -> int64 -> gram
    tc::mbar_wait(&sh->acc_bar, (uint32_t)(seg_no & 1));
    tc::tc_fence_after();
    {
      const int lg = warp & 3, ch = warp >> 2;  // TMEM lane group, column slice of 128 / (warps / 4)
      constexpr int CW = 128 / (kGtcWarps / 4);
      const int a = blkA + lg * 32 + lane;
      const uint32_t trow = tmem + ((uint32_t)(lg * 32) << 16);
      int64_t* grow = gram + (l * E + a) * E + blkB;
#pragma unroll 1
      for (int b0 = ch * CW; b0 < ch * CW + CW; b0 += 16) {
        uint32_t ll[16], lh[16], hl2[16], hh[16];
        tc::tmem_ld16(trow + b0, ll);
        tc::tmem_ld16(trow + 128 + b0, lh);
        tc::tmem_ld16(trow + 256 + b0, hl2);
        tc::tmem_ld16(trow + 384 + b0, hh);
        tc::tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const uint64_t g = (uint64_t)ll[i] + ((uint64_t)lh[i] + (uint64_t)hl2[i]) * 256ull + (uint64_t)hh[i] * 65536ull;
          if (g) atomicAdd(reinterpret_cast<unsigned long long*>(grow + b0 + i), (unsigned long long)g);
        }
      }
    }
    tc::tc_fence_before();
    __syncthreads();
    ++seg_no;
    p += seg_len;
  }

  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<512>(tmem);
}

}  // namespace gem

using namespace gem;

static int gram_tc_launch(const int32_t* hist, int64_t L, int64_t T, int32_t E, int64_t* gram, cudaStream_t st) {
  const int nbk = E / 128;
  GramPairs diag{}, off{};
  int nd = 0, no = 0;
  for (int a = 0; a < nbk; ++a)
    for (int b = a; b < nbk; ++b) {
      if (a == b) diag.p[nd++] = make_int2(a, b);
      else off.p[no++] = make_int2(a, b);
    }
  const int64_t total = L * T;
  const size_t smem = (size_t)kGtcStages * kGtcStageBytes + sizeof(GramTcShared);
  const int sms = num_sms();
  auto run = [&](auto kern, int npairs, const GramPairs& pp) -> int {
    GEM_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int64_t ctas = sms / npairs;
    if (ctas < 1) ctas = 1;
    int64_t range = (total + ctas - 1) / ctas;
    range = ((range + 127) / 128) * 128;  // whole stages where the layer boundaries allow
    ctas = (total + range - 1) / range;
    kern<<<dim3((unsigned)ctas, (unsigned)npairs), kGtcThreads, smem, st>>>(hist, T, E, total, range, pp, gram);
    GEM_CHECK_LAUNCH("gram_tc_kernel");
    return GEM_OK;
  };
  int rc = run(gram_tc_kernel<1>, nd, diag);
  if (rc == GEM_OK && no) rc = run(gram_tc_kernel<2>, no, off);
  return rc;
}

extern "C" int gem_step_gram_tc(const int32_t* hist, int64_t L, int64_t T, int32_t E, int64_t* gram, void* stream) {
  GEM_REQUIRE(hist && gram && L >= 1 && T >= 1, "gem_step_gram_tc: bad arguments");
  GEM_REQUIRE(E >= 128 && E <= 512 && E % 128 == 0, "gem_step_gram_tc: E must be 128, 256, 384 or 512 (got %d)", E);
  return gram_tc_launch(hist, L, T, E, gram, as_stream(stream));
}
