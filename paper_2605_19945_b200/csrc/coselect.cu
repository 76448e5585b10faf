// K2b: token-level co-selection counts (north-star subsystem (1))
//
//     cosel[l][a][b] += #tokens n of layer l whose top-k set S_n holds both a and b
//
// i.e. OᵀO for the 0/1 selection indicator O [N, E] of each layer. The diagonal
// is the number of tokens that selected a, which equals K1's colsum[l][a]
// whenever a token's ids are distinct (router top-k) -- a built-in parity link.
// Ids outside [0, E) are ignored (K1 counts them as dropped); a repeated id
// inside one token counts once (indicator semantics). int32 output, full
// symmetric matrix; the caller guarantees every count stays below 2^31
// (it is at most the number of tokens).
//
// The reference has no counterpart: its only co-activation statistic is the
// step-level Pearson correlation (/root/reference/pkg/src/gemap/trace.py:100-113),
// which K2 (gram_tc.cu) feeds.
//
// Two kernels, both exact (integer-only), chosen by measurement:
//
//  * coselect_tc_kernel (E <= 256): OᵀO as an int8 one-hot contraction on the
//    5th-generation tensor cores, tcgen05.mma kind::i8 with s32 accumulators in
//    TMEM. Warp-specialised, persistent (two CTAs per SM at E <= 128, one at
//    E <= 256), each over a contiguous range of the flattened (layer, token)
//    space:
//      - warp 5 (TMA): one 1-D cp.async.bulk per 128-token stage moves the
//        stage's ids into a shared-memory ring, completing on an mbarrier;
//      - warps 0-3 (producers): lane = token; each lane reads its own k ids from
//        the ring, the warp zeroes its two 16-token K slices of the one-hot
//        operand tile and sets byte (expert, token) = 1 for every valid id --
//        the tile is Oᵀ in the K-major no-swizzle UMMA layout (tc.cuh);
//      - warp 4 (MMA): one elected thread issues, per 32 tokens,
//        D[128 x N] += Oᵀ[block] · O, with A and B descriptors on the SAME tile
//        (E <= 128: one 128x128x32 MMA; E <= 256: 128x256 for expert block 0 and
//        128x128 for the block-1 diagonal block, the lower-left block is the
//        mirror), and frees the stage with tcgen05.commit;
//      - at every layer-segment end the producers drain TMEM (tcgen05.ld) and
//        add the segment's counts to cosel with global reductions.
//    The one-hot expansion is 8-16x the id bytes, so it never leaves shared
//    memory: HBM sees the ids once and the [E,E] result once per segment.
//  * coselect_scatter_kernel (any E): CUDA-core reference kernel -- per token,
//    every pair of its distinct valid ids increments an upper-triangle counter
//    in shared memory (global memory when the triangle does not fit), flushed
//    per layer segment. Used for E > 256, unaligned id buffers and k*id_bytes >
//    32, and as the tensor-core kernel's cross-check.
#include "gem_common.cuh"
#include "tc.cuh"

namespace gem {

constexpr int kCsTok = 128;                     // tokens per pipeline stage
constexpr int kCsProd = 4;                      // producer / epilogue warps (32 tokens each, TMEM lane quarters)
constexpr int kCsThreads = (kCsProd + 2) * 32;  // + MMA warp + TMA warp
constexpr int kCsMaxTokBytes = 32;              // k * id_bytes on the tensor-core path

#ifndef GEM_CS_IDRING
#define GEM_CS_IDRING 32768  // bytes of the TMA id ring per CTA
#endif
#ifndef GEM_CS_STAGES1
#define GEM_CS_STAGES1 4  // E <= 128: 4 x 16 KB operand stages -> two CTAs per SM
#endif

// IDB: bytes of one id-ring slot (kCsTok tokens x 16 or 32 bytes); the id ring
// is 32 KB deep either way (16 or 8 stages of 128 tokens in flight per CTA),
// enough outstanding TMA bytes to cover HBM latency at the kernel's id rate
template <int EB, int IDB>
struct CsGeo {
  static constexpr int EP = 128 * EB;                // padded experts (operand rows)
  static constexpr int SLICE = EP * 16;              // bytes of one 16-token K slice
  // K-slice stride: +64 bytes of padding shift the second slice of a warp by
  // 16 banks, so lanes t and t+16 (same byte column, adjacent slices) stop
  // colliding in the one-hot scatter; the MMA never reads the padding
  static constexpr int LBO = SLICE + 64;
  static constexpr int STAGE = LBO * (kCsTok / 16);  // one-hot bytes per stage
  static constexpr int STAGES = EB == 1 ? GEM_CS_STAGES1 : 4;  // powers of two: ring
  static constexpr int ISTAGES = GEM_CS_IDRING / IDB;
  static constexpr size_t SMEM_EST = (size_t)STAGES * STAGE + (size_t)ISTAGES * IDB + 512;
  static constexpr int CTAS_PER_SM = EB == 1 ? (SMEM_EST <= 74 * 1024 ? 3 : (STAGES <= 4 ? 2 : 1)) : 1;
  static constexpr uint32_t TMEM_COLS = EB == 1 ? 128 : 512;
  static constexpr size_t SMEM = (size_t)STAGES * STAGE + (size_t)ISTAGES * IDB + 512;
};

struct CsBars {
  uint64_t ids_full[16], ids_empty[16], op_full[8], op_empty[8], acc_full, acc_empty;
  uint32_t tmem_base;
};

constexpr uint32_t kCsIdesc128 = tc::instr_desc(/*S32*/ 2, /*u8*/ 0, /*u8*/ 0, 128, 128);
constexpr uint32_t kCsIdesc256 = tc::instr_desc(/*S32*/ 2, /*u8*/ 0, /*u8*/ 0, 128, 256);

template <typename IdT>
__device__ __forceinline__ uint32_t id_as_u32(IdT v) {
  return (uint32_t)(int32_t)v;  // negative ids become >= E and are skipped
}

// TOKB: bytes of one token's ids when they can be read as 16-byte vectors (16
// or 32), 0 for the scalar path.
template <typename IdT, int EB, int TOKB, int IDB>
__global__ void __launch_bounds__(kCsThreads, (CsGeo<EB, IDB>::CTAS_PER_SM))
coselect_tc_kernel(const IdT* __restrict__ ids, int64_t N, int k, int E, int64_t total, int64_t range,
                   int32_t* __restrict__ out) {
  using G = CsGeo<EB, IDB>;
  constexpr int kMaxIds = kCsMaxTokBytes / (int)sizeof(IdT);
  extern __shared__ __align__(1024) unsigned char cs_smem[];
  unsigned char* op = cs_smem;
  unsigned char* idr = cs_smem + G::STAGES * G::STAGE;
  CsBars* sh = reinterpret_cast<CsBars*>(idr + G::ISTAGES * IDB);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t s0 = (int64_t)blockIdx.x * range;
  const int64_t s1 = imin64(s0 + range, total);
  if (s0 >= s1) return;
  const int tok_bytes = k * (int)sizeof(IdT);

  if (tid == 0) {
    for (int i = 0; i < G::ISTAGES; ++i) {
      tc::mbar_init(&sh->ids_full[i], 1);
      tc::mbar_init(&sh->ids_empty[i], kCsProd);
    }
    for (int i = 0; i < G::STAGES; ++i) {
      tc::mbar_init(&sh->op_full[i], kCsProd);
      tc::mbar_init(&sh->op_empty[i], 1);
    }
    tc::mbar_init(&sh->acc_full, 1);
    tc::mbar_init(&sh->acc_empty, kCsProd);
    tc::fence_mbar_init();
  }
  if (warp == 0) tc::tmem_alloc<G::TMEM_COLS>(&sh->tmem_base);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = sh->tmem_base;

  if (warp == kCsProd + 1) {
    // ---------------- TMA: ids of each stage -> shared ring
    if (lane == 0) {
      uint32_t g = 0;
      for (int64_t p = s0; p < s1;) {
        const int64_t seg = imin64(s1 - p, N - p % N);
        for (int64_t j = 0; j < seg; j += kCsTok, ++g) {
          const int is = (int)(g % G::ISTAGES);
          if (g >= G::ISTAGES) {
            tc::mbar_wait(&sh->ids_empty[is], (g / G::ISTAGES - 1) & 1);
            tc::fence_async_smem();  // the producers' generic reads of the slot before the async-proxy refill
          }
          const uint32_t bytes = (uint32_t)(imin64(kCsTok, seg - j) * tok_bytes);
          tc::mbar_arrive_expect_tx(&sh->ids_full[is], bytes);
          tc::bulk_load_1d(idr + is * IDB, ids + (p + j) * k, bytes, &sh->ids_full[is]);
        }
        p += seg;
      }
    }
  } else if (warp == kCsProd) {
    // ---------------- MMA issuer
    if (lane == 0) {
      uint32_t g = 0;
      int segno = 0;
      const uint32_t op_addr = tc::smem_u32(op);
      for (int64_t p = s0; p < s1; ++segno) {
        const int64_t seg = imin64(s1 - p, N - p % N);
        const int64_t nst = (seg + kCsTok - 1) / kCsTok;
        for (int64_t st = 0; st < nst; ++st, ++g) {
          const int s = (int)(g % G::STAGES);
          tc::mbar_wait(&sh->op_full[s], (g / G::STAGES) & 1);
          if (st == 0 && segno > 0) tc::mbar_wait(&sh->acc_empty, (uint32_t)((segno - 1) & 1));
          tc::tc_fence_after();
          const uint32_t base = op_addr + (uint32_t)(s * G::STAGE);
#pragma unroll
          for (int ks = 0; ks < kCsTok / 32; ++ks) {
            const uint32_t kb = base + (uint32_t)(ks * 2 * G::LBO);
            const uint32_t acc = (st > 0 || ks > 0) ? 1u : 0u;
            const uint64_t d0 = tc::smem_desc(kb, G::LBO, 128);
            if (EB == 1) {
              tc::mma_i8(tmem, d0, d0, kCsIdesc128, acc);
            } else {
              const uint64_t d1 = tc::smem_desc(kb + 128 * 16, G::LBO, 128);
              tc::mma_i8(tmem, d0, d0, kCsIdesc256, acc);        // rows 0..127 x cols 0..255
              tc::mma_i8(tmem + 256, d1, d1, kCsIdesc128, acc);  // rows 128..255 x cols 128..255
            }
          }
          tc::mma_commit(&sh->op_empty[s]);
          if (st + 1 == nst) tc::mma_commit(&sh->acc_full);
        }
        p += seg;
      }
    }
  } else {
    // ---------------- producers (lane = token of the stage) + segment epilogue
    uint32_t g = 0;
    int segno = 0;
    const int tok = warp * 32 + lane;
    for (int64_t p = s0; p < s1; ++segno) {
      const int64_t l = p / N;
      const int64_t seg = imin64(s1 - p, N - p % N);
      const int64_t nst = (seg + kCsTok - 1) / kCsTok;
      for (int64_t st = 0; st < nst; ++st, ++g) {
        const int s = (int)(g % G::STAGES), is = (int)(g % G::ISTAGES);
        const bool valid = tok < imin64(kCsTok, seg - st * kCsTok);
        uint32_t idv[kMaxIds];
        tc::mbar_wait(&sh->ids_full[is], (g / G::ISTAGES) & 1);
        if (valid) {
          const unsigned char* tp = idr + is * IDB + tok * tok_bytes;
          if (TOKB > 0) {
            uint32_t w[TOKB > 0 ? TOKB / 4 : 1];
#pragma unroll
            for (int v = 0; v < TOKB / 16; ++v) {
              const uint4 q = reinterpret_cast<const uint4*>(tp)[v];
              w[4 * v] = q.x; w[4 * v + 1] = q.y; w[4 * v + 2] = q.z; w[4 * v + 3] = q.w;
            }
#pragma unroll
            for (int i = 0; i < kMaxIds; ++i) {
              if (sizeof(IdT) == 2) idv[i] = (uint32_t)(int32_t)(int16_t)(w[i >> 1] >> ((i & 1) * 16));
              else idv[i] = w[i];
            }
          } else {
#pragma unroll
            for (int i = 0; i < kMaxIds; ++i)
              idv[i] = i < k ? id_as_u32(reinterpret_cast<const IdT*>(tp)[i]) : 0xffffffffu;
          }
        }
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&sh->ids_empty[is]);
        if (g >= G::STAGES) tc::mbar_wait(&sh->op_empty[s], (g / G::STAGES - 1) & 1);
        unsigned char* slab = op + s * G::STAGE + warp * 2 * G::LBO;  // this warp's two 16-token K slices
#pragma unroll
        for (int i = lane; i < 2 * G::EP; i += 32)
          *reinterpret_cast<uint4*>(slab + (i / G::EP) * G::LBO + (i % G::EP) * 16) = make_uint4(0u, 0u, 0u, 0u);
        __syncwarp();
        if (valid) {
          unsigned char* col = slab + (lane >> 4) * G::LBO + (lane & 15);
#pragma unroll
          for (int i = 0; i < kMaxIds; ++i)
            if (i < k && idv[i] < (uint32_t)E) col[idv[i] * 16] = 1;
        }
        tc::fence_async_smem();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&sh->op_full[s]);

        if (st + 1 == nst) {
          // ---- segment epilogue: TMEM lanes [32w, 32w+32) -> cosel[l]
          tc::mbar_wait(&sh->acc_full, (uint32_t)(segno & 1));
          tc::tc_fence_after();
          int32_t* ol = out + l * (int64_t)E * E;
          const uint32_t trow = tmem + ((uint32_t)(warp * 32) << 16);
          const int a0 = warp * 32 + lane;
#pragma unroll 1
          for (int c0 = 0; c0 < (EB == 1 ? 128 : 384); c0 += 16) {
            uint32_t v[16];
            tc::tmem_ld16(trow + c0, v);
            tc::tmem_ld_wait();
            const int a = c0 < 256 ? a0 : 128 + a0;             // block-1 rows live in columns [256, 384)
            const int b0 = c0 < 256 ? c0 : 128 + (c0 - 256);
            if (a < E) {
#pragma unroll
              for (int i = 0; i < 16; ++i) {
                const int b = b0 + i;
                if (b < E && v[i]) {
                  atomicAdd(ol + (int64_t)a * E + b, (int)v[i]);
                  if (EB == 2 && c0 < 256 && b >= 128) atomicAdd(ol + (int64_t)b * E + a, (int)v[i]);
                }
              }
            }
          }
          tc::tc_fence_before();
          __syncwarp();
          if (lane == 0) tc::mbar_arrive(&sh->acc_empty);
        }
      }
      p += seg;
    }
  }
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<G::TMEM_COLS>(tmem);
}

// ---------------------------------------------------------------------------
// CUDA-core kernel: per token, every pair of distinct valid ids increments an
// upper-triangle counter tri(a <= b) (shared memory when it fits, else global).
constexpr int kCsScatterThreads = 512;
constexpr int kCsScatterMaxK = 32;

__device__ __forceinline__ int64_t tri_index(int a, int b, int E) {  // a <= b
  return (int64_t)a * E - (int64_t)a * (a - 1) / 2 + (b - a);
}

template <typename IdT, bool SMEM>
__global__ void __launch_bounds__(kCsScatterThreads)
coselect_scatter_kernel(const IdT* __restrict__ ids, int64_t N, int k, int E, int64_t total, int64_t range,
                        int32_t* __restrict__ out) {
  extern __shared__ uint32_t tri[];
  const int64_t ntri = (int64_t)E * (E + 1) / 2;
  const int64_t s0 = (int64_t)blockIdx.x * range;
  const int64_t s1 = imin64(s0 + range, total);
  if (s0 >= s1) return;
  if (SMEM) {
    for (int64_t q = threadIdx.x; q < ntri; q += blockDim.x) tri[q] = 0;
    __syncthreads();
  }
  for (int64_t p = s0; p < s1;) {
    const int64_t l = p / N;
    const int64_t seg = imin64(s1 - p, N - p % N);
    int32_t* ol = out + l * (int64_t)E * E;
    for (int64_t j = p + threadIdx.x; j < p + seg; j += blockDim.x) {
      const IdT* tp = ids + j * k;
      int d[kCsScatterMaxK];
      int m = 0;
      for (int i = 0; i < k; ++i) {
        const uint32_t e = id_as_u32(tp[i]);
        if (e >= (uint32_t)E) continue;
        bool dup = false;
        for (int q = 0; q < m; ++q) dup |= (d[q] == (int)e);
        if (!dup) d[m++] = (int)e;
      }
      for (int x = 0; x < m; ++x)
        for (int y = x; y < m; ++y) {
          const int a = min(d[x], d[y]), b = max(d[x], d[y]);
          if (SMEM) {
            atomicAdd(&tri[tri_index(a, b, E)], 1u);
          } else {
            atomicAdd(ol + (int64_t)a * E + b, 1);
            if (a != b) atomicAdd(ol + (int64_t)b * E + a, 1);
          }
        }
    }
    if (SMEM) {
      __syncthreads();
      for (int64_t q = threadIdx.x; q < (int64_t)E * E; q += blockDim.x) {
        const int a = (int)(q / E), b = (int)(q % E);
        if (b < a) continue;
        const int64_t t = tri_index(a, b, E);
        const uint32_t v = tri[t];
        if (v) {
          atomicAdd(ol + (int64_t)a * E + b, (int)v);
          if (a != b) atomicAdd(ol + (int64_t)b * E + a, (int)v);
        }
      }
      __syncthreads();
      for (int64_t q = threadIdx.x; q < ntri; q += blockDim.x) tri[q] = 0;
      __syncthreads();
    }
    p += seg;
  }
}

// ---------------------------------------------------------------------------
// launchers

static int64_t cs_range(int64_t total, int64_t ctas, int64_t align) {
  int64_t r = (total + ctas - 1) / ctas;
  return ((r + align - 1) / align) * align;
}

template <typename IdT, int EB, int TOKB, int IDB>
static int launch_cs_tc(const void* ids, int64_t L, int64_t N, int k, int E, int32_t* out, cudaStream_t st) {
  auto kern = coselect_tc_kernel<IdT, EB, TOKB, IDB>;
  const size_t smem = CsGeo<EB, IDB>::SMEM;
  GEM_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int64_t total = L * N;
  int per_sm = 1;
  GEM_CHECK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kCsThreads, smem));
  if (per_sm < 1) per_sm = 1;
  int64_t ctas = imin64((int64_t)num_sms() * per_sm, (total + kCsTok - 1) / kCsTok);
  const int64_t range = cs_range(total, ctas, kCsTok);
  ctas = (total + range - 1) / range;
  kern<<<(unsigned)ctas, kCsThreads, smem, st>>>((const IdT*)ids, N, k, E, total, range, out);
  GEM_CHECK_LAUNCH("coselect_tc_kernel");
  return GEM_OK;
}

template <typename IdT, int EB>
static int dispatch_cs_tc(const void* ids, int64_t L, int64_t N, int k, int E, int32_t* out, cudaStream_t st) {
  const int tb = k * (int)sizeof(IdT);
  if (tb == 16) return launch_cs_tc<IdT, EB, 16, 2048>(ids, L, N, k, E, out, st);
  if (tb == 32) return launch_cs_tc<IdT, EB, 32, 4096>(ids, L, N, k, E, out, st);
  if (tb < 16) return launch_cs_tc<IdT, EB, 0, 2048>(ids, L, N, k, E, out, st);
  return launch_cs_tc<IdT, EB, 0, 4096>(ids, L, N, k, E, out, st);
}

static size_t cs_scatter_smem(int E) { return (size_t)E * (E + 1) / 2 * sizeof(uint32_t); }

template <typename IdT>
static int launch_cs_scatter(const void* ids, int64_t L, int64_t N, int k, int E, int32_t* out, cudaStream_t st) {
  const size_t smem = cs_scatter_smem(E);
  const bool in_smem = smem <= 200 * 1024;
  const int64_t total = L * N;
  int per_sm = 1;
  if (in_smem) {
    auto kern = coselect_scatter_kernel<IdT, true>;
    GEM_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    GEM_CHECK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kCsScatterThreads, smem));
    if (per_sm < 1) per_sm = 1;
    int64_t ctas = imin64((int64_t)num_sms() * per_sm, (total + kCsScatterThreads - 1) / kCsScatterThreads);
    const int64_t range = cs_range(total, ctas, kCsScatterThreads);
    ctas = (total + range - 1) / range;
    kern<<<(unsigned)ctas, kCsScatterThreads, smem, st>>>((const IdT*)ids, N, k, E, total, range, out);
  } else {
    int64_t ctas = imin64((int64_t)num_sms() * 4, (total + kCsScatterThreads - 1) / kCsScatterThreads);
    const int64_t range = cs_range(total, ctas, kCsScatterThreads);
    ctas = (total + range - 1) / range;
    coselect_scatter_kernel<IdT, false>
        <<<(unsigned)ctas, kCsScatterThreads, 0, st>>>((const IdT*)ids, N, k, E, total, range, out);
  }
  GEM_CHECK_LAUNCH("coselect_scatter_kernel");
  return GEM_OK;
}

}  // namespace gem

using namespace gem;

static int cs_check(const char* who, const void* ids, int32_t id_bytes, int64_t L, int64_t N, int32_t k, int32_t E,
                    const int32_t* out) {
  GEM_REQUIRE(ids && out, "%s: null pointer", who);
  GEM_REQUIRE(id_bytes == 2 || id_bytes == 4, "%s: id_bytes must be 2 or 4", who);
  GEM_REQUIRE(L >= 1 && N >= 1 && k >= 1 && k <= kCsScatterMaxK && E >= 1 && E <= 1024,
              "%s: bad shape L=%lld N=%lld k=%d E=%d (k <= 32, E <= 1024)", who, (long long)L, (long long)N, k, E);
  GEM_REQUIRE(N < (1LL << 31), "%s: more than 2^31 - 1 tokens per layer would overflow the int32 counts", who);
  return GEM_OK;
}

extern "C" int gem_coselect_path(const void* ids, int32_t id_bytes, int64_t N, int32_t k, int32_t E) {
  const int64_t tb = (int64_t)k * id_bytes;
  const bool aligned = (reinterpret_cast<uintptr_t>(ids) & 15) == 0 && (N * tb) % 16 == 0;
  return (E >= 1 && E <= 256 && tb <= kCsMaxTokBytes && aligned) ? 1 : 0;
}

extern "C" int gem_coselect_tc(const void* ids, int32_t id_bytes, int64_t L, int64_t N, int32_t k, int32_t E,
                               int32_t* cosel, void* stream) {
  int rc = cs_check("gem_coselect_tc", ids, id_bytes, L, N, k, E, cosel);
  if (rc) return rc;
  GEM_REQUIRE(gem_coselect_path(ids, id_bytes, N, k, E) == 1,
              "gem_coselect_tc: needs E <= 256, k*id_bytes <= 32, a 16-byte aligned buffer and N*k*id_bytes %% 16 == 0");
  cudaStream_t st = as_stream(stream);
  if (id_bytes == 2) {
    return E <= 128 ? dispatch_cs_tc<int16_t, 1>(ids, L, N, k, E, cosel, st)
                    : dispatch_cs_tc<int16_t, 2>(ids, L, N, k, E, cosel, st);
  }
  return E <= 128 ? dispatch_cs_tc<int32_t, 1>(ids, L, N, k, E, cosel, st)
                  : dispatch_cs_tc<int32_t, 2>(ids, L, N, k, E, cosel, st);
}

extern "C" int gem_coselect_scatter(const void* ids, int32_t id_bytes, int64_t L, int64_t N, int32_t k, int32_t E,
                                    int32_t* cosel, void* stream) {
  int rc = cs_check("gem_coselect_scatter", ids, id_bytes, L, N, k, E, cosel);
  if (rc) return rc;
  cudaStream_t st = as_stream(stream);
  if (id_bytes == 2) return launch_cs_scatter<int16_t>(ids, L, N, k, E, cosel, st);
  return launch_cs_scatter<int32_t>(ids, L, N, k, E, cosel, st);
}

extern "C" int gem_coselect(const void* ids, int32_t id_bytes, int64_t L, int64_t N, int32_t k, int32_t E,
                            int32_t* cosel, void* stream) {
  if (gem_coselect_path(ids, id_bytes, N, k, E) == 1) return gem_coselect_tc(ids, id_bytes, L, N, k, E, cosel, stream);
  return gem_coselect_scatter(ids, id_bytes, L, N, k, E, cosel, stream);
}
