/*
 * gemcore.h — C ABI of libgemcore.so, the B200 (sm_100a) implementation of
 * GEM's data-parallel core (arXiv 2605.19945, reference package `gemap` 0.1.0).
 *
 * Two tiers:
 *
 *  1. The reference's kernel-backend protocol (HOST pointers, synchronous).
 *     `gemap.kernels.get_backend()` returns a module with exactly three
 *     functions (/root/reference/pkg/src/gemap/kernels.py:22-47); these three
 *     entry points replace them 1:1, same argument meaning, same results bit
 *     for bit, same "(False,-1,-1,inf) when no cross pair" convention:
 *       gem_ref_eval_curve_packed      <- _kernels.pyx:58-73  eval_curve_packed
 *       gem_ref_swap_candidate_score   <- _kernels.pyx:90-117 swap_candidate_score
 *       gem_ref_best_swap              <- _kernels.pyx:120-160 best_swap
 *     They copy host buffers to the device, run, and copy the result back.
 *
 *  2. Batched DEVICE-pointer entry points (async on the caller's stream) that
 *     the Python package drives for compute_stats / score_mapping / replay /
 *     search (trace.py:87-114, mapping.py:146-208, search.py:134-312) and the
 *     new north-star paths (top-k id ingestion, co-activation, classification,
 *     thousands-of-candidates scoring).
 *
 * Conventions: every function returns 0 (GEM_OK) or a negative status; the
 * message of the last failure on the calling thread is gem_last_error().
 * `stream` is a cudaStream_t (NULL = legacy default stream). No entry point
 * allocates device memory except the host-pointer tier and the search
 * driver's internal reductions; there is no global mutable state.
 */
#ifndef GEMCORE_H
#define GEMCORE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GEM_OK 0
#define GEM_ERR_INVALID (-1)   /* bad argument (shape, size, pointer)      */
#define GEM_ERR_CUDA (-2)      /* a CUDA runtime call failed               */
#define GEM_ERR_MISMATCH (-3)  /* incremental swap score != full rescore   */
#define GEM_ERR_RANGE (-4)     /* a load exceeded the LUT / int32 range    */

/* expert classes written by gem_classify */
#define GEM_CLASS_OTHER 0
#define GEM_CLASS_CONSISTENT 1
#define GEM_CLASS_TEMPORAL 2

const char* gem_version(void);
const char* gem_last_error(void);
/* sm count, compute capability of the current device */
int gem_device_info(int* sm_count, int* cc_major, int* cc_minor);

/* ======================================================================
 * Tier 1: reference backend protocol (host pointers; kernels.py:22-47)
 * Curve arrays are the packed form built by _Instance (search.py:110-114):
 * xs_flat i64[sum S_g], ys_flat f64[sum S_g], offsets i64[G+1],
 * dense_limits i64[G].
 * ==================================================================== */
int gem_ref_eval_curve_packed(const int64_t* xs_flat, const double* ys_flat,
                              const int64_t* offsets, const int64_t* dense_limits,
                              int64_t num_gpus, int64_t gpu,
                              const int64_t* counts, int64_t n, double* out);

/* tokens i64[T,E], assignment i64[E], loads i64[T,G], lat f64[T,G] */
int gem_ref_swap_candidate_score(const int64_t* tokens, int64_t steps, int64_t experts,
                                 const int64_t* assignment, const int64_t* loads,
                                 const double* lat, int64_t num_gpus,
                                 const int64_t* xs_flat, const double* ys_flat,
                                 const int64_t* offsets, const int64_t* dense_limits,
                                 int64_t i, int64_t j, double* out);

int gem_ref_best_swap(const int64_t* tokens, int64_t steps, int64_t experts,
                      const int64_t* assignment, const int64_t* loads, const double* lat,
                      int64_t num_gpus, const int64_t* xs_flat, const double* ys_flat,
                      const int64_t* offsets, const int64_t* dense_limits,
                      int32_t* found, int64_t* best_i, int64_t* best_j, double* best_cand);

/* ======================================================================
 * Tier 2: device entry points
 * ==================================================================== */

/* --- K9: synthetic router top-k ids (test-input generator) -------------
 * ids[l][n][s] for local tokens n in [0,N) whose global index is
 * token_offset+n; step = global_token / B. Per (layer, step): consistent
 * experts (role 1) are on with probability p_consistent/2^32, temporal group
 * g (role 2+g) is jointly on with p_burst/2^32 at weight*burst_mult,
 * background (role 0) is always on. Each token draws k distinct experts
 * proportionally to the gated integer weights (Philox4x32-10, rejection of
 * repeats, deterministic fallback). id_bytes is 2 (int16) or 4 (int32). */
int gem_gen_topk(int64_t L, int64_t N, int32_t k, int32_t B, int32_t E,
                 const uint32_t* weight, const int8_t* role,
                 uint32_t p_consistent, uint32_t p_burst, uint32_t burst_mult,
                 uint64_t seed, int64_t token_offset, int32_t id_bytes, void* ids,
                 void* stream);

/* --- K1: ids -> per-step histograms + per-expert totals -----------------
 * ids [L,N,k] (int16 or int32); T = ceil(N/B) local steps per layer.
 * hist[l][t][e] = #tokens of step t that chose e (int32, [L,T,E]).
 * colsum[l][e] += sum_t hist, active[l][e] += #(hist>0),
 * heavy[l][e] += #(hist>0 and hist*E >= sum_e' hist[t][e'])  (steps in which
 * e got at least its fair share; drives the consistent-expert class),
 * dropped[l] += ids outside [0,E): these four are ACCUMULATED (zero them
 * first), so token-range shards can all-reduce them. hist rows are
 * overwritten. */
int gem_topk_hist(const void* ids, int32_t id_bytes, int64_t L, int64_t N, int32_t k,
                  int32_t B, int32_t E, int32_t* hist, int64_t* colsum, int32_t* active,
                  int32_t* heavy, int64_t* dropped, void* stream);

/* The same for one chunk of a longer trace (streamed router dumps, token-range
 * shards written into a full-length histogram): the chunk's ceil(N/B) step
 * rows of layer l go to hist + l*hist_rows*E (pass hist + t0*E for a chunk
 * that starts at step t0); hist_rows >= ceil(N/B). */
int gem_topk_hist_rows(const void* ids, int32_t id_bytes, int64_t L, int64_t N, int32_t k,
                       int32_t B, int32_t E, int32_t* hist, int64_t hist_rows, int64_t* colsum,
                       int32_t* active, int32_t* heavy, int64_t* dropped, void* stream);

/* hist [L,T,E] (int32) -> colsum/active/heavy (accumulated) — for traces
 * given as counts (ExpertTrace) instead of ids. */
int gem_hist_colstats(const int32_t* hist, int64_t L, int64_t T, int32_t E,
                      int64_t* colsum, int32_t* active, int32_t* heavy, void* stream);

/* --- K2: step-level co-activation Gram, gram[l][a][b] = sum_t h_a h_b -----
 * int64, exact (callers guarantee sum fits int64). ACCUMULATED; the upper
 * triangle a <= b is authoritative (128x128 / 64x64 tiles straddling the
 * diagonal also fill some a > b cells).
 * max_count: an upper bound on every hist value that the caller guarantees
 * (for ids: tokens_per_step * top_k), or -1 if unknown. With E a multiple of
 * 128 (<= 512) and 0 <= max_count <= 65535 the tensor-core kernel runs
 * (gem_step_gram_path() == 1: tcgen05 kind::i8 on two u8 limbs, s32 TMEM
 * accumulators, int64 combine), otherwise the CUDA-core kernel (path 0).
 * Both are exact and give identical results. */
int gem_step_gram(const int32_t* hist, int64_t L, int64_t T, int32_t E, int64_t max_count,
                  int64_t* gram, void* stream);
int gem_step_gram_path(int32_t E, int64_t max_count);
/* the two implementations, callable directly (tests, kernel benchmarks) */
int gem_step_gram_cc(const int32_t* hist, int64_t L, int64_t T, int32_t E, int64_t* gram,
                     void* stream);
int gem_step_gram_tc(const int32_t* hist, int64_t L, int64_t T, int32_t E, int64_t* gram,
                     void* stream);

/* --- K2b: token-level co-selection counts (north-star (1); no reference
 * counterpart -- its only co-activation statistic is the step-level Pearson of
 * trace.py:100-113, fed by K2) ---------------------------------------------
 * cosel[l][a][b] += #tokens of layer l whose top-k ids contain both a and b
 * (OᵀO of the 0/1 selection indicator; ids outside [0,E) ignored, a repeated
 * id within a token counts once). int32 [L,E,E], full symmetric matrix,
 * ACCUMULATED (zero it first); diag == K1's colsum when ids are distinct.
 * ids [L,N,k] int16/int32 as for gem_topk_hist. gem_coselect runs the tcgen05
 * kind::i8 kernel when gem_coselect_path() == 1 (E <= 256, k*id_bytes <= 32,
 * 16-byte aligned ids with N*k*id_bytes % 16 == 0), else the CUDA-core
 * scatter kernel; both are exact and agree bit for bit. */
int gem_coselect(const void* ids, int32_t id_bytes, int64_t L, int64_t N, int32_t k, int32_t E,
                 int32_t* cosel, void* stream);
int gem_coselect_path(const void* ids, int32_t id_bytes, int64_t N, int32_t k, int32_t E);
int gem_coselect_tc(const void* ids, int32_t id_bytes, int64_t L, int64_t N, int32_t k, int32_t E,
                    int32_t* cosel, void* stream);
int gem_coselect_scatter(const void* ids, int32_t id_bytes, int64_t L, int64_t N, int32_t k,
                         int32_t E, int32_t* cosel, void* stream);

/* --- K3: statistics finalisation (trace.py:87-114) -------------------------
 * mean_util = colsum/total, active_frac = active/T (IEEE, bit-exact);
 * corr = Pearson from exact integer statistics (0 on zero variance,
 * clamped, unit diagonal, exactly symmetric). Any output may be NULL. */
int gem_stats_finalize(const int64_t* colsum, const int32_t* active, const int64_t* gram,
                       int64_t L, int64_t T, int32_t E, double* mean_util,
                       double* active_frac, double* corr, void* stream);

/* --- K3b: consistent / temporal classification ----------------------------
 * (consistent = heavily used in almost every step,
 * temporal = heavily used only in some steps, correlated with each other)
 * consistent:  heavy*cons_den >= cons_num*T   (heavy from K1 / colstats)
 * temporal:    not consistent, heavy > 0, and r(e,f) >= corr_num/corr_den
 *              (exact int128 predicate) for some other such f
 * group:       connected components of the temporal correlation graph,
 *              labelled by their lowest expert index; -1 otherwise.
 * Asynchronous: *err_flag (device, zeroed by the caller) becomes nonzero if a
 * correlation statistic exceeds the exact int128 predicate range; the caller
 * checks it when it next reads results (no host synchronisation here). */
int gem_classify(const int64_t* colsum, const int32_t* heavy, const int64_t* gram,
                 int64_t L, int64_t T, int32_t E, int64_t cons_num, int64_t cons_den,
                 int64_t corr_num, int64_t corr_den, int8_t* cls, int16_t* group,
                 int32_t* err_flag, void* stream);

/* --- K4: curve evaluation ----------------------------------------------- */
/* out[i] = C_gpu(counts[i]) (profiles.py:157-190, _kernels.pyx:18-55);
 * asynchronous: the curve bounds offsets[gpu..gpu+1] / dense_limits[gpu] are
 * device data read by the kernel; an empty curve sets *err_flag (may be NULL)
 * to GEM_ERR_INVALID. */
int gem_eval_curve(const int64_t* xs_flat, const double* ys_flat, const int64_t* offsets,
                   const int64_t* dense_limits, int32_t gpu, const int64_t* counts, int64_t n,
                   double* out, int32_t* err_flag, void* stream);
/* equal_latency_load (profiles.py:308-333): *out = the largest n_b with
 * C_gpu_b(n_b) <= C_gpu_a(n_a), doubling then bisection saturating at
 * max_search, the reference's probe sequence on one device thread. */
int gem_equal_latency_load(const int64_t* xs_flat, const double* ys_flat, const int64_t* offsets,
                           const int64_t* dense_limits, int32_t gpu_a, int32_t gpu_b, int64_t n_a,
                           int64_t max_search, int64_t* out, void* stream);
/* lut[g][n] = C_g(n) for n in [0, nmax]  (f64 [G, nmax+1]) */
int gem_curve_lut(const int64_t* xs_flat, const double* ys_flat, const int64_t* offsets,
                  const int64_t* dense_limits, int32_t G, int64_t nmax, double* lut,
                  void* stream);

/* --- K5: straggler scoring (mapping.py:146-166) ---------------------------
 * hist [L,T,E] int32; cand [C,L,E] int8 (GPU of each expert per layer);
 * layer_scores[c][l] = serial-in-t sum of max_g lut[g][load_g(t)];
 * total[c] = serial-in-l sum of layer_scores[c][:]. Either output may be
 * NULL. Loads above nmax -> GEM_ERR_RANGE (flag set on device). */
int gem_score_batch(const int32_t* hist, int64_t L, int64_t T, int32_t E, int32_t G,
                    const int8_t* cand, int64_t C, const double* lut, int64_t nmax,
                    double* layer_scores, double* total, int32_t* err_flag, void* stream);

/* The two implementations behind gem_score_batch (which tries the first and
 * falls back to the second):
 *  - gem_score_batch_tc: candidate loads as a one-hot GEMM on tcgen05
 *    (kind::i8: u8 limbs of counts < 4096, exact s32 loads); every load is
 *    looked up in an order-key table (u16, or u32 past 65,536 distinct
 *    latencies; rows split between shared memory and a global table when too
 *    long) and each (candidate, layer) chain adds the exact fp64 value of its
 *    step maxima serially in t. Needs E in {64, 128, 256}, G in {4, 8, 16,
 *    32}. Returns 1 (nothing done) when a precondition fails. Stream-ordered
 *    scratch; ONE host sync (the launch geometry depends on the load window),
 *    two when the clamped rows hold more than 65,536 entries.
 *  - gem_score_batch_v1: CUDA cores, any shape (E <= 256). */
int gem_score_batch_tc(const int32_t* hist, int64_t L, int64_t T, int32_t E, int32_t G,
                       const int8_t* cand, int64_t C, const double* lut, int64_t nmax,
                       double* layer_scores, int32_t* err_flag, void* stream);
int gem_score_batch_v1(const int32_t* hist, int64_t L, int64_t T, int32_t E, int32_t G,
                       const int8_t* cand, int64_t C, const double* lut, int64_t nmax,
                       double* layer_scores, int32_t* err_flag, void* stream);

/* total[c] = serial-in-l sum of layer_scores[c][0..L) (cli.py:427 aggregate order) */
int gem_layer_sum(const double* layer_scores, int64_t C, int64_t L, double* total, void* stream);

/* replay of one layer under one mapping (mapping.py:169-198): per-step GPU
 * loads [T,G] (int64), latencies [T,G], step max, straggler (lowest index),
 * total (serial), busy time per GPU (serial), token totals per GPU. */
int gem_replay(const int32_t* hist, int64_t T, int32_t E, int32_t G, const int8_t* assign,
               const double* lut, int64_t nmax, int64_t* loads, double* lat, double* step_max,
               int32_t* straggler, double* total, double* busy, int64_t* gpu_tokens,
               int32_t* err_flag, void* stream);

/* --- K6/K7/K8: GEM-Place search (search.py:134-239) -----------------------
 * R runs; run r searches layer run_layer[r] of hist [L,T,E].
 * If needs_greedy[r], assign[r] is produced by the greedy placement in
 * expert order order[r][:] (search.py:134-164); otherwise assign[r] is the
 * seed mapping. Then best-swap refinement (search.py:209-239) with the
 * reference's convergence rules. Outputs: assign (in/out, int8 [R,E]),
 * trajectory f64 [R, traj_cap] (score after init and after every swap),
 * swaps [R], final_score [R]. The workspace must be at least
 * gem_search_workspace_bytes(...) bytes of device memory. */
size_t gem_search_workspace_bytes(int64_t R, int64_t T, int32_t E, int32_t G);
/* Restart orders (search.py:188-193): order[r] = the experts by descending
 * keys[r][e], ascending index on ties -- the reference's
 * np.lexsort((arange(E), -keys)). keys f64 [R, E] (the host computes them with
 * the reference's generator), order int16 [R, E]. */
int gem_restart_order(const double* keys, int64_t R, int32_t E, int16_t* order, void* stream);
int gem_search_runs(const int32_t* hist, int64_t L, int64_t T, int32_t E, int32_t G,
                    const double* lut, int64_t nmax, int64_t R, const int32_t* run_layer,
                    const uint8_t* needs_greedy, const int16_t* order, int8_t* assign,
                    double threshold, int64_t swap_cap, int64_t traj_cap, double* trajectory,
                    int32_t* swaps, double* final_score, void* workspace,
                    size_t workspace_bytes, void* stream);

/* single best-swap scan for R runs given their assignments (tests/bench) */
int gem_best_swap_runs(const int32_t* hist, int64_t L, int64_t T, int32_t E, int32_t G,
                       const double* lut, int64_t nmax, int64_t R, const int32_t* run_layer,
                       const int8_t* assign, int32_t* found, int32_t* best_i, int32_t* best_j,
                       double* best_cand, void* workspace, size_t workspace_bytes,
                       void* stream);

/* --- scale study (scale.py:100-129) ---------------------------------------
 * draws [S, nmax] f64 (host-drawn with the reference's generator), sizes [K]
 * strictly increasing in [1, nmax]: gaps[k][s] = (max - min) / max over
 * draws[s][0 .. sizes[k]) -- the mean over s is taken by the caller. */
int gem_scale_gaps(const double* draws, int64_t S, int64_t nmax, const int64_t* sizes, int32_t K,
                   double* gaps, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* GEMCORE_H */
