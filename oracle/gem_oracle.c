/*
 * gem_oracle.c — CPU ORACLE (test infrastructure only; never on the product path).
 *
 * A scalar C restatement of the reference algorithms on the GEM hot path, used
 * by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg to check
 * the CUDA kernels. Each function cites the reference code it restates:
 *   /root/reference/pkg/src/gemap/_kernels.pyx   (curve eval, best_swap, ...)
 *   /root/reference/pkg/src/gemap/search.py      (greedy, refine)
 *   /root/reference/pkg/src/gemap/mapping.py     (score, replay)
 *   /root/reference/pkg/src/gemap/trace.py       (statistics)
 * plus the north-star additions the reference does not have (top-k id
 * ingestion, co-activation Gram, classification, the Philox id generator),
 * which are defined in DESIGN.md and restated here independently of the
 * CUDA sources. Pinning: see oracle/README.md and tests/test_oracle.py.
 *
 * Build: compiled with -O2 -ffp-contract=off (the reference's own flag,
 * pkg/setup.py:17) so no FMA contraction changes a bit.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- curves */
/* _kernels.pyx:18-55 (_eval_one); profiles.py:106-135 (CostCurve.cost) */
double or_eval_one(const int64_t* xs, const double* ys, int64_t size, int64_t dense_limit, int64_t n) {
  if (n <= 0) return 0.0;
  int64_t lo = 0, hi = size;
  while (lo < hi) {
    int64_t mid = (lo + hi) / 2;
    if (xs[mid] < n) lo = mid + 1;
    else hi = mid;
  }
  int64_t idx = lo;
  if (idx < size && xs[idx] == n) return ys[idx];
  if (n <= dense_limit) return ys[idx];
  int64_t x0, x1;
  double y0, y1;
  if (idx == size) {
    if (size == 1) { x0 = 0; y0 = 0.0; }
    else { x0 = xs[size - 2]; y0 = ys[size - 2]; }
    x1 = xs[size - 1]; y1 = ys[size - 1];
  } else if (idx == 0) {
    x0 = 0; y0 = 0.0; x1 = xs[0]; y1 = ys[0];
  } else {
    x0 = xs[idx - 1]; y0 = ys[idx - 1]; x1 = xs[idx]; y1 = ys[idx];
  }
  return y0 + (y1 - y0) * (double)(n - x0) / (double)(x1 - x0);
}

static double curve(const int64_t* xs, const double* ys, const int64_t* off, const int64_t* dl, int g, int64_t n) {
  return or_eval_one(xs + off[g], ys + off[g], off[g + 1] - off[g], dl[g], n);
}

/* _kernels.pyx:58-73 */
void or_eval_curve_packed(const int64_t* xs, const double* ys, const int64_t* off, const int64_t* dl, int64_t gpu,
                          const int64_t* counts, int64_t n, double* out) {
  for (int64_t i = 0; i < n; ++i) out[i] = curve(xs, ys, off, dl, (int)gpu, counts[i]);
}

/* ---------------------------------------------------------------- scoring */
/* loads[t][g] = sum_{e: a[e]=g} tokens[t][e]   (mapping.py:146-152) */
static void load_matrix(const int64_t* tok, int64_t T, int64_t E, int64_t G, const int64_t* a, int64_t* loads) {
  memset(loads, 0, sizeof(int64_t) * T * G);
  for (int64_t t = 0; t < T; ++t)
    for (int64_t e = 0; e < E; ++e) loads[t * G + a[e]] += tok[t * E + e];
}

/* mapping.py:162-166 + _util.py:8-18: serial fp64 over steps of the row max */
double or_score(const int64_t* tok, int64_t T, int64_t E, int64_t G, const int64_t* a, const int64_t* xs,
                const double* ys, const int64_t* off, const int64_t* dl) {
  int64_t* loads = (int64_t*)malloc(sizeof(int64_t) * (T * G + 1));
  load_matrix(tok, T, E, G, a, loads);
  double total = 0.0;
  for (int64_t t = 0; t < T; ++t) {
    double m = curve(xs, ys, off, dl, 0, loads[t * G]);
    for (int64_t g = 1; g < G; ++g) {
      double v = curve(xs, ys, off, dl, (int)g, loads[t * G + g]);
      if (v > m) m = v;
    }
    total = total + m;
  }
  free(loads);
  return total;
}

/* mapping.py:169-198 (per-step arrays; the host assembles the report) */
void or_replay(const int64_t* tok, int64_t T, int64_t E, int64_t G, const int64_t* a, const int64_t* xs,
               const double* ys, const int64_t* off, const int64_t* dl, int64_t* loads, double* lat,
               double* step_max, int32_t* straggler, double* total, double* busy) {
  load_matrix(tok, T, E, G, a, loads);
  double tot = 0.0;
  for (int64_t g = 0; g < G; ++g) busy[g] = 0.0;
  for (int64_t t = 0; t < T; ++t) {
    double m = 0.0;
    int32_t arg = 0;
    for (int64_t g = 0; g < G; ++g) {
      double v = curve(xs, ys, off, dl, (int)g, loads[t * G + g]);
      lat[t * G + g] = v;
      if (g == 0 || v > m) { m = v; arg = (int32_t)g; }
      busy[g] = busy[g] + v;
    }
    step_max[t] = m;
    straggler[t] = arg;
    tot = tot + m;
  }
  *total = tot;
}

/* _kernels.pyx:76-87: pother[a][b][t] = max over g not in {a,b} of lat[t][g] */
static void pair_other_max(const double* lat, int64_t T, int64_t G, double* pother) {
  for (int64_t a = 0; a < G; ++a)
    for (int64_t b = 0; b < G; ++b)
      for (int64_t t = 0; t < T; ++t) {
        double mx = -INFINITY;
        for (int64_t g = 0; g < G; ++g)
          if (g != a && g != b && lat[t * G + g] > mx) mx = lat[t * G + g];
        pother[(a * G + b) * T + t] = mx;
      }
}

static double pair_score(const int64_t* tok, int64_t T, int64_t E, int64_t G, const int64_t* asg, const int64_t* loads,
                         const double* pother_ab, const int64_t* xs, const double* ys, const int64_t* off,
                         const int64_t* dl, int64_t i, int64_t j) {
  int a = (int)asg[i], b = (int)asg[j];
  double cand = 0.0;
  for (int64_t t = 0; t < T; ++t) {
    double la = curve(xs, ys, off, dl, a, loads[t * G + a] - tok[t * E + i] + tok[t * E + j]);
    double lb = curve(xs, ys, off, dl, b, loads[t * G + b] - tok[t * E + j] + tok[t * E + i]);
    double m = pother_ab[t];
    if (la > m) m = la;
    if (lb > m) m = lb;
    cand = cand + m;
  }
  return cand;
}

/* _kernels.pyx:90-117 */
double or_swap_candidate_score(const int64_t* tok, int64_t T, int64_t E, const int64_t* asg, const int64_t* loads,
                               const double* lat, int64_t G, const int64_t* xs, const double* ys, const int64_t* off,
                               const int64_t* dl, int64_t i, int64_t j) {
  int a = (int)asg[i], b = (int)asg[j];
  double* po = (double*)malloc(sizeof(double) * (T + 1));
  for (int64_t t = 0; t < T; ++t) {
    double m = -INFINITY;
    for (int64_t g = 0; g < G; ++g)
      if (g != a && g != b && lat[t * G + g] > m) m = lat[t * G + g];
    po[t] = m;
  }
  double s = pair_score(tok, T, E, G, asg, loads, po, xs, ys, off, dl, i, j);
  free(po);
  return s;
}

/* _kernels.pyx:120-160: first strict minimum over cross-GPU pairs i<j */
int or_best_swap(const int64_t* tok, int64_t T, int64_t E, const int64_t* asg, const int64_t* loads, const double* lat,
                 int64_t G, const int64_t* xs, const double* ys, const int64_t* off, const int64_t* dl,
                 int64_t* bi, int64_t* bj, double* bc) {
  double* pother = (double*)malloc(sizeof(double) * (G * G * T + 1));
  pair_other_max(lat, T, G, pother);
  double best = INFINITY;
  int64_t best_i = -1, best_j = -1;
  for (int64_t i = 0; i < E; ++i) {
    int64_t a = asg[i];
    for (int64_t j = i + 1; j < E; ++j) {
      int64_t b = asg[j];
      if (b == a) continue;
      double cand = pair_score(tok, T, E, G, asg, loads, pother + (a * G + b) * T, xs, ys, off, dl, i, j);
      if (cand < best) { best = cand; best_i = i; best_j = j; }
    }
  }
  free(pother);
  *bi = best_i;
  *bj = best_j;
  *bc = best_i < 0 ? INFINITY : best;
  return best_i >= 0;
}

/* search.py:134-164 (_greedy_assignment): lat starts at 0.0; strict < lowest g */
void or_greedy(const int64_t* tok, int64_t T, int64_t E, int64_t G, const int64_t* xs, const double* ys,
               const int64_t* off, const int64_t* dl, const int64_t* order, int64_t* asg) {
  int64_t cap = E / G;
  int64_t* loads = (int64_t*)calloc((size_t)(T * G + 1), sizeof(int64_t));
  double* lat = (double*)calloc((size_t)(T * G + 1), sizeof(double));
  double* cand = (double*)malloc(sizeof(double) * (T + 1));
  double* best_lat = (double*)malloc(sizeof(double) * (T + 1));
  int64_t* counts = (int64_t*)calloc((size_t)G + 1, sizeof(int64_t));
  for (int64_t e = 0; e < E; ++e) asg[e] = -1;
  for (int64_t k = 0; k < E; ++k) {
    int64_t e = order[k];
    int64_t best_gpu = -1;
    double best_score = INFINITY;
    for (int64_t g = 0; g < G; ++g) {
      if (counts[g] == cap) continue;
      double score = 0.0;
      for (int64_t t = 0; t < T; ++t) {
        double cl = curve(xs, ys, off, dl, (int)g, loads[t * G + g] + tok[t * E + e]);
        cand[t] = cl;
        double sc = cl;
        if (G > 1) {
          double others = -INFINITY;
          for (int64_t h = 0; h < G; ++h)
            if (h != g && lat[t * G + h] > others) others = lat[t * G + h];
          sc = others > cl ? others : cl;
        }
        score = score + sc;
      }
      if (score < best_score) {
        best_score = score;
        best_gpu = g;
        memcpy(best_lat, cand, sizeof(double) * T);
      }
    }
    asg[e] = best_gpu;
    counts[best_gpu] += 1;
    for (int64_t t = 0; t < T; ++t) {
      loads[t * G + best_gpu] += tok[t * E + e];
      lat[t * G + best_gpu] = best_lat[t];
    }
  }
  free(loads); free(lat); free(cand); free(best_lat); free(counts);
}

static double full_score_from_loads(const int64_t* loads, int64_t T, int64_t G, const int64_t* xs, const double* ys,
                                    const int64_t* off, const int64_t* dl, double* lat) {
  double s = 0.0;
  for (int64_t t = 0; t < T; ++t) {
    double m = 0.0;
    for (int64_t g = 0; g < G; ++g) {
      double v = curve(xs, ys, off, dl, (int)g, loads[t * G + g]);
      lat[t * G + g] = v;
      if (g == 0 || v > m) m = v;
    }
    s = s + m;
  }
  return s;
}

/* search.py:209-239 (_refine_assignment). Returns swaps; -1 on a rescore mismatch. */
int64_t or_refine(const int64_t* tok, int64_t T, int64_t E, int64_t G, const int64_t* xs, const double* ys,
                  const int64_t* off, const int64_t* dl, int64_t* asg, double threshold, int64_t cap,
                  double* traj, int64_t traj_cap, double* final_score) {
  int64_t* loads = (int64_t*)malloc(sizeof(int64_t) * (T * G + 1));
  double* lat = (double*)malloc(sizeof(double) * (T * G + 1));
  load_matrix(tok, T, E, G, asg, loads);
  double score = full_score_from_loads(loads, T, G, xs, ys, off, dl, lat);
  if (traj_cap > 0) traj[0] = score;
  int64_t swaps = 0;
  int mismatch = 0;
  while (swaps < cap) {
    int64_t i, j;
    double cand;
    int found = or_best_swap(tok, T, E, asg, loads, lat, G, xs, ys, off, dl, &i, &j, &cand);
    if (!found || !(cand < score)) break;
    if (1.0 - cand / score < threshold) break;
    int64_t a = asg[i], b = asg[j];
    asg[i] = b;
    asg[j] = a;
    for (int64_t t = 0; t < T; ++t) {
      int64_t d = tok[t * E + j] - tok[t * E + i];
      loads[t * G + a] += d;
      loads[t * G + b] -= d;
    }
    score = full_score_from_loads(loads, T, G, xs, ys, off, dl, lat);
    if (score != cand) mismatch = 1;
    swaps += 1;
    if (swaps < traj_cap) traj[swaps] = score;
  }
  *final_score = score;
  free(loads);
  free(lat);
  return mismatch ? -1 : swaps;
}

/* ------------------------------------------------------------ statistics */
/* exact integer statistics of trace.py:87-114 */
/* colsum, active = #(h>0) (trace.py:95-98), and heavy = #(h>0 and h*E >=
 * row total): the steps in which e received at least its fair share
 * (the consistent-expert statistic). */
void or_colstats(const int64_t* tok, int64_t T, int64_t E, int64_t* colsum, int64_t* active, int64_t* heavy) {
  for (int64_t e = 0; e < E; ++e) { colsum[e] = 0; active[e] = 0; heavy[e] = 0; }
  for (int64_t t = 0; t < T; ++t) {
    int64_t row = 0;
    for (int64_t e = 0; e < E; ++e) row += tok[t * E + e];
    for (int64_t e = 0; e < E; ++e) {
      const int64_t h = tok[t * E + e];
      colsum[e] += h;
      active[e] += h > 0;
      heavy[e] += h > 0 && h * E >= row;
    }
  }
}

void or_gram(const int64_t* tok, int64_t T, int64_t E, int64_t* gram) {
  memset(gram, 0, sizeof(int64_t) * E * E);
  for (int64_t t = 0; t < T; ++t)
    for (int64_t a = 0; a < E; ++a) {
      int64_t ha = tok[t * E + a];
      if (!ha) continue;
      for (int64_t b = 0; b < E; ++b) gram[a * E + b] += ha * tok[t * E + b];
    }
}

/* classification: consistent = active*cd >= cn*T;
 * temporal = not consistent and r >= rn/rd with another non-consistent expert;
 * group = connected component (lowest index). Returns 0, or 1 on range overflow. */
/* consistent: heavy in >= cn/cd of the steps; temporal: not consistent,
 * heavy in some step, Pearson r >= rn/rd with another such expert (exact
 * int128 predicate); groups = connected components, lowest index labels. */
int or_classify(const int64_t* colsum, const int64_t* heavy, const int64_t* gram, int64_t T, int64_t E,
                int64_t cn, int64_t cd, int64_t rn, int64_t rd, int8_t* cls, int16_t* group) {
  typedef __int128 i128;
  const i128 lim = (i128)1 << 60;
  int err = 0;
  unsigned char* adj = (unsigned char*)calloc((size_t)(E * E + 1), 1);
  /* 3 = burst candidate (heavy somewhere, not consistent) until confirmed */
  for (int64_t e = 0; e < E; ++e) cls[e] = ((i128)heavy[e] * cd >= (i128)cn * T) ? 1 : (heavy[e] > 0 ? 3 : 0);
  for (int64_t a = 0; a < E; ++a)
    for (int64_t b = a + 1; b < E; ++b) {
      if (cls[a] != 3 || cls[b] != 3) continue;
      i128 sa = colsum[a], sb = colsum[b];
      i128 va = (i128)T * gram[a * E + a] - sa * sa;
      i128 vb = (i128)T * gram[b * E + b] - sb * sb;
      if (va == 0 || vb == 0) continue;
      i128 num = (i128)T * gram[a * E + b] - sa * sb;
      if (num <= 0) continue;
      if (num >= lim || va >= lim || vb >= lim) { err = 1; continue; }
      if ((i128)(rd * rd) * (num * num) >= (i128)(rn * rn) * (va * vb)) adj[a * E + b] = adj[b * E + a] = 1;
    }
  int32_t* label = (int32_t*)malloc(sizeof(int32_t) * (E + 1));
  for (int64_t e = 0; e < E; ++e) {
    int any = 0;
    for (int64_t f = 0; f < E; ++f) any |= adj[e * E + f];
    if (cls[e] == 3) cls[e] = any ? 2 : 0;
    label[e] = cls[e] == 2 ? (int32_t)e : -1;
  }
  /* connected components by repeated min-label relaxation */
  int changed = 1;
  while (changed) {
    changed = 0;
    for (int64_t e = 0; e < E; ++e) {
      if (label[e] < 0) continue;
      for (int64_t f = 0; f < E; ++f)
        if (adj[e * E + f] && label[f] < label[e]) { label[e] = label[f]; changed = 1; }
    }
  }
  for (int64_t e = 0; e < E; ++e) group[e] = (int16_t)label[e];
  free(adj);
  free(label);
  return err;
}

/* ------------------------------------------------------ top-k ingestion */
/* hist[l][t][e] = #{n in step t, s : ids[l][n][s] == e}; ids outside [0,E) dropped */
void or_topk_hist(const void* ids, int id_bytes, int64_t L, int64_t N, int64_t k, int64_t B, int64_t E,
                  int64_t* hist, int64_t* dropped) {
  int64_t T = (N + B - 1) / B;
  memset(hist, 0, sizeof(int64_t) * L * T * E);
  for (int64_t l = 0; l < L; ++l) {
    dropped[l] = 0;
    for (int64_t n = 0; n < N; ++n)
      for (int64_t s = 0; s < k; ++s) {
        int64_t idx = (l * N + n) * k + s;
        uint32_t id = id_bytes == 2 ? (uint32_t)((const uint16_t*)ids)[idx] : ((const uint32_t*)ids)[idx];
        if (id < (uint32_t)E) hist[(l * T + n / B) * E + id] += 1;
        else dropped[l] += 1;
      }
  }
}

/* ------------------------------------------------------ Philox generator */
/* Philox4x32-10 (Salmon et al., SC'11), written independently of csrc/ */
static void philox10(uint32_t c[4], uint32_t k0, uint32_t k1) {
  for (int r = 0; r < 10; ++r) {
    uint64_t p0 = (uint64_t)0xD2511F53u * c[0];
    uint64_t p1 = (uint64_t)0xCD9E8D57u * c[2];
    uint32_t n0 = (uint32_t)(p1 >> 32) ^ c[1] ^ k0;
    uint32_t n1 = (uint32_t)p1;
    uint32_t n2 = (uint32_t)(p0 >> 32) ^ c[3] ^ k1;
    uint32_t n3 = (uint32_t)p0;
    c[0] = n0; c[1] = n1; c[2] = n2; c[3] = n3;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
}

void or_philox4x32_10(const uint32_t ctr[4], uint32_t k0, uint32_t k1, uint32_t out[4]) {
  uint32_t c[4] = {ctr[0], ctr[1], ctr[2], ctr[3]};
  philox10(c, k0, k1);
  memcpy(out, c, sizeof(c));
}

static uint32_t draw(uint64_t seed, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  uint32_t ctr[4] = {a, b, c, d};
  philox10(ctr, (uint32_t)seed, (uint32_t)(seed >> 32));
  return ctr[0];
}

/* the generator contract of gem_gen_topk (include/gemcore.h) */
/* layers [layer0, layer0 + L) of the trace (weight/role rows of those layers) */
void or_gen_topk_l(int64_t L, int64_t layer0, int64_t N, int64_t k, int64_t B, int64_t E, const uint32_t* weight,
                   const int8_t* role, uint32_t p_cons, uint32_t p_burst, uint32_t burst_mult, uint64_t seed,
                   int64_t token_offset, int id_bytes, void* ids);

void or_gen_topk(int64_t L, int64_t N, int64_t k, int64_t B, int64_t E, const uint32_t* weight, const int8_t* role,
                 uint32_t p_cons, uint32_t p_burst, uint32_t burst_mult, uint64_t seed, int64_t token_offset,
                 int id_bytes, void* ids) {
  or_gen_topk_l(L, 0, N, k, B, E, weight, role, p_cons, p_burst, burst_mult, seed, token_offset, id_bytes, ids);
}

void or_gen_topk_l(int64_t L, int64_t layer0, int64_t N, int64_t k, int64_t B, int64_t E, const uint32_t* weight,
                   const int8_t* role, uint32_t p_cons, uint32_t p_burst, uint32_t burst_mult, uint64_t seed,
                   int64_t token_offset, int id_bytes, void* ids) {
  uint64_t* w = (uint64_t*)malloc(sizeof(uint64_t) * (E + 1));
  uint64_t* cdf = (uint64_t*)malloc(sizeof(uint64_t) * (E + 1));
  int64_t chosen[64];
  int64_t cur_step = -1;
  for (int64_t l = 0; l < L; ++l) {
    cur_step = -1;
    for (int64_t n = 0; n < N; ++n) {
      int64_t gt = token_offset + n;
      int64_t step = gt / B;
      if (step != cur_step) {
        cur_step = step;
        for (int64_t e = 0; e < E; ++e) {
          int r = role[l * E + e];
          uint64_t v = weight[l * E + e];
          if (r == 1) {
            if (draw(seed, (uint32_t)step, (uint32_t)(step >> 32), (uint32_t)(l + layer0), 0x80000000u | (uint32_t)e) >= p_cons) v = 0;
          } else if (r >= 2) {
            if (draw(seed, (uint32_t)step, (uint32_t)(step >> 32), (uint32_t)(l + layer0), 0xC0000000u | (uint32_t)(r - 2)) < p_burst)
              v *= burst_mult;
            else
              v = 0;
          }
          w[e] = v;
        }
        uint64_t run = 0;
        for (int64_t e = 0; e < E; ++e) { run += w[e]; cdf[e] = run; }
      }
      uint64_t total = cdf[E - 1];
      for (int64_t s = 0; s < k; ++s) {
        int64_t pick = -1;
        if (total > 0) {
          for (int a = 0; a < 32 && pick < 0; ++a) {
            uint32_t u = draw(seed, (uint32_t)gt, (uint32_t)(gt >> 32), (uint32_t)(l + layer0), (uint32_t)(s * 64 + a));
            uint64_t r = ((uint64_t)u * total) >> 32;
            int64_t e = 0;
            while (cdf[e] <= r) ++e; /* first e with cdf[e] > r */
            int dup = 0;
            for (int64_t q = 0; q < s; ++q) dup |= chosen[q] == e;
            if (!dup) pick = e;
          }
        }
        for (int pass = 0; pass < 2 && pick < 0; ++pass)
          for (int64_t e = 0; e < E && pick < 0; ++e) {
            if (pass == 0 && w[e] == 0) continue;
            int dup = 0;
            for (int64_t q = 0; q < s; ++q) dup |= chosen[q] == e;
            if (!dup) pick = e;
          }
        chosen[s] = pick;
        int64_t idx = (l * N + n) * k + s;
        if (id_bytes == 2) ((int16_t*)ids)[idx] = (int16_t)pick;
        else ((int32_t*)ids)[idx] = (int32_t)pick;
      }
    }
  }
  free(w);
  free(cdf);
}
