/*
 * ORACLE / TEST INFRASTRUCTURE — not product code. See bfsim_oracle.h.
 *
 * Plain-C restatement of the reference's hot path. Each function cites the
 * reference file:line it follows (paths relative to
 * /root/reference/proj/include/bfsim/). Compiled with -ffp-contract=off so
 * dt = C + t*max and r2 = x*x + y*y round exactly as the reference build
 * (SURVEY.md F6). Integer-valued loads are carried in int64 (F5); the
 * reference's double arithmetic on them is exact below 2^53.
 *
 * Deliberately simple data structures (insertion-ordered per-worker lists,
 * an ordered waiting array): this is the checker, not the product.
 */
#include "bfsim_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---------------- libstdc++ <random> restatements ---------------- */

#define MT_N 312
#define MT_M 156
#define MT_A 0xB5026F5AA96619E9ULL
#define MT_UPPER 0xFFFFFFFF80000000ULL
#define MT_LOWER 0x000000007FFFFFFFULL

/* mersenne_twister_engine::seed (bits/random.tcc, mt19937_64 parameters). */
void oracle_mt64_seed(oracle_mt64_t* g, uint64_t seed) {
  g->mt[0] = seed;
  for (int i = 1; i < MT_N; ++i) {
    uint64_t x = g->mt[i - 1];
    g->mt[i] = 6364136223846793005ULL * (x ^ (x >> 62)) + (uint64_t)i;
  }
  g->idx = MT_N;
}

static void mt64_twist(oracle_mt64_t* g) {
  for (int i = 0; i < MT_N; ++i) {
    uint64_t x = (g->mt[i] & MT_UPPER) | (g->mt[(i + 1) % MT_N] & MT_LOWER);
    uint64_t xa = x >> 1;
    if (x & 1ULL) xa ^= MT_A;
    g->mt[i] = g->mt[(i + MT_M) % MT_N] ^ xa;
  }
  g->idx = 0;
}

uint64_t oracle_mt64_next(oracle_mt64_t* g) {
  if (g->idx >= MT_N) mt64_twist(g);
  uint64_t y = g->mt[g->idx++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= y >> 43;
  return y;
}

/* generate_canonical<double,53> with a 64-bit engine: one call, (double)u / 2^64,
 * clamped below 1 (random.tcc:3349-3381). */
double oracle_canonical(oracle_mt64_t* g) {
  double r = (double)oracle_mt64_next(g) / 18446744073709551616.0;
  if (r >= 1.0) r = nextafter(1.0, 0.0);
  return r;
}

/* normal_distribution polar method, fresh object per call (no saved value),
 * random.tcc:1809-1844; called from make_preview, policies.hpp:75. */
double oracle_normal(oracle_mt64_t* g, double mean, double sigma) {
  double x, y, r2;
  do {
    x = 2.0 * oracle_canonical(g) - 1.0;
    y = 2.0 * oracle_canonical(g) - 1.0;
    r2 = x * x + y * y;
  } while (r2 > 1.0 || r2 == 0.0);
  double mult = sqrt(-2 * log(r2) / r2);
  double ret = y * mult;
  return ret * sigma + mean;
}

/* ---------------- policy operator (policies.hpp) ---------------- */

typedef struct {
  const double* w; /* preview w[0..H] */
} pv_ref_t;

/* fcfs_assign, policies.hpp:100-114. */
static int64_t assign_fcfs(int n_waiting, int G, const int32_t* caps, int32_t* pairs) {
  int32_t* cap = (int32_t*)malloc(sizeof(int32_t) * (size_t)(G > 0 ? G : 1));
  long free_total = 0;
  for (int g = 0; g < G; ++g) {
    cap[g] = caps[g];
    free_total += caps[g];
  }
  int64_t u = 0;
  for (int i = 0; i < n_waiting && free_total > 0; ++i) {
    int best = -1;
    for (int g = 0; g < G; ++g)
      if (best < 0 || cap[g] > cap[best]) best = g;
    pairs[2 * u] = i;
    pairs[2 * u + 1] = best;
    ++u;
    --cap[best];
    --free_total;
  }
  free(cap);
  return u;
}

/* jsq_assign, policies.hpp:118-138. */
static int64_t assign_jsq(int n_waiting, int G, const int32_t* caps, const int32_t* counts,
                          int32_t* pairs) {
  int32_t* cap = (int32_t*)malloc(sizeof(int32_t) * (size_t)(2 * (G > 0 ? G : 1)));
  int32_t* cnt = cap + G;
  for (int g = 0; g < G; ++g) {
    cap[g] = caps[g];
    cnt[g] = counts[g];
  }
  int64_t u = 0;
  for (int i = 0; i < n_waiting; ++i) {
    int best = -1;
    for (int g = 0; g < G; ++g) {
      if (cap[g] <= 0) continue;
      if (best < 0 || cnt[g] < cnt[best]) best = g;
    }
    if (best < 0) break;
    pairs[2 * u] = i;
    pairs[2 * u + 1] = best;
    ++u;
    --cap[best];
    ++cnt[best];
  }
  free(cap);
  return u;
}

static const double* g_sort_w0; /* qsort context */
typedef struct {
  double w0;
  int idx;
  int seq;
} sort_item_t;
static int cmp_w0_asc_stable(const void* a, const void* b) {
  const sort_item_t* x = (const sort_item_t*)a;
  const sort_item_t* y = (const sort_item_t*)b;
  if (x->w0 < y->w0) return -1;
  if (x->w0 > y->w0) return 1;
  return x->seq - y->seq;
}
static int cmp_w0_desc_stable(const void* a, const void* b) {
  const sort_item_t* x = (const sort_item_t*)a;
  const sort_item_t* y = (const sort_item_t*)b;
  if (x->w0 > y->w0) return -1;
  if (x->w0 < y->w0) return 1;
  return x->seq - y->seq;
}
static int cmp_pair(const void* a, const void* b) {
  const int32_t* x = (const int32_t*)a;
  const int32_t* y = (const int32_t*)b;
  if (x[0] != y[0]) return x[0] - y[0];
  return x[1] - y[1];
}

/* bfio_assign_greedy, policies.hpp:269-370.
 * Phase 1 (:274-323) literally: stable sort by w0 ascending, pick the last
 * unused entry with w0 <= deficit, else the first unused entry.
 * Sort of the selection by w0 descending, stable (:324-326).
 * Phase 2 (:339-367) in the restated O(G*(H+1)) form: the
 * horizon cost after adding preview w to worker g is, up to a g-independent
 * term, G * sum_h max(M_h, F_h[g] + w_h) with M_h the max over ALL workers;
 * ties break on (loads[0][g], g) exactly as :355. Exact for integer-valued
 * doubles (F5). Assignments sorted by (waiting idx, worker) (:368). */
static int64_t assign_greedy(int n_waiting, const pv_ref_t* waiting, int G, const int32_t* caps,
                             const double* futures, int H, int32_t* pairs) {
  const int H1 = H + 1;
  long total_cap = 0;
  for (int g = 0; g < G; ++g) total_cap += caps[g];
  long U = n_waiting < total_cap ? n_waiting : total_cap;
  int* order = (int*)malloc(sizeof(int) * (size_t)(U > 0 ? U : 1));
  long n_order = 0;
  if ((long)n_waiting == U) {
    for (long i = 0; i < U; ++i) order[n_order++] = (int)i;
  } else {
    double* load = (double*)malloc(sizeof(double) * (size_t)G);
    int* fs = (int*)malloc(sizeof(int) * (size_t)G);
    double target = 0.0;
    for (int g = 0; g < G; ++g) {
      load[g] = futures[(size_t)g * H1];
      fs[g] = caps[g];
      if (load[g] > target) target = load[g];
    }
    sort_item_t* by = (sort_item_t*)malloc(sizeof(sort_item_t) * (size_t)n_waiting);
    for (int i = 0; i < n_waiting; ++i) {
      by[i].w0 = waiting[i].w[0];
      by[i].idx = i;
      by[i].seq = i;
    }
    qsort(by, (size_t)n_waiting, sizeof(sort_item_t), cmp_w0_asc_stable);
    char* used = (char*)calloc((size_t)n_waiting, 1);
    for (long left = U; left > 0; --left) {
      int g = -1;
      for (int j = 0; j < G; ++j)
        if (fs[j] > 0 && (g < 0 || load[j] < load[g])) g = j;
      if (g < 0) break;
      double deficit = target - load[g];
      int pick = -1;
      for (int j = n_waiting - 1; j >= 0; --j) {
        if (used[j]) continue;
        if (by[j].w0 <= deficit) {
          pick = j;
          break;
        }
      }
      if (pick < 0)
        for (int j = 0; j < n_waiting; ++j)
          if (!used[j]) {
            pick = j;
            break;
          }
      if (pick < 0) break;
      used[pick] = 1;
      int i = by[pick].idx;
      order[n_order++] = i;
      load[g] += waiting[i].w[0];
      if (load[g] > target) target = load[g];
      --fs[g];
    }
    free(used);
    free(by);
    free(fs);
    free(load);
  }
  /* stable sort by w0 descending */
  sort_item_t* ord = (sort_item_t*)malloc(sizeof(sort_item_t) * (size_t)(n_order > 0 ? n_order : 1));
  for (long j = 0; j < n_order; ++j) {
    ord[j].w0 = waiting[order[j]].w[0];
    ord[j].idx = order[j];
    ord[j].seq = (int)j;
  }
  qsort(ord, (size_t)n_order, sizeof(sort_item_t), cmp_w0_desc_stable);

  /* phase 2 */
  int32_t* cap = (int32_t*)malloc(sizeof(int32_t) * (size_t)G);
  double* F = (double*)malloc(sizeof(double) * (size_t)G * H1); /* [g][h] */
  double* M = (double*)malloc(sizeof(double) * (size_t)H1);
  for (int h = 0; h < H1; ++h) M[h] = 0.0;
  for (int g = 0; g < G; ++g) {
    cap[g] = caps[g];
    for (int h = 0; h < H1; ++h) {
      F[(size_t)g * H1 + h] = futures[(size_t)g * H1 + h];
      if (F[(size_t)g * H1 + h] > M[h]) M[h] = F[(size_t)g * H1 + h];
    }
  }
  int64_t u = 0;
  for (long j = 0; j < n_order; ++j) {
    const double* w = waiting[ord[j].idx].w;
    int best = -1;
    double best_c = 0.0, best_l = 0.0;
    for (int g = 0; g < G; ++g) {
      if (cap[g] <= 0) continue;
      double c = 0.0;
      for (int h = 0; h < H1; ++h) {
        double v = F[(size_t)g * H1 + h] + w[h];
        c += v > M[h] ? v : M[h];
      }
      double l = F[(size_t)g * H1];
      if (best < 0 || c < best_c || (c == best_c && l < best_l)) {
        best = g;
        best_c = c;
        best_l = l;
      }
    }
    if (best < 0) break;
    pairs[2 * u] = ord[j].idx;
    pairs[2 * u + 1] = best;
    ++u;
    --cap[best];
    for (int h = 0; h < H1; ++h) {
      double v = F[(size_t)best * H1 + h] + w[h];
      F[(size_t)best * H1 + h] = v;
      if (v > M[h]) M[h] = v;
    }
  }
  qsort(pairs, (size_t)u, 2 * sizeof(int32_t), cmp_pair);
  free(M);
  free(F);
  free(cap);
  free(ord);
  free(order);
  return u;
}

int oracle_assign(int policy, int n_waiting, const double* previews, int G, const int32_t* caps,
                  const int32_t* active_counts, const double* futures, int H, int32_t* pairs,
                  int64_t* n_pairs) {
  switch (policy) {
    case BFSIM_POLICY_FCFS:
      *n_pairs = assign_fcfs(n_waiting, G, caps, pairs);
      return BFSIM_OK;
    case BFSIM_POLICY_JSQ:
      *n_pairs = assign_jsq(n_waiting, G, caps, active_counts, pairs);
      return BFSIM_OK;
    case BFSIM_POLICY_BFIO_GREEDY: {
      pv_ref_t* pv = (pv_ref_t*)malloc(sizeof(pv_ref_t) * (size_t)(n_waiting > 0 ? n_waiting : 1));
      for (int i = 0; i < n_waiting; ++i) pv[i].w = previews + (size_t)i * (H + 1);
      *n_pairs = assign_greedy(n_waiting, pv, G, caps, futures, H, pairs);
      free(pv);
      return BFSIM_OK;
    }
    default:
      return BFSIM_EINVAL;
  }
}

/* ---------------- simulation state ---------------- */

/* make_preview, policies.hpp:67-90, for a request with prefill s, decode o,
 * integer drift d (profile[j] = s + d*j, drift_profile workload.hpp:73-85). */
static void make_preview(double* w, int64_t s, int64_t o, int64_t d, int64_t tau, int H, int mode,
                         double sigma, oracle_mt64_t* rng) {
  int64_t remaining = o - tau;
  int64_t predicted = remaining;
  if (mode == BFSIM_LOOKAHEAD_NOISY && rng != NULL && sigma > 0.0) {
    double n = oracle_normal(rng, 0.0, sigma);
    int64_t r = remaining + lround(n);
    predicted = r > 1 ? r : 1;
  } else if (mode == BFSIM_LOOKAHEAD_TRUNCATED) {
    predicted = remaining > (int64_t)H + 1 ? remaining : (int64_t)H + 1;
  }
  w[0] = (double)(s + d * tau);
  for (int h = 1; h <= H; ++h) {
    if (h < predicted) {
      int64_t j = tau + h < o - 1 ? tau + h : o - 1;
      w[h] = (double)(s + d * j);
    } else {
      w[h] = 0.0;
    }
  }
}

static int drift_ok(double drift) {
  return drift >= 0.0 && drift == floor(drift) && drift < 1e9;
}

static int power_ok(const bfsim_scenario_t* sc) {
  /* PowerModel::validate, metrics_power.hpp:17-21 */
  if (!(sc->p_idle > 0.0 && sc->p_idle < sc->p_max)) return 0;
  if (!(sc->mfu_sat > 0.0 && sc->mfu_sat <= 1.0)) return 0;
  if (!(sc->gamma > 0.0 && sc->gamma < 1.0)) return 0;
  return 1;
}

/* power(), metrics_power.hpp:24-27 */
static double power_of(double u, const bfsim_scenario_t* sc) {
  return sc->p_idle + (sc->p_max - sc->p_idle) * pow(u, sc->gamma);
}

/* Per-step accounting of compute_metrics (metrics.hpp:17-76,106-122) done as
 * running sums in the reference's summation order. */
typedef struct {
  double imb_acc;   /* avg_imbalance accumulator (metrics.hpp:24-29) */
  double tokens;    /* throughput (metrics.hpp:32-40) */
  double elapsed;
  double energy;    /* energy (metrics.hpp:67-76) */
  double imb_total; /* compute_metrics :116-121 */
  double workload;
  int64_t imb_i, work_i, tok_i;
  int64_t records;
} acct_t;

static void acct_step(acct_t* a, const int64_t* L, int G, int64_t mx, int64_t ac, double dt,
                      const bfsim_scenario_t* sc) {
  double sum = 0.0, mxd = 0.0;
  int64_t sum_i = 0;
  for (int g = 0; g < G; ++g) {
    double l = (double)L[g];
    if (l > mxd) mxd = l;
    sum += l;
    sum_i += L[g];
  }
  double imb = (double)G * mxd - sum; /* imbalance(), metrics.hpp:17-22 */
  a->imb_acc += imb;
  a->tokens += (double)ac;
  a->elapsed += dt;
  /* utilization (metrics.hpp:56-62) + energy (:67-76) */
  double p = 0.0;
  for (int g = 0; g < G; ++g) {
    double u = mxd > 0.0 ? (double)L[g] / mxd : 0.0;
    p += power_of(u, sc);
  }
  a->energy += dt * p;
  a->imb_total += imb;
  a->workload += sum;
  a->imb_i += (int64_t)G * mx - sum_i;
  a->work_i += sum_i;
  a->tok_i += ac;
  a->records += 1;
}

/* compute_metrics, metrics.hpp:106-122 (tpot 0 when nothing completed). */
static void acct_finish(const acct_t* a, double tpot_sum, int64_t tpot_n, bfsim_result_t* r) {
  r->imb_total_i = a->imb_i;
  r->total_workload_i = a->work_i;
  r->tokens_i = a->tok_i;
  r->records = a->records;
  r->elapsed = a->elapsed;
  r->tpot_sum = tpot_sum;
  if (a->records == 0) {
    r->flags |= BFSIM_FLAG_EMPTY;
    return; /* tools/bfsim.cpp:133-137: MetricsReport{} */
  }
  r->avg_imbalance = a->imb_acc / (double)a->records;
  r->throughput = a->tokens / a->elapsed;
  r->tpot = tpot_n > 0 ? tpot_sum / (double)tpot_n : 0.0;
  r->energy = a->energy;
  r->imb_total = a->imb_total;
  r->total_workload = a->workload;
  r->eta_sum = a->workload > 0.0 ? a->imb_total / a->workload : 0.0;
}

/* ---------------- Simulation::run (engine.hpp:95-188) ---------------- */

int oracle_run_poisson(const bfsim_scenario_t* sc, const bfsim_request_t* trace, int64_t n,
                       int64_t step_cap, double* o_clock_start, double* o_dt, double* o_max_load,
                       int64_t* o_active_count, double* o_loads, int32_t* o_arrival_step,
                       int32_t* o_start_step, int32_t* o_worker, double* o_admit_clock,
                       double* o_finish_clock, bfsim_result_t* res) {
  memset(res, 0, sizeof(*res));
  const int G = sc->workers, B = sc->batch, H = sc->horizon, H1 = sc->horizon + 1;
  /* SimConfig::validate, engine.hpp:31-36 */
  if (G < 1 || B < 1 || sc->overhead < 0.0 || sc->per_token <= 0.0 || H < 0 || sc->max_steps < 1 ||
      !power_ok(sc) || !drift_ok(sc->drift) || sc->policy == BFSIM_POLICY_BFIO_EXACT ||
      sc->policy < 0 || sc->policy > 3) {
    res->status = BFSIM_EINVAL;
    return BFSIM_EINVAL;
  }
  const int64_t d = (int64_t)sc->drift;
  const int need_views = sc->policy == BFSIM_POLICY_BFIO_GREEDY;

  int64_t* x = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1)); /* start step */
  int32_t* wk = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
  double* admit = (double*)calloc((size_t)(n > 0 ? n : 1), sizeof(double));
  double* finish = (double*)calloc((size_t)(n > 0 ? n : 1), sizeof(double));
  int32_t* arr_step = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
  char* done = (char*)calloc((size_t)(n > 0 ? n : 1), 1);
  for (int64_t i = 0; i < n; ++i) {
    x[i] = -1;
    wk[i] = -1;
    arr_step[i] = -1;
  }
  int64_t* act = (int64_t*)malloc(sizeof(int64_t) * (size_t)G * B); /* active_[g], insertion order */
  int32_t* nact = (int32_t*)calloc((size_t)G, sizeof(int32_t));
  int64_t* waiting = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
  int64_t nw = 0;
  int64_t* L = (int64_t*)malloc(sizeof(int64_t) * (size_t)G);
  int32_t* caps = (int32_t*)malloc(sizeof(int32_t) * (size_t)G);
  int32_t* cnts = (int32_t*)malloc(sizeof(int32_t) * (size_t)G);
  double* fut = (double*)malloc(sizeof(double) * (size_t)G * H1);
  double* pvbuf = NULL;
  pv_ref_t* pvs = NULL;
  int32_t* pairs = (int32_t*)malloc(sizeof(int32_t) * 2 * (size_t)G * B);
  char* taken = NULL;
  double* tmpw = (double*)malloc(sizeof(double) * (size_t)H1);
  oracle_mt64_t* rng = (oracle_mt64_t*)malloc(sizeof(oracle_mt64_t));
  oracle_mt64_seed(rng, sc->seed); /* rng_(config.seed), engine.hpp:98 */

  acct_t acct;
  memset(&acct, 0, sizeof(acct));
  double clock = 0.0;
  int64_t nxt = 0, n_done = 0, k = 0;
  int status = BFSIM_OK;
  for (;;) {
    /* while (!all_done() && steps < max_steps), engine.hpp:171 */
    if (n_done == n) break;
    if (k >= sc->max_steps) {
      status = BFSIM_PARTIAL;
      break;
    }
    /* reveal, engine.hpp:123-128 */
    while (nxt < n && trace[nxt].arrival_time <= clock) {
      arr_step[nxt] = (int32_t)k;
      waiting[nw++] = nxt;
      ++nxt;
    }
    /* views, engine.hpp:204-231. GCC evaluates assign()'s arguments right to
     * left, so worker_views draws before waiting_views. */
    for (int g = 0; g < G; ++g) {
      caps[g] = B - nact[g];
      cnts[g] = nact[g];
      for (int h = 0; h < H1; ++h) fut[(size_t)g * H1 + h] = 0.0;
      if (!need_views) continue;
      for (int j = 0; j < nact[g]; ++j) {
        int64_t i = act[(size_t)g * B + j];
        make_preview(tmpw, trace[i].prefill, trace[i].decode, d, k - x[i], H, sc->lookahead,
                     sc->noise_sigma, rng);
        for (int h = 0; h < H1; ++h) fut[(size_t)g * H1 + h] += tmpw[h];
      }
    }
    if (need_views) {
      pvbuf = (double*)realloc(pvbuf, sizeof(double) * (size_t)(nw > 0 ? nw : 1) * H1);
      pvs = (pv_ref_t*)realloc(pvs, sizeof(pv_ref_t) * (size_t)(nw > 0 ? nw : 1));
      for (int64_t j = 0; j < nw; ++j) {
        int64_t i = waiting[j];
        make_preview(pvbuf + (size_t)j * H1, trace[i].prefill, trace[i].decode, d, 0, H,
                     sc->lookahead, sc->noise_sigma, rng);
        pvs[j].w = pvbuf + (size_t)j * H1;
      }
    }
    /* assign, policies.hpp:372-382 */
    int64_t np = 0;
    if (sc->policy == BFSIM_POLICY_FCFS)
      np = assign_fcfs((int)nw, G, caps, pairs);
    else if (sc->policy == BFSIM_POLICY_JSQ)
      np = assign_jsq((int)nw, G, caps, cnts, pairs);
    else
      np = assign_greedy((int)nw, pvs, G, caps, fut, H, pairs);
    /* apply, engine.hpp:233-253 */
    taken = (char*)realloc(taken, (size_t)(nw > 0 ? nw : 1));
    memset(taken, 0, (size_t)(nw > 0 ? nw : 1));
    for (int64_t p = 0; p < np; ++p) {
      int wi = pairs[2 * p], g = pairs[2 * p + 1];
      if (wi < 0 || wi >= nw || g < 0 || g >= G || nact[g] >= B || taken[wi]) {
        status = BFSIM_ELOGIC;
        goto out;
      }
      int64_t i = waiting[wi];
      taken[wi] = 1;
      wk[i] = g;
      x[i] = k;
      admit[i] = clock;
      act[(size_t)g * B + nact[g]++] = i;
      res->admitted += 1;
    }
    {
      int64_t w2 = 0;
      for (int64_t j = 0; j < nw; ++j)
        if (!taken[j]) waiting[w2++] = waiting[j];
      nw = w2;
    }
    /* loads, max, dt, clock: engine.hpp:136-146 */
    int64_t ac = 0, mx = 0;
    for (int g = 0; g < G; ++g) {
      L[g] = 0;
      for (int j = 0; j < nact[g]; ++j) {
        int64_t i = act[(size_t)g * B + j];
        L[g] += trace[i].prefill + d * (k - x[i]);
      }
      ac += nact[g];
      if (L[g] > mx) mx = L[g];
    }
    double dtk = sc->overhead + sc->per_token * (double)mx;
    double cs = clock;
    clock += dtk;
    if (k < step_cap) {
      if (o_clock_start) o_clock_start[k] = cs;
      if (o_dt) o_dt[k] = dtk;
      if (o_max_load) o_max_load[k] = (double)mx;
      if (o_active_count) o_active_count[k] = ac;
      if (o_loads)
        for (int g = 0; g < G; ++g) o_loads[(size_t)k * G + g] = (double)L[g];
    } else {
      res->flags |= BFSIM_FLAG_STEP_OVERFLOW;
    }
    acct_step(&acct, L, G, mx, ac, dtk, sc);
    /* progress + completion, engine.hpp:149-157; erase at next step start :118-120 */
    for (int g = 0; g < G; ++g) {
      int keep = 0;
      for (int j = 0; j < nact[g]; ++j) {
        int64_t i = act[(size_t)g * B + j];
        if (k - x[i] + 1 >= trace[i].decode) {
          finish[i] = clock;
          done[i] = 1;
          ++n_done;
        } else {
          act[(size_t)g * B + keep++] = i;
        }
      }
      nact[g] = keep;
    }
    ++k;
  }
out:
  res->steps_run = k;
  res->clock = clock;
  res->completed = n_done;
  {
    /* tpot over requests in id order, metrics.hpp:43-53 */
    double acc = 0.0;
    int64_t cnt = 0;
    for (int64_t i = 0; i < n; ++i) {
      if (!done[i]) continue;
      acc += (finish[i] - admit[i]) / (double)trace[i].decode;
      ++cnt;
    }
    acct_finish(&acct, acc, cnt, res);
  }
  for (int64_t i = 0; i < n; ++i) {
    if (o_arrival_step) o_arrival_step[i] = arr_step[i];
    if (o_start_step) o_start_step[i] = (int32_t)x[i];
    if (o_worker) o_worker[i] = wk[i];
    if (o_admit_clock) o_admit_clock[i] = admit[i];
    if (o_finish_clock) o_finish_clock[i] = finish[i];
  }
  res->status = status;
  free(rng);
  free(tmpw);
  free(taken);
  free(pairs);
  free(pvs);
  free(pvbuf);
  free(fut);
  free(cnts);
  free(caps);
  free(L);
  free(waiting);
  free(nact);
  free(act);
  free(done);
  free(arr_step);
  free(finish);
  free(admit);
  free(wk);
  free(x);
  return status;
}

/* ---------------- run_overloaded (oracle.hpp:138-244) ---------------- */

int oracle_run_overloaded(const bfsim_scenario_t* sc, const bfsim_sample_t* stream,
                          int64_t stream_len, int32_t s_max, int64_t step_cap,
                          double* o_clock_start, double* o_dt, double* o_max_load,
                          int64_t* o_active_count, double* o_loads, int32_t* o_start_step,
                          int32_t* o_worker, int64_t timing_cap, int32_t* t_id, double* t_admit,
                          double* t_finish, int64_t* t_decode, int64_t* n_timings,
                          bfsim_result_t* res) {
  memset(res, 0, sizeof(*res));
  *n_timings = 0;
  const int G = sc->workers, B = sc->batch, H = sc->horizon, H1 = sc->horizon + 1;
  if (G < 1 || B < 1 || H < 0 || s_max < 1 || !drift_ok(sc->drift) || !power_ok(sc) ||
      sc->policy == BFSIM_POLICY_BFIO_EXACT || sc->policy < 0 || sc->policy > 3 || sc->steps < 0 ||
      sc->warmup < 0) {
    res->status = BFSIM_EINVAL;
    return BFSIM_EINVAL;
  }
  const int64_t d = (int64_t)sc->drift;
  const int64_t total = sc->warmup + sc->steps;
  /* min_pool, oracle.hpp:169-170 */
  const int64_t min_pool = (int64_t)(sc->backlog * (double)G * (double)B);

  int64_t* pool = (int64_t*)malloc(sizeof(int64_t) * (size_t)(stream_len > 0 ? stream_len : 1));
  int64_t np_ = 0, next_sample = 0;
  int64_t* cls = (int64_t*)calloc((size_t)s_max + 1, sizeof(int64_t));
  typedef struct {
    int64_t si, age, id;
    double admit;
  } act_t;
  act_t* act = (act_t*)malloc(sizeof(act_t) * (size_t)G * B);
  int32_t* nact = (int32_t*)calloc((size_t)G, sizeof(int32_t));
  int64_t* L = (int64_t*)malloc(sizeof(int64_t) * (size_t)G);
  int32_t* caps = (int32_t*)malloc(sizeof(int32_t) * (size_t)G);
  int32_t* cnts = (int32_t*)malloc(sizeof(int32_t) * (size_t)G);
  double* fut = (double*)malloc(sizeof(double) * (size_t)G * H1);
  double* tmpw = (double*)malloc(sizeof(double) * (size_t)H1);
  int32_t* pairs = (int32_t*)malloc(sizeof(int32_t) * 2 * (size_t)G * B);
  double* pvbuf = NULL;
  pv_ref_t* pvs = NULL;
  char* taken = NULL;
  if (o_start_step)
    for (int64_t i = 0; i < stream_len; ++i) o_start_step[i] = -1;
  if (o_worker)
    for (int64_t i = 0; i < stream_len; ++i) o_worker[i] = -1;

  acct_t acct;
  memset(&acct, 0, sizeof(acct));
  double clock = 0.0, tpot_acc = 0.0;
  int64_t tpot_n = 0, next_id = 0, k = 0;
  int status = BFSIM_OK;
  for (k = 0; k < total; ++k) {
    long free_slots = 0;
    for (int g = 0; g < G; ++g) free_slots += B - nact[g];
    /* top-up until Def. 1 holds and the backlog is met, oracle.hpp:167-183;
     * is_overloaded_at, workload.hpp:325-335 */
    for (;;) {
      int64_t largest = 0;
      for (int c = 1; c <= s_max; ++c)
        if (cls[c] > largest) largest = cls[c];
      if (np_ >= min_pool && np_ - largest >= free_slots) break;
      if (next_sample >= stream_len) {
        status = BFSIM_ESTREAM;
        goto out;
      }
      int s = stream[next_sample].prefill;
      if (s >= 1 && s <= s_max) cls[s] += 1;
      pool[np_++] = next_sample++;
    }
    /* views, oracle.hpp:185-199 (perfect previews) */
    for (int g = 0; g < G; ++g) {
      caps[g] = B - nact[g];
      cnts[g] = nact[g];
      for (int h = 0; h < H1; ++h) fut[(size_t)g * H1 + h] = 0.0;
      if (sc->policy != BFSIM_POLICY_BFIO_GREEDY) continue;
      for (int j = 0; j < nact[g]; ++j) {
        const act_t* a = &act[(size_t)g * B + j];
        make_preview(tmpw, stream[a->si].prefill, stream[a->si].decode, d, a->age, H,
                     BFSIM_LOOKAHEAD_PERFECT, 0.0, NULL);
        for (int h = 0; h < H1; ++h) fut[(size_t)g * H1 + h] += tmpw[h];
      }
    }
    int64_t npairs = 0;
    if (sc->policy == BFSIM_POLICY_FCFS) {
      npairs = assign_fcfs((int)np_, G, caps, pairs);
    } else if (sc->policy == BFSIM_POLICY_JSQ) {
      npairs = assign_jsq((int)np_, G, caps, cnts, pairs);
    } else {
      pvbuf = (double*)realloc(pvbuf, sizeof(double) * (size_t)(np_ > 0 ? np_ : 1) * H1);
      pvs = (pv_ref_t*)realloc(pvs, sizeof(pv_ref_t) * (size_t)(np_ > 0 ? np_ : 1));
      for (int64_t j = 0; j < np_; ++j) {
        int64_t si = pool[j];
        make_preview(pvbuf + (size_t)j * H1, stream[si].prefill, stream[si].decode, d, 0, H,
                     BFSIM_LOOKAHEAD_PERFECT, 0.0, NULL);
        pvs[j].w = pvbuf + (size_t)j * H1;
      }
      npairs = assign_greedy((int)np_, pvs, G, caps, fut, H, pairs);
    }
    /* admit, oracle.hpp:203-210 */
    taken = (char*)realloc(taken, (size_t)(np_ > 0 ? np_ : 1));
    memset(taken, 0, (size_t)(np_ > 0 ? np_ : 1));
    for (int64_t p = 0; p < npairs; ++p) {
      int wi = pairs[2 * p], g = pairs[2 * p + 1];
      int64_t si = pool[wi];
      act_t* a = &act[(size_t)g * B + nact[g]++];
      a->si = si;
      a->age = 0;
      a->admit = clock;
      a->id = next_id++;
      taken[wi] = 1;
      if (o_start_step) o_start_step[si] = (int32_t)k;
      if (o_worker) o_worker[si] = g;
      int s = stream[si].prefill;
      if (s >= 1 && s <= s_max) cls[s] -= 1;
      res->admitted += 1;
    }
    {
      int64_t w2 = 0;
      for (int64_t j = 0; j < np_; ++j)
        if (!taken[j]) pool[w2++] = pool[j];
      np_ = w2;
    }
    /* record, oracle.hpp:212-223 */
    int64_t ac = 0, mx = 0;
    for (int g = 0; g < G; ++g) {
      L[g] = 0;
      for (int j = 0; j < nact[g]; ++j) {
        const act_t* a = &act[(size_t)g * B + j];
        L[g] += stream[a->si].prefill + d * a->age;
      }
      ac += nact[g];
      if (L[g] > mx) mx = L[g];
    }
    double dtk = sc->overhead + sc->per_token * (double)mx;
    double cs = clock;
    clock += dtk;
    if (k < step_cap) {
      if (o_clock_start) o_clock_start[k] = cs;
      if (o_dt) o_dt[k] = dtk;
      if (o_max_load) o_max_load[k] = (double)mx;
      if (o_active_count) o_active_count[k] = ac;
      if (o_loads)
        for (int g = 0; g < G; ++g) o_loads[(size_t)k * G + g] = (double)L[g];
    } else {
      res->flags |= BFSIM_FLAG_STEP_OVERFLOW;
    }
    if (k >= sc->warmup) acct_step(&acct, L, G, mx, ac, dtk, sc);
    /* age + erase_if done -> timings, oracle.hpp:225-240 */
    for (int g = 0; g < G; ++g) {
      int keep = 0;
      for (int j = 0; j < nact[g]; ++j) {
        act_t a = act[(size_t)g * B + j];
        a.age += 1;
        int64_t o = stream[a.si].decode;
        if (a.age >= o) {
          if (*n_timings < timing_cap) {
            if (t_id) t_id[*n_timings] = (int32_t)a.id;
            if (t_admit) t_admit[*n_timings] = a.admit;
            if (t_finish) t_finish[*n_timings] = clock;
            if (t_decode) t_decode[*n_timings] = o;
          }
          *n_timings += 1;
          tpot_acc += (clock - a.admit) / (double)o;
          ++tpot_n;
        } else {
          act[(size_t)g * B + keep++] = a;
        }
      }
      nact[g] = keep;
    }
  }
out:
  res->steps_run = k;
  res->clock = clock;
  res->completed = tpot_n;
  res->consumed = next_sample;
  acct_finish(&acct, tpot_acc, tpot_n, res);
  res->status = status;
  free(taken);
  free(pvs);
  free(pvbuf);
  free(pairs);
  free(tmpw);
  free(fut);
  free(cnts);
  free(caps);
  free(L);
  free(nact);
  free(act);
  free(cls);
  free(pool);
  return status;
}
