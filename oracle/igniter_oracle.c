/*
 * igniter_oracle.c -- CPU restatement of the iGniter provisioning hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA
 * library in paper_2211_01713_b200/csrc; it is never linked into the product.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference leg may load it.
 *
 * It restates, operation by operation, the reference package gpuplanner
 * (/root/reference/pkg/src/gpuplanner, CPython 3.12):
 *   appropriate_batch      planner.py:76-92
 *   _lower_bound_units     planner.py:95-120
 *   _Entry                 model.py:239-270
 *   _eval_entries          model.py:273-317
 *   _alloc_units (Alg. 2)  planner.py:133-162
 *   plan (Alg. 1)          planner.py:258-325 (+ _build_plan planner.py:218-246,
 *                          predict_gpu model.py:320-343)
 *   builtin sum of floats  CPython 3.12 Python/bltinmodule.c builtin_sum_impl
 *                          (Neumaier-compensated; SURVEY.md finding 1)
 *
 * Every fp64 operation is rounded separately in the reference's left-to-right
 * association; build with -ffp-contract=off (no FMA contraction) and without
 * -ffast-math.  Pinned against fixtures produced by the real reference:
 * tests/golden/make_golden.py -> tests/test_oracle_golden.py.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "igniter_oracle.h"

/* workload SoA field indices (paper_2211_01713_b200/layout.py WL_FIELDS) */
enum { F_SLO, F_RATE, F_DLOAD, F_DFB, F_NK, F_KSCH, F_K1, F_K2, F_K3, F_K4, F_K5,
       F_AP, F_BP, F_AC, F_BC, F_ACACHE, F_NF };
/* hardware fields (layout.py HW_FIELDS) */
enum { H_PMAX, H_FMAX, H_PIDLE, H_BW, H_AF, H_ASCH, H_BSCH, H_RUNIT, H_RMAX,
       H_PRICE, H_FMINFRAC };

#define WLF(wl, ld, f, i) ((wl)[(int64_t)(f) * (ld) + (i)])

/* Python max(a, b): b only if b > a.  min(a, b): b only if b < a. */
static inline double py_max(double a, double b) { return (b > a) ? b : a; }
static inline double py_min(double a, double b) { return (b < a) ? b : a; }

/* CPython 3.12 sum(list_of_floats) with start=0 (int). */
static double py_sum(const double *x, int n) {
  if (n <= 0) return 0.0;
  double s = 0.0 + x[0];
  double c = 0.0;
  for (int k = 1; k < n; ++k) {
    double v = x[k];
    double t = s + v;
    if (fabs(s) >= fabs(v)) c += (s - t) + v;
    else c += (v - t) + s;
    s = t;
  }
  if (c != 0.0 && isfinite(c)) s += c;
  return s;
}

/* ---- entry constants: model.py:253-270 -------------------------------- */
typedef struct {
  int w;            /* workload index (input order) */
  double batch;     /* int in the reference; exact as double */
  double gamma, k4, k5, k_sch, nk, acache, ap, bp, ac, bc;
  double t_load, t_fb, t_half;
} entry_t;

static void make_entry(entry_t *e, const double *wl, int64_t ld, int i, int b,
                       const double *hw) {
  double bd = (double)b;
  e->w = i;
  e->batch = bd;
  e->gamma = ((WLF(wl, ld, F_K1, i) * bd) * bd + WLF(wl, ld, F_K2, i) * bd) + WLF(wl, ld, F_K3, i);
  e->k4 = WLF(wl, ld, F_K4, i);
  e->k5 = WLF(wl, ld, F_K5, i);
  e->k_sch = WLF(wl, ld, F_KSCH, i);
  e->nk = WLF(wl, ld, F_NK, i);
  e->acache = WLF(wl, ld, F_ACACHE, i);
  e->ap = WLF(wl, ld, F_AP, i);
  e->bp = WLF(wl, ld, F_BP, i);
  e->ac = WLF(wl, ld, F_AC, i);
  e->bc = WLF(wl, ld, F_BC, i);
  e->t_load = (WLF(wl, ld, F_DLOAD, i) * bd) / hw[H_BW];
  e->t_fb = (WLF(wl, ld, F_DFB, i) * bd) / hw[H_BW];
  e->t_half = WLF(wl, ld, F_SLO, i) / 2.0;
}

static void set_err(igo_err *err, int code, int w, double a, double b, double c) {
  if (!err) return;
  err->code = code;
  err->workload = w;
  err->a = a;
  err->b = b;
  err->c = c;
}

/* model.py:273-317.  rows may be NULL (decision-only callers still need
 * t_inf, which is written to tinf).  Returns 0 or an error code. */
static int eval_entries(const entry_t *const *es, const double *rs, int n,
                        const double *hw, double *rows /* n x 10 or NULL */,
                        double *tinf /* n or NULL */, double *scratch /* 3n */,
                        igo_err *err) {
  double delta = (n <= 1) ? 0.0 : py_max(0.0, hw[H_ASCH] * (double)n + hw[H_BSCH]);
  double *k_acts = scratch, *powers = scratch + n, *caches = scratch + 2 * n;
  for (int i = 0; i < n; ++i) {
    const entry_t *e = es[i];
    double r = rs[i];
    double denom = r + e->k4;
    if (denom <= 0) {
      set_err(err, IGO_E_DENOM, e->w, denom, r, e->k4);
      return IGO_E_DENOM;
    }
    double k_act = e->gamma / denom + e->k5;
    if (k_act <= 0) {
      set_err(err, IGO_E_ACTIVE_TIME, e->w, k_act, e->batch, r);
      return IGO_E_ACTIVE_TIME;
    }
    double ability = e->batch / k_act;
    double c = e->ac * ability + e->bc;
    k_acts[i] = k_act;
    powers[i] = e->ap * ability + e->bp;
    caches[i] = py_min(1.0, py_max(0.0, c));
  }
  double p_dem = hw[H_PIDLE] + py_sum(powers, n);
  double f;
  if (p_dem <= hw[H_PMAX]) f = hw[H_FMAX];
  else f = py_max(hw[H_FMINFRAC] * hw[H_FMAX], hw[H_FMAX] + hw[H_AF] * (p_dem - hw[H_PMAX]));
  double cache_total = py_sum(caches, n);
  double scale = f / hw[H_FMAX];
  for (int i = 0; i < n; ++i) {
    const entry_t *e = es[i];
    double t_sch = (e->k_sch + delta) * e->nk;
    double co_cache = cache_total - caches[i];
    double t_act = k_acts[i] * (1.0 + e->acache * co_cache);
    double t_gpu = (t_sch + t_act) / scale;
    double t_inf = (e->t_load + t_gpu) + e->t_fb;
    if (tinf) tinf[i] = t_inf;
    if (rows) {
      double *row = rows + 10 * i;
      row[0] = e->t_load;
      row[1] = t_sch;
      row[2] = t_act;
      row[3] = f;
      row[4] = t_gpu;
      row[5] = e->t_fb;
      row[6] = t_inf;
      row[7] = (e->batch / (t_gpu + e->t_fb)) * 1000.0;
      row[8] = powers[i];
      row[9] = caches[i];
    }
  }
  return 0;
}

/* ---- prologue: planner.py:76-120 -------------------------------------- */
static int prologue_one(const double *wl, int64_t ld, int i, const double *hw,
                        int b_max, int cap, int *b_out, int *lb_out, igo_err *err) {
  double slo = WLF(wl, ld, F_SLO, i), rate_rps = WLF(wl, ld, F_RATE, i);
  double dl = WLF(wl, ld, F_DLOAD, i), dfb = WLF(wl, ld, F_DFB, i);
  double bw = hw[H_BW];
  double rate = rate_rps / 1000.0;
  double bx = ceil(((slo * rate) * bw) / (2.0 * (bw + rate * dl)));
  if (!(bx > 1.0)) bx = 1.0;
  if (bx > (double)b_max) {
    set_err(err, IGO_E_BATCH_CAP, i, bx, (double)b_max, 0.0);
    return IGO_E_BATCH_CAP;
  }
  int b = (int)bx;
  double bd = (double)b;
  double delta = ((slo / 2.0 - ((dl + dfb) * bd) / bw) - WLF(wl, ld, F_K5, i)) -
                 WLF(wl, ld, F_KSCH, i) * WLF(wl, ld, F_NK, i);
  if (delta <= 0) {
    set_err(err, IGO_E_INFEASIBLE_SLO, i, delta, 0.0, 0.0);
    *b_out = b;
    return IGO_E_INFEASIBLE_SLO;
  }
  double gamma = ((WLF(wl, ld, F_K1, i) * bd) * bd + WLF(wl, ld, F_K2, i) * bd) + WLF(wl, ld, F_K3, i);
  double ux = ceil(gamma / (delta * hw[H_RUNIT]) - WLF(wl, ld, F_K4, i) / hw[H_RUNIT]);
  if (!(ux > 1.0)) ux = 1.0;
  if (ux > (double)cap) {
    set_err(err, IGO_E_INFEASIBLE_RES, i, ux, 0.0, 0.0);
    *b_out = b;
    return IGO_E_INFEASIBLE_RES;
  }
  *b_out = b;
  *lb_out = (int)ux;
  return 0;
}

int igo_max_units(const double *hw) {
  /* int(round(r_max / r_unit)): Python round() is round-half-even */
  return (int)nearbyint(hw[H_RMAX] / hw[H_RUNIT]);
}

int igo_prologue(const double *wl, int64_t ld, int m, const double *hw, int b_max,
                 int32_t *batch, int32_t *lb, int32_t *code) {
  int cap = igo_max_units(hw);
  int first = 0;
  for (int i = 0; i < m; ++i) {
    int b = -1, u = -1;
    igo_err e;
    int rc = prologue_one(wl, ld, i, hw, b_max, cap, &b, &u, &e);
    batch[i] = (rc == IGO_E_BATCH_CAP) ? -1 : b;
    lb[i] = rc ? -1 : u;
    code[i] = rc;
    if (rc && !first) first = rc;
  }
  return first;
}

int igo_eval_states(const double *wl, int64_t ld, const int32_t *batch, const double *r,
                    const int64_t *ptr, int n_states, const double *hw, double *rows,
                    igo_err *err) {
  int nmax = 0;
  for (int s = 0; s < n_states; ++s)
    if (ptr[s + 1] - ptr[s] > nmax) nmax = (int)(ptr[s + 1] - ptr[s]);
  entry_t *ents = malloc(sizeof(entry_t) * (nmax + 1));
  const entry_t **eps = malloc(sizeof(entry_t *) * (nmax + 1));
  double *scratch = malloc(sizeof(double) * 3 * (nmax + 1));
  int rc = 0;
  for (int s = 0; s < n_states && !rc; ++s) {
    int n = (int)(ptr[s + 1] - ptr[s]);
    for (int k = 0; k < n; ++k) {
      int64_t gi = ptr[s] + k;
      make_entry(&ents[k], wl, ld, (int)gi, batch[gi], hw);
      eps[k] = &ents[k];
    }
    rc = eval_entries(eps, r + ptr[s], n, hw, rows + 10 * ptr[s], NULL, scratch, err);
  }
  free(ents);
  free(eps);
  free(scratch);
  return rc;
}

/* ---- Alg. 2: planner.py:133-162 --------------------------------------- */
typedef struct {
  double *rs, *tinf, *scratch;
} alloc_ws_t;

static int alloc_units(const entry_t *const *es, int *units, int n, const double *hw,
                       int cap, int64_t *model_evals, alloc_ws_t *ws, igo_err *err) {
  int flag = 1;
  for (;;) {
    int total = 0;
    for (int i = 0; i < n; ++i) total += units[i];
    if (!(total <= cap && flag)) break;
    flag = 0;
    int have_rows = 0;
    for (int i = 0; i < n; ++i) {
      if (!have_rows) {
        for (int k = 0; k < n; ++k) ws->rs[k] = (double)units[k] * hw[H_RUNIT];
        int rc = eval_entries(es, ws->rs, n, hw, NULL, ws->tinf, ws->scratch, err);
        if (rc) return rc;
        if (model_evals) *model_evals += n;
        have_rows = 1;
      }
      if (ws->tinf[i] > es[i]->t_half) {
        units[i] += 1;
        flag = 1;
        have_rows = 0;
      }
    }
  }
  return 0;
}

int igo_alloc_units(const double *wl, int64_t ld, const int32_t *batch, const double *r,
                    const int64_t *ptr, int n_states, const double *hw, int32_t *units_out,
                    igo_err *err) {
  int cap = igo_max_units(hw);
  int nmax = 0;
  for (int s = 0; s < n_states; ++s)
    if (ptr[s + 1] - ptr[s] > nmax) nmax = (int)(ptr[s + 1] - ptr[s]);
  entry_t *ents = malloc(sizeof(entry_t) * (nmax + 1));
  const entry_t **eps = malloc(sizeof(entry_t *) * (nmax + 1));
  double *buf = malloc(sizeof(double) * 5 * (nmax + 1));
  alloc_ws_t ws = {buf, buf + (nmax + 1), buf + 2 * (nmax + 1)};
  int rc = 0;
  for (int s = 0; s < n_states && !rc; ++s) {
    int n = (int)(ptr[s + 1] - ptr[s]);
    for (int k = 0; k < n; ++k) {
      int64_t gi = ptr[s] + k;
      make_entry(&ents[k], wl, ld, (int)gi, batch[gi], hw);
      eps[k] = &ents[k];
      units_out[gi] = (int32_t)nearbyint(r[gi] / hw[H_RUNIT]); /* planner.py:184-185 */
    }
    rc = alloc_units(eps, units_out + ptr[s], n, hw, cap, NULL, &ws, err);
  }
  free(ents);
  free(eps);
  free(buf);
  return rc;
}

/* ---- Alg. 1: planner.py:258-325 --------------------------------------- */
typedef struct {
  const int32_t *rank;
  const int32_t *lb;
} sort_ctx_t;

static __thread const sort_ctx_t *t_sort_ctx; /* qsort has no context argument */

static int cmp_order(const void *a, const void *b) {
  int i = *(const int *)a, j = *(const int *)b;
  const sort_ctx_t *c = t_sort_ctx;
  /* sorted(key=(-lb, name)) planner.py:284: larger lb first, then name */
  if (c->lb[i] != c->lb[j]) return (c->lb[i] > c->lb[j]) ? -1 : 1;
  return (c->rank[i] < c->rank[j]) ? -1 : (c->rank[i] > c->rank[j]);
}

int igo_plan(const double *wl, int64_t ld, int m, const double *hw, int b_max,
             const int32_t *name_rank, int32_t *gpu_of, int32_t *pos, int32_t *units_out,
             int32_t *batch_out, int32_t *lb_out, double *pred, int32_t *gpu_count,
             int64_t *stats /* [model_evals, candidate_gpus, resident_reads] */, igo_err *err) {
  int cap = igo_max_units(hw);
  if (err) memset(err, 0, sizeof(*err));
  if (stats) stats[0] = stats[1] = stats[2] = 0;
  /* prologue in input order: planner.py:280-282 (batch before lb per workload) */
  for (int i = 0; i < m; ++i) {
    int b = 0, u = 0;
    int rc = prologue_one(wl, ld, i, hw, b_max, cap, &b, &u, err);
    if (rc) return rc;
    batch_out[i] = b;
    lb_out[i] = u;
  }
  int *order = malloc(sizeof(int) * (m > 0 ? m : 1));
  for (int i = 0; i < m; ++i) order[i] = i;
  sort_ctx_t sc = {name_rank, lb_out};
  t_sort_ctx = &sc;
  qsort(order, m, sizeof(int), cmp_order);

  entry_t *ents = malloc(sizeof(entry_t) * (m > 0 ? m : 1));
  for (int i = 0; i < m; ++i) make_entry(&ents[i], wl, ld, i, batch_out[i], hw);
  /* per GPU: resident workload ids and units, at most cap residents (units >= 1) */
  int stride = cap + 1;
  int *g_res = malloc(sizeof(int) * (size_t)(m > 0 ? m : 1) * stride);
  int *g_units = malloc(sizeof(int) * (size_t)(m > 0 ? m : 1) * stride);
  int *g_n = calloc(m > 0 ? m : 1, sizeof(int));
  int *g_occ = calloc(m > 0 ? m : 1, sizeof(int));
  int G = 0;
  const entry_t **eps = malloc(sizeof(entry_t *) * (stride + 1));
  int *cand = malloc(sizeof(int) * (stride + 1));
  int *best = malloc(sizeof(int) * (stride + 1));
  double *buf = malloc(sizeof(double) * 5 * (stride + 1));
  alloc_ws_t ws = {buf, buf + (stride + 1), buf + 2 * (stride + 1)};
  int64_t *evals = stats ? &stats[0] : NULL;
  int rc = 0;

  for (int step = 0; step < m && !rc; ++step) {
    int w = order[step];
    int need = lb_out[w];
    int best_j = -1, best_inter = cap, best_n = 0;
    for (int j = 0; j < G; ++j) {
      int occupied = g_occ[j];
      if (occupied + need > cap) continue;
      if (stats) {
        stats[1] += 1;
        stats[2] += g_n[j];
      }
      int n = g_n[j] + 1;
      for (int k = 0; k < n - 1; ++k) {
        eps[k] = &ents[g_res[(size_t)j * stride + k]];
        cand[k] = g_units[(size_t)j * stride + k];
      }
      eps[n - 1] = &ents[w];
      cand[n - 1] = need;
      rc = alloc_units(eps, cand, n, hw, cap, evals, &ws, err);
      if (rc) break;
      int total = 0;
      for (int k = 0; k < n; ++k) total += cand[k];
      if (total <= cap) {
        int inter = total - occupied;
        if (inter < best_inter) {
          best_j = j;
          best_inter = inter;
          best_n = n;
          memcpy(best, cand, sizeof(int) * n);
        }
      }
    }
    if (rc) break;
    if (best_j < 0) {
      g_res[(size_t)G * stride] = w;
      g_units[(size_t)G * stride] = need;
      g_n[G] = 1;
      g_occ[G] = need;
      G++;
    } else {
      int *res = g_res + (size_t)best_j * stride;
      int *un = g_units + (size_t)best_j * stride;
      res[best_n - 1] = w;
      int occ = 0;
      for (int k = 0; k < best_n; ++k) {
        un[k] = best[k];
        occ += best[k];
      }
      g_n[best_j] = best_n;
      g_occ[best_j] = occ;
    }
  }

  /* _build_plan (planner.py:218-246) -> predict_gpu per GPU (model.py:320-343) */
  double *rs = malloc(sizeof(double) * (stride + 1));
  double *rowbuf = malloc(sizeof(double) * 10 * (stride + 1));
  for (int j = 0; j < G && !rc; ++j) {
    int n = g_n[j];
    for (int k = 0; k < n; ++k) {
      eps[k] = &ents[g_res[(size_t)j * stride + k]];
      rs[k] = (double)g_units[(size_t)j * stride + k] * hw[H_RUNIT];
    }
    double total_r = py_sum(rs, n);
    if (total_r > hw[H_RMAX] + 1e-9) {
      set_err(err, IGO_E_OVERALLOC, -1, total_r, hw[H_RMAX], 0.0);
      rc = IGO_E_OVERALLOC;
      break;
    }
    rc = eval_entries(eps, rs, n, hw, rowbuf, NULL, ws.scratch, err);
    if (rc) break;
    for (int k = 0; k < n; ++k) {
      int w = g_res[(size_t)j * stride + k];
      gpu_of[w] = j;
      pos[w] = k;
      units_out[w] = g_units[(size_t)j * stride + k];
      if (pred) memcpy(pred + 10 * (size_t)w, rowbuf + 10 * k, sizeof(double) * 10);
    }
  }
  if (gpu_count) *gpu_count = G;
  free(rs);
  free(rowbuf);
  free(order);
  free(ents);
  free(g_res);
  free(g_units);
  free(g_n);
  free(g_occ);
  free(eps);
  free(cand);
  free(best);
  free(buf);
  return rc;
}

/* ---- scenario batch on host threads (the CPU baseline arm) ------------ */
typedef struct {
  const double *wl;
  int64_t scen_stride;
  int m;
  const double *hw;
  int b_max;
  const int32_t *name_rank;
  int32_t *gpu_of, *pos, *units, *gpu_count;
  double *pred; /* nullable: the _build_plan rows (planner.py:218-246) */
  int64_t *stats;
  int s_begin, s_end, rc;
} batch_job_t;

static void *batch_worker(void *arg) {
  batch_job_t *j = (batch_job_t *)arg;
  int m = j->m;
  int32_t *pos = malloc(sizeof(int32_t) * m), *bt = malloc(sizeof(int32_t) * m);
  int32_t *lb = malloc(sizeof(int32_t) * m);
  for (int s = j->s_begin; s < j->s_end; ++s) {
    igo_err e;
    int rc = igo_plan(j->wl + (int64_t)s * j->scen_stride, m, m, j->hw, j->b_max,
                      j->name_rank, j->gpu_of + (int64_t)s * m,
                      j->pos ? j->pos + (int64_t)s * m : pos, j->units + (int64_t)s * m, bt, lb,
                      j->pred ? j->pred + (int64_t)s * m * 10 : NULL, j->gpu_count + s,
                      j->stats ? j->stats + 3 * s : NULL, &e);
    if (rc && !j->rc) j->rc = rc;
  }
  free(pos);
  free(bt);
  free(lb);
  return NULL;
}

int igo_plan_batch(const double *wl, int n_scen, int m, const double *hw, int b_max,
                   const int32_t *name_rank, int32_t *gpu_of, int32_t *pos, int32_t *units,
                   double *pred, int32_t *gpu_count, int64_t *stats, int n_threads) {
  if (n_threads < 1) n_threads = 1;
  if (n_threads > n_scen) n_threads = n_scen > 0 ? n_scen : 1;
  pthread_t *th = malloc(sizeof(pthread_t) * n_threads);
  batch_job_t *jobs = malloc(sizeof(batch_job_t) * n_threads);
  int per = n_scen / n_threads, extra = n_scen % n_threads, s0 = 0;
  for (int t = 0; t < n_threads; ++t) {
    int cnt = per + (t < extra);
    jobs[t] = (batch_job_t){wl, (int64_t)F_NF * m, m, hw, b_max, name_rank,
                            gpu_of, pos, units, gpu_count, pred, stats, s0, s0 + cnt, 0};
    s0 += cnt;
    pthread_create(&th[t], NULL, batch_worker, &jobs[t]);
  }
  int rc = 0;
  for (int t = 0; t < n_threads; ++t) {
    pthread_join(th[t], NULL);
    if (jobs[t].rc && !rc) rc = jobs[t].rc;
  }
  free(th);
  free(jobs);
  return rc;
}

/* ---- solo candidate grid: oracle.py:64-114 for one-workload groups ----
 * For every (w, b in 1..b_max): scan u = 1..cap like _Search.best_group_alloc
 * (oracle.py:77-114) and record the first u passing _Search._feasible
 * (oracle.py:64-75) on the single-entry state _eval_entries([_Entry(b)], [u*r_unit]);
 * 0 if none, -code if an evaluation raised first. */
int igo_solo_grid(const double *wl, int64_t ld, int m, const double *hw, int b_max,
                  int32_t *min_units, int64_t *n_evals) {
  int cap = igo_max_units(hw);
  int64_t ev = 0;
  for (int w = 0; w < m; ++w) {
    for (int b = 1; b <= b_max; ++b) {
      entry_t e;
      make_entry(&e, wl, ld, w, b, hw);
      const entry_t *ep = &e;
      double rate = WLF(wl, ld, F_RATE, w);
      int res = 0;
      for (int u = 1; u <= cap; ++u) {
        double r = (double)u * hw[H_RUNIT], row[10], scratch[3];
        igo_err err;
        ++ev;
        int rc = eval_entries(&ep, &r, 1, hw, row, NULL, scratch, &err);
        if (rc) { res = -rc; break; }
        if (row[6] > e.t_half || row[7] < rate) continue;
        res = u;
        break;
      }
      min_units[(int64_t)w * b_max + (b - 1)] = res;
    }
  }
  if (n_evals) *n_evals = ev;
  return 0;
}

/* ---- online stream: planner.py:290-319 in arrival order --------------
 * No reference API exists (plan() always sorts, planner.py:284); this is the
 * driver over the reference internals that tests/golden/make_golden.py
 * (stream_reference) runs: each arrival gets its batch and lower bound
 * (planner.py:280-282) and is placed by one Alg. 1 step against the
 * persistent state; an arrival whose prologue or candidate evaluation
 * raises is rejected (code = error) and leaves the state unchanged. */
int igo_stream(const double *wl, int64_t ld, int n, const double *hw, int b_max,
               int32_t *gpu_of, int32_t *pos, int32_t *code, int32_t *units_final,
               int32_t *gpu_count, int64_t *stats) {
  int cap = igo_max_units(hw);
  int stride = cap + 1;
  int nn = n > 0 ? n : 1;
  entry_t *ents = malloc(sizeof(entry_t) * nn);
  int *lbv = malloc(sizeof(int) * nn);
  int *g_res = malloc(sizeof(int) * (size_t)nn * stride);
  int *g_units = malloc(sizeof(int) * (size_t)nn * stride);
  int *g_n = calloc(nn, sizeof(int));
  int *g_occ = calloc(nn, sizeof(int));
  const entry_t **eps = malloc(sizeof(entry_t *) * (stride + 1));
  int *cand = malloc(sizeof(int) * (stride + 1));
  int *best = malloc(sizeof(int) * (stride + 1));
  double *buf = malloc(sizeof(double) * 5 * (stride + 1));
  alloc_ws_t ws = {buf, buf + (stride + 1), buf + 2 * (stride + 1)};
  int G = 0;
  if (stats) stats[0] = stats[1] = 0;
  for (int a = 0; a < n; ++a) {
    gpu_of[a] = -1;
    pos[a] = -1;
    code[a] = 0;
    int b = 0, need = 0;
    igo_err e;
    int rc = prologue_one(wl, ld, a, hw, b_max, cap, &b, &need, &e);
    if (rc) {
      code[a] = rc;
      continue;
    }
    lbv[a] = need;
    make_entry(&ents[a], wl, ld, a, b, hw);
    int best_j = -1, best_inter = cap, best_n = 0;
    for (int j = 0; j < G && !rc; ++j) {
      int occupied = g_occ[j];
      if (occupied + need > cap) continue;
      if (stats) stats[1] += 1;
      int nres = g_n[j] + 1;
      for (int k = 0; k < nres - 1; ++k) {
        eps[k] = &ents[g_res[(size_t)j * stride + k]];
        cand[k] = g_units[(size_t)j * stride + k];
      }
      eps[nres - 1] = &ents[a];
      cand[nres - 1] = need;
      rc = alloc_units(eps, cand, nres, hw, cap, stats ? &stats[0] : NULL, &ws, &e);
      if (rc) break;
      int total = 0;
      for (int k = 0; k < nres; ++k) total += cand[k];
      if (total <= cap && total - occupied < best_inter) {
        best_j = j;
        best_inter = total - occupied;
        best_n = nres;
        memcpy(best, cand, sizeof(int) * nres);
      }
    }
    if (rc) {
      code[a] = rc;
      continue;
    }
    if (best_j < 0) {
      g_res[(size_t)G * stride] = a;
      g_units[(size_t)G * stride] = need;
      g_n[G] = 1;
      g_occ[G] = need;
      best_j = G++;
    } else {
      int occ = 0;
      g_res[(size_t)best_j * stride + best_n - 1] = a;
      for (int k = 0; k < best_n; ++k) {
        g_units[(size_t)best_j * stride + k] = best[k];
        occ += best[k];
      }
      g_n[best_j] = best_n;
      g_occ[best_j] = occ;
    }
    gpu_of[a] = best_j;
    pos[a] = g_n[best_j] - 1;
  }
  for (int a = 0; a < n; ++a) units_final[a] = 0;
  for (int j = 0; j < G; ++j)
    for (int k = 0; k < g_n[j]; ++k)
      units_final[g_res[(size_t)j * stride + k]] = g_units[(size_t)j * stride + k];
  if (gpu_count) *gpu_count = G;
  free(ents); free(lbv); free(g_res); free(g_units); free(g_n); free(g_occ);
  free(eps); free(cand); free(best); free(buf);
  return 0;
}

/* ---- exhaustive oracle group search: oracle.py:64-114 -----------------
 * For every non-empty subset (members in the caller's order = name order,
 * oracle.py:86) the lexicographic minimum of (total, unit tuple) over the
 * feasible vectors on the grid with total <= max_units, packed like
 * igp_group_search_device; ~0 when none.  Returns the first evaluation error
 * code met (0 if none). */
int igo_group_search(const double *wl, int64_t ld, int n, const int32_t *batch, const double *hw,
                     const int32_t *grid, int n_grid, uint64_t *best) {
  int cap = igo_max_units(hw);
  int first_err = 0;
  entry_t ents[8];
  for (int w = 0; w < n; ++w) make_entry(&ents[w], wl, ld, w, batch[w], hw);
  for (int mask = 1; mask < (1 << n); ++mask) {
    int idx[8], k = 0;
    for (int w = 0; w < n; ++w)
      if ((mask >> w) & 1) idx[k++] = w;
    uint64_t b = ~(uint64_t)0;
    int digit[8] = {0};
    for (;;) {
      int sum = 0, units[8];
      for (int d = 0; d < k; ++d) {
        units[d] = grid[digit[d]];
        sum += units[d];
      }
      if (sum <= cap) {
        const entry_t *eps[8];
        double rs[8], rows[80], scratch[24];
        for (int d = 0; d < k; ++d) {
          eps[d] = &ents[idx[d]];
          rs[d] = (double)units[d] * hw[H_RUNIT];
        }
        igo_err e;
        int rc = eval_entries(eps, rs, k, hw, rows, NULL, scratch, &e);
        if (rc) {
          if (!first_err) first_err = rc;
        } else {
          int ok = 1;
          for (int d = 0; d < k && ok; ++d)
            if (rows[10 * d + 6] > eps[d]->t_half || rows[10 * d + 7] < WLF(wl, ld, F_RATE, idx[d]))
              ok = 0;
          if (ok) {
            uint64_t key = (uint64_t)sum;
            for (int d = 0; d < k; ++d) key = (key << 9) | (uint64_t)units[d];
            if (key < b) b = key;
          }
        }
      }
      int d = k - 1;
      while (d >= 0 && ++digit[d] == n_grid) digit[d--] = 0;
      if (d < 0) break;
    }
    best[mask] = b;
  }
  return first_err;
}
