/* Experiment (round 1): Alg. 1 evaluation counts under three pruning regimes.
 * Build: gcc -O2 -ffp-contract=off -o /tmp/ideal tools/experiments/prune_bound.c -lm -lpthread
 * Input: binary [16][m] fp64 workload table + [m] int32 name ranks (V100, r_unit 0.025). */
#include "../../oracle/igniter_oracle.c"
#include <stdio.h>
typedef struct { long long evals, cands, started; } cnt_t;
/* Alg. 2 with early exit on overflow / key > bound; returns 1 if pruned/overflow, else 0 (feasible) */
static int alloc_pruned(const entry_t *const *es, int *units, int n, const double *hw, int cap,
                        int occ, unsigned long long bound, int j, long long *evals, alloc_ws_t *ws) {
  int flag = 1, total = 0;
  for (int i = 0; i < n; ++i) total += units[i];
  while (total <= cap && flag) {
    flag = 0;
    int have = 0;
    for (int i = 0; i < n; ++i) {
      if (!have) {
        for (int k = 0; k < n; ++k) ws->rs[k] = (double)units[k] * hw[H_RUNIT];
        igo_err e;
        eval_entries(es, ws->rs, n, hw, NULL, ws->tinf, ws->scratch, &e);
        *evals += 1;
        have = 1;
      }
      if (ws->tinf[i] > es[i]->t_half) {
        units[i] += 1; flag = 1; have = 0; total += 1;
        if (total > cap) return 1;
        unsigned long long key = ((unsigned long long)(total - occ) << 32) | (unsigned)j;
        if (key > bound) return 1;
      }
    }
  }
  return total > cap;
}
int main(int argc, char **argv) {
  int m = atoi(argv[1]);
  FILE *f = fopen(argv[2], "rb");
  double *wl = malloc(sizeof(double) * 16 * m);
  fread(wl, 8, 16 * m, f);
  int32_t *rank = malloc(4 * m);
  fread(rank, 4, m, f);
  fclose(f);
  double hw[11] = {300.0, 1530.0, 53.5, 10.0, -1.025, 0.00475, -0.00902, 0.025, 1.0, 3.06, 0.3};
  int cap = igo_max_units(hw), b_max = 32;
  int32_t *batch = malloc(4 * m), *lb = malloc(4 * m), *code = malloc(4 * m);
  igo_prologue(wl, m, m, hw, b_max, batch, lb, code);
  int *order = malloc(sizeof(int) * m);
  for (int i = 0; i < m; ++i) order[i] = i;
  sort_ctx_t sc = {rank, lb};
  t_sort_ctx = &sc;
  qsort(order, m, sizeof(int), cmp_order);
  entry_t *ents = malloc(sizeof(entry_t) * m);
  for (int i = 0; i < m; ++i) make_entry(&ents[i], wl, m, i, batch[i], hw);
  int stride = cap + 1;
  int *g_res = malloc(sizeof(int) * m * stride), *g_units = malloc(sizeof(int) * m * stride);
  int *g_n = calloc(m, sizeof(int)), *g_occ = calloc(m, sizeof(int));
  const entry_t **eps = malloc(sizeof(void *) * (stride + 1));
  int *cand = malloc(sizeof(int) * (stride + 1)), *best = malloc(sizeof(int) * (stride + 1));
  double *buf = malloc(sizeof(double) * 5 * (stride + 1));
  alloc_ws_t ws = {buf, buf + (stride + 1), buf + 2 * (stride + 1)};
  long long ref_evals = 0, ref_cands = 0, ideal_evals = 0, ideal_started = 0, seq_evals = 0, seq_started = 0;
  long long zero_bump_steps = 0;
  int G = 0;
  for (int step = 0; step < m; ++step) {
    int w = order[step], need = lb[w];
    int best_j = -1, best_inter = cap, best_n = 0;
    /* reference: full Alg. 2 on every candidate */
    for (int j = 0; j < G; ++j) {
      if (g_occ[j] + need > cap) continue;
      ref_cands++;
      int n = g_n[j] + 1;
      for (int k = 0; k < n - 1; ++k) { eps[k] = &ents[g_res[j * stride + k]]; cand[k] = g_units[j * stride + k]; }
      eps[n - 1] = &ents[w]; cand[n - 1] = need;
      int64_t ev = 0;
      igo_err e;
      alloc_units(eps, cand, n, hw, cap, &ev, &ws, &e);
      ref_evals += ev / n;
      int total = 0;
      for (int k = 0; k < n; ++k) total += cand[k];
      if (total <= cap && total - g_occ[j] < best_inter) { best_j = j; best_inter = total - g_occ[j]; best_n = n; memcpy(best, cand, sizeof(int) * n); }
    }
    if (best_j >= 0 && best_inter == need) zero_bump_steps++;
    unsigned long long B = best_j < 0 ? ~0ull : (((unsigned long long)best_inter << 32) | (unsigned)best_j);
    unsigned long long run = ~0ull;
    for (int j = 0; j < G; ++j) {
      if (g_occ[j] + need > cap) continue;
      unsigned long long k0 = ((unsigned long long)need << 32) | (unsigned)j;
      int n = g_n[j] + 1;
      /* ideal: bound known */
      if (k0 <= B) {
        ideal_started++;
        for (int k = 0; k < n - 1; ++k) { eps[k] = &ents[g_res[j * stride + k]]; cand[k] = g_units[j * stride + k]; }
        eps[n - 1] = &ents[w]; cand[n - 1] = need;
        alloc_pruned(eps, cand, n, hw, cap, g_occ[j], B, j, &ideal_evals, &ws);
      }
      /* sequential with running best */
      if (k0 <= run) {
        seq_started++;
        for (int k = 0; k < n - 1; ++k) { eps[k] = &ents[g_res[j * stride + k]]; cand[k] = g_units[j * stride + k]; }
        eps[n - 1] = &ents[w]; cand[n - 1] = need;
        int pr = alloc_pruned(eps, cand, n, hw, cap, g_occ[j], run, j, &seq_evals, &ws);
        if (!pr) {
          int total = 0;
          for (int k = 0; k < n; ++k) total += cand[k];
          unsigned long long key = ((unsigned long long)(total - g_occ[j]) << 32) | (unsigned)j;
          if (key < run) run = key;
        }
      }
    }
    if (best_j < 0) { g_res[G * stride] = w; g_units[G * stride] = need; g_n[G] = 1; g_occ[G] = need; G++; }
    else { int occ = 0; g_res[best_j * stride + best_n - 1] = w; for (int k = 0; k < best_n; ++k) { g_units[best_j * stride + k] = best[k]; occ += best[k]; } g_n[best_j] = best_n; g_occ[best_j] = occ; }
  }
  printf("m=%d G=%d ref_cands=%lld ref_evals=%lld | ideal: started=%lld evals=%lld | sequential: started=%lld evals=%lld | zero-bump steps=%lld\n",
         m, G, ref_cands, ref_evals, ideal_started, ideal_evals, seq_started, seq_evals, zero_bump_steps);
  return 0;
}
