/* Experiment: evaluations under a sequential running-best prune for different candidate orders. */
#include "../../oracle/igniter_oracle.c"
#include <stdio.h>
static int alloc_pruned(const entry_t *const *es, int *units, int n, const double *hw, int cap,
                        int occ, unsigned long long bound, int j, long long *evals, alloc_ws_t *ws) {
  int flag = 1, total = 0;
  for (int i = 0; i < n; ++i) total += units[i];
  while (total <= cap && flag) {
    flag = 0; int have = 0;
    for (int i = 0; i < n; ++i) {
      if (!have) { for (int k = 0; k < n; ++k) ws->rs[k] = (double)units[k] * hw[H_RUNIT]; igo_err e;
        eval_entries(es, ws->rs, n, hw, NULL, ws->tinf, ws->scratch, &e); *evals += 1; have = 1; }
      if (ws->tinf[i] > es[i]->t_half) { units[i] += 1; flag = 1; have = 0; total += 1;
        if (total > cap) return 1;
        unsigned long long key = ((unsigned long long)(total - occ) << 32) | (unsigned)j;
        if (key > bound) return 1; }
    }
  }
  return total > cap;
}
static double *g_key; static int cmpk(const void *a, const void *b) { double x = g_key[*(int*)a], y = g_key[*(int*)b]; return x < y ? -1 : x > y; }
int main(int argc, char **argv) {
  int m = atoi(argv[1]); FILE *f = fopen(argv[2], "rb");
  double *wl = malloc(sizeof(double) * 16 * m); if (fread(wl, 8, 16 * m, f)) {}
  int32_t *rank = malloc(4 * m); if (fread(rank, 4, m, f)) {} fclose(f);
  double hw[11] = {300.0, 1530.0, 53.5, 10.0, -1.025, 0.00475, -0.00902, 0.025, 1.0, 3.06, 0.3};
  int cap = igo_max_units(hw);
  int32_t *batch = malloc(4 * m), *lb = malloc(4 * m), *code = malloc(4 * m);
  igo_prologue(wl, m, m, hw, 32, batch, lb, code);
  int *order = malloc(sizeof(int) * m); for (int i = 0; i < m; ++i) order[i] = i;
  sort_ctx_t sc = {rank, lb}; t_sort_ctx = &sc; qsort(order, m, sizeof(int), cmp_order);
  entry_t *ents = malloc(sizeof(entry_t) * m); for (int i = 0; i < m; ++i) make_entry(&ents[i], wl, m, i, batch[i], hw);
  int stride = cap + 1;
  int *g_res = malloc(sizeof(int) * m * stride), *g_units = malloc(sizeof(int) * m * stride);
  int *g_n = calloc(m, sizeof(int)), *g_occ = calloc(m, sizeof(int));
  double *g_pw = calloc(m, sizeof(double)), *g_ca = calloc(m, sizeof(double));
  const entry_t **eps = malloc(sizeof(void *) * (stride + 1));
  int *cand = malloc(sizeof(int) * (stride + 1)), *best = malloc(sizeof(int) * (stride + 1));
  double *buf = malloc(sizeof(double) * 5 * (stride + 1)); alloc_ws_t ws = {buf, buf + (stride + 1), buf + 2 * (stride + 1)};
  long long ev[6] = {0}; int G = 0;
  int *cl = malloc(sizeof(int) * m); double *key = malloc(sizeof(double) * m); g_key = key;
  for (int step = 0; step < m; ++step) {
    int w = order[step], need = lb[w];
    int best_j = -1, best_inter = cap, best_n = 0;
    for (int j = 0; j < G; ++j) {
      if (g_occ[j] + need > cap) continue;
      int n = g_n[j] + 1;
      for (int k = 0; k < n - 1; ++k) { eps[k] = &ents[g_res[j * stride + k]]; cand[k] = g_units[j * stride + k]; }
      eps[n - 1] = &ents[w]; cand[n - 1] = need; int64_t e2 = 0; igo_err e;
      alloc_units(eps, cand, n, hw, cap, &e2, &ws, &e);
      int total = 0; for (int k = 0; k < n; ++k) total += cand[k];
      if (total <= cap && total - g_occ[j] < best_inter) { best_j = j; best_inter = total - g_occ[j]; best_n = n; memcpy(best, cand, sizeof(int) * n); }
    }
    /* orders: 0 asc j, 1 desc slack, 2 asc residents, 3 asc power sum, 4 desc slack then asc power, 5 asc (power+1000*cache) */
    for (int o = 0; o < 6; ++o) {
      int nc = 0;
      for (int j = 0; j < G; ++j) if (g_occ[j] + need <= cap) {
        cl[nc++] = j;
        double sl = cap - g_occ[j];
        key[j] = o == 0 ? j : o == 1 ? -sl + j * 1e-9 : o == 2 ? g_n[j] + j * 1e-9 : o == 3 ? g_pw[j] : o == 4 ? -sl * 1e6 + g_pw[j] : g_pw[j] + 1000.0 * g_ca[j];
      }
      qsort(cl, nc, sizeof(int), cmpk);
      unsigned long long run = ~0ull;
      for (int c = 0; c < nc; ++c) {
        int j = cl[c]; unsigned long long k0 = ((unsigned long long)need << 32) | (unsigned)j;
        if (k0 > run) continue;
        int n = g_n[j] + 1;
        for (int k = 0; k < n - 1; ++k) { eps[k] = &ents[g_res[j * stride + k]]; cand[k] = g_units[j * stride + k]; }
        eps[n - 1] = &ents[w]; cand[n - 1] = need;
        int pr = alloc_pruned(eps, cand, n, hw, cap, g_occ[j], run, j, &ev[o], &ws);
        if (!pr) { int total = 0; for (int k = 0; k < n; ++k) total += cand[k];
          unsigned long long kk = ((unsigned long long)(total - g_occ[j]) << 32) | (unsigned)j; if (kk < run) run = kk; }
      }
    }
    int jj;
    if (best_j < 0) { jj = G; g_res[G * stride] = w; g_units[G * stride] = need; g_n[G] = 1; g_occ[G] = need; G++; }
    else { jj = best_j; int occ = 0; g_res[best_j * stride + best_n - 1] = w; for (int k = 0; k < best_n; ++k) { g_units[best_j * stride + k] = best[k]; occ += best[k]; } g_n[best_j] = best_n; g_occ[best_j] = occ; }
    /* power / cache sums of jj */
    double pw = 0, ca = 0;
    for (int k = 0; k < g_n[jj]; ++k) { const entry_t *e = &ents[g_res[jj * stride + k]]; double r = g_units[jj * stride + k] * hw[H_RUNIT];
      double ka = e->gamma / (r + e->k4) + e->k5, ab = e->batch / ka; pw += e->ap * ab + e->bp; double c = e->ac * ab + e->bc; ca += c < 0 ? 0 : c > 1 ? 1 : c; }
    g_pw[jj] = pw; g_ca[jj] = ca;
  }
  printf("m=%d evals: ascj=%lld descslack=%lld ascres=%lld ascpow=%lld slack+pow=%lld pow+cache=%lld\n", m, ev[0], ev[1], ev[2], ev[3], ev[4], ev[5]);
}
