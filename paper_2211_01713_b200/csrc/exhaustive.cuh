// exhaustive.cuh -- the exhaustive oracle's group search on the device.
//
// Restates _Search.best_group_alloc (oracle.py:77-114) for every non-empty
// subset of up to IGP_GS_MAXN workloads at once.  The reference recurses over
// the unit grid, evaluating a unit vector only if it beats the best so far,
// and returns the lexicographic minimum of (total units, unit tuple) over the
// feasible vectors with total <= max_units (oracle.py:93-110).  That minimum
// does not depend on evaluation order, so the device enumerates every vector
// of every subset in parallel, tests feasibility exactly like _Search._feasible
// (oracle.py:64-75: _eval_entries, then t_inf <= t_half and throughput >=
// rate for every member), and keeps the minimum packed key per subset with
// one atomicMin.  Members of a subset are in the caller's order, which is
// name order (oracle.py:86).
//
// Included by igniter_kernels.cu.
#pragma once

namespace igp {

constexpr int GS_MAXN = IGP_GS_MAXN;

struct GroupSearchParams {
  Hw hw;
  int n, n_grid;
  const double *wl;        // [16][n]
  const int32_t *batch;    // [n]
  const int32_t *grid;     // [n_grid] ascending units
  unsigned long long *best;  // [1 << n] packed (total, u_1..u_k), ~0 = infeasible
  int32_t *err;            // first evaluation error code seen (0 = none)
  long long base[(1 << GS_MAXN) + 1];  // combo index offset of each subset
};

// key = total << (9 k) | u_1 << (9 (k - 1)) | ... | u_k   (units <= 256 < 2^9)
__global__ void __launch_bounds__(256) k_group_search(GroupSearchParams G) {
  const long long total = G.base[(1 << G.n)];
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x; g < total; g += stride) {
    int mask = 1;
    while (G.base[mask + 1] <= g) ++mask;  // at most 2^GS_MAXN - 1 subsets
    long long local = g - G.base[mask];
    int idx[GS_MAXN], units[GS_MAXN];
    int k = 0, sum = 0;
    for (int w = 0; w < G.n; ++w)
      if ((mask >> w) & 1) idx[k++] = w;
    // mixed-radix digits, the LAST member fastest (the reference's recursion order)
    for (int d = k - 1; d >= 0; --d) {
      units[d] = G.grid[local % G.n_grid];
      local /= G.n_grid;
      sum += units[d];
    }
    if (sum > G.hw.cap) continue;  // oracle.py:104-105
    const Hw &hw = G.hw;
    const long long ld = G.n;
    // _eval_entries (model.py:273-317) on the subset, entries in member order
    double ka[GS_MAXN], pw[GS_MAXN], ca[GS_MAXN];
    int bad = 0;
    for (int d = 0; d < k && !bad; ++d) {
      const int w = idx[d];
      const double bd = (double)G.batch[w];
      const double gamma = ((G.wl[IGP_WL_K1 * ld + w] * bd) * bd + G.wl[IGP_WL_K2 * ld + w] * bd) +
                           G.wl[IGP_WL_K3 * ld + w];
      const Solo so = solo_at(gamma, G.wl[IGP_WL_K4 * ld + w], G.wl[IGP_WL_K5 * ld + w], bd,
                              G.wl[IGP_WL_ALPHA_P * ld + w], G.wl[IGP_WL_BETA_P * ld + w],
                              G.wl[IGP_WL_ALPHA_CU * ld + w], G.wl[IGP_WL_BETA_CU * ld + w],
                              (double)units[d] * hw.runit);  // oracle.py:70
      if (so.err) bad = so.err;
      ka[d] = so.ka;
      pw[d] = so.pw;
      ca[d] = so.ca;
    }
    if (bad) {
      atomicCAS(G.err, 0, bad);
      continue;
    }
    Neumaier fp, fc;
    fp.first(pw[0]);
    fc.first(ca[0]);
    for (int d = 1; d < k; ++d) {
      fp.add(pw[d]);
      fc.add(ca[d]);
    }
    const double f = frequency(hw, hw.pidle + fp.result());
    const double C = fc.result();
    const double scale = f / hw.fmax;
    const double dl = delta_sch(hw, k);
    bool feasible = true;
    for (int d = 0; d < k && feasible; ++d) {
      const int w = idx[d];
      const double bd = (double)G.batch[w];
      const double t_sch = (G.wl[IGP_WL_KSCH * ld + w] + dl) * G.wl[IGP_WL_NK * ld + w];
      const double t_act = ka[d] * (1.0 + G.wl[IGP_WL_ALPHA_CACHE * ld + w] * (C - ca[d]));
      const double t_gpu = (t_sch + t_act) / scale;
      const double t_load = (G.wl[IGP_WL_DLOAD * ld + w] * bd) / hw.bw;
      const double t_fb = (G.wl[IGP_WL_DFB * ld + w] * bd) / hw.bw;
      const double t_inf = (t_load + t_gpu) + t_fb;
      const double thr = (bd / (t_gpu + t_fb)) * 1000.0;
      // oracle.py:73: row[_T_INF] > t_half or row[_THROUGHPUT] < rate_rps
      if (t_inf > G.wl[IGP_WL_SLO * ld + w] / 2.0 || thr < G.wl[IGP_WL_RATE * ld + w])
        feasible = false;
    }
    if (!feasible) continue;
    unsigned long long key = (unsigned long long)sum;
    for (int d = 0; d < k; ++d) key = (key << 9) | (unsigned long long)units[d];
    atomicMin(&G.best[mask], key);
  }
}

}  // namespace igp
