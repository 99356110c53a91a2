// grid.cuh -- the solo candidate grid (BASELINE config 3, "full candidate grid").
//
// Every (workload w, batch b in 1..b_max, units u in 1..cap) point is one
// single-entry device state of _eval_entries (model.py:273-317) tested with the
// reference's feasibility predicate _Search._feasible (oracle.py:64-75):
//     feasible  <=>  not (t_inf > t_half  or  throughput < rate_rps)
// The entry is _Entry(spec, coef, b, hw) (model.py:253-270) at that batch.
// For each (w, b) the grid reports the smallest feasible u, scanning u upward
// exactly like _Search.best_group_alloc (oracle.py:77-114) does for a
// one-workload group; an evaluation that raises before a feasible point ends
// the scan with the negated error code.  Per workload the cheapest feasible
// point (min u, then min b) is reduced in a second pass.
//
// Included by igniter_kernels.cu (needs Hw, py_max/py_min, frequency).
#pragma once

namespace igp {

struct GridParams {
  Hw hw;
  int m, b_max;
  const double *wl;            // [16][m]
  int32_t *min_units;          // [m][b_max]
  int32_t *best_u, *best_b;    // [m]
  unsigned long long *evals;   // points evaluated (nullable)
};

// One (w, b) row: scan u = 1..cap.  Returns u, 0 (none) or -code.
__device__ __forceinline__ int grid_row(const GridParams &G, int w, int b, int &n_eval) {
  const Hw &hw = G.hw;
  const double *wl = G.wl;
  const long long ld = G.m;
  const double bd = (double)b;
  // _Entry at batch b (model.py:257-270)
  const double gamma = ((wl[IGP_WL_K1 * ld + w] * bd) * bd + wl[IGP_WL_K2 * ld + w] * bd) +
                       wl[IGP_WL_K3 * ld + w];
  const double k4 = wl[IGP_WL_K4 * ld + w], k5 = wl[IGP_WL_K5 * ld + w];
  const double ap = wl[IGP_WL_ALPHA_P * ld + w], bp = wl[IGP_WL_BETA_P * ld + w];
  const double ac = wl[IGP_WL_ALPHA_CU * ld + w], bc = wl[IGP_WL_BETA_CU * ld + w];
  const double acache = wl[IGP_WL_ALPHA_CACHE * ld + w];
  const double t_load = (wl[IGP_WL_DLOAD * ld + w] * bd) / hw.bw;
  const double t_fb = (wl[IGP_WL_DFB * ld + w] * bd) / hw.bw;
  const double t_half = wl[IGP_WL_SLO * ld + w] / 2.0;
  const double rate = wl[IGP_WL_RATE * ld + w];
  // n == 1: delta = 0.0 (model.py:281)
  const double t_sch = (wl[IGP_WL_KSCH * ld + w] + 0.0) * wl[IGP_WL_NK * ld + w];
  int e = 0;
  int res = 0;
  for (int u = 1; u <= hw.cap; ++u) {
    ++e;
    const double r = (double)u * hw.runit;  // oracle.py:70
    const double denom = r + k4;
    if (denom <= 0) {
      res = -IGP_E_DENOM;
      break;
    }
    const double k_act = gamma / denom + k5;
    if (k_act <= 0) {
      res = -IGP_E_ACTIVE_TIME;
      break;
    }
    const double ability = bd / k_act;
    const double pw = ap * ability + bp;
    const double ca = py_min(1.0, py_max(0.0, ac * ability + bc));
    // sum([x]) == 0 + x (CPython builtin sum, one term)
    const double f = frequency(hw, hw.pidle + __dadd_rn(0.0, pw));
    const double C = __dadd_rn(0.0, ca);
    const double x = t_sch + k_act * (1.0 + acache * (C - ca));
    // f == F gives scale = F / F = 1.0 (finite F > 0) and x / 1.0 == x exactly:
    // the division only matters when the power cap binds
    const double t_gpu = (f == hw.fmax && hw.margin_ok) ? x : x / (f / hw.fmax);
    const double t_inf = (t_load + t_gpu) + t_fb;
    if (t_inf > t_half) continue;                           // oracle.py:73 (short-circuit or)
    if ((bd / (t_gpu + t_fb)) * 1000.0 < rate) continue;    // oracle.py:73
    res = u;
    break;
  }
  n_eval = e;
  return res;
}

// thread per (w, b); b fastest so a warp shares one workload's coefficients
__global__ void __launch_bounds__(256) k_solo_grid(GridParams G) {
  const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long tot = (long long)G.m * G.b_max;
  int n_eval = 0;
  if (gid < tot) {
    const int w = (int)(gid / G.b_max);
    const int b = (int)(gid % G.b_max) + 1;
    G.min_units[gid] = grid_row(G, w, b, n_eval);
  }
  if (G.evals) {
    unsigned long long v = (unsigned long long)n_eval;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0 && v) atomicAdd(G.evals, v);
  }
}

// warp per workload: cheapest feasible point (min u, then min b)
__global__ void k_grid_best(GridParams G) {
  const long long wid = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (wid >= G.m) return;
  const int32_t *row = G.min_units + wid * G.b_max;
  unsigned best = 0xffffffffu;  // (u << 16) | b
  for (int b0 = lane; b0 < G.b_max; b0 += 32) {
    const int u = row[b0];
    if (u > 0) {
      const unsigned key = ((unsigned)u << 16) | (unsigned)(b0 + 1);
      best = key < best ? key : best;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned v = __shfl_xor_sync(0xffffffffu, best, o);
    best = v < best ? v : best;
  }
  if (lane == 0) {
    G.best_u[wid] = best == 0xffffffffu ? 0 : (int32_t)(best >> 16);
    G.best_b[wid] = best == 0xffffffffu ? 0 : (int32_t)(best & 0xffffu);
  }
}

}  // namespace igp
