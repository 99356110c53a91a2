// igniter_kernels.cu -- B200 (sm_100a) kernels and C-ABI for the iGniter
// provisioning hot path.  See include/igniter_b200.h for the contract and
// DESIGN.md for the layout/roofline discussion.
//
// Reference restated (file:line in /root/reference/pkg/src/gpuplanner):
//   appropriate_batch     planner.py:76-92      -> prologue_one()
//   _lower_bound_units    planner.py:95-120     -> prologue_one()
//   sorted(-lb, name)     planner.py:284        -> k_sort
//   _Entry                model.py:239-270      -> k_build
//   _eval_entries         model.py:273-317      -> run_candidate() fold/check,
//                                                  k_eval_states, predict phase
//   _alloc_units (Alg. 2) planner.py:133-162    -> run_candidate(), k_alloc_units
//   plan (Alg. 1)         planner.py:290-319    -> k_plan step loop
//   _build_plan           planner.py:218-246    -> k_plan predict phase
//   predict_gpu           model.py:320-343      -> k_eval_states (check_capacity)
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -fmad=false -O3 -lineinfo
// (-fmad=false is REQUIRED: CPython rounds every multiply and add separately).
#include <cuda_runtime.h>

#include <climits>
#include <cstdint>
#include <cstdio>
#include <cstring>

#include "exact_fp64.cuh"

namespace igp {

constexpr unsigned FULL = 0xffffffffu;
constexpr unsigned long long NO_KEY = ~0ull;

static thread_local char g_last_err[256] = "";

static Hw make_hw(const double *h, int b_max) {
  Hw hw;
  hw.pmax = h[IGP_HW_PMAX];
  hw.fmax = h[IGP_HW_FMAX];
  hw.pidle = h[IGP_HW_PIDLE];
  hw.bw = h[IGP_HW_BW];
  hw.af = h[IGP_HW_ALPHA_F];
  hw.asch = h[IGP_HW_ALPHA_SCH];
  hw.bsch = h[IGP_HW_BETA_SCH];
  hw.runit = h[IGP_HW_RUNIT];
  hw.rmax = h[IGP_HW_RMAX];
  hw.price = h[IGP_HW_PRICE];
  hw.fminfrac = h[IGP_HW_FMIN_FRAC];
  hw.fmin = hw.fminfrac * hw.fmax;  // HardwareProfile.f_min_mhz (model.py:108-110)
  // int(round(r_max / r_unit)): CPython round() on a float is half-to-even,
  // which is what nearbyint does in the default rounding mode.
  hw.cap = (int)nearbyint(hw.rmax / hw.runit);
  hw.b_max = b_max;
  return hw;
}

// ---------------------------------------------------------------------------
// Prologue: planner.py:76-120 for workload i.  Returns 0 or an error code;
// `opnd` carries the message operand (b, delta or units).
// ---------------------------------------------------------------------------
__device__ int prologue_one(const double *wl, long long ld, int i, const Hw &hw,
                            const int32_t *batch_in, int &b_out, int &lb_out, double &opnd) {
  const double slo = wl[IGP_WL_SLO * ld + i];
  const double bw = hw.bw;
  int b;
  if (batch_in) {
    b = batch_in[i];
  } else {
    const double rate = wl[IGP_WL_RATE * ld + i] / 1000.0;  // planner.py:80
    const double dl = wl[IGP_WL_DLOAD * ld + i];
    double bx = ceil(((slo * rate) * bw) / (2.0 * (bw + rate * dl)));  // :81-84
    if (!(bx > 1.0)) bx = 1.0;                                         // :85 max(1, b)
    if (bx > (double)hw.b_max) {                                       // :86
      opnd = bx;
      b_out = -1;
      lb_out = -1;
      return IGP_E_BATCH_CAP;
    }
    b = (int)bx;
  }
  b_out = b;
  const double bd = (double)b;
  const double dl = wl[IGP_WL_DLOAD * ld + i], dfb = wl[IGP_WL_DFB * ld + i];
  const double delta = ((slo / 2.0 - ((dl + dfb) * bd) / bw) - wl[IGP_WL_K5 * ld + i]) -
                       wl[IGP_WL_KSCH * ld + i] * wl[IGP_WL_NK * ld + i];  // :101-106
  if (delta <= 0) {
    opnd = delta;
    lb_out = -1;
    return IGP_E_INFEASIBLE_SLO;
  }
  const double gamma = ((wl[IGP_WL_K1 * ld + i] * bd) * bd + wl[IGP_WL_K2 * ld + i] * bd) +
                       wl[IGP_WL_K3 * ld + i];  // :112
  double ux = ceil(gamma / (delta * hw.runit) - wl[IGP_WL_K4 * ld + i] / hw.runit);  // :113
  if (!(ux > 1.0)) ux = 1.0;                                                          // :114
  if (ux > (double)hw.cap) {                                                          // :115
    opnd = ux;
    lb_out = -1;
    return IGP_E_INFEASIBLE_RES;
  }
  lb_out = (int)ux;
  return 0;
}

// Entry constants for workload i at batch b (model.py:253-270).
__device__ __forceinline__ void entry_consts(const double *wl, long long ld, int i, int b,
                                             const Hw &hw, double *cold, double *slot) {
  const double bd = (double)b;
  cold[C_GAMMA] = ((wl[IGP_WL_K1 * ld + i] * bd) * bd + wl[IGP_WL_K2 * ld + i] * bd) +
                  wl[IGP_WL_K3 * ld + i];
  cold[C_K4] = wl[IGP_WL_K4 * ld + i];
  cold[C_K5] = wl[IGP_WL_K5 * ld + i];
  cold[C_BATCH] = bd;
  cold[C_AP] = wl[IGP_WL_ALPHA_P * ld + i];
  cold[C_BP] = wl[IGP_WL_BETA_P * ld + i];
  cold[C_AC] = wl[IGP_WL_ALPHA_CU * ld + i];
  cold[C_BC] = wl[IGP_WL_BETA_CU * ld + i];
  cold[C_KSCH] = wl[IGP_WL_KSCH * ld + i];
  cold[C_NK] = wl[IGP_WL_NK * ld + i];
  slot[S_ACACHE] = wl[IGP_WL_ALPHA_CACHE * ld + i];
  slot[S_TLOAD] = (wl[IGP_WL_DLOAD * ld + i] * bd) / hw.bw;
  slot[S_TFB] = (wl[IGP_WL_DFB * ld + i] * bd) / hw.bw;
  slot[S_THALF] = wl[IGP_WL_SLO * ld + i] / 2.0;
}

// ---------------------------------------------------------------------------
// Plan workspace layout (per scenario arrays, S scenarios back to back)
// ---------------------------------------------------------------------------
struct WsLayout {
  size_t by_rank, order, slot, cold, serr, nres, occ, geidx, gunits, lane_units, risky, perr;
  size_t total;
  int lanes;  // scratch lanes per scenario
};

static size_t align_up(size_t x) { return (x + 255) & ~(size_t)255; }

static WsLayout ws_layout(int S, int m, int cap, int flags) {
  WsLayout L;
  size_t off = 0;
  size_t Sm = (size_t)S * (size_t)(m > 0 ? m : 1);
  int capx = cap > 0 ? cap : 1;
  L.lanes = (flags & IGP_F_CTA) ? 256 : 32;
  L.by_rank = off; off = align_up(off + Sm * 4);
  L.order = off; off = align_up(off + Sm * 4);
  L.slot = off; off = align_up(off + Sm * S_NF * 8);
  L.cold = off; off = align_up(off + Sm * C_NF * 8);
  L.serr = off; off = align_up(off + Sm * 4);
  L.nres = off; off = align_up(off + Sm * 4);
  L.occ = off; off = align_up(off + Sm * 4);
  L.geidx = off; off = align_up(off + Sm * capx * 4);
  L.gunits = off; off = align_up(off + Sm * capx * 2);
  L.lane_units = off; off = align_up(off + (size_t)S * L.lanes * capx * 2);
  L.risky = off; off = align_up(off + (size_t)S * 4);
  L.perr = off; off = align_up(off + (size_t)S * 4);
  L.total = off;
  return L;
}

struct PlanParams {
  Hw hw;
  int S, m, flags;
  const double *wl;        // [S][16][m]
  const int32_t *rank;     // name ranks
  int rank_stride;
  // workspace
  int32_t *by_rank, *order, *serr, *nres, *occ, *geidx, *risky, *perr;
  double *slot, *cold;
  uint16_t *gunits, *lane_units;
  int lanes;
  // outputs
  int32_t *gpu_of, *pos, *units, *batch, *lb, *gpu_count;
  double *pred;
  int64_t *stats;
  igp_error *err;
};

// thread per (scenario, workload): batch, lb, error key, risk flag, by_rank
__global__ void k_prologue_plan(PlanParams P) {
  long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= (long long)P.S * P.m) return;
  int s = (int)(gid / P.m), i = (int)(gid % P.m);
  const double *wl = P.wl + (size_t)s * IGP_WL_NF * P.m;
  int b = -1, u = -1;
  double opnd;
  int rc = prologue_one(wl, P.m, i, P.hw, nullptr, b, u, opnd);
  size_t o = (size_t)s * P.m + i;
  P.batch[o] = b;
  P.lb[o] = u;
  const int32_t *rk = P.rank + (size_t)s * P.rank_stride;
  P.by_rank[(size_t)s * P.m + rk[i]] = i;
  if (rc) {
    atomicMin(&P.perr[s], i);  // first error in INPUT order (planner.py:280-282)
    return;
  }
  // Risk screen for NonPositiveDenominatorError: denom(u) = u*r_unit + k4 is
  // non-decreasing in u and k_act(u) = gamma/denom(u) + k5 is monotone in u
  // (direction = sign of gamma) under round-to-nearest, so the extremes of the
  // reachable range [lb, cap] decide whether any evaluation can raise.
  double cold[C_NF], slot[S_NF];
  entry_consts(wl, P.m, i, b, P.hw, cold, slot);
  Solo a = solo_from_cold(cold, (double)u * P.hw.runit);
  Solo c = solo_from_cold(cold, (double)P.hw.cap * P.hw.runit);
  if (a.err || c.err) atomicOr(&P.risky[s], 1);
}

// warp per scenario: stable counting sort by (-lb, name rank) (planner.py:284)
__global__ void k_sort(PlanParams P) {
  __shared__ int hist[4][257];
  int w = threadIdx.x / 32, lane = threadIdx.x % 32;
  int s = blockIdx.x * 4 + w;
  if (s >= P.S) return;
  if (P.perr[s] != INT_MAX) return;
  const int cap = P.hw.cap, m = P.m;
  const int32_t *lb = P.lb + (size_t)s * m;
  const int32_t *byr = P.by_rank + (size_t)s * m;
  int32_t *order = P.order + (size_t)s * m;
  int *h = hist[w];
  for (int b = lane; b <= cap; b += 32) h[b] = 0;
  __syncwarp();
  for (int i = lane; i < m; i += 32) atomicAdd(&h[cap - lb[i]], 1);
  __syncwarp();
  if (lane == 0) {
    int acc = 0;
    for (int b = 0; b < cap; ++b) {
      int c = h[b];
      h[b] = acc;
      acc += c;
    }
  }
  __syncwarp();
  const unsigned lt = (1u << lane) - 1u;
  for (int base = 0; base < m; base += 32) {
    int r = base + lane;
    bool act = r < m;
    unsigned am = __ballot_sync(FULL, act);
    if (act) {
      int i = byr[r];
      int key = cap - lb[i];
      unsigned peers = __match_any_sync(am, key);
      int before = __popc(peers & lt);
      order[h[key] + before] = i;
      __syncwarp(am);
      if (before == 0) h[key] += __popc(peers);
    }
    __syncwarp();
  }
}

// thread per (scenario, sorted position k): entry constants + solo at lb
__global__ void k_build(PlanParams P) {
  long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= (long long)P.S * P.m) return;
  int s = (int)(gid / P.m), k = (int)(gid % P.m);
  if (P.perr[s] != INT_MAX) return;
  size_t sm = (size_t)s * P.m;
  int i = P.order[sm + k];
  const double *wl = P.wl + (size_t)s * IGP_WL_NF * P.m;
  double cold[C_NF], slot[S_NF];
  int b = P.batch[sm + i], u = P.lb[sm + i];
  entry_consts(wl, P.m, i, b, P.hw, cold, slot);
  cold[C_LB] = (double)u;
  cold[C_WIN] = (double)i;
  Solo so = solo_from_cold(cold, (double)u * P.hw.runit);
  slot[S_KA] = so.ka;
  slot[S_PW] = so.pw;
  slot[S_CA] = so.ca;
  slot[S_TSN] = 0.0;
  double *cd = P.cold + (sm + k) * C_NF;
  double *sd = P.slot + (sm + k) * S_NF;
#pragma unroll
  for (int f = 0; f < C_NF; ++f) cd[f] = cold[f];
#pragma unroll
  for (int f = 0; f < S_NF; ++f) sd[f] = slot[f];
  P.serr[sm + k] = so.err;
}

// ---------------------------------------------------------------------------
// Candidate evaluation: Alg. 2 (planner.py:133-162) on residents_j + [new].
// ---------------------------------------------------------------------------
enum { R_FEAS = 0, R_INFEAS = 1, R_PRUNED = 2, R_ERROR = 3 };

template <int MAXN>
struct Cand {
  int idx[MAXN];
  int u[MAXN];
  double ka[MAXN], pw[MAXN], ca[MAXN];
};

struct Scn {
  const double *cold;
  const double *slot;
  const int32_t *serr, *nres, *occ, *geidx;
  const uint16_t *gunits;
  int cap;
};

struct ErrOut {
  int code, e;
  double a, b, c;
};

__device__ __forceinline__ void err_operands(const Hw &hw, const double *ce, int u, int code,
                                             ErrOut &eo) {
  double r = (double)u * hw.runit;
  double denom = r + ce[C_K4];
  eo.code = code;
  if (code == IGP_E_DENOM) {
    eo.a = denom;
    eo.b = r;
    eo.c = ce[C_K4];
  } else {
    eo.a = ce[C_GAMMA] / denom + ce[C_K5];
    eo.b = ce[C_BATCH];
    eo.c = r;
  }
}

// Runs one candidate.  exact: reference evaluation sequence (no overflow exit,
// no prune), counts evaluations and surfaces NonPositiveDenominatorError at the
// evaluation where the reference raises it.  Fast mode (exact == false) stops
// at the first unit overflow (units only grow, so the candidate is already
// infeasible) and when its running (inter, j) key can no longer beat the best
// key found so far in this step (inter only grows); neither changes the
// placement decision.
template <int MAXN>
__device__ int run_candidate(const Hw &hw, const Scn &sc, int j, int k, int need, double tsch_new,
                             bool exact, const volatile unsigned long long *best, Cand<MAXN> &cd,
                             int &n_out, int &sum_out, long long &evals, long long &calls,
                             ErrOut &eo) {
  const int cap = sc.cap;
  const int nres = sc.nres[j];
  const int n = nres + 1;
  const int occ = sc.occ[j];
  const int32_t *gi = sc.geidx + (size_t)j * cap;
  const uint16_t *gu = sc.gunits + (size_t)j * cap;
  for (int q = 0; q < nres; ++q) {
    int e = gi[q];
    cd.idx[q] = e;
    cd.u[q] = gu[q];
    const double *sl = sc.slot + (size_t)e * S_NF;
    cd.ka[q] = sl[S_KA];
    cd.pw[q] = sl[S_PW];
    cd.ca[q] = sl[S_CA];
  }
  {
    const double *sl = sc.slot + (size_t)k * S_NF;
    cd.idx[nres] = k;
    cd.u[nres] = need;
    cd.ka[nres] = sl[S_KA];
    cd.pw[nres] = sl[S_PW];
    cd.ca[nres] = sl[S_CA];
  }
  n_out = n;
  int sum = occ + need;
  int pend = -1, pend_code = 0;
  if (exact) {
    for (int q = 0; q < n; ++q) {
      int ec = sc.serr[cd.idx[q]];
      if (ec) {
        pend = q;
        pend_code = ec;
        break;
      }
    }
  }
  bool flag = true;
  double C = 0.0, scale = 1.0;
  while (sum <= cap && flag) {
    flag = false;
    bool need_eval = true;
    for (int i = 0; i < n; ++i) {
      if (need_eval) {
        if (pend >= 0) {
          err_operands(hw, sc.cold + (size_t)cd.idx[pend] * C_NF, cd.u[pend], pend_code, eo);
          eo.e = cd.idx[pend];
          sum_out = sum;
          return R_ERROR;
        }
        // _eval_entries device-level terms (model.py:299-305)
        Neumaier fp, fc;
        fp.first(cd.pw[0]);
        fc.first(cd.ca[0]);
        for (int q = 1; q < n; ++q) {
          fp.add(cd.pw[q]);
          fc.add(cd.ca[q]);
        }
        const double p_dem = hw.pidle + fp.result();
        const double f = frequency(hw, p_dem);
        C = fc.result();
        scale = f / hw.fmax;
        evals += n;
        calls += 1;
        need_eval = false;
      }
      // per-resident terms (model.py:308-313); only t_inf is tested (planner.py:158)
      const int e = cd.idx[i];
      const double *sl = sc.slot + (size_t)e * S_NF;
      const double t_sch = (i == n - 1) ? tsch_new : sl[S_TSN];
      const double co_cache = C - cd.ca[i];
      const double t_act = cd.ka[i] * (1.0 + sl[S_ACACHE] * co_cache);
      const double x = t_sch + t_act;
      const double t_gpu = (scale == 1.0) ? x : x / scale;  // x / 1.0 == x exactly
      const double t_inf = (sl[S_TLOAD] + t_gpu) + sl[S_TFB];
      if (t_inf > sl[S_THALF]) {
        cd.u[i] += 1;
        sum += 1;
        const Solo so = solo_from_cold(sc.cold + (size_t)e * C_NF, (double)cd.u[i] * hw.runit);
        cd.ka[i] = so.ka;
        cd.pw[i] = so.pw;
        cd.ca[i] = so.ca;
        if (exact && so.err && pend < 0) {
          pend = i;
          pend_code = so.err;
        }
        flag = true;
        need_eval = true;
        if (!exact) {
          if (sum > cap) {
            sum_out = sum;
            return R_INFEAS;
          }
          unsigned long long key = ((unsigned long long)(sum - occ) << 32) | (unsigned)j;
          if (key > *best) {
            sum_out = sum;
            return R_PRUNED;
          }
        }
      }
    }
  }
  sum_out = sum;
  return (sum <= cap) ? R_FEAS : R_INFEAS;
}

struct GroupSmem {
  unsigned long long best;
  unsigned long long tot[3];  // model_evals, eval calls, candidates
  int err_flag;
  int win_thread;
  int err_gpu;
};

template <int GW>
__device__ __forceinline__ void group_sync() {
  if (GW == 1) __syncwarp();
  else __syncthreads();
}

__device__ __forceinline__ int warp_sum(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  return v;
}

// One scenario per group of GW warps (GW == 1: four independent scenarios per
// 128-thread CTA; GW > 1: one scenario per CTA).
template <int MAXN, int GW>
__global__ void __launch_bounds__(GW == 1 ? 128 : GW * 32)
k_plan(PlanParams P) {
  constexpr int GT = GW * 32;
  constexpr int GPB = (GW == 1) ? 4 : 1;
  __shared__ GroupSmem gsm[GPB];
  __shared__ int qsm[GPB * GW][64];
  const int grp = threadIdx.x / GT, t = threadIdx.x % GT, wi = t / 32, lane = t % 32;
  const int s = blockIdx.x * GPB + grp;
  if (s >= P.S) return;
  GroupSmem &gs = gsm[grp];
  int *q = qsm[grp * GW + wi];
  const Hw &hw = P.hw;
  const int m = P.m, cap = hw.cap;
  const size_t sm = (size_t)s * m;
  igp_error *err = P.err + s;

  if (P.perr[s] != INT_MAX) {  // prologue error, input order (planner.py:280-282)
    if (t == 0) {
      int i = P.perr[s], b, u;
      double opnd = 0.0;
      const double *wl = P.wl + (size_t)s * IGP_WL_NF * m;
      int rc = prologue_one(wl, m, i, hw, nullptr, b, u, opnd);
      err->code = rc;
      err->workload = i;
      err->gpu = -1;
      err->a = opnd;
      err->b = (double)hw.b_max;
      err->c = 0.0;
      P.gpu_count[s] = 0;
      if (P.stats) {
        const long long z = (P.flags & IGP_F_STATS) ? 0 : -1;
        P.stats[4 * s] = z;
        P.stats[4 * s + 1] = z;
        P.stats[4 * s + 2] = z;
        P.stats[4 * s + 3] = 0;
      }
    }
    return;
  }

  Scn sc;
  sc.cold = P.cold + sm * C_NF;
  sc.slot = P.slot + sm * S_NF;
  sc.serr = P.serr + sm;
  sc.nres = P.nres + sm;
  sc.occ = P.occ + sm;
  sc.geidx = P.geidx + sm * cap;
  sc.gunits = P.gunits + sm * cap;
  sc.cap = cap;
  double *slot = P.slot + sm * S_NF;
  int32_t *serr = P.serr + sm;
  int32_t *nres = P.nres + sm;
  int32_t *occ = P.occ + sm;
  int32_t *geidx = P.geidx + sm * cap;
  uint16_t *gunits = P.gunits + sm * cap;
  uint16_t *lane_units = P.lane_units + (size_t)s * P.lanes * cap;
  const bool exact = (P.flags & IGP_F_STATS) || P.risky[s];
  const unsigned lt = (1u << lane) - 1u;

  Cand<MAXN> cd;
  int G = 0;
  // per-thread counters: committed totals and the current step's share
  long long tot_evals = 0, tot_calls = 0, tot_cands = 0;
  long long st_evals = 0, st_calls = 0, st_cands = 0;
  bool failed = false;
  ErrOut eo_fail;
  eo_fail.code = 0;

  for (int k = 0; k < m; ++k) {
    const double *ck = sc.cold + (size_t)k * C_NF;
    const int need = (int)ck[C_LB];
    const double ksch = ck[C_KSCH], nk = ck[C_NK];
    if (t == 0) {
      gs.best = NO_KEY;
      gs.err_flag = 0;
    }
    group_sync<GW>();
    unsigned long long my_best = NO_KEY;

    auto process = [&](int j) {
      int n = 0, sum = 0;
      long long ev = 0, calls = 0;
      ErrOut eo;
      const double tsch_new = (ksch + delta_sch(hw, nres[j] + 1)) * nk;
      int r = run_candidate<MAXN>(hw, sc, j, k, need, tsch_new, exact, &gs.best, cd, n, sum, ev,
                                  calls, eo);
      st_evals += ev;
      st_calls += calls;
      st_cands += 1;
      if (r == R_ERROR) {
        atomicOr(&gs.err_flag, 1);
      } else if (r == R_FEAS) {
        unsigned long long key = ((unsigned long long)(sum - occ[j]) << 32) | (unsigned)j;
        if (key < my_best) {
          my_best = key;
          uint16_t *lu = lane_units + (size_t)t * cap;
          for (int qq = 0; qq < n; ++qq) lu[qq] = (uint16_t)cd.u[qq];
        }
        atomicMin(&gs.best, key);
      }
    };

    // prefilter (planner.py:297-299) + ballot compaction into a per-warp queue
    int qn = 0;
    for (int base = wi * 32; base < G; base += GT) {
      const int j = base + lane;
      const bool pass = (j < G) && (occ[j] + need <= cap);
      const unsigned mask = __ballot_sync(FULL, pass);
      if (pass) q[qn + __popc(mask & lt)] = j;
      qn += __popc(mask);
      __syncwarp();
      if (qn >= 32) {
        process(q[lane]);
        __syncwarp();
        qn -= 32;
        if (lane < qn) q[lane] = q[lane + 32];
        __syncwarp();
      }
    }
    if (lane < qn) process(q[lane]);
    group_sync<GW>();

    if (gs.err_flag) {
      // exact mode only: replay this step in the reference's candidate order
      // to find the first raising candidate and the PlanStats at that point.
      if (t == 0) {
        for (int j = 0; j < G; ++j) {
          if (occ[j] + need > cap) continue;
          tot_cands++;
          int n = 0, sum = 0;
          long long ev = 0, calls = 0;
          ErrOut eo;
          const double tsch_new = (ksch + delta_sch(hw, nres[j] + 1)) * nk;
          int r = run_candidate<MAXN>(hw, sc, j, k, need, tsch_new, true, &gs.best, cd, n, sum, ev,
                                      calls, eo);
          tot_evals += ev;
          tot_calls += calls;
          if (r == R_ERROR) {
            eo_fail = eo;
            break;
          }
        }
      }
      failed = true;
      break;
    }
    tot_evals += st_evals;
    tot_calls += st_calls;
    tot_cands += st_cands;
    st_evals = st_calls = st_cands = 0;
    const unsigned long long bk = gs.best;
    if (bk != NO_KEY && my_best == bk) gs.win_thread = t;
    group_sync<GW>();

    // commit (planner.py:312-319), warp 0 of the group
    if (wi == 0) {
      if (bk == NO_KEY) {
        if (lane == 0) {
          nres[G] = 1;
          occ[G] = need;
          geidx[(size_t)G * cap] = k;
          gunits[(size_t)G * cap] = (uint16_t)need;
          slot[(size_t)k * S_NF + S_TSN] = (ksch + delta_sch(hw, 2)) * nk;
        }
      } else {
        const int j = (int)(bk & 0xffffffffu);
        const uint16_t *lu = lane_units + (size_t)gs.win_thread * cap;
        const int n = nres[j] + 1;
        const double dnext = delta_sch(hw, n + 1);
        int part = 0;
        for (int r = lane; r < n; r += 32) {
          const int e = (r == n - 1) ? k : geidx[(size_t)j * cap + r];
          const int nu = lu[r];
          const int ou = (r == n - 1) ? need : gunits[(size_t)j * cap + r];
          const double *ce = sc.cold + (size_t)e * C_NF;
          double *se = slot + (size_t)e * S_NF;
          if (nu != ou) {
            Solo so = solo_from_cold(ce, (double)nu * hw.runit);
            se[S_KA] = so.ka;
            se[S_PW] = so.pw;
            se[S_CA] = so.ca;
            serr[e] = so.err;
          }
          se[S_TSN] = (ce[C_KSCH] + dnext) * ce[C_NK];
          gunits[(size_t)j * cap + r] = (uint16_t)nu;
          if (r == n - 1) geidx[(size_t)j * cap + r] = k;
          part += nu;
        }
        part = warp_sum(part);
        if (lane == 0) {
          occ[j] = part;
          nres[j] = n;
        }
      }
    }
    if (bk == NO_KEY) G += 1;
    __threadfence_block();
    group_sync<GW>();
  }

  // group totals of the counters
  if (t == 0) gs.tot[0] = gs.tot[1] = gs.tot[2] = 0;
  group_sync<GW>();
  atomicAdd(&gs.tot[0], (unsigned long long)tot_evals);
  atomicAdd(&gs.tot[1], (unsigned long long)tot_calls);
  atomicAdd(&gs.tot[2], (unsigned long long)tot_cands);
  group_sync<GW>();
  if (t == 0 && P.stats) {
    const bool st_ok = (P.flags & IGP_F_STATS) || failed;
    P.stats[4 * s] = st_ok ? (long long)gs.tot[0] : -1;
    P.stats[4 * s + 1] = st_ok ? (long long)gs.tot[2] : -1;
    P.stats[4 * s + 2] = st_ok ? (long long)gs.tot[1] : -1;
    P.stats[4 * s + 3] = (long long)gs.tot[1];
  }

  if (failed) {
    if (t == 0) {
      err->code = eo_fail.code;
      err->workload = (int)sc.cold[(size_t)eo_fail.e * C_NF + C_WIN];
      err->gpu = -1;
      err->a = eo_fail.a;
      err->b = eo_fail.b;
      err->c = eo_fail.c;
      P.gpu_count[s] = G;
    }
    return;
  }

  // _build_plan (planner.py:218-246): predict_gpu per device (model.py:320-343)
  if (t == 0) gs.err_gpu = INT_MAX;
  group_sync<GW>();
  int my_err_gpu = INT_MAX;
  ErrOut my_eo;
  my_eo.code = 0;
  const bool want_pred = P.pred && !(P.flags & IGP_F_NO_PRED);
  for (int j = t; j < G; j += GT) {
    const int n = nres[j];
    const int32_t *gi = geidx + (size_t)j * cap;
    const uint16_t *gu = gunits + (size_t)j * cap;
    // capacity check: sum(a.r) with a.r = u * r_unit (model.py:331-335)
    Neumaier cs;
    cs.first((double)gu[0] * hw.runit);
    for (int qq = 1; qq < n; ++qq) cs.add((double)gu[qq] * hw.runit);
    const double total_r = cs.result();
    int ecode = 0;
    if (total_r > hw.rmax + 1e-9) {
      ecode = IGP_E_OVERALLOC;
      if (j < my_err_gpu) {
        my_err_gpu = j;
        my_eo.code = ecode;
        my_eo.e = -1;
        my_eo.a = total_r;
        my_eo.b = hw.rmax;
        my_eo.c = 0.0;
      }
    }
    Neumaier fp, fc;
    for (int qq = 0; qq < n; ++qq) {
      const int e = gi[qq];
      const Solo so = solo_from_cold(sc.cold + (size_t)e * C_NF, (double)gu[qq] * hw.runit);
      if (!ecode && so.err) {
        ecode = so.err;
        if (j < my_err_gpu) {
          my_err_gpu = j;
          err_operands(hw, sc.cold + (size_t)e * C_NF, gu[qq], so.err, my_eo);
          my_eo.e = e;
        }
      }
      cd.ka[qq] = so.ka;
      cd.ca[qq] = so.ca;
      cd.pw[qq] = so.pw;
      if (qq == 0) {
        fp.first(so.pw);
        fc.first(so.ca);
      } else {
        fp.add(so.pw);
        fc.add(so.ca);
      }
    }
    const double f = frequency(hw, hw.pidle + fp.result());
    const double C = fc.result();
    const double scale = f / hw.fmax;
    const double dl = delta_sch(hw, n);
    for (int qq = 0; qq < n; ++qq) {
      const int e = gi[qq];
      const double *ce = sc.cold + (size_t)e * C_NF;
      const double *se = slot + (size_t)e * S_NF;
      const int w_in = (int)ce[C_WIN];
      P.gpu_of[sm + w_in] = j;
      P.pos[sm + w_in] = qq;
      P.units[sm + w_in] = gu[qq];
      if (want_pred) {
        const double t_sch = (ce[C_KSCH] + dl) * ce[C_NK];
        const double t_act = cd.ka[qq] * (1.0 + se[S_ACACHE] * (C - cd.ca[qq]));
        const double t_gpu = (t_sch + t_act) / scale;
        const double t_inf = (se[S_TLOAD] + t_gpu) + se[S_TFB];
        double *row = P.pred + (sm + w_in) * 10;
        row[0] = se[S_TLOAD];
        row[1] = t_sch;
        row[2] = t_act;
        row[3] = f;
        row[4] = t_gpu;
        row[5] = se[S_TFB];
        row[6] = t_inf;
        row[7] = (ce[C_BATCH] / (t_gpu + se[S_TFB])) * 1000.0;
        row[8] = cd.pw[qq];
        row[9] = cd.ca[qq];
      }
    }
  }
  if (my_err_gpu != INT_MAX) atomicMin(&gs.err_gpu, my_err_gpu);
  group_sync<GW>();
  const int eg = gs.err_gpu;
  if (eg != INT_MAX && my_err_gpu == eg) {
    err->code = my_eo.code;
    err->workload = my_eo.e >= 0 ? (int)sc.cold[(size_t)my_eo.e * C_NF + C_WIN] : -1;
    err->gpu = eg;
    err->a = my_eo.a;
    err->b = my_eo.b;
    err->c = my_eo.c;
  }
  if (t == 0) {
    if (eg == INT_MAX) {
      err->code = 0;
      err->workload = -1;
      err->gpu = -1;
      err->a = err->b = err->c = 0.0;
    }
    P.gpu_count[s] = G;
  }
}

// ---------------------------------------------------------------------------
// Batched _eval_entries / predict_gpu: thread per device state.
// ---------------------------------------------------------------------------
struct RowEntry {
  double gamma, k4, k5, batch, ap, bp, ac, bc, ksch, nk, acache, t_load, t_fb;
};

__device__ __forceinline__ RowEntry row_entry(const double *wl, long long ld, int i, int b,
                                              const Hw &hw) {
  RowEntry r;
  const double bd = (double)b;
  r.gamma = ((wl[IGP_WL_K1 * ld + i] * bd) * bd + wl[IGP_WL_K2 * ld + i] * bd) + wl[IGP_WL_K3 * ld + i];
  r.k4 = wl[IGP_WL_K4 * ld + i];
  r.k5 = wl[IGP_WL_K5 * ld + i];
  r.batch = bd;
  r.ap = wl[IGP_WL_ALPHA_P * ld + i];
  r.bp = wl[IGP_WL_BETA_P * ld + i];
  r.ac = wl[IGP_WL_ALPHA_CU * ld + i];
  r.bc = wl[IGP_WL_BETA_CU * ld + i];
  r.ksch = wl[IGP_WL_KSCH * ld + i];
  r.nk = wl[IGP_WL_NK * ld + i];
  r.acache = wl[IGP_WL_ALPHA_CACHE * ld + i];
  r.t_load = (wl[IGP_WL_DLOAD * ld + i] * bd) / hw.bw;
  r.t_fb = (wl[IGP_WL_DFB * ld + i] * bd) / hw.bw;
  return r;
}

__device__ __forceinline__ void set_err(igp_error *e, int code, int w, double a, double b, double c) {
  e->code = code;
  e->workload = w;
  e->gpu = -1;
  e->pad = 0;
  e->a = a;
  e->b = b;
  e->c = c;
}

// Evaluates state [b0, b0+n) with the given units source; returns 0 or error.
// Writes t_inf (tinf != null) or full rows (rows != null).
template <typename RFn>
__device__ int eval_state(const double *wl, long long ld, const int32_t *batch, long long b0, int n,
                          const Hw &hw, RFn rfn, double *rows, igp_error *e, double *tinf_i,
                          int want_i) {
  const double dl = delta_sch(hw, n);
  Neumaier fp, fc;
  for (int q = 0; q < n; ++q) {
    const long long gi = b0 + q;
    const RowEntry re = row_entry(wl, ld, (int)gi, batch[gi], hw);
    const double r = rfn(q);
    const Solo so = solo_at(re.gamma, re.k4, re.k5, re.batch, re.ap, re.bp, re.ac, re.bc, r);
    if (so.err) {
      const double denom = r + re.k4;
      if (so.err == IGP_E_DENOM) set_err(e, so.err, (int)gi, denom, r, re.k4);
      else set_err(e, so.err, (int)gi, re.gamma / denom + re.k5, re.batch, r);
      return so.err;
    }
    if (q == 0) {
      fp.first(so.pw);
      fc.first(so.ca);
    } else {
      fp.add(so.pw);
      fc.add(so.ca);
    }
  }
  const double f = frequency(hw, hw.pidle + fp.result());
  const double C = fc.result();
  const double scale = f / hw.fmax;
  for (int q = 0; q < n; ++q) {
    if (!rows && q != want_i) continue;
    const long long gi = b0 + q;
    const RowEntry re = row_entry(wl, ld, (int)gi, batch[gi], hw);
    const double r = rfn(q);
    const Solo so = solo_at(re.gamma, re.k4, re.k5, re.batch, re.ap, re.bp, re.ac, re.bc, r);
    const double t_sch = (re.ksch + dl) * re.nk;
    const double t_act = so.ka * (1.0 + re.acache * (C - so.ca));
    const double t_gpu = (t_sch + t_act) / scale;
    const double t_inf = (re.t_load + t_gpu) + re.t_fb;
    if (tinf_i) *tinf_i = t_inf;
    if (rows) {
      double *row = rows + gi * 10;
      row[0] = re.t_load;
      row[1] = t_sch;
      row[2] = t_act;
      row[3] = f;
      row[4] = t_gpu;
      row[5] = re.t_fb;
      row[6] = t_inf;
      row[7] = (re.batch / (t_gpu + re.t_fb)) * 1000.0;
      row[8] = so.pw;
      row[9] = so.ca;
    }
  }
  return 0;
}

__global__ void k_eval_states(const double *wl, int n_rows, const int32_t *batch, const double *r,
                              const int64_t *ptr, int n_states, Hw hw, int check_capacity,
                              double *rows, igp_error *err, int *first_err) {
  int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n_states) return;
  const long long b0 = ptr[s];
  const int n = (int)(ptr[s + 1] - b0);
  igp_error *e = err + s;
  set_err(e, 0, -1, 0.0, 0.0, 0.0);
  if (check_capacity && n > 0) {
    Neumaier cs;
    cs.first(r[b0]);
    for (int q = 1; q < n; ++q) cs.add(r[b0 + q]);
    const double tot = cs.result();
    if (tot > hw.rmax + 1e-9) {
      set_err(e, IGP_E_OVERALLOC, -1, tot, hw.rmax, 0.0);
      atomicMin(first_err, s);
      return;
    }
  }
  if (n == 0) return;
  const double *rr = r + b0;
  int rc = eval_state(wl, n_rows, batch, b0, n, hw, [&](int q) { return rr[q]; }, rows, e,
                      nullptr, -1);
  if (rc) atomicMin(first_err, s);
}

// Alg. 2 (planner.py:133-162), reference evaluation sequence, one thread per state.
__global__ void k_alloc_units(const double *wl, int n_rows, const int32_t *batch, const double *r,
                              const int64_t *ptr, int n_states, Hw hw, int32_t *units,
                              igp_error *err, int *first_err) {
  int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n_states) return;
  const long long b0 = ptr[s];
  const int n = (int)(ptr[s + 1] - b0);
  igp_error *e = err + s;
  set_err(e, 0, -1, 0.0, 0.0, 0.0);
  int32_t *u = units + b0;
  for (int q = 0; q < n; ++q) u[q] = (int32_t)nearbyint(r[b0 + q] / hw.runit);  // planner.py:184-185
  auto rfn = [&](int q) { return (double)u[q] * hw.runit; };
  bool flag = true;
  for (;;) {
    long long total = 0;
    for (int q = 0; q < n; ++q) total += u[q];
    if (!(total <= hw.cap && flag)) break;
    flag = false;
    bool need_eval = true;
    for (int i = 0; i < n; ++i) {
      if (need_eval) {
        // validate the whole state once (errors surface in entry order)
        int rc = eval_state(wl, n_rows, batch, b0, n, hw, rfn, nullptr, e, nullptr, -1);
        if (rc) {
          atomicMin(first_err, s);
          return;
        }
        need_eval = false;
      }
      double t_inf = 0.0;
      eval_state(wl, n_rows, batch, b0, n, hw, rfn, nullptr, e, &t_inf, i);
      const double t_half = wl[IGP_WL_SLO * (long long)n_rows + b0 + i] / 2.0;
      if (t_inf > t_half) {
        u[i] += 1;
        flag = true;
        need_eval = true;
      }
    }
  }
}

// thread per workload: appropriate_batch / _lower_bound_units
__global__ void k_prologue(const double *wl, int m, Hw hw, const int32_t *batch_in, int32_t *batch,
                           int32_t *lb, int32_t *code, int *first_err) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  int b = -1, u = -1;
  double opnd = 0.0;
  int rc = prologue_one(wl, m, i, hw, batch_in, b, u, opnd);
  batch[i] = b;
  lb[i] = u;
  code[i] = rc;
  if (rc) atomicMin(first_err, i);
}

__global__ void k_prologue_err(const double *wl, int m, Hw hw, const int32_t *batch_in,
                               const int *first_err, igp_error *err) {
  int i = *first_err;
  if (i == INT_MAX) {
    set_err(err, 0, -1, 0.0, 0.0, 0.0);
    return;
  }
  int b, u;
  double opnd = 0.0;
  int rc = prologue_one(wl, m, i, hw, batch_in, b, u, opnd);
  set_err(err, rc, i, opnd, (double)hw.b_max, 0.0);
}

__global__ void k_fill_int(int *p, int n, int v) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = v;
}

}  // namespace igp

// ===========================================================================
// C-ABI
// ===========================================================================
using namespace igp;

static int cuda_fail(cudaError_t e) {
  snprintf(g_last_err, sizeof(g_last_err), "%s", cudaGetErrorString(e));
  return IGP_E_CUDA;
}
#define CK(x)                              \
  do {                                     \
    cudaError_t e_ = (x);                  \
    if (e_ != cudaSuccess) return cuda_fail(e_); \
  } while (0)

static inline unsigned nblk(long long n, int t) { return (unsigned)((n + t - 1) / t); }

template <int MAXN>
static void launch_plan(const PlanParams &P, cudaStream_t st) {
  if (P.flags & IGP_F_CTA) {
    k_plan<MAXN, 8><<<P.S, 256, 0, st>>>(P);
  } else {
    k_plan<MAXN, 1><<<nblk(P.S, 4), 128, 0, st>>>(P);
  }
}

extern "C" {

int igp_abi_version(void) { return IGP_ABI_VERSION; }
int igp_max_cap(void) { return 256; }
const char *igp_last_error_string(void) { return g_last_err; }

size_t igp_plan_workspace_bytes(int n_scen, int m, const double *hw, int b_max, int flags) {
  Hw h = make_hw(hw, b_max);
  return ws_layout(n_scen, m, h.cap, flags).total;
}

static int plan_device_impl(const double *wl, int n_scen, int m, const double *hw_h, int b_max,
                            const int32_t *name_rank, int rank_stride, int32_t *gpu_of,
                            int32_t *pos, int32_t *units, int32_t *batch, int32_t *lb,
                            double *pred, int32_t *gpu_count, int64_t *stats, igp_error *err,
                            void *workspace, size_t workspace_bytes, int flags, void *stream,
                            int stages) {
  if (n_scen < 0 || m < 0 || !hw_h) return IGP_E_ARG;
  if (n_scen == 0) return IGP_E_OK;
  Hw hw = make_hw(hw_h, b_max);
  if (hw.cap < 1) return IGP_E_ARG;
  if (hw.cap > igp_max_cap()) return IGP_E_CAPACITY;
  WsLayout L = ws_layout(n_scen, m, hw.cap, flags);
  if (workspace_bytes < L.total || !workspace) return IGP_E_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  char *ws = (char *)workspace;
  PlanParams P;
  P.hw = hw;
  P.S = n_scen;
  P.m = m;
  P.flags = flags;
  P.wl = wl;
  P.rank = name_rank;
  P.rank_stride = rank_stride;
  P.by_rank = (int32_t *)(ws + L.by_rank);
  P.order = (int32_t *)(ws + L.order);
  P.slot = (double *)(ws + L.slot);
  P.cold = (double *)(ws + L.cold);
  P.serr = (int32_t *)(ws + L.serr);
  P.nres = (int32_t *)(ws + L.nres);
  P.occ = (int32_t *)(ws + L.occ);
  P.geidx = (int32_t *)(ws + L.geidx);
  P.gunits = (uint16_t *)(ws + L.gunits);
  P.lane_units = (uint16_t *)(ws + L.lane_units);
  P.lanes = L.lanes;
  P.risky = (int32_t *)(ws + L.risky);
  P.perr = (int32_t *)(ws + L.perr);
  P.gpu_of = gpu_of;
  P.pos = pos;
  P.units = units;
  P.batch = batch;
  P.lb = lb;
  P.pred = pred;
  P.gpu_count = gpu_count;
  P.stats = stats;
  P.err = err;
  if (stages & 1) {
    CK(cudaMemsetAsync(P.risky, 0, (size_t)n_scen * 4, st));
    k_fill_int<<<nblk(n_scen, 256), 256, 0, st>>>(P.perr, n_scen, INT_MAX);
    if (m > 0) {
      long long tot = (long long)n_scen * m;
      k_prologue_plan<<<nblk(tot, 256), 256, 0, st>>>(P);
      k_sort<<<nblk(n_scen, 4), 128, 0, st>>>(P);
      k_build<<<nblk(tot, 256), 256, 0, st>>>(P);
    }
  }
  if (stages & 2) {
    if (hw.cap <= 48) launch_plan<48>(P, st);
    else if (hw.cap <= 128) launch_plan<128>(P, st);
    else launch_plan<256>(P, st);
  }
  CK(cudaGetLastError());
  return IGP_E_OK;
}

#define PLAN_ARGS_DECL                                                                          \
  const double *wl, int n_scen, int m, const double *hw_h, int b_max, const int32_t *name_rank, \
      int rank_stride, int32_t *gpu_of, int32_t *pos, int32_t *units, int32_t *batch,           \
      int32_t *lb, double *pred, int32_t *gpu_count, int64_t *stats, igp_error *err,             \
      void *workspace, size_t workspace_bytes, int flags, void *stream
#define PLAN_ARGS_PASS                                                                        \
  wl, n_scen, m, hw_h, b_max, name_rank, rank_stride, gpu_of, pos, units, batch, lb, pred,     \
      gpu_count, stats, err, workspace, workspace_bytes, flags, stream

int igp_plan_batch_device(PLAN_ARGS_DECL) { return plan_device_impl(PLAN_ARGS_PASS, 3); }
int igp_plan_prepare_device(PLAN_ARGS_DECL) { return plan_device_impl(PLAN_ARGS_PASS, 1); }
int igp_plan_place_device(PLAN_ARGS_DECL) { return plan_device_impl(PLAN_ARGS_PASS, 2); }

int igp_plan_batch_host(const double *wl, int n_scen, int m, const double *hw_h, int b_max,
                        const int32_t *name_rank, int rank_stride, int32_t *gpu_of, int32_t *pos,
                        int32_t *units, int32_t *batch, int32_t *lb, double *pred,
                        int32_t *gpu_count, int64_t *stats, igp_error *err, void *workspace,
                        size_t workspace_bytes, int flags, void *stream) {
  if (n_scen < 0 || m < 0 || !hw_h) return IGP_E_ARG;
  if (n_scen == 0) return IGP_E_OK;
  Hw hw = make_hw(hw_h, b_max);
  if (hw.cap < 1) return IGP_E_ARG;
  if (hw.cap > igp_max_cap()) return IGP_E_CAPACITY;
  WsLayout L = ws_layout(n_scen, m, hw.cap, flags);
  // device I/O buffers are carved after the planning scratch
  size_t Sm = (size_t)n_scen * (m > 0 ? m : 1);
  size_t rank_n = rank_stride ? Sm : (size_t)(m > 0 ? m : 1);
  size_t off = L.total;
  size_t o_wl = off; off = align_up(off + Sm * IGP_WL_NF * 8);
  size_t o_rank = off; off = align_up(off + rank_n * 4);
  size_t o_i32 = off; off = align_up(off + Sm * 4 * 5);
  size_t o_pred = off; off = align_up(off + (pred ? Sm * 80 : 0));
  size_t o_gc = off; off = align_up(off + (size_t)n_scen * 4);
  size_t o_st = off; off = align_up(off + (size_t)n_scen * 32);
  size_t o_err = off; off = align_up(off + (size_t)n_scen * sizeof(igp_error));
  if (!workspace || workspace_bytes < off) return IGP_E_ARG;
  char *ws = (char *)workspace;
  cudaStream_t st = (cudaStream_t)stream;
  double *d_wl = (double *)(ws + o_wl);
  int32_t *d_rank = (int32_t *)(ws + o_rank);
  int32_t *d_i32 = (int32_t *)(ws + o_i32);
  double *d_pred = pred ? (double *)(ws + o_pred) : nullptr;
  int32_t *d_gc = (int32_t *)(ws + o_gc);
  int64_t *d_st = (int64_t *)(ws + o_st);
  igp_error *d_err = (igp_error *)(ws + o_err);
  if (m > 0) {
    CK(cudaMemcpyAsync(d_wl, wl, Sm * IGP_WL_NF * 8, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(d_rank, name_rank, rank_n * 4, cudaMemcpyHostToDevice, st));
  }
  int rc = igp_plan_batch_device(d_wl, n_scen, m, hw_h, b_max, d_rank, rank_stride, d_i32,
                                 d_i32 + Sm, d_i32 + 2 * Sm, d_i32 + 3 * Sm, d_i32 + 4 * Sm, d_pred,
                                 d_gc, stats ? d_st : nullptr, d_err, workspace, L.total, flags,
                                 stream);
  if (rc) return rc;
  if (m > 0) {
    if (gpu_of) CK(cudaMemcpyAsync(gpu_of, d_i32, Sm * 4, cudaMemcpyDeviceToHost, st));
    if (pos) CK(cudaMemcpyAsync(pos, d_i32 + Sm, Sm * 4, cudaMemcpyDeviceToHost, st));
    if (units) CK(cudaMemcpyAsync(units, d_i32 + 2 * Sm, Sm * 4, cudaMemcpyDeviceToHost, st));
    if (batch) CK(cudaMemcpyAsync(batch, d_i32 + 3 * Sm, Sm * 4, cudaMemcpyDeviceToHost, st));
    if (lb) CK(cudaMemcpyAsync(lb, d_i32 + 4 * Sm, Sm * 4, cudaMemcpyDeviceToHost, st));
    if (pred) CK(cudaMemcpyAsync(pred, d_pred, Sm * 80, cudaMemcpyDeviceToHost, st));
  }
  CK(cudaMemcpyAsync(gpu_count, d_gc, (size_t)n_scen * 4, cudaMemcpyDeviceToHost, st));
  if (stats) CK(cudaMemcpyAsync(stats, d_st, (size_t)n_scen * 32, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(err, d_err, (size_t)n_scen * sizeof(igp_error), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  for (int s = 0; s < n_scen; ++s)
    if (err[s].code) return err[s].code;
  return IGP_E_OK;
}

static int *scratch_int(cudaStream_t st, int *&p) {
  if (cudaMallocAsync((void **)&p, sizeof(int), st) != cudaSuccess) return nullptr;
  return p;
}

int igp_eval_states_device(const double *wl, int n_rows, const int32_t *batch, const double *r,
                           const int64_t *ptr, int n_states, const double *hw_h, int check_capacity,
                           double *rows, igp_error *err, void *stream) {
  if (n_states < 0 || n_rows < 0 || !hw_h) return IGP_E_ARG;
  if (n_states == 0) return IGP_E_OK;
  cudaStream_t st = (cudaStream_t)stream;
  Hw hw = make_hw(hw_h, 0);
  int *fe = nullptr;
  if (!scratch_int(st, fe)) return cuda_fail(cudaGetLastError());
  k_fill_int<<<1, 1, 0, st>>>(fe, 1, INT_MAX);
  k_eval_states<<<nblk(n_states, 128), 128, 0, st>>>(wl, n_rows, batch, r, ptr, n_states, hw,
                                                     check_capacity, rows, err, fe);
  CK(cudaFreeAsync(fe, st));
  CK(cudaGetLastError());
  return IGP_E_OK;
}

int igp_alloc_units_device(const double *wl, int n_rows, const int32_t *batch, const double *r,
                           const int64_t *ptr, int n_states, const double *hw_h, int32_t *units,
                           igp_error *err, void *stream) {
  if (n_states < 0 || n_rows < 0 || !hw_h) return IGP_E_ARG;
  if (n_states == 0) return IGP_E_OK;
  cudaStream_t st = (cudaStream_t)stream;
  Hw hw = make_hw(hw_h, 0);
  int *fe = nullptr;
  if (!scratch_int(st, fe)) return cuda_fail(cudaGetLastError());
  k_fill_int<<<1, 1, 0, st>>>(fe, 1, INT_MAX);
  k_alloc_units<<<nblk(n_states, 128), 128, 0, st>>>(wl, n_rows, batch, r, ptr, n_states, hw, units,
                                                     err, fe);
  CK(cudaFreeAsync(fe, st));
  CK(cudaGetLastError());
  return IGP_E_OK;
}

int igp_prologue_device(const double *wl, int m, const double *hw_h, int b_max,
                        const int32_t *batch_in, int32_t *batch, int32_t *lb, int32_t *code,
                        igp_error *err, void *stream) {
  if (m < 0 || !hw_h) return IGP_E_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  Hw hw = make_hw(hw_h, b_max);
  int *fe = nullptr;
  if (!scratch_int(st, fe)) return cuda_fail(cudaGetLastError());
  k_fill_int<<<1, 1, 0, st>>>(fe, 1, INT_MAX);
  if (m > 0) k_prologue<<<nblk(m, 256), 256, 0, st>>>(wl, m, hw, batch_in, batch, lb, code, fe);
  k_prologue_err<<<1, 1, 0, st>>>(wl, m, hw, batch_in, fe, err);
  CK(cudaFreeAsync(fe, st));
  CK(cudaGetLastError());
  return IGP_E_OK;
}

}  // extern "C"
