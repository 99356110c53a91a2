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

#include <cub/device/device_segmented_sort.cuh>
#include <nvtx3/nvToolsExt.h>

#include <climits>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <vector>

#include "exact_fp64.cuh"

namespace igp {

#ifndef IGP_MINB_WARP
#define IGP_MINB_WARP 4
#endif
#ifndef IGP_MINB_CTA
#define IGP_MINB_CTA 1
#endif

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
  hw.margin_ok = (hw.fmax > 0.0 && hw.fmin > 0.0 && std::isfinite(hw.fmax) &&
                  std::isfinite(hw.fmin) && std::isfinite(hw.pidle) && std::isfinite(hw.pmax) &&
                  std::isfinite(hw.af)) ? 1 : 0;
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

}  // namespace igp

#include "place.cuh"
#include "window.cuh"
#include "fast.cuh"
#include "smem_plan.cuh"
#include "grid.cuh"
#ifndef IGP_GS_MAXN
#define IGP_GS_MAXN 6
#endif
#include "exhaustive.cuh"
#include "simulate.cuh"
#include "components.cuh"

namespace igp {

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

// NVTX range over one C-ABI call (header-only nvtx3: a no-op unless a tool
// such as Nsight Systems / ncu --nvtx injects itself)
struct NvtxRange {
  explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};
#define IGP_NVTX() NvtxRange nvtx_range_(__func__)

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

template <int GW>
static size_t place_smem() {
  return (size_t)(GW == 1 ? 128 : GW * 32) * lane_smem_bytes();
}

// Per-device launch facts of one kernel instantiation: the opt-in dynamic
// shared memory attribute is set, and the occupancy queried, once per device
// ordinal (the attribute belongs to the device's context), under a lock.
struct DevOcc {
  int per_sm = -1, sms = 0;
};
template <typename Kern>
static DevOcc dev_occupancy(Kern kern, int threads, size_t smem) {
  static std::mutex mu;
  static std::map<std::pair<const void *, int>, DevOcc> cache;  // (kernel, device)
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> g(mu);
  DevOcc &o = cache[{(const void *)kern, dev}];
  if (o.per_sm < 0) {
    cudaDeviceGetAttribute(&o.sms, cudaDevAttrMultiProcessorCount, dev);
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o.per_sm, kern, threads, smem) !=
            cudaSuccess ||
        o.per_sm < 1)
      o.per_sm = 1;
  }
  return o;
}

// one-warp scenarios of at least this many workloads use the 5-CTA build
#ifndef IGP_MINB5_FROM_M
#define IGP_MINB5_FROM_M 4000
#endif
#ifndef IGP_MINB_BIG
#define IGP_MINB_BIG 5  // resident CTAs per SM of the large-plan one-warp build
#endif

template <int MAXN, int GW, bool HWS = false, int MINB = 0, bool LEAN = false>
static unsigned place_grid(int S) {
  // persistent launch: at most as many groups as can be co-resident
  const DevOcc o = dev_occupancy(k_place<MAXN, GW, false, HWS, MINB, LEAN>, GW == 1 ? 128 : GW * 32,
                                 place_smem<GW>());
  const int gpb = (GW == 1) ? 4 : 1;
  const long long want = (S + gpb - 1) / gpb;
  const long long cap = (long long)o.per_sm * o.sms;
  return (unsigned)(want < cap ? want : cap);
}

static size_t fast_smem() { return 128 * fast_lane_smem(); }

template <int MAXN>
static unsigned fast_grid(int S) {
  const DevOcc o = dev_occupancy(k_place_fast<MAXN>, 128, fast_smem());
  const long long want = (S + 3) / 4;
  const long long cap = (long long)o.per_sm * o.sms;
  return (unsigned)(want < cap ? want : cap);
}

template <int MAXN>
static void launch_place(const PlanParams &P, cudaStream_t st) {
  if (P.crec) {  // the certified-margin fast kernel plans what it can; k_place the rest
    cudaMemsetAsync(P.sched, 0, sizeof(int32_t), st);
    k_place_fast<MAXN><<<fast_grid<MAXN>(P.S), 128, fast_smem(), st>>>(P);
  }
  cudaMemsetAsync(P.sched, 0, sizeof(int32_t), st);
  if (P.hand && !P.crec && !P.hw_s && !(P.flags & (IGP_F_CTA | IGP_F_GW2 | IGP_F_GW4 | IGP_F_SMEM))) {
    // the lean pass (no exact-sequence code), then the full pass below plans
    // only the scenarios it declined
    if (P.m >= IGP_MINB5_FROM_M && MAXN == 48)
      k_place<MAXN, 1, false, false, IGP_MINB_BIG, true>
          <<<place_grid<MAXN, 1, false, IGP_MINB_BIG, true>(P.S), 128, place_smem<1>(), st>>>(P);
    else
      k_place<MAXN, 1, false, false, 0, true>
          <<<place_grid<MAXN, 1, false, 0, true>(P.S), 128, place_smem<1>(), st>>>(P);
    cudaMemsetAsync(P.sched, 0, sizeof(int32_t), st);
  }
  if (P.hw_s) {  // one profile per scenario: one CTA or one warp per scenario
    if (P.flags & IGP_F_CTA)
      k_place<MAXN, 8, false, true>
          <<<place_grid<MAXN, 8, true>(P.S), 256, place_smem<8>(), st>>>(P);
    else
      k_place<MAXN, 1, false, true>
          <<<place_grid<MAXN, 1, true>(P.S), 128, place_smem<1>(), st>>>(P);
    return;
  }
  if (P.flags & IGP_F_CTA) {
    k_place<MAXN, 8><<<place_grid<MAXN, 8>(P.S), 256, place_smem<8>(), st>>>(P);
  } else if (P.flags & IGP_F_GW4) {
    k_place<MAXN, 4><<<place_grid<MAXN, 4>(P.S), 128, place_smem<4>(), st>>>(P);
  } else if (P.flags & IGP_F_GW2) {
    k_place<MAXN, 2><<<place_grid<MAXN, 2>(P.S), 64, place_smem<2>(), st>>>(P);
  } else if (P.m >= IGP_MINB5_FROM_M && MAXN == 48) {
    k_place<MAXN, 1, false, false, IGP_MINB_BIG>
        <<<place_grid<MAXN, 1, false, IGP_MINB_BIG>(P.S), 128, place_smem<1>(), st>>>(P);
  } else {
    k_place<MAXN, 1><<<place_grid<MAXN, 1>(P.S), 128, place_smem<1>(), st>>>(P);
  }
}

// One scenario on the whole GPU: the cooperative step kernel, then the
// per-CTA kernel, which writes the plan (or, when the cooperative kernel
// declined because the exact sequence is needed, plans it itself).
#ifndef COOP_M_PER_CTA
#define COOP_M_PER_CTA 64
#endif

template <int MAXN>
static int launch_place_coop(PlanParams P, cudaStream_t st) {
  const DevOcc o = dev_occupancy(k_place<MAXN, 1, true>, 128, place_smem<1>());
  const int per_sm = o.per_sm, sms = o.sms;
  int grid = per_sm * sms;
  if (grid * 128 > COOP_MAX_LANES) grid = COOP_MAX_LANES / 128;
  // no more CTAs than the step's candidates can use (a step of m workloads has
  // about m / 40 candidates at 2.5% units); bits 16..27 of flags override
  const int want_ctas = (P.flags >> 16) & 0xfff;
  const int by_m = (P.m + COOP_M_PER_CTA - 1) / COOP_M_PER_CTA;
  const int lim = want_ctas ? want_ctas : (by_m > 1 ? by_m : 1);
  if (grid > lim) grid = lim;
  CK(cudaMemsetAsync(P.coop, 0, sizeof(CoopState), st));
  // plan mode: the slack order starts empty before any warp reads it (the
  // kernel has no grid-wide barrier before its first step); stream mode: it
  // persists, and so does the pool top
  if (!P.stream) CK(cudaMemsetAsync(P.sE, 0, sizeof(int32_t) * (P.hw.cap + 2), st));
  else CK(cudaMemcpyAsync(&P.coop->pool_top, P.sstate + 1, sizeof(int32_t),
                          cudaMemcpyDeviceToDevice, st));
  CK(cudaMemsetAsync(P.coop->best, 0xff, sizeof(P.coop->best), st));
  void *args[] = {&P};
  CK(cudaLaunchCooperativeKernel((const void *)k_place<MAXN, 1, true>, dim3(grid), dim3(128), args,
                                 place_smem<1>(), st));
  launch_place<MAXN>(P, st);
  return IGP_E_OK;
}

// The largest dynamic shared memory one CTA of k_plan_smem may use (device limit
// minus its static state), queried once per device.
static size_t smem_plan_limit() {
  static std::mutex mu;
  static std::map<int, size_t> cache;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> g(mu);
  auto it = cache.find(dev);
  if (it != cache.end()) return it->second;
  int optin = 0;
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  const size_t lim = optin > 4096 ? (size_t)optin - 4096 : 0;
  cache[dev] = lim;
  return lim;
}

// One plan per CTA with the search state in shared memory (smem_plan.cuh),
// then the per-CTA kernel, which writes the plan (or plans a declined scenario).
template <int MAXN>
static void launch_smem(PlanParams P, size_t bytes, cudaStream_t st) {
  if (P.hw_s) {
    cudaFuncSetAttribute(k_plan_smem<MAXN, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)bytes);
    k_plan_smem<MAXN, true><<<P.S, SMEM_WARPS * 32, bytes, st>>>(P);
  } else {
    cudaFuncSetAttribute(k_plan_smem<MAXN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    k_plan_smem<MAXN><<<P.S, SMEM_WARPS * 32, bytes, st>>>(P);
  }
  launch_place<MAXN>(P, st);
}

// One scenario in windows of speculative steps (window.cuh), then the per-CTA
// kernel, which writes the plan (or plans it itself when the windowed kernel
// declined because the exact sequence is needed).
template <int MAXN>
static int launch_place_win(PlanParams P, cudaStream_t st) {
  CK(cudaMemsetAsync(P.coop, 0, sizeof(CoopState), st));
  k_place_win<MAXN><<<1, WIN_THREADS, 0, st>>>(P);
  launch_place<MAXN>(P, st);
  return IGP_E_OK;
}

extern "C" {

int igp_abi_version(void) { return IGP_ABI_VERSION; }
int igp_max_cap(void) { return 256; }
const char *igp_last_error_string(void) { return g_last_err; }

// The largest max_units over the call's profiles (one, or n_scen with IGP_F_HWS).
static int cap_of(const double *hw, int n_scen, int b_max, int flags) {
  int cap = make_hw(hw, b_max).cap;
  if (flags & IGP_F_HWS)
    for (int s = 1; s < n_scen; ++s) {
      const int c = make_hw(hw + (size_t)s * IGP_HW_NF, b_max).cap;
      if (c > cap) cap = c;
    }
  return cap;
}

int igp_plan_batch_slots(int m, const double *hw, int b_max, int flags) {
  if (!hw || m < 0) return -IGP_E_ARG;
  const int cap = make_hw(hw, b_max).cap;
  if (cap < 1 || cap > igp_max_cap()) return -IGP_E_ARG;
  auto slots = [&](auto kern, int threads, size_t smem, int gpb) {
    const DevOcc o = dev_occupancy(kern, threads, smem);
    return o.per_sm * o.sms * gpb;
  };
  const bool cta = flags & IGP_F_CTA;
  if (fast_path(flags))
    return cap <= 48    ? slots(k_place_fast<48>, 128, fast_smem(), 4)
           : cap <= 128 ? slots(k_place_fast<128>, 128, fast_smem(), 4)
                        : slots(k_place_fast<256>, 128, fast_smem(), 4);
  if (cap <= 48)
    return cta ? slots(k_place<48, 8>, 256, place_smem<8>(), 1)
           : m >= IGP_MINB5_FROM_M ? slots(k_place<48, 1, false, false, IGP_MINB_BIG>, 128, place_smem<1>(), 4)
                                   : slots(k_place<48, 1>, 128, place_smem<1>(), 4);
  if (cap <= 128)
    return cta ? slots(k_place<128, 8>, 256, place_smem<8>(), 1)
               : slots(k_place<128, 1>, 128, place_smem<1>(), 4);
  return cta ? slots(k_place<256, 8>, 256, place_smem<8>(), 1)
             : slots(k_place<256, 1>, 128, place_smem<1>(), 4);
}

size_t igp_plan_workspace_bytes(int n_scen, int m, const double *hw, int b_max, int flags) {
  return ws_layout(n_scen, m, cap_of(hw, n_scen, b_max, flags), flags).total;
}

static int plan_device_impl(const double *wl, int n_scen, int m, const double *hw_h, int b_max,
                            const int32_t *name_rank, int rank_stride, int32_t *gpu_of,
                            int32_t *pos, int32_t *units, int32_t *batch, int32_t *lb,
                            double *pred, int32_t *gpu_count, int64_t *stats, igp_error *err,
                            void *workspace, size_t workspace_bytes, int flags, void *stream,
                            int stages) {
  IGP_NVTX();
  if (n_scen < 0 || m < 0 || !hw_h) return IGP_E_ARG;
  if (n_scen == 0) return IGP_E_OK;
  if ((flags & IGP_F_HWS) && (flags & IGP_F_COOP)) return IGP_E_ARG;
  Hw hw = make_hw(hw_h, b_max);
  std::vector<Hw> hws;
  if (flags & IGP_F_HWS) {
    hws.resize(n_scen);
    for (int s = 0; s < n_scen; ++s) {
      hws[s] = make_hw(hw_h + (size_t)s * IGP_HW_NF, b_max);
      if (hws[s].cap < 1) return IGP_E_ARG;
      if (hws[s].cap > hw.cap) hw.cap = hws[s].cap;  // layout / dispatch size
    }
  }
  if (hw.cap < 1) return IGP_E_ARG;
  if (hw.cap > igp_max_cap()) return IGP_E_CAPACITY;
  if (m >= (1 << 23)) return IGP_E_CAPACITY;  // candidate keys pack j into 23 bits
  WsLayout L = ws_layout(n_scen, m, hw.cap, flags);
  if (workspace_bytes < L.total || !workspace) return IGP_E_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  char *ws = (char *)workspace;
  PlanParams P;
  P.hw = hw;
  P.hw_s = nullptr;
  P.cap_ld = hw.cap;
  if (flags & IGP_F_HWS) {
    // pageable source: the copy is staged before cudaMemcpyAsync returns
    CK(cudaMemcpyAsync(ws + L.hws, hws.data(), hws.size() * sizeof(Hw), cudaMemcpyHostToDevice,
                       st));
    P.hw_s = (const Hw *)(ws + L.hws);
  }
  P.S = n_scen;
  P.m = m;
  P.flags = flags;
  P.k0 = 0;
  P.k1 = m;
  P.stream = 0;
  P.code = nullptr;
  P.sstate = nullptr;
  if ((flags & IGP_F_WIN) && (n_scen != 1 || hw.cap > 128 || (flags & (IGP_F_COOP | IGP_F_HWS))))
    flags &= ~IGP_F_WIN;  // the windowed kernel plans one scenario of max_units <= 128
  P.coop = (flags & (IGP_F_COOP | IGP_F_WIN)) && n_scen == 1 ? (CoopState *)(ws + L.coop)
                                                            : nullptr;
  P.win_tid = (int32_t *)(ws + L.win_tid);
  P.sdesc = (unsigned long long *)(ws + L.sdesc);
  P.sj = (int32_t *)(ws + L.sj);
  P.spos = (int32_t *)(ws + L.spos);
  P.sE = (int32_t *)(ws + L.sE);
  P.nxt = (double *)(ws + L.nxt);
  // the layout (sized with the caller's flags) holds the compact tiles
  const bool fast = L.cnext > L.crec && fast_path(flags) && !P.coop;
  P.crec = fast ? (CRec *)(ws + L.crec) : nullptr;
  P.cnext = fast ? (CNext *)(ws + L.cnext) : nullptr;
  // IGP_F_SMEM: the shared-memory plan kernel when the scenario's state fits
  const size_t smem_need =
      smem_layout(m, L.pool_recs, hw.cap).total;
  const bool smem = !fast && !P.coop && (flags & IGP_F_SMEM) && (flags & IGP_F_CTA) &&
                    !(flags & IGP_F_STATS) && m > 0 &&
                    smem_need <= smem_plan_limit();
  const bool lean = !fast && !smem && !P.coop && lean_path(flags);
  P.hand = (fast || smem || lean) ? (Hand *)(ws + L.hand) : nullptr;
  // the fast kernel's decision margin; IGP_FAST_DELTA raises it (tests force the
  // exact fallback with it); it is never lowered below FAST_DELTA
  P.fast_delta = FAST_DELTA;
  if (const char *e = getenv("IGP_FAST_DELTA")) {
    const double d = atof(e);
    if (d > FAST_DELTA) P.fast_delta = d;
  }
  P.wl = wl;
  P.rank = name_rank;
  P.rank_stride = rank_stride;
  P.lanes = L.lanes;
  P.pool_recs = L.pool_recs;
  P.by_rank = (int32_t *)(ws + L.by_rank);
  P.order = (int32_t *)(ws + L.order);
  P.cold = (double *)(ws + L.cold);
  P.nw = (double *)(ws + L.nw);
  P.tbl = (double *)(ws + L.tbl);
  P.gstate = (unsigned long long *)(ws + L.gstate);
  P.gstride = L.gstride;
  P.gcap = (int32_t *)(ws + L.gcap);
  P.gfold = (double *)(ws + L.gfold);
  P.rec = (double *)(ws + L.rec);
  P.frec = (double *)(ws + L.frec);
  P.pfx = (double *)(ws + L.pfx);
  P.meta = (Meta *)(ws + L.meta);
  P.lane_units = (uint16_t *)(ws + L.lane_units);
  P.sflags = (int32_t *)(ws + L.sflags);
  P.perr = (int32_t *)(ws + L.perr);
  P.sched = (int32_t *)(ws + L.sched);
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
    CK(cudaMemsetAsync(P.sflags, 0, (size_t)n_scen * 4, st));
    // every byte of the error records (incl. padding) is defined for the caller
    CK(cudaMemsetAsync(err, 0, (size_t)n_scen * sizeof(igp_error), st));
    k_fill_int<<<nblk(n_scen, 256), 256, 0, st>>>(P.perr, n_scen, INT_MAX);
    if (m > 0) {
      const long long tot = (long long)n_scen * m;
      k_prologue_plan<<<nblk(tot, 256), 256, 0, st>>>(P);
      k_sort<<<nblk(n_scen, 4), 128, 0, st>>>(P);
      k_build<<<nblk(tot, 256), 256, 0, st>>>(P);
      k_table<<<nblk(tot * TB, 256), 256, 0, st>>>(P);
    }
  }
  if (stages & 2) {
    if (P.coop && (flags & IGP_F_WIN)) {
      const int rc = hw.cap <= 48 ? launch_place_win<48>(P, st) : launch_place_win<128>(P, st);
      if (rc) return rc;
    } else if (P.coop) {
      int rc;
      if (hw.cap <= 48) rc = launch_place_coop<48>(P, st);
      else if (hw.cap <= 128) rc = launch_place_coop<128>(P, st);
      else rc = launch_place_coop<256>(P, st);
      if (rc) return rc;
    } else if (P.hand && (flags & IGP_F_SMEM)) {  // the shared-memory plan kernel
      const size_t bytes = smem_layout(m, P.pool_recs, hw.cap).total;
      if (hw.cap <= 48) launch_smem<48>(P, bytes, st);
      else if (hw.cap <= 128) launch_smem<128>(P, bytes, st);
      else launch_smem<256>(P, bytes, st);
    } else if (hw.cap <= 48) {
      launch_place<48>(P, st);
    } else if (hw.cap <= 128) {
      launch_place<128>(P, st);
    } else {
      launch_place<256>(P, st);
    }
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

// igp_plan_batch_host pipelines the batch in up to HOST_CHUNKS scenario
// chunks, each on its own stream with its own slice of the workspace: chunk
// c's kernels overlap chunk c+1's H2D copy and chunk c-1's D2H copy, and the
// chunks' persistent place kernels share the SMs (each sized to half the resident
// warp slots, so together they fill the GPU).
static constexpr int HOST_CHUNKS = 2;  // measured: 2 chunks 1340 ms, 1: 1364, 4: 2107 (uneven
                                       // co-residency of four persistent grids)
static constexpr int HOST_CHUNK_MIN = 128;  // scenarios per chunk before splitting

static int host_chunks(int n_scen, int flags) {
  if (flags & IGP_F_COOP) return 1;
  int nc = n_scen / HOST_CHUNK_MIN;
  if (const char *e = getenv("IGP_HOST_CHUNKS")) nc = atoi(e);  // A/B experiments
  return nc < 1 ? 1 : nc > HOST_CHUNKS ? HOST_CHUNKS : nc;
}

struct HostChunkLayout {
  size_t plan, o_wl, o_rank, o_i32, o_pred, o_gc, o_st, o_err, per_chunk;
};

static HostChunkLayout host_chunk_layout(int sc, int m, int cap, int flags, int rank_stride,
                                         int want_pred) {
  HostChunkLayout H;
  const size_t Sm = (size_t)sc * (m > 0 ? m : 1);
  const size_t rank_n = rank_stride ? Sm : (size_t)(m > 0 ? m : 1);
  size_t off = ws_layout(sc, m, cap, flags).total;
  H.plan = off;
  H.o_wl = off; off = align_up(off + Sm * IGP_WL_NF * 8);
  H.o_rank = off; off = align_up(off + rank_n * 4);
  H.o_i32 = off; off = align_up(off + Sm * 4 * 5);
  H.o_pred = off; off = align_up(off + (want_pred ? Sm * 80 : 0));
  H.o_gc = off; off = align_up(off + (size_t)sc * 4);
  H.o_st = off; off = align_up(off + (size_t)sc * 8 * IGP_NSTAT);
  H.o_err = off; off = align_up(off + (size_t)sc * sizeof(igp_error));
  H.per_chunk = off;
  return H;
}

size_t igp_plan_host_workspace_bytes(int n_scen, int m, const double *hw, int b_max, int flags,
                                     int rank_stride, int want_pred) {
  if (n_scen <= 0 || !hw) return 256;
  const int nc = host_chunks(n_scen, flags);
  const int sc = (n_scen + nc - 1) / nc;
  return (size_t)nc * host_chunk_layout(sc, m, cap_of(hw, n_scen, b_max, flags), flags,
                                        rank_stride, want_pred).per_chunk;
}

// per-thread, per-device chunk streams and events (created on first use)
struct HostStreams {
  int dev = -1;
  cudaStream_t s[HOST_CHUNKS];
  cudaEvent_t start, done[HOST_CHUNKS];
};

static int host_streams(HostStreams *&out) {
  static thread_local HostStreams cache[8];
  int dev = 0;
  CK(cudaGetDevice(&dev));
  HostStreams &h = cache[dev & 7];
  if (h.dev != dev) {
    for (int c = 0; c < HOST_CHUNKS; ++c) {
      CK(cudaStreamCreateWithFlags(&h.s[c], cudaStreamNonBlocking));
      CK(cudaEventCreateWithFlags(&h.done[c], cudaEventDisableTiming));
    }
    CK(cudaEventCreateWithFlags(&h.start, cudaEventDisableTiming));
    h.dev = dev;
  }
  out = &h;
  return IGP_E_OK;
}

int igp_plan_batch_host(const double *wl, int n_scen, int m, const double *hw_h, int b_max,
                        const int32_t *name_rank, int rank_stride, int32_t *gpu_of, int32_t *pos,
                        int32_t *units, int32_t *batch, int32_t *lb, double *pred,
                        int32_t *gpu_count, int64_t *stats, igp_error *err, void *workspace,
                        size_t workspace_bytes, int flags, void *stream) {
  IGP_NVTX();
  if (n_scen < 0 || m < 0 || !hw_h) return IGP_E_ARG;
  if (n_scen == 0) return IGP_E_OK;
  Hw hw = make_hw(hw_h, b_max);
  hw.cap = cap_of(hw_h, n_scen, b_max, flags);
  if (hw.cap < 1) return IGP_E_ARG;
  if (hw.cap > igp_max_cap()) return IGP_E_CAPACITY;
  const int want_pred = pred != nullptr && !(flags & IGP_F_NO_PRED);
  const int nc = host_chunks(n_scen, flags);
  const int sc_max = (n_scen + nc - 1) / nc;
  const HostChunkLayout H = host_chunk_layout(sc_max, m, hw.cap, flags, rank_stride, want_pred);
  cudaStream_t st = (cudaStream_t)stream;
  void *owned = nullptr;  // workspace == NULL, bytes == 0: the library allocates it on the stream
  if (!workspace && workspace_bytes == 0) {
    CK(cudaMallocAsync(&owned, (size_t)nc * H.per_chunk, st));
    workspace = owned;
    workspace_bytes = (size_t)nc * H.per_chunk;
  }
  if (!workspace || workspace_bytes < (size_t)nc * H.per_chunk) return IGP_E_ARG;
  HostStreams *hs = nullptr;
  if (nc > 1) {
    int rc = host_streams(hs);
    if (rc) return rc;
    CK(cudaEventRecord(hs->start, st));  // the chunks follow the caller's prior work
  }
  const size_t mm = (size_t)(m > 0 ? m : 1);
  // two passes: every chunk's H2D copies and kernels are queued before the
  // first D2H copy, so a D2H into pageable memory (which returns only when it
  // is done) cannot hold back the later chunks' work
  for (int pass = 0; pass < 2; ++pass) {
    for (int c = 0; c < nc; ++c) {
      const int s0 = c * sc_max;
      const int sc = (n_scen - s0) < sc_max ? (n_scen - s0) : sc_max;
      if (sc <= 0) break;
      cudaStream_t cs = nc > 1 ? hs->s[c] : st;
      char *ws = (char *)workspace + (size_t)c * H.per_chunk;
      const size_t Sm = (size_t)sc * mm, Sm0 = (size_t)s0 * mm;
      const size_t rank_n = rank_stride ? Sm : mm;
      double *d_wl = (double *)(ws + H.o_wl);
      int32_t *d_rank = (int32_t *)(ws + H.o_rank);
      int32_t *d_i32 = (int32_t *)(ws + H.o_i32);
      double *d_pred = want_pred ? (double *)(ws + H.o_pred) : nullptr;
      int32_t *d_gc = (int32_t *)(ws + H.o_gc);
      int64_t *d_st = (int64_t *)(ws + H.o_st);
      igp_error *d_err = (igp_error *)(ws + H.o_err);
      if (pass == 0) {
        if (nc > 1) CK(cudaStreamWaitEvent(cs, hs->start, 0));
        if (m > 0) {
          CK(cudaMemcpyAsync(d_wl, wl + Sm0 * IGP_WL_NF, Sm * IGP_WL_NF * 8,
                             cudaMemcpyHostToDevice, cs));
          CK(cudaMemcpyAsync(d_rank, name_rank + (rank_stride ? Sm0 : 0), rank_n * 4,
                             cudaMemcpyHostToDevice, cs));
        }
        const double *hw_c = (flags & IGP_F_HWS) ? hw_h + (size_t)s0 * IGP_HW_NF : hw_h;
        int rc = igp_plan_batch_device(d_wl, sc, m, hw_c, b_max, d_rank, rank_stride, d_i32,
                                       d_i32 + Sm, d_i32 + 2 * Sm, d_i32 + 3 * Sm,
                                       d_i32 + 4 * Sm, d_pred, d_gc, stats ? d_st : nullptr,
                                       d_err, ws, H.plan, flags, cs);
        if (rc) return rc;
        continue;
      }
      if (m > 0) {
        if (gpu_of) CK(cudaMemcpyAsync(gpu_of + Sm0, d_i32, Sm * 4, cudaMemcpyDeviceToHost, cs));
        if (pos) CK(cudaMemcpyAsync(pos + Sm0, d_i32 + Sm, Sm * 4, cudaMemcpyDeviceToHost, cs));
        if (units)
          CK(cudaMemcpyAsync(units + Sm0, d_i32 + 2 * Sm, Sm * 4, cudaMemcpyDeviceToHost, cs));
        if (batch)
          CK(cudaMemcpyAsync(batch + Sm0, d_i32 + 3 * Sm, Sm * 4, cudaMemcpyDeviceToHost, cs));
        if (lb)
          CK(cudaMemcpyAsync(lb + Sm0, d_i32 + 4 * Sm, Sm * 4, cudaMemcpyDeviceToHost, cs));
        if (want_pred)
          CK(cudaMemcpyAsync(pred + Sm0 * 10, d_pred, Sm * 80, cudaMemcpyDeviceToHost, cs));
      }
      CK(cudaMemcpyAsync(gpu_count + s0, d_gc, (size_t)sc * 4, cudaMemcpyDeviceToHost, cs));
      if (stats)
        CK(cudaMemcpyAsync(stats + (size_t)s0 * IGP_NSTAT, d_st, (size_t)sc * 8 * IGP_NSTAT,
                           cudaMemcpyDeviceToHost, cs));
      CK(cudaMemcpyAsync(err + s0, d_err, (size_t)sc * sizeof(igp_error),
                         cudaMemcpyDeviceToHost, cs));
      if (nc > 1) {
        CK(cudaEventRecord(hs->done[c], cs));
        CK(cudaStreamWaitEvent(st, hs->done[c], 0));
      }
    }
  }
  if (owned) CK(cudaFreeAsync(owned, st));
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
  IGP_NVTX();
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
  IGP_NVTX();
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
  IGP_NVTX();
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

// ---------------------------------------------------------------------------
// Online stream (BASELINE config 5).  The workspace holds the plan workspace
// for (n_streams, capacity) followed by the arrival tables and the
// persistent per-stream state.
// ---------------------------------------------------------------------------
struct StreamLayout {
  WsLayout L;
  size_t wl, batch, lb, code, gpu_of, pos, units, pred, sstate, gc, err, total;
};

static StreamLayout stream_layout(int S, int C, int cap, int flags) {
  StreamLayout X;
  // a single stream may run any push on the whole GPU (IGP_F_COOP per push):
  // its layout always reserves the cooperative lanes
  X.L = ws_layout(S, C, cap, S == 1 ? (flags | IGP_F_COOP) : (flags & ~IGP_F_COOP));
  const size_t SC = (size_t)S * (C > 0 ? C : 1);
  size_t off = X.L.total;
  X.wl = off; off = align_up(off + SC * IGP_WL_NF * 8);
  X.batch = off; off = align_up(off + SC * 4);
  X.lb = off; off = align_up(off + SC * 4);
  X.code = off; off = align_up(off + SC * 4);
  X.gpu_of = off; off = align_up(off + SC * 4);
  X.pos = off; off = align_up(off + SC * 4);
  X.units = off; off = align_up(off + SC * 4);
  X.pred = off; off = align_up(off + SC * 80);
  X.sstate = off; off = align_up(off + (size_t)S * 16);
  X.gc = off; off = align_up(off + (size_t)S * 4);
  X.err = off; off = align_up(off + (size_t)S * sizeof(igp_error));
  X.total = off;
  return X;
}

static void stream_params(PlanParams &P, const StreamLayout &X, char *ws, const Hw &hw, int S,
                          int C, int flags) {
  const WsLayout &L = X.L;
  P.hw = hw;
  P.hw_s = nullptr;
  P.cap_ld = hw.cap;
  P.S = S;
  P.m = C;
  P.flags = flags;
  P.stream = 1;
  P.wl = (const double *)(ws + X.wl);
  P.rank = nullptr;
  P.rank_stride = 0;
  P.lanes = L.lanes;
  P.gstride = L.gstride;
  P.pool_recs = L.pool_recs;
  P.by_rank = (int32_t *)(ws + L.by_rank);
  P.order = (int32_t *)(ws + L.order);
  P.cold = (double *)(ws + L.cold);
  P.nw = (double *)(ws + L.nw);
  P.tbl = (double *)(ws + L.tbl);
  P.gstate = (unsigned long long *)(ws + L.gstate);
  P.gcap = (int32_t *)(ws + L.gcap);
  P.gfold = (double *)(ws + L.gfold);
  P.rec = (double *)(ws + L.rec);
  P.frec = (double *)(ws + L.frec);
  P.pfx = (double *)(ws + L.pfx);
  P.meta = (Meta *)(ws + L.meta);
  P.lane_units = (uint16_t *)(ws + L.lane_units);
  P.sflags = (int32_t *)(ws + L.sflags);
  P.perr = (int32_t *)(ws + L.perr);
  P.sched = (int32_t *)(ws + L.sched);
  P.batch = (int32_t *)(ws + X.batch);
  P.lb = (int32_t *)(ws + X.lb);
  P.code = (int32_t *)(ws + X.code);
  P.gpu_of = (int32_t *)(ws + X.gpu_of);
  P.pos = (int32_t *)(ws + X.pos);
  P.units = (int32_t *)(ws + X.units);
  P.pred = nullptr;
  P.sstate = (int32_t *)(ws + X.sstate);
  P.coop = nullptr;
  P.win_tid = (int32_t *)(ws + L.win_tid);
  P.sdesc = (unsigned long long *)(ws + L.sdesc);
  P.sj = (int32_t *)(ws + L.sj);
  P.spos = (int32_t *)(ws + L.spos);
  P.sE = (int32_t *)(ws + L.sE);
  P.nxt = (double *)(ws + L.nxt);
  P.crec = nullptr;
  P.cnext = nullptr;
  P.hand = nullptr;
  P.fast_delta = FAST_DELTA;
  P.gpu_count = (int32_t *)(ws + X.gc);
  P.stats = nullptr;
  P.err = (igp_error *)(ws + X.err);
}

size_t igp_stream_workspace_bytes(int n_streams, int capacity, const double *hw, int b_max,
                                  int flags) {
  Hw h = make_hw(hw, b_max);
  return stream_layout(n_streams, capacity, h.cap, flags).total;
}

int igp_stream_reset_device(int n_streams, int capacity, const double *hw_h, int b_max,
                            void *workspace, size_t workspace_bytes, int flags, void *stream) {
  IGP_NVTX();
  if (n_streams < 1 || capacity < 1 || !hw_h || !workspace || (flags & IGP_F_HWS)) return IGP_E_ARG;
  Hw hw = make_hw(hw_h, b_max);
  if (hw.cap < 1) return IGP_E_ARG;
  if (hw.cap > igp_max_cap()) return IGP_E_CAPACITY;
  StreamLayout X = stream_layout(n_streams, capacity, hw.cap, flags);
  if (workspace_bytes < X.total) return IGP_E_ARG;
  CK(cudaMemsetAsync((char *)workspace + X.sstate, 0, (size_t)n_streams * 16,
                     (cudaStream_t)stream));
  CK(cudaMemsetAsync((char *)workspace + X.err, 0, (size_t)n_streams * sizeof(igp_error),
                     (cudaStream_t)stream));
  // empty slack orders: a first push may run on the cooperative kernel, which
  // does not initialise them
  CK(cudaMemsetAsync((char *)workspace + X.L.sE, 0,
                     (size_t)n_streams * (hw.cap + 2) * sizeof(int32_t), (cudaStream_t)stream));
  return IGP_E_OK;
}

int igp_stream_push_device(const double *wl_new, int n_streams, int k0, int n, int capacity,
                           const double *hw_h, int b_max, int32_t *gpu_of, int32_t *pos,
                           int32_t *code, int64_t *stats, igp_error *err, void *workspace,
                           size_t workspace_bytes, int flags, void *stream) {
  IGP_NVTX();
  if (n_streams < 1 || capacity < 1 || k0 < 0 || n < 0 || k0 + n > capacity || !hw_h ||
      !workspace)
    return IGP_E_ARG;
  if (capacity >= (1 << 23)) return IGP_E_CAPACITY;  // candidate keys pack j into 23 bits
  if (n == 0) return IGP_E_OK;
  Hw hw = make_hw(hw_h, b_max);
  if (hw.cap < 1) return IGP_E_ARG;
  if (hw.cap > igp_max_cap()) return IGP_E_CAPACITY;
  StreamLayout X = stream_layout(n_streams, capacity, hw.cap, flags);
  if (workspace_bytes < X.total) return IGP_E_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  char *ws = (char *)workspace;
  const size_t S = (size_t)n_streams;
  // append the arrivals: [S][16][n] -> columns [k0, k0 + n) of [S][16][capacity]
  CK(cudaMemcpy2DAsync(ws + X.wl + (size_t)k0 * 8, (size_t)capacity * 8, wl_new, (size_t)n * 8,
                       (size_t)n * 8, S * IGP_WL_NF, cudaMemcpyDeviceToDevice, st));
  PlanParams P;
  stream_params(P, X, ws, hw, n_streams, capacity, flags);
  P.k0 = k0;
  P.k1 = k0 + n;
  P.stats = stats;
  const long long tot = (long long)S * n;
  k_prologue_plan<<<nblk(tot, 256), 256, 0, st>>>(P);
  k_build<<<nblk(tot, 256), 256, 0, st>>>(P);
  k_table<<<nblk(tot * TB, 256), 256, 0, st>>>(P);
  if ((flags & IGP_F_COOP) && n_streams == 1) {
    // one stream on the whole GPU: the cooperative step kernel runs the
    // arrivals, the per-CTA kernel resumes at the first one that needs the
    // exact sequence (an input that can raise) and persists the state
    P.coop = (CoopState *)(ws + X.L.coop);
    int rc;
    if (hw.cap <= 48) rc = launch_place_coop<48>(P, st);
    else if (hw.cap <= 128) rc = launch_place_coop<128>(P, st);
    else rc = launch_place_coop<256>(P, st);
    if (rc) return rc;
  } else if (hw.cap <= 48) {
    launch_place<48>(P, st);
  } else if (hw.cap <= 128) {
    launch_place<128>(P, st);
  } else {
    launch_place<256>(P, st);
  }
  CK(cudaGetLastError());
  const size_t dp = (size_t)capacity * 4, sp = (size_t)n * 4;
  if (gpu_of)
    CK(cudaMemcpy2DAsync(gpu_of, sp, ws + X.gpu_of + (size_t)k0 * 4, dp, sp, S,
                         cudaMemcpyDeviceToDevice, st));
  if (pos)
    CK(cudaMemcpy2DAsync(pos, sp, ws + X.pos + (size_t)k0 * 4, dp, sp, S,
                         cudaMemcpyDeviceToDevice, st));
  if (code)
    CK(cudaMemcpy2DAsync(code, sp, ws + X.code + (size_t)k0 * 4, dp, sp, S,
                         cudaMemcpyDeviceToDevice, st));
  if (err)
    CK(cudaMemcpyAsync(err, ws + X.err, S * sizeof(igp_error), cudaMemcpyDeviceToDevice, st));
  return IGP_E_OK;
}

int igp_stream_snapshot_device(int n_streams, int n_arrivals, int capacity, const double *hw_h,
                               int b_max, int32_t *gpu_of, int32_t *pos, int32_t *units,
                               double *pred, int32_t *gpu_count, igp_error *err,
                               void *workspace, size_t workspace_bytes, int flags,
                               void *stream) {
  IGP_NVTX();
  if (n_streams < 1 || capacity < 1 || n_arrivals < 0 || n_arrivals > capacity || !hw_h ||
      !workspace)
    return IGP_E_ARG;
  Hw hw = make_hw(hw_h, b_max);
  if (hw.cap < 1) return IGP_E_ARG;
  if (hw.cap > igp_max_cap()) return IGP_E_CAPACITY;
  StreamLayout X = stream_layout(n_streams, capacity, hw.cap, flags);
  if (workspace_bytes < X.total) return IGP_E_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  char *ws = (char *)workspace;
  const size_t S = (size_t)n_streams;
  PlanParams P;
  stream_params(P, X, ws, hw, n_streams, capacity, flags & ~IGP_F_NO_PRED);
  P.k0 = P.k1 = n_arrivals;
  P.pred = (double *)(ws + X.pred);
  if (hw.cap <= 48) launch_place<48>(P, st);
  else if (hw.cap <= 128) launch_place<128>(P, st);
  else launch_place<256>(P, st);
  CK(cudaGetLastError());
  if (n_arrivals > 0) {
    const size_t dp = (size_t)capacity * 4, sp = (size_t)n_arrivals * 4;
    if (gpu_of)
      CK(cudaMemcpy2DAsync(gpu_of, sp, ws + X.gpu_of, dp, sp, S, cudaMemcpyDeviceToDevice, st));
    if (pos) CK(cudaMemcpy2DAsync(pos, sp, ws + X.pos, dp, sp, S, cudaMemcpyDeviceToDevice, st));
    if (units)
      CK(cudaMemcpy2DAsync(units, sp, ws + X.units, dp, sp, S, cudaMemcpyDeviceToDevice, st));
    if (pred)
      CK(cudaMemcpy2DAsync(pred, sp * 20, ws + X.pred, dp * 20, sp * 20, S,
                           cudaMemcpyDeviceToDevice, st));
  }
  if (gpu_count) CK(cudaMemcpyAsync(gpu_count, ws + X.gc, S * 4, cudaMemcpyDeviceToDevice, st));
  if (err) CK(cudaMemcpyAsync(err, ws + X.err, S * sizeof(igp_error), cudaMemcpyDeviceToDevice, st));
  return IGP_E_OK;
}

int igp_group_search_device(const double *wl, int n, const int32_t *batch, const double *hw_h,
                            const int32_t *grid, int n_grid, unsigned long long *best,
                            int32_t *err, void *stream) {
  IGP_NVTX();
  if (n < 1 || n > IGP_GS_MAXN || n_grid < 1 || !hw_h || !grid || !best || !err)
    return IGP_E_ARG;
  Hw hw = make_hw(hw_h, 0);
  if (hw.cap < 1) return IGP_E_ARG;
  if (hw.cap > igp_max_cap()) return IGP_E_CAPACITY;
  cudaStream_t st = (cudaStream_t)stream;
  GroupSearchParams G;
  G.hw = hw;
  G.n = n;
  G.n_grid = n_grid;
  G.wl = wl;
  G.batch = batch;
  G.grid = grid;
  G.best = best;
  G.err = err;
  long long acc = 0;
  G.base[0] = 0;
  for (int mask = 1; mask <= (1 << n); ++mask) {
    G.base[mask] = acc;
    if (mask == (1 << n)) break;
    long long c = 1;
    for (int b = 0; b < n; ++b)
      if ((mask >> b) & 1) c *= n_grid;
    acc += c;
  }
  G.base[1 << n] = acc;
  CK(cudaMemsetAsync(best, 0xff, sizeof(unsigned long long) << n, st));
  CK(cudaMemsetAsync(err, 0, sizeof(int32_t), st));
  long long blocks = (acc + 255) / 256;
  if (blocks > 148 * 64) blocks = 148 * 64;
  if (blocks < 1) blocks = 1;
  k_group_search<<<(unsigned)blocks, 256, 0, st>>>(G);
  CK(cudaGetLastError());
  return IGP_E_OK;
}

int igp_simulate_device(int n, const double *rate, const int32_t *batch, const double *service,
                        double duration_ms, double warmup_ms, const int64_t *seg, double *lat,
                        double *starts, double *sorted, int64_t *seg_end, int32_t *max_depth,
                        int32_t *backlog, int32_t *completed, double *p50, double *p99,
                        double *achieved, void *stream) {
  IGP_NVTX();
  if (n < 0 || !(duration_ms >= warmup_ms) || !(warmup_ms >= 0.0)) return IGP_E_ARG;
  if (n == 0) return IGP_E_OK;
  cudaStream_t st = (cudaStream_t)stream;
  SimParams S;
  S.n = n;
  S.duration = duration_ms;
  S.warmup = warmup_ms;
  S.rate = rate;
  S.batch = batch;
  S.service = service;
  S.seg = (const long long *)seg;
  S.lat = lat;
  S.starts = starts;
  S.seg_end = (long long *)seg_end;
  S.max_depth = max_depth;
  S.backlog = backlog;
  S.completed = completed;
  k_sim_replay<<<nblk(n, 128), 128, 0, st>>>(S);
  CK(cudaGetLastError());
  long long total = 0;
  CK(cudaMemcpyAsync(&total, seg + n, sizeof(long long), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  size_t tmp_bytes = 0;
  CK(cub::DeviceSegmentedSort::SortKeys(nullptr, tmp_bytes, lat, sorted, total, n, seg, seg_end,
                                        st));
  void *tmp = nullptr;
  CK(cudaMallocAsync(&tmp, tmp_bytes > 0 ? tmp_bytes : 1, st));
  CK(cub::DeviceSegmentedSort::SortKeys(tmp, tmp_bytes, lat, sorted, total, n, seg, seg_end, st));
  CK(cudaFreeAsync(tmp, st));
  k_sim_report<<<nblk(n, 128), 128, 0, st>>>(S, sorted, p50, p99, achieved);
  CK(cudaGetLastError());
  return IGP_E_OK;
}

int igp_solo_grid_device(const double *wl, int m, const double *hw_h, int b_max,
                         int32_t *min_units, int32_t *best_u, int32_t *best_b,
                         unsigned long long *n_evals, void *stream) {
  IGP_NVTX();
  if (m < 0 || b_max < 1 || !hw_h) return IGP_E_ARG;
  Hw hw = make_hw(hw_h, b_max);
  if (hw.cap < 1) return IGP_E_ARG;
  if (m == 0) return IGP_E_OK;
  cudaStream_t st = (cudaStream_t)stream;
  GridParams G;
  G.hw = hw;
  G.m = m;
  G.b_max = b_max;
  G.wl = wl;
  G.min_units = min_units;
  G.best_u = best_u;
  G.best_b = best_b;
  G.evals = n_evals;
  if (n_evals) CK(cudaMemsetAsync(n_evals, 0, sizeof(unsigned long long), st));
  k_solo_grid<<<nblk((long long)m * b_max, 256), 256, 0, st>>>(G);
  if (best_u && best_b) k_grid_best<<<nblk((long long)m * 32, 256), 256, 0, st>>>(G);
  CK(cudaGetLastError());
  return IGP_E_OK;
}

int igp_components_device(int n, const double *wl, const int32_t *batch, const double *r,
                          const double *co_cache, const int32_t *n_col, const double *p_dem,
                          const double *hw_h, double *out, int32_t *code, void *stream) {
  IGP_NVTX();
  if (n < 0 || !hw_h) return IGP_E_ARG;
  if (n == 0) return IGP_E_OK;
  if (!wl || !batch || !r || !co_cache || !n_col || !p_dem || !out || !code) return IGP_E_ARG;
  CompParams C;
  C.n = n;
  C.hw = make_hw(hw_h, 1);
  C.wl = wl;
  C.batch = batch;
  C.r = r;
  C.co_cache = co_cache;
  C.n_col = n_col;
  C.p_dem = p_dem;
  C.out = out;
  C.code = code;
  k_components<<<nblk(n, 128), 128, 0, (cudaStream_t)stream>>>(C);
  CK(cudaGetLastError());
  return IGP_E_OK;
}

int igp_power_demand_device(int n, const double *powers, const double *hw_h, double *out,
                            void *stream) {
  IGP_NVTX();
  if (n < 0 || !hw_h || !out || (n > 0 && !powers)) return IGP_E_ARG;
  k_power_demand<<<1, 32, 0, (cudaStream_t)stream>>>(n, powers, make_hw(hw_h, 1), out);
  CK(cudaGetLastError());
  return IGP_E_OK;
}

}  // extern "C"
