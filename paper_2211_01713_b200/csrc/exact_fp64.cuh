// exact_fp64.cuh -- CPython-exact fp64 building blocks for the iGniter model.
//
// The whole translation unit is compiled with -fmad=false, so every a*b+c in
// this file is a DMUL followed by a DADD, each rounded to nearest-even exactly
// like CPython's float ops.  Division is the IEEE-exact DIV sequence (CUDA
// double division is always correctly rounded).  Association follows the
// reference expressions left to right.
#pragma once

#include <cstdint>

#include "../../include/igniter_b200.h"

namespace igp {

// Hardware profile with the derived constants the kernels use.
struct Hw {
  double pmax, fmax, pidle, bw, af, asch, bsch, runit, rmax, price, fminfrac;
  double fmin;  // f_min_mhz = f_min_frac * freq_max_mhz  (model.py:108-110)
  int cap;      // max_units = int(round(r_max / r_unit)) (planner.py:72-73)
  int margin_ok;  // scale = f / fmax is finite and > 0 for every reachable f
  int b_max;
};

// Python max(a, b) / min(a, b): the second argument wins only on a strict
// comparison, so ties, NaNs and signed zeros resolve exactly like CPython.
__device__ __forceinline__ double py_max(double a, double b) { return (b > a) ? b : a; }
__device__ __forceinline__ double py_min(double a, double b) { return (b < a) ? b : a; }

// CPython 3.12 builtin sum over floats with start=0 (Python/bltinmodule.c,
// builtin_sum_impl): the first term enters as int(0) + x0, the rest go
// through Neumaier's compensated step; the compensation is added at the end
// only when it is non-zero and finite.  The fold order is the resident order.
struct Neumaier {
  double s, c;
  __device__ __forceinline__ void first(double x0) {
    s = __dadd_rn(0.0, x0);
    c = 0.0;
  }
  __device__ __forceinline__ void add(double x) {
    const double t = s + x;
    // c += (s - t) + x if |s| >= |x| else (x - t) + s: same operations on
    // selected operands, branch-free
    const bool big = fabs(s) >= fabs(x);
    const double a = big ? s : x, b = big ? x : s;
    c += (a - t) + b;
    s = t;
  }
  __device__ __forceinline__ double result() const {
    return (c != 0.0 && isfinite(c)) ? s + c : s;
  }
};

// Scheduling-delay increase for n co-located workloads (model.py:201-209 /
// model.py:281).
__device__ __forceinline__ double delta_sch(const Hw &hw, int n) {
  return (n <= 1) ? 0.0 : py_max(0.0, hw.asch * (double)n + hw.bsch);
}

// Power-capped frequency (model.py:300-303).
__device__ __forceinline__ double frequency(const Hw &hw, double p_dem) {
  if (p_dem <= hw.pmax) return hw.fmax;
  return py_max(hw.fmin, hw.fmax + hw.af * (p_dem - hw.pmax));
}

// Per-workload constants that the allocation loop needs when a unit changes
// (model.py:253-266).  Stored as 12 doubles per workload.
enum { C_GAMMA = 0, C_K4, C_K5, C_BATCH, C_AP, C_BP, C_AC, C_BC, C_KSCH, C_NK, C_LB, C_WIN, C_NF };
// Per-workload resident state read by every check (64 B, one half line):
// solo k_act / power / cache at the current units, t_sch for the next
// candidate size, and the transfer / budget constants.
enum { S_KA = 0, S_PW, S_CA, S_TSN, S_ACACHE, S_TLOAD, S_TFB, S_THALF, S_NF };

struct Solo {
  double ka, pw, ca;
  int err;  // 0, IGP_E_DENOM or IGP_E_ACTIVE_TIME
};

// First loop body of _eval_entries (model.py:285-297) for one entry at r.
__device__ __forceinline__ Solo solo_at(double gamma, double k4, double k5, double batch,
                                        double ap, double bp, double ac, double bc, double r) {
  Solo o;
  o.err = 0;
  double denom = r + k4;
  if (denom <= 0) o.err = IGP_E_DENOM;
  double k_act = gamma / denom + k5;
  if (!o.err && k_act <= 0) o.err = IGP_E_ACTIVE_TIME;
  double ability = batch / k_act;
  double c = ac * ability + bc;
  o.ka = k_act;
  o.pw = ap * ability + bp;
  o.ca = py_min(1.0, py_max(0.0, c));
  return o;
}

__device__ __forceinline__ Solo solo_from_cold(const double *cold, double r) {
  return solo_at(cold[C_GAMMA], cold[C_K4], cold[C_K5], cold[C_BATCH], cold[C_AP], cold[C_BP],
                 cold[C_AC], cold[C_BC], r);
}

}  // namespace igp
