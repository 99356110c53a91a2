// components.cuh -- the latency model's scalar component functions
// (model.py:159-236), batched: one thread per query.
//
// These are the public helpers the reference exposes beside predict_gpu
// (transfer_latencies, solo_active_time, solo_power, solo_cache_util,
// sched_delay_increase, sched_delay, active_time_with_interference,
// gpu_frequency, power_demand).  Each column is computed with the operation
// order of its reference function, so results are bit-identical.
#pragma once

namespace igp {

// output columns per query
enum {
  K_TLOAD = 0,  // transfer_latencies[0]          model.py:159-165
  K_TFB,        // transfer_latencies[1]
  K_DENOM,      // r + k4 (the operand of the denominator error)
  K_KACT,       // solo_active_time               model.py:168-175
  K_POWER,      // solo_power                     model.py:186-190
  K_CACHE,      // solo_cache_util                model.py:193-198
  K_SCHINC,     // sched_delay_increase           model.py:201-209
  K_SCHED,      // sched_delay                    model.py:212-216
  K_ACTINT,     // active_time_with_interference  model.py:219-223
  K_FREQ,       // gpu_frequency                  model.py:231-236
  K_NF
};

struct CompParams {
  int n;
  Hw hw;
  const double *wl;       // [IGP_WL_NF][n] query fields, field-major like the plan tables
  const int32_t *batch;   // [n]
  const double *r;        // [n] resource fraction
  const double *co_cache; // [n] co-runners' summed cache utilisation
  const int32_t *n_col;   // [n] co-located workloads
  const double *p_dem;    // [n] device power demand (W)
  double *out;            // [n][K_NF]
  int32_t *code;          // [n] 0, IGP_E_DENOM (r + k4 <= 0) or IGP_E_ACTIVE_TIME (k_act <= 0)
};

__global__ void k_components(CompParams C) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= C.n) return;
#define w(f) C.wl[(size_t)(f) * C.n + i]
  const Hw &hw = C.hw;
  double *o = C.out + (size_t)i * K_NF;
  const double b = (double)C.batch[i], r = C.r[i];
  o[K_TLOAD] = (w(IGP_WL_DLOAD) * b) / hw.bw;
  o[K_TFB] = (w(IGP_WL_DFB) * b) / hw.bw;
  const double denom = r + w(IGP_WL_K4);
  o[K_DENOM] = denom;
  int code = 0;
  double k_act = 0.0;
  if (denom <= 0.0) {
    code = IGP_E_DENOM;
  } else {
    // (k1 * batch * batch + k2 * batch + k3) / denom + k5
    k_act = (((w(IGP_WL_K1) * b) * b + w(IGP_WL_K2) * b) + w(IGP_WL_K3)) / denom + w(IGP_WL_K5);
    if (k_act <= 0.0) code = IGP_E_ACTIVE_TIME;
  }
  o[K_KACT] = k_act;
  const double ab = b / k_act;
  o[K_POWER] = w(IGP_WL_ALPHA_P) * ab + w(IGP_WL_BETA_P);
  o[K_CACHE] = py_min(1.0, py_max(0.0, w(IGP_WL_ALPHA_CU) * ab + w(IGP_WL_BETA_CU)));
  const double inc = delta_sch(hw, C.n_col[i]);
  o[K_SCHINC] = inc;
  o[K_SCHED] = (w(IGP_WL_KSCH) + inc) * w(IGP_WL_NK);
  o[K_ACTINT] = k_act * (1.0 + w(IGP_WL_ALPHA_CACHE) * C.co_cache[i]);
  o[K_FREQ] = frequency(hw, C.p_dem[i]);
  C.code[i] = code;
#undef w
}

// power_demand (model.py:226-228): idle draw + CPython sum of the solo powers
__global__ void k_power_demand(int n, const double *powers, Hw hw, double *out) {
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  if (n == 0) {
    *out = hw.pidle;  // sum([]) is int 0; pidle + 0 == pidle
    return;
  }
  Neumaier f;
  f.first(powers[0]);
  for (int i = 1; i < n; ++i) f.add(powers[i]);
  *out = hw.pidle + f.result();
}

}  // namespace igp
