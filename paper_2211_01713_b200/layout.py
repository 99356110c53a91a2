"""Column layouts shared by the C-ABI, the oracle and the golden fixtures.

A workload table is structure-of-arrays, field-major: ``wl[f * m + i]`` is
field ``f`` of workload ``i`` (input order), all fp64.  ``n_kernels`` is an
integer in the reference (``model.py:51``) but only ever enters arithmetic as
``k_sch_ms * n_kernels`` (``model.py:216``, ``planner.py:105``), where CPython
converts it to a double exactly; storing it as fp64 is therefore bit-neutral.

The hardware record mirrors ``HardwareProfile`` (``model.py:73-110``).
The breakdown row mirrors ``LatencyBreakdown`` field order (``model.py:133-146``),
which is also the tuple order of ``_eval_entries`` (``model.py:315-316``).
"""

# workload fields: WorkloadSpec (model.py:19-27) then WorkloadCoefficients (model.py:40-62)
WL_FIELDS = (
    "slo_ms", "rate_rps", "d_load_mb", "d_feedback_mb",
    "n_kernels", "k_sch_ms", "k1", "k2", "k3", "k4", "k5",
    "alpha_power_w", "beta_power_w", "alpha_cacheutil", "beta_cacheutil",
    "alpha_cache",
)
WL_NF = len(WL_FIELDS)  # 16
WL = {name: i for i, name in enumerate(WL_FIELDS)}

HW_FIELDS = (
    "power_max_w", "freq_max_mhz", "power_idle_w", "pcie_bw_mb_per_ms",
    "alpha_f", "alpha_sch_ms", "beta_sch_ms", "r_unit", "r_max",
    "price_per_hour", "f_min_frac",
)
HW_NF = len(HW_FIELDS)  # 11

ROW_FIELDS = (
    "t_load_ms", "t_sch_ms", "t_act_ms", "freq_mhz", "t_gpu_ms",
    "t_feedback_ms", "t_inf_ms", "throughput_rps", "power_w", "cache_util",
)
ROW_NF = len(ROW_FIELDS)  # 10

# error codes carried across the C-ABI (include/igniter_b200.h, IGP_E_*)
E_OK = 0
E_BATCH_CAP = 1          # BatchCapExceededError      planner.py:86-91
E_INFEASIBLE_SLO = 2     # InfeasibleSloError         planner.py:107-111
E_INFEASIBLE_RES = 3     # InfeasibleResourceError    planner.py:115-119
E_DENOM = 4              # NonPositiveDenominatorError model.py:286-290 (r + k4 <= 0)
E_ACTIVE_TIME = 5        # NonPositiveDenominatorError model.py:178-183 (k_act <= 0)
E_OVERALLOC = 6          # OverAllocatedError         model.py:331-335
E_CAPACITY = 7           # scratch capacity exceeded (library limit, not a model error)
E_CUDA = 8               # CUDA runtime failure
E_ARG = 9                # invalid argument at the boundary


def hw_vector(hw):
    """Pack any object with HardwareProfile attributes into HW_FIELDS order."""
    return [float(getattr(hw, f)) for f in HW_FIELDS]


def spec_coef_row(spec, coef):
    """One workload's 16 fields in WL_FIELDS order from (spec, coef) objects."""
    return [
        float(spec.slo_ms), float(spec.rate_rps), float(spec.d_load_mb),
        float(spec.d_feedback_mb), float(coef.n_kernels), float(coef.k_sch_ms),
        float(coef.k1), float(coef.k2), float(coef.k3), float(coef.k4),
        float(coef.k5), float(coef.alpha_power_w), float(coef.beta_power_w),
        float(coef.alpha_cacheutil), float(coef.beta_cacheutil),
        float(coef.alpha_cache),
    ]
