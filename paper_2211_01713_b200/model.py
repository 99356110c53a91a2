"""Interference-aware latency model: drop-in types and device-backed evaluation.

Types keep the reference's field names, defaults and validation
(``gpuplanner/model.py:19-156``).  Evaluation of a device state --
``_eval_entries`` (``model.py:273-317``) and ``predict_gpu``
(``model.py:320-343``) -- runs in the sm_100a kernel ``k_eval_states``
through ``igp_eval_states_device``; there is no host implementation.

Units: latencies in ms, sizes in MB, bandwidth in MB/ms, frequency in MHz,
power in W; rates are req/s at the API boundary.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Mapping, Sequence

import numpy as np

from . import _device
from .errors import native_exception
from .layout import E_ACTIVE_TIME, E_DENOM, WL_NF, hw_vector, spec_coef_row


@dataclass(frozen=True)
class WorkloadSpec:
    """SLO (ms), arrival rate (req/s) and per-request transfer sizes (MB)."""

    name: str
    slo_ms: float
    rate_rps: float
    d_load_mb: float
    d_feedback_mb: float

    def __post_init__(self):
        if not self.name:
            raise ValueError("workload name must be non-empty")
        if self.slo_ms <= 0:
            raise ValueError(f"slo_ms must be positive, got {self.slo_ms}")
        if self.rate_rps <= 0:
            raise ValueError(f"rate_rps must be positive, got {self.rate_rps}")
        if self.d_load_mb < 0 or self.d_feedback_mb < 0:
            raise ValueError("transfer sizes must be non-negative")


@dataclass(frozen=True)
class WorkloadCoefficients:
    """Fitted per-workload coefficients (active time k1..k5, power/cache lines)."""

    n_kernels: int
    k_sch_ms: float
    k1: float
    k2: float
    k3: float
    k4: float
    k5: float
    alpha_power_w: float
    beta_power_w: float
    alpha_cacheutil: float
    beta_cacheutil: float
    alpha_cache: float

    def __post_init__(self):
        if self.n_kernels < 1:
            raise ValueError(f"n_kernels must be >= 1, got {self.n_kernels}")
        if self.k_sch_ms < 0:
            raise ValueError(f"k_sch_ms must be >= 0, got {self.k_sch_ms}")
        if self.alpha_cache < 0:
            raise ValueError(f"alpha_cache must be >= 0, got {self.alpha_cache}")


@dataclass(frozen=True)
class HardwareProfile:
    """Device coefficients, allocation granularity and hourly price."""

    gpu_type: str
    power_max_w: float
    freq_max_mhz: float
    power_idle_w: float
    pcie_bw_mb_per_ms: float
    alpha_f: float
    alpha_sch_ms: float
    beta_sch_ms: float
    r_unit: float = 0.025
    r_max: float = 1.0
    price_per_hour: float = 1.0
    f_min_frac: float = 0.3

    def __post_init__(self):
        if self.power_idle_w < 0 or self.power_max_w <= self.power_idle_w:
            raise ValueError("requires power_max_w > power_idle_w >= 0")
        if self.freq_max_mhz <= 0:
            raise ValueError(f"freq_max_mhz must be positive, got {self.freq_max_mhz}")
        if self.pcie_bw_mb_per_ms <= 0:
            raise ValueError("pcie_bw_mb_per_ms must be positive")
        if self.r_max != 1.0:
            raise ValueError(f"r_max must be 1.0, got {self.r_max}")
        if not 0 < self.r_unit <= self.r_max:
            raise ValueError(f"r_unit must be in (0, {self.r_max}], got {self.r_unit}")
        if self.price_per_hour <= 0:
            raise ValueError("price_per_hour must be positive")
        if not 0 < self.f_min_frac <= 1:
            raise ValueError("f_min_frac must be in (0, 1]")

    @property
    def f_min_mhz(self) -> float:
        return self.f_min_frac * self.freq_max_mhz


@dataclass(frozen=True)
class Allocation:
    """A workload's resource fraction r and batch size on one device."""

    workload: str
    r: float
    batch: int

    def __post_init__(self):
        if self.r <= 0:
            raise ValueError(f"r must be positive, got {self.r}")
        if self.batch < 1:
            raise ValueError(f"batch must be >= 1, got {self.batch}")


@dataclass(frozen=True)
class LatencyBreakdown:
    """One resident's predicted latency terms, throughput, solo power and cache."""

    t_load_ms: float
    t_sch_ms: float
    t_act_ms: float
    freq_mhz: float
    t_gpu_ms: float
    t_feedback_ms: float
    t_inf_ms: float
    throughput_rps: float
    power_w: float
    cache_util: float


@dataclass(frozen=True)
class SloCheck:
    latency_ok: bool
    throughput_ok: bool

    @property
    def ok(self) -> bool:
        return self.latency_ok and self.throughput_ok


def slo_check(breakdown: LatencyBreakdown, spec: WorkloadSpec) -> SloCheck:
    """Half-SLO latency budget and arrival-rate floor (model.py:346-351)."""
    return SloCheck(
        latency_ok=bool(breakdown.t_inf_ms <= spec.slo_ms / 2.0),
        throughput_ok=bool(breakdown.throughput_rps >= spec.rate_rps),
    )


# ---- component functions (model.py:159-236), evaluated on the device --------
# Each call is one igp_components_device launch over a single query; the
# columns follow include/igniter_b200.h.
_K_TLOAD, _K_TFB, _K_DENOM, _K_KACT, _K_POWER, _K_CACHE, _K_SCHINC, _K_SCHED, _K_ACTINT, \
    _K_FREQ = range(10)


def _component(hw, *, spec=None, coef=None, batch=1, r=1.0, co_cache=0.0, n_col=1, p_dem=0.0):
    row = np.zeros((WL_NF, 1))
    if coef is not None:
        row[:, 0] = spec_coef_row(spec, coef) if spec is not None else \
            spec_coef_row(_ZeroSpec, coef)
    elif spec is not None:
        row[:, 0] = spec_coef_row(spec, _UnitCoef)
    out, code = _device.components(row, [batch], [r], [co_cache], [n_col], [p_dem],
                                   hw_vector(hw))
    return out[0], int(code[0])


class _ZeroSpec:  # spec fields a coefficient-only query does not read
    slo_ms = rate_rps = d_load_mb = d_feedback_mb = 0.0


class _NEUTRAL_HW:  # hardware fields the hardware-independent columns do not read
    power_max_w = freq_max_mhz = pcie_bw_mb_per_ms = r_max = price_per_hour = f_min_frac = 1.0
    power_idle_w = alpha_f = alpha_sch_ms = beta_sch_ms = 0.0
    r_unit = 0.025


class _UnitCoef:  # coefficient fields a spec-only query does not read
    n_kernels = 1
    k_sch_ms = k1 = k2 = k3 = k5 = alpha_power_w = beta_power_w = 0.0
    alpha_cacheutil = beta_cacheutil = alpha_cache = 0.0
    k4 = 1.0


def _solo(coef, batch, r, need_positive):
    out, code = _component(_NEUTRAL_HW, coef=coef, batch=batch, r=r)
    if code == E_DENOM:
        raise native_exception(code, float(out[_K_DENOM]), float(r), float(coef.k4))
    if need_positive and code == E_ACTIVE_TIME:
        raise native_exception(code, float(out[_K_KACT]), batch, float(r))
    return out


def transfer_latencies(spec: WorkloadSpec, batch: int, hw: HardwareProfile) -> tuple[float, float]:
    """PCIe load/feedback latency of one batch, in ms (model.py:159-165)."""
    out, _ = _component(hw, spec=spec, batch=batch)
    return float(out[_K_TLOAD]), float(out[_K_TFB])


def solo_active_time(coef: WorkloadCoefficients, batch: int, r: float) -> float:
    """GPU active time (ms) of a batch running alone (model.py:168-175)."""
    return float(_solo(coef, batch, r, False)[_K_KACT])


def solo_power(coef: WorkloadCoefficients, batch: int, r: float) -> float:
    """Solo power draw (W), linear in batch / k_act (model.py:186-190)."""
    return float(_solo(coef, batch, r, True)[_K_POWER])


def solo_cache_util(coef: WorkloadCoefficients, batch: int, r: float) -> float:
    """Solo L2-cache utilisation clamped to [0, 1] (model.py:193-198)."""
    return float(_solo(coef, batch, r, True)[_K_CACHE])


def sched_delay_increase(hw: HardwareProfile, n_colocated: int) -> float:
    """Per-kernel scheduling-delay increase (ms) from co-location (model.py:201-209)."""
    out, _ = _component(hw, n_col=n_colocated)
    return float(out[_K_SCHINC])


def sched_delay(coef: WorkloadCoefficients, hw: HardwareProfile, n_colocated: int) -> float:
    """Total kernel scheduling delay (ms) for one batch (model.py:212-216)."""
    out, _ = _component(hw, coef=coef, n_col=n_colocated)
    return float(out[_K_SCHED])


def active_time_with_interference(coef: WorkloadCoefficients, batch: int, r: float,
                                  co_cache_sum: float) -> float:
    """Active time (ms) inflated by co-runners' summed cache use (model.py:219-223)."""
    out, code = _component(_NEUTRAL_HW, coef=coef, batch=batch, r=r, co_cache=co_cache_sum)
    if code == E_DENOM:
        raise native_exception(code, float(out[_K_DENOM]), float(r), float(coef.k4))
    return float(out[_K_ACTINT])


def power_demand(hw: HardwareProfile, solo_powers) -> float:
    """Device power demand (W): idle draw + the residents' solo power (model.py:226-228)."""
    return _device.power_demand([float(p) for p in solo_powers], hw_vector(hw))


def gpu_frequency(hw: HardwareProfile, p_demand: float) -> float:
    """Operating frequency (MHz) under the power cap (model.py:231-236)."""
    out, _ = _component(hw, p_dem=p_demand)
    return float(out[_K_FREQ])


class _Entry:
    """A (spec, coefficients, batch) triple prepared for device evaluation.

    The device forms the pre-reduced constants itself (k_build / row_entry);
    this host object keeps ``spec`` and ``coef`` for marshalling and exposes
    the reference's attributes (model.py:239-270: ``gamma``, ``k4`` ...
    ``t_load``, ``t_feedback``, ``t_half``, ``rate_rps``), so modules that
    import ``_Entry`` (oracle.py:16-22, baselines.py:19-28) read the same
    values.  They are formed on first access with the reference's operations
    in the reference's order (CPython floats: identical bits).
    """

    __slots__ = ("name", "batch", "spec", "coef", "t_half", "rate_rps", "_hw")

    def __init__(self, spec, coef, batch: int, hw=None):
        self.name = spec.name
        self.batch = batch
        self.spec = spec
        self.coef = coef
        self.t_half = spec.slo_ms / 2.0
        self.rate_rps = spec.rate_rps
        self._hw = hw

    @property
    def gamma(self):
        c, b = self.coef, self.batch
        return c.k1 * b * b + c.k2 * b + c.k3

    k4 = property(lambda self: self.coef.k4)
    k5 = property(lambda self: self.coef.k5)
    k_sch = property(lambda self: self.coef.k_sch_ms)
    n_kernels = property(lambda self: self.coef.n_kernels)
    alpha_cache = property(lambda self: self.coef.alpha_cache)
    alpha_p = property(lambda self: self.coef.alpha_power_w)
    beta_p = property(lambda self: self.coef.beta_power_w)
    alpha_c = property(lambda self: self.coef.alpha_cacheutil)
    beta_c = property(lambda self: self.coef.beta_cacheutil)

    @property
    def t_load(self):
        return self.spec.d_load_mb * self.batch / self._hw.pcie_bw_mb_per_ms

    @property
    def t_feedback(self):
        return self.spec.d_feedback_mb * self.batch / self._hw.pcie_bw_mb_per_ms


def _states_to_arrays(states):
    """[(entries, rs), ...] -> SoA workload table, batch, r, CSR ptr."""
    n = sum(len(e) for e, _ in states)
    wl = np.empty((WL_NF, n), dtype=np.float64)
    batch = np.empty(n, np.int32)
    r = np.empty(n, np.float64)
    ptr = np.zeros(len(states) + 1, np.int64)
    k = 0
    for s, (entries, rs) in enumerate(states):
        for e, rv in zip(entries, rs):
            wl[:, k] = spec_coef_row(e.spec, e.coef)
            batch[k] = e.batch
            r[k] = rv
            k += 1
        ptr[s + 1] = k
    return wl, batch, r, ptr


def _raise_state_error(rec, hw):
    raise native_exception(int(rec["code"]), float(rec["a"]), float(rec["b"]),
                           float(rec["c"]), hw=hw)


def eval_states(states, hw, check_capacity=False):
    """Evaluate many device states in one launch; returns a list of row lists.

    Raises the first error in state order, as a sequential loop over the
    reference's _eval_entries / predict_gpu would."""
    if not states:
        return []
    wl, batch, r, ptr = _states_to_arrays(states)
    rows, err = _device.eval_states(wl, batch, r, ptr, hw_vector(hw), check_capacity)
    bad = np.nonzero(err["code"])[0]
    if len(bad):
        _raise_state_error(err[bad[0]], hw)
    return [[tuple(float(v) for v in rows[i]) for i in range(ptr[s], ptr[s + 1])]
            for s in range(len(states))]


def _eval_entries(entries: Sequence[_Entry], rs: Sequence[float], hw: HardwareProfile):
    """Device evaluation of one state; tuples in LatencyBreakdown order."""
    if len(entries) == 0:
        return []
    return eval_states([(list(entries), list(rs))], hw)[0]


def predict_gpu(
    allocations: Sequence[Allocation],
    specs: Mapping[str, WorkloadSpec],
    coefs: Mapping[str, WorkloadCoefficients],
    hw: HardwareProfile,
) -> dict[str, LatencyBreakdown]:
    """Every resident's breakdown under co-location (capacity check first)."""
    if len(allocations) == 0:
        return {}
    entries = [_Entry(specs[a.workload], coefs[a.workload], a.batch, hw) for a in allocations]
    rows = eval_states([(entries, [a.r for a in allocations])], hw, check_capacity=True)[0]
    return {a.workload: LatencyBreakdown(*(float(v) for v in row))
            for a, row in zip(allocations, rows)}
