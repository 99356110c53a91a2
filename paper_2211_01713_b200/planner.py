"""Provisioning API (drop-in for ``gpuplanner.planner``), executed on the B200.

Signatures, return types, tie-breaks and exceptions follow the reference
(``gpuplanner/planner.py:38-364``).  The work behind each call runs in the
sm_100a library:

* ``plan``              -> ``igp_plan_batch_device`` (prologue, sort, Alg. 1
                           with Alg. 2 per candidate, _build_plan predictions)
* ``alloc_gpus``        -> ``igp_alloc_units_device`` (Alg. 2)
* ``appropriate_batch`` / ``lower_bound_resources`` -> ``igp_prologue_device``

Host code only validates inputs (duplicate names, planner.py:249-255),
ranks names in Python string order for the sort tie-break (planner.py:284),
marshals structure-of-arrays buffers, and assembles the result objects.
"""

from __future__ import annotations

from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field, fields
from itertools import chain
from operator import attrgetter
from typing import Mapping, Sequence

import numpy as np

from . import _device
from .errors import (
    BatchCapExceededError,
    InfeasibleError,
    InfeasibleResourceError,
    InfeasibleSloError,
    native_exception,
)
from .layout import E_BATCH_CAP, WL_FIELDS, WL_NF, hw_vector, spec_coef_row
from .model import (
    Allocation,
    HardwareProfile,
    LatencyBreakdown,
    WorkloadCoefficients,
    WorkloadSpec,
    _Entry,
    predict_gpu,
    slo_check,
)

DEFAULT_BATCH_CAP = 32
IGP_F_STATS = 1
IGP_F_CTA = 4
IGP_F_SMEM = 8
IGP_F_COOP = 16
CTA_MIN_WORKLOADS = 512      # one CTA per plan: 12.6 ms vs 22.5 ms (one warp) at 1k workloads
COOP_MIN_WORKLOADS = 10_000  # whole-GPU steps: 16.2 vs 19.5 us/step (one CTA) at 15k, 16.8 vs 23.5 at 20k;
                             # one CTA wins below 10k (13.1 vs 16.5 at 5k) and ties at 10k


@dataclass
class GpuPlan:
    """Allocations committed to one device, with model predictions."""

    gpu_index: int
    allocations: list[Allocation]
    predicted: dict[str, LatencyBreakdown]
    fragment_r: float


@dataclass
class Plan:
    """Provisioning plan over devices of one GPU type."""

    strategy: str
    gpu_type: str
    gpus: list[GpuPlan]
    cost_per_hour: float
    per_workload_r_inter: dict[str, float]
    diagnostics: list[str] = field(default_factory=list)

    @property
    def gpu_count(self) -> int:
        return len(self.gpus)


@dataclass
class PlanStats:
    """Reference operation counters (planner.py:64-69): model_evals counts
    per-resident model evaluations, candidate_gpus (workload, GPU) trials."""

    model_evals: int = 0
    candidate_gpus: int = 0


def max_units(hw) -> int:
    return int(round(hw.r_max / hw.r_unit))


def _one_workload_table(spec, coef=None) -> np.ndarray:
    wl = np.zeros((WL_NF, 1), dtype=np.float64)
    if coef is None:
        wl[:4, 0] = [spec.slo_ms, spec.rate_rps, spec.d_load_mb, spec.d_feedback_mb]
        wl[4, 0] = 1.0
    else:
        wl[:, 0] = spec_coef_row(spec, coef)
    return wl


def appropriate_batch(spec: WorkloadSpec, hw: HardwareProfile,
                      b_max: int = DEFAULT_BATCH_CAP) -> int:
    """Eq. 19 batch (planner.py:76-92), computed by the device prologue."""
    batch, _, code, err = _device.prologue(_one_workload_table(spec), hw_vector(hw), b_max)
    if code[0] == E_BATCH_CAP:
        raise native_exception(E_BATCH_CAP, float(err["a"]), 0.0, 0.0, spec=spec, hw=hw,
                               b_max=b_max)
    return int(batch[0])


def _lower_bound_units(spec, coef, hw, batch: int) -> int:
    """Eq. 20 lower bound in allocation units (planner.py:95-120)."""
    _, lb, code, err = _device.prologue(_one_workload_table(spec, coef), hw_vector(hw),
                                        DEFAULT_BATCH_CAP, batch_in=np.array([batch], np.int32))
    if code[0]:
        raise native_exception(int(code[0]), float(err["a"]), 0.0, 0.0, spec=spec, hw=hw)
    return int(lb[0])


def lower_bound_resources(spec, coef, hw, batch: int) -> float:
    """Minimum solo resource fraction meeting the half-SLO (planner.py:123-130)."""
    return _lower_bound_units(spec, coef, hw, batch) * hw.r_unit


def alloc_gpus(
    specs: Mapping[str, WorkloadSpec],
    coefs: Mapping[str, WorkloadCoefficients],
    hw: HardwareProfile,
    current: Sequence[Allocation],
    workload: str,
    batch: int,
    r_lower: float,
) -> list[Allocation]:
    """Alg. 2 for residents + newcomer (planner.py:165-192); a result summing
    beyond r_max is the reference's infeasibility marker."""
    names = [a.workload for a in current] + [workload]
    batches = [a.batch for a in current] + [batch]
    rs = [a.r for a in current] + [r_lower]
    wl = np.empty((WL_NF, len(names)), dtype=np.float64)
    for k, nm in enumerate(names):
        wl[:, k] = spec_coef_row(specs[nm], coefs[nm])
    units, err = _device.alloc_units(wl, np.array(batches, np.int32), np.array(rs),
                                     np.array([0, len(names)], np.int64), hw_vector(hw))
    if err[0]["code"]:
        e = err[0]
        raise native_exception(int(e["code"]), float(e["a"]), float(e["b"]), float(e["c"]), hw=hw)
    return [Allocation(nm, int(u) * hw.r_unit, b) for nm, u, b in zip(names, units, batches)]


def violation_diagnostics(gpus: Sequence[GpuPlan], specs: Mapping[str, WorkloadSpec]) -> list[str]:
    """Readable SLO violations of predicted plans (planner.py:195-215)."""
    out = []
    for gpu in gpus:
        for alloc in gpu.allocations:
            spec = specs[alloc.workload]
            bd = gpu.predicted[alloc.workload]
            chk = slo_check(bd, spec)
            if not chk.latency_ok:
                out.append(f"{alloc.workload} on gpu {gpu.gpu_index}: predicted latency "
                           f"{bd.t_inf_ms:.3f} ms exceeds half-SLO {spec.slo_ms / 2.0:.3f} ms")
            if not chk.throughput_ok:
                out.append(f"{alloc.workload} on gpu {gpu.gpu_index}: predicted throughput "
                           f"{bd.throughput_rps:.1f} req/s below rate {spec.rate_rps:.1f} req/s")
    return out


def _build_plan(strategy, hw, placement, specs, coefs, lb_units) -> Plan:
    """Plan from explicit (names, units, batches) per device; predictions for
    all devices are evaluated in ONE device launch (planner.py:218-246)."""
    cap = max_units(hw)
    allocs_per_gpu = []
    states = []
    for names, units, batches in placement:
        allocations = [Allocation(nm, u * hw.r_unit, b) for nm, u, b in zip(names, units, batches)]
        allocs_per_gpu.append(allocations)
        states.append(([_Entry(specs[a.workload], coefs[a.workload], a.batch, hw)
                        for a in allocations], [a.r for a in allocations]))
    from .model import eval_states
    rows_per_gpu = eval_states([s for s in states if s[0]], hw, check_capacity=True)
    gpus = []
    r_inter: dict[str, float] = {}
    it = iter(rows_per_gpu)
    for index, ((names, units, batches), allocations) in enumerate(zip(placement, allocs_per_gpu)):
        rows = next(it) if allocations else []
        predicted = {a.workload: LatencyBreakdown(*(float(v) for v in row))
                     for a, row in zip(allocations, rows)}
        gpus.append(GpuPlan(index, allocations, predicted, (cap - sum(units)) * hw.r_unit))
        for nm, u in zip(names, units):
            r_inter[nm] = (u - lb_units[nm]) * hw.r_unit
    return Plan(strategy=strategy, gpu_type=hw.gpu_type, gpus=gpus,
                cost_per_hour=len(gpus) * hw.price_per_hour, per_workload_r_inter=r_inter)


def _check_unique_names(workloads) -> None:
    names = [s.name for s, _ in workloads]
    if len(set(names)) != len(names):
        dup = sorted({n for n in names if names.count(n) > 1})
        raise ValueError(f"duplicate workload names: {dup}")


def name_ranks(names: Sequence[str]) -> np.ndarray:
    """Position of each name in Python string order (planner.py:284 tie-break)."""
    order = sorted(range(len(names)), key=names.__getitem__)
    rank = np.empty(len(names), np.int32)
    rank[np.asarray(order, dtype=np.int64)] = np.arange(len(names), dtype=np.int32)
    return rank


_SPEC_GET = attrgetter(*WL_FIELDS[:4])
_COEF_GET = attrgetter(*WL_FIELDS[4:])


def workload_table(workloads) -> np.ndarray:
    """(spec, coef) pairs -> [16, m] float64 SoA table (layout.WL_FIELDS):
    C-level attribute gathers streamed into numpy (about 1 us per workload)."""
    m = len(workloads)
    wl = np.empty((WL_NF, m), dtype=np.float64)
    if m:
        specs = [w[0] for w in workloads]
        coefs = [w[1] for w in workloads]
        wl[:4] = np.fromiter(chain.from_iterable(map(_SPEC_GET, specs)), np.float64,
                             count=4 * m).reshape(m, 4).T
        wl[4:] = np.fromiter(chain.from_iterable(map(_COEF_GET, coefs)), np.float64,
                             count=(WL_NF - 4) * m).reshape(m, WL_NF - 4).T
    return wl


_LB_FIELDS = tuple(f.name for f in fields(LatencyBreakdown))
_AL_FIELDS = tuple(f.name for f in fields(Allocation))
_new = object.__new__
_set = object.__setattr__


def _frozen(cls, names, values):
    """A frozen dataclass instance from already-validated device outputs,
    without the per-field __setattr__ of the generated __init__ (the values
    are exactly those the reference constructor would store)."""
    o = _new(cls)
    _set(o, "__dict__", dict(zip(names, values)))
    return o


class _DevicePlan(Plan):
    """A Plan assembled from one scenario's device arrays.  The per-GPU
    objects (GpuPlan, Allocation, LatencyBreakdown: ~3 per workload) are
    built on first access of ``gpus`` / ``per_workload_r_inter``; everything
    else is set at once.  Equal to the eagerly built Plan in every field."""

    def __getattr__(self, name):  # only reached while the lazy fields are unset
        if name in ("gpus", "per_workload_r_inter") and "_arrays" in self.__dict__:
            self._materialize()
            return self.__dict__[name]
        raise AttributeError(name)

    @property
    def gpu_count(self) -> int:
        return self.__dict__["_g"]

    def __eq__(self, other):
        if not isinstance(other, Plan):
            return NotImplemented
        return all(getattr(self, f.name) == getattr(other, f.name) for f in fields(Plan))

    __hash__ = None

    def __reduce__(self):
        return (Plan, tuple(getattr(self, f.name) for f in fields(Plan)))

    def _materialize(self):
        workloads, hw, g, gpu_of, pos, units, batch, lb, pred = self.__dict__.pop("_arrays")
        m = len(workloads)
        names = [w[0].name for w in workloads]
        order = np.lexsort((pos, gpu_of)).tolist()
        ends = np.cumsum(np.bincount(gpu_of, minlength=g)).tolist()
        units_l, batch_l = units.tolist(), batch.tolist()
        inter_l = ((units - lb) * hw.r_unit).tolist()
        r_l = (units * hw.r_unit).tolist()
        rows = pred.tolist()
        cap = max_units(hw)
        gpus, r_inter, start = [], {}, 0
        for j in range(g):
            allocations, predicted, used = [], {}, 0
            for i in order[start:ends[j]]:
                name = names[i]
                used += units_l[i]
                allocations.append(_frozen(Allocation, _AL_FIELDS, (name, r_l[i], batch_l[i])))
                predicted[name] = _frozen(LatencyBreakdown, _LB_FIELDS, rows[i])
                r_inter[name] = inter_l[i]
            start = ends[j]
            gpus.append(GpuPlan(j, allocations, predicted, (cap - used) * hw.r_unit))
        assert start == m
        self.__dict__["gpus"] = gpus
        self.__dict__["per_workload_r_inter"] = r_inter


def _plan_from_arrays(res, s, workloads, hw) -> Plan:
    """The reference Plan object of one scenario's device outputs (lazily
    materialised, see _DevicePlan)."""
    p = _new(_DevicePlan)
    g = int(res["gpu_count"][s])
    p.__dict__.update(
        strategy="igniter", gpu_type=hw.gpu_type, cost_per_hour=g * hw.price_per_hour,
        diagnostics=[], _g=g,
        _arrays=(workloads, hw, g, res["gpu_of"][s], res["pos"][s], res["units"][s],
                 res["batch"][s], res["lb"][s], res["pred"][s]))
    return p


def _raise_plan_error(rec, workloads, hw, b_max):
    code = int(rec["code"])
    w = int(rec["workload"])
    spec = workloads[w][0] if w >= 0 else None
    raise native_exception(code, float(rec["a"]), float(rec["b"]), float(rec["c"]),
                           spec=spec, hw=hw, b_max=b_max)


def plan(
    workloads: Sequence[tuple[WorkloadSpec, WorkloadCoefficients]],
    hw: HardwareProfile,
    *,
    b_max: int = DEFAULT_BATCH_CAP,
    stats: PlanStats | None = None,
) -> Plan:
    """Greedy minimum-interference provisioning (Alg. 1, planner.py:258-325).

    Workloads are placed in descending order of their solo lower bound (names
    break ties); each goes to the open device whose joint reallocation (Alg. 2)
    adds the fewest units, lowest index on ties, else to a new device.  With
    ``stats`` the device runs the reference's exact evaluation sequence and
    the counters match the reference's PlanStats bit for bit."""
    _check_unique_names(workloads)
    m = len(workloads)
    wl = workload_table(workloads)
    rank = name_ranks([s.name for s, _ in workloads])
    flags = IGP_F_STATS if stats is not None else 0
    if m >= CTA_MIN_WORKLOADS:
        flags |= IGP_F_CTA  # one CTA per plan: many warps share each step's candidates
    if stats is None and m < COOP_MIN_WORKLOADS:
        # the search state in shared memory, one warp per candidate (csrc/smem_plan.cuh;
        # the library uses the per-CTA kernel when it does not fit): C2 (1k) 5.4 vs
        # 9.8 ms, 300 workloads 1.25 vs 2.5 ms (one CTA) / 3.0 ms (one warp)
        flags |= IGP_F_SMEM | IGP_F_CTA
    if m >= COOP_MIN_WORKLOADS:
        # every warp of the GPU shares each step; the device falls back to the
        # per-CTA kernel when the exact sequence is needed (stats, raising input)
        flags |= IGP_F_COOP | IGP_F_CTA
    res = _device.plan_device(wl, hw_vector(hw), b_max, rank, flags=flags)
    rec = res["err"][0]
    if stats is not None:
        stats.model_evals += int(res["stats"][0][0])
        stats.candidate_gpus += int(res["stats"][0][1])
    if int(rec["code"]):
        _raise_plan_error(rec, workloads, hw, b_max)
    return _plan_from_arrays(res, 0, workloads, hw)


def _cta_per_scenario(S: int, m: int, device=None) -> bool:
    """One CTA per scenario while the batch fits in one or two waves over the
    SMs (B200, measured: 16 x 1k 10.3 vs 16.5 ms, 148 x 1k 11.0 vs 18.5 ms,
    148 x 10k 176 vs 726 ms; one warp per scenario wins from 296 x 1k on)."""
    if m < CTA_MIN_WORKLOADS:
        return False
    sms = _device.sm_count(device)
    return S <= sms or (m >= COOP_MIN_WORKLOADS and S <= 2 * sms)


def plan_many(scenarios, hw: HardwareProfile, *, b_max: int = DEFAULT_BATCH_CAP,
              stats: list | None = None, devices=None) -> list:
    """Plan independent scenarios (lists of (spec, coef) of equal length) in
    one launch per device: one warp per scenario, or one CTA per scenario for
    small batches of large scenarios.  ``devices`` (e.g. ``["cuda:0",
    "cuda:1"]``) splits the batch into contiguous blocks planned concurrently,
    one host thread per device (scenarios are independent, no
    collective).  Returns a list with a Plan or the exception instance the
    reference would raise for each scenario."""
    if not scenarios:
        return []
    m = len(scenarios[0])
    assert all(len(sc) == m for sc in scenarios), "scenarios must have equal workload counts"
    for sc in scenarios:
        _check_unique_names(sc)
    if stats is not None:
        assert len(stats) == len(scenarios)
    devices = list(devices) if devices else [None]
    from .shard import shard_bounds
    blocks = [shard_bounds(len(scenarios), r, len(devices)) for r in range(len(devices))]

    def run(r):
        a, b = blocks[r]
        if a == b:
            return []
        return _plan_block(scenarios[a:b], hw, b_max, None if stats is None else stats[a:b],
                           devices[r])

    if len(devices) == 1:
        return run(0)
    with ThreadPoolExecutor(len(devices)) as ex:
        parts = list(ex.map(run, range(len(devices))))
    return [p for part in parts for p in part]


def _plan_block(scenarios, hw, b_max, stats, device):
    m = len(scenarios[0])
    wl = np.stack([workload_table(sc) for sc in scenarios])
    rank = np.stack([name_ranks([s.name for s, _ in sc]) for sc in scenarios])
    flags = IGP_F_STATS if stats is not None else 0
    if _cta_per_scenario(len(scenarios), m, device):
        flags |= IGP_F_CTA
        if stats is None:
            flags |= IGP_F_SMEM  # shared-memory state per CTA when it fits
    res = _device.plan_device(wl, hw_vector(hw), b_max, rank, flags=flags, device=device)
    out = []
    for s, sc in enumerate(scenarios):
        if stats is not None:
            stats[s].model_evals += int(res["stats"][s][0])
            stats[s].candidate_gpus += int(res["stats"][s][1])
        rec = res["err"][s]
        if int(rec["code"]):
            try:
                _raise_plan_error(rec, sc, hw, b_max)
            except Exception as exc:  # noqa: BLE001 - returned, not swallowed
                out.append(exc)
            continue
        out.append(_plan_from_arrays(res, s, sc, hw))
    return out


def plan_cost(p: Plan, hw: HardwareProfile) -> float:
    """Devices times unit price (planner.py:328-330)."""
    return len(p.gpus) * hw.price_per_hour


def select_gpu_type(
    workloads: Sequence[WorkloadSpec],
    profiles: Sequence[HardwareProfile],
    coefs_by_type: Mapping[str, Mapping[str, WorkloadCoefficients]],
    *,
    b_max: int = DEFAULT_BATCH_CAP,
) -> Plan:
    """Cheapest plan over GPU types, first profile on ties; infeasible types
    are skipped (planner.py:333-364).

    Every type is one scenario of ONE device launch (IGP_F_HWS: one hardware
    profile per scenario, each with its own coefficient table); the
    reference's sequential semantics are then replayed on the results in
    profile order: a missing coefficient table raises ValueError when its
    type is reached, a non-planning error (NonPositiveDenominatorError, ...)
    of an earlier type propagates first, and planning errors skip the type."""
    tables, missing = [], None
    for t, hw in enumerate(profiles):
        try:
            coefs = coefs_by_type[hw.gpu_type]
            tables.append(workload_table([(s, coefs[s.name]) for s in workloads]))
        except KeyError as exc:
            missing = (t, hw, exc)
            break
    res = None
    if tables:
        _check_unique_names([(s, None) for s in workloads])  # the first type's plan() check
        n = len(tables)
        rank = name_ranks([s.name for s in workloads])
        hv = np.stack([np.asarray(hw_vector(hw), np.float64) for hw in profiles[:n]])
        if n <= _device.sm_count():
            # one CTA per type with the search state in shared memory (the library
            # falls back to the per-CTA kernel when it does not fit): 4 types x 1k
            flags = IGP_F_SMEM | IGP_F_CTA
        else:
            flags = IGP_F_CTA if _cta_per_scenario(n, len(workloads)) else 0
        res = _device.plan_device(np.stack(tables), hv, b_max, rank, flags=flags)
    best: Plan | None = None
    last_error: Exception | None = None
    for t in range(len(tables)):
        hw = profiles[t]
        coefs = coefs_by_type[hw.gpu_type]
        pairs = [(s, coefs[s.name]) for s in workloads]
        rec = res["err"][t]
        if int(rec["code"]):
            try:
                _raise_plan_error(rec, pairs, hw, b_max)
            except (InfeasibleSloError, InfeasibleResourceError, BatchCapExceededError) as exc:
                last_error = exc
                continue
        candidate = _plan_from_arrays(res, t, pairs, hw)
        if best is None or candidate.cost_per_hour < best.cost_per_hour:
            best = candidate
    if missing is not None:
        t, hw, exc = missing
        raise ValueError(f"missing coefficients for GPU type {hw.gpu_type}: {exc}") from exc
    if best is None:
        raise InfeasibleError(f"no GPU type can host all workloads ({last_error})")
    return best
