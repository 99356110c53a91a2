"""ctypes binding of libigniter_b200.so for the reference package (include/igniter_b200.h).

The file a maintainer drops into the reference as ``gpuplanner/_b200.py``
("Reference-side binding").  It depends only on numpy and
ctypes -- no torch -- and on sibling modules of the package it is installed
in (``.model``, ``.planner``, ``.errors``) for the result and exception
classes, so ``plan()`` below returns the reference's own ``Plan`` objects.

    from gpuplanner import _b200
    p = _b200.plan(workloads, hw, b_max=32, stats=None)   # == gpuplanner.plan

Replaces the computation of ``plan`` (planner.py:258-325): the prologue
(:280-282), the (-lb, name) sort (:284), Alg. 1 with Alg. 2 per candidate
(:290-319, :133-162) and the ``_build_plan`` predictions (:218-246) run in
``igp_plan_batch_host``; this module only marshals arrays and assembles the
reference's result objects (planner.py:218-246).
"""

import ctypes
import os

import numpy as np

IGP_F_STATS = 1
IGP_F_CTA = 4
IGP_F_COOP = 16

WL_FIELDS = ("slo_ms", "rate_rps", "d_load_mb", "d_feedback_mb")
COEF_FIELDS = ("n_kernels", "k_sch_ms", "k1", "k2", "k3", "k4", "k5", "alpha_power_w",
               "beta_power_w", "alpha_cacheutil", "beta_cacheutil", "alpha_cache")
HW_FIELDS = ("power_max_w", "freq_max_mhz", "power_idle_w", "pcie_bw_mb_per_ms", "alpha_f",
             "alpha_sch_ms", "beta_sch_ms", "r_unit", "r_max", "price_per_hour", "f_min_frac")


class IgpError(ctypes.Structure):
    _fields_ = [("code", ctypes.c_int32), ("workload", ctypes.c_int32),
                ("gpu", ctypes.c_int32), ("pad", ctypes.c_int32),
                ("a", ctypes.c_double), ("b", ctypes.c_double), ("c", ctypes.c_double)]


_lib = None


def lib():
    """libigniter_b200.so from $IGP_LIB (else the dynamic loader's search path)."""
    global _lib
    if _lib is None:
        L = ctypes.CDLL(os.environ.get("IGP_LIB", "libigniter_b200.so"))
        vp, i, sz = ctypes.c_void_p, ctypes.c_int, ctypes.c_size_t
        L.igp_plan_batch_host.restype = i
        L.igp_plan_batch_host.argtypes = [vp, i, i, vp, i, vp, i] + [vp] * 10 + [sz, i, vp]
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def plan_arrays(workloads, hw, b_max=32, flags=0):
    """One plan on the GPU; per-workload arrays in input order plus the
    GPU count, the PlanStats counters and the error record."""
    m = len(workloads)
    wl = np.empty((16, m))
    for k, (s, c) in enumerate(workloads):
        wl[:, k] = [float(getattr(s, f)) for f in WL_FIELDS] + \
                   [float(getattr(c, f)) for f in COEF_FIELDS]
    names = [s.name for s, _ in workloads]
    rank = np.empty(m, np.int32)
    rank[np.array(sorted(range(m), key=names.__getitem__), dtype=np.int64)] = \
        np.arange(m, dtype=np.int32)
    h = np.array([float(getattr(hw, f)) for f in HW_FIELDS])
    out = {k: np.empty(max(m, 1), np.int32) for k in ("gpu_of", "pos", "units", "batch", "lb")}
    pred = np.empty((max(m, 1), 10))
    gc = np.zeros(1, np.int32)
    st = np.zeros(6, np.int64)
    err = IgpError()
    # workspace NULL / 0 bytes: the library allocates it on the (default) stream
    rc = lib().igp_plan_batch_host(_p(wl), 1, m, _p(h), int(b_max), _p(rank), 0,
                                   _p(out["gpu_of"]), _p(out["pos"]), _p(out["units"]),
                                   _p(out["batch"]), _p(out["lb"]), _p(pred), _p(gc), _p(st),
                                   ctypes.byref(err), None, 0, int(flags), None)
    return rc, err, out, pred, int(gc[0]), st


def _exception(err, workloads, hw, b_max):
    from . import errors as E  # the host package's exception classes
    code = err.code
    spec = workloads[err.workload][0] if err.workload >= 0 else None
    if code == 1:
        return E.BatchCapExceededError(
            spec.name, f"needs batch {int(err.a)} > cap {b_max}; a single replica cannot meet "
                       f"{spec.rate_rps} req/s within {spec.slo_ms} ms")
    if code == 2:
        return E.InfeasibleSloError(
            spec.name, f"latency budget exhausted by fixed terms (delta={err.a:.6f} ms)")
    if code == 3:
        return E.InfeasibleResourceError(
            spec.name, f"needs {int(err.a) * hw.r_unit:.3f} of a device even running alone")
    if code == 4:
        return E.NonPositiveDenominatorError(
            f"r + k4 = {err.a} must be positive (r={err.b}, k4={err.c})")
    if code == 5:
        return E.NonPositiveDenominatorError(
            f"active time {err.a} ms at (batch={int(err.b)}, r={err.c}) must be positive; "
            "coefficients are corrupt")
    if code == 6:
        return E.OverAllocatedError(f"allocated {err.a:.6f} exceeds r_max {hw.r_max}")
    return RuntimeError(f"libigniter_b200 error {code}")


def plan(workloads, hw, *, b_max=32, stats=None):
    """Drop-in body of gpuplanner.plan (planner.py:258-325) on the GPU."""
    from .model import Allocation, LatencyBreakdown
    from .planner import GpuPlan, Plan, _check_unique_names
    _check_unique_names(workloads)  # planner.py:273 (ValueError on duplicates)
    m = len(workloads)
    flags = IGP_F_STATS if stats is not None else 0
    if m >= 512:
        flags |= IGP_F_CTA
    rc, err, out, pred, g, st = plan_arrays(workloads, hw, b_max, flags)
    if stats is not None:
        stats.model_evals += int(st[0])
        stats.candidate_gpus += int(st[1])
    if err.code:
        raise _exception(err, workloads, hw, b_max)
    if rc:
        raise RuntimeError(f"libigniter_b200 rejected the call ({rc})")
    cap = int(round(hw.r_max / hw.r_unit))
    members = [[] for _ in range(g)]
    for i in np.lexsort((out["pos"][:m], out["gpu_of"][:m])):
        members[out["gpu_of"][i]].append(int(i))
    gpus, r_inter = [], {}
    for j, mem in enumerate(members):
        allocations, predicted, used = [], {}, 0
        for i in mem:
            name, u = workloads[i][0].name, int(out["units"][i])
            used += u
            allocations.append(Allocation(name, u * hw.r_unit, int(out["batch"][i])))
            predicted[name] = LatencyBreakdown(*(float(v) for v in pred[i]))
            r_inter[name] = (u - int(out["lb"][i])) * hw.r_unit
        gpus.append(GpuPlan(j, allocations, predicted, (cap - used) * hw.r_unit))
    return Plan(strategy="igniter", gpu_type=hw.gpu_type, gpus=gpus,
                cost_per_hour=len(gpus) * hw.price_per_hour, per_workload_r_inter=r_inter)
