"""Exception hierarchy of the drop-in surface.

Names, base classes and constructor signatures match the reference's
``gpuplanner.errors`` (``errors.py:4-68``) so ``except`` clauses written
against the reference keep working.  The native library reports failures as
``IGP_E_*`` codes plus operands (include/igniter_b200.h); ``raise_native``
turns one such record into the exception the reference raises, with the
reference's message text.
"""

from __future__ import annotations


class GpuPlannerError(Exception):
    """Root of every error raised by this package."""


class NonPositiveDenominatorError(GpuPlannerError):
    """r + k4 (or the resulting active time) is not positive."""


class OverAllocatedError(GpuPlannerError):
    """A device's summed resource fractions exceed r_max."""


class InsufficientDataError(GpuPlannerError):
    """Calibration input too small (kept for API parity; calibration is out of scope)."""


class DegenerateDesignError(GpuPlannerError):
    """Rank-deficient regression design (API parity only)."""


class ZeroVarianceError(GpuPlannerError):
    """Constant regressor (API parity only)."""


class PlanningError(GpuPlannerError):
    """A workload cannot be provisioned; ``.workload`` names it."""

    def __init__(self, workload: str, message: str):
        self.workload = workload
        super().__init__(f"{workload}: {message}")


class InfeasibleSloError(PlanningError):
    """Fixed latency terms already exhaust the half-SLO budget."""


class InfeasibleResourceError(PlanningError):
    """Even the whole device is below the solo resource lower bound."""


class BatchCapExceededError(PlanningError):
    """The arrival rate needs a batch beyond the cap."""


class InfeasibleError(GpuPlannerError):
    """No candidate satisfies the constraints."""


class BudgetExceededError(GpuPlannerError):
    """Enumeration budget exhausted (API parity only)."""


class UnstableQueueError(GpuPlannerError):
    """Simulated queue grew beyond bound; the offered rate is not sustainable."""

    def __init__(self, workload: str, depth: int, bound: int):
        self.workload = workload
        self.depth = depth
        super().__init__(f"{workload}: queue depth {depth} exceeds {bound} at horizon end")


class ProblemFormatError(GpuPlannerError):
    """Malformed input document (API parity only)."""


def _reference_errors():
    """The reference's ``gpuplanner.errors`` module when it is importable in
    this process and is not this package under an alias, else None."""
    import importlib
    import importlib.util
    import os
    import sys
    if os.environ.get("IGP_OWN_ERRORS"):
        return None
    here = os.path.dirname(os.path.abspath(__file__))
    mod = sys.modules.get("gpuplanner.errors")
    if mod is None:
        top = sys.modules.get("gpuplanner")
        if top is not None and os.path.dirname(os.path.abspath(getattr(top, "__file__", "") or
                                                                "/")) == here:
            return None
        try:
            spec = importlib.util.find_spec("gpuplanner")
        except (ImportError, ValueError):
            return None
        if spec is None or (spec.origin and os.path.dirname(os.path.abspath(spec.origin)) == here):
            return None
        try:
            mod = importlib.import_module("gpuplanner.errors")
        except Exception:  # noqa: BLE001 - a broken reference install: keep our own classes
            return None
    path = getattr(mod, "__file__", None)
    if not path or os.path.dirname(os.path.abspath(path)) == here:
        return None
    return mod


# When the reference package is importable, its exception classes ARE this
# package's: `except gpuplanner.errors.PlanningError` written against the
# reference keeps catching what this package raises (class identity, not just
# names).  Our definitions above are the same hierarchy for when it is not.
_REF = _reference_errors()
if _REF is not None:
    for _n in ("GpuPlannerError", "NonPositiveDenominatorError", "OverAllocatedError",
               "InsufficientDataError", "DegenerateDesignError", "ZeroVarianceError",
               "PlanningError", "InfeasibleSloError", "InfeasibleResourceError",
               "BatchCapExceededError", "InfeasibleError", "BudgetExceededError",
               "UnstableQueueError", "ProblemFormatError"):
        if hasattr(_REF, _n):
            globals()[_n] = getattr(_REF, _n)


class NativeError(GpuPlannerError):
    """The CUDA library failed for a reason that has no reference counterpart."""


# IGP_E_* codes (include/igniter_b200.h)
E_OK, E_BATCH_CAP, E_INFEASIBLE_SLO, E_INFEASIBLE_RES = 0, 1, 2, 3
E_DENOM, E_ACTIVE_TIME, E_OVERALLOC, E_CAPACITY, E_CUDA, E_ARG = 4, 5, 6, 7, 8, 9


def native_exception(code, a, b, c, *, spec=None, hw=None, b_max=None, detail=""):
    """Build the reference exception for a native error record.

    Message templates follow the reference raise sites:
    planner.py:87-91, :107-111, :115-119; model.py:178-183, :286-290, :331-335.
    """
    if code == E_BATCH_CAP:
        return BatchCapExceededError(
            spec.name,
            f"needs batch {int(a)} > cap {b_max}; a single replica cannot meet "
            f"{spec.rate_rps} req/s within {spec.slo_ms} ms",
        )
    if code == E_INFEASIBLE_SLO:
        return InfeasibleSloError(
            spec.name, f"latency budget exhausted by fixed terms (delta={a:.6f} ms)")
    if code == E_INFEASIBLE_RES:
        return InfeasibleResourceError(
            spec.name, f"needs {int(a) * hw.r_unit:.3f} of a device even running alone")
    if code == E_DENOM:
        return NonPositiveDenominatorError(
            f"r + k4 = {a} must be positive (r={b}, k4={c})")
    if code == E_ACTIVE_TIME:
        return NonPositiveDenominatorError(
            f"active time {a} ms at (batch={int(b)}, r={c}) must be positive; "
            f"coefficients are corrupt")
    if code == E_OVERALLOC:
        return OverAllocatedError(f"allocated {a:.6f} exceeds r_max {hw.r_max}")
    return NativeError(f"native error code {code}{': ' + detail if detail else ''}")
