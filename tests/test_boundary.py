"""The drop-in boundary, seen from the reference's side.

* Exception identity: when the reference package ``gpuplanner`` is importable,
  this package raises the reference's own exception classes, so
  ``except gpuplanner.errors.PlanningError`` keeps catching (errors.py).
* The reference-side ctypes stub (integration/_b200.py, shown in
  INTEGRATION.md): installed into a temporary copy of the reference package
  it imports and binds the library (CPU, needs /root/reference); on the B200
  its ``plan()`` reproduces the reference-generated plan fixtures and raises
  the reference's exceptions (GPU; the stub's sibling modules are this
  package's API-identical ones, since the reference source does not travel).
"""
import os
import shutil
import subprocess
import sys
import textwrap

import numpy as np
import pytest

import golden_io as G
from instances import hw_from_golden, workloads_from_golden

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_SRC = "/root/reference/pkg/src"
STUB = os.path.join(REPO, "integration", "_b200.py")
LIB = os.path.join(REPO, "paper_2211_01713_b200", "_lib", "libigniter_b200.so")
needs_ref = pytest.mark.skipif(not os.path.isdir(os.path.join(REF_SRC, "gpuplanner")),
                               reason="reference source not present (GPU box)")


def _run(code, env_extra):
    env = dict(os.environ, **env_extra)
    r = subprocess.run([sys.executable, "-c", textwrap.dedent(code)], env=env,
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    return r.stdout


@needs_ref
def test_exception_classes_are_the_references():
    out = _run("""
        import gpuplanner.errors as ref
        import paper_2211_01713_b200 as igp
        from paper_2211_01713_b200 import errors, planner
        names = ["GpuPlannerError", "PlanningError", "InfeasibleSloError",
                 "InfeasibleResourceError", "BatchCapExceededError",
                 "NonPositiveDenominatorError", "OverAllocatedError", "InfeasibleError",
                 "BudgetExceededError", "UnstableQueueError"]
        assert all(getattr(errors, n) is getattr(ref, n) for n in names)
        assert planner.InfeasibleSloError is ref.InfeasibleSloError
        assert issubclass(errors.NativeError, ref.GpuPlannerError)
        e = errors.native_exception(2, 0.5, 0.0, 0.0, spec=igp.WorkloadSpec("w", 1, 1, 0, 0))
        try:
            raise e
        except ref.PlanningError as caught:
            print("caught", type(caught).__module__, caught.workload)
    """, {"PYTHONPATH": f"{REPO}:{REF_SRC}"})
    assert "caught gpuplanner.errors w" in out


def test_exception_classes_standalone_without_reference():
    out = _run("""
        import sys
        sys.modules["gpuplanner"] = None  # reference not importable
        from paper_2211_01713_b200 import errors
        assert errors._REF is None
        assert errors.PlanningError.__module__ == "paper_2211_01713_b200.errors"
        print("own")
    """, {"PYTHONPATH": REPO})
    assert "own" in out


@needs_ref
def test_stub_installs_into_a_copy_of_the_reference(tmp_path):
    from paper_2211_01713_b200 import _native
    _native.build()
    dst = tmp_path / "gpuplanner"
    shutil.copytree(os.path.join(REF_SRC, "gpuplanner"), dst)
    shutil.copy(STUB, dst / "_b200.py")
    out = _run("""
        import gpuplanner
        from gpuplanner import _b200
        L = _b200.lib()
        assert L.igp_plan_batch_host and L.igp_plan_host_workspace_bytes
        assert L.igp_abi_version() == 1
        from gpuplanner.planner import GpuPlan, Plan, _check_unique_names  # what the stub uses
        from gpuplanner.model import Allocation, LatencyBreakdown
        print("stub bound", _b200.HW_FIELDS[-1])
    """, {"PYTHONPATH": str(tmp_path), "IGP_LIB": LIB})
    assert "stub bound f_min_frac" in out


def _stub_host_package(tmp_path):
    """A package holding the stub as `_b200`, its siblings re-exporting this
    package's API-identical model / planner / errors modules."""
    pkg = tmp_path / "stubhost"
    pkg.mkdir()
    (pkg / "__init__.py").write_text("")
    for mod in ("model", "planner", "errors"):
        (pkg / f"{mod}.py").write_text(
            f"from paper_2211_01713_b200.{mod} import *  # noqa\n"
            f"from paper_2211_01713_b200.{mod} import __dict__ as _d\n"
            "globals().update({k: v for k, v in _d.items() if not k.startswith('__')})\n")
    shutil.copy(STUB, pkg / "_b200.py")
    sys.path.insert(0, str(tmp_path))
    import importlib
    return importlib.import_module("stubhost._b200")


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["plan_c1_twelve", "plan_rand1k_seed7", "plan_rand600_r01",
                                  "plan_err_slo", "plan_err_denom"])
def test_stub_plan_matches_reference_fixtures(tmp_path, monkeypatch, case):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2211_01713_b200 import PlanStats, _native, errors
    _native.load()
    monkeypatch.setenv("IGP_LIB", LIB)
    stub = _stub_host_package(tmp_path)
    d = G.load(case)
    wls, hw = workloads_from_golden(d), hw_from_golden(d)
    stats = PlanStats()
    if str(d["err_class"]):
        with pytest.raises(errors.GpuPlannerError) as ei:
            stub.plan(wls, hw, b_max=int(d["b_max"]), stats=stats)
        assert type(ei.value).__name__ == str(d["err_class"])
        assert str(ei.value) == str(d["err_msg"])
        return
    p = stub.plan(wls, hw, b_max=int(d["b_max"]), stats=stats)
    assert p.gpu_count == int(d["gpu_count"])
    assert stats.model_evals == int(d["model_evals"])
    assert stats.candidate_gpus == int(d["candidate_gpus"])
    idx = {s.name: i for i, (s, _) in enumerate(wls)}
    for g in p.gpus:
        for k, a in enumerate(g.allocations):
            i = idx[a.workload]
            assert (g.gpu_index, k, a.batch) == (int(d["gpu_of"][i]), int(d["pos"][i]),
                                                 int(d["batch"][i]))
            assert a.r == float(d["r"][i])
            assert np.float64(g.predicted[a.workload].t_inf_ms).view(np.int64) == \
                G.bits(d["pred"][i, 6])
    assert p.cost_per_hour == float(d["cost"])


def test_entry_exposes_the_reference_constants():
    """_Entry keeps the reference's attributes (model.py:239-270) bit for bit."""
    import sys
    sys.path.insert(0, "/root/reference/pkg/src")
    gm = pytest.importorskip("gpuplanner.model")
    from paper_2211_01713_b200 import model as mm
    from instances import make_v100, random_instance
    import numpy as np
    hw = make_v100()
    for spec, coef in random_instance(np.random.default_rng(3), 20, hw):
        b = 1 + len(spec.name) % 7
        ours, ref = mm._Entry(spec, coef, b, hw), gm._Entry(spec, coef, b, hw)
        for a in gm._Entry.__slots__:
            assert getattr(ours, a) == getattr(ref, a), a
