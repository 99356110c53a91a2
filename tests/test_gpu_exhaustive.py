"""Exhaustive oracle on the GPU (igp_group_search_device + exhaustive_plan)
against the reference's exhaustive_plan fixtures and the CPU oracle, plus the
SPEC acceptance properties that need the oracle."""
import numpy as np
import pytest

import golden_io as G
from instances import hw_from_golden, make_v100, random_instance, workloads_from_golden

import paper_2211_01713_b200 as igp
from paper_2211_01713_b200 import errors
from paper_2211_01713_b200.exhaustive import OracleBudget, exhaustive_plan, group_search

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.parametrize("case", G.names("oracle_"))
def test_exhaustive_plan_matches_reference(case):
    d = G.load(case)
    wls = workloads_from_golden(d)
    hw = hw_from_golden(d)
    budget = OracleBudget(max_gpus=int(d["max_gpus"]),
                          r_grid_units=tuple(int(x) for x in d["grid"]) or None)
    if str(d["err_class"]):
        with pytest.raises(errors.GpuPlannerError) as ei:
            exhaustive_plan(wls, hw, budget=budget, b_max=int(d["b_max"]))
        assert type(ei.value).__name__ == str(d["err_class"])
        assert str(ei.value) == str(d["err_msg"])
        return
    p = exhaustive_plan(wls, hw, budget=budget, b_max=int(d["b_max"]))
    assert p.strategy == "oracle" and len(p.gpus) == int(d["gpu_count"])
    idx = {s.name: i for i, (s, _) in enumerate(wls)}
    for g in p.gpus:
        for a in g.allocations:
            i = idx[a.workload]
            assert g.gpu_index == int(d["gpu_of"][i])
            assert int(round(a.r / hw.r_unit)) == int(d["units"][i])
            bd = g.predicted[a.workload]
            row = [bd.t_load_ms, bd.t_sch_ms, bd.t_act_ms, bd.freq_mhz, bd.t_gpu_ms,
                   bd.t_feedback_ms, bd.t_inf_ms, bd.throughput_rps, bd.power_w, bd.cache_util]
            np.testing.assert_array_equal(G.bits(row), G.bits(d["pred"][i]))
    assert p.cost_per_hour == float(d["cost"])


@pytest.mark.parametrize("r_unit,n", [(0.01, 4), (0.025, 6)])
def test_group_search_vs_cpu_oracle(oracle_lib, r_unit, n):
    hw = make_v100(r_unit=r_unit)
    rng = np.random.default_rng(4242)
    from paper_2211_01713_b200.layout import hw_vector, spec_coef_row
    for _ in range(3):
        inst = random_instance(rng, n, hw)
        specs = {s.name: s for s, _ in inst}
        coefs = {s.name: c for s, c in inst}
        names = sorted(specs)
        batches = {nm: igp.appropriate_batch(specs[nm], hw) for nm in names}
        cap = igp.max_units(hw)
        grid = list(range(1, cap + 1))
        dev = group_search(specs, coefs, batches, names, hw, grid)
        wl = np.array([spec_coef_row(specs[nm], coefs[nm]) for nm in names]).T.copy()
        best, rc = oracle_lib.group_search(wl, np.array([batches[nm] for nm in names]),
                                           np.array(hw_vector(hw)), np.array(grid))
        assert rc == 0
        from paper_2211_01713_b200.exhaustive import decode_keys
        assert dev == decode_keys(best, len(names))


def test_spec_acceptance_4_theorem1_tightness():
    """for 200 seeded random feasible workloads the oracle's
    single-workload optimum equals lower_bound_resources (grid scan), and one
    unit less violates the half-SLO."""
    hw = make_v100()
    rng = np.random.default_rng(478)
    inst = random_instance(rng, 200, hw)
    matches = 0
    for spec, coef in inst:
        p = exhaustive_plan([(spec, coef)], hw)
        b = igp.appropriate_batch(spec, hw)
        lb = igp.lower_bound_resources(spec, coef, hw, b)
        a = p.gpus[0].allocations[0]
        matches += abs(a.r - lb) < 1e-12
        if a.r > hw.r_unit:
            below = igp.predict_gpu([igp.Allocation(spec.name, a.r - hw.r_unit, b)],
                                    {spec.name: spec}, {spec.name: coef}, hw)[spec.name]
            chk = igp.slo_check(below, spec)
            assert not (chk.latency_ok and chk.throughput_ok)
    assert matches == 200


def test_spec_acceptance_5_oracle_gap():
    """on 100 seeded instances of <= 3 workloads the greedy plan
    is feasible, matches the oracle's GPU count on >= 80% and never uses
    fewer GPUs than the oracle."""
    hw = make_v100()
    rng = np.random.default_rng(479)
    same = 0
    for t in range(100):
        inst = random_instance(rng, 1 + t % 3, hw)
        o = exhaustive_plan(inst, hw)
        g = igp.plan(inst, hw)
        assert len(g.gpus) >= len(o.gpus)
        same += len(g.gpus) == len(o.gpus)
        specs = {s.name: s for s, _ in inst}
        for gp in g.gpus:
            for a in gp.allocations:
                assert igp.slo_check(gp.predicted[a.workload], specs[a.workload]).latency_ok
    assert same >= 80
