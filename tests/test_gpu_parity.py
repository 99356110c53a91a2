"""CUDA path vs the reference (golden fixtures) and vs the CPU oracle.

Every comparison is bit-exact: placements, units, batches, lower bounds,
PlanStats and the fp64 breakdown rows (compared as int64 bit patterns; the
north_star tolerance of 1e-9 relative is therefore met with margin 0).
"""
import numpy as np
import pytest

import golden_io as G
from instances import (c3_instance, hw_from_golden, make_v100, random_instance,
                       twelve_workload_instance, workloads_from_golden)

import paper_2211_01713_b200 as igp
from paper_2211_01713_b200 import _device, errors
from paper_2211_01713_b200.layout import hw_vector
from paper_2211_01713_b200.planner import (IGP_F_COOP, IGP_F_CTA, IGP_F_STATS, name_ranks,
                                           workload_table)

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2211_01713_b200 import _native
    _native.load()


def _plan_arrays_from_plan(p, workloads, r_unit):
    idx = {s.name: i for i, (s, _) in enumerate(workloads)}
    m = len(workloads)
    gpu_of = np.full(m, -1, np.int32)
    pos = np.full(m, -1, np.int32)
    units = np.zeros(m, np.int32)
    batch = np.zeros(m, np.int32)
    pred = np.zeros((m, 10))
    for g in p.gpus:
        for k, a in enumerate(g.allocations):
            i = idx[a.workload]
            gpu_of[i], pos[i], batch[i] = g.gpu_index, k, a.batch
            units[i] = int(round(a.r / r_unit))
            bd = g.predicted[a.workload]
            pred[i] = [bd.t_load_ms, bd.t_sch_ms, bd.t_act_ms, bd.freq_mhz, bd.t_gpu_ms,
                       bd.t_feedback_ms, bd.t_inf_ms, bd.throughput_rps, bd.power_w, bd.cache_util]
    return gpu_of, pos, units, batch, pred


@pytest.mark.parametrize("with_stats", [True, False])
@pytest.mark.parametrize("case", G.names("plan_"))
def test_plan_api_matches_reference_golden(case, with_stats):
    d = G.load(case)
    wls = workloads_from_golden(d)
    hw = hw_from_golden(d)
    stats = igp.PlanStats() if with_stats else None
    if str(d["err_class"]):
        with pytest.raises(errors.GpuPlannerError) as ei:
            igp.plan(wls, hw, b_max=int(d["b_max"]), stats=stats)
        assert type(ei.value).__name__ == str(d["err_class"])
        assert str(ei.value) == str(d["err_msg"])
        if with_stats:
            assert stats.model_evals == int(d["model_evals"])
            assert stats.candidate_gpus == int(d["candidate_gpus"])
        return
    p = igp.plan(wls, hw, b_max=int(d["b_max"]), stats=stats)
    gpu_of, pos, units, batch, pred = _plan_arrays_from_plan(p, wls, hw.r_unit)
    np.testing.assert_array_equal(gpu_of, d["gpu_of"])
    np.testing.assert_array_equal(pos, d["pos"])
    np.testing.assert_array_equal(units, d["units"])
    np.testing.assert_array_equal(batch, d["batch"])
    np.testing.assert_array_equal(G.bits(pred), G.bits(d["pred"]))
    assert p.cost_per_hour == float(d["cost"])
    np.testing.assert_array_equal(G.bits([g.fragment_r for g in p.gpus]), G.bits(d["fragment"]))
    r_inter = np.array([p.per_workload_r_inter[s.name] for s, _ in wls])
    np.testing.assert_array_equal(G.bits(r_inter), G.bits(d["r_inter"]))
    for g in p.gpus:
        for a in g.allocations:
            i = [s.name for s, _ in wls].index(a.workload)
            assert a.r == float(d["r"][i])
    if with_stats:
        assert stats.model_evals == int(d["model_evals"])
        assert stats.candidate_gpus == int(d["candidate_gpus"])


@pytest.mark.parametrize("case", G.names("eval_states_"))
def test_eval_states_match_reference_rows(case):
    d = G.load(case)
    rows, err = _device.eval_states(d["wl"], d["batch"], d["r"], d["ptr"], d["hw"])
    assert (err["code"] == 0).all()
    np.testing.assert_array_equal(G.bits(rows), G.bits(d["rows"]))


@pytest.mark.parametrize("case", G.names("prologue_"))
def test_prologue_matches_reference(case):
    d = G.load(case)
    b, lb, code, err = _device.prologue(d["wl"], d["hw"], int(d["b_max"]))
    np.testing.assert_array_equal(code, d["code"])
    np.testing.assert_array_equal(b[code != 1], d["batch"][code != 1])
    np.testing.assert_array_equal(lb[code == 0], d["lb"][code == 0])
    first = np.nonzero(code)[0]
    assert int(err["workload"]) == (int(first[0]) if len(first) else -1)


def test_alloc_units_match_reference():
    d = G.load("alloc_v100")
    u, err = _device.alloc_units(d["wl"], d["batch"], d["r"], d["ptr"], d["hw"])
    assert (err["code"] == 0).all()
    np.testing.assert_array_equal(u, d["units"])


def _compare_to_oracle(res, s, wl, hw_vec, b_max, rank, oracle, stats=False):
    o = oracle.plan(wl, hw_vec, b_max, rank)
    assert o["rc"] == int(res["err"][s]["code"])
    if o["rc"]:
        return o
    for k in ("gpu_of", "pos", "units", "batch", "lb"):
        np.testing.assert_array_equal(res[k][s], o[k], err_msg=k)
    assert int(res["gpu_count"][s]) == o["gpu_count"]
    np.testing.assert_array_equal(G.bits(res["pred"][s]), G.bits(o["pred"]))
    if stats:
        assert int(res["stats"][s][0]) == o["model_evals"]
        assert int(res["stats"][s][1]) == o["candidate_gpus"]
        assert int(res["stats"][s][4]) == o["resident_reads"]
    return o


@pytest.mark.parametrize("flags", [0, IGP_F_STATS, IGP_F_CTA, IGP_F_CTA | IGP_F_STATS, 32, 64,
                                   64 | IGP_F_STATS])
def test_scenario_batch_vs_oracle(oracle_lib, flags):
    """Scenario batches in every group width: one warp (default), two / four
    warps (IGP_F_GW2 = 32, IGP_F_GW4 = 64) and one CTA per scenario."""
    hw = make_v100()
    rng = np.random.default_rng(123)
    scen = [random_instance(rng, 300, hw) for _ in range(12)]
    wl = np.stack([workload_table(sc) for sc in scen])
    rank = np.stack([name_ranks([s.name for s, _ in sc]) for sc in scen])
    res = _device.plan_device(wl, hw_vector(hw), 32, rank, flags=flags)
    for s in range(len(scen)):
        _compare_to_oracle(res, s, wl[s], np.array(hw_vector(hw)), 32, rank[s], oracle_lib,
                           stats=bool(flags & IGP_F_STATS))


def test_plan_many_matches_single_plans():
    hw = make_v100()
    rng = np.random.default_rng(5)
    scen = [random_instance(rng, 80, hw) for _ in range(6)]
    stats = [igp.PlanStats() for _ in scen]
    many = igp.plan_many(scen, hw, stats=stats)
    for sc, p, st in zip(scen, many, stats):
        st1 = igp.PlanStats()
        q = igp.plan(sc, hw, stats=st1)
        assert [[(a.workload, a.r, a.batch) for a in g.allocations] for g in p.gpus] == \
               [[(a.workload, a.r, a.batch) for a in g.allocations] for g in q.gpus]
        assert (st.model_evals, st.candidate_gpus) == (st1.model_evals, st1.candidate_gpus)


def test_plan_many_cta_path_vs_oracle(oracle_lib):
    """Few large scenarios take one CTA each (planner._cta_per_scenario)."""
    from paper_2211_01713_b200.planner import _cta_per_scenario
    hw = make_v100()
    rng = np.random.default_rng(77)
    scen = [random_instance(rng, 600, hw) for _ in range(3)]
    assert _cta_per_scenario(len(scen), 600)
    many = igp.plan_many(scen, hw)
    for sc, p in zip(scen, many):
        wl = workload_table(sc)
        r = oracle_lib.plan(wl, np.array(hw_vector(hw)), 32, name_ranks([s.name for s, _ in sc]))
        units = {a.workload: int(round(a.r / hw.r_unit)) for g in p.gpus for a in g.allocations}
        gpu_of = {a.workload: gi for gi, g in enumerate(p.gpus) for a in g.allocations}
        names = [s.name for s, _ in sc]
        assert [gpu_of[n] for n in names] == list(r["gpu_of"])
        assert [units[n] for n in names] == list(r["units"])


def test_r_unit_001_and_c3_generator_vs_oracle(oracle_lib):
    hw = make_v100(r_unit=0.01)
    rng = np.random.default_rng(2211)
    scen = [c3_instance(rng, 500, hw) for _ in range(4)]
    wl = np.stack([workload_table(sc) for sc in scen])
    rank = np.stack([name_ranks([s.name for s, _ in sc]) for sc in scen])
    for flags in (0, IGP_F_STATS, IGP_F_CTA):
        res = _device.plan_device(wl, hw_vector(hw), 128, rank, flags=flags)
        for s in range(len(scen)):
            _compare_to_oracle(res, s, wl[s], np.array(hw_vector(hw)), 128, rank[s], oracle_lib,
                               stats=bool(flags & IGP_F_STATS))


def test_full_size_10k_plan_vs_oracle(oracle_lib):
    """BASELINE metric size: one 10k-workload plan, bit-exact vs the oracle."""
    from paper_2211_01713_b200 import synth
    hw = make_v100()
    wl, names = synth.scenarios(1, 10_000, hw, seed=77)
    rank = name_ranks(list(names))
    for flags in (0, IGP_F_CTA):
        res = _device.plan_device(wl, hw_vector(hw), 32, rank, flags=flags)
        _compare_to_oracle(res, 0, wl[0], np.array(hw_vector(hw)), 32, rank, oracle_lib)


def test_reference_error_messages_and_types():
    hw = make_v100()
    spec = igp.WorkloadSpec("w", 200.0, 2000.0, 0.0, 0.0)
    with pytest.raises(errors.BatchCapExceededError, match="w"):
        igp.appropriate_batch(spec, hw)
    assert igp.appropriate_batch(spec, hw, b_max=512) == 200  # test_planner.py:64-66
    for slo, rate, exp in [(15.0, 500.0, 4), (40.0, 400.0, 8), (60.0, 200.0, 6)]:
        assert igp.appropriate_batch(igp.WorkloadSpec("w", slo, rate, 0.574, 0.004), hw) == exp
    coef = igp.WorkloadCoefficients(100, 0.002, 0.001, 0.05, 0.5, 0.05, 0.2, 50.0, 60.0, 0.05, 0.10, 0.25)
    assert igp.lower_bound_resources(igp.WorkloadSpec("resnet", 40.0, 400.0, 0.574, 0.004), coef, hw, 8) == 0.025
    assert igp.lower_bound_resources(igp.WorkloadSpec("w", 22.0, 400.0, 0.574, 0.004), coef, hw, 8) == 0.05
    with pytest.raises(errors.InfeasibleSloError, match="w"):
        igp.lower_bound_resources(igp.WorkloadSpec("w", 1.2, 400.0, 0.574, 0.004), coef, hw, 8)


def test_predict_gpu_known_values_and_overallocation():
    hw = make_v100()
    spec = igp.WorkloadSpec("resnet", 40.0, 400.0, 0.574, 0.004)
    coef = igp.WorkloadCoefficients(100, 0.002, 0.001, 0.05, 0.5, 0.05, 0.2, 50.0, 60.0, 0.05, 0.10, 0.25)
    bd = igp.predict_gpu([igp.Allocation("resnet", 0.025, 8)], {"resnet": spec}, {"resnet": coef}, hw)["resnet"]
    assert bd.t_gpu_ms == pytest.approx(13.253333333333334, rel=1e-12)   # test_model.py:153-160
    assert bd.t_inf_ms == pytest.approx(13.715733333333333, rel=1e-12)
    assert bd.freq_mhz == 1530.0
    assert bd.throughput_rps == pytest.approx(603.4760218860637, rel=1e-12)
    assert igp.predict_gpu([], {}, {}, hw) == {}
    other = igp.WorkloadSpec("other", 40.0, 400.0, 0.574, 0.004)
    with pytest.raises(errors.OverAllocatedError):
        igp.predict_gpu([igp.Allocation("resnet", 0.6, 8), igp.Allocation("other", 0.45, 8)],
                        {"resnet": spec, "other": other}, {"resnet": coef, "other": coef}, hw)
    bad = igp.WorkloadCoefficients(100, 0.002, 0.001, 0.05, 0.5, -0.5, 0.2, 50.0, 60.0, 0.05, 0.10, 0.25)
    with pytest.raises(errors.NonPositiveDenominatorError, match="r \\+ k4"):
        igp.predict_gpu([igp.Allocation("resnet", 0.3, 8)], {"resnet": spec}, {"resnet": bad}, hw)


def test_boundary_corunner_alloc():
    """test_planner.py:126-157: exact t_inf == t_half boundary."""
    hw = make_v100(alpha_sch_ms=0.0, beta_sch_ms=0.0)
    res_spec = igp.WorkloadSpec("resident", 40.0, 100.0, 0.0, 0.0)
    res_coef = igp.WorkloadCoefficients(1, 0.0, 0.0, 0.0, 10.0, 0.0, 0.0, 0.0, 10.0, 0.0, 0.0, 0.5)
    solo = igp.predict_gpu([igp.Allocation("resident", 0.5, 2)], {"resident": res_spec},
                           {"resident": res_coef}, hw)
    assert solo["resident"].t_inf_ms == 20.0
    new_spec = igp.WorkloadSpec("new", 40.0, 50.0, 0.0, 0.0)
    new_coef = igp.WorkloadCoefficients(1, 0.0, 0.0, 0.0, 0.5, 0.0, 0.0, 0.0, 10.0, 0.0, 0.3, 0.0)
    specs = {"resident": res_spec, "new": new_spec}
    coefs = {"resident": res_coef, "new": new_coef}
    result = igp.alloc_gpus(specs, coefs, hw, [igp.Allocation("resident", 0.5, 2)], "new", 1, 0.025)
    by = {a.workload: a for a in result}
    assert by["resident"].r > 0.5


def test_select_gpu_type_cheaper_type_wins():
    v100 = make_v100()
    t4 = igp.HardwareProfile("t4", 70.0, 1590.0, 10.0, 10.0, -1.0, 0.00475, -0.00902,
                             price_per_hour=0.526)

    def simple(name, k3):
        return (igp.WorkloadSpec(name, 40.0, 100.0, 0.0, 0.0),
                igp.WorkloadCoefficients(1, 0.0, 0.0, 0.0, k3, 0.0, 0.0, 0.0, 10.0, 0.0, 0.0, 0.0))
    specs = [simple(f"w{i:02d}", 9.9)[0] for i in range(15)]
    chosen = igp.select_gpu_type(specs, [v100, t4], {
        "v100": {s.name: simple(s.name, 9.9)[1] for s in specs},
        "t4": {s.name: simple(s.name, 19.8)[1] for s in specs}})
    assert chosen.gpu_type == "t4" and len(chosen.gpus) == 15
    assert round(chosen.cost_per_hour, 2) == 7.89


def test_twelve_workload_order_invariance():
    hw = make_v100()
    w = twelve_workload_instance()
    a = igp.plan(w, hw)
    b = igp.plan(list(reversed(w)), hw)
    assert [[(x.workload, x.r, x.batch) for x in g.allocations] for g in a.gpus] == \
           [[(x.workload, x.r, x.batch) for x in g.allocations] for g in b.gpus]


@pytest.mark.parametrize("case", G.names("plan_"))
@pytest.mark.parametrize("flags", [IGP_F_COOP, IGP_F_COOP | IGP_F_CTA, IGP_F_COOP | IGP_F_STATS])
def test_cooperative_single_plan_matches_reference_golden(case, flags):
    """Grid-cooperative single plan (and its device-side fallback for stats /
    raising inputs) against the reference fixtures."""
    d = G.load(case)
    rank = name_ranks([str(n) for n in d["names"]])
    res = _device.plan_device(d["wl"], d["hw"], int(d["b_max"]), rank, flags=flags)
    if str(d["err_class"]):
        assert int(res["err"][0]["code"]) == int(d["err_code"])
        return
    assert int(res["err"][0]["code"]) == 0
    for k in ("gpu_of", "pos", "units", "batch", "lb"):
        np.testing.assert_array_equal(res[k][0], d[k], err_msg=k)
    np.testing.assert_array_equal(G.bits(res["pred"][0]), G.bits(d["pred"]))
    if flags & IGP_F_STATS:
        assert int(res["stats"][0][0]) == int(d["model_evals"])
        assert int(res["stats"][0][1]) == int(d["candidate_gpus"])


def test_cooperative_10k_and_r01_vs_oracle(oracle_lib):
    from paper_2211_01713_b200 import synth
    hw = make_v100()
    wl, names = synth.scenarios(1, 10_000, hw, seed=91)
    rank = name_ranks(list(names))
    res = _device.plan_device(wl, hw_vector(hw), 32, rank, flags=IGP_F_COOP | IGP_F_CTA)
    _compare_to_oracle(res, 0, wl[0], np.array(hw_vector(hw)), 32, rank, oracle_lib)
    hw = make_v100(r_unit=0.01)
    wl, names = synth.scenarios(1, 3000, hw, seed=92, slo=(20.0, 100.0), rate=(50.0, 6000.0),
                                b_max=128)
    rank = name_ranks(list(names))
    res = _device.plan_device(wl, hw_vector(hw), 128, rank, flags=IGP_F_COOP)
    _compare_to_oracle(res, 0, wl[0], np.array(hw_vector(hw)), 128, rank, oracle_lib)


@pytest.mark.parametrize("case", G.names("doc_"))
def test_plan_document_matches_reference_text(case):
    """plan_to_document (problem.py:305-341) of the device plan is the
    reference's JSON document, character for character."""
    import json
    from paper_2211_01713_b200.document import allocations_from_document, plan_to_document
    d = G.load(case)
    wls = workloads_from_golden(d)
    hw = hw_from_golden(d)
    specs = {s.name: s for s, _ in wls}
    doc = plan_to_document(igp.plan(wls, hw), specs)
    assert json.dumps(doc) == str(d["document"])
    rev = plan_to_document(igp.plan(list(reversed(wls)), hw), specs)  # test_planner.py:208-213
    assert rev == doc
    allocs = allocations_from_document(doc)
    assert sum(len(a) for a in allocs) == len(wls)


def _random_states(rng, n_states, nmax, r_unit, floor=False):
    """Random device states over wide coefficient ranges (test_model_properties.py
    ranges), half of them at unit multiples, the rest at arbitrary r."""
    counts = rng.integers(1, nmax + 1, n_states)
    n = int(counts.sum())
    wl = np.empty((16, n))
    wl[0] = rng.uniform(1.0, 200.0, n)
    wl[1] = rng.uniform(1.0, 2000.0, n)
    wl[2] = rng.uniform(0.0, 2.0, n)
    wl[3] = rng.uniform(0.0, 0.5, n)
    wl[4] = rng.integers(1, 501, n)
    wl[5] = rng.uniform(0.0, 0.01, n)
    wl[6] = rng.uniform(0.0, 0.02, n)
    wl[7] = rng.uniform(0.0, 0.2, n)
    wl[8] = rng.uniform(0.0, 20.0, n)
    wl[9] = rng.uniform(0.0, 2.0, n)
    wl[10] = rng.uniform(1e-3, 1.0, n)
    wl[11] = rng.uniform(0.0, 2000.0 if floor else 100.0, n)
    wl[12] = rng.uniform(0.0, 400.0 if floor else 200.0, n)
    wl[13] = rng.uniform(0.0, 0.2, n)
    wl[14] = rng.uniform(0.0, 0.5, n)
    wl[15] = rng.uniform(0.0, 1.0, n)
    batch = rng.integers(1, 129, n).astype(np.int32)
    u = rng.integers(1, int(round(1.0 / r_unit)) + 1, n)
    r = np.where(rng.random(n) < 0.5, u * r_unit, rng.uniform(0.001, 1.0, n))
    ptr = np.zeros(n_states + 1, np.int64)
    np.cumsum(counts, out=ptr[1:])
    return wl, batch, r, ptr


@pytest.mark.parametrize("r_unit,nmax,floor", [(0.025, 12, False), (0.01, 30, False),
                                               (0.025, 8, True)])
def test_eval_states_million_random_states_vs_oracle(oracle_lib, r_unit, nmax, floor):
    """_eval_entries rows bit-equal on >= 1e6 random
    device states (n = 1..nmax; cap binding, f_min floor and clamps included)."""
    rng = np.random.default_rng(int(r_unit * 1000) + nmax)
    n_states = 1_000_000 if not floor else 200_000
    wl, batch, r, ptr = _random_states(rng, n_states, nmax, r_unit, floor)
    hw = np.array(hw_vector(make_v100(r_unit=r_unit)))
    rows, err = _device.eval_states(wl, batch, r, ptr, hw)
    orows, rc = oracle_lib.eval_states(wl, batch, r, ptr, hw)
    assert rc == 0 and (err["code"] == 0).all()
    np.testing.assert_array_equal(G.bits(rows), G.bits(orows))
    f = rows[:, 3]
    assert (f < hw[1]).mean() > 0.1  # the power cap binds in a good share of states
    if floor:
        assert (f == hw[10] * hw[1]).mean() > 0.1  # f_min floor reached
