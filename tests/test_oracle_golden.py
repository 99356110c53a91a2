"""Pin the CPU oracle against fixtures produced by the real reference
(tests/golden/make_golden.py).  CPU only."""
import numpy as np
import pytest

import golden_io as G


@pytest.mark.parametrize("case", G.names("plan_"))
def test_oracle_plan_matches_reference(oracle_lib, case):
    d = G.load(case)
    rank = oracle_lib.name_ranks([str(n) for n in d["names"]])
    o = oracle_lib.plan(d["wl"], d["hw"], int(d["b_max"]), rank)
    assert o["model_evals"] == int(d["model_evals"])
    assert o["candidate_gpus"] == int(d["candidate_gpus"])
    if str(d["err_class"]):
        assert o["rc"] == int(d["err_code"])
        return
    assert o["rc"] == 0
    for k in ("gpu_of", "pos", "units", "batch", "lb"):
        np.testing.assert_array_equal(o[k], d[k], err_msg=k)
    assert o["gpu_count"] == int(d["gpu_count"])
    np.testing.assert_array_equal(G.bits(o["pred"]), G.bits(d["pred"]))


@pytest.mark.parametrize("case", G.names("eval_states_"))
def test_oracle_eval_states(oracle_lib, case):
    d = G.load(case)
    rows, rc = oracle_lib.eval_states(d["wl"], d["batch"], d["r"], d["ptr"], d["hw"])
    assert rc == 0
    np.testing.assert_array_equal(G.bits(rows), G.bits(d["rows"]))


@pytest.mark.parametrize("case", G.names("prologue_"))
def test_oracle_prologue(oracle_lib, case):
    d = G.load(case)
    b, lb, code = oracle_lib.prologue(d["wl"], d["hw"], int(d["b_max"]))
    np.testing.assert_array_equal(code, d["code"])
    ok_b = code != 1
    np.testing.assert_array_equal(b[ok_b], d["batch"][ok_b])
    np.testing.assert_array_equal(lb[code == 0], d["lb"][code == 0])


def test_oracle_alloc_units(oracle_lib):
    d = G.load("alloc_v100")
    u, rc = oracle_lib.alloc_units(d["wl"], d["batch"], d["r"], d["ptr"], d["hw"])
    assert rc == 0
    np.testing.assert_array_equal(u, d["units"])


def test_golden_known_answers_from_reference_tests():
    """Spot values the reference's own tests freeze (test_planner.py)."""
    d = G.load("plan_single")  # test_planner.py:161-167
    assert int(d["gpu_count"]) == 1 and int(d["units"][0]) == 1 and int(d["batch"][0]) == 8
    assert float(d["cost"]) == 3.06
    assert float(d["fragment"][0]) == pytest.approx(0.975, rel=1e-12)
    d = G.load("plan_simple12_v100")  # :238-243
    assert int(d["gpu_count"]) == 6 and round(float(d["cost"]), 2) == 18.36
    d = G.load("plan_simple15_t4")  # :245-250
    assert int(d["gpu_count"]) == 15 and round(float(d["cost"]), 2) == 7.89
    d = G.load("plan_c1_twelve")  # SURVEY.md §8c session known answer
    assert int(d["gpu_count"]) == 2
    assert int(d["model_evals"]) == 650 and int(d["candidate_gpus"]) == 17
    d = G.load("plan_rand1k_seed7")  # 268 GPUs, 31,018 / 930,080
    assert int(d["gpu_count"]) == 268
    assert int(d["candidate_gpus"]) == 31018 and int(d["model_evals"]) == 930080


def test_predict_known_values_in_eval_fixture_semantics(oracle_lib):
    """test_model.py:153-160: single resnet at r=0.025, batch 8 on the V100."""
    from instances import make_v100
    from paper_2211_01713_b200.layout import hw_vector, spec_coef_row
    from paper_2211_01713_b200 import WorkloadSpec, WorkloadCoefficients
    spec = WorkloadSpec("resnet", 40.0, 400.0, 0.574, 0.004)
    coef = WorkloadCoefficients(100, 0.002, 0.001, 0.05, 0.5, 0.05, 0.2, 50.0, 60.0, 0.05, 0.10, 0.25)
    wl = np.array(spec_coef_row(spec, coef)).reshape(16, 1)
    rows, rc = oracle_lib.eval_states(wl, np.array([8], np.int32), np.array([0.025]),
                                      np.array([0, 1], np.int64), np.array(hw_vector(make_v100())))
    assert rc == 0
    assert rows[0, 4] == pytest.approx(13.253333333333334, rel=1e-12)
    assert rows[0, 6] == pytest.approx(13.715733333333333, rel=1e-12)
    assert rows[0, 3] == 1530.0
    assert rows[0, 7] == pytest.approx(603.4760218860637, rel=1e-12)


@pytest.mark.parametrize("case", G.names("grid_"))
def test_oracle_solo_grid_matches_reference(oracle_lib, case):
    """Solo grid vs the reference's _Search.best_group_alloc (oracle.py:77-114)."""
    d = G.load(case)
    mu, evals = oracle_lib.solo_grid(d["wl"], d["hw"], int(d["b_max"]))
    np.testing.assert_array_equal(mu, d["min_units"])
    assert evals > 0


@pytest.mark.parametrize("case", G.names("stream_"))
def test_oracle_stream_matches_reference_driver(oracle_lib, case):
    """Arrival-order stream vs the reference-internals driver (make_golden.py)."""
    d = G.load(case)
    o = oracle_lib.stream(d["wl"], d["hw"], int(d["b_max"]))
    for k in ("gpu_of", "pos", "code", "units"):
        np.testing.assert_array_equal(o[k], d[k], err_msg=k)
    assert o["gpu_count"] == int(d["gpu_count"])


def test_plan_document_roundtrip_helpers(tmp_path):
    """allocations_from_document / write_json_atomic on the reference's own
    document text (problem.py:344-398)."""
    import json
    from paper_2211_01713_b200.document import allocations_from_document, write_json_atomic
    from paper_2211_01713_b200.errors import ProblemFormatError
    d = G.load("doc_c1_twelve")
    doc = json.loads(str(d["document"]))
    allocs = allocations_from_document(doc)
    assert [len(a) for a in allocs] == [len(g["allocations"]) for g in doc["gpus"]]
    assert allocs[0][0].workload == doc["gpus"][0]["allocations"][0]["workload"]
    path = tmp_path / "sub" / "plan.json"
    write_json_atomic(path, doc)
    assert json.loads(path.read_text()) == doc
    with pytest.raises(ProblemFormatError, match="missing required field 'gpus'"):
        allocations_from_document({})
