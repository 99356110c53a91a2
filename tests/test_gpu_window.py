"""The windowed speculative single-plan kernel (IGP_F_WIN, csrc/window.cuh)
against the reference's plan fixtures and the CPU oracle: placements, units,
batches, lower bounds and the _build_plan rows bit for bit, and the
reference's exceptions for inputs that raise (declined to the per-CTA
kernel)."""
import numpy as np
import pytest

import golden_io as G
from instances import make_v100, random_instance

pytestmark = pytest.mark.gpu

IGP_F_CTA, IGP_F_STATS, IGP_F_WIN = 4, 1, 1 << 28


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _check(res, o):
    for k in ("gpu_of", "pos", "units", "batch", "lb"):
        np.testing.assert_array_equal(res[k][0], o[k], err_msg=k)
    assert int(res["gpu_count"][0]) == int(o["gpu_count"])
    np.testing.assert_array_equal(G.bits(res["pred"][0]), G.bits(o["pred"]))


@pytest.mark.parametrize("case", G.names("plan_"))
def test_window_plan_matches_reference_fixture(case):
    from paper_2211_01713_b200 import _device
    from paper_2211_01713_b200.planner import name_ranks
    d = G.load(case)
    res = _device.plan_device(d["wl"], d["hw"], int(d["b_max"]), name_ranks(list(d["names"])),
                              flags=IGP_F_WIN | IGP_F_CTA)
    code = int(res["err"][0]["code"])
    if str(d["err_class"]):
        assert code == int(d["err_code"])
        return
    assert code == 0
    o = {k: d[k] for k in ("gpu_of", "pos", "units", "batch", "lb", "pred")}
    o["gpu_count"] = int(d["gpu_count"])
    _check(res, o)


@pytest.mark.parametrize("m,seed,r_unit,b_max", [(40, 1, 0.025, 32), (300, 2, 0.025, 32),
                                                 (1000, 7, 0.025, 32), (2500, 3, 0.025, 32),
                                                 (1200, 4, 0.01, 128), (700, 5, 0.05, 32)])
def test_window_plan_vs_oracle(oracle_lib, m, seed, r_unit, b_max):
    from paper_2211_01713_b200 import _device, synth
    from paper_2211_01713_b200.layout import hw_vector
    from paper_2211_01713_b200.planner import name_ranks
    hw = make_v100(r_unit=r_unit)
    kw = dict(slo=(20.0, 100.0), rate=(50.0, 6000.0), b_max=128) if b_max == 128 else {}
    wl, names = synth.scenarios(1, m, hw, seed=seed, **kw)
    rank = name_ranks(list(names))
    hv = np.array(hw_vector(hw))
    res = _device.plan_device(wl, hv, b_max, rank, flags=IGP_F_WIN | IGP_F_CTA)
    assert int(res["err"][0]["code"]) == 0
    _check(res, oracle_lib.plan(wl[0], hv, b_max, rank))


def test_window_plan_reference_10k():
    from paper_2211_01713_b200 import _device
    from paper_2211_01713_b200.planner import name_ranks
    d = G.load("ref_plan_10k")
    res = _device.plan_device(d["wl"], d["hw"], 32,
                              name_ranks(list(d["names"])), flags=IGP_F_WIN | IGP_F_CTA)
    assert int(res["err"][0]["code"]) == 0
    o = {k: d[k] for k in ("gpu_of", "pos", "units", "batch", "lb", "pred")}
    o["gpu_count"] = int(d["gpu_count"])
    _check(res, o)


def test_window_declines_to_exact_stats():
    """With PlanStats the windowed kernel declines; the per-CTA kernel runs the
    reference's exact sequence (same plan, exact counters)."""
    from paper_2211_01713_b200 import _device
    from paper_2211_01713_b200.planner import name_ranks
    d = G.load("plan_rand1k_seed7")
    res = _device.plan_device(d["wl"], d["hw"], 32, name_ranks(list(d["names"])),
                              flags=IGP_F_WIN | IGP_F_CTA | IGP_F_STATS)
    assert int(res["stats"][0][0]) == int(d["model_evals"])
    np.testing.assert_array_equal(res["units"][0], d["units"])
