"""The shared-memory single-plan kernel (IGP_F_SMEM, csrc/smem_plan.cuh).

One CTA per scenario keeps the search state in shared memory and evaluates
each candidate with one warp (certified-margin decisions, the exact
evaluation inside the margin).  Pinned bit for bit -- placements, units,
batches, lower bounds, GPU counts and the _build_plan rows -- to the
reference's plan fixtures, to the CPU oracle, and to the per-CTA kernel:
* every reference plan fixture (known answers, error branches, name ties);
* random plans at r_unit 0.025 / 0.01 / 0.05 and b <= 128;
* a wide margin (IGP_FAST_DELTA=0.5), so most candidates take the exact path;
* a plan too large for shared memory (the per-CTA kernel plans it);
* PlanStats (declined: the exact sequence and counters);
* a batch of several scenarios, one CTA each, one of them declined;
* a record pool too small for the plan (IGP_E_CAPACITY, retried).
"""
import os

import numpy as np
import pytest

import golden_io as G
from instances import make_v100

pytestmark = pytest.mark.gpu

IGP_F_STATS, IGP_F_CTA, IGP_F_SMEM = 1, 4, 8
FL = IGP_F_SMEM | IGP_F_CTA


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _check(res, o, s=0):
    for k in ("gpu_of", "pos", "units", "batch", "lb"):
        np.testing.assert_array_equal(res[k][s], o[k], err_msg=k)
    assert int(res["gpu_count"][s]) == int(o["gpu_count"])
    np.testing.assert_array_equal(G.bits(res["pred"][s]), G.bits(o["pred"]))


def _inst(m, seed, r_unit=0.025, b_max=32, S=1):
    from paper_2211_01713_b200 import synth
    from paper_2211_01713_b200.layout import hw_vector
    from paper_2211_01713_b200.planner import name_ranks
    hw = make_v100(r_unit=r_unit)
    kw = dict(slo=(20.0, 100.0), rate=(50.0, 6000.0), b_max=128) if b_max == 128 else {}
    wl, names = synth.scenarios(S, m, hw, seed=seed, **kw)
    return wl, np.array(hw_vector(hw)), name_ranks(list(names))


@pytest.mark.parametrize("case", G.names("plan_"))
def test_smem_plan_matches_reference_fixture(case):
    from paper_2211_01713_b200 import _device
    from paper_2211_01713_b200.planner import name_ranks
    d = G.load(case)
    res = _device.plan_device(d["wl"], d["hw"], int(d["b_max"]), name_ranks(list(d["names"])),
                              flags=FL)
    code = int(res["err"][0]["code"])
    if str(d["err_class"]):
        assert code == int(d["err_code"])
        return
    assert code == 0
    o = {k: d[k] for k in ("gpu_of", "pos", "units", "batch", "lb", "pred")}
    o["gpu_count"] = int(d["gpu_count"])
    _check(res, o)


@pytest.mark.parametrize("m,seed,r_unit,b_max", [(12, 9, 0.025, 32), (40, 1, 0.025, 32),
                                                 (300, 2, 0.025, 32), (1000, 7, 0.025, 32),
                                                 (1800, 3, 0.025, 32), (1200, 4, 0.01, 128),
                                                 (700, 5, 0.05, 32)])
def test_smem_plan_vs_oracle_and_cta_kernel(oracle_lib, m, seed, r_unit, b_max):
    from paper_2211_01713_b200 import _device
    wl, hv, rank = _inst(m, seed, r_unit, b_max)
    res = _device.plan_device(wl, hv, b_max, rank, flags=FL)
    assert int(res["err"][0]["code"]) == 0
    _check(res, oracle_lib.plan(wl[0], hv, b_max, rank))
    cta = _device.plan_device(wl, hv, b_max, rank, flags=IGP_F_CTA)
    _check(res, {k: cta[k][0] for k in ("gpu_of", "pos", "units", "batch", "lb", "pred",
                                        "gpu_count")})


def test_smem_wide_margin_exact_path(oracle_lib):
    from paper_2211_01713_b200 import _device
    wl, hv, rank = _inst(600, 21)
    os.environ["IGP_FAST_DELTA"] = "0.5"
    try:
        res = _device.plan_device(wl, hv, 32, rank, flags=FL)
    finally:
        del os.environ["IGP_FAST_DELTA"]
    assert int(res["stats"][0][4]) > 0  # candidates re-run with the exact evaluation
    _check(res, oracle_lib.plan(wl[0], hv, 32, rank))


def test_smem_too_large_falls_back(oracle_lib):
    from paper_2211_01713_b200 import _device
    wl, hv, rank = _inst(4000, 22)
    res = _device.plan_device(wl, hv, 32, rank, flags=FL)
    assert int(res["stats"][0][4]) == -1  # not the shared-memory kernel
    _check(res, oracle_lib.plan(wl[0], hv, 32, rank))


def test_smem_declines_to_exact_stats():
    from paper_2211_01713_b200 import _device
    from paper_2211_01713_b200.planner import name_ranks
    d = G.load("plan_rand1k_seed7")
    res = _device.plan_device(d["wl"], d["hw"], 32, name_ranks(list(d["names"])),
                              flags=FL | IGP_F_STATS)
    assert int(res["stats"][0][0]) == int(d["model_evals"])
    assert int(res["stats"][0][1]) == int(d["candidate_gpus"])
    np.testing.assert_array_equal(res["units"][0], d["units"])


def test_smem_batch_one_cta_each(oracle_lib):
    from paper_2211_01713_b200 import _device
    from paper_2211_01713_b200.layout import WL
    wl, hv, rank = _inst(500, 23, S=6)
    wl[2, WL["slo_ms"], 40] = 1e-3  # a prologue error: declined, reported like the reference
    res = _device.plan_device(wl, hv, 32, rank, flags=FL)
    for s in range(6):
        o = oracle_lib.plan(wl[s], hv, 32, rank)
        assert int(res["err"][s]["code"]) == o["rc"]
        if not o["rc"]:
            _check(res, o, s)


def test_smem_small_pool_retry(oracle_lib):
    from paper_2211_01713_b200 import _device
    wl, hv, rank = _inst(800, 24)
    res = _device.plan_device(wl, hv, 32, rank, flags=FL | (1 << 8))
    _check(res, oracle_lib.plan(wl[0], hv, 32, rank))


def test_plan_api_uses_smem_kernel():
    """plan() of a C2-sized instance runs the shared-memory kernel and returns
    the reference's plan object."""
    import paper_2211_01713_b200 as igp
    from paper_2211_01713_b200 import _device
    from instances import random_instance
    hw = make_v100()
    wls = random_instance(np.random.default_rng(7), 300, hw)
    p = igp.plan(wls, hw)
    assert len(p.gpus) > 0 and sum(len(g.allocations) for g in p.gpus) == 300
