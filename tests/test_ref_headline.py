"""Reference-run fixtures at the headline size.

ref_plan_10k.npz -- the unmodified reference plan() (CPython 3.12) on scenario 0
of bench.py's batch (10,000 workloads, seed 2211; tests/golden/make_ref_10k.py):
2,654 GPUs, 73,041,794 model_evals, 183 s of CPython.  The oracle (CPU) and the
B200 (through plan() and through the batch C-ABI, inside a full-size batch) must
reproduce it bit for bit, _build_plan rows and PlanStats included.

c3_prefix_ref.npz -- the reference plan() on the top-K workloads of the C3
100,000-workload instance (greedy prefix property): pins the oracle, and the
B200's cooperative kernel, on the first K steps of the C3 plan with the
reference's own output.
"""
import os
import sys

import numpy as np
import pytest

import golden_io as G
from instances import make_v100, workloads_from_golden

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden"))


def _hv():
    from paper_2211_01713_b200.layout import hw_vector
    return np.array(hw_vector(make_v100()))


def _check(out, d, s=None):
    pick = (lambda a: a[s]) if s is not None else (lambda a: a)
    for k in ("gpu_of", "pos", "units", "batch", "lb"):
        if k in d:
            np.testing.assert_array_equal(pick(out[k]), d[k].astype(np.int32), err_msg=k)
    np.testing.assert_array_equal(G.bits(pick(out["pred"])), G.bits(d["pred"]))


def test_bench_scenario0_is_the_fixture_instance():
    from paper_2211_01713_b200 import synth
    d = G.load("ref_plan_10k")
    wl, _ = synth.scenario_batch(2368, 10_000, make_v100(), seed=int(d["seed"]), indices=[0])
    np.testing.assert_array_equal(G.bits(wl[0]), G.bits(d["wl"]))


def test_oracle_matches_reference_10k(oracle_lib):
    d = G.load("ref_plan_10k")
    rank = oracle_lib.name_ranks(list(d["names"]))
    o = oracle_lib.plan(d["wl"], _hv(), 32, rank)
    assert o["rc"] == 0
    _check(o, d)
    assert o["gpu_count"] == int(d["gpu_count"]) == 2654
    assert o["model_evals"] == int(d["model_evals"])
    assert o["candidate_gpus"] == int(d["candidate_gpus"])


def _c3_prefix_instance():
    import make_c3_100k as C3
    d = G.load("c3_prefix_ref")
    hw, wl, names = C3.instance()
    order = d["order"].astype(np.int64)
    return d, hw, wl[:, order], [names[i] for i in order]


@pytest.mark.slow
def test_oracle_matches_reference_c3_prefix(oracle_lib):
    from paper_2211_01713_b200.layout import hw_vector
    d, hw, sub, names = _c3_prefix_instance()
    o = oracle_lib.plan(sub, np.array(hw_vector(hw)), int(d["b_max"]),
                        oracle_lib.name_ranks(names))
    assert o["rc"] == 0
    _check(o, d)
    assert o["model_evals"] == int(d["model_evals"])
    assert o["candidate_gpus"] == int(d["candidate_gpus"])


# ---------------------------------------------------------------- B200 -----
@pytest.fixture
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


@pytest.mark.gpu
@pytest.mark.parametrize("with_stats", [False, True])
def test_plan_api_matches_reference_10k(cuda, with_stats):
    import paper_2211_01713_b200 as igp
    d = G.load("ref_plan_10k")
    wls = workloads_from_golden(d)
    stats = igp.PlanStats() if with_stats else None
    p = igp.plan(wls, make_v100(), b_max=32, stats=stats)
    assert p.gpu_count == int(d["gpu_count"])
    idx = {s.name: i for i, (s, _) in enumerate(wls)}
    units = np.zeros(len(wls), np.int32)
    pred = np.zeros((len(wls), 10))
    for g in p.gpus:
        for k, a in enumerate(g.allocations):
            i = idx[a.workload]
            assert g.gpu_index == int(d["gpu_of"][i]) and k == int(d["pos"][i])
            units[i] = int(round(a.r / 0.025))
            bd = g.predicted[a.workload]
            pred[i] = [bd.t_load_ms, bd.t_sch_ms, bd.t_act_ms, bd.freq_mhz, bd.t_gpu_ms,
                       bd.t_feedback_ms, bd.t_inf_ms, bd.throughput_rps, bd.power_w, bd.cache_util]
    np.testing.assert_array_equal(units, d["units"])
    np.testing.assert_array_equal(G.bits(pred), G.bits(d["pred"]))
    if with_stats:
        assert stats.model_evals == int(d["model_evals"])
        assert stats.candidate_gpus == int(d["candidate_gpus"])


@pytest.mark.gpu
def test_batch_abi_matches_reference_10k_inside_full_batch(cuda):
    """The headline path: scenario 0 (and copies of it in the middle and at the
    LAST index of the bench's batch -- two waves of the place kernel's resident
    slots, 5,920 scenarios on a B200 -- so an offset bug at the far end shows)
    planned by igp_plan_batch_host / igp_plan_batch_device."""
    from paper_2211_01713_b200 import _device
    from paper_2211_01713_b200.planner import name_ranks
    d = G.load("ref_plan_10k")
    S = 2 * _device.batch_slots(10_000, _hv(), 32)  # bench.py: WAVES x slots
    wl = np.empty((S, 16, 10_000))
    wl[:] = d["wl"][None]
    rank = name_ranks(list(d["names"]))
    out = _device.plan_host(wl, _hv(), 32, rank, want_pred=True)
    assert (out["err"]["code"] == 0).all()
    for s in (0, S // 2, S - 1):
        _check(out, d, s)
    res = _device.plan_device(wl[[0, -1]], _hv(), 32, rank, flags=1)  # exact PlanStats
    for s in (0, 1):
        _check(res, d, s)
        assert int(res["stats"][s][0]) == int(d["model_evals"])
        assert int(res["stats"][s][1]) == int(d["candidate_gpus"])


@pytest.mark.gpu
def test_cooperative_plan_matches_reference_c3_prefix(cuda):
    from paper_2211_01713_b200 import _device
    from paper_2211_01713_b200.layout import hw_vector
    from paper_2211_01713_b200.planner import IGP_F_COOP, IGP_F_CTA, name_ranks
    d, hw, sub, names = _c3_prefix_instance()
    res = _device.plan_device(sub, hw_vector(hw), int(d["b_max"]), name_ranks(names),
                              flags=IGP_F_CTA | IGP_F_COOP)
    assert int(res["err"][0]["code"]) == 0
    _check(res, d, 0)
