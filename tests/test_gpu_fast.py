"""The certified-margin fast kernel (csrc/fast.cuh) on the B200.

With IGP_F_FAST, batches of one-warp scenarios run k_place_fast first (it is
opt-in: slower than the exact kernel on the latency-bound batch, DESIGN.md
section 6).  Every Alg. 2 decision
(planner.py:158) is taken from fp32 compact tiles with an error bound, and a
candidate with a decision inside the bound is re-run with the exact
evaluation.  These tests pin the fast path to the exact-evaluation kernel
(the default) and to the CPU oracle bit for bit -- placements, units,
batches, lower bounds, GPU counts and the _build_plan rows -- including:
* a wide margin (IGP_FAST_DELTA=0.5), so most candidates take the exact
  fallback mid-way;
* r_unit 0.01 / b <= 128 scenarios (max_units 100, GPUs with more than the
  8 staged residents: exact fallback per candidate);
* batches mixing scenarios the fast kernel must decline (a prologue error,
  alpha_cache above the screen) with ordinary ones;
* a record pool too small for the plan (IGP_E_CAPACITY, retried).
"""
import os

import numpy as np
import pytest

from instances import make_v100

pytestmark = pytest.mark.gpu

IGP_F_FAST = 1 << 29
KEYS = ("gpu_of", "pos", "units", "batch", "lb", "gpu_count")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _batch(S, m, hw, seed, **kw):
    from paper_2211_01713_b200 import synth
    from paper_2211_01713_b200.planner import name_ranks
    wl, names = synth.scenario_batch(S, m, hw, seed=seed, **kw)
    return wl, name_ranks(list(names))


def _hv(hw):
    from paper_2211_01713_b200.layout import hw_vector
    return np.array(hw_vector(hw))


def _same(a, b, idx=None):
    sel = (lambda x: x) if idx is None else (lambda x: x[idx])
    for k in KEYS:
        np.testing.assert_array_equal(sel(a[k]), sel(b[k]), err_msg=k)
    np.testing.assert_array_equal(sel(a["pred"]).view(np.int64), sel(b["pred"]).view(np.int64))
    np.testing.assert_array_equal(sel(a["err"]["code"]), sel(b["err"]["code"]))


def _vs_oracle(res, wl, hv, b_max, rank, idx):
    from oracle import oracle
    for s in idx:
        o = oracle.plan(wl[s], hv, b_max, rank)
        assert int(res["err"][s]["code"]) == o["rc"]
        if o["rc"]:
            continue
        for k in ("gpu_of", "pos", "units", "batch", "lb"):
            np.testing.assert_array_equal(res[k][s], o[k], err_msg=f"scenario {s}: {k}")
        assert int(res["gpu_count"][s]) == int(o["gpu_count"])
        np.testing.assert_array_equal(res["pred"][s].view(np.int64), o["pred"].view(np.int64))


def test_fast_equals_exact_kernel_and_oracle():
    from paper_2211_01713_b200 import _device
    hw = make_v100()
    hv = _hv(hw)
    wl, rank = _batch(96, 1500, hw, seed=11)
    fast = _device.plan_device(wl, hv, 32, rank, flags=IGP_F_FAST)
    slow = _device.plan_device(wl, hv, 32, rank)
    _same(fast, slow)
    _vs_oracle(fast, wl, hv, 32, rank, [0, 47, 95])


def test_wide_margin_forces_the_exact_fallback():
    from paper_2211_01713_b200 import _device
    hw = make_v100()
    hv = _hv(hw)
    wl, rank = _batch(32, 800, hw, seed=12)
    base = _device.plan_device(wl, hv, 32, rank)
    os.environ["IGP_FAST_DELTA"] = "0.5"
    try:
        wide = _device.plan_device(wl, hv, 32, rank, flags=IGP_F_FAST)
    finally:
        del os.environ["IGP_FAST_DELTA"]
    _same(wide, base)
    _vs_oracle(wide, wl, hv, 32, rank, [0, 31])


def test_r_unit_001_many_residents():
    from paper_2211_01713_b200 import _device
    hw = make_v100(r_unit=0.01)
    hv = _hv(hw)
    wl, rank = _batch(16, 1200, hw, seed=13, slo=(20.0, 100.0), rate=(50.0, 6000.0), b_max=128)
    fast = _device.plan_device(wl, hv, 128, rank, flags=IGP_F_FAST)
    slow = _device.plan_device(wl, hv, 128, rank)
    _same(fast, slow)
    _vs_oracle(fast, wl, hv, 128, rank, [0, 15])


def test_declined_scenarios_in_a_batch():
    from paper_2211_01713_b200 import _device
    from paper_2211_01713_b200.layout import WL
    hw = make_v100()
    hv = _hv(hw)
    wl, rank = _batch(12, 600, hw, seed=14)
    wl[3, WL["alpha_cache"], 17] = 40.0      # above the fast screen: SF_NO_FAST
    wl[5, WL["slo_ms"], 100] = 1e-3          # InfeasibleSlo in the prologue
    wl[7, WL["k4"], :] = -1.0                # reachable non-positive denominators: risky
    fast = _device.plan_device(wl, hv, 32, rank, flags=IGP_F_FAST)
    slow = _device.plan_device(wl, hv, 32, rank)
    _same(fast, slow)
    assert int(fast["err"][5]["code"]) != 0
    _vs_oracle(fast, wl, hv, 32, rank, range(12))


def test_small_pool_capacity_retry():
    from paper_2211_01713_b200 import _device
    hw = make_v100()
    hv = _hv(hw)
    wl, rank = _batch(8, 700, hw, seed=15)
    slow = _device.plan_device(wl, hv, 32, rank)
    tight = _device.plan_device(wl, hv, 32, rank, flags=IGP_F_FAST | 1 << 8)  # pool of 1 x m records: retried
    _same(tight, slow)


def test_host_entry_with_the_fast_path():
    import torch
    from paper_2211_01713_b200 import _device
    hw = make_v100()
    hv = _hv(hw)
    wl, rank = _batch(300, 500, hw, seed=16)
    dev = _device.plan_device(wl, hv, 32, rank)
    host = _device.plan_host(torch.from_numpy(wl).pin_memory().numpy(), hv, 32, rank,
                             flags=IGP_F_FAST)
    _same(host, dev)
