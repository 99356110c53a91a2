"""BASELINE config 3 at full size: one 100,000-workload plan (r_unit 0.01,
b <= 128) on the GPU, bit-exact against the CPU oracle's plan of the same
seeded instance (tests/golden/c3_plan_100k.npz, tests/golden/make_c3_100k.py).
The oracle is pinned to the reference on the C3-style fixtures and, when the
fixture was made, on a reference prefix run (greedy prefix property)."""
import os
import sys

import numpy as np
import pytest

import golden_io as G

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden"))


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def test_c3_100k_plan_bit_exact():
    import make_c3_100k as C3
    from paper_2211_01713_b200 import _device
    from paper_2211_01713_b200.layout import hw_vector
    from paper_2211_01713_b200.planner import IGP_F_COOP, IGP_F_CTA, name_ranks
    d = G.load("c3_plan_100k")
    hw, wl, names = C3.instance()
    res = _device.plan_device(wl, hw_vector(hw), C3.B_MAX, name_ranks(names),
                              flags=IGP_F_CTA | IGP_F_COOP)
    assert int(res["err"][0]["code"]) == 0
    assert int(res["gpu_count"][0]) == int(d["gpu_count"])
    for k in ("gpu_of", "pos", "units", "batch", "lb"):
        np.testing.assert_array_equal(res[k][0], d[k].astype(np.int32), err_msg=k)
    np.testing.assert_array_equal(G.bits(res["pred"][0][:, 6]), G.bits(d["pred_t_inf"]))
