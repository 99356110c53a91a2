"""The model's component functions (model.py:159-236) on the device against
the reference's own values and exception texts (tests/golden/modelfn_*.npz).
Columns are compared bit for bit; error rows by code and message."""
import numpy as np
import pytest

import golden_io as G
from instances import hw_from_golden, workloads_from_golden

import paper_2211_01713_b200 as igp
from paper_2211_01713_b200 import _device, errors
from paper_2211_01713_b200.layout import E_ACTIVE_TIME, E_DENOM

pytestmark = pytest.mark.gpu

COLS = ["t_load", "t_fb", None, "k_act", "power", "cache", "sch_inc", "sched", "act_int", "freq"]


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.parametrize("case", G.names("modelfn_"))
def test_batched_columns_match_reference(case):
    d = G.load(case)
    out, code = _device.components(d["wl"], d["q_batch"], d["q_r"], d["q_co"], d["q_ncol"],
                                   d["q_pdem"], d["hw"])
    denom_err = np.array([m.startswith("NonPositiveDenominatorError: r + k4") for m in d["msg_k_act"]])
    act_err = np.array([m != "" for m in d["msg_power"]]) & ~denom_err
    np.testing.assert_array_equal(code == E_DENOM, denom_err)
    np.testing.assert_array_equal(code == E_ACTIVE_TIME, act_err)
    for j, name in enumerate(COLS):
        if name is None:
            continue
        ok = d[f"msg_{name}"] == ""
        np.testing.assert_array_equal(G.bits(out[ok, j]), G.bits(d[f"fn_{name}"][ok]), err_msg=name)


@pytest.mark.parametrize("case", G.names("modelfn_"))
def test_public_functions_and_messages(case):
    d = G.load(case)
    hw = hw_from_golden(d)
    wls = workloads_from_golden(d)
    calls = {
        "t_load": lambda i, sp, c: igp.transfer_latencies(sp, int(d["q_batch"][i]), hw)[0],
        "t_fb": lambda i, sp, c: igp.transfer_latencies(sp, int(d["q_batch"][i]), hw)[1],
        "k_act": lambda i, sp, c: igp.solo_active_time(c, int(d["q_batch"][i]), float(d["q_r"][i])),
        "power": lambda i, sp, c: igp.solo_power(c, int(d["q_batch"][i]), float(d["q_r"][i])),
        "cache": lambda i, sp, c: igp.solo_cache_util(c, int(d["q_batch"][i]), float(d["q_r"][i])),
        "sch_inc": lambda i, sp, c: igp.sched_delay_increase(hw, int(d["q_ncol"][i])),
        "sched": lambda i, sp, c: igp.sched_delay(c, hw, int(d["q_ncol"][i])),
        "act_int": lambda i, sp, c: igp.active_time_with_interference(
            c, int(d["q_batch"][i]), float(d["q_r"][i]), float(d["q_co"][i])),
        "freq": lambda i, sp, c: igp.gpu_frequency(hw, float(d["q_pdem"][i])),
    }
    for i in range(0, 40):  # every query kind (i % 10), including both error kinds
        sp, c = wls[i]
        for name, fn in calls.items():
            msg = str(d[f"msg_{name}"][i])
            if msg:
                with pytest.raises(errors.NonPositiveDenominatorError) as ei:
                    fn(i, sp, c)
                assert f"{type(ei.value).__name__}: {ei.value}" == msg
            else:
                assert G.bits([fn(i, sp, c)]) == G.bits([d[f"fn_{name}"][i]]), (name, i)


@pytest.mark.parametrize("case", G.names("modelfn_"))
def test_power_demand_matches_reference(case):
    d = G.load(case)
    hw = hw_from_golden(d)
    ptr, vals = d["pd_ptr"], d["pd_vals"]
    got = [igp.power_demand(hw, list(vals[ptr[k]:ptr[k + 1]])) for k in range(len(ptr) - 1)]
    np.testing.assert_array_equal(G.bits(got), G.bits(d["pd_out"]))
