"""Exhaustive oracle (oracle.py:130-201): the CPU oracle's per-subset grid
search plus the host partition choice against the reference's own
exhaustive_plan fixtures (tests/golden/oracle_*.npz).  CPU only."""
import numpy as np
import pytest

import golden_io as G

from paper_2211_01713_b200.exhaustive import decode_keys, select_partition


def _plan_via_oracle(d, oracle_lib):
    wl, hw = d["wl"], d["hw"]
    names = [str(x) for x in d["names"]]
    m = len(names)
    b, lb, code = oracle_lib.prologue(wl, hw, int(d["b_max"]))
    if (code != 0).any():
        return None, int(code[code != 0][0])
    order = sorted(range(m), key=names.__getitem__)
    cap = oracle_lib.lib().igo_max_units(hw.ctypes.data_as(__import__("ctypes").c_void_p))
    grid = d["grid"] if len(d["grid"]) else np.arange(1, cap + 1)
    best, rc = oracle_lib.group_search(wl[:, order], b[order], hw, np.sort(grid))
    assert rc == 0
    sorted_names = [names[i] for i in order]
    blocks = select_partition(sorted_names, decode_keys(best, m), int(d["max_gpus"]))
    return blocks, 0


@pytest.mark.parametrize("case", G.names("oracle_"))
def test_oracle_exhaustive_matches_reference(oracle_lib, case):
    d = G.load(case)
    names = [str(x) for x in d["names"]]
    if str(d["err_class"]) == "BudgetExceededError":
        assert len(names) > 4
        return
    blocks, code = _plan_via_oracle(d, oracle_lib)
    if str(d["err_class"]):
        assert str(d["err_class"]) == "InfeasibleError" and blocks is None
        return
    assert code == 0 and blocks is not None
    gpu_of = np.full(len(names), -1)
    units = np.zeros(len(names), np.int32)
    for j, block in enumerate(blocks):
        for nm, u in block:
            gpu_of[names.index(nm)] = j
            units[names.index(nm)] = u
    np.testing.assert_array_equal(gpu_of, d["gpu_of"])
    np.testing.assert_array_equal(units, d["units"])
