"""The C-ABI library loads and exports every symbol include/*.h declares
(no compute without a GPU).  CPU only."""
import glob
import os
import re

import pytest

from paper_2211_01713_b200 import _native

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    syms = set()
    for h in glob.glob(os.path.join(REPO, "include", "*.h")):
        text = open(h).read()
        text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
        syms |= set(re.findall(r"\b(igp_\w+)\s*\(", text))
    return sorted(syms)


def test_header_declares_entry_points():
    syms = declared_symbols()
    for must in ("igp_plan_batch_device", "igp_plan_batch_host", "igp_eval_states_device",
                 "igp_alloc_units_device", "igp_prologue_device", "igp_plan_workspace_bytes"):
        assert must in syms


def test_library_exports_all_declared_symbols():
    lib = _native.load()
    for s in declared_symbols():
        assert hasattr(lib, s), s
    assert set(declared_symbols()) == set(_native.PROTOTYPES)


def test_abi_version_and_limits():
    lib = _native.load()
    assert lib.igp_abi_version() == 1
    assert lib.igp_max_cap() >= 100


def test_workspace_sizing_is_monotone():
    import numpy as np
    from paper_2211_01713_b200.layout import hw_vector
    from instances import make_v100
    lib = _native.load()
    h = np.array(hw_vector(make_v100()))
    p = h.ctypes.data_as(__import__("ctypes").c_void_p)
    a = lib.igp_plan_workspace_bytes(1, 1000, p, 32, 0)
    b = lib.igp_plan_workspace_bytes(2, 1000, p, 32, 0)
    c = lib.igp_plan_workspace_bytes(2, 2000, p, 32, 0)
    assert 0 < a < b < c


def test_compute_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2211_01713_b200 import appropriate_batch
    from instances import make_v100
    from paper_2211_01713_b200 import WorkloadSpec
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        appropriate_batch(WorkloadSpec("w", 40.0, 400.0, 0.5, 0.01), make_v100())
