"""Debug helper: one cooperative plan (m, r_unit, b_max, flags) vs the oracle."""
import os, sys
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO); sys.path.insert(0, os.path.join(REPO, "tests"))
import numpy as np
from oracle import oracle
from paper_2211_01713_b200 import _device, synth
from paper_2211_01713_b200.layout import hw_vector
from paper_2211_01713_b200.planner import name_ranks
from instances import make_v100
m, ru, bm, fl = int(sys.argv[1]), float(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
hw = make_v100(r_unit=ru)
kw = dict(slo=(20.0, 100.0), rate=(50.0, 6000.0), b_max=128) if bm == 128 else {}
wl, names = synth.scenarios(1, m, hw, seed=92, **kw)
rank = name_ranks(list(names))
res = _device.plan_device(wl, hw_vector(hw), bm, rank, flags=fl)
o = oracle.plan(wl[0], np.array(hw_vector(hw)), bm, rank)
print("err", res["err"][0]["code"], "gpus", res["gpu_count"][0], o["gpu_count"],
      "units equal", np.array_equal(res["units"][0], o["units"]))
