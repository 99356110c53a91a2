"""One single plan (for ncu): python tools/profile_single.py m r_unit b_max flags"""
import os, sys
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO); sys.path.insert(0, os.path.join(REPO, "tests"))
import numpy as np, torch
from paper_2211_01713_b200 import _device, synth
from paper_2211_01713_b200.layout import hw_vector
from paper_2211_01713_b200.planner import name_ranks
from instances import make_v100
m, ru, bm, fl = int(sys.argv[1]), float(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
hw = make_v100(r_unit=ru)
kw = dict(slo=(20.0, 100.0), rate=(50.0, 6000.0), b_max=128) if bm == 128 else {}
wl, names = synth.scenarios(1, m, hw, seed=2211, **kw)
for _ in range(2):
    r = _device.plan_device(wl, hw_vector(hw), bm, name_ranks(list(names)), flags=fl, want_pred=False)
torch.cuda.synchronize()
print("gpus", r["gpu_count"], "stats", r["stats"][0].tolist())
