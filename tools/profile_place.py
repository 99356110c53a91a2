"""Run prepare+place twice on one synthetic batch (for ncu: profile the 2nd k_place).

usage: python tools/profile_place.py S m flags   (S=0: the bench batch, one scenario per slot)"""
import ctypes, os, sys
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import numpy as np, torch
from paper_2211_01713_b200 import _device, _native, synth
from paper_2211_01713_b200.layout import hw_vector
from paper_2211_01713_b200.model import HardwareProfile
from paper_2211_01713_b200.planner import name_ranks

S = int(sys.argv[1]) if len(sys.argv) > 1 else 1184
m = int(sys.argv[2]) if len(sys.argv) > 2 else 10000
flags = int(sys.argv[3]) if len(sys.argv) > 3 else 0
hw = HardwareProfile("v100", 300.0, 1530.0, 53.5, 10.0, -1.025, 0.00475, -0.00902, r_unit=0.025, price_per_hour=3.06)
if S == 0:  # one scenario per resident slot, as bench.py
    S = _device.batch_slots(m, hw_vector(hw), 32, flags)
wl, names = synth.scenario_batch(S, m, hw, seed=2211)
for rep in range(2):
    res = _device.plan_device(wl, hw_vector(hw), 32, name_ranks(list(names)), flags=flags, want_pred=False)
torch.cuda.synchronize()
print("gpus", res["gpu_count"][:4], "evals_run", res["stats"][:, 3].sum())
