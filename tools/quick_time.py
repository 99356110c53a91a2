"""Ad-hoc timing of the plan kernel on synthetic 10k scenario batches."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
from paper_2211_01713_b200 import synth, _device
from paper_2211_01713_b200.planner import name_ranks, IGP_F_CTA
from paper_2211_01713_b200.layout import hw_vector
from instances import make_v100

hw = make_v100()
for S, m, flags in [(1, 10000, 0), (1, 10000, IGP_F_CTA), (148, 10000, 0), (592, 10000, 0), (1184, 10000, 0), (4096, 1000, 0)]:
    wl, names = synth.scenarios(S, m, hw, seed=1)
    rank = name_ranks(list(names))
    _device.plan_device(wl[:1], hw_vector(hw), 32, rank, flags=flags, want_pred=False)
    torch.cuda.synchronize()
    t = time.perf_counter()
    res = _device.plan_device(wl, hw_vector(hw), 32, rank, flags=flags, want_pred=False)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    print(f"S={S} m={m} flags={flags}: {dt:.3f}s  {S/dt:.2f} plans/s  gpus={res['gpu_count'][:3]} err={np.unique(res['err']['code'])}", flush=True)
