"""A/B of igp_plan_batch_host chunking (IGP_HOST_CHUNKS) at the headline batch."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2211_01713_b200 import _device, synth  # noqa: E402
from paper_2211_01713_b200.layout import hw_vector  # noqa: E402
from paper_2211_01713_b200.planner import name_ranks  # noqa: E402

S, m = int(sys.argv[1]) if len(sys.argv) > 1 else 2368, 10_000
hw = bench.hardware()
hv = np.array(hw_vector(hw))
wl, names = synth.scenario_batch(S, m, hw, seed=2211)
rk = name_ranks(list(names))
wl_p = torch.from_numpy(wl).pin_memory().numpy()
out = {k: torch.empty((S, m), dtype=torch.int32).pin_memory().numpy()
       for k in ("gpu_of", "pos", "units", "batch", "lb")}
out["pred"] = torch.empty((S, m, 10), dtype=torch.float64).pin_memory().numpy()
out["gpu_count"] = torch.empty(S, dtype=torch.int32).pin_memory().numpy()
out["stats"] = torch.empty((S, 6), dtype=torch.int64).pin_memory().numpy()
out["err"] = torch.zeros(S * _device._native.err_dtype().itemsize, dtype=torch.uint8).pin_memory().numpy().view(_device._native.err_dtype())
for nc in sys.argv[2:] or ["1", "2", "4", "8"]:
    os.environ["IGP_HOST_CHUNKS"] = nc
    _device.plan_host(wl_p, hv, 32, rk, out=out)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(2):
        _device.plan_host(wl_p, hv, 32, rk, out=out)
    dt = (time.perf_counter() - t) / 2
    print(f"chunks {nc}: {dt * 1e3:.1f} ms/step, {S / dt:.1f} plans/s", flush=True)
d_wl = torch.from_numpy(wl).cuda()
for sub in (S // 4, S):
    t = time.perf_counter()
    _device.plan_device(wl[:sub], hv, 32, rk)
    torch.cuda.synchronize()
    t = time.perf_counter()
    _device.plan_device(wl[:sub], hv, 32, rk)
    torch.cuda.synchronize()
    print(f"plan_device S={sub}: {(time.perf_counter() - t) * 1e3:.1f} ms", flush=True)
