"""Single-plan latency per kernel: one warp, one CTA (IGP_F_CTA), the
shared-memory CTA kernel (IGP_F_SMEM), the windowed speculative kernel
(IGP_F_WIN) and the grid-cooperative kernel (IGP_F_COOP).

usage: python tools/single_plan.py [cfg ...]   cfg = m[:r_unit[:b_max]] (default: C2 1000, 5000,
       10000, C3 100000:0.01:128).  Device-timed with CUDA events, inputs resident."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import numpy as np  # noqa: E402
from bench_configs import DevicePlan  # noqa: E402

from paper_2211_01713_b200 import synth  # noqa: E402
from paper_2211_01713_b200.layout import hw_vector  # noqa: E402
from paper_2211_01713_b200.planner import IGP_F_COOP, IGP_F_CTA, name_ranks  # noqa: E402
from instances import make_v100  # noqa: E402

IGP_F_WIN = 1 << 28
IGP_F_SMEM = 8
cfgs = sys.argv[1:] or ["1000", "5000", "10000", "100000:0.01:128"]
for c in cfgs:
    parts = c.split(":")
    m = int(parts[0])
    r_unit = float(parts[1]) if len(parts) > 1 else 0.025
    b_max = int(parts[2]) if len(parts) > 2 else 32
    hw = make_v100(r_unit=r_unit)
    kw = dict(slo=(20.0, 100.0), rate=(50.0, 6000.0), b_max=128) if b_max == 128 else {}
    seed = 7 if m == 1000 else 2211
    wl, names = synth.scenarios(1, m, hw, seed=seed, **kw)
    rk = name_ranks(list(names))
    hv = np.array(hw_vector(hw))
    out = {}
    units = {}
    for tag, fl in (("warp", 0), ("cta", IGP_F_CTA), ("smem", IGP_F_SMEM | IGP_F_CTA),
                    ("win", IGP_F_WIN | IGP_F_CTA), ("coop", IGP_F_COOP | IGP_F_CTA)):
        if (tag == "coop" and m < 5000) or (tag == "warp" and m > 2000) or (tag == "win" and m > 20000):
            continue
        dp = DevicePlan(wl, hv, b_max, rk, fl)
        reps = 1 if m >= 50_000 else 5
        out[tag] = dp.time(reps)
        units[tag] = dp.i32[2].cpu().numpy().copy()
        del dp
    same = all(np.array_equal(units[t], units["cta"]) for t in units)
    print(json.dumps(dict(m=m, r_unit=r_unit, b_max=b_max, ms=out,
                          us_per_step={t: v * 1e3 / m for t, v in out.items()},
                          plans_identical=bool(same))), flush=True)
