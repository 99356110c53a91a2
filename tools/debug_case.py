"""Compare one golden plan case through the device path in fast and exact modes; print diffs."""
import os, sys
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO); sys.path.insert(0, os.path.join(REPO, "tests"))
import numpy as np
import golden_io as G
from paper_2211_01713_b200 import _device
from paper_2211_01713_b200.planner import name_ranks
case = sys.argv[1] if len(sys.argv) > 1 else "plan_c1_twelve"
d = G.load(case)
rank = name_ranks([str(x) for x in d["names"]])
for flags in (0, 1, 4, 5):
    r = _device.plan_device(d["wl"], d["hw"], int(d["b_max"]), rank, flags=flags)
    msg = []
    for k in ("gpu_of", "pos", "units", "batch", "lb"):
        if not np.array_equal(r[k][0], d[k]):
            msg.append(f"{k}: got {r[k][0][:20]} want {d[k][:20]}")
    if not np.array_equal(r["pred"][0].view(np.int64), d["pred"].view(np.int64)):
        bad = np.nonzero((r["pred"][0] != d["pred"]).any(1))[0]
        msg.append(f"pred rows differ: {bad[:10]}")
    msg.append(f"stats {r['stats'][0].tolist()} want {int(d['model_evals'])},{int(d['candidate_gpus'])} err {r['err'][0]['code']}")
    print(case, "flags", flags, "|", " ; ".join(msg))
