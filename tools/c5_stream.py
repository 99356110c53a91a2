"""BASELINE config 5 as specified: ONE online stream of N arrivals (C2
generator, seed 5, arrival order) on one B200, pushed in fixed-size pushes.

  python tools/c5_stream.py [N=1000000] [push=4096] [--check K]

Prints one JSON line: arrivals/s over the whole stream (device-timed with CUDA
events around every push, inputs resident in HBM), the per-segment rates, the
GPU count, and -- with --check K -- a bit-exact comparison of the first K
arrivals' admissions against the CPU oracle's arrival-order driver (plus the
oracle's arrivals/s on one core).  COOP_FROM / CTAS env vars override the
whole-GPU policy of stream.push_flags for A/B runs."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2211_01713_b200 import stream as stream_mod, synth  # noqa: E402
from paper_2211_01713_b200.layout import hw_vector  # noqa: E402
from paper_2211_01713_b200.model import HardwareProfile  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
N = int(args[0]) if args else 1_000_000
PUSH = int(args[1]) if len(args) > 1 else 4096
CHECK = int(sys.argv[sys.argv.index("--check") + 1]) if "--check" in sys.argv else 0
if "COOP_FROM" in os.environ:
    stream_mod.COOP_FROM_ARRIVALS = int(os.environ["COOP_FROM"])
if "CTAS" in os.environ:
    stream_mod.coop_ctas = lambda k: int(os.environ["CTAS"])
hw = HardwareProfile("v100", 300.0, 1530.0, 53.5, 10.0, -1.025, 0.00475, -0.00902,
                     r_unit=0.025, price_per_hour=3.06)
N = (N // PUSH) * PUSH
t0 = time.perf_counter()
wl, _ = synth.scenarios(1, N, hw, seed=5)
gen_s = time.perf_counter() - t0
d_wl = torch.from_numpy(np.ascontiguousarray(
    wl[0].reshape(16, N // PUSH, PUSH).transpose(1, 0, 2))).cuda()
sp = stream_mod.StreamPlanner(hw, capacity=N, whole_gpu=True)
evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
       for _ in range(N // PUSH)]
outs = []
torch.cuda.synchronize()
for c in range(N // PUSH):
    evs[c][0].record()
    g, p, cd = sp.push_device(d_wl[c][None])
    evs[c][1].record()
    outs.append((g.clone(), p.clone(), cd.clone()) if CHECK and c * PUSH < CHECK else None)
torch.cuda.synchronize()
sp.check_errors()
ms = np.array([a.elapsed_time(b) for a, b in evs])
snap = sp.snapshot()
segs = {}
for lo, hi in ((0, 10_000), (10_000, 100_000), (100_000, 500_000), (500_000, N)):
    sel = [c for c in range(N // PUSH) if lo <= c * PUSH < hi]
    if sel:
        segs[f"{lo}-{hi}"] = {"arrivals_per_s": len(sel) * PUSH / (ms[sel].sum() / 1e3),
                              "us_per_arrival": ms[sel].sum() * 1e3 / (len(sel) * PUSH)}
line = {"config": "C5: one stream of %d arrivals (C2 generator seed 5, arrival order)" % N,
        "arrivals_per_s": N / (ms.sum() / 1e3), "seconds": ms.sum() / 1e3, "push": PUSH,
        "gpu_count": int(snap["gpu_count"][0]), "segments": segs,
        "policy": {"coop_from": stream_mod.COOP_FROM_ARRIVALS,
                   "ctas_at_end": stream_mod.coop_ctas(N)},
        "generate_s": gen_s}
if CHECK:
    from oracle import oracle
    K = (CHECK // PUSH) * PUSH
    t0 = time.perf_counter()
    o = oracle.stream(wl[0][:, :K], np.array(hw_vector(hw)), 32)
    line["oracle_arrivals_per_s_1core"] = K / (time.perf_counter() - t0)
    g = np.concatenate([x[0].cpu().numpy()[0] for x in outs if x is not None])[:K]
    p = np.concatenate([x[1].cpu().numpy()[0] for x in outs if x is not None])[:K]
    cd = np.concatenate([x[2].cpu().numpy()[0] & 0xFF for x in outs if x is not None])[:K]
    ok = (np.array_equal(g, o["gpu_of"]) and np.array_equal(p, o["pos"]) and
          np.array_equal(cd, o["code"]))
    line["check"] = {"arrivals": K, "bit_exact_admissions": bool(ok),
                     "oracle_model_evals": o["model_evals"],
                     "oracle_candidate_gpus": o["candidate_gpus"]}
print(json.dumps(line), flush=True)
