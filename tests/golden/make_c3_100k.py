"""C3 fixture: one 100,000-workload plan (r_unit 0.01, b <= 128) by the CPU oracle.

Run from the repo root (CPU only, a few minutes):  python tests/golden/make_c3_100k.py

The instance is regenerated from its seed by paper_2211_01713_b200.synth (C3
distributions: slo U(20,100) ms, rate U(50,6000) req/s, rejection through
Eq. 19/20 at b_max 128), so only the plan is stored.  Names are w{i:04d} as
in the reference generator (support.py:102), so beyond 10,000 workloads the
name tie-break order differs from index order (SURVEY.md finding 9).

The oracle itself is pinned against the reference's own plan() on the
C3-style fixtures (plan_c3style_800.npz); when /root/reference is present
this script additionally runs the reference plan() on the first K workloads
of the sorted order and checks the oracle against it on that prefix.
"""
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.dirname(HERE))

from oracle import oracle  # noqa: E402
from paper_2211_01713_b200 import synth  # noqa: E402
from paper_2211_01713_b200.layout import hw_vector  # noqa: E402
from instances import make_v100  # noqa: E402

M, SEED, B_MAX = 100_000, 2211, 128


def instance():
    hw = make_v100(r_unit=0.01)
    wl, names = synth.scenarios(1, M, hw, seed=SEED, slo=(20.0, 100.0), rate=(50.0, 6000.0),
                                b_max=B_MAX)
    return hw, wl[0], list(names)


def main():
    hw, wl, names = instance()
    rank = oracle.name_ranks(names)
    t0 = time.perf_counter()
    o = oracle.plan(wl, np.array(hw_vector(hw)), B_MAX, rank)
    dt = time.perf_counter() - t0
    assert o["rc"] == 0, o["err"]
    print(f"oracle plan: {o['gpu_count']} GPUs, evals {o['model_evals']}, "
          f"cands {o['candidate_gpus']}, {dt:.1f} s")
    np.savez_compressed(os.path.join(HERE, "c3_plan_100k.npz"),
                        gpu_of=o["gpu_of"], pos=o["pos"], units=o["units"].astype(np.int16),
                        batch=o["batch"].astype(np.int16), lb=o["lb"].astype(np.int16),
                        pred_t_inf=o["pred"][:, 6], gpu_count=np.int64(o["gpu_count"]),
                        model_evals=np.int64(o["model_evals"]),
                        candidate_gpus=np.int64(o["candidate_gpus"]),
                        seed=np.int64(SEED), m=np.int64(M), b_max=np.int64(B_MAX),
                        oracle_seconds=np.float64(dt))
    if os.path.isdir("/root/reference/pkg/src") and len(sys.argv) > 1:
        prefix_check(hw, wl, names, o, int(sys.argv[1]))


def prefix_check(hw, wl, names, o, K):
    """Reference plan() on the top-K workloads of the sorted order equals the
    oracle on the same K (greedy prefix property, SURVEY.md finding 7)."""
    sys.path.insert(0, "/root/reference/pkg/src")
    import gpuplanner as gp
    from paper_2211_01713_b200.layout import WL_FIELDS
    order = sorted(range(M), key=lambda i: (-int(o["lb"][i]), names[i]))[:K]
    specs = []
    for i in order:
        f = {k: float(wl[j, i]) for j, k in enumerate(WL_FIELDS)}
        specs.append((gp.WorkloadSpec(names[i], f["slo_ms"], f["rate_rps"], f["d_load_mb"],
                                      f["d_feedback_mb"]),
                      gp.WorkloadCoefficients(int(f["n_kernels"]), f["k_sch_ms"], f["k1"], f["k2"],
                                              f["k3"], f["k4"], f["k5"], f["alpha_power_w"],
                                              f["beta_power_w"], f["alpha_cacheutil"],
                                              f["beta_cacheutil"], f["alpha_cache"])))
    ghw = gp.HardwareProfile(**{k: getattr(hw, k) for k in hw.__dataclass_fields__})
    t0 = time.perf_counter()
    p = gp.plan(specs, ghw, b_max=B_MAX)
    dt = time.perf_counter() - t0
    sub = wl[:, order]
    op = oracle.plan(sub, np.array(hw_vector(hw)), B_MAX, oracle.name_ranks([names[i] for i in order]))
    ref_units = {a.workload: round(a.r / hw.r_unit) for g in p.gpus for a in g.allocations}
    ref_gpu = {a.workload: g.gpu_index for g in p.gpus for a in g.allocations}
    ok = all(ref_units[names[i]] == op["units"][k] and ref_gpu[names[i]] == op["gpu_of"][k]
             for k, i in enumerate(order))
    print(f"prefix K={K}: reference {len(p.gpus)} GPUs in {dt:.1f} s; oracle matches: {ok}")
    assert ok


if __name__ == "__main__":
    main()
