"""Reference-run fixtures at the headline size (10,000 workloads) and a
reference-run prefix of the C3 100k instance.

Run from the repo root (needs /root/reference, which is NOT on the GPU box;
about 2 min + 2-5 min of CPython):

    python tests/golden/make_ref_10k.py            # both fixtures
    python tests/golden/make_ref_10k.py 10k        # only ref_plan_10k.npz
    python tests/golden/make_ref_10k.py prefix     # only c3_prefix_ref.npz

ref_plan_10k.npz  -- the UNMODIFIED reference ``plan()`` (with PlanStats) on
    scenario 0 of bench.py's batch: ``synth.scenario_batch(S, 10000, V100,
    seed=2211, indices=[0])`` (per-scenario seeds, so the instance does not
    depend on S).  Stored: the workload table, every output in input order
    and all ten _build_plan breakdown fields, the counters and the CPython
    runtime.  Checked against the oracle (CPU) and the B200 (GPU tests).

c3_prefix_ref.npz -- the reference ``plan()`` on the top-K workloads (sorted
    by (-lb, name), planner.py:284) of the C3 100,000-workload instance of
    make_c3_100k.py (r_unit 0.01, b <= 128).  K = 45,000: the first ~40,000
    sorted workloads need more than half a device each, so real packing starts
    near there.  By the greedy prefix
    property these are exactly the full plan's first K steps; the fixture pins
    the oracle and the B200 on that prefix with the reference's own output.
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, HERE)

assert sys.version_info >= (3, 12), "golden fixtures need CPython >= 3.12 (Neumaier sum)"

M10K, SEED10K, S_BENCH = 10_000, 2211, 2368
K_PREFIX = int(os.environ.get("K_PREFIX", "45000"))


def to_reference(wl, names, gp):
    from paper_2211_01713_b200.layout import WL_FIELDS
    out = []
    for i in range(wl.shape[1]):
        f = {k: float(wl[j, i]) for j, k in enumerate(WL_FIELDS)}
        out.append((gp.WorkloadSpec(str(names[i]), f["slo_ms"], f["rate_rps"], f["d_load_mb"],
                                    f["d_feedback_mb"]),
                    gp.WorkloadCoefficients(int(f["n_kernels"]), f["k_sch_ms"], f["k1"], f["k2"],
                                            f["k3"], f["k4"], f["k5"], f["alpha_power_w"],
                                            f["beta_power_w"], f["alpha_cacheutil"],
                                            f["beta_cacheutil"], f["alpha_cache"])))
    return out


def ref_10k():
    import make_golden as mg
    from paper_2211_01713_b200 import synth
    from instances import make_v100
    hw_ours = make_v100()
    wl, names = synth.scenario_batch(S_BENCH, M10K, hw_ours, seed=SEED10K, indices=[0])
    wl = wl[0]
    ghw = mg.gp.HardwareProfile(**{k: getattr(hw_ours, k) for k in hw_ours.__dataclass_fields__})
    workloads = to_reference(wl, names, mg.gp)
    out, dt = mg.run_plan_case(workloads, ghw, b_max=32)
    assert str(out["err_class"]) == "", out["err_msg"]
    out["wl"] = wl
    out["seed"] = np.int64(SEED10K)
    out["scenario"] = np.int64(0)
    print(f"reference plan(10k): {int(out['gpu_count'])} GPUs, model_evals "
          f"{int(out['model_evals'])}, candidate_gpus {int(out['candidate_gpus'])}, {dt:.1f} s")
    np.savez_compressed(os.path.join(HERE, "ref_plan_10k.npz"), **out)


def c3_prefix():
    import make_c3_100k as c3
    import make_golden as mg
    from oracle import oracle
    from paper_2211_01713_b200.layout import hw_vector
    hw, wl, names = c3.instance()
    hv = np.array(hw_vector(hw))
    b, lb, code = oracle.prologue(wl, hv, c3.B_MAX)
    assert (code == 0).all()
    order = sorted(range(c3.M), key=lambda i: (-int(lb[i]), names[i]))[:K_PREFIX]
    sub = wl[:, order]
    sub_names = [names[i] for i in order]
    ghw = mg.gp.HardwareProfile(**{k: getattr(hw, k) for k in hw.__dataclass_fields__})
    out, dt = mg.run_plan_case(to_reference(sub, sub_names, mg.gp), ghw, b_max=c3.B_MAX)
    assert str(out["err_class"]) == "", out["err_msg"]
    print(f"reference plan(top-{K_PREFIX} of C3 100k): {int(out['gpu_count'])} GPUs, "
          f"model_evals {int(out['model_evals'])}, {dt:.1f} s")
    np.savez_compressed(
        os.path.join(HERE, "c3_prefix_ref.npz"), order=np.array(order, np.int32),
        gpu_of=out["gpu_of"], pos=out["pos"], units=out["units"].astype(np.int16),
        batch=out["batch"].astype(np.int16), lb=out["lb"].astype(np.int16), pred=out["pred"],
        gpu_count=out["gpu_count"],
        model_evals=out["model_evals"], candidate_gpus=out["candidate_gpus"],
        ref_seconds=out["ref_seconds"], k=np.int64(K_PREFIX), seed=np.int64(c3.SEED),
        m=np.int64(c3.M), b_max=np.int64(c3.B_MAX))


if __name__ == "__main__":
    what = sys.argv[1] if len(sys.argv) > 1 else "all"
    if what in ("all", "10k"):
        ref_10k()
    if what in ("all", "prefix"):
        c3_prefix()
