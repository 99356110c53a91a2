#!/usr/bin/env python
"""Measure every BASELINE.json config on one B200 (bench.py covers the headline).

  C1  paper 4-model mix, 12 workloads: plan() latency through the public API
  C2  1,000 synthetic workloads, r_unit 0.025, b <= 32: single-plan latency
  C3  100,000 workloads, r_unit 0.01, b <= 128: single-plan latency and the
      full solo candidate grid (100,000 x 128 batches x 100 units)
  C4  4,096 independent 1k-workload scenarios: plans/s
  C5  online re-provisioning stream as BASELINE defines it: ONE stream of 1M
      arrivals (C2 generator, seed 5), per-CTA steps for the first 16k
      arrivals then every step on the whole GPU: arrivals/s, bit-exact on a
      24,576-arrival oracle prefix (tools/c5_stream.py)
  C5-tenants  1,000 independent streams x 1,000 arrivals (a tenant batch,
      not C5): arrivals/s
  api   plan_many() through the object API (host marshalling + lazily built
        Plan objects included): plans/s at 148 x 10k
  select  select_gpu_type over 4 GPU types x 1,000 workloads: one launch

Every number is device time (CUDA events on the launching stream, after
warm-up) with inputs resident in HBM unless the line says otherwise.  One JSON
line per config on stdout.  CPU oracle timings are given beside them where
cheap (1 host thread).
"""
import ctypes
import json
import os
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2211_01713_b200 import _device, _native, synth  # noqa: E402
from paper_2211_01713_b200.layout import hw_vector  # noqa: E402
from paper_2211_01713_b200.planner import IGP_F_COOP, IGP_F_CTA, IGP_F_SMEM, IGP_F_STATS, name_ranks  # noqa: E402

dev = torch.device("cuda", 0)
lib = _native.lib_for_compute()
P = _device._ptr


def emit(d):
    print(json.dumps(d), flush=True)


def events():
    return torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


class DevicePlan:
    """Device-resident buffers for repeated igp_plan_batch_device calls."""

    def __init__(self, wl, hv, b_max, rank, flags):
        self.S, _, self.m = wl.shape
        self.hv, self.b_max, self.flags = hv, b_max, flags
        self.d_wl = torch.from_numpy(wl).to(dev)
        self.d_rk = torch.from_numpy(rank).to(dev)
        S, m = self.S, self.m
        self.i32 = torch.empty((5, S, m), dtype=torch.int32, device=dev)
        self.gc = torch.empty(S, dtype=torch.int32, device=dev)
        self.st = torch.empty((S, 6), dtype=torch.int64, device=dev)
        self.err = torch.empty((S, 40), dtype=torch.uint8, device=dev)
        self.ws = torch.empty(max(_device.plan_workspace_bytes(S, m, hv, b_max, fl)
                                  for fl in (flags, flags | IGP_F_STATS)),
                              dtype=torch.uint8, device=dev)

    def run(self, flags=None):
        fl = self.flags if flags is None else flags
        i = self.i32
        rc = lib.igp_plan_batch_device(
            P(self.d_wl), self.S, self.m, _device._np_ptr(self.hv), self.b_max, P(self.d_rk),
            self.m if self.d_rk.dim() == 2 else 0, P(i[0]), P(i[1]), P(i[2]), P(i[3]), P(i[4]),
            ctypes.c_void_p(0), P(self.gc), P(self.st), P(self.err), P(self.ws), self.ws.numel(),
            fl, ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
        assert rc == 0, rc

    def time(self, reps=3):
        self.run()
        torch.cuda.synchronize()
        a, b = events()
        a.record()
        for _ in range(reps):
            self.run()
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) / reps

    def ref_stats(self):
        self.run(self.flags | IGP_F_STATS)
        torch.cuda.synchronize()
        st = self.st.cpu().numpy()
        return dict(model_evals=int(st[:, 0].sum()), candidate_gpus=int(st[:, 1].sum()),
                    eval_calls=int(st[:, 2].sum()), resident_reads=int(st[:, 4].sum()))


def c1():
    import paper_2211_01713_b200 as igp
    from instances import make_v100, twelve_workload_instance
    from oracle import oracle
    hw = make_v100()
    w = twelve_workload_instance()
    for _ in range(5):
        igp.plan(w, hw)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    n = 50
    for _ in range(n):
        p = igp.plan(w, hw)
    api_ms = (time.perf_counter() - t0) / n * 1e3
    wl = np.stack([np.array(igp.planner.workload_table(w))])
    rk = name_ranks([s.name for s, _ in w])
    dp = DevicePlan(wl, np.array(hw_vector(hw)), 32, rk, IGP_F_SMEM | IGP_F_CTA)  # plan()'s kernel
    dev_ms = dp.time(20)
    t0 = time.perf_counter()
    for _ in range(200):
        oracle.plan(wl[0], np.array(hw_vector(hw)), 32, rk)
    cpu_ms = (time.perf_counter() - t0) / 200 * 1e3
    emit(dict(config="C1", workload="twelve_workload_instance (paper Table 3 mix), V100 profile",
              gpus=len(p.gpus), api_ms_per_plan=api_ms, device_ms_per_plan=dev_ms,
              cpu_oracle_ms_per_plan=cpu_ms, cpu_reference_published_ms=3.64,
              note="api = igp.plan() end to end incl. host marshalling and H2D/D2H"))


def c2():
    from instances import make_v100
    hw = make_v100()
    hv = np.array(hw_vector(hw))
    wl, names = synth.scenarios(1, 1000, hw, seed=7)
    rk = name_ranks(list(names))
    out = {}
    for tag, fl in (("warp", 0), ("cta", IGP_F_CTA), ("coop", IGP_F_COOP | IGP_F_CTA),
                    ("smem", IGP_F_SMEM | IGP_F_CTA)):
        dp = DevicePlan(wl, hv, 32, rk, fl)
        out[tag] = dp.time(10)
    st = dp.ref_stats()
    from oracle import oracle
    t0 = time.perf_counter()
    for _ in range(5):
        oracle.plan(wl[0], hv, 32, rk)
    cpu_ms = (time.perf_counter() - t0) / 5 * 1e3
    emit(dict(config="C2", workload="1 plan of 1,000 synthetic workloads, r_unit 0.025, b<=32",
              cpu_oracle_ms_per_plan_1core=cpu_ms,
              ms_per_plan_warp=out["warp"], ms_per_plan_cta=out["cta"],
              ms_per_plan_coop=out["coop"], ms_per_plan_smem=out["smem"],
              kernel_plan_api="smem (IGP_F_SMEM | IGP_F_CTA: shared-memory state, warp per candidate)",
              us_per_step=min(out.values()) * 1e3 / 1000, reference_counters=st,
              candidate_evals_per_s=st["model_evals"] / (min(out.values()) / 1e3)))


def c3():
    from instances import make_v100
    hw = make_v100(r_unit=0.01)
    hv = np.array(hw_vector(hw))
    m = 100_000
    wl, names = synth.scenarios(1, m, hw, seed=2211, slo=(20.0, 100.0), rate=(50.0, 6000.0),
                                b_max=128)
    rk = name_ranks(list(names))
    dp = DevicePlan(wl, hv, 128, rk, IGP_F_CTA | IGP_F_COOP)
    plan_ms = dp.time(1)
    st = dp.ref_stats()
    from oracle import oracle
    sub = np.ascontiguousarray(wl[0][:, :10_000])
    t0 = time.perf_counter()
    o = oracle.plan(sub, hv, 128, name_ranks(list(names[:10_000])))
    cpu_sub = time.perf_counter() - t0
    emit(dict(config="C3-plan",
              cpu_oracle_10k_subset_s=cpu_sub,
              cpu_oracle_10k_subset_evals_per_s=o["model_evals"] / cpu_sub, workload="1 plan of 100,000 workloads, r_unit 0.01, b<=128 "
                                         "(grid-cooperative)",
              ms_per_plan=plan_ms, us_per_step=plan_ms * 1e3 / m, gpus=int(dp.gc[0].item()),
              reference_counters=st, candidate_evals_per_s=st["model_evals"] / (plan_ms / 1e3),
              cpu_oracle_s_per_plan=162.0,
              cpu_oracle_note="tests/golden/make_c3_100k.py on 1 core of the build container"))
    # full solo candidate grid
    d_wl = torch.from_numpy(np.ascontiguousarray(wl[0])).to(dev)
    d_min = torch.empty((m, 128), dtype=torch.int32, device=dev)
    d_best = torch.empty((2, m), dtype=torch.int32, device=dev)
    d_ev = torch.zeros(1, dtype=torch.int64, device=dev)
    s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)

    def grid(ev):
        rc = lib.igp_solo_grid_device(P(d_wl), m, _device._np_ptr(hv), 128, P(d_min), P(d_best[0]),
                                      P(d_best[1]), P(d_ev) if ev else ctypes.c_void_p(0), s)
        assert rc == 0
    grid(True)
    torch.cuda.synchronize()
    evals = int(d_ev.item())
    a, b = events()
    a.record()
    for _ in range(5):
        grid(False)
    b.record()
    torch.cuda.synchronize()
    g_ms = a.elapsed_time(b) / 5
    points = m * 128 * 100
    emit(dict(config="C3-grid", workload="solo grid 100,000 workloads x b 1..128 x u 1..100",
              ms=g_ms, grid_points=points, grid_points_per_s=points / (g_ms / 1e3),
              points_evaluated=evals, evaluated_per_s=evals / (g_ms / 1e3),
              note="scan stops at the first feasible u per (w, b) like best_group_alloc"))


def c3grid():
    """Only the solo grid of C3 (for a focused ncu capture)."""
    from instances import make_v100
    hw = make_v100(r_unit=0.01)
    hv = np.array(hw_vector(hw))
    m = 100_000
    wl, _ = synth.scenarios(1, m, hw, seed=2211, slo=(20.0, 100.0), rate=(50.0, 6000.0), b_max=128)
    r = _device.solo_grid(wl[0], hv, 128)
    emit(dict(config="C3-grid-only", feasible_points=int((r["min_units"] > 0).sum())))


def c4():
    from instances import make_v100
    hw = make_v100()
    hv = np.array(hw_vector(hw))
    wl, names = synth.scenarios(4096, 1000, hw, seed=4096)
    rk = name_ranks(list(names))
    dp = DevicePlan(wl, hv, 32, rk, 0)
    ms = dp.time(3)
    st = dp.ref_stats()
    from oracle import oracle
    threads = os.cpu_count() or 1
    n_cpu = max(64, threads)
    t0 = time.perf_counter()
    oracle.plan_batch(wl[:n_cpu], hv, 32, rk, threads)
    cpu_s = time.perf_counter() - t0
    emit(dict(config="C4", cpu_oracle_plans_per_s=n_cpu / cpu_s, cpu_threads=threads,
              cpu_sample=f"{n_cpu} scenarios on {threads} threads", workload="4,096 scenarios x 1,000 workloads, 1 GPU (bench.py --gpus N shards)",
              ms=ms, plans_per_s=4096 / (ms / 1e3), reference_counters=st,
              candidate_evals_per_s=st["model_evals"] / (ms / 1e3)))


def c5():
    import subprocess
    out = subprocess.run([sys.executable, os.path.join(REPO, "tools", "c5_stream.py"), "1000000",
                          "4096", "--check", "24576"], capture_output=True, text=True, check=True)
    d = json.loads(out.stdout.strip().splitlines()[-1])
    d["config"] = "C5"
    d["workload"] = "one stream of 1M arrivals (C2 generator seed 5), arrival order, pushes of 4096"
    emit(d)


def c5tenants():
    from instances import make_v100
    from paper_2211_01713_b200.stream import StreamPlanner
    hw = make_v100()
    S, L, chunk = 1000, 1000, 100
    wl, _ = synth.scenarios(S, L, hw, seed=5)
    d_wl = torch.from_numpy(wl).to(dev)
    chunks = [d_wl[:, :, k:k + chunk].contiguous() for k in range(0, L, chunk)]
    by_width = {}
    for tag, fl in (("1 warp", 0), ("2 warps", 32), ("4 warps", 64)):
        sp = StreamPlanner(hw, capacity=L, n_streams=S, flags=fl)
        for c in chunks:  # warm-up pass
            sp.push_device(c)
        torch.cuda.synchronize()
        sp.reset()
        a, b = events()
        a.record()
        for c in chunks:
            sp.push_device(c)
        b.record()
        torch.cuda.synchronize()
        by_width[tag] = a.elapsed_time(b)
        del sp
        torch.cuda.empty_cache()
    best = min(by_width, key=by_width.get)
    ms = by_width[best]
    from oracle import oracle
    from paper_2211_01713_b200.layout import hw_vector as _hv
    t0 = time.perf_counter()
    oracle.stream(wl[0], np.array(_hv(hw)), 32)
    cpu_s = time.perf_counter() - t0
    emit(dict(config="C5-tenants", cpu_oracle_arrivals_per_s_1core=L / cpu_s,
              workload=f"{S} independent streams x {L} arrivals (a tenant batch, not BASELINE C5), "
                       f"pushes of {chunk} arrivals per stream",
              ms=ms, arrivals_per_s=S * L / (ms / 1e3), us_per_push=ms * 1e3 / len(chunks),
              group_width=best, ms_by_group_width=by_width,
              multi_gpu="independent streams shard across ranks (SURVEY §8e option B)"))


def api():
    """plan_many through the object API: (spec, coef) objects in, Plan objects out."""
    import paper_2211_01713_b200 as igp
    from instances import make_v100
    hw = make_v100()
    S, m = 148, 10_000
    wl, names = synth.scenario_batch(S, m, hw, seed=2211)
    scen = []
    for s_ in range(S):
        scen.append([(igp.WorkloadSpec(str(names[i]), *map(float, wl[s_, :4, i])),
                      igp.WorkloadCoefficients(int(wl[s_, 4, i]), *map(float, wl[s_, 5:, i])))
                     for i in range(m)])
    igp.plan_many(scen[:8], hw)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    plans = igp.plan_many(scen, hw)
    dt = time.perf_counter() - t0
    t1 = time.perf_counter()
    n_alloc = sum(len(g.allocations) for g in plans[0].gpus)
    mat_ms = (time.perf_counter() - t1) * 1e3
    t0 = time.perf_counter()
    tabs = [igp.planner.workload_table(sc) for sc in scen[:16]]
    marshal_ms = (time.perf_counter() - t0) / 16 * 1e3
    emit(dict(config="api", workload=f"plan_many({S} scenarios x {m} workloads) via the object API",
              plans_per_s=S / dt, s=dt, host_marshal_ms_per_10k_plan=marshal_ms,
              plan_object_materialise_ms_per_10k_plan=mat_ms, allocations_plan0=n_alloc,
              note="includes workload_table/name ranks per scenario, H2D, kernels, D2H; Plan "
                   "objects are built lazily on first access of .gpus"))
    del tabs


def select():
    """select_gpu_type over 4 types in one launch vs one plan() per type."""
    import paper_2211_01713_b200 as igp
    from instances import make_v100, random_instance
    rng = np.random.default_rng(3)
    base = random_instance(rng, 1000, make_v100())
    specs = [s for s, _ in base]
    types = [make_v100(gpu_type="a"), make_v100(gpu_type="b", r_unit=0.01, price_per_hour=2.9),
             make_v100(gpu_type="c", power_max_w=150.0, price_per_hour=2.5),
             make_v100(gpu_type="d", r_unit=0.05, price_per_hour=2.2)]
    coefs = {hw.gpu_type: {s.name: c for s, c in base} for hw in types}
    igp.select_gpu_type(specs, types, coefs)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5):
        best = igp.select_gpu_type(specs, types, coefs)
    one = (time.perf_counter() - t0) / 5
    t0 = time.perf_counter()
    for _ in range(5):
        for hw in types:
            igp.plan([(s, coefs[hw.gpu_type][s.name]) for s in specs], hw)
    seq = (time.perf_counter() - t0) / 5
    emit(dict(config="select", workload="select_gpu_type, 4 GPU types x 1,000 workloads",
              ms_one_launch=one * 1e3, ms_sequential_plans=seq * 1e3, chosen=best.gpu_type,
              gpus=best.gpu_count))


if __name__ == "__main__":
    which = sys.argv[1:] or ["c1", "c2", "c3", "c4", "c5", "c5tenants", "api", "select"]
    torch.cuda.set_device(0)
    for w in which:
        globals()[w]()
