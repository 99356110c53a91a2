#!/usr/bin/env python
"""Measure every BASELINE.json config on one B200 (bench.py covers the headline).

  C1  paper 4-model mix, 12 workloads: plan() latency through the public API
  C2  1,000 synthetic workloads, r_unit 0.025, b <= 32: single-plan latency
  C3  100,000 workloads, r_unit 0.01, b <= 128: single-plan latency and the
      full solo candidate grid (100,000 x 128 batches x 100 units)
  C4  4,096 independent 1k-workload scenarios: plans/s
  C5  online stream: 1,000 streams x 1,000 arrivals (1M arrivals), pushed 100
      arrivals at a time: arrivals/s

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
from paper_2211_01713_b200.planner import IGP_F_COOP, IGP_F_CTA, IGP_F_STATS, name_ranks  # noqa: E402

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
        self.ws = torch.empty(_device.plan_workspace_bytes(S, m, hv, b_max, flags | IGP_F_STATS),
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
    dp = DevicePlan(wl, np.array(hw_vector(hw)), 32, rk, 0)
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
    for tag, fl in (("warp", 0), ("cta", IGP_F_CTA), ("coop", IGP_F_COOP | IGP_F_CTA)):
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
              ms_per_plan_coop=out["coop"],
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
    sp = StreamPlanner(hw, capacity=L, n_streams=S, flags={"1 warp": 0, "2 warps": 32, "4 warps": 64}[best])
    for c in chunks:
        sp.push_device(c)
    snap = sp.snapshot()
    from oracle import oracle
    from paper_2211_01713_b200.layout import hw_vector as _hv
    t0 = time.perf_counter()
    oracle.stream(wl[0], np.array(_hv(hw)), 32)
    cpu_s = time.perf_counter() - t0
    emit(dict(config="C5", cpu_oracle_arrivals_per_s_1core=L / cpu_s,
              cpu_sample=f"one stream of {L} arrivals on 1 core", workload=f"{S} independent streams x {L} arrivals = {S * L} arrivals, "
                                    f"pushes of {chunk} arrivals per stream",
              ms=ms, arrivals_per_s=S * L / (ms / 1e3), us_per_push=ms * 1e3 / len(chunks),
              group_width=best, ms_by_group_width=by_width,
              gpus_open=int(snap["gpu_count"].sum()),
              rejected=int((snap["gpu_of"] < 0).sum()),
              multi_gpu="independent streams shard across ranks (SURVEY §8e option B)"))


if __name__ == "__main__":
    which = sys.argv[1:] or ["c1", "c2", "c3", "c4", "c5"]
    torch.cuda.set_device(0)
    for w in which:
        globals()[w]()
