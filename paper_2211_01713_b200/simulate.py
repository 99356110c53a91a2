"""Deterministic request-level replay of a plan (drop-in for ``gpuplanner.simulate``).

Every workload of a plan is served by one process. Requests queue until a full
batch is waiting and the server is idle; the whole batch then runs for the
predicted inference latency of that device's co-location state (``t_inf``
from ``predict_gpu``, evaluated on the device). End-to-end latency covers
batch formation, queueing and execution, and is judged against the full SLO
(``simulate.py:1-8``).

The replay of all workloads, the per-workload sort of measured latencies and
the percentiles run in one device call (``igp_simulate_device``). They follow
``simulate._run_workload`` (``simulate.py:98-136``) and the report of
``simulate.simulate`` (``simulate.py:139-198``). Poisson arrivals behave as
in the reference on CPython >= 3.11: its tuple seed
(``random.Random((seed, offset))``, ``simulate.py:86``) raises ``TypeError``.
"""

from __future__ import annotations

import math
import random
from dataclasses import dataclass
from typing import Mapping

import numpy as np

from . import _device, _native
from .errors import UnstableQueueError
from .model import predict_gpu

UNSTABLE_QUEUE_FACTOR = 10


@dataclass(frozen=True)
class SimConfig:
    duration_ms: float
    warmup_ms: float = 0.0
    arrival: str = "constant"  # "constant" or "poisson"
    seed: int = 0

    def __post_init__(self):
        if not 0 <= self.warmup_ms <= self.duration_ms:
            raise ValueError("requires duration_ms >= warmup_ms >= 0")
        if self.arrival not in ("constant", "poisson"):
            raise ValueError(f"unknown arrival process: {self.arrival}")


@dataclass(frozen=True)
class RequestRecord:
    workload: str
    arrival_ms: float
    dispatch_ms: float
    complete_ms: float


@dataclass(frozen=True)
class WorkloadReport:
    workload: str
    offered_rps: float
    achieved_rps: float
    p50_ms: float
    p99_ms: float
    max_queue_depth: int
    completed: int
    violation: bool  # p99 beyond the full latency SLO


@dataclass(frozen=True)
class SimReport:
    duration_ms: float
    warmup_ms: float
    workloads: list[WorkloadReport]

    @property
    def violations(self) -> list[str]:
        return [w.workload for w in self.workloads if w.violation]


def replay_arrays(rate_rps, batch, service_ms, cfg: SimConfig, device=None, *, starts=False):
    """Device replay of n workloads; numpy arrays in, dict of numpy arrays out.
    With starts=True the result also holds every batch's start time
    (``starts``, workload w's batches from ``seg[w]``)."""
    torch = _device._torch()
    lib = _native.lib_for_compute()
    device = _device._dev(device)
    rate = np.ascontiguousarray(rate_rps, np.float64)
    n = len(rate)
    bound = np.array([math.ceil(cfg.duration_ms * r / 1000.0) + 2 for r in rate], np.int64)
    seg = np.zeros(n + 1, np.int64)
    np.cumsum(bound, out=seg[1:])
    total = int(seg[-1]) if n else 0
    with torch.cuda.device(device):
        d = {k: _device._to_dev(v, device) for k, v in (
            ("rate", rate), ("batch", np.asarray(batch, np.int32)),
            ("service", np.asarray(service_ms, np.float64)), ("seg", seg))}
        scratch = torch.empty((3, max(total, 1)), dtype=torch.float64, device=device)
        seg_end = torch.empty(max(n, 1), dtype=torch.int64, device=device)
        i32 = torch.empty((3, max(n, 1)), dtype=torch.int32, device=device)
        f64 = torch.empty((3, max(n, 1)), dtype=torch.float64, device=device)
        P = _device._ptr
        rc = lib.igp_simulate_device(n, P(d["rate"]), P(d["batch"]), P(d["service"]),
                                     float(cfg.duration_ms), float(cfg.warmup_ms), P(d["seg"]),
                                     P(scratch[0]), P(scratch[1]), P(scratch[2]), P(seg_end),
                                     P(i32[0]), P(i32[1]), P(i32[2]), P(f64[0]), P(f64[1]),
                                     P(f64[2]), _device._stream(device))
        _device._check(rc)
        oi = i32.cpu().numpy()[:, :n]
        of = f64.cpu().numpy()[:, :n]
        out = dict(max_depth=oi[0], backlog=oi[1], completed=oi[2], p50=of[0], p99=of[1],
                   achieved=of[2])
        if starts:
            out.update(starts=scratch[1].cpu().numpy(), seg=seg)
    return out


def arrival_count(rate_rps: float, duration_ms: float) -> int:
    """Number of constant-rate arrivals t_k = k * (1000 / rate) < duration
    (``_arrival_times``, simulate.py:79-85), without the loop."""
    if not duration_ms > 0.0:
        return 0
    spacing = 1000.0 / rate_rps
    k = max(1, math.ceil(duration_ms / spacing))
    while k * spacing < duration_ms:
        k += 1
    while k > 1 and (k - 1) * spacing >= duration_ms:
        k -= 1
    return k


def _workload_trace(name, rate_rps, batch, service_ms, starts, cfg):
    """The RequestRecords of one workload in the reference's order
    (simulate.py:118-124): batch after batch, members in arrival order."""
    spacing = 1000.0 / rate_rps
    out = []
    for q in range(arrival_count(rate_rps, cfg.duration_ms) // batch):
        start = float(starts[q])
        done = start + service_ms
        out.extend(RequestRecord(name, r * spacing if r else 0.0, start, done)
                   for r in range(q * batch, (q + 1) * batch))
    return out


def write_trace_csv(path, trace) -> None:
    """Per-request trace: workload,arrival_ms,dispatch_ms,complete_ms (simulate.py:201-209)."""
    with open(path, "w") as handle:
        handle.write("workload,arrival_ms,dispatch_ms,complete_ms\n")
        for r in trace:
            handle.write(f"{r.workload},{r.arrival_ms!r},{r.dispatch_ms!r},{r.complete_ms!r}\n")


def simulate(plan, specs: Mapping, coefs: Mapping, hw, cfg: SimConfig, *, collect_trace: bool = False):
    """Replay every workload of a plan; interference is frozen at plan time.
    With collect_trace=True returns (report, trace) like the reference
    (simulate.py:192-198); the trace is rebuilt from the device's batch start
    times (arrival k at k * spacing, completion at start + t_inf)."""
    items = []  # (name, batch, service t_inf)
    for gpu in plan.gpus:
        predicted = predict_gpu(gpu.allocations, specs, coefs, hw)
        for alloc in gpu.allocations:
            items.append((alloc.workload, alloc.batch, predicted[alloc.workload].t_inf_ms))
    items.sort()
    if cfg.arrival == "poisson" and items:
        random.Random((cfg.seed, 0))  # the reference's seed: TypeError on CPython >= 3.11
    r = replay_arrays([specs[n].rate_rps for n, _, _ in items], [b for _, b, _ in items],
                      [s for _, _, s in items], cfg, starts=collect_trace)
    reports = []
    trace = []
    for i, (name, batch, _) in enumerate(items):
        if int(r["backlog"][i]) > UNSTABLE_QUEUE_FACTOR * batch:
            raise UnstableQueueError(name, int(r["backlog"][i]), UNSTABLE_QUEUE_FACTOR * batch)
        done = int(r["completed"][i])
        p99 = float(r["p99"][i])
        reports.append(WorkloadReport(
            workload=name, offered_rps=specs[name].rate_rps, achieved_rps=float(r["achieved"][i]),
            p50_ms=float(r["p50"][i]), p99_ms=p99, max_queue_depth=int(r["max_depth"][i]),
            completed=done, violation=bool(done) and p99 > specs[name].slo_ms))
        if collect_trace:
            trace.extend(_workload_trace(name, specs[name].rate_rps, batch, items[i][2],
                                         r["starts"][r["seg"][i]:], cfg))
    report = SimReport(cfg.duration_ms, cfg.warmup_ms, reports)
    if collect_trace:
        return report, trace
    return report
