"""Generate golden fixtures by running the UNMODIFIED reference in this container.

Run from the repo root (needs /root/reference, which is NOT on the GPU box):

    python tests/golden/make_golden.py

It imports ``gpuplanner`` read-only from ``/root/reference/pkg/src`` and the
reference's own test generators from ``/root/reference/pkg/tests/support.py``
(``random_instance`` ``support.py:190-195``, ``twelve_workload_instance``
``support.py:232-243``, ``make_v100`` ``support.py:122-125``), runs the
reference ``plan()`` / ``predict_gpu()`` / ``alloc_gpus()`` /
``appropriate_batch()`` / ``_lower_bound_units()`` and freezes inputs and
outputs as ``.npz`` files next to this script.  The fixtures are what the
oracle is pinned against (tests/test_oracle_golden.py) and what the CUDA
path is checked against on the GPU box (tests/test_gpu_parity.py).

CPython must be 3.12+: builtin ``sum`` of floats is Neumaier-compensated
from 3.12 on and the reference depends on it (SURVEY.md finding 1).
"""

from __future__ import annotations

import dataclasses
import json
import math
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, "/root/reference/pkg/tests")

assert sys.version_info >= (3, 12), "golden fixtures need CPython >= 3.12 (Neumaier sum)"

import gpuplanner as gp  # noqa: E402
from gpuplanner import errors as gerr  # noqa: E402
from gpuplanner import model as gmodel  # noqa: E402
from gpuplanner import planner as gplanner  # noqa: E402
import support  # noqa: E402

from paper_2211_01713_b200 import layout  # noqa: E402

ERR_CODE = {
    "BatchCapExceededError": layout.E_BATCH_CAP,
    "InfeasibleSloError": layout.E_INFEASIBLE_SLO,
    "InfeasibleResourceError": layout.E_INFEASIBLE_RES,
    "NonPositiveDenominatorError": None,  # resolved from the message
    "OverAllocatedError": layout.E_OVERALLOC,
}


def err_code(exc):
    name = type(exc).__name__
    if name == "NonPositiveDenominatorError":
        return layout.E_DENOM if str(exc).startswith("r + k4") else layout.E_ACTIVE_TIME
    return ERR_CODE[name]


def pack_instance(workloads, hw, b_max):
    m = len(workloads)
    wl = np.zeros((layout.WL_NF, m), dtype=np.float64)
    for i, (s, c) in enumerate(workloads):
        wl[:, i] = layout.spec_coef_row(s, c)
    names = np.array([s.name for s, _ in workloads])
    return dict(
        wl=wl, names=names, hw=np.array(layout.hw_vector(hw)),
        gpu_type=np.array(hw.gpu_type), b_max=np.int64(b_max),
    )


def run_plan_case(workloads, hw, b_max=32):
    """Reference plan() with stats; outputs re-indexed by input order."""
    out = pack_instance(workloads, hw, b_max)
    m = len(workloads)
    stats = gplanner.PlanStats()
    t0 = time.perf_counter()
    try:
        p = gp.plan(workloads, hw, b_max=b_max, stats=stats)
    except gerr.GpuPlannerError as exc:
        out.update(err_class=np.array(type(exc).__name__), err_msg=np.array(str(exc)),
                   err_code=np.int64(err_code(exc)),
                   model_evals=np.int64(stats.model_evals),
                   candidate_gpus=np.int64(stats.candidate_gpus))
        return out, time.perf_counter() - t0
    dt = time.perf_counter() - t0
    idx = {s.name: i for i, (s, _) in enumerate(workloads)}
    gpu_of = np.full(m, -1, np.int32)
    pos = np.full(m, -1, np.int32)
    r = np.zeros(m)
    units = np.zeros(m, np.int32)
    batch = np.zeros(m, np.int32)
    pred = np.zeros((m, layout.ROW_NF))
    r_inter = np.zeros(m)
    lb = np.zeros(m, np.int32)
    for g in p.gpus:
        for k, a in enumerate(g.allocations):
            i = idx[a.workload]
            gpu_of[i] = g.gpu_index
            pos[i] = k
            r[i] = a.r
            units[i] = int(round(a.r / hw.r_unit))
            assert units[i] * hw.r_unit == a.r
            batch[i] = a.batch
            bd = g.predicted[a.workload]
            pred[i] = [getattr(bd, f) for f in layout.ROW_FIELDS]
    for name, v in p.per_workload_r_inter.items():
        r_inter[idx[name]] = v
    for i, (s, c) in enumerate(workloads):
        lb[i] = gplanner._lower_bound_units(s, c, hw, batch[i])
    out.update(
        gpu_of=gpu_of, pos=pos, r=r, units=units, batch=batch, pred=pred,
        r_inter=r_inter, lb=lb,
        fragment=np.array([g.fragment_r for g in p.gpus]),
        cost=np.float64(p.cost_per_hour), gpu_count=np.int64(len(p.gpus)),
        model_evals=np.int64(stats.model_evals),
        candidate_gpus=np.int64(stats.candidate_gpus),
        err_class=np.array(""), err_msg=np.array(""), err_code=np.int64(0),
        ref_seconds=np.float64(dt),
    )
    return out, dt


def simple_workload(name, k3, *, slo_ms=40.0, rate_rps=100.0):
    # test_planner.py:37-45
    spec = gp.WorkloadSpec(name, slo_ms, rate_rps, 0.0, 0.0)
    coef = gp.WorkloadCoefficients(
        n_kernels=1, k_sch_ms=0.0, k1=0.0, k2=0.0, k3=k3, k4=0.0, k5=0.0,
        alpha_power_w=0.0, beta_power_w=10.0,
        alpha_cacheutil=0.0, beta_cacheutil=0.0, alpha_cache=0.0,
    )
    return spec, coef


def c3_feasible_workload(rng, name, hw, b_max=128):
    """SURVEY.md §8d C3 generator: support.py:168-187 with slo U(20,100),
    rate U(50,6000) and rejection through appropriate_batch(spec, hw, 128)."""
    for _ in range(200):
        spec = gp.WorkloadSpec(
            name=name,
            slo_ms=float(rng.uniform(20.0, 100.0)),
            rate_rps=float(rng.uniform(50.0, 6000.0)),
            d_load_mb=float(rng.uniform(0.05, 1.0)),
            d_feedback_mb=float(rng.uniform(0.001, 0.05)),
        )
        coef = support.random_coefficients(rng)
        try:
            b = gp.appropriate_batch(spec, hw, b_max)
            gp.lower_bound_resources(spec, coef, hw, b)
        except gerr.PlanningError:
            continue
        return spec, coef
    raise RuntimeError("no feasible workload")


def wide_coef(rng):
    """Wide coefficient draws (test_model_properties.py:25-40 ranges)."""
    return gp.WorkloadCoefficients(
        n_kernels=int(rng.integers(1, 501)),
        k_sch_ms=float(rng.uniform(0.0, 0.01)),
        k1=float(rng.uniform(0.0, 0.02)),
        k2=float(rng.uniform(0.0, 0.2)),
        k3=float(rng.uniform(0.0, 20.0)),
        k4=float(rng.uniform(0.0, 2.0)),
        k5=float(rng.uniform(1e-3, 1.0)),
        alpha_power_w=float(rng.uniform(0.0, 100.0)),
        beta_power_w=float(rng.uniform(0.0, 200.0)),
        alpha_cacheutil=float(rng.uniform(0.0, 0.2)),
        beta_cacheutil=float(rng.uniform(0.0, 0.5)),
        alpha_cache=float(rng.uniform(0.0, 1.0)),
    )


def wide_spec(rng, name):
    return gp.WorkloadSpec(
        name, float(rng.uniform(1.0, 200.0)), float(rng.uniform(1.0, 2000.0)),
        float(rng.uniform(0.0, 2.0)), float(rng.uniform(0.0, 0.5)),
    )


def eval_states_case(rng, count, hw, nmax=12, r_unit=0.025, floor_bias=False):
    """Random device states through the reference _eval_entries
    (model.py:273-317); CSR layout: state s owns rows ptr[s]:ptr[s+1]."""
    wl_rows, rs, batches, ptr, rows = [], [], [], [0], []
    cap = int(round(1.0 / r_unit))
    for _ in range(count):
        n = int(rng.integers(1, nmax + 1))
        entries, r_list = [], []
        for k in range(n):
            spec, coef = wide_spec(rng, f"s{k}"), wide_coef(rng)
            if floor_bias:
                coef = gp.WorkloadCoefficients(**{**coef.__dict__,
                                                  "alpha_power_w": float(rng.uniform(200, 2000)),
                                                  "beta_power_w": float(rng.uniform(100, 400))})
            b = int(rng.integers(1, 33))
            u = int(rng.integers(1, cap + 1))
            r = u * r_unit if rng.random() < 0.8 else float(rng.uniform(0.001, 1.0))
            entries.append(gmodel._Entry(spec, coef, b, hw))
            wl_rows.append(layout.spec_coef_row(spec, coef))
            batches.append(b)
            r_list.append(r)
        out = gmodel._eval_entries(entries, r_list, hw)
        rows.extend(out)
        rs.extend(r_list)
        ptr.append(ptr[-1] + n)
    return dict(
        wl=np.array(wl_rows).T.copy(), batch=np.array(batches, np.int32),
        r=np.array(rs), ptr=np.array(ptr, np.int64), rows=np.array(rows),
        hw=np.array(layout.hw_vector(hw)),
    )


def prologue_case(rng, count, hw, b_max):
    """appropriate_batch (planner.py:76-92) + _lower_bound_units (:95-120)
    over wide random workloads, including every error branch."""
    wl_rows, b_out, lb_out, code = [], [], [], []
    for i in range(count):
        spec = gp.WorkloadSpec(
            f"p{i}", float(rng.uniform(0.5, 200.0)), float(rng.uniform(1.0, 8000.0)),
            float(rng.uniform(0.0, 2.0)), float(rng.uniform(0.0, 0.5)))
        coef = wide_coef(rng)
        if rng.random() < 0.1:
            coef = gp.WorkloadCoefficients(**{**coef.__dict__, "k3": float(rng.uniform(20, 800))})
        wl_rows.append(layout.spec_coef_row(spec, coef))
        try:
            b = gp.appropriate_batch(spec, hw, b_max)
        except gerr.PlanningError as exc:
            b_out.append(-1); lb_out.append(-1); code.append(err_code(exc))
            continue
        try:
            lb = gplanner._lower_bound_units(spec, coef, hw, b)
        except gerr.PlanningError as exc:
            b_out.append(b); lb_out.append(-1); code.append(err_code(exc))
            continue
        b_out.append(b); lb_out.append(lb); code.append(0)
    return dict(wl=np.array(wl_rows).T.copy(), batch=np.array(b_out, np.int32),
                lb=np.array(lb_out, np.int32), code=np.array(code, np.int32),
                hw=np.array(layout.hw_vector(hw)), b_max=np.int64(b_max))


def alloc_case(rng, count, hw):
    """alloc_gpus (planner.py:165-192): random residents + one newcomer."""
    wl_rows, batch, r_in, ptr, units_out = [], [], [], [0], []
    cap = gplanner.max_units(hw)
    for _ in range(count):
        inst = support.random_instance(rng, int(rng.integers(1, 9)), hw)
        specs = {s.name: s for s, _ in inst}
        coefs = {s.name: c for s, c in inst}
        bs = [gp.appropriate_batch(s, hw) for s, _ in inst]
        lbs = [gplanner._lower_bound_units(s, c, hw, b) for (s, c), b in zip(inst, bs)]
        current = []
        used = 0
        for (s, _), b, lb in zip(inst[:-1], bs[:-1], lbs[:-1]):
            u = lb + int(rng.integers(0, 3))
            if used + u > cap - lbs[-1]:
                break
            used += u
            current.append(gp.Allocation(s.name, u * hw.r_unit, b))
        new_s = inst[-1][0]
        res = gp.alloc_gpus(specs, coefs, hw, current, new_s.name, bs[-1],
                            lbs[-1] * hw.r_unit)
        names = [a.workload for a in current] + [new_s.name]
        for nm, a in zip(names, res):
            wl_rows.append(layout.spec_coef_row(specs[nm], coefs[nm]))
            batch.append(a.batch)
            units_out.append(int(round(a.r / hw.r_unit)))
        r_in.extend([a.r for a in current] + [lbs[-1] * hw.r_unit])
        ptr.append(ptr[-1] + len(names))
    return dict(wl=np.array(wl_rows).T.copy(), batch=np.array(batch, np.int32),
                r=np.array(r_in), ptr=np.array(ptr, np.int64),
                units=np.array(units_out, np.int32), hw=np.array(layout.hw_vector(hw)))


def denom_error_workload(name, k4, k3=-1.0, slo=40.0):
    spec = gp.WorkloadSpec(name, slo, 100.0, 0.1, 0.01)
    coef = gp.WorkloadCoefficients(
        n_kernels=10, k_sch_ms=0.001, k1=0.0, k2=0.0, k3=k3, k4=k4, k5=0.2,
        alpha_power_w=10.0, beta_power_w=20.0, alpha_cacheutil=0.02,
        beta_cacheutil=0.05, alpha_cache=0.1)
    return spec, coef


def grid_case(workloads, hw, b_max):
    """Per (w, b): the reference's own one-workload grid search,
    _Search.best_group_alloc([w]) (oracle.py:77-114), with the entry built at
    batch b.  Records the minimal feasible units, 0 if none, -code if an
    evaluation raised (NonPositiveDenominatorError)."""
    from gpuplanner import oracle as goracle
    out = pack_instance(workloads, hw, b_max)
    m = len(workloads)
    specs = {s.name: s for s, _ in workloads}
    budget = goracle.OracleBudget(max_candidates=10**12)
    res = np.zeros((m, b_max), np.int32)
    for i, (s, c) in enumerate(workloads):
        for b in range(1, b_max + 1):
            search = goracle._Search(specs, {s.name: gmodel._Entry(s, c, b, hw)}, hw, budget)
            try:
                r = search.best_group_alloc([s.name])
            except gerr.NonPositiveDenominatorError as exc:
                res[i, b - 1] = -err_code(exc)
                continue
            res[i, b - 1] = 0 if r is None else r[0]
    out.update(min_units=res)
    return out


def stream_reference(workloads, hw, b_max=32):
    """Online arrival-order provisioning over the reference's own internals
    (no reference API exists, plan() always sorts).  Each
    arrival is one step of planner.py:290-319 against the persistent state,
    with the batch and lower bound of planner.py:280-282; an arrival whose
    prologue or candidate evaluation raises is rejected and leaves the state
    unchanged.  Returns per-arrival GPU, position and error code, plus the
    final units of every admitted arrival."""
    cap = gplanner.max_units(hw)
    names, entries, units = [], [], []
    n = len(workloads)
    gpu_of = np.full(n, -1, np.int32)
    pos = np.full(n, -1, np.int32)
    code = np.zeros(n, np.int32)
    where = {}
    for a, (spec, coef) in enumerate(workloads):
        try:
            b = gp.appropriate_batch(spec, hw, b_max)
            need = gplanner._lower_bound_units(spec, coef, hw, b)
        except gerr.PlanningError as exc:
            code[a] = err_code(exc)
            continue
        entry = gmodel._Entry(spec, coef, b, hw)
        best_j, best_inter, best_units = -1, cap, None
        try:
            for j in range(len(names)):
                occupied = sum(units[j])
                if occupied + need > cap:
                    continue
                cand = gplanner._alloc_units(entries[j] + [entry], units[j] + [need], hw, cap)
                total = sum(cand)
                if total <= cap and total - occupied < best_inter:
                    best_j, best_inter, best_units = j, total - occupied, cand
        except gerr.NonPositiveDenominatorError as exc:
            code[a] = err_code(exc)
            continue
        if best_j < 0:
            names.append([a]); entries.append([entry]); units.append([need])
            best_j = len(names) - 1
        else:
            names[best_j].append(a); entries[best_j].append(entry); units[best_j] = list(best_units)
        gpu_of[a] = best_j
        pos[a] = len(names[best_j]) - 1
    final_units = np.zeros(n, np.int32)
    for j, mem in enumerate(names):
        for k, a in enumerate(mem):
            final_units[a] = units[j][k]
    return gpu_of, pos, code, final_units


def oracle_case(workloads, hw, budget=None, b_max=32):
    """The reference's exhaustive_plan (oracle.py:130-201) on a tiny instance."""
    from gpuplanner import oracle as goracle
    out = pack_instance(workloads, hw, b_max)
    grid = budget.r_grid_units if budget and budget.r_grid_units else ()
    out.update(max_gpus=np.int64(budget.max_gpus if budget else 3), grid=np.array(grid, np.int64))
    m = len(workloads)
    try:
        p = goracle.exhaustive_plan(workloads, hw, budget=budget, b_max=b_max)
    except gerr.GpuPlannerError as exc:
        out.update(err_class=np.array(type(exc).__name__), err_msg=np.array(str(exc)))
        return out
    idx = {s.name: i for i, (s, _) in enumerate(workloads)}
    gpu_of = np.full(m, -1, np.int32)
    units = np.zeros(m, np.int32)
    pred = np.zeros((m, layout.ROW_NF))
    for g in p.gpus:
        for a in g.allocations:
            i = idx[a.workload]
            gpu_of[i] = g.gpu_index
            units[i] = int(round(a.r / hw.r_unit))
            pred[i] = [getattr(g.predicted[a.workload], f) for f in layout.ROW_FIELDS]
    out.update(err_class=np.array(""), err_msg=np.array(""), gpu_of=gpu_of, units=units, pred=pred,
               gpu_count=np.int64(len(p.gpus)), cost=np.float64(p.cost_per_hour))
    return out


def simulate_case(workloads, hw, cfg, plan=None):
    """The reference's simulate() (simulate.py:139-198) on a plan; the replay
    inputs (rate, batch, predicted t_inf) are stored in report order."""
    import importlib
    gsim = importlib.import_module("gpuplanner.simulate")
    out = pack_instance(workloads, hw, 32)
    specs = {s.name: s for s, _ in workloads}
    coefs = {s.name: c for s, c in workloads}
    p = plan or gp.plan(workloads, hw)
    items = []
    for g in p.gpus:
        pred = gp.predict_gpu(g.allocations, specs, coefs, hw)
        for a in g.allocations:
            items.append((a.workload, a.batch, pred[a.workload].t_inf_ms))
    items.sort()
    out.update(duration=np.float64(cfg.duration_ms), warmup=np.float64(cfg.warmup_ms),
               arrival=np.array(cfg.arrival), sim_names=np.array([n for n, _, _ in items]),
               rate=np.array([specs[n].rate_rps for n, _, _ in items]),
               sim_batch=np.array([b for _, b, _ in items], np.int32),
               service=np.array([t for _, _, t in items]))
    try:
        rep = gsim.simulate(p, specs, coefs, hw, cfg)
    except Exception as exc:  # noqa: BLE001 - the fixture records the reference's failure
        out.update(err_class=np.array(type(exc).__name__), err_msg=np.array(str(exc)))
        return out
    out.update(err_class=np.array(""), err_msg=np.array(""),
               achieved=np.array([w.achieved_rps for w in rep.workloads]),
               p50=np.array([w.p50_ms for w in rep.workloads]),
               p99=np.array([w.p99_ms for w in rep.workloads]),
               max_depth=np.array([w.max_queue_depth for w in rep.workloads], np.int32),
               completed=np.array([w.completed for w in rep.workloads], np.int32),
               violation=np.array([w.violation for w in rep.workloads]))
    return out


def trace_case(workloads, hw, cfg):
    """simulate(..., collect_trace=True): the per-request records
    (simulate.py:192-197), as workload index + fp64 arrays."""
    import importlib
    gsim = importlib.import_module("gpuplanner.simulate")
    out = simulate_case(workloads, hw, cfg)
    specs = {s.name: s for s, _ in workloads}
    coefs = {s.name: c for s, c in workloads}
    _, trace = gsim.simulate(gp.plan(workloads, hw), specs, coefs, hw, cfg, collect_trace=True)
    index = {str(n): i for i, n in enumerate(out["sim_names"])}
    out.update(trace_w=np.array([index[r.workload] for r in trace], np.int32),
               trace_arrival=np.array([r.arrival_ms for r in trace]),
               trace_dispatch=np.array([r.dispatch_ms for r in trace]),
               trace_complete=np.array([r.complete_ms for r in trace]))
    return out


def modelfn_case(seed, n, hw):
    """The model's component functions (model.py:159-236) on n random queries,
    including r + k4 <= 0 and k_act <= 0 rows; '' / message per function."""
    from gpuplanner import model as gm
    rng = np.random.default_rng(seed)
    wls, batch, r, co, ncol, pdem = [], [], [], [], [], []
    for i in range(n):
        c = support.random_coefficients(rng)
        kind = i % 10
        if kind == 8:  # r + k4 <= 0
            c = dataclasses.replace(c, k4=-float(rng.uniform(0.3, 1.2)))
        elif kind == 9:  # k_act <= 0
            c = dataclasses.replace(c, k5=-float(rng.uniform(50.0, 500.0)))
        sp = gp.WorkloadSpec(f"q{i}", float(rng.uniform(20, 100)), float(rng.uniform(50, 6000)),
                             float(rng.uniform(0.05, 1.0)), float(rng.uniform(0.001, 0.05)))
        wls.append((sp, c))
        batch.append(int(rng.integers(1, 129)))
        r.append(float(rng.integers(1, 41)) * hw.r_unit)
        co.append(float(rng.uniform(0.0, 3.0)))
        ncol.append(int(rng.integers(0, 12)))
        pdem.append(float(rng.uniform(0.5, 2.5)) * hw.power_max_w)
    out = pack_instance(wls, hw, 128)

    def run(fn):
        vals, msgs = [], []
        for i, (sp, c) in enumerate(wls):
            try:
                vals.append(float(fn(i, sp, c)))
                msgs.append("")
            except Exception as exc:  # noqa: BLE001 - recorded for the parity test
                vals.append(float("nan"))
                msgs.append(f"{type(exc).__name__}: {exc}")
        return np.array(vals), np.array(msgs)

    cols = {
        "t_load": lambda i, sp, c: gm.transfer_latencies(sp, batch[i], hw)[0],
        "t_fb": lambda i, sp, c: gm.transfer_latencies(sp, batch[i], hw)[1],
        "k_act": lambda i, sp, c: gm.solo_active_time(c, batch[i], r[i]),
        "power": lambda i, sp, c: gm.solo_power(c, batch[i], r[i]),
        "cache": lambda i, sp, c: gm.solo_cache_util(c, batch[i], r[i]),
        "sch_inc": lambda i, sp, c: gm.sched_delay_increase(hw, ncol[i]),
        "sched": lambda i, sp, c: gm.sched_delay(c, hw, ncol[i]),
        "act_int": lambda i, sp, c: gm.active_time_with_interference(c, batch[i], r[i], co[i]),
        "freq": lambda i, sp, c: gm.gpu_frequency(hw, pdem[i]),
    }
    for k, fn in cols.items():
        v, m = run(fn)
        out[f"fn_{k}"] = v
        out[f"msg_{k}"] = m
    lists = [[float(x) for x in rng.uniform(10.0, 150.0, int(rng.integers(0, 14)))] for _ in range(64)]
    lists[1] = [1e16, 1.0, -1e16, 3.5]  # compensation matters
    out.update(q_batch=np.array(batch, np.int32), q_r=np.array(r), q_co=np.array(co),
               q_ncol=np.array(ncol, np.int32), q_pdem=np.array(pdem),
               pd_ptr=np.cumsum([0] + [len(x) for x in lists]).astype(np.int64),
               pd_vals=np.array([x for xs in lists for x in xs]),
               pd_out=np.array([gm.power_demand(hw, xs) for xs in lists]))
    return out


def stream_case(workloads, hw, b_max=32):
    out = pack_instance(workloads, hw, b_max)
    gpu_of, pos, code, units = stream_reference(workloads, hw, b_max)
    out.update(gpu_of=gpu_of, pos=pos, code=code, units=units,
               gpu_count=np.int64(gpu_of.max() + 1 if (gpu_of >= 0).any() else 0))
    return out


def main():
    groups = set(sys.argv[1:]) or {"plan", "component", "grid", "stream", "oracle", "document",
                                   "simulate"}
    mpath = os.path.join(HERE, "manifest.json")
    manifest = json.load(open(mpath))["cases"] if os.path.exists(mpath) else {}
    v100 = support.make_v100()

    def save(name, d, note):
        np.savez_compressed(os.path.join(HERE, name + ".npz"), **d)
        manifest[name] = note
        print(f"{name}: {note}", flush=True)

    # ---- plan() cases -------------------------------------------------
    plan_cases = []
    plan_cases.append(("plan_c1_twelve", support.twelve_workload_instance(), v100, 32,
                       "C1: twelve_workload_instance on make_v100 (support.py:106-151)"))
    plan_cases.append(("plan_c1_twelve_reversed",
                       list(reversed(support.twelve_workload_instance())), v100, 32,
                       "C1 reversed input order (test_planner.py:208-213)"))
    rng = np.random.default_rng(7)
    for m in (20, 40, 80):  # test_planner.py:225-234 draws these sequentially
        plan_cases.append((f"plan_rand{m}_seq7", support.random_instance(rng, m, v100), v100, 32,
                           f"random_instance m={m}, shared default_rng(7) stream"))
    plan_cases.append(("plan_single", [(support.demo_spec(), support.demo_coef())], v100, 32,
                       "test_planner.py:161-167"))
    coef2 = support.demo_coef(alpha_cache=0.0, alpha_power_w=5.0, beta_power_w=20.0)
    plan_cases.append(("plan_two_copies", [(support.demo_spec("a"), coef2),
                                           (support.demo_spec("b"), coef2)], v100, 32,
                       "test_planner.py:169-181"))
    plan_cases.append(("plan_simple12_v100", [simple_workload(f"w{i:02d}", 9.9) for i in range(12)],
                       v100, 32, "test_planner.py:238-243 (6 GPUs, $18.36)"))
    t4 = gp.HardwareProfile("t4", 70.0, 1590.0, 10.0, 10.0, -1.0, 0.00475, -0.00902,
                            price_per_hour=0.526)
    plan_cases.append(("plan_simple15_t4", [simple_workload(f"w{i:02d}", 19.8) for i in range(15)],
                       t4, 32, "test_planner.py:245-250 (15 GPUs, $7.89)"))
    plan_cases.append(("plan_rand1k_seed7", support.random_instance(np.random.default_rng(7), 1000, v100),
                       v100, 32, "C2: random_instance(default_rng(7), 1000), r_unit 0.025"))
    plan_cases.append(("plan_rand1k_seed1", support.random_instance(np.random.default_rng(1), 1000, v100),
                       v100, 32, "C2: random_instance(default_rng(1), 1000), r_unit 0.025"))
    hw01 = support.make_v100(r_unit=0.01)
    plan_cases.append(("plan_rand600_r01", support.random_instance(np.random.default_rng(3), 600, hw01),
                       hw01, 32, "random_instance(default_rng(3), 600), r_unit 0.01 (cap 100)"))
    rng3 = np.random.default_rng(2211)
    c3 = [c3_feasible_workload(rng3, f"w{i:06d}", hw01) for i in range(800)]
    plan_cases.append(("plan_c3style_800", c3, hw01, 128,
                       "C3 generator (slo U(20,100), rate U(50,6000), b<=128, r_unit 0.01), 800 workloads"))
    # names whose string order differs from numeric order (SURVEY finding 9)
    rngn = np.random.default_rng(11)
    inst = support.random_instance(rngn, 400, v100)
    perm = rngn.permutation(400)
    inst = [(gp.WorkloadSpec(f"w{int(perm[i]) * 37 % 1009}", s.slo_ms, s.rate_rps, s.d_load_mb,
                             s.d_feedback_mb), c) for i, (s, c) in enumerate(inst)]
    plan_cases.append(("plan_names_mixed400", inst, v100, 32,
                       "400 workloads, names w<k> of mixed length (string vs numeric order)"))
    # identical workloads: every sort key ties on lb, every argmin ties on inter
    ident = [(gp.WorkloadSpec(f"t{i}", 40.0, 300.0, 0.5, 0.01), support.demo_coef()) for i in range(60)]
    plan_cases.append(("plan_identical60", ident, v100, 32,
                       "60 identical workloads: sort/argmin ties resolved by name / lowest index"))
    # hardware variants: floor binding (tiny power cap), no scheduling term
    hw_floor = support.make_v100(power_max_w=80.0, power_idle_w=53.5, alpha_f=-8.0)
    plan_cases.append(("plan_floor300", support.random_instance(np.random.default_rng(5), 300, hw_floor),
                       hw_floor, 32, "tight power cap: f_min floor binds in most evaluations"))
    # error cases
    inst = support.random_instance(np.random.default_rng(9), 30, v100)
    bad = gp.WorkloadSpec("impossible", 0.9, 100.0, 0.574, 0.004)
    plan_cases.append(("plan_err_slo", inst[:10] + [(bad, support.demo_coef())] + inst[10:], v100, 32,
                       "InfeasibleSloError (test_planner.py:215-218) after 10 good workloads"))
    dense = gp.WorkloadSpec("dense", 1.2, 100.0, 0.574, 0.004)
    plan_cases.append(("plan_err_res", inst[:5] + [(dense, support.demo_coef())] + inst[5:], v100, 32,
                       "InfeasibleResourceError (test_planner.py:220-223)"))
    capx = gp.WorkloadSpec("capx", 200.0, 2000.0, 0.0, 0.0)
    plan_cases.append(("plan_err_batch", inst[:3] + [(capx, support.demo_coef())] + inst[3:], v100, 32,
                       "BatchCapExceededError (test_planner.py:59-62) mid-input"))
    # r + k4 <= 0 on a workload that enters the plan: lb*r_unit + k4 < 0
    plan_cases.append(("plan_err_denom", inst[:12] + [denom_error_workload("neg", -0.5)] + inst[12:],
                       v100, 32, "NonPositiveDenominatorError raised mid-plan by _eval_entries"))
    # k_act <= 0 branch: negative gamma keeps lb small while k_act stays negative
    spec_k, coef_k = denom_error_workload("negk", 0.05, k3=-3.0)
    plan_cases.append(("plan_err_kact", inst[:7] + [(spec_k, coef_k)] + inst[7:], v100, 32,
                       "NonPositiveDenominatorError (active-time variant) mid-plan"))
    plan_cases.append(("plan_err_denom_alone", [denom_error_workload("solo_neg", -0.5)], v100, 32,
                       "denominator error surfaced only by _build_plan/predict_gpu"))

    for name, wls, hw, bmax, note in plan_cases if "plan" in groups else []:
        d, dt = run_plan_case(wls, hw, bmax)
        extra = f" [{str(d['err_class'])}]" if str(d["err_class"]) else (
            f" -> {int(d['gpu_count'])} GPUs, evals={int(d['model_evals'])}, "
            f"cands={int(d['candidate_gpus'])}, {dt:.2f}s")
        save(name, d, note + extra)

    # ---- solo candidate grid (BASELINE config 3) --------------------------
    if "grid" in groups:
        rng = np.random.default_rng(2212)
        c3 = [c3_feasible_workload(rng, f"g{i:03d}", hw01) for i in range(40)]
        save("grid_c3_40", grid_case(c3, hw01, 128),
             "solo grid: 40 C3-generator workloads x b 1..128 x u 1..100 (oracle.py:77-114)")
        inst = support.random_instance(np.random.default_rng(2213), 60, v100)
        save("grid_v100_60", grid_case(inst, v100, 32),
             "solo grid: 60 random_instance workloads x b 1..32 x u 1..40")
        odd = [denom_error_workload("gneg", -0.5), denom_error_workload("gnegk", 0.05, k3=-3.0),
               (support.demo_spec("gfloor"), support.demo_coef(alpha_power_w=400.0, beta_power_w=300.0)),
               (gp.WorkloadSpec("gtight", 1.0, 5000.0, 0.9, 0.05), support.demo_coef()),
               (gp.WorkloadSpec("gloose", 200.0, 10.0, 0.0, 0.0), support.demo_coef())]
        rngw = np.random.default_rng(2214)
        odd += [(wide_spec(rngw, f"gw{i}"), wide_coef(rngw)) for i in range(25)]
        save("grid_edge_30", grid_case(odd, v100, 48),
             "solo grid edge cases: denominator / active-time errors, f_min floor, "
             "infeasible everywhere, wide coefficients")

    # ---- online stream (BASELINE config 5): arrival order, no sort ---------
    if "stream" in groups:
        save("stream_c2_600", stream_case(support.random_instance(np.random.default_rng(505), 600, v100),
                                          v100), "stream: 600 random_instance arrivals in arrival order")
        save("stream_r01_300", stream_case(support.random_instance(np.random.default_rng(506), 300, hw01),
                                           hw01), "stream: 300 arrivals, r_unit 0.01 (cap 100)")
        inst = support.random_instance(np.random.default_rng(507), 120, v100)
        mix = (inst[:20] + [(gp.WorkloadSpec("s_slo", 0.9, 100.0, 0.574, 0.004), support.demo_coef())]
               + inst[20:40] + [(gp.WorkloadSpec("s_cap", 200.0, 2000.0, 0.0, 0.0), support.demo_coef())]
               + inst[40:60] + [denom_error_workload("s_neg", -0.5)] + inst[60:80]
               + [denom_error_workload("s_negk", 0.05, k3=-3.0)] + inst[80:])
        save("stream_errors_124", stream_case(mix, v100),
             "stream with rejected arrivals: infeasible SLO, batch cap, r + k4 <= 0, k_act <= 0")

    # ---- exhaustive oracle (oracle.py:130-201), SURVEY §8f row 2 -----------
    if "oracle" in groups:
        from gpuplanner import oracle as goracle
        rng = np.random.default_rng(808)
        for i in range(24):
            m = 1 + i % 4
            save(f"oracle_rand{i:02d}", oracle_case(support.random_instance(rng, m, v100), v100),
                 f"exhaustive_plan on random_instance m={m}")
        hw20 = support.make_v100(r_unit=0.05)
        for i in range(4):
            save(f"oracle_r05_{i}", oracle_case(support.random_instance(rng, 4, hw20), hw20),
                 "exhaustive_plan, r_unit 0.05 (cap 20), 4 workloads")
        coarse = goracle.OracleBudget(r_grid_units=(1, 2, 3, 5, 8, 13, 21, 34))
        for i in range(3):
            save(f"oracle_grid_{i}", oracle_case(support.random_instance(rng, 3, v100), v100, coarse),
                 "exhaustive_plan with a custom unit grid")
        heavy = [(gp.WorkloadSpec(f"h{i}", 30.0, 450.0, 0.9, 0.05), support.demo_coef(k3=6.0))
                 for i in range(4)]
        save("oracle_err_infeasible", oracle_case(heavy, v100, goracle.OracleBudget(max_gpus=1)),
             "InfeasibleError: four heavy workloads on one device")
        save("oracle_err_budget", oracle_case(support.random_instance(rng, 5, v100), v100),
             "BudgetExceededError: five workloads")
        save("oracle_twelve_sub4", oracle_case(support.twelve_workload_instance()[:4], v100),
             "exhaustive_plan on the first four C1 workloads")

    # ---- plan documents (problem.py:305-341), SURVEY §8f row 1 -------------
    if "document" in groups:
        from gpuplanner import problem as gproblem
        for name, wls, hw in (("doc_c1_twelve", support.twelve_workload_instance(), v100),
                              ("doc_rand80", support.random_instance(np.random.default_rng(80), 80, v100), v100),
                              ("doc_r01_40", support.random_instance(np.random.default_rng(81), 40, hw01), hw01)):
            p = gp.plan(wls, hw)
            doc = gproblem.plan_to_document(p, {s.name: s for s, _ in wls})
            d = pack_instance(wls, hw, 32)
            d.update(document=np.array(json.dumps(doc)))
            save(name, d, "reference plan_to_document(plan(...)) as JSON text")

    # ---- request-level replay (simulate.py:139-198), SURVEY §8f row 4 -------
    if "simulate" in groups:
        import importlib
        gsim = importlib.import_module("gpuplanner.simulate")
        twelve = support.twelve_workload_instance()
        save("sim_c1_30s", simulate_case(twelve, v100, gsim.SimConfig(30_000.0, 1_000.0)),
             "simulate(plan(C1), 30 s, warmup 1 s) -- SPEC acceptance 7 window")
        inst = support.random_instance(np.random.default_rng(90), 60, v100)
        save("sim_rand60_10s", simulate_case(inst, v100, gsim.SimConfig(10_000.0, 500.0)),
             "simulate(plan(random_instance 60)), 10 s")
        save("sim_rand60_nowarm", simulate_case(inst, v100, gsim.SimConfig(2_000.0)),
             "simulate, 2 s, no warm-up")
        save("sim_allwarm", simulate_case(twelve[:5], v100, gsim.SimConfig(500.0, 500.0)),
             "simulate with warmup == duration (no measured requests)")
        slow = [(gp.WorkloadSpec(f"u{i}", 40.0, 400.0, 0.5, 0.01), support.demo_coef()) for i in range(2)]
        over = gp.Plan("manual", "v100", [gp.GpuPlan(0, [gp.Allocation("u0", 0.025, 1),
                                                         gp.Allocation("u1", 0.025, 1)], {}, 0.95)],
                       3.06, {})
        save("sim_unstable", simulate_case(slow, v100, gsim.SimConfig(5_000.0), plan=over),
             "UnstableQueueError: batch 1 at 2.5% of a device cannot keep up")
        save("sim_poisson", simulate_case(twelve[:3], v100, gsim.SimConfig(1_000.0, arrival="poisson")),
             "poisson arrivals: the reference's tuple seed raises TypeError on CPython 3.12")

    if "modelfn" in groups:
        save("modelfn_v100", modelfn_case(11, 1000, v100), "model.py:159-236 component functions")
        save("modelfn_r01", modelfn_case(12, 500, support.make_v100(r_unit=0.01)),
             "component functions, r_unit 0.01")

    if "simtrace" in groups:
        import importlib
        gsim = importlib.import_module("gpuplanner.simulate")
        twelve = support.twelve_workload_instance()
        save("simtrace_c1_allwarm", trace_case(twelve[:5], v100, gsim.SimConfig(500.0, 500.0)),
             "simulate(..., collect_trace=True), warmup == duration")
        inst = support.random_instance(np.random.default_rng(90), 60, v100)
        save("simtrace_rand60", trace_case(inst, v100, gsim.SimConfig(200.0, 50.0)),
             "simulate(..., collect_trace=True), 60 workloads, 200 ms")

    # ---- component cases ------------------------------------------------
    if "component" not in groups:
        with open(mpath, "w") as fh:
            json.dump({"python": sys.version.split()[0], "numpy": np.__version__,
                       "cases": manifest}, fh, indent=1, sort_keys=True)
        return
    save("eval_states_v100", eval_states_case(np.random.default_rng(101), 1000, v100),
         "1000 random device states, n=1..12, wide coefficients (_eval_entries rows)")
    save("eval_states_floor", eval_states_case(np.random.default_rng(102), 600, v100, floor_bias=True),
         "600 states biased onto the f_min floor")
    save("eval_states_r01", eval_states_case(np.random.default_rng(103), 500, hw01, nmax=30, r_unit=0.01),
         "500 states, r_unit 0.01, up to 30 residents")
    save("prologue_v100", prologue_case(np.random.default_rng(104), 6000, v100, 32),
         "6000 workloads: appropriate_batch + _lower_bound_units incl. error codes")
    save("prologue_r01_b128", prologue_case(np.random.default_rng(105), 6000, hw01, 128),
         "6000 workloads, r_unit 0.01, b_max 128")
    save("alloc_v100", alloc_case(np.random.default_rng(106), 400, v100),
         "400 alloc_gpus calls (Alg. 2) on random residents")

    with open(mpath, "w") as fh:
        json.dump({"python": sys.version.split()[0], "numpy": np.__version__,
                   "cases": manifest}, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
