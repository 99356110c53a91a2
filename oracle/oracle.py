"""ctypes front-end for the CPU oracle (oracle/igniter_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's CPU-baseline legs, never by the product package.  The functions
here mirror the reference call sites they check (see igniter_oracle.c).
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")


class IgoErr(ctypes.Structure):
    _fields_ = [("code", ctypes.c_int32), ("workload", ctypes.c_int32),
                ("a", ctypes.c_double), ("b", ctypes.c_double), ("c", ctypes.c_double)]


def build(force: bool = False) -> str:
    src = os.path.join(HERE, "igniter_oracle.c")
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < os.path.getmtime(src):
        subprocess.check_call(["make", "-s", "-C", HERE, "-B", "liboracle.so"])
    return LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        _lib = ctypes.CDLL(LIB_PATH)
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def name_ranks(names) -> np.ndarray:
    """Rank of each name under Python string order (planner.py:284 tie-break)."""
    order = sorted(range(len(names)), key=lambda i: names[i])
    rank = np.empty(len(names), np.int32)
    rank[np.array(order, dtype=np.int64)] = np.arange(len(names), dtype=np.int32)
    return rank


def plan(wl: np.ndarray, hw, b_max: int, rank: np.ndarray):
    """Alg. 1 with exact PlanStats; returns a dict of per-workload arrays."""
    wl = np.ascontiguousarray(wl, np.float64)
    m = wl.shape[1]
    hw = np.ascontiguousarray(hw, np.float64)
    rank = np.ascontiguousarray(rank, np.int32)
    out = {k: np.full(m, -1, np.int32) for k in ("gpu_of", "pos", "units", "batch", "lb")}
    pred = np.zeros((m, 10))
    gc = np.zeros(1, np.int32)
    stats = np.zeros(3, np.int64)
    err = IgoErr()
    rc = lib().igo_plan(_p(wl), ctypes.c_int64(m), ctypes.c_int(m), _p(hw), ctypes.c_int(b_max),
                        _p(rank), _p(out["gpu_of"]), _p(out["pos"]), _p(out["units"]),
                        _p(out["batch"]), _p(out["lb"]), _p(pred), _p(gc), _p(stats),
                        ctypes.byref(err))
    out.update(pred=pred, gpu_count=int(gc[0]), model_evals=int(stats[0]),
               candidate_gpus=int(stats[1]), resident_reads=int(stats[2]), rc=int(rc),
               err=(err.code, err.workload, err.a, err.b, err.c))
    return out


def plan_batch(wl: np.ndarray, hw, b_max: int, rank: np.ndarray, threads: int, stats=False,
               pred=False):
    """S independent scenarios wl[S, 16, m] on `threads` host threads; with
    pred=True also the _build_plan rows (planner.py:218-246) and positions."""
    wl = np.ascontiguousarray(wl, np.float64)
    S, _, m = wl.shape
    hw = np.ascontiguousarray(hw, np.float64)
    rank = np.ascontiguousarray(rank, np.int32)
    gpu_of = np.zeros((S, m), np.int32)
    units = np.zeros((S, m), np.int32)
    pos = np.zeros((S, m), np.int32) if pred else None
    rows = np.zeros((S, m, 10)) if pred else None
    gc = np.zeros(S, np.int32)
    st = np.zeros((S, 3), np.int64) if stats else None
    rc = lib().igo_plan_batch(_p(wl), ctypes.c_int(S), ctypes.c_int(m), _p(hw), ctypes.c_int(b_max),
                              _p(rank), _p(gpu_of), _p(pos) if pred else None, _p(units),
                              _p(rows) if pred else None, _p(gc), _p(st) if stats else None,
                              ctypes.c_int(threads))
    return dict(gpu_of=gpu_of, pos=pos, units=units, pred=rows, gpu_count=gc, stats=st, rc=int(rc))


def prologue(wl: np.ndarray, hw, b_max: int):
    wl = np.ascontiguousarray(wl, np.float64)
    m = wl.shape[1]
    hw = np.ascontiguousarray(hw, np.float64)
    b = np.zeros(m, np.int32)
    lb = np.zeros(m, np.int32)
    code = np.zeros(m, np.int32)
    lib().igo_prologue(_p(wl), ctypes.c_int64(m), ctypes.c_int(m), _p(hw), ctypes.c_int(b_max),
                       _p(b), _p(lb), _p(code))
    return b, lb, code


def eval_states(wl, batch, r, ptr, hw):
    wl = np.ascontiguousarray(wl, np.float64)
    n = wl.shape[1]
    batch = np.ascontiguousarray(batch, np.int32)
    r = np.ascontiguousarray(r, np.float64)
    ptr = np.ascontiguousarray(ptr, np.int64)
    hw = np.ascontiguousarray(hw, np.float64)
    rows = np.zeros((n, 10))
    err = IgoErr()
    rc = lib().igo_eval_states(_p(wl), ctypes.c_int64(n), _p(batch), _p(r), _p(ptr),
                               ctypes.c_int(len(ptr) - 1), _p(hw), _p(rows), ctypes.byref(err))
    return rows, int(rc)


def alloc_units(wl, batch, r, ptr, hw):
    wl = np.ascontiguousarray(wl, np.float64)
    n = wl.shape[1]
    batch = np.ascontiguousarray(batch, np.int32)
    r = np.ascontiguousarray(r, np.float64)
    ptr = np.ascontiguousarray(ptr, np.int64)
    hw = np.ascontiguousarray(hw, np.float64)
    units = np.zeros(n, np.int32)
    err = IgoErr()
    rc = lib().igo_alloc_units(_p(wl), ctypes.c_int64(n), _p(batch), _p(r), _p(ptr),
                               ctypes.c_int(len(ptr) - 1), _p(hw), _p(units), ctypes.byref(err))
    return units, int(rc)


def solo_grid(wl, hw, b_max: int):
    """min feasible units per (workload, batch) -- oracle.py:64-114 semantics."""
    wl = np.ascontiguousarray(wl, np.float64)
    m = wl.shape[1]
    hw = np.ascontiguousarray(hw, np.float64)
    out = np.zeros((m, b_max), np.int32)
    ev = np.zeros(1, np.int64)
    lib().igo_solo_grid(_p(wl), ctypes.c_int64(m), ctypes.c_int(m), _p(hw), ctypes.c_int(b_max),
                        _p(out), _p(ev))
    return out, int(ev[0])


def stream(wl, hw, b_max: int):
    """Arrival-order provisioning (one planner.py:290-319 step per arrival,
    rejected arrivals leave the state unchanged)."""
    wl = np.ascontiguousarray(wl, np.float64)
    n = wl.shape[1]
    hw = np.ascontiguousarray(hw, np.float64)
    gpu_of = np.zeros(n, np.int32)
    pos = np.zeros(n, np.int32)
    code = np.zeros(n, np.int32)
    units = np.zeros(n, np.int32)
    gc = np.zeros(1, np.int32)
    st = np.zeros(2, np.int64)
    lib().igo_stream(_p(wl), ctypes.c_int64(n), ctypes.c_int(n), _p(hw), ctypes.c_int(b_max),
                     _p(gpu_of), _p(pos), _p(code), _p(units), _p(gc), _p(st))
    return dict(gpu_of=gpu_of, pos=pos, code=code, units=units, gpu_count=int(gc[0]),
                model_evals=int(st[0]), candidate_gpus=int(st[1]))


def group_search(wl, batch, hw, grid):
    """Per-subset minimal (total, units) keys of the exhaustive oracle
    (oracle.py:77-114), packed like igp_group_search_device."""
    wl = np.ascontiguousarray(wl, np.float64)
    n = wl.shape[1]
    hw = np.ascontiguousarray(hw, np.float64)
    batch = np.ascontiguousarray(batch, np.int32)
    grid = np.ascontiguousarray(grid, np.int32)
    best = np.zeros(1 << n, np.uint64)
    rc = lib().igo_group_search(_p(wl), ctypes.c_int64(n), ctypes.c_int(n), _p(batch), _p(hw),
                                _p(grid), ctypes.c_int(len(grid)), _p(best))
    return best, int(rc)
