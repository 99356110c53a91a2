"""Exhaustive reference planner for tiny instances (drop-in for ``gpuplanner.oracle``).

The reference (``oracle.py:130-201``) enumerates every partition of at most
``max_workloads`` workloads onto at most ``max_gpus`` devices and, for every
block, the minimal feasible allocation on the unit grid
(``_Search.best_group_alloc``, ``oracle.py:77-114``).  Here the grid search of
every subset of the workloads runs in one device launch
(``igp_group_search_device``).  The partition walk (at most 15 partitions of
4 workloads) and the lexicographic choice (``oracle.py:181-185``) are host
bookkeeping over those per-subset results.  The plan is then built by
``_build_plan`` (``planner.py:218-246``), with device predictions.

Differences from the reference (also in include/igniter_b200.h and
INTEGRATION.md):
* ``OracleBudget.max_candidates`` counts the reference's own pruned
  evaluations. It is not reproduced, because the device evaluates the whole
  grid.
* A ``NonPositiveDenominatorError`` is raised if any grid vector raises.
* The device search takes at most 6 workloads (``IGP_GS_MAXN``, 2^6 subsets
  of up to cap^6 grid vectors): ``exhaustive_plan`` raises
  ``BudgetExceededError`` above that even when ``max_workloads`` allows
  more.  The reference's default budget is 4 workloads.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Iterator, Sequence

import numpy as np

from . import _device, _native
from .errors import BudgetExceededError, InfeasibleError, NonPositiveDenominatorError
from .layout import E_ACTIVE_TIME, E_DENOM, WL_NF, hw_vector, spec_coef_row
from .planner import (DEFAULT_BATCH_CAP, _build_plan, _check_unique_names, _lower_bound_units,
                      appropriate_batch, max_units)

MAX_GROUP = 6  # IGP_GS_MAXN


@dataclass(frozen=True)
class OracleBudget:
    """Enumeration limits; the grid defaults to every allocation unit (oracle.py:37-44)."""

    max_workloads: int = 4
    max_gpus: int = 3
    max_candidates: int = 100_000_000
    r_grid_units: tuple[int, ...] | None = None


def _mask_partitions(full: int, max_blocks: int) -> Iterator[list[int]]:
    """Every set partition of the bits of ``full`` into at most ``max_blocks``
    blocks, as lists of bitmasks.  Each block is the lowest bit not yet placed
    plus a subset of the bits above it, so every partition appears once.  The
    order differs from the reference's generator (oracle.py:117-127), which
    does not matter: the choice below is a strict lexicographic minimum over
    keys that are distinct for distinct partitions."""
    if full == 0:
        yield []
        return
    if max_blocks == 0:
        return
    low = full & -full
    rest = full ^ low
    sub = rest
    while True:
        for tail in _mask_partitions(rest & ~sub, max_blocks - 1):
            yield [low | sub] + tail
        if sub == 0:
            break
        sub = (sub - 1) & rest


def decode_keys(best, n):
    """Packed per-subset keys -> {mask: (total, (u, ...)) or None}; the units
    follow the subset's members in name order."""
    out = {}
    for mask in range(1, 1 << n):
        key = int(best[mask])
        if key == (1 << 64) - 1:
            out[mask] = None
            continue
        k = bin(mask).count("1")
        out[mask] = (key >> (9 * k), tuple((key >> (9 * (k - 1 - d))) & 0x1FF for d in range(k)))
    return out


def select_partition(names, results, max_gpus):
    """The partition minimising (device count, total units, signature) over
    the per-subset optima (the choice of oracle.py:170-190), as its sorted
    blocks of (name, units) pairs, or None when no partition is feasible."""
    n = len(names)
    best = None
    for blocks in _mask_partitions((1 << n) - 1, max_gpus):
        found = [results[b] for b in blocks]
        if any(r is None for r in found):
            continue
        signature = tuple(sorted(
            tuple(zip((names[i] for i in range(n) if (b >> i) & 1), r[1]))
            for b, r in zip(blocks, found)))
        key = (len(blocks), sum(r[0] for r in found), signature)
        if best is None or key < best:
            best = key
    return None if best is None else list(best[2])


def group_search(specs, coefs, batches, names, hw, grid):
    """Minimal feasible (total, units) of every subset of ``names`` (name
    order), or None: {subset bitmask over names: (total, (u, ...))}."""
    torch = _device._torch()
    lib = _native.lib_for_compute()
    n = len(names)
    if n > MAX_GROUP:
        raise BudgetExceededError(f"device group search handles at most {MAX_GROUP} workloads")
    wl = np.empty((WL_NF, n))
    for i, nm in enumerate(names):
        wl[:, i] = spec_coef_row(specs[nm], coefs[nm])
    device = _device._dev(None)
    h = _device.hw_array(hw_vector(hw))
    with torch.cuda.device(device):
        d_wl = _device._to_dev(wl, device)
        d_b = _device._to_dev(np.array([batches[nm] for nm in names], np.int32), device)
        d_g = _device._to_dev(np.asarray(grid, np.int32), device)
        d_best = torch.empty(1 << n, dtype=torch.int64, device=device)
        d_err = torch.empty(1, dtype=torch.int32, device=device)
        rc = lib.igp_group_search_device(_device._ptr(d_wl), n, _device._ptr(d_b),
                                         _device._np_ptr(h), _device._ptr(d_g), len(grid),
                                         _device._ptr(d_best), _device._ptr(d_err),
                                         _device._stream(device))
        _device._check(rc)
        best = d_best.cpu().numpy().view(np.uint64)
        err = int(d_err.item())
    if err in (E_DENOM, E_ACTIVE_TIME):
        raise NonPositiveDenominatorError(
            "a unit vector of the exhaustive grid has a non-positive r + k4 or active time")
    return decode_keys(best, n)


def exhaustive_plan(workloads, hw, *, budget: OracleBudget | None = None,
                    b_max: int = DEFAULT_BATCH_CAP):
    """Optimal plan by full enumeration; raises InfeasibleError when none
    exists (oracle.py:130-201)."""
    budget = budget or OracleBudget()
    _check_unique_names(workloads)
    if len(workloads) > budget.max_workloads:
        raise BudgetExceededError(
            f"oracle accepts at most {budget.max_workloads} workloads, got {len(workloads)}")
    specs = {s.name: s for s, _ in workloads}
    coefs = {s.name: c for s, c in workloads}
    batches = {s.name: appropriate_batch(s, hw, b_max) for s, _ in workloads}
    lb_units = {s.name: _lower_bound_units(s, c, hw, batches[s.name]) for s, c in workloads}
    cap = max_units(hw)
    grid = tuple(sorted(budget.r_grid_units or range(1, cap + 1)))
    names = sorted(specs)
    results = group_search(specs, coefs, batches, names, hw, grid) if names else {}

    best_blocks = select_partition(names, results, budget.max_gpus)
    if best_blocks is None:
        raise InfeasibleError(f"no feasible plan within {budget.max_gpus} devices")
    placement = [([nm for nm, _ in block], [u for _, u in block], [batches[nm] for nm, _ in block])
                 for block in best_blocks]
    return _build_plan("oracle", hw, placement, specs, coefs, lb_units)
