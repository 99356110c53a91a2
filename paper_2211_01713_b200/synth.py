"""Synthetic scenario batches for benchmarks (not used by plan()).

Draws workloads from the distributions of the reference's test generator
(``pkg/tests/support.py:59-103``: slo U(20,80) ms, rate U(50,500) req/s,
d_load U(0.05,1), d_feedback U(0.001,0.05), coefficients per
``random_coefficients``) but vectorised over whole batches with numpy, so a
4,096 x 10,000 batch takes seconds instead of minutes.  Like the reference
generator it rejects workloads a single device cannot host alone: the
rejection predicate restates Eq. 19/20 (planner.py:76-120) in elementwise
numpy fp64 (one rounding per operation, same association).  The stream is
NOT the reference's (use tests/instances.py for that); it is seeded and
deterministic.
"""

from __future__ import annotations

import numpy as np

from .layout import WL, WL_NF


def _feasible(wl: np.ndarray, hw, b_max: int) -> np.ndarray:
    slo, rate_rps = wl[WL["slo_ms"]], wl[WL["rate_rps"]]
    dl, dfb = wl[WL["d_load_mb"]], wl[WL["d_feedback_mb"]]
    bw = hw.pcie_bw_mb_per_ms
    rate = rate_rps / 1000.0
    b = np.maximum(1.0, np.ceil(((slo * rate) * bw) / (2.0 * (bw + rate * dl))))
    ok = b <= b_max
    delta = ((slo / 2.0 - ((dl + dfb) * b) / bw) - wl[WL["k5"]]) - wl[WL["k_sch_ms"]] * wl[WL["n_kernels"]]
    ok &= delta > 0
    gamma = ((wl[WL["k1"]] * b) * b + wl[WL["k2"]] * b) + wl[WL["k3"]]
    with np.errstate(divide="ignore", invalid="ignore"):
        u = np.maximum(1.0, np.ceil(gamma / (delta * hw.r_unit) - wl[WL["k4"]] / hw.r_unit))
    cap = int(round(hw.r_max / hw.r_unit))
    ok &= u <= cap
    return ok


def _draw(rng, n, slo, rate):
    wl = np.empty((WL_NF, n), dtype=np.float64)
    wl[WL["slo_ms"]] = rng.uniform(slo[0], slo[1], n)
    wl[WL["rate_rps"]] = rng.uniform(rate[0], rate[1], n)
    wl[WL["d_load_mb"]] = rng.uniform(0.05, 1.0, n)
    wl[WL["d_feedback_mb"]] = rng.uniform(0.001, 0.05, n)
    wl[WL["n_kernels"]] = rng.integers(20, 301, n).astype(np.float64)
    wl[WL["k_sch_ms"]] = rng.uniform(0.0005, 0.004, n)
    wl[WL["k1"]] = rng.uniform(0.0, 0.01, n)
    wl[WL["k2"]] = rng.uniform(0.01, 0.1, n)
    wl[WL["k3"]] = rng.uniform(0.5, 10.0, n)
    wl[WL["k4"]] = rng.uniform(0.0, 0.2, n)
    wl[WL["k5"]] = rng.uniform(0.05, 0.5, n)
    wl[WL["alpha_power_w"]] = rng.uniform(10.0, 60.0, n)
    wl[WL["beta_power_w"]] = rng.uniform(20.0, 80.0, n)
    wl[WL["alpha_cacheutil"]] = rng.uniform(0.01, 0.08, n)
    wl[WL["beta_cacheutil"]] = rng.uniform(0.02, 0.15, n)
    wl[WL["alpha_cache"]] = rng.uniform(0.0, 0.4, n)
    return wl


def scenarios(n_scen: int, m: int, hw, seed: int = 0, *, slo=(20.0, 80.0),
              rate=(50.0, 500.0), b_max: int = 32, out: np.ndarray | None = None):
    """Return (wl [S,16,m] float64, names [m]) of feasible synthetic workloads.

    Names are ``w{i:04d}`` like the reference generator, so for m > 10,000 the
    string tie-break order differs from index order (SURVEY.md finding 9)."""
    rng = np.random.default_rng(seed)
    total = n_scen * m
    wl = out if out is not None else np.empty((n_scen, WL_NF, m), dtype=np.float64)
    flat = np.empty((WL_NF, total), dtype=np.float64)
    filled = 0
    while filled < total:
        need = total - filled
        cand = _draw(rng, int(need * 1.6) + 64, slo, rate)
        good = cand[:, _feasible(cand, hw, b_max)]
        take = min(need, good.shape[1])
        flat[:, filled:filled + take] = good[:, :take]
        filled += take
    wl[...] = flat.reshape(WL_NF, n_scen, m).transpose(1, 0, 2)
    names = np.array([f"w{i:04d}" for i in range(m)])
    return wl, names


def scenario_batch(n_scen: int, m: int, hw, seed: int = 0, *, indices=None,
                   slo=(20.0, 80.0), rate=(50.0, 500.0), b_max: int = 32):
    """Like ``scenarios`` but scenario s draws from its own stream
    (``SeedSequence([seed, s])``), so any subset of a batch can be rebuilt
    on its own: ``indices`` selects the scenarios to return (default: all
    n_scen).  The benchmark's GPU arm plans the whole batch and its CPU arms
    plan, and check, a subset of the SAME scenarios."""
    idx = range(n_scen) if indices is None else [int(i) for i in indices]
    wl = np.empty((len(idx), WL_NF, m), dtype=np.float64)
    for o, s in enumerate(idx):
        if not 0 <= s < n_scen:
            raise IndexError(f"scenario {s} outside the batch of {n_scen}")
        rng = np.random.default_rng(np.random.SeedSequence([seed, s]))
        filled = 0
        while filled < m:
            cand = _draw(rng, int((m - filled) * 1.6) + 64, slo, rate)
            good = cand[:, _feasible(cand, hw, b_max)]
            take = min(m - filled, good.shape[1])
            wl[o, :, filled:filled + take] = good[:, :take]
            filled += take
    names = np.array([f"w{i:04d}" for i in range(m)])
    return wl, names
