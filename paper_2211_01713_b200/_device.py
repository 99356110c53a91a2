"""Array-level bridge between host numpy buffers and the C-ABI.

PyTorch is used only as plumbing: device allocations, the current CUDA stream
and pinned host staging.  Every computation happens in the sm_100a kernels of
``csrc/igniter_kernels.cu``; nothing here computes model values.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native
from .layout import HW_NF, WL_NF

def _torch():
    import torch
    return torch


def _dev(device=None):
    torch = _torch()
    if device is None:
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device(device)


def _to_dev(a: np.ndarray, device):
    torch = _torch()
    return torch.from_numpy(np.ascontiguousarray(a)).to(device)


def _ptr(t) -> ctypes.c_void_p:
    return ctypes.c_void_p(t.data_ptr()) if t is not None else ctypes.c_void_p(0)


def _np_ptr(a) -> ctypes.c_void_p:
    return ctypes.c_void_p(a.ctypes.data) if a is not None else ctypes.c_void_p(0)


def _stream(device):
    return ctypes.c_void_p(_torch().cuda.current_stream(device).cuda_stream)


def sm_count(device=None) -> int:
    return _torch().cuda.get_device_properties(_dev(device)).multi_processor_count


def workspace(nbytes: int, device=None, tag="plan"):
    """A device byte buffer of at least nbytes for one call.

    Allocated per call through the torch caching allocator on the current
    stream of `device`: the allocator recycles the block only after the work
    queued on that stream, so concurrent calls from several threads or streams
    never share scratch (the reference is pure Python and safe to call from
    several threads; so is this)."""
    torch = _torch()
    device = _dev(device)
    return torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=device)


IGP_F_HWS = 128  # include/igniter_b200.h: one hardware profile per scenario


def hw_array(hw_vec) -> np.ndarray:
    """One profile [HW_NF], or one per scenario [S, HW_NF] (IGP_F_HWS)."""
    h = np.ascontiguousarray(np.asarray(hw_vec, dtype=np.float64))
    assert h.shape[-1] == HW_NF and h.ndim in (1, 2)
    return h


def _hw_flags(h, flags):
    return flags | IGP_F_HWS if h.ndim == 2 else flags


def _check(rc: int):
    if rc == 8:  # IGP_E_CUDA
        raise RuntimeError(f"CUDA failure in libigniter_b200: {_native.last_error()}")
    if rc in (7, 9):
        from .errors import NativeError
        raise NativeError(
            "libigniter_b200 rejected the call "
            + ("(capacity: max_units(hw) exceeds igp_max_cap() or m >= 2^23)" if rc == 7
               else "(bad argument)"))


def _pool_overflow():
    from .errors import NativeError
    return NativeError("libigniter_b200: a scenario outgrew the largest record pool "
                       f"({POOL_RETRY} x m records)")


def batch_slots(m, hw_vec, b_max=32, flags=0, device=None) -> int:
    """Scenarios of m workloads the place kernel runs concurrently on `device`
    (one wave)."""
    torch = _torch()
    lib = _native.lib_for_compute()
    with torch.cuda.device(_dev(device)):
        n = int(lib.igp_plan_batch_slots(int(m), _np_ptr(hw_array(hw_vec)), int(b_max),
                                         int(flags)))
    if n <= 0:
        _check(-n)
    return n


def plan_workspace_bytes(S, m, hw_vec, b_max, flags):
    lib = _native.load()
    h = hw_array(hw_vec)
    return int(lib.igp_plan_workspace_bytes(S, m, _np_ptr(h), b_max, _hw_flags(h, flags)))


POOL_RETRY = 14  # tiles 4m + 8G <= 12m records plus <= 2m header slots always suffice


def plan_device(wl, hw_vec, b_max, rank, flags=0, device=None, want_pred=True):
    """Plan S scenarios; wl is [S,16,m] (or [16,m]) float64, rank [m] or [S,m].

    Returns numpy arrays (all per scenario, input order).  A scenario whose
    tiles outgrow the default record pool (IGP_E_CAPACITY) is re-planned with
    the pool size that is sufficient for any plan."""
    res = _plan_device_once(wl, hw_vec, b_max, rank, flags, device, want_pred)
    if (res["err"]["code"] == 7).any() and ((flags >> 8) & 0xFF) < POOL_RETRY:
        res = _plan_device_once(wl, hw_vec, b_max, rank, (flags & ~0xFF00) | (POOL_RETRY << 8),
                                device, want_pred)
    return res


def _plan_device_once(wl, hw_vec, b_max, rank, flags, device, want_pred):
    torch = _torch()
    lib = _native.lib_for_compute()
    device = _dev(device)
    wl = np.asarray(wl, dtype=np.float64)
    if wl.ndim == 2:
        wl = wl[None]
    S, nf, m = wl.shape
    assert nf == WL_NF
    rank = np.asarray(rank, dtype=np.int32)
    rank_stride = m if rank.ndim == 2 else 0
    h = hw_array(hw_vec)
    assert h.ndim == 1 or h.shape[0] == S, "one hardware profile per scenario"
    flags = _hw_flags(h, flags)
    with torch.cuda.device(device):
        d_wl = _to_dev(wl, device)
        d_rank = _to_dev(rank, device)
        # every output in one device buffer (one D2H copy): fp64 rows first,
        # then stats (int64), the int32 arrays and the error records
        mm = max(m, 1)
        n_pred = S * mm * 10 if want_pred else 0
        esz = ctypes.sizeof(_native.IgpError)
        o_st = n_pred * 8
        o_i32 = o_st + S * 6 * 8
        o_gc = o_i32 + 5 * S * mm * 4
        o_err = (o_gc + S * 4 + 7) // 8 * 8
        out = torch.empty(o_err + S * esz, dtype=torch.uint8, device=device)
        base = out.data_ptr()
        vp = ctypes.c_void_p
        i32p = [vp(base + o_i32 + f * S * mm * 4) for f in range(5)]
        nbytes = plan_workspace_bytes(S, m, h, b_max, flags)
        ws = workspace(nbytes, device)
        rc = lib.igp_plan_batch_device(
            _ptr(d_wl), S, m, _np_ptr(h), int(b_max), _ptr(d_rank), rank_stride,
            *i32p, vp(base) if want_pred else vp(0), vp(base + o_gc), vp(base + o_st),
            vp(base + o_err), _ptr(ws), ws.numel(), int(flags), _stream(device))
        _check(rc)
        host = out.cpu().numpy()
        out_i = host[o_i32:o_gc].view(np.int32).reshape(5, S, mm)[:, :, :m]
        res = dict(gpu_of=out_i[0], pos=out_i[1], units=out_i[2], batch=out_i[3], lb=out_i[4],
                   gpu_count=host[o_gc:o_gc + S * 4].view(np.int32),
                   stats=host[o_st:o_i32].view(np.int64).reshape(S, 6),
                   err=host[o_err:].view(_native.err_dtype()).reshape(S))
        if want_pred:
            res["pred"] = host[:n_pred * 8].view(np.float64).reshape(S, mm, 10)[:, :m]
    return res


def plan_host(wl, hw_vec, b_max, rank, flags=0, device=None, want_pred=True, out=None):
    """Host-buffer entry (igp_plan_batch_host): H2D, kernels, D2H, sync in one call.

    `wl`/`rank` should be pinned (page-locked) numpy views for full PCIe
    bandwidth; `out` may carry preallocated (pinned) output arrays.  Per-scenario
    planning errors are left in out["err"] (codes 1-6, as plan_device); a
    scenario whose tiles outgrow the default record pool is re-planned with the
    pool size that suffices for any plan, like plan_device."""
    torch = _torch()
    lib = _native.lib_for_compute()
    device = _dev(device)
    S, nf, m = wl.shape
    rank_stride = m if rank.ndim == 2 else 0
    h = hw_array(hw_vec)
    flags = _hw_flags(h, flags)
    if out is None:
        out = dict(gpu_of=np.empty((S, m), np.int32), pos=np.empty((S, m), np.int32),
                   units=np.empty((S, m), np.int32), batch=np.empty((S, m), np.int32),
                   lb=np.empty((S, m), np.int32), gpu_count=np.empty(S, np.int32),
                   stats=np.empty((S, 6), np.int64),
                   err=np.zeros(S, _native.err_dtype()))
        if want_pred:
            out["pred"] = np.empty((S, m, 10))
    with torch.cuda.device(device):
        for attempt in range(2):
            nbytes = host_workspace_bytes(S, m, h, b_max, flags, rank_stride, want_pred)
            ws = workspace(nbytes, device)
            rc = lib.igp_plan_batch_host(
                _np_ptr(wl), S, m, _np_ptr(h), int(b_max), _np_ptr(rank), rank_stride,
                _np_ptr(out["gpu_of"]), _np_ptr(out["pos"]), _np_ptr(out["units"]),
                _np_ptr(out["batch"]), _np_ptr(out["lb"]),
                _np_ptr(out.get("pred")) if want_pred else ctypes.c_void_p(0),
                _np_ptr(out["gpu_count"]), _np_ptr(out["stats"]), _np_ptr(out["err"]),
                _ptr(ws), ws.numel(), int(flags), _stream(device))
            del ws
            if rc in (8, 9):
                _check(rc)
            overflow = (out["err"]["code"] == 7).any()
            if rc == 7 and not overflow:
                _check(rc)  # a call-level limit, not a scenario's pool
            if not overflow:
                break
            if attempt or ((flags >> 8) & 0xFF) >= POOL_RETRY:
                raise _pool_overflow()
            flags = (flags & ~0xFF00) | (POOL_RETRY << 8)
    return out


def host_workspace_bytes(S, m, hw_vec, b_max, flags, rank_stride, want_pred):
    lib = _native.load()
    h = hw_array(hw_vec)
    return int(lib.igp_plan_host_workspace_bytes(S, m, _np_ptr(h), int(b_max),
                                                 int(_hw_flags(h, flags)), int(rank_stride),
                                                 int(bool(want_pred))))


def eval_states(wl, batch, r, ptr, hw_vec, check_capacity=False, device=None):
    """Batched _eval_entries rows for CSR device states."""
    torch = _torch()
    lib = _native.lib_for_compute()
    device = _dev(device)
    wl = np.asarray(wl, np.float64)
    n_rows = wl.shape[1]
    n_states = len(ptr) - 1
    h = hw_array(hw_vec)
    with torch.cuda.device(device):
        d_wl = _to_dev(wl, device)
        d_b = _to_dev(np.asarray(batch, np.int32), device)
        d_r = _to_dev(np.asarray(r, np.float64), device)
        d_p = _to_dev(np.asarray(ptr, np.int64), device)
        d_rows = torch.empty((max(n_rows, 1), 10), dtype=torch.float64, device=device)
        d_err = torch.empty((max(n_states, 1), ctypes.sizeof(_native.IgpError)),
                            dtype=torch.uint8, device=device)
        rc = lib.igp_eval_states_device(_ptr(d_wl), n_rows, _ptr(d_b), _ptr(d_r), _ptr(d_p),
                                        n_states, _np_ptr(h), int(bool(check_capacity)),
                                        _ptr(d_rows), _ptr(d_err), _stream(device))
        _check(rc)
        rows = d_rows.cpu().numpy()[:n_rows]
        err = d_err.cpu().numpy().view(_native.err_dtype()).reshape(-1)[:n_states]
    return rows, err


def components(wl, batch, r, co_cache, n_col, p_dem, hw_vec, device=None):
    """The model's component functions for n queries (igp_components_device):
    ([n, 10] fp64 columns, [n] int32 error codes)."""
    torch = _torch()
    lib = _native.lib_for_compute()
    device = _dev(device)
    wl = np.ascontiguousarray(wl, np.float64)
    n = wl.shape[1]
    h = hw_array(hw_vec)
    with torch.cuda.device(device):
        d = [_to_dev(np.ascontiguousarray(a, t), device) for a, t in (
            (wl, np.float64), (batch, np.int32), (r, np.float64), (co_cache, np.float64),
            (n_col, np.int32), (p_dem, np.float64))]
        d_out = torch.empty((max(n, 1), 10), dtype=torch.float64, device=device)
        d_code = torch.empty(max(n, 1), dtype=torch.int32, device=device)
        rc = lib.igp_components_device(n, *[_ptr(x) for x in d], _np_ptr(h), _ptr(d_out),
                                       _ptr(d_code), _stream(device))
        _check(rc)
        return d_out.cpu().numpy()[:n], d_code.cpu().numpy()[:n]


def power_demand(powers, hw_vec, device=None) -> float:
    """hw idle draw + the CPython sum of the solo powers (igp_power_demand_device)."""
    torch = _torch()
    lib = _native.lib_for_compute()
    device = _dev(device)
    p = np.ascontiguousarray(powers, np.float64)
    with torch.cuda.device(device):
        d_p = _to_dev(p if len(p) else np.zeros(1), device)
        d_out = torch.empty(1, dtype=torch.float64, device=device)
        _check(lib.igp_power_demand_device(len(p), _ptr(d_p), _np_ptr(hw_array(hw_vec)),
                                           _ptr(d_out), _stream(device)))
        return float(d_out.cpu()[0])


def alloc_units(wl, batch, r, ptr, hw_vec, device=None):
    """Batched Alg. 2 (reference evaluation sequence)."""
    torch = _torch()
    lib = _native.lib_for_compute()
    device = _dev(device)
    wl = np.asarray(wl, np.float64)
    n_rows = wl.shape[1]
    n_states = len(ptr) - 1
    h = hw_array(hw_vec)
    with torch.cuda.device(device):
        d_wl = _to_dev(wl, device)
        d_b = _to_dev(np.asarray(batch, np.int32), device)
        d_r = _to_dev(np.asarray(r, np.float64), device)
        d_p = _to_dev(np.asarray(ptr, np.int64), device)
        d_u = torch.empty(max(n_rows, 1), dtype=torch.int32, device=device)
        d_err = torch.empty((max(n_states, 1), ctypes.sizeof(_native.IgpError)),
                            dtype=torch.uint8, device=device)
        rc = lib.igp_alloc_units_device(_ptr(d_wl), n_rows, _ptr(d_b), _ptr(d_r), _ptr(d_p),
                                        n_states, _np_ptr(h), _ptr(d_u), _ptr(d_err),
                                        _stream(device))
        _check(rc)
        units = d_u.cpu().numpy()[:n_rows]
        err = d_err.cpu().numpy().view(_native.err_dtype()).reshape(-1)[:n_states]
    return units, err


def prologue(wl, hw_vec, b_max, batch_in=None, device=None):
    """appropriate_batch / _lower_bound_units for m workloads."""
    torch = _torch()
    lib = _native.lib_for_compute()
    device = _dev(device)
    wl = np.asarray(wl, np.float64)
    m = wl.shape[1]
    h = hw_array(hw_vec)
    with torch.cuda.device(device):
        d_wl = _to_dev(wl, device)
        d_bin = _to_dev(np.asarray(batch_in, np.int32), device) if batch_in is not None else None
        o = torch.empty((3, max(m, 1)), dtype=torch.int32, device=device)
        d_err = torch.empty(ctypes.sizeof(_native.IgpError), dtype=torch.uint8, device=device)
        rc = lib.igp_prologue_device(_ptr(d_wl), m, _np_ptr(h), int(b_max), _ptr(d_bin),
                                     _ptr(o[0]), _ptr(o[1]), _ptr(o[2]), _ptr(d_err),
                                     _stream(device))
        _check(rc)
        on = o.cpu().numpy()[:, :m]
        err = d_err.cpu().numpy().view(_native.err_dtype())[0]
    return on[0], on[1], on[2], err


def solo_grid(wl, hw_vec, b_max, device=None, count_evals=True):
    """Solo candidate grid: min feasible units per (workload, batch) plus the
    cheapest point per workload (igp_solo_grid_device)."""
    torch = _torch()
    lib = _native.lib_for_compute()
    device = _dev(device)
    wl = np.asarray(wl, np.float64)
    m = wl.shape[1]
    h = hw_array(hw_vec)
    with torch.cuda.device(device):
        d_wl = _to_dev(wl, device)
        d_min = torch.empty((max(m, 1), b_max), dtype=torch.int32, device=device)
        d_best = torch.empty((2, max(m, 1)), dtype=torch.int32, device=device)
        d_ev = torch.zeros(1, dtype=torch.int64, device=device) if count_evals else None
        rc = lib.igp_solo_grid_device(_ptr(d_wl), m, _np_ptr(h), int(b_max), _ptr(d_min),
                                      _ptr(d_best[0]), _ptr(d_best[1]), _ptr(d_ev),
                                      _stream(device))
        _check(rc)
        out = dict(min_units=d_min.cpu().numpy()[:m], best_u=d_best[0].cpu().numpy()[:m],
                   best_b=d_best[1].cpu().numpy()[:m])
        out["evals"] = int(d_ev.item()) if count_evals else -1
    return out
