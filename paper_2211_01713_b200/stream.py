"""Online re-provisioning stream on the B200 (BASELINE config 5).

The reference has no online API: ``plan()`` always sorts its workloads
(``planner.py:284``).  ``StreamPlanner`` applies one step of the greedy
placement (``planner.py:290-319``) per arrival, in arrival order, to device
state that persists across ``push`` calls.  Each arrival gets its batch and
lower bound from ``planner.py:76-120``.  An arrival whose prologue or
candidate evaluation raises the reference's ``PlanningError`` /
``NonPositiveDenominatorError`` is rejected and leaves the state unchanged.
This is the semantics of the reference-internals driver in
``tests/golden/make_golden.py`` (``stream_reference``).

Several independent streams (tenants) advance together: each push appends
the same number of arrivals to every stream, and one launch runs them all.
The per-GPU Neumaier fold states cached on the device make each arrival's
interference recompute incremental.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _device, _native
from .layout import ROW_NF, WL_NF, hw_vector, spec_coef_row

ERROR_NAMES = {1: "BatchCapExceededError", 2: "InfeasibleSloError", 3: "InfeasibleResourceError",
               4: "NonPositiveDenominatorError", 5: "NonPositiveDenominatorError"}


IGP_F_CTA = 4   # include/igniter_b200.h: one CTA per stream
IGP_F_COOP = 16  # a single stream's push on the whole GPU (cooperative steps)
IGP_F_GW2 = 32  # two warps per stream
COOP_FROM_ARRIVALS = 16_384  # whole_gpu streams: per-CTA steps before, cooperative after


def coop_ctas(k: int) -> int:
    """CTAs of the cooperative kernel for a push starting at arrival k of one
    stream: candidates per arrival grow about linearly with the arrivals so far
    (~3% of them), and 128 lanes per CTA each take one candidate; 0 = all."""
    return min(max(k // 1024, 16), 0xFFF)


class StreamPlanner:
    """n_streams independent arrival streams of up to ``capacity`` arrivals each."""

    def __init__(self, hw, *, capacity: int, n_streams: int = 1, b_max: int = 32, device=None,
                 flags: int | None = None, whole_gpu: bool = False):
        torch = _device._torch()
        self.lib = _native.lib_for_compute()
        self.hw = hw
        self.hv = _device.hw_array(hw_vector(hw))
        self.device = _device._dev(device)
        if whole_gpu and int(n_streams) != 1:
            raise ValueError("whole_gpu runs ONE stream on every SM")
        self.whole_gpu = bool(whole_gpu)
        if flags is None and whole_gpu:
            flags = IGP_F_CTA
        if flags is None:
            # two warps per stream while the streams leave warp slots free
            # (1,000 streams: 20.3 ms vs 24.6 ms with one warp, config 5)
            slots = torch.cuda.get_device_properties(self.device).multi_processor_count * 16
            flags = IGP_F_GW2 if 2 * int(n_streams) <= slots else 0
        self.S, self.C, self.b_max, self.flags = int(n_streams), int(capacity), int(b_max), int(flags)
        self.k = 0
        nbytes = int(self.lib.igp_stream_workspace_bytes(self.S, self.C, _device._np_ptr(self.hv),
                                                         self.b_max, self.flags))
        self.ws = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
        self._out = torch.empty((3, self.S, self.C), dtype=torch.int32, device=self.device)
        self.stats = torch.zeros((self.S, 6), dtype=torch.int64, device=self.device)
        self.err = torch.zeros((self.S, ctypes.sizeof(_native.IgpError)), dtype=torch.uint8,
                               device=self.device)
        self.reset()

    def _stream(self):
        return _device._stream(self.device)

    def reset(self):
        with _device._torch().cuda.device(self.device):
            rc = self.lib.igp_stream_reset_device(self.S, self.C, _device._np_ptr(self.hv),
                                                  self.b_max, _device._ptr(self.ws),
                                                  self.ws.numel(), self.flags, self._stream())
        _device._check(rc)
        self.k = 0

    def push_flags(self) -> int:
        """Flags of the next push: a whole_gpu stream runs its first
        COOP_FROM_ARRIVALS arrivals in one CTA (a step has few candidates),
        then every step on the whole GPU (cooperative kernel)."""
        if self.whole_gpu and self.k >= COOP_FROM_ARRIVALS:
            return self.flags | IGP_F_COOP | (coop_ctas(self.k) << 16)
        return self.flags

    def push_device(self, wl_new, flags: int | None = None):
        """Append n arrivals to every stream; ``wl_new`` is a float64 CUDA
        tensor [S, 16, n] on this device.  Returns device int32 tensors
        (gpu_of, pos, code) of shape [S, n]: the GPU and position each arrival
        was admitted to (-1 when rejected) and its IGP_E_* code."""
        S, nf, n = wl_new.shape
        assert S == self.S and nf == WL_NF and wl_new.is_contiguous()
        if self.k + n > self.C:
            raise ValueError(f"stream capacity {self.C} exceeded ({self.k} + {n})")
        out = self._out.view(-1)[: 3 * self.S * n].view(3, self.S, n)
        fl = self.push_flags() if flags is None else int(flags)
        with _device._torch().cuda.device(self.device):
            rc = self.lib.igp_stream_push_device(
                _device._ptr(wl_new), self.S, self.k, n, self.C, _device._np_ptr(self.hv),
                self.b_max, _device._ptr(out[0]), _device._ptr(out[1]), _device._ptr(out[2]),
                _device._ptr(self.stats), _device._ptr(self.err), _device._ptr(self.ws),
                self.ws.numel(), fl, self._stream())
        _device._check(rc)
        self.k += n
        return out[0], out[1], out[2]

    def push_arrays(self, wl_new: np.ndarray):
        """Host variant of push_device: numpy [S, 16, n] in, numpy arrays out."""
        torch = _device._torch()
        wl_new = np.ascontiguousarray(wl_new, dtype=np.float64)
        if wl_new.ndim == 2:
            wl_new = wl_new[None]
        with torch.cuda.device(self.device):
            d = torch.from_numpy(wl_new).to(self.device)
            g, p, c = self.push_device(d)
            g, p, c = (x.cpu().numpy().copy() for x in (g, p, c))
            self.check_errors()
        return dict(gpu_of=g, pos=p, code=c & 0xFF)

    def check_errors(self):
        """Raise if a stream's device state broke (record pool overflow)."""
        codes = self.err.cpu().numpy().view(_native.err_dtype()).reshape(self.S)["code"]
        if (codes != 0).any():
            from .errors import NativeError
            bad = int(np.nonzero(codes)[0][0])
            raise NativeError(f"stream {bad}: device state error {int(codes[bad])} "
                              "(record pool exhausted: recreate with a larger pool factor)")

    def push(self, workloads):
        """Append one arrival list per stream (lists of equal length of
        (WorkloadSpec, WorkloadCoefficients)).  Returns, per stream, a list
        of the GPU index each arrival joined, or the name of the reference
        exception that rejected it."""
        if workloads and hasattr(workloads[0][0], "slo_ms"):  # one flat list: a single stream
            workloads = [workloads]
        n = len(workloads[0])
        assert all(len(w) == n for w in workloads), "every stream gets the same number of arrivals"
        wl = np.empty((self.S, WL_NF, n))
        for s, ws in enumerate(workloads):
            for i, (spec, coef) in enumerate(ws):
                wl[s, :, i] = spec_coef_row(spec, coef)
        r = self.push_arrays(wl)
        return [[int(g) if g >= 0 else ERROR_NAMES.get(int(c), f"error {int(c)}")
                 for g, c in zip(r["gpu_of"][s], r["code"][s])] for s in range(self.S)]

    def snapshot(self, with_predictions: bool = False):
        """Current placement of every arrival so far: arrays [S, k] of GPU,
        position and units (units 0 / GPU -1 for rejected arrivals), the GPU
        count per stream and, optionally, the predict_gpu breakdown rows."""
        torch = _device._torch()
        S, k = self.S, self.k
        with torch.cuda.device(self.device):
            o = torch.empty((3, S, max(k, 1)), dtype=torch.int32, device=self.device)
            pred = (torch.empty((S, max(k, 1), ROW_NF), dtype=torch.float64, device=self.device)
                    if with_predictions else None)
            gc = torch.empty(S, dtype=torch.int32, device=self.device)
            err = torch.empty((S, ctypes.sizeof(_native.IgpError)), dtype=torch.uint8,
                              device=self.device)
            rc = self.lib.igp_stream_snapshot_device(
                S, k, self.C, _device._np_ptr(self.hv), self.b_max, _device._ptr(o[0]),
                _device._ptr(o[1]), _device._ptr(o[2]), _device._ptr(pred), _device._ptr(gc),
                _device._ptr(err), _device._ptr(self.ws), self.ws.numel(), self.flags,
                self._stream())
            _device._check(rc)
            on = o.cpu().numpy()[:, :, :k]
            res = dict(gpu_of=on[0], pos=on[1], units=on[2], gpu_count=gc.cpu().numpy(),
                       err=err.cpu().numpy().view(_native.err_dtype()).reshape(S))
            if with_predictions:
                res["pred"] = pred.cpu().numpy()[:, :k]
        return res
