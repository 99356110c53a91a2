"""Loader and ctypes prototypes for the sm_100a library (include/igniter_b200.h).

There is no fallback: if ``_lib/libigniter_b200.so`` is missing or cannot be
loaded, or no CUDA device is visible, every compute entry point raises.
``build()`` compiles the library in-tree with nvcc (``__graft_entry__.build``
calls it); the .so travels with the repository snapshot to the GPU box.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(PKG)
LIB_DIR = os.path.join(PKG, "_lib")
LIB_PATH = os.environ.get("IGP_LIB") or os.path.join(LIB_DIR, "libigniter_b200.so")
SOURCES = [os.path.join(PKG, "csrc", "igniter_kernels.cu")]
DEPS = SOURCES + [os.path.join(PKG, "csrc", "exact_fp64.cuh"), os.path.join(PKG, "csrc", "place.cuh"),
                  os.path.join(PKG, "csrc", "grid.cuh"), os.path.join(PKG, "csrc", "exhaustive.cuh"),
                  os.path.join(PKG, "csrc", "simulate.cuh"), os.path.join(PKG, "csrc", "components.cuh"),
                  os.path.join(PKG, "csrc", "window.cuh"), os.path.join(PKG, "csrc", "fast.cuh"),
                  os.path.join(PKG, "csrc", "smem_plan.cuh"),
                  os.path.join(REPO, "include", "igniter_b200.h")]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-fmad=false",  # CPython rounds every * and + separately: no FMA contraction
    "-Xcompiler", "-fPIC", "-shared",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.isabs(cand) and os.path.exists(cand) or not os.path.isabs(cand)):
            return cand
    return "nvcc"


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile the CUDA library in-tree (sm_100a).  Returns the .so path."""
    os.makedirs(LIB_DIR, exist_ok=True)
    stale = force or not os.path.exists(LIB_PATH) or any(
        os.path.getmtime(d) > os.path.getmtime(LIB_PATH) for d in DEPS)
    if stale:
        cmd = [nvcc(), *NVCC_FLAGS, "-o", LIB_PATH + ".tmp", *SOURCES]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        subprocess.check_call(cmd)
        os.replace(LIB_PATH + ".tmp", LIB_PATH)
    return LIB_PATH


class IgpError(ctypes.Structure):
    _fields_ = [("code", ctypes.c_int32), ("workload", ctypes.c_int32),
                ("gpu", ctypes.c_int32), ("pad", ctypes.c_int32),
                ("a", ctypes.c_double), ("b", ctypes.c_double), ("c", ctypes.c_double)]


ERR_DTYPE = None  # numpy structured dtype mirroring IgpError, set lazily


def err_dtype():
    global ERR_DTYPE
    if ERR_DTYPE is None:
        import numpy as np
        ERR_DTYPE = np.dtype([("code", np.int32), ("workload", np.int32), ("gpu", np.int32),
                              ("pad", np.int32), ("a", np.float64), ("b", np.float64),
                              ("c", np.float64)])
        assert ERR_DTYPE.itemsize == ctypes.sizeof(IgpError)
    return ERR_DTYPE


_VP = ctypes.c_void_p
_I = ctypes.c_int
_SZ = ctypes.c_size_t

# name -> (restype, argtypes); mirrors include/igniter_b200.h
PROTOTYPES = {
    "igp_abi_version": (_I, []),
    "igp_max_cap": (_I, []),
    "igp_last_error_string": (ctypes.c_char_p, []),
    "igp_plan_workspace_bytes": (_SZ, [_I, _I, _VP, _I, _I]),
    "igp_plan_batch_slots": (_I, [_I, _VP, _I, _I]),
    "igp_plan_host_workspace_bytes": (_SZ, [_I, _I, _VP, _I, _I, _I, _I]),
    "igp_plan_batch_device": (_I, [_VP, _I, _I, _VP, _I, _VP, _I, _VP, _VP, _VP, _VP, _VP,
                                   _VP, _VP, _VP, _VP, _VP, _SZ, _I, _VP]),
    "igp_plan_prepare_device": (_I, [_VP, _I, _I, _VP, _I, _VP, _I, _VP, _VP, _VP, _VP, _VP,
                                     _VP, _VP, _VP, _VP, _VP, _SZ, _I, _VP]),
    "igp_plan_place_device": (_I, [_VP, _I, _I, _VP, _I, _VP, _I, _VP, _VP, _VP, _VP, _VP,
                                   _VP, _VP, _VP, _VP, _VP, _SZ, _I, _VP]),
    "igp_plan_batch_host": (_I, [_VP, _I, _I, _VP, _I, _VP, _I, _VP, _VP, _VP, _VP, _VP,
                                 _VP, _VP, _VP, _VP, _VP, _SZ, _I, _VP]),
    "igp_eval_states_device": (_I, [_VP, _I, _VP, _VP, _VP, _I, _VP, _I, _VP, _VP, _VP]),
    "igp_alloc_units_device": (_I, [_VP, _I, _VP, _VP, _VP, _I, _VP, _VP, _VP, _VP]),
    "igp_prologue_device": (_I, [_VP, _I, _VP, _I, _VP, _VP, _VP, _VP, _VP, _VP]),
    "igp_solo_grid_device": (_I, [_VP, _I, _VP, _I, _VP, _VP, _VP, _VP, _VP]),
    "igp_group_search_device": (_I, [_VP, _I, _VP, _VP, _VP, _I, _VP, _VP, _VP]),
    "igp_simulate_device": (_I, [_I, _VP, _VP, _VP, ctypes.c_double, ctypes.c_double, _VP, _VP,
                                 _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP]),
    "igp_components_device": (_I, [_I, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP]),
    "igp_power_demand_device": (_I, [_I, _VP, _VP, _VP, _VP]),
    "igp_stream_workspace_bytes": (_SZ, [_I, _I, _VP, _I, _I]),
    "igp_stream_reset_device": (_I, [_I, _I, _VP, _I, _VP, _SZ, _I, _VP]),
    "igp_stream_push_device": (_I, [_VP, _I, _I, _I, _I, _VP, _I, _VP, _VP, _VP, _VP, _VP, _VP,
                                    _SZ, _I, _VP]),
    "igp_stream_snapshot_device": (_I, [_I, _I, _I, _VP, _I, _VP, _VP, _VP, _VP, _VP, _VP, _VP,
                                        _SZ, _I, _VP]),
}

_lib = None


def load(path: str | None = None):
    """Load the library (no GPU needed for loading/symbol lookup)."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = path or LIB_PATH
    if not os.path.exists(p):
        raise ImportError(
            f"{p} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback)")
    lib = ctypes.CDLL(p)
    for name, (res, args) in PROTOTYPES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if path is None:
        _lib = lib
    return lib


def lib_for_compute():
    """The library, after checking that a CUDA device is present."""
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2211_01713_b200 needs a CUDA device (sm_100a); "
                           "there is no CPU fallback")
    return load()


def last_error() -> str:
    return (load().igp_last_error_string() or b"").decode()
