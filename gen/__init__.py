"""Seeded synthetic input generator (see gen/norm_gen.h).

Shared by the oracle side and the CUDA side; contains no arithmetic of the
method.  ``fill_host`` writes a numpy float32 array, ``fill_cuda`` a CUDA
torch tensor (the device fill lives in its own ``libnormgen_cuda.so``, not in
libnorm, so the product library carries only the method).
"""
import ctypes
import os

import numpy as np

_DIR = os.path.dirname(os.path.abspath(__file__))

UNIT, CONST, RAMP, SIGNED, WIDE = range(5)
DISTS = {"unit": UNIT, "const": CONST, "ramp": RAMP, "signed": SIGNED, "wide": WIDE}

_host = None
_cuda = None


def _load_host():
    global _host
    if _host is None:
        path = os.path.join(_DIR, "libnormgen.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run `make` (or __graft_entry__.build())")
        lib = ctypes.CDLL(path)
        lib.ng_fill_host.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_uint64,
                                     ctypes.c_int, ctypes.c_int64]
        lib.ng_fill_host.restype = ctypes.c_int
        lib.ng_value_host.argtypes = [ctypes.c_uint64, ctypes.c_int, ctypes.c_int64]
        lib.ng_value_host.restype = ctypes.c_float
        _host = lib
    return _host


def _load_cuda():
    global _cuda
    if _cuda is None:
        path = os.path.join(_DIR, "libnormgen_cuda.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run `make` (or __graft_entry__.build())")
        lib = ctypes.CDLL(path)
        lib.ng_fill_cuda.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_uint64,
                                     ctypes.c_int, ctypes.c_int64, ctypes.c_void_p]
        lib.ng_fill_cuda.restype = ctypes.c_int
        _cuda = lib
    return _cuda


def _dist(d):
    return DISTS[d] if isinstance(d, str) else int(d)


def fill_host(arr, seed=0, dist=UNIT, offset=0):
    """Fill a contiguous float32 numpy array (or CPU torch tensor) in place."""
    if hasattr(arr, "data_ptr"):
        assert arr.dtype.__str__() == "torch.float32" and arr.is_contiguous()
        ptr, n = arr.data_ptr(), arr.numel()
    else:
        assert arr.dtype == np.float32 and arr.flags["C_CONTIGUOUS"]
        ptr, n = arr.ctypes.data, arr.size
    rc = _load_host().ng_fill_host(ptr, n, seed, _dist(dist), offset)
    if rc:
        raise ValueError(f"ng_fill_host failed ({rc})")
    return arr


def make_host(n, seed=0, dist=UNIT, offset=0):
    return fill_host(np.empty(n, dtype=np.float32), seed, dist, offset)


def value(seed, dist, i):
    return _load_host().ng_value_host(seed, _dist(dist), i)


def fill_cuda(t, seed=0, dist=UNIT, offset=0, stream=None):
    """Fill a contiguous float32 CUDA tensor in place on ``stream`` (default: current)."""
    import torch
    assert t.is_cuda and t.dtype == torch.float32 and t.is_contiguous()
    s = stream if stream is not None else torch.cuda.current_stream(t.device)
    rc = _load_cuda().ng_fill_cuda(t.data_ptr(), t.numel(), seed, _dist(dist), offset,
                                   s.cuda_stream)
    if rc:
        raise RuntimeError(f"ng_fill_cuda failed ({rc})")
    return t
