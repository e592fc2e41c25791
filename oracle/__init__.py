"""CPU oracle for Fig. 1 `normalize` — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package.  It wraps the plain C oracle
``oracle/norm_oracle.c`` (fp64 + exact superaccumulator) with ctypes over numpy
arrays; it shares no code with the CUDA path.  See ``norm_oracle.h`` for the
passage each function follows and its parity-pin status.
"""
import ctypes
import os

import numpy as np

_DIR = os.path.dirname(os.path.abspath(__file__))
LITERAL, DENSE = 0, 1
_MODES = {"literal": LITERAL, "dense": DENSE}
_lib = None


def _mode(m):
    return _MODES[m] if isinstance(m, str) else int(m)


def lib():
    global _lib
    if _lib is None:
        path = os.path.join(_DIR, "liboracle.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run `make` (or __graft_entry__.build())")
        L = ctypes.CDLL(path)
        i64, vp, u64p = ctypes.c_int64, ctypes.c_void_p, ctypes.POINTER(ctypes.c_uint64)
        L.oracle_grid_blocks.argtypes = [i64]
        L.oracle_grid_blocks.restype = i64
        L.oracle_tid.argtypes = [i64, i64, ctypes.c_int]
        L.oracle_tid.restype = i64
        L.oracle_coverage_brute.argtypes = [i64, ctypes.c_int, vp]
        L.oracle_coverage_closed.argtypes = [i64, ctypes.c_int, ctypes.POINTER(i64),
                                             ctypes.POINTER(i64)]
        L.oracle_is_covered.argtypes = [i64, ctypes.c_int, i64]
        for f in ("oracle_sum_seq", "oracle_sum_exact", "oracle_sum_abs_exact"):
            getattr(L, f).argtypes = [vp, i64]
            getattr(L, f).restype = ctypes.c_double
        for f in ("oracle_form_thread", "oracle_form_block", "oracle_form_hoisted"):
            getattr(L, f).argtypes = [vp, vp, i64, ctypes.c_int, u64p]
        L.oracle_form_hoisted_mt.argtypes = [vp, vp, i64, ctypes.c_int, ctypes.c_int, u64p]
        L.oracle_sum_exact_mt.argtypes = [vp, i64, ctypes.c_int]
        L.oracle_sum_exact_mt.restype = ctypes.c_double
        L.oracle_rows_sum_exact.argtypes = [vp, vp, i64, i64, i64]
        L.oracle_rows.argtypes = [vp, vp, i64, i64, i64, i64, ctypes.c_int]
        L.oracle_replay.argtypes = [vp, vp, i64, ctypes.c_int, ctypes.c_float]
        L.oracle_softmax_rows.argtypes = [vp, vp, i64, i64, i64, i64]
        L.oracle_log_softmax_rows.argtypes = [vp, vp, i64, i64, i64, i64]
        dp = ctypes.POINTER(ctypes.c_double)
        L.oracle_nll_forward.argtypes = [vp, dp, vp, vp, vp, i64, i64, i64, ctypes.c_int, i64]
        L.oracle_nll_backward.argtypes = [vp, vp, vp, vp, ctypes.c_double, i64, i64, i64,
                                          ctypes.c_int, i64]
        L.oracle_bpnn_layerforward.argtypes = [vp, vp, vp, i64, i64]
        L.oracle_normalize_backward.argtypes = [vp, vp, vp, ctypes.c_double, i64, ctypes.c_int]
        L.oracle_softmax_backward_rows.argtypes = [vp, vp, vp, i64, i64, ctypes.c_int]
        _lib = L
    return _lib


def _f32(a):
    a = np.ascontiguousarray(a, dtype=np.float32)
    return a, a.ctypes.data


def grid_blocks(n):
    return lib().oracle_grid_blocks(n)


def tid(b, t, mode="literal"):
    return lib().oracle_tid(b, t, _mode(mode))


def coverage_brute(n, mode="literal"):
    mult = np.zeros(max(n, 1), dtype=np.uint32)
    assert lib().oracle_coverage_brute(n, _mode(mode), mult.ctypes.data) == 0
    return mult[:n]


def coverage_closed(n, mode="literal"):
    c, p = ctypes.c_int64(), ctypes.c_int64()
    assert lib().oracle_coverage_closed(n, _mode(mode), ctypes.byref(c), ctypes.byref(p)) == 0
    return c.value, p.value


def is_covered(n, i, mode="literal"):
    return bool(lib().oracle_is_covered(n, _mode(mode), i))


def covered_mask(n, mode="literal"):
    """Boolean mask of C(n) from the closed form (vectorised over i)."""
    count, prefix = coverage_closed(n, mode)
    i = np.arange(n, dtype=np.int64)
    if prefix >= 0:
        return i < prefix
    G = grid_blocks(n)
    return (i % 32) < G


def sum_seq(x):
    x, p = _f32(x)
    return lib().oracle_sum_seq(p, x.size)


def sum_exact(x):
    x, p = _f32(x)
    return lib().oracle_sum_exact(p, x.size)


def sum_abs_exact(x):
    x, p = _f32(x)
    return lib().oracle_sum_abs_exact(p, x.size)


def _form(fname, inp, mode, out=None):
    inp, pin = _f32(inp)
    if out is None:
        out = np.zeros_like(inp)
    assert out.dtype == np.float32 and out.flags["C_CONTIGUOUS"] and out.size == inp.size
    adds = ctypes.c_uint64(0)
    rc = getattr(lib(), fname)(out.ctypes.data, pin, inp.size, _mode(mode), ctypes.byref(adds))
    if rc:
        raise ValueError(f"{fname} rejected its arguments")
    return out, adds.value


def form_thread(inp, mode="literal", out=None):
    """Fig. 1 as written: O(N^2) adds. Returns (out, adds)."""
    return _form("oracle_form_thread", inp, mode, out)


def form_block(inp, mode="literal", out=None):
    """Per-block shared-memory variant: O(N^2/B) adds."""
    return _form("oracle_form_block", inp, mode, out)


def form_hoisted(inp, mode="literal", out=None):
    """After parallel LICM: O(N) adds."""
    return _form("oracle_form_hoisted", inp, mode, out)


def form_hoisted_mt(inp, mode="literal", threads=None, out=None):
    """Form 3 on `threads` host threads (default: all cores): exact per-chunk
    accumulators merged in chunk order, so bit-identical to form_hoisted.  Used to
    time the oracle on the host's cores (bench.py cpu_baseline)."""
    inp, pin = _f32(inp)
    if out is None:
        out = np.zeros_like(inp)
    assert out.dtype == np.float32 and out.flags["C_CONTIGUOUS"] and out.size == inp.size
    threads = (os.cpu_count() or 1) if threads is None else threads
    adds = ctypes.c_uint64(0)
    rc = lib().oracle_form_hoisted_mt(out.ctypes.data, pin, inp.size, _mode(mode), int(threads),
                                      ctypes.byref(adds))
    if rc:
        raise ValueError("oracle_form_hoisted_mt rejected its arguments")
    return out, adds.value


def sum_exact_mt(x, threads=None):
    """oracle_sum_exact on `threads` host threads (default: all cores); same value."""
    x, p = _f32(x)
    threads = (os.cpu_count() or 1) if threads is None else threads
    return lib().oracle_sum_exact_mt(p, x.size, int(threads))


def rows_sum_exact(x2d):
    """Exact sum of every row of a 2-D float32 array, correctly rounded to fp64."""
    x2d = np.ascontiguousarray(x2d, dtype=np.float32)
    R, C = x2d.shape
    S = np.zeros(R, dtype=np.float64)
    assert lib().oracle_rows_sum_exact(S.ctypes.data, x2d.ctypes.data, R, C, C) == 0
    return S


def normalize(inp, mode="literal", out=None):
    return form_hoisted(inp, mode, out)[0]


def rows(inp2d, mode="literal", out=None):
    inp2d = np.ascontiguousarray(inp2d, dtype=np.float32)
    R, C = inp2d.shape
    if out is None:
        out = np.zeros_like(inp2d)
    rc = lib().oracle_rows(out.ctypes.data, inp2d.ctypes.data, R, C, out.shape[1], C, _mode(mode))
    assert rc == 0
    return out


def replay(inp, s, mode="literal", out=None):
    inp, pin = _f32(inp)
    if out is None:
        out = np.zeros_like(inp)
    assert lib().oracle_replay(out.ctypes.data, pin, inp.size, _mode(mode), float(s)) == 0
    return out


# ------------------------------------------------ NEXT-2: softmax and ClassNLL

RED = {"none": 0, "mean": 1, "sum": 2}


def softmax_rows(x2d, log=False):
    """Row softmax (or log-softmax) in fp64, rounded once to fp32."""
    x2d = np.ascontiguousarray(x2d, dtype=np.float32)
    R, C = x2d.shape
    out = np.zeros_like(x2d)
    f = lib().oracle_log_softmax_rows if log else lib().oracle_softmax_rows
    assert f(out.ctypes.data, x2d.ctypes.data, R, C, C, C) == 0
    return out


def nll_forward(logp, target, weight=None, reduction="mean", ignore_index=-100):
    """ClassNLLCriterion_updateOutput in fp64: (loss, total_weight)."""
    logp = np.ascontiguousarray(logp, dtype=np.float32)
    target = np.ascontiguousarray(target, dtype=np.int64)
    N, C = logp.shape
    w = None if weight is None else np.ascontiguousarray(weight, dtype=np.float32)
    loss = np.zeros(max(N, 1) if reduction == "none" else 1, dtype=np.float64)
    tw = ctypes.c_double()
    rc = lib().oracle_nll_forward(loss.ctypes.data, ctypes.byref(tw), logp.ctypes.data,
                                  target.ctypes.data, None if w is None else w.ctypes.data,
                                  N, C, C, RED[reduction], ignore_index)
    assert rc == 0
    return (loss[:N] if reduction == "none" else loss[0]), tw.value


def nll_backward(grad_out, target, C, weight=None, reduction="mean", ignore_index=-100,
                 total_weight=1.0):
    """ClassNLLCriterion_updateGradInput in fp64: dense [N, C] gradient."""
    target = np.ascontiguousarray(target, dtype=np.int64)
    N = target.size
    g = np.ascontiguousarray(np.atleast_1d(grad_out), dtype=np.float64)
    w = None if weight is None else np.ascontiguousarray(weight, dtype=np.float32)
    grad = np.zeros((N, C), dtype=np.float64)
    rc = lib().oracle_nll_backward(grad.ctypes.data, g.ctypes.data, target.ctypes.data,
                                   None if w is None else w.ctypes.data, float(total_weight),
                                   N, C, C, RED[reduction], ignore_index)
    assert rc == 0
    return grad


# ------------------------------------------------ gradients (autograd of the ops)

def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def normalize_backward(g, y, S, mode="literal"):
    """d(sum g*y)/dx of the functional normalize y = normalize(x) (uncovered y_j = x_j),
    from g, y and the divisor S, in fp64: gx_j = [j in C] g_j / S + [j not in C] g_j -
    sum_{i in C} g_i y_i / S."""
    g, y = _f64(g), _f64(y)
    gx = np.empty_like(g)
    assert lib().oracle_normalize_backward(gx.ctypes.data, g.ctypes.data, y.ctypes.data, float(S),
                                           g.size, _mode(mode)) == 0
    return gx


def rows_normalize_backward(g2d, y2d, S_rows, mode="literal"):
    """normalize_backward of every row (row r with its own divisor S_rows[r])."""
    g2d, y2d = _f64(g2d), _f64(y2d)
    return np.stack([normalize_backward(g2d[r], y2d[r], S_rows[r], mode) for r in range(g2d.shape[0])]) \
        if g2d.shape[0] else np.empty_like(g2d)


def softmax_backward_rows(g2d, y2d, log=False):
    """Row softmax gradient y (g - sum g y), or log-softmax g - exp(y) sum g, in fp64."""
    g2d, y2d = _f64(g2d), _f64(y2d)
    R, C = g2d.shape
    gx = np.empty_like(g2d)
    assert lib().oracle_softmax_backward_rows(gx.ctypes.data, g2d.ctypes.data, y2d.ctypes.data, R, C,
                                              int(bool(log))) == 0
    return gx


# ------------------------------------------------ NEXT-4: backprop layerforward

def bpnn_layerforward(input_units, hidden_weights, hid=16):
    """Rodinia bpnn_layerforward (Fig. backprop) step by step in fp32.
    input_units: fp32[in + 1]; hidden_weights: fp32[(in + 1), hid + 1] (not modified).
    Returns (hidden_after, output[in])."""
    inp = np.ascontiguousarray(input_units, dtype=np.float32)
    hw = np.array(hidden_weights, dtype=np.float32, copy=True, order="C")
    n_in = inp.size - 1
    out = np.zeros(max(n_in, 1), dtype=np.float32)
    rc = lib().oracle_bpnn_layerforward(inp.ctypes.data, hw.ctypes.data, out.ctypes.data, n_in, hid)
    if rc:
        raise ValueError("bad backprop arguments (hid == 16, in % 16 == 0)")
    return hw, out[:n_in]
