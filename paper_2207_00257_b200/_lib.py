"""ctypes marshalling for libnorm.so (see include/libnorm.h for semantics)."""
import ctypes
import os

_DIR = os.path.dirname(os.path.abspath(__file__))
# LIBNORM_SO overrides the library path; used only by tests/test_gpu_faults.py to
# load the fault-injected builds in a subprocess.
_SO = os.environ.get("LIBNORM_SO") or os.path.join(_DIR, "libnorm.so")

INDEX = {"literal": 0, "dense": 1}
PATH = {"auto": 0, "two_pass": 1, "fused": 2, "small": 3, "mid": 4, "cluster": 5}
STATUS = ["NORM_OK", "NORM_ERR_INVALID_VALUE", "NORM_ERR_OVERLAP", "NORM_ERR_CUDA",
          "NORM_ERR_NCCL", "NORM_ERR_WORKSPACE", "NORM_ERR_UNSUPPORTED"]


class NormOpts(ctypes.Structure):
    _fields_ = [("stream", ctypes.c_void_p), ("index", ctypes.c_int32), ("path", ctypes.c_int32),
                ("sum_out", ctypes.c_void_p), ("sum_out_f64", ctypes.c_void_p),
                ("workspace", ctypes.c_void_p), ("workspace_bytes", ctypes.c_size_t),
                ("flags", ctypes.c_uint32), ("reserved", ctypes.c_uint32)]


FLAG_TRUSTED_PTRS = 1  # NORM_FLAG_TRUSTED_PTRS


class NormShard(ctypes.Structure):
    _fields_ = [("nranges", ctypes.c_int32), ("begin", ctypes.c_int64 * 2),
                ("len", ctypes.c_int64 * 2)]

    def ranges(self):
        return [(self.begin[k], self.len[k]) for k in range(self.nranges)]


class NormError(RuntimeError):
    def __init__(self, status, detail):
        self.status = status
        name = STATUS[status] if 0 <= status < len(STATUS) else str(status)
        super().__init__(f"{name}: {detail}")


_lib = None


def lib():
    """Load libnorm.so (built in-tree by `make` / __graft_entry__.build()); raise if absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(_SO):
            raise ImportError(f"{_SO} is missing: build it with `make` (no CPU fallback exists)")
        L = ctypes.CDLL(_SO)
        i64, i32, vp = ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p
        optp = ctypes.POINTER(NormOpts)
        sig = {
            "norm_launch": [vp, vp, i64],
            "norm_launch_ex": [vp, vp, i64, optp],
            "norm_launch_host": [vp, vp, i64, optp],
            "norm_launch_form": [vp, vp, i64, i32, optp],
            "norm_graph_create": [ctypes.POINTER(vp), vp, vp, i64, optp],
            "norm_graph_launch": [vp, vp],
            "norm_graph_destroy": [vp],
            "norm_softmax_rows": [vp, vp, i64, i64, i64, i64, i32, optp],
            "norm_bpnn_layerforward": [vp, vp, vp, i64, i64, i32, optp],
            "norm_nll_forward": [vp, vp, vp, vp, vp, i64, i64, i64, i32, i64, optp],
            "norm_nll_backward": [vp, vp, vp, vp, vp, i64, i64, i64, i32, i64, optp],
            "norm_rows": [vp, vp, i64, i64, i64, i64, optp],
            "norm_launch_backward": [vp, vp, vp, vp, i64, optp],
            "norm_rows_backward": [vp, vp, vp, vp, i64, i64, i64, optp],
            "norm_softmax_rows_backward": [vp, vp, vp, i64, i64, i64, i32, optp],
            "norm_coverage": [i64, i32, ctypes.POINTER(i64), ctypes.POINTER(i64)],
            "norm_workspace_bytes": [i64, optp, ctypes.POINTER(ctypes.c_size_t)],
            "norm_algorithmic_bytes": [i64, i32, ctypes.POINTER(i64)],
            "norm_choose_path": [i64, i64, i32, ctypes.POINTER(i32)],
            "norm_comm_unique_id": [ctypes.c_char_p],
            "norm_comm_init": [ctypes.POINTER(vp), i32, i32, ctypes.c_char_p],
            "norm_comm_destroy": [vp],
            "norm_comm_set_mode": [vp, i32],
            "norm_plan_shards": [i64, i32, i32, i32, ctypes.POINTER(NormShard)],
            "norm_launch_sharded": [vp, vp, vp, ctypes.POINTER(NormShard), i64, optp],
            "norm_shard_partial": [vp, vp, i64, optp],
            "norm_peer_create": [ctypes.POINTER(vp), i32, i32, ctypes.c_char_p],
            "norm_peer_connect": [vp, ctypes.c_char_p],
            "norm_peer_destroy": [vp],
            "norm_launch_sharded_peer": [vp, vp, vp, ctypes.POINTER(NormShard), i64, optp],
            "norm_shard_finish": [vp, vp, ctypes.POINTER(NormShard), i64, vp, i32, optp],
        }
        for name, args in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = ctypes.c_int
        L.norm_debug_set_events.argtypes = [vp, vp]
        L.norm_debug_set_events.restype = ctypes.c_int
        L.norm_cache_release.argtypes = []
        L.norm_cache_release.restype = ctypes.c_int
        L.norm_status_string.argtypes = [ctypes.c_int]
        L.norm_status_string.restype = ctypes.c_char_p
        L.norm_last_error.argtypes = []
        L.norm_last_error.restype = ctypes.c_char_p
        _lib = L
    return _lib


def cache_release():
    """Free libnorm's internal workspaces and host-staging buffers (norm_cache_release)."""
    _check(lib().norm_cache_release())


def status_string(s):
    return lib().norm_status_string(s).decode()


def last_error():
    return lib().norm_last_error().decode()


def _check(st):
    if st != 0:
        raise NormError(st, last_error())


def _enum(table, v):
    return table[v] if isinstance(v, str) else int(v)


def _ptr(t):
    return None if t is None else t.data_ptr()


def _stream_handle(stream, device=None):
    import torch
    if stream is None:
        stream = torch.cuda.current_stream(device)
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


def _opts(index, path, stream, sum_out, sum_out_f64, workspace=None, device=None, flags=0):
    o = NormOpts()
    o.stream = _stream_handle(stream, device)
    o.index = _enum(INDEX, index)
    o.path = _enum(PATH, path)
    o.sum_out = _ptr(sum_out)
    o.sum_out_f64 = _ptr(sum_out_f64)
    o.flags = flags
    if workspace is not None:
        o.workspace = workspace.data_ptr()
        o.workspace_bytes = workspace.numel() * workspace.element_size()
    return o


class _call:
    """Context of one libnorm call from Python: makes the tensors' device current
    (libnorm launches on the current device; a tensor on another GPU would be a
    device fault) and, for the bench, arms norm_debug_set_events with a
    (begin, end) torch.cuda.Event pair for the duration of the call."""
    __slots__ = ("dev", "events", "prev")

    def __init__(self, device, events=None):
        self.dev = device
        self.events = events
        self.prev = None

    def __enter__(self):
        import torch
        if self.dev is not None and self.dev.type == "cuda":
            idx = self.dev.index if self.dev.index is not None else torch.cuda.current_device()
            cur = torch.cuda.current_device()
            if idx != cur:
                self.prev = cur
                torch.cuda.set_device(idx)
        if self.events is not None:
            for ev in self.events:  # torch creates the CUDA event lazily, on first record
                if not ev.cuda_event:
                    ev.record()
            lib().norm_debug_set_events(self.events[0].cuda_event, self.events[1].cuda_event)
        return self

    def __exit__(self, *a):
        if self.events is not None:
            lib().norm_debug_set_events(None, None)
        if self.prev is not None:
            import torch
            torch.cuda.set_device(self.prev)
        return False


def _check_f32(t, name, cuda=True):
    import torch
    if t.dtype != torch.float32:
        raise TypeError(f"{name} must be float32")
    if cuda and not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor")


def normalize(out, inp, index="literal", path="auto", stream=None, sum_out=None,
              sum_out_f64=None, workspace=None, events=None, trusted=False):
    """out[C(n)] = inp[C(n)] / sum(inp) on the GPU (norm_launch_ex).  Returns out.

    out, inp: contiguous float32 CUDA tensors of equal numel (out may be inp).
    sum_out / sum_out_f64: optional 1-element float32 / float64 CUDA tensors.
    events: optional (begin, end) torch.cuda.Event pair recorded around the call's
    dominant kernel (norm_debug_set_events).
    trusted: pass NORM_FLAG_TRUSTED_PTRS (skip libnorm's per-pointer checks; the
    tensors are CUDA tensors of one device, checked here) -- for launch-bound sizes.
    """
    _check_f32(out, "out")
    _check_f32(inp, "inp")
    if not (out.is_contiguous() and inp.is_contiguous()) or out.numel() != inp.numel():
        raise ValueError("out and inp must be contiguous with equal numel")
    flags = 0
    if trusted:
        for t in (out, sum_out, sum_out_f64):
            if t is not None and (not t.is_cuda or t.device != inp.device):
                raise ValueError("trusted=True needs every tensor on inp's CUDA device")
        flags = FLAG_TRUSTED_PTRS
    o = _opts(index, path, stream, sum_out, sum_out_f64, workspace, inp.device, flags)
    with _call(inp.device, events):
        _check(lib().norm_launch_ex(out.data_ptr(), inp.data_ptr(), inp.numel(), ctypes.byref(o)))
    return out


FORM = {"hoisted": 0, "per_block": 1, "per_thread": 2}


def normalize_form(out, inp, form="hoisted", index="literal", stream=None, sum_out=None,
                   sum_out_f64=None):
    """Fig. 1 before / after parallel LICM (norm_launch_form): "per_thread" (as
    printed, O(N^2)), "per_block" (shared-memory comment, O(N^2/B)) or "hoisted"."""
    _check_f32(out, "out")
    _check_f32(inp, "inp")
    if not (out.is_contiguous() and inp.is_contiguous()) or out.numel() != inp.numel():
        raise ValueError("out and inp must be contiguous with equal numel")
    o = _opts(index, "auto", stream, sum_out, sum_out_f64, device=inp.device)
    with _call(inp.device):
        _check(lib().norm_launch_form(out.data_ptr(), inp.data_ptr(), inp.numel(), _enum(FORM, form),
                                      ctypes.byref(o)))
    return out


REDUCTION = {"none": 0, "mean": 1, "sum": 2}


def softmax_rows(out, inp, log=False, stream=None):
    """Row softmax / log-softmax of 2-D float32 CUDA tensors (norm_softmax_rows)."""
    _check_f32(out, "out")
    _check_f32(inp, "inp")
    if out.dim() != 2 or out.shape != inp.shape:
        raise ValueError("out and inp must be 2-D with equal shapes")
    if out.shape[1] > 1 and (out.stride(1) != 1 or inp.stride(1) != 1):
        raise ValueError("rows must have unit column stride")
    o = _opts("literal", "auto", stream, None, None, device=inp.device)
    with _call(inp.device):
        _check(lib().norm_softmax_rows(out.data_ptr(), inp.data_ptr(), inp.shape[0], inp.shape[1],
                                       out.stride(0), inp.stride(0), 1 if log else 0, ctypes.byref(o)))
    return out


def nll_forward(logp, target, weight=None, reduction="mean", ignore_index=-100, stream=None):
    """ClassNLLCriterion_updateOutput: returns (loss, total_weight) CUDA tensors."""
    import torch
    _check_f32(logp, "logp")
    if logp.dim() != 2 or (logp.shape[1] > 1 and logp.stride(1) != 1):
        raise ValueError("logp must be 2-D with unit column stride")
    if target.dtype != torch.int64 or not target.is_cuda or not target.is_contiguous():
        raise ValueError("target must be a contiguous int64 CUDA tensor")
    N, C = logp.shape
    red = _enum(REDUCTION, reduction)
    loss = torch.empty(N if red == 0 else 1, dtype=torch.float32, device=logp.device)
    tw = torch.empty(1, dtype=torch.float32, device=logp.device)
    o = _opts("literal", "auto", stream, None, None, device=logp.device)
    with _call(logp.device):
        _check(lib().norm_nll_forward(loss.data_ptr(), tw.data_ptr(), logp.data_ptr(), target.data_ptr(),
                                      _ptr(weight), N, C, logp.stride(0), red, ignore_index,
                                      ctypes.byref(o)))
    return (loss if red == 0 else loss[0]), tw


def nll_backward(grad_out, logp_shape, target, total_weight, weight=None, reduction="mean",
                 ignore_index=-100, grad=None, stream=None):
    """ClassNLLCriterion_updateGradInput: returns the dense [N, C] float32 gradient."""
    import torch
    N, C = logp_shape
    if grad is None:
        grad = torch.empty((N, C), dtype=torch.float32, device=target.device)
    o = _opts("literal", "auto", stream, None, None, device=target.device)
    with _call(target.device):
        _check(lib().norm_nll_backward(grad.data_ptr(), grad_out.data_ptr(), target.data_ptr(),
                                       _ptr(weight), _ptr(total_weight), N, C, grad.stride(0),
                                       _enum(REDUCTION, reduction), ignore_index, ctypes.byref(o)))
    return grad


BP_VARIANT = {"printed": 0, "eliminated": 1, "register": 2, "tma": 3}


def bpnn_layerforward(input_units, hidden, output, variant="register", stream=None):
    """Rodinia backprop layer-forward (Fig. backprop): updates `hidden` in place and
    writes the per-block column sums to `output` (norm_bpnn_layerforward)."""
    for t, nm in ((input_units, "input"), (hidden, "hidden"), (output, "output")):
        _check_f32(t, nm)
        if not t.is_contiguous():
            raise ValueError(f"{nm} must be contiguous")
    n_in = input_units.numel() - 1
    hid = hidden.shape[-1] - 1 if hidden.dim() == 2 else 16
    if hidden.numel() != (n_in + 1) * (hid + 1) or output.numel() < n_in:
        raise ValueError("shapes: input [in+1], hidden [in+1, hid+1], output [in]")
    o = _opts("literal", "auto", stream, None, None, device=hidden.device)
    with _call(hidden.device):
        _check(lib().norm_bpnn_layerforward(input_units.data_ptr(), hidden.data_ptr(), output.data_ptr(),
                                            n_in, hid, _enum(BP_VARIANT, variant), ctypes.byref(o)))
    return hidden, output


class BoundNormalize:
    """One normalize call bound to fixed tensors for launch-bound Python callers
    (configs 1-2: n = 1024, 2^20 + 7): the tensors are validated, the options
    struct (stream, index, path, outputs, NORM_FLAG_TRUSTED_PTRS) built and the
    ctypes argument tuple prepared once; each ``()`` is a single norm_launch_ex
    call on the stream given at construction (default: the current stream then).
    The tensors must stay alive and on their device; the device must be current
    at call time (checked: a call on another device is refused, not launched).
    Same kernels and results as ``normalize``."""

    __slots__ = ("_keep", "_fn", "_args", "_dev")

    def __init__(self, out, inp, index="literal", path="auto", stream=None, sum_out=None, sum_out_f64=None):
        _check_f32(out, "out")
        _check_f32(inp, "inp")
        if not (out.is_contiguous() and inp.is_contiguous()) or out.numel() != inp.numel():
            raise ValueError("out and inp must be contiguous with equal numel")
        for t in (out, sum_out, sum_out_f64):
            if t is not None and (not t.is_cuda or t.device != inp.device):
                raise ValueError("every tensor must be on inp's CUDA device")
        self._keep = (out, inp, sum_out, sum_out_f64)
        o = _opts(index, path, stream, sum_out, sum_out_f64, None, inp.device, FLAG_TRUSTED_PTRS)
        self._dev = inp.device.index if inp.device.index is not None else 0
        self._fn = lib().norm_launch_ex
        self._args = (ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(inp.data_ptr()),
                      ctypes.c_int64(inp.numel()), ctypes.byref(o), o)

    def __call__(self):
        import torch
        if torch.cuda.current_device() != self._dev:
            raise ValueError(f"BoundNormalize: device {self._dev} is not current")
        a = self._args
        st = self._fn(a[0], a[1], a[2], a[3])
        if st != 0:
            raise NormError(st, last_error())
        return self._keep[0]


class NormGraph:
    """One normalize call captured as a CUDA graph (norm_graph_create): replay with
    launch(stream) -- one cudaGraphLaunch for the reduce + scale pair."""

    def __init__(self, out, inp, index="literal", path="auto", sum_out=None, sum_out_f64=None):
        _check_f32(out, "out")
        _check_f32(inp, "inp")
        if not (out.is_contiguous() and inp.is_contiguous()) or out.numel() != inp.numel():
            raise ValueError("out and inp must be contiguous with equal numel")
        self._keep = (out, inp, sum_out, sum_out_f64)  # the graph holds raw pointers
        o = _opts(index, path, None, sum_out, sum_out_f64, device=inp.device)
        h = ctypes.c_void_p()
        with _call(inp.device):
            _check(lib().norm_graph_create(ctypes.byref(h), out.data_ptr(), inp.data_ptr(), inp.numel(),
                                           ctypes.byref(o)))
        self._h = h
        self._device = inp.device

    def launch(self, stream=None):
        with _call(self._device):
            _check(lib().norm_graph_launch(self._h, _stream_handle(stream, self._device)))

    def destroy(self):
        if self._h:
            _check(lib().norm_graph_destroy(self._h))
            self._h = None

    def __del__(self):
        try:
            self.destroy()
        except Exception:  # noqa: BLE001 - interpreter shutdown
            pass


def normalize_rows(out, inp, index="literal", stream=None, sum_out=None, sum_out_f64=None):
    """Row-wise normalize of 2-D float32 CUDA tensors (unit column stride)."""
    _check_f32(out, "out")
    _check_f32(inp, "inp")
    if out.dim() != 2 or inp.dim() != 2 or out.shape != inp.shape:
        raise ValueError("out and inp must be 2-D with equal shapes")
    if (out.shape[1] > 1 and (out.stride(1) != 1 or inp.stride(1) != 1)):
        raise ValueError("rows must have unit column stride")
    rows, cols = inp.shape
    o = _opts(index, "auto", stream, sum_out, sum_out_f64, device=inp.device)
    with _call(inp.device):
        _check(lib().norm_rows(out.data_ptr(), inp.data_ptr(), rows, cols, out.stride(0),
                               inp.stride(0), ctypes.byref(o)))
    return out


def _check_same(ts, names, shape=None):
    ref = ts[0]
    for t, nm in zip(ts, names):
        _check_f32(t, nm)
        if t.device != ref.device or t.shape != ref.shape or not t.is_contiguous():
            raise ValueError(f"{nm} must be a contiguous tensor of {tuple(ref.shape)} on {ref.device}")


def normalize_backward(gx, g, y, s, index="literal", stream=None):
    """Gradient of the functional normalize y = normalize(x) (norm_launch_backward):
    gx = ([j in C] ? g / s : g) - sum_{i in C} g_i y_i / s.  s: the forward's 1-element
    divisor tensor.  gx may be g or y.  Returns gx."""
    _check_same([gx, g, y], ["gx", "g", "y"])
    _check_f32(s, "s")
    o = _opts(index, "auto", stream, None, None, device=g.device)
    with _call(g.device):
        _check(lib().norm_launch_backward(gx.data_ptr(), g.data_ptr(), y.data_ptr(), s.data_ptr(), g.numel(),
                                          ctypes.byref(o)))
    return gx


def normalize_rows_backward(gx, g, y, s, index="literal", stream=None):
    """Row-wise normalize_backward of contiguous 2-D tensors (norm_rows_backward); s: the
    forward's per-row divisors (float32[rows])."""
    _check_same([gx, g, y], ["gx", "g", "y"])
    _check_f32(s, "s")
    if g.dim() != 2 or s.numel() != g.shape[0]:
        raise ValueError("2-D g / y / gx and one divisor per row")
    o = _opts(index, "auto", stream, None, None, device=g.device)
    with _call(g.device):
        _check(lib().norm_rows_backward(gx.data_ptr(), g.data_ptr(), y.data_ptr(), s.data_ptr(), g.shape[0],
                                        g.shape[1], g.shape[1], ctypes.byref(o)))
    return gx


def softmax_rows_backward(gx, g, y, log=False, stream=None):
    """Row softmax gradient y (g - sum g y), or log-softmax g - exp(y) sum g, of contiguous
    2-D tensors (norm_softmax_rows_backward).  gx may be g or y.  Returns gx."""
    _check_same([gx, g, y], ["gx", "g", "y"])
    if g.dim() != 2:
        raise ValueError("2-D tensors expected")
    o = _opts("literal", "auto", stream, None, None, device=g.device)
    with _call(g.device):
        _check(lib().norm_softmax_rows_backward(gx.data_ptr(), g.data_ptr(), y.data_ptr(), g.shape[0],
                                                g.shape[1], g.shape[1], 1 if log else 0, ctypes.byref(o)))
    return gx


def normalize_host(out, inp, index="literal", stream=None, sum_out=None, sum_out_f64=None):
    """End-to-end entry on HOST buffers (norm_launch_host): CPU float32 tensors or numpy
    arrays (pin them for overlapped copies).  Enqueued on `stream`; synchronise it
    before reading `out`."""
    import numpy as np

    def hp(a):
        if isinstance(a, np.ndarray):
            assert a.dtype == np.float32 and a.flags["C_CONTIGUOUS"]
            return a.ctypes.data, a.size
        _check_f32(a, "host buffer", cuda=False)
        assert not a.is_cuda and a.is_contiguous()
        return a.data_ptr(), a.numel()

    po, no = hp(out)
    pi, ni = hp(inp)
    if no != ni:
        raise ValueError("size mismatch")
    o = _opts(index, "auto", stream, sum_out, sum_out_f64)
    _check(lib().norm_launch_host(po, pi, ni, ctypes.byref(o)))
    return out


def coverage(n, index="literal"):
    """(|C(n)|, prefix_len or -1) — host-only."""
    c, p = ctypes.c_int64(), ctypes.c_int64()
    _check(lib().norm_coverage(n, _enum(INDEX, index), ctypes.byref(c), ctypes.byref(p)))
    return c.value, p.value


def algorithmic_bytes(n, index="literal"):
    """4n + 8|C(n)|: the roofline numerator of one call — host-only."""
    b = ctypes.c_int64()
    _check(lib().norm_algorithmic_bytes(n, _enum(INDEX, index), ctypes.byref(b)))
    return b.value


def choose_path(n, covered_prefix, path="auto"):
    """The path name a call over n elements with covered set [0, covered_prefix)
    (-1: not a prefix) takes on the current device (norm_choose_path)."""
    c = ctypes.c_int32()
    _check(lib().norm_choose_path(n, covered_prefix, _enum(PATH, path), ctypes.byref(c)))
    return {v: k for k, v in PATH.items()}[c.value]


def workspace_bytes(n=0):
    b = ctypes.c_size_t()
    _check(lib().norm_workspace_bytes(n, None, ctypes.byref(b)))
    return b.value


def plan_shards(n, world, index="literal", coverage_balanced=True):
    """List (per rank) of [(begin, len), ...] global ranges — host-only."""
    plan = (NormShard * world)()
    _check(lib().norm_plan_shards(n, world, _enum(INDEX, index), int(bool(coverage_balanced)), plan))
    return [p.ranges() for p in plan]


def _shard_struct(ranges):
    s = NormShard()
    s.nranges = len(ranges)
    for k, (b, ln) in enumerate(ranges):
        s.begin[k] = b
        s.len[k] = ln
    return s


def normalize_sharded_via(out_local, in_local, ranges, n_global, all_gather, index="literal",
                          stream=None, sum_out=None, sum_out_f64=None, events=None):
    """The sharded path with a caller-supplied exchange (norm_shard_partial ->
    all_gather(partial: 1-element float64 CUDA tensor) -> float64 CUDA tensor of the W
    partials in rank order -> norm_shard_finish).  E.g. torch.distributed over gloo."""
    import torch
    _check_f32(out_local, "out_local")
    _check_f32(in_local, "in_local")
    if in_local.numel() != sum(ln for _, ln in ranges) or out_local.numel() != in_local.numel():
        raise ValueError("local buffers must hold exactly the shard's elements")
    part = torch.empty(1, dtype=torch.float64, device=in_local.device)
    o = _opts(index, "auto", stream, sum_out, sum_out_f64, device=in_local.device)
    with _call(in_local.device, events):
        _check(lib().norm_shard_partial(part.data_ptr(), in_local.data_ptr(), in_local.numel(),
                                        ctypes.byref(o)))
    parts = all_gather(part)
    if parts.dtype != torch.float64 or not parts.is_cuda or not parts.is_contiguous():
        raise ValueError("all_gather must return a contiguous float64 CUDA tensor")
    shard = _shard_struct(ranges)
    with _call(in_local.device):
        _check(lib().norm_shard_finish(out_local.data_ptr(), in_local.data_ptr(), ctypes.byref(shard),
                                       n_global, parts.data_ptr(), parts.numel(), ctypes.byref(o)))
    return out_local


class Comm:
    """NCCL communicator for norm_launch_sharded (one process per GPU).

    The 128-byte NCCL unique id is created on rank 0 and broadcast through the
    torch.distributed process group (any backend)."""

    def __init__(self, group=None, allreduce=False):
        import torch.distributed as dist
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        uid = ctypes.create_string_buffer(128)
        if self.rank == 0:
            _check(lib().norm_comm_unique_id(uid))
        obj = [bytes(uid.raw) if self.rank == 0 else None]
        dist.broadcast_object_list(obj, src=0, group=group)
        uid = ctypes.create_string_buffer(obj[0], 128)
        h = ctypes.c_void_p()
        _check(lib().norm_comm_init(ctypes.byref(h), self.world, self.rank, uid))
        self._h = h
        if allreduce:
            _check(lib().norm_comm_set_mode(self._h, 1))

    def normalize_sharded(self, out_local, in_local, ranges, n_global, index="literal",
                          stream=None, sum_out=None, sum_out_f64=None, events=None):
        _check_f32(out_local, "out_local")
        _check_f32(in_local, "in_local")
        shard = _shard_struct(ranges)
        if in_local.numel() != sum(ln for _, ln in ranges) or out_local.numel() != in_local.numel():
            raise ValueError("local buffers must hold exactly the shard's elements")
        o = _opts(index, "auto", stream, sum_out, sum_out_f64, device=in_local.device)
        with _call(in_local.device, events):
            _check(lib().norm_launch_sharded(self._h, out_local.data_ptr(), in_local.data_ptr(),
                                             ctypes.byref(shard), n_global, ctypes.byref(o)))
        return out_local

    def destroy(self):
        if self._h:
            _check(lib().norm_comm_destroy(self._h))
            self._h = None


class PeerComm:
    """Fused peer-memory exchange (norm_peer_*): the rank partial travels from the
    reduce kernel straight into the peers' mailboxes; no collective is launched.
    The 64-byte CUDA IPC handles are all-gathered through the torch.distributed
    process group (any backend).  Set-up failures are agreed on collectively, so
    either every rank gets a PeerComm or every rank raises (callers can fall
    back consistently)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self._h = None

        def agree(ok, what):
            flags = [None] * self.world
            dist.all_gather_object(flags, (bool(ok), what), group=group)
            bad = [f"rank {r}: {w}" for r, (o, w) in enumerate(flags) if not o]
            if bad:
                if self._h:
                    lib().norm_peer_destroy(self._h)
                    self._h = None
                raise RuntimeError("peer exchange unavailable: " + "; ".join(bad))

        h = ctypes.c_void_p()
        buf = ctypes.create_string_buffer(64)
        st = lib().norm_peer_create(ctypes.byref(h), self.world, self.rank, buf)
        if st == 0:
            self._h = h
        agree(st == 0, "" if st == 0 else f"norm_peer_create: {last_error()}")
        handles = [None] * self.world
        dist.all_gather_object(handles, bytes(buf.raw), group=group)
        allh = ctypes.create_string_buffer(b"".join(handles), 64 * self.world)
        st = lib().norm_peer_connect(self._h, allh)
        agree(st == 0, "" if st == 0 else f"norm_peer_connect: {last_error()}")

    def normalize_sharded(self, out_local, in_local, ranges, n_global, index="literal",
                          stream=None, sum_out=None, sum_out_f64=None, events=None, path="auto"):
        _check_f32(out_local, "out_local")
        _check_f32(in_local, "in_local")
        if in_local.numel() != sum(ln for _, ln in ranges) or out_local.numel() != in_local.numel():
            raise ValueError("local buffers must hold exactly the shard's elements")
        shard = _shard_struct(ranges)
        o = _opts(index, path, stream, sum_out, sum_out_f64, device=in_local.device)
        with _call(in_local.device, events):
            _check(lib().norm_launch_sharded_peer(self._h, out_local.data_ptr(), in_local.data_ptr(),
                                                  ctypes.byref(shard), n_global, ctypes.byref(o)))
        return out_local

    def destroy(self):
        if self._h:
            _check(lib().norm_peer_destroy(self._h))
            self._h = None


# ---------------------------------------------------------------------------
# The C ABI's own names (include/libnorm.h), for callers who think in the C API.
# Each is the same ctypes marshalling as the Pythonic spelling above.

def norm_launch(out, inp):
    """norm_launch(out, in, n): Fig. 1 launch() after LICM (literal index, current stream)."""
    return normalize(out, inp, index="literal")


def norm_launch_ex(out, inp, index="literal", path="auto", stream=None, sum_out=None,
                   sum_out_f64=None, workspace=None, events=None):
    return normalize(out, inp, index, path, stream, sum_out, sum_out_f64, workspace, events)


def norm_launch_host(out_host, in_host, index="literal", stream=None, sum_out=None, sum_out_f64=None):
    return normalize_host(out_host, in_host, index, stream, sum_out, sum_out_f64)


def norm_launch_form(out, inp, form, index="literal", stream=None, sum_out=None, sum_out_f64=None):
    return normalize_form(out, inp, form, index, stream, sum_out, sum_out_f64)


def norm_rows(out, inp, index="literal", stream=None, sum_out=None, sum_out_f64=None):
    return normalize_rows(out, inp, index, stream, sum_out, sum_out_f64)


def norm_softmax_rows(out, inp, kind="softmax", stream=None):
    return softmax_rows(out, inp, log=(kind in ("log_softmax", 1)), stream=stream)


def norm_softmax_rows_backward(gx, g, y, kind="softmax", stream=None):
    return softmax_rows_backward(gx, g, y, log=(kind in ("log_softmax", 1)), stream=stream)


norm_launch_backward = normalize_backward
norm_rows_backward = normalize_rows_backward
norm_graph_create = NormGraph
norm_nll_forward = nll_forward
norm_nll_backward = nll_backward
norm_bpnn_layerforward = bpnn_layerforward
norm_coverage = coverage
norm_algorithmic_bytes = algorithmic_bytes
norm_choose_path = choose_path
norm_workspace_bytes = workspace_bytes
norm_plan_shards = plan_shards
norm_cache_release = cache_release
norm_status_string = status_string
norm_last_error = last_error


def norm_debug_set_events(begin=None, end=None):
    """norm_debug_set_events: (begin, end) torch.cuda.Event pair recorded around the
    dominant kernel of every later call on this thread; (None, None) turns it off."""
    if begin is None or end is None:
        _check(lib().norm_debug_set_events(None, None))
        return
    for ev in (begin, end):
        if not ev.cuda_event:
            ev.record()
    _check(lib().norm_debug_set_events(begin.cuda_event, end.cuda_event))
