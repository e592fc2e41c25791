"""PyTorch operator registration for libnorm.

The paper's MocCUDA runs PyTorch's own CUDA kernels unchanged on a CPU by
interposing on the runtime; the B200-side analogue is to make
libnorm's kernels callable from PyTorch code as ordinary operators, visible to
the dispatcher, autograd-opaque and traceable by torch.compile:

    torch.ops.libnorm.normalize(x, index="dense")       -> Tensor
    torch.ops.libnorm.normalize_rows(x, index="dense")  -> Tensor   (2-D, per row)
    torch.ops.libnorm.normalize_(x, index="literal")    -> None     (in place)
    torch.ops.libnorm.softmax(x, log=False)              -> Tensor   (2-D, per row; NEXT-2)

Functional forms return a fresh tensor whose covered elements are x[i] / s and
whose uncovered elements (literal index, reading R1) are copies of x — i.e. the
in-place semantics of Fig. 1 applied to a copy.  CUDA float32 only; there is no
CPU kernel and no fallback (calls on CPU tensors raise).

Training (the paper runs PyTorch training through its kernels):
`softmax` is differentiable (its backward is norm_softmax_rows_backward), and so
are the divisor-returning forms, whose backward is norm_launch_backward /
norm_rows_backward:

    torch.ops.libnorm.normalize_fwd(x, index)       -> (y, s)    s = the fp32 divisor
    torch.ops.libnorm.normalize_rows_fwd(x, index)  -> (y, s)    s = one divisor per row

`normalize` / `normalize_rows` themselves stay autograd-opaque (they do not keep
the divisor); `Normalize` and `normalize_autograd` use the differentiable forms.

Import this module to register the ops.
"""
import torch

from . import _lib

_INDEXES = ("literal", "dense")


def _check(x, name="x"):
    if x.dtype != torch.float32 or not x.is_cuda:
        raise RuntimeError(f"libnorm ops take CUDA float32 tensors ({name} is {x.dtype} on {x.device})")


@torch.library.custom_op("libnorm::normalize", mutates_args=())
def normalize(x: torch.Tensor, index: str = "dense") -> torch.Tensor:
    _check(x)
    out = x.contiguous().clone()
    _lib.normalize(out, out, index=index)
    return out


@normalize.register_fake
def _(x, index="dense"):
    return torch.empty_like(x, memory_format=torch.contiguous_format)


@torch.library.custom_op("libnorm::normalize_rows", mutates_args=())
def normalize_rows(x: torch.Tensor, index: str = "dense") -> torch.Tensor:
    _check(x)
    if x.dim() != 2:
        raise RuntimeError("libnorm::normalize_rows expects a 2-D tensor")
    out = x.contiguous().clone()
    _lib.normalize_rows(out, out, index=index)
    return out


@normalize_rows.register_fake
def _(x, index="dense"):
    return torch.empty_like(x, memory_format=torch.contiguous_format)


@torch.library.custom_op("libnorm::normalize_", mutates_args=("x",))
def normalize_(x: torch.Tensor, index: str = "literal") -> None:
    _check(x)
    if not x.is_contiguous():
        raise RuntimeError("libnorm::normalize_ needs a contiguous tensor")
    _lib.normalize(x, x, index=index)


@torch.library.custom_op("libnorm::softmax", mutates_args=())
def softmax(x: torch.Tensor, log: bool = False) -> torch.Tensor:
    """Row softmax / log-softmax of a 2-D tensor (norm_softmax_rows): the
    "aggregation operations like Softmax" the paper transpiles."""
    _check(x)
    if x.dim() != 2:
        raise RuntimeError("libnorm::softmax expects a 2-D tensor")
    src = x.contiguous()
    out = torch.empty_like(src)
    _lib.softmax_rows(out, src, log=log)
    return out


@softmax.register_fake
def _(x, log=False):
    return torch.empty_like(x, memory_format=torch.contiguous_format)


# ------------------------------------------------------------------ autograd

@torch.library.custom_op("libnorm::softmax_backward", mutates_args=())
def softmax_backward(g: torch.Tensor, y: torch.Tensor, log: bool = False) -> torch.Tensor:
    """norm_softmax_rows_backward: y (g - sum g y), or g - exp(y) sum g for log-softmax."""
    _check(g, "g")
    _check(y, "y")
    g, y = g.contiguous(), y.contiguous()
    gx = torch.empty_like(y)
    _lib.softmax_rows_backward(gx, g, y, log=log)
    return gx


@softmax_backward.register_fake
def _(g, y, log=False):
    return torch.empty_like(y, memory_format=torch.contiguous_format)


def _softmax_setup(ctx, inputs, output):
    ctx.log = inputs[1] if len(inputs) > 1 else False
    ctx.save_for_backward(output)


def _softmax_bwd(ctx, grad):
    (y,) = ctx.saved_tensors
    return torch.ops.libnorm.softmax_backward(grad, y, ctx.log), None


softmax.register_autograd(_softmax_bwd, setup_context=_softmax_setup)


@torch.library.custom_op("libnorm::normalize_fwd", mutates_args=())
def normalize_fwd(x: torch.Tensor, index: str = "dense") -> tuple[torch.Tensor, torch.Tensor]:
    """normalize (functional form) returning (y, s), s the fp32 divisor used."""
    _check(x)
    out = x.contiguous().clone()
    s = torch.zeros(1, dtype=torch.float32, device=x.device)
    _lib.normalize(out, out, index=index, sum_out=s)
    return out, s


@normalize_fwd.register_fake
def _(x, index="dense"):
    return (torch.empty_like(x, memory_format=torch.contiguous_format),
            x.new_empty(1, dtype=torch.float32))


@torch.library.custom_op("libnorm::normalize_backward", mutates_args=())
def normalize_backward(g: torch.Tensor, y: torch.Tensor, s: torch.Tensor, index: str = "dense") -> torch.Tensor:
    """norm_launch_backward: ([j in C] ? g / s : g) - sum_{i in C} g_i y_i / s."""
    _check(g, "g")
    _check(y, "y")
    g, y = g.contiguous(), y.contiguous()
    gx = torch.empty_like(y)
    _lib.normalize_backward(gx, g, y, s, index=index)
    return gx


@normalize_backward.register_fake
def _(g, y, s, index="dense"):
    return torch.empty_like(y, memory_format=torch.contiguous_format)


def _nfwd_setup(ctx, inputs, output):
    ctx.index = inputs[1] if len(inputs) > 1 else "dense"
    ctx.save_for_backward(*output)


def _nfwd_bwd(ctx, gy, gs):
    y, s = ctx.saved_tensors
    gx = None
    if gy is not None:
        gx = torch.ops.libnorm.normalize_backward(gy, y, s, ctx.index)
    if gs is not None:  # ds/dx_j = 1
        gx = gs.expand_as(y) if gx is None else gx + gs
    return gx, None


normalize_fwd.register_autograd(_nfwd_bwd, setup_context=_nfwd_setup)


@torch.library.custom_op("libnorm::normalize_rows_fwd", mutates_args=())
def normalize_rows_fwd(x: torch.Tensor, index: str = "dense") -> tuple[torch.Tensor, torch.Tensor]:
    """normalize_rows (functional form) returning (y, s), s one fp32 divisor per row."""
    _check(x)
    if x.dim() != 2:
        raise RuntimeError("libnorm::normalize_rows_fwd expects a 2-D tensor")
    out = x.contiguous().clone()
    s = torch.zeros(x.shape[0], dtype=torch.float32, device=x.device)
    _lib.normalize_rows(out, out, index=index, sum_out=s)
    return out, s


@normalize_rows_fwd.register_fake
def _(x, index="dense"):
    return (torch.empty_like(x, memory_format=torch.contiguous_format),
            x.new_empty(x.shape[0], dtype=torch.float32))


@torch.library.custom_op("libnorm::normalize_rows_backward", mutates_args=())
def normalize_rows_backward(g: torch.Tensor, y: torch.Tensor, s: torch.Tensor,
                            index: str = "dense") -> torch.Tensor:
    """norm_rows_backward: normalize_backward of every row with its own divisor."""
    _check(g, "g")
    _check(y, "y")
    g, y = g.contiguous(), y.contiguous()
    gx = torch.empty_like(y)
    _lib.normalize_rows_backward(gx, g, y, s, index=index)
    return gx


@normalize_rows_backward.register_fake
def _(g, y, s, index="dense"):
    return torch.empty_like(y, memory_format=torch.contiguous_format)


def _nrfwd_bwd(ctx, gy, gs):
    y, s = ctx.saved_tensors
    gx = None
    if gy is not None:
        gx = torch.ops.libnorm.normalize_rows_backward(gy, y, s, ctx.index)
    if gs is not None:  # ds_r/dx_rj = 1
        gx = gs[:, None].expand_as(y) if gx is None else gx + gs[:, None]
    return gx, None


normalize_rows_fwd.register_autograd(_nrfwd_bwd, setup_context=_nfwd_setup)


def normalize_autograd(x: torch.Tensor, index: str = "dense") -> torch.Tensor:
    """Differentiable normalize: 1-D -> normalize_fwd, 2-D -> per row (normalize_rows_fwd)."""
    if x.dim() == 1:
        return torch.ops.libnorm.normalize_fwd(x, index)[0]
    return torch.ops.libnorm.normalize_rows_fwd(x, index)[0]


class Normalize(torch.nn.Module):
    """x / x.sum(dim=-1, keepdim=True) over the last dimension (dense index) via libnorm;
    differentiable (backward: norm_launch_backward / norm_rows_backward)."""

    def __init__(self, index: str = "dense"):
        super().__init__()
        assert index in _INDEXES
        self.index = index

    def forward(self, x):
        if x.dim() == 1:
            return torch.ops.libnorm.normalize_fwd(x, self.index)[0]
        shape = x.shape
        return torch.ops.libnorm.normalize_rows_fwd(x.reshape(-1, shape[-1]), self.index)[0].view(shape)
