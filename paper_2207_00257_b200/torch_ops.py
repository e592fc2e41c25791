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


class Normalize(torch.nn.Module):
    """x / x.sum(dim=-1, keepdim=True) over the last dimension (dense index) via libnorm."""

    def __init__(self, index: str = "dense"):
        super().__init__()
        assert index in _INDEXES
        self.index = index

    def forward(self, x):
        if x.dim() == 1:
            return torch.ops.libnorm.normalize(x, self.index)
        shape = x.shape
        return torch.ops.libnorm.normalize_rows(x.reshape(-1, shape[-1]), self.index).view(shape)
