"""libnorm — Fig. 1 `normalize` of arxiv 2207.00257 on B200 (sm_100a).

Thin ctypes binding over the C ABI in ``include/libnorm.h`` (argument
marshalling only: every step of the path runs in the CUDA kernels of
``libnorm.so``).  PyTorch supplies device memory, the current stream and the
process group; nothing here computes on the CPU, and there is no fallback:
if ``libnorm.so`` is missing or the device is not sm_100, calls raise.

    out[i] = in[i] / sum(in)   for i in the covered set C(n) of the launch
    normalize<<<(n+31)/32, 32>>> with tid = blockIdx.x + blockDim.x*threadIdx.x
    (PAPER.md:98-119); uncovered outputs are untouched.
"""
from ._lib import (  # noqa: F401
    norm_launch,
    norm_launch_ex,
    norm_launch_host,
    norm_launch_form,
    norm_rows,
    norm_softmax_rows,
    norm_nll_forward,
    norm_nll_backward,
    norm_bpnn_layerforward,
    norm_launch_backward,
    norm_rows_backward,
    norm_softmax_rows_backward,
    norm_coverage,
    norm_algorithmic_bytes,
    norm_choose_path,
    norm_workspace_bytes,
    norm_plan_shards,
    norm_cache_release,
    norm_status_string,
    norm_last_error,
    norm_debug_set_events,
    Comm,
    PeerComm,
    NormError,
    algorithmic_bytes,
    choose_path,
    cache_release,
    coverage,
    last_error,
    lib,
    normalize,
    normalize_form,
    NormGraph,
    BoundNormalize,
    norm_graph_create,
    FORM,
    normalize_host,
    normalize_rows,
    softmax_rows,
    normalize_backward,
    normalize_rows_backward,
    softmax_rows_backward,
    bpnn_layerforward,
    BP_VARIANT,
    nll_forward,
    nll_backward,
    REDUCTION,
    plan_shards,
    normalize_sharded_via,
    status_string,
    workspace_bytes,
    INDEX,
    PATH,
)

__all__ = [
    "normalize", "normalize_form", "NormGraph", "BoundNormalize", "FORM", "normalize_rows", "softmax_rows", "normalize_backward", "normalize_rows_backward", "softmax_rows_backward", "bpnn_layerforward", "BP_VARIANT", "nll_forward", "nll_backward", "REDUCTION", "normalize_host", "coverage", "algorithmic_bytes", "choose_path",
    "cache_release", "plan_shards", "normalize_sharded_via", "workspace_bytes", "Comm", "PeerComm", "NormError", "lib", "status_string",
    "last_error", "INDEX", "PATH",
]
