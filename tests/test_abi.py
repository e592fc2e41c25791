"""C-ABI checks that need no GPU: the library loads, exports every symbol the
header declares, validates arguments before touching CUDA, and its host-only
functions (coverage, byte accounting, shard planner) agree with the oracle."""
import ctypes
import os
import random
import re

import numpy as np
import pytest

import oracle
import paper_2207_00257_b200 as L
from conftest import ROOT

HDR = os.path.join(ROOT, "include", "libnorm.h")


def declared_functions():
    src = open(HDR).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[a-z_]+\s*\*?\s*(norm_[a-z_0-9]+)\s*\(", src, flags=re.M)))


def test_header_symbols_exported():
    names = declared_functions()
    assert len(names) >= 14, names
    lib = L.lib()
    for n in names:
        assert hasattr(lib, n), n


def test_no_internal_symbols_exported():
    out = os.popen(f"nm -D --defined-only {L._lib._SO}").read()
    exported = {l.split()[-1] for l in out.splitlines() if " T " in l}
    ours = {s for s in exported if s.startswith("norm_")}
    assert ours == set(declared_functions())


def test_status_strings():
    for i, name in enumerate(L._lib.STATUS):
        assert L.status_string(i) == name


@pytest.mark.parametrize("mode", ["literal", "dense"])
def test_coverage_matches_oracle(mode):
    ns = list(range(0, 3000)) + [random.Random(2).randrange(1, 1 << 40) for _ in range(300)]
    ns += [2**20 + 7, 2**20 - 1, 2**28, 2**32, 32 * (2**31 - 1)]
    for n in ns:
        assert L.coverage(n, mode) == oracle.coverage_closed(n, mode), (n, mode)


def test_algorithmic_bytes_golden():
    # SURVEY.md §8(d) / BASELINE.md §3 byte table: 4n + 8|C(n)|
    assert L.algorithmic_bytes(1024) == 12288
    assert L.algorithmic_bytes(2**20 + 7) == 4464420
    assert L.algorithmic_bytes(2**28) == 1140858624
    assert L.algorithmic_bytes(2**32) == 18253618944
    assert L.algorithmic_bytes(2**32, "dense") == 51539607552
    assert L.algorithmic_bytes(0) == 0


@pytest.mark.parametrize("mode,balanced", [("literal", True), ("literal", False), ("dense", True)])
@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_plan_shards_partition(mode, balanced, world):
    for n in [0, 1, 7, 100, 993, 1025, 2**20 + 7, 2**28, 2**32, 12345678901]:
        plan = L.plan_shards(n, world, mode, balanced)
        assert len(plan) == world
        ranges = sorted(r for p in plan for r in p)
        pos = 0
        for b, ln in ranges:
            assert b == pos and ln > 0
            pos += ln
        assert pos == n
        for p in plan:
            assert [b for b, _ in p] == sorted(b for b, _ in p) and len(p) <= 2
        if world == 1:
            assert plan[0] == ([(0, n)] if n else [])
        count, prefix = L.coverage(n, mode)
        cov_per_rank = [sum(max(0, min(b + ln, prefix) - b) for b, ln in p) for p in plan] if prefix >= 0 else None
        if cov_per_rank and n > 64 * world:
            if balanced or mode == "dense":
                assert max(cov_per_rank) - min(cov_per_rank) <= 8 + prefix % 8 + 8 * world
            tot = [sum(ln for _, ln in p) for p in plan]
            if not balanced or mode == "dense":
                assert max(tot) - min(tot) <= 8 * world


def test_invalid_arguments_rejected_before_cuda():
    lib = L.lib()
    vp = ctypes.c_void_p
    E = L._lib.STATUS.index
    assert lib.norm_launch(vp(4096), vp(8192), -1) == E("NORM_ERR_INVALID_VALUE")
    assert lib.norm_launch(None, vp(8192), 10) == E("NORM_ERR_INVALID_VALUE")
    assert lib.norm_launch(vp(4098), vp(8192), 10) == E("NORM_ERR_INVALID_VALUE")  # misaligned
    assert lib.norm_launch(vp(4096), vp(4096 + 16), 10) == E("NORM_ERR_OVERLAP")
    assert lib.norm_launch(vp(4096), vp(4096), 0) == E("NORM_OK")  # n == 0: no-op
    assert lib.norm_launch(None, None, 0) == E("NORM_OK")
    o = L._lib.NormOpts()
    o.index = 7
    assert lib.norm_launch_ex(vp(4096), vp(8192), 1, ctypes.byref(o)) == E("NORM_ERR_INVALID_VALUE")
    o.index, o.path = 0, 9
    assert lib.norm_launch_ex(vp(4096), vp(8192), 1, ctypes.byref(o)) == E("NORM_ERR_INVALID_VALUE")
    o.path = 0
    o.flags = 2  # unknown flag bit
    assert lib.norm_launch_ex(vp(4096), vp(8192), 1, ctypes.byref(o)) == E("NORM_ERR_INVALID_VALUE")
    o.flags, o.reserved = 0, 1
    assert lib.norm_launch_ex(vp(4096), vp(8192), 1, ctypes.byref(o)) == E("NORM_ERR_INVALID_VALUE")
    assert lib.norm_shard_partial(vp(4096), vp(8192), 8, ctypes.byref(o)) == E("NORM_ERR_INVALID_VALUE")
    # literal grid beyond gridDim.x: G = ceil(n/32) > 2^31 - 1
    big = 32 * (2**31 - 1) + 1
    assert lib.norm_launch(vp(1 << 44), vp(1 << 46), big) == E("NORM_ERR_UNSUPPORTED")
    # rows
    assert lib.norm_rows(vp(4096), vp(1 << 30), 2, 10, 5, 10, None) == E("NORM_ERR_INVALID_VALUE")
    assert lib.norm_rows(vp(4096), vp(4096 + 40), 4, 10, 10, 10, None) == E("NORM_ERR_OVERLAP")
    assert lib.norm_rows(vp(4096), vp(8192), 0, 10, 10, 10, None) == E("NORM_OK")
    assert "overlap" in L.last_error() or L.last_error() != ""
    # sharded: bad shard
    s = L._lib.NormShard()
    s.nranges = 3
    assert lib.norm_launch_sharded(vp(1), vp(4096), vp(8192), ctypes.byref(s), 10, None) == E("NORM_ERR_INVALID_VALUE")
    assert lib.norm_plan_shards(10, 0, 0, 1, None) == E("NORM_ERR_INVALID_VALUE")


def test_cuda_errors_are_reported_not_raised():
    import torch
    if torch.cuda.is_available():
        pytest.skip("CPU-only check")
    st = L.lib().norm_launch(ctypes.c_void_p(4096), ctypes.c_void_p(1 << 20), 100)
    assert st == L._lib.STATUS.index("NORM_ERR_CUDA")
    assert "cuda" in L.last_error().lower()


def test_python_binding_rejects_cpu_tensors():
    import torch
    x = torch.ones(16)
    with pytest.raises(ValueError):
        L.normalize(x, x)


def test_unique_id_on_host():
    a = ctypes.create_string_buffer(128)
    assert L.lib().norm_comm_unique_id(a) == 0
    assert any(a.raw)


def test_binding_has_c_names():
    # the binding offers every host-callable C entry under its C name (sharded / comm
    # entries live on Comm / PeerComm / normalize_sharded_via)
    skip = {"norm_comm_unique_id", "norm_comm_init", "norm_comm_destroy", "norm_comm_set_mode",
            "norm_launch_sharded", "norm_shard_partial", "norm_shard_finish", "norm_peer_create",
            "norm_peer_connect", "norm_peer_destroy", "norm_launch_sharded_peer",
            "norm_graph_launch", "norm_graph_destroy"}
    for name in declared_functions():
        if name not in skip:
            assert hasattr(L, name), name
    assert L.norm_coverage(2**32) == (134218720, 134218720)


def test_opts_layout_matches_header():
    """norm_opts_t as ctypes sees it == the C struct (offsets of every field)."""
    import subprocess
    import tempfile
    src = r"""
#include <stddef.h>
#include <stdio.h>
#include "libnorm.h"
int main(void) {
  printf("%zu %zu %zu %zu %zu %zu %zu %zu %zu %zu\n", sizeof(norm_opts_t),
         offsetof(norm_opts_t, stream), offsetof(norm_opts_t, index), offsetof(norm_opts_t, path),
         offsetof(norm_opts_t, sum_out), offsetof(norm_opts_t, sum_out_f64),
         offsetof(norm_opts_t, workspace), offsetof(norm_opts_t, workspace_bytes),
         offsetof(norm_opts_t, flags), offsetof(norm_opts_t, reserved));
  return 0;
}
"""
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "o.c")
        with open(c, "w") as f:
            f.write(src)
        exe = os.path.join(d, "o")
        subprocess.run(["gcc", "-std=c11", "-I", os.path.join(ROOT, "include"), c, "-o", exe], check=True)
        got = [int(v) for v in subprocess.run([exe], capture_output=True, text=True, check=True).stdout.split()]
    O = L._lib.NormOpts
    want = [ctypes.sizeof(O)] + [getattr(O, f).offset for f in
                                 ("stream", "index", "path", "sum_out", "sum_out_f64", "workspace",
                                  "workspace_bytes", "flags", "reserved")]
    assert got == want
