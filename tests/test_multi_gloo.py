"""World-size-2 host-side coverage of the sharded path (gloo, CPU).

No GPU here, so the device steps of norm_launch_sharded are emulated per rank
with the oracle (test infrastructure): each rank takes its shard from libnorm's
planner, computes its partial, the partials are all-gathered over gloo exactly
like the 8-byte ncclAllGather, combined in rank order, and the rank's covered
outputs are produced by replay.  Checks: the plan covers [0, n) once, every rank
derives bit-identical s, s is within 1e-6 of the exact sum, and the union of the
local outputs equals the single-process oracle result.  The NCCL unique-id
broadcast used by Comm is exercised over the same process group."""
import ctypes
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, mode, balanced, dist_kind, result_q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import gen
    import oracle
    import paper_2207_00257_b200 as L
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        plan = L.plan_shards(n, world, mode, balanced)
        mine = plan[rank]
        local = np.concatenate([gen.make_host(ln, seed=3, dist=dist_kind, offset=b) for b, ln in mine]) \
            if mine else np.zeros(0, np.float32)
        part = torch.tensor([oracle.sum_exact(local)], dtype=torch.float64)
        parts = [torch.zeros(1, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(parts, part)
        S = 0.0
        for p in parts:  # rank order, as the scale prologue does
            S += float(p[0])
        s = np.float32(S)
        # local covered outputs by replay over the global coverage
        out = []
        off = 0
        for b, ln in mine:
            idx = np.arange(b, b + ln, dtype=np.int64)
            cov = np.array([oracle.is_covered(n, int(i), mode) for i in idx]) if ln < 5000 else \
                (idx < oracle.coverage_closed(n, mode)[1] if oracle.coverage_closed(n, mode)[1] >= 0 else (idx % 32) < oracle.grid_blocks(n))
            seg = local[off:off + ln]
            o = np.where(cov, seg / s, np.float32(np.nan)).astype(np.float32)
            out.append((b, o))
            off += ln
        # Comm's unique-id broadcast path
        uid = ctypes.create_string_buffer(128)
        if rank == 0:
            assert L.lib().norm_comm_unique_id(uid) == 0
        obj = [bytes(uid.raw) if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        result_q.put((rank, float(s), S, out, obj[0]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n,mode,balanced,dist_kind", [
    (2**20 + 7, "literal", True, 0),
    (2**20 + 7, "literal", False, 3),
    (3 * 2**16 + 5, "dense", True, 4),
    (700, "literal", True, 2),   # residue coverage (G < 32)
])
def test_two_rank_sharded_semantics(n, mode, balanced, dist_kind):
    import gen
    import oracle
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n, mode, balanced, dist_kind, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    assert res[0][1] == res[1][1] and res[0][2] == res[1][2]  # bit-identical s on every rank
    assert res[0][4] == res[1][4]                            # same NCCL unique id
    x = gen.make_host(n, seed=3, dist=dist_kind)
    S = oracle.sum_exact(x)
    scale = oracle.sum_abs_exact(x) if dist_kind == 3 else abs(S)
    assert abs(res[0][2] - S) <= 1e-6 * scale
    ref = oracle.normalize(x, mode, out=np.full(n, np.nan, np.float32))
    full = np.full(n, np.nan, np.float32)
    for _, _, _, out, _ in res:
        for b, o in out:
            full[b:b + len(o)] = o
    cov = oracle.covered_mask(n, mode)
    assert np.array_equal(np.isnan(full), ~cov)
    rel = np.abs(full[cov] - ref[cov]) / np.maximum(np.abs(ref[cov]), 1e-30)
    assert rel.max() <= 1e-5
