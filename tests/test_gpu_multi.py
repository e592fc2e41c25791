"""Multi-rank sharded path on ONE GPU: W processes (gloo process group) share
cuda:0 and run the real device kernels of the sharded path — norm_shard_partial
-> all-gather of the 8-byte partials (gloo, in rank order) -> norm_shard_finish.
This is norm_launch_sharded with the ncclAllGather swapped for gloo (NCCL
refuses two ranks on one device).  Checks every rank's outputs against the
oracle, the bit-identical divisor on all ranks, and the 1e-6 bound on s."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, mode, balanced, q, exchange="gather", values="unit"):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import gen
    import paper_2207_00257_b200 as L
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        ranges = L.plan_shards(n, world, mode, balanced)[rank]
        nloc = sum(ln for _, ln in ranges)
        inp = torch.empty(max(nloc, 1), device="cuda")[:nloc]
        off = 0
        for b, ln in ranges:
            gen.fill_cuda(inp[off:off + ln], seed=11, dist=values, offset=b)
            off += ln
        out = torch.full((nloc,), -5.0, device="cuda")
        s = torch.zeros(1, device="cuda")

        def ag(part):
            lst = [torch.zeros(1, dtype=torch.float64) for _ in range(world)]
            dist.all_gather(lst, part.cpu())
            return torch.cat(lst).cuda()

        if exchange == "gather":
            L.normalize_sharded_via(out, inp, ranges, n, ag, index=mode, sum_out=s)
        else:  # fused peer-memory exchange (CUDA IPC mailboxes), several epochs
            pc = L.PeerComm()
            ref = torch.full((nloc,), -5.0, device="cuda")
            sref = torch.zeros(1, device="cuda")
            L.normalize_sharded_via(ref, inp, ranges, n, ag, index=mode, sum_out=sref)
            path = "fused" if exchange.startswith("peer-fused") else ("two_pass" if exchange == "peer-2p" else "auto")
            first = None
            for _ in range(7):
                out.fill_(-5.0)
                pc.normalize_sharded(out, inp, ranges, n, index=mode, sum_out=s, path=path)
                torch.cuda.synchronize()
                if values == "unit":  # grid values: every summation order gives the same bits
                    assert torch.equal(out, ref) and torch.equal(s, sref)
                elif first is None:
                    first = (out.clone(), s.clone())
                else:  # other inputs: the fused partial's order differs from the gathered one,
                    assert torch.equal(out, first[0]) and torch.equal(s, first[1])  # but repeats
            dist.barrier()
            pc.destroy()
        torch.cuda.synchronize()
        q.put((rank, ranges, float(s.item()), out.cpu().numpy(), inp.cpu().numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n,mode,balanced,exchange,values", [
    (2, 2**20 + 7, "literal", True, "gather", "unit"),
    (3, 2**20 + 7, "literal", False, "gather", "unit"),
    (4, 3 * 2**20 + 5, "dense", True, "gather", "unit"),
    (2, 700, "literal", True, "gather", "unit"),
    (2, 2**22 + 7, "literal", True, "peer", "unit"),
    (4, 3 * 2**20 + 5, "dense", True, "peer", "unit"),
    (3, 700, "literal", True, "peer", "unit"),  # ranks without covered elements still wait every epoch
    # one fused kernel per rank (reduce, grid barrier, publish + mailbox wait, scale)
    (2, 2**22 + 7, "literal", True, "peer-fused", "unit"),
    (3, 3 * 2**20 + 5, "dense", True, "peer-fused", "unit"),
    (2, 2**20 + 7, "literal", False, "peer-fused", "unit"),  # one-range plan: rank 1 has nothing covered
    (2, 2**26 + 7, "literal", True, "peer", "unit"),  # AUTO picks fused per rank (local input > L2)
    (2, 2**26 + 7, "literal", True, "peer-2p", "unit"),
    (8, 2**23 + 7, "literal", True, "peer-fused", "unit"),  # the 8-rank mailbox protocol (8 processes, one GPU)
    (8, 2**23 + 7, "literal", True, "peer-2p", "unit"),
    # wide-exponent inputs: s bit-identical on every rank and run, within 1e-6 of the exact sum
    (3, 2**23 + 7, "literal", True, "peer-fused", "wide"),
    (4, 2**22 + 9, "dense", True, "peer-fused", "wide"),
])
def test_sharded_ranks_on_one_gpu(world, n, mode, balanced, exchange, values):
    import gen
    import oracle
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, n, mode, balanced, q, exchange, values))
          for r in range(world)]
    for p in ps:
        p.start()
    res = sorted([q.get(timeout=300) for _ in range(world)], key=lambda t: t[0])
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    svals = {r[2] for r in res}
    assert len(svals) == 1  # bit-identical divisor on every rank
    sv = np.float32(res[0][2])
    x = gen.make_host(n, seed=11, dist=values)
    S = oracle.sum_exact(x)
    assert abs(float(sv) - S) <= 1e-6 * S
    full = np.full(n, -5.0, np.float32)
    for _, ranges, _, out, inp in res:
        off = 0
        for b, ln in ranges:
            assert inp[off:off + ln].tobytes() == x[b:b + ln].tobytes()
            full[b:b + ln] = out[off:off + ln]
            off += ln
    rep = oracle.replay(x, sv, mode, out=np.full(n, -5.0, np.float32))
    assert full.tobytes() == rep.tobytes()
    ref = oracle.normalize(x, mode, out=np.full(n, -5.0, np.float32))
    cov = oracle.covered_mask(n, mode)
    assert np.max(np.abs(full[cov] - ref[cov]) / ref[cov]) <= 1e-5
