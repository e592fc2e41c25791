"""Multi-GPU normalize with libnorm: one process per GPU, each holding its shard.

    python -m torch.distributed.run --nproc-per-node 8 --master-addr 127.0.0.1 \
        examples/sharded_normalize.py --numel 4294967296

Every rank generates its own ranges of the global n-element input in HBM (the
coverage-balanced shard plan: a slice of Fig. 1's covered prefix and a slice of
the rest), then one call per rank does the whole step: local reduce, the 8-byte
partial stored straight into every rank's mailbox over NVLink (CUDA IPC peer
memory), rank-order combine, scale of the locally covered elements.  Every rank
ends with the same divisor s, bit for bit.  NORM_EXAMPLE_BACKEND=gloo with
NORM_EXAMPLE_DEVICE=0 runs all ranks on one GPU (the peer mailboxes are then
same-device IPC mappings); with backend nccl the example can also use
libnorm's NCCL exchange (--exchange nccl).
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch
import torch.distributed as dist

import gen
import paper_2207_00257_b200 as L


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--numel", type=int, default=2**28)
    ap.add_argument("--index", default="literal", choices=["literal", "dense"])
    ap.add_argument("--exchange", default="p2p", choices=["p2p", "nccl"])
    args = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    dev = int(os.environ.get("NORM_EXAMPLE_DEVICE", local))
    torch.cuda.set_device(dev)
    dist.init_process_group(os.environ.get("NORM_EXAMPLE_BACKEND", "nccl"))

    n = args.numel
    mine = L.plan_shards(n, world, args.index, True)[rank]  # [(global begin, length), ...]
    nloc = sum(ln for _, ln in mine)
    x = torch.empty(nloc, device="cuda")
    off = 0
    for begin, ln in mine:  # this rank's slices of the global input, generated in place
        gen.fill_cuda(x[off:off + ln], seed=7, dist="unit", offset=begin)
        off += ln
    y = torch.empty_like(x)
    s = torch.zeros(1, device="cuda")

    comm = L.PeerComm() if args.exchange == "p2p" else L.Comm()
    comm.normalize_sharded(y, x, mine, n, index=args.index, sum_out=s)
    torch.cuda.synchronize()

    everyone = [None] * world
    dist.all_gather_object(everyone, s.item())
    if rank == 0:
        same = all(v == everyone[0] for v in everyone)
        print(f"world={world} n={n} index={args.index} exchange={args.exchange}: s={everyone[0]!r} "
              f"identical on every rank: {same}")
    comm.destroy()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
