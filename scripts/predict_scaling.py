"""Per-rank cost of the sharded literal n = 2^32 step at W = 1/2/4/8, measured on
ONE B200: each rank's shard (coverage-balanced plan) is run through the real
fused peer-memory path (norm_launch_sharded_peer: reduce kernel that publishes
its partial into the mailbox, scale kernel whose prologue waits on it) with a
world-1 mailbox.  The kernels, grid sizes, PDL edge and mailbox protocol are the
ones a W-GPU run executes; only the NVLink latency of the remote stores is
missing.  Prints, per W, the slowest rank's time and the implied aggregate GB/s
(= algorithmic bytes / slowest rank) against W x the one-GPU figure.

    python scripts/predict_scaling.py [--steps 20] [--index literal]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import torch.distributed as dist

    import gen
    import paper_2207_00257_b200 as L

    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--index", default="literal")
    ap.add_argument("--numel", type=int, default=2**32)
    ap.add_argument("--only", type=int, default=0, help="run this W only (e.g. under ncu)")
    ap.add_argument("--plan", default="balanced", choices=["balanced", "uniform"])
    args = ap.parse_args()
    n = args.numel
    torch.cuda.set_device(0)
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29533")
    dist.init_process_group("gloo", rank=0, world_size=1)
    pc = L.PeerComm()
    stream = torch.cuda.current_stream()
    algo = L.algorithmic_bytes(n, args.index)
    res = {}
    base = None
    for W in ((args.only,) if args.only else (1, 2, 4, 8)):
        plan = L.plan_shards(n, W, args.index, args.plan == "balanced")
        ranks = sorted({0, W // 2, W - 1})
        per = {}
        for k in ranks:
            mine = plan[k]
            nloc = sum(ln for _, ln in mine)
            inp = torch.empty(nloc, dtype=torch.float32, device="cuda")
            off = 0
            for b, ln in mine:
                gen.fill_cuda(inp[off:off + ln], seed=2207, dist="unit", offset=b)
                off += ln
            out = torch.empty_like(inp)
            for _ in range(args.warmup):
                pc.normalize_sharded(out, inp, mine, n, index=args.index)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            a.record(stream)
            for _ in range(args.steps):
                pc.normalize_sharded(out, inp, mine, n, index=args.index)
            b.record(stream)
            torch.cuda.synchronize()
            per[k] = a.elapsed_time(b) / args.steps
            del inp, out
            torch.cuda.empty_cache()
        slow = max(per.values())
        gbs = algo / (slow / 1e3) / 1e9
        if base is None:
            base = gbs / W
        res[W] = {"rank_ms": per, "slowest_ms": slow, "aggregate_gbs": gbs,
                  "vs_W_x_one_gpu": gbs / (W * base)}
        print(f"W={W}: per-rank ms {', '.join(f'r{k}={v:.4f}' for k, v in per.items())}  "
              f"-> {gbs:8.1f} GB/s aggregate, {gbs / (W * base):.3f} of W x one GPU", flush=True)
    pc.destroy()
    print(json.dumps({"index": args.index, "plan": args.plan, "n": n, "steps": args.steps, "results": res}))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
