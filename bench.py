#!/usr/bin/env python
"""bench.py — libnorm throughput on B200 (BASELINE.json metric:
"normalize GB/s and % of HBM peak, n=2^32 fp32, at 1/2/4/8 B200").

One step = one normalize of the whole workload (hoisted global sum over all n
elements, then the scale of the covered elements): two kernels (reduce, scale)
per rank, plus one 8-byte ncclAllGather when N > 1.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload vector|rows|fused28]
                  [--index literal|dense] [--impl libnorm|reference]

For N > 1 launch with torchrun (one process per GPU).  Rank 0 prints ONE JSON line.
value = algorithmic bytes of the whole job (4n + 8|C(n)|) per second
of the max-over-ranks device time.  Inputs (16 GiB at n = 2^32) are far larger than
the 126 MB L2, so no flush is needed between steps (the rows / 2^28 workloads flush).
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAK_FALLBACK_GBS = 6650.0  # /opt/skills/guides/B200_PROFILING.md fallback (earlier pool measurement)
DATASHEET_GBS = 8000.0


def load_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs: torch copy, read+write bytes)"
    except Exception:
        return PEAK_FALLBACK_GBS, "fallback (B200_PROFILING.md)"


def load_traffic(workload, index):
    """dram__bytes_read.sum + dram__bytes_write.sum per reduce launch, from the
    committed ncu --set full summary (profiles/), or None."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return d.get(f"{workload}:{index}")
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled DURING the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index):
        self.dev = device_index
        self.proc = None
        self.path = f"/tmp/libnorm_clocks_{os.getpid()}.csv"

    def __enter__(self):
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=self.f, stderr=subprocess.DEVNULL)
            time.sleep(0.3)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.2)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.f.close()

    def summary(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


class L2Flush:
    """Between timed steps: write a 256 MiB buffer (> the 126 MB L2, the timing
    rule), then read a second 256 MiB buffer so the dirty lines of the write are
    written back to HBM here, outside the timed region, instead of during the
    next timed kernel (measured: ~18 us of foreign write-back otherwise at 2^28)."""

    def __init__(self):
        import torch
        self.w = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
        self.r = torch.ones(64 << 20, dtype=torch.float32, device="cuda")

    def __call__(self):
        self.w.zero_()
        self.r.sum()


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def oracle_sample(index, n_sample=2**28, reps=10):
    """Time the CPU oracle (form 3, hoisted O(N)) as it stands, single-threaded,
    on a bounded sample of the same workload; returns GB/s of algorithmic bytes."""
    import gen
    import oracle
    import paper_2207_00257_b200 as L
    x = gen.make_host(n_sample, seed=2207, dist="unit")
    out = x.copy()
    times = []
    for _ in range(reps):
        t0 = time.perf_counter()
        oracle.form_hoisted(x, index, out=out)
        times.append(time.perf_counter() - t0)
    t = statistics.median(times)
    b = L.algorithmic_bytes(n_sample, index)
    return {"value": b / t / 1e9, "unit": "GB/s", "cores": 1, "kind": "oracle",
            "sample": f"oracle form 3 (hoisted sum + scale, fp64 exact sum), n={n_sample} "
                      f"{index} index, median of {reps}, {t:.3f} s each, 1 thread of "
                      f"{os.cpu_count()} ({cpu_model()})"}


# --------------------------------------------------------------------------- arms

def _wait_for_cuda(timeout_s=90):
    """A freshly handed-over box can briefly refuse CUDA initialisation, and the
    CUDA runtime caches that failure per process: probe in subprocesses first."""
    probe = [sys.executable, "-c", "import torch, sys; sys.exit(0 if torch.cuda.is_available() else 1)"]
    deadline = time.time() + timeout_s
    while time.time() < deadline:
        if subprocess.run(probe, capture_output=True).returncode == 0:
            return
        time.sleep(5)


def dist_setup(args):
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        if world == 1 and args.gpus > 1:
            raise SystemExit("--gpus N > 1 needs torchrun (one process per GPU)")
    if world > 1:
        backend = os.environ.get("NORM_BENCH_BACKEND", "nccl")  # gloo: harness tests on one GPU
        dev = local if backend == "nccl" else int(os.environ.get("NORM_BENCH_DEVICE", local))
        torch.cuda.set_device(dev)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group(backend)
    else:
        torch.cuda.set_device(0)
    return world, rank, local


def _dev():
    import torch.distributed as dist
    return "cuda" if dist.get_backend() == "nccl" else "cpu"


def max_over_ranks(v, world):
    import torch
    import torch.distributed as dist
    if world == 1:
        return v
    t = torch.tensor([v], dtype=torch.float64, device=_dev())
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def host_all_gather(world):
    """All-gather of the 8-byte partial over the default process group (used by
    --exchange host: norm_shard_partial -> this -> norm_shard_finish)."""
    import torch
    import torch.distributed as dist

    def ag(part):
        if _dev() == "cuda":
            out = torch.empty(world, dtype=torch.float64, device="cuda")
            dist.all_gather_into_tensor(out, part)
            return out
        lst = [torch.zeros(1, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(lst, part.cpu())
        return torch.cat(lst).cuda()
    return ag


def barrier(world):
    import torch
    import torch.distributed as dist
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()



def workload_name(n, index):
    """The workload key shared by both arms' JSON lines."""
    e = n.bit_length() - 1
    size = f"2^{e}" if n == 1 << e else str(n)
    return f"normalize n={size} fp32 (Fig. 1), {index} index"


def run_reference(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    n_sample = 2**26
    steps = []
    import gen
    import oracle
    import paper_2207_00257_b200 as L
    x = gen.make_host(n_sample, seed=2207, dist="unit")
    out = x.copy()
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        oracle.form_hoisted(x, args.index, out=out)
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            steps.append(dt)
    ms = 1e3 * sum(steps) / len(steps)
    b = L.algorithmic_bytes(n_sample, args.index)
    v = b / (ms / 1e3) / 1e9
    line = {
        "impl": "reference", "metric": "normalize GB/s and % of HBM peak, n=2^32 fp32, at 1/2/4/8 B200",
        "value": v, "unit": "GB/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload_name(args.n, args.index),
                   "sample": f"CPU oracle (form 3, hoisted) on a bounded sample: n={n_sample} per step; "
                             f"value = the sample's algorithmic bytes / its time",
                   "n": args.n, "sample_n": n_sample, "index": args.index},
        "cpu_baseline": {"value": v, "unit": "GB/s", "cores": 1, "kind": "oracle",
                         "sample": f"n={n_sample} per step, 1 thread of {os.cpu_count()} ({cpu_model()})"},
        "e2e": {"value": v, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_vector(args, world, rank, local):
    import torch
    import gen
    import paper_2207_00257_b200 as L

    n = args.n
    index = args.index
    plan = L.plan_shards(n, world, index, args.plan == "balanced")
    mine = plan[rank]
    nloc = sum(ln for _, ln in mine)
    inp = torch.empty(max(nloc, 1), dtype=torch.float32, device="cuda")[:nloc]
    off = 0
    for b, ln in mine:  # each rank generates its own global ranges in HBM
        gen.fill_cuda(inp[off:off + ln], seed=2207, dist="unit", offset=b)
        off += ln
    out = torch.empty_like(inp)
    torch.cuda.synchronize()
    comm = None
    exchange_note = None
    if world > 1 and args.exchange == "p2p":
        # the fused peer-memory exchange, cross-checked once against the gathered
        # partials (same kernels, exchange over the process group); any failure or
        # mismatch falls back to NCCL and is recorded in the JSON line
        try:
            comm = L.PeerComm()
            s_p = torch.zeros(1, device="cuda")
            s_g = torch.zeros(1, device="cuda")
            comm.normalize_sharded(out, inp, mine, n, index=index, sum_out=s_p)
            L.normalize_sharded_via(out, inp, mine, n, host_all_gather(world), index=index, sum_out=s_g)
            torch.cuda.synchronize()
            ok = torch.tensor([1.0 if torch.equal(s_p, s_g) else 0.0], device=_dev() if _dev() == "cuda" else "cpu")
            import torch.distributed as dist
            dist.all_reduce(ok, op=dist.ReduceOp.MIN)
            if ok.item() != 1.0:
                raise RuntimeError("p2p divisor != gathered divisor")
        except Exception as e:  # noqa: BLE001
            exchange_note = f"p2p unavailable ({e}); fell back to nccl"
            print(f"[bench] {exchange_note}", file=sys.stderr)
            comm = None
            args.exchange = "nccl"
    if world > 1 and args.exchange in ("nccl", "nccl-allreduce") and comm is None:
        comm = L.Comm(allreduce=args.exchange == "nccl-allreduce")
    ag = host_all_gather(world) if world > 1 and args.exchange == "host" else None
    stream = torch.cuda.current_stream()

    def step(ev=None):
        if world == 1:
            L.normalize(out, inp, index=index, path=args.path, events=ev)
        elif comm is not None:
            comm.normalize_sharded(out, inp, mine, n, index=index, events=ev)
        else:
            L.normalize_sharded_via(out, inp, mine, n, ag, index=index, events=ev)

    for _ in range(args.warmup):
        step()
    # Timed region: K whole steps, bracketed by barrier + sync.  The reduce
    # kernel's own duration is taken in a second, instrumented pass (events
    # recorded by libnorm around the reduce launch, on the launch stream),
    # because an event between the two kernels disables their programmatic
    # dependent launch and would perturb the step being timed.
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier(world)
    with ClockSampler(local) as clk:
        t0.record(stream)
        for k in range(args.steps):
            step()
        t1.record(stream)
        torch.cuda.synchronize()
    barrier(world)
    ms_local = t0.elapsed_time(t1) / args.steps
    ms = max_over_ranks(ms_local, world)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    i0, i1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier(world)
    i0.record(stream)
    for k in range(args.steps):
        step(evs[k])
    i1.record(stream)
    torch.cuda.synchronize()
    barrier(world)
    ms_instr = i0.elapsed_time(i1) / args.steps
    red_ms = [b.elapsed_time(e) for b, e in evs]
    red_ms_avg = sum(red_ms) / len(red_ms)
    algo = L.algorithmic_bytes(n, index)
    value = algo / (ms / 1e3) / 1e9
    peak, peak_src = load_peak()
    # the kernel the events bracket: the reduce (two-pass: 4 bytes per owned
    # element) or, when this rank's call is one fused kernel, that kernel
    # (4 bytes per owned element + 8 per locally covered element)
    cov_count_g, prefix_g = L.coverage(n, index)
    lloc = local_covered_prefix(mine, prefix_g)
    if world == 1:
        kpath = L.choose_path(n, prefix_g, args.path)
    elif comm is not None and isinstance(comm, L.PeerComm):
        kpath = L.choose_path(nloc, lloc, "auto")
    else:
        kpath = "two_pass"
    fused_step = kpath == "fused"
    red_bytes = 4 * nloc + (8 * lloc if fused_step else 0)
    # in-run calibration on the same buffers: a torch copy stream
    # (read + write bytes) and a torch read-only stream (torch.sum)
    calib = {}
    if nloc >= (1 << 24):
        def _t(fn, reps=5):
            fn()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            for _ in range(reps):
                fn()
            b.record(stream)
            torch.cuda.synchronize()
            return a.elapsed_time(b) / reps
        cms = _t(lambda: out.copy_(inp))
        rms = _t(lambda: torch.sum(inp))
        calib = {"torch_copy_gbs": 8 * nloc / (cms / 1e3) / 1e9, "torch_sum_gbs": 4 * nloc / (rms / 1e3) / 1e9,
                 "note": "same-run torch streams on this rank's buffers (copy counts read+write bytes)"}
    achieved = red_bytes / (red_ms_avg / 1e3) / 1e9
    extra = {}
    # per-step distribution (events between steps; PDL acts inside a step, so
    # these do not perturb it) and, at N = 1, the same step replayed as a CUDA
    # graph (norm_graph_create: reduce + scale captured with their PDL edge)
    sev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    barrier(world)
    sev[0].record(stream)
    for k in range(args.steps):
        step()
        sev[k + 1].record(stream)
    torch.cuda.synchronize()
    barrier(world)
    per = sorted(sev[k].elapsed_time(sev[k + 1]) for k in range(args.steps))
    stats = {"median_ms": max_over_ranks(statistics.median(per), world),
             "min_ms": max_over_ranks(per[0], world),
             "p90_ms": max_over_ranks(per[min(len(per) - 1, int(0.9 * len(per)))], world)}
    if world == 1:
        g = L.NormGraph(out, inp, index=index, path=args.path)
        for _ in range(2):
            g.launch()
        barrier(world)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(args.steps):
            g.launch()
        b.record(stream)
        torch.cuda.synchronize()
        gms = a.elapsed_time(b) / args.steps
        stats["graph_ms_per_step"] = gms
        stats["graph_value"] = L.algorithmic_bytes(n, index) / (gms / 1e3) / 1e9
        g.destroy()
    extra["step_stats"] = stats
    # dense-index figure on the same buffers (caption reading R1), reported beside the headline
    if args.also_dense and index == "literal" and (world == 1 or comm is not None):
        dense_mine = L.plan_shards(n, world, "dense", True)[rank]
        if dense_mine == mine or world == 1:
            for _ in range(2):
                L.normalize(out, inp, index="dense", path="auto") if comm is None else \
                    comm.normalize_sharded(out, inp, mine, n, index="dense")
            barrier(world)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            for _ in range(args.steps):
                L.normalize(out, inp, index="dense", path="auto") if comm is None else \
                    comm.normalize_sharded(out, inp, mine, n, index="dense")
            b.record(stream)
            torch.cuda.synchronize()
            dms = max_over_ranks(a.elapsed_time(b) / args.steps, world)
            dbytes = L.algorithmic_bytes(n, "dense")
            extra["dense_index"] = {"value": dbytes / (dms / 1e3) / 1e9, "unit": "GB/s", "ms_per_step": dms,
                                    "frac_of_peak": dbytes / (dms / 1e3) / 1e9 / (world * peak)}
    # e2e: same metric through the public API with host buffers, copies inside the timed region
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, world, rank, local, mine, n, index)
    launches_per_step = 1 if fused_step else 2
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = oracle_sample(index)
    if rank != 0:
        return
    cov_count, prefix = L.coverage(n, index)
    line = {
        "metric": "normalize GB/s and % of HBM peak, n=2^32 fp32, at 1/2/4/8 B200",
        "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f32", "data": "synthetic",
        "config": {"workload": workload_name(n, index),
                   "path": kpath + (" per rank" if world > 1 else ""),
                   "exchange_desc": ("8 B per rank: " + {
                       "nccl": "ncclAllGather", "nccl-allreduce": "ncclAllReduce",
                       "p2p": "peer-memory stores into every rank's mailbox from the reduce / fused kernel",
                       "host": "all-gather over the torch.distributed group"}[args.exchange]) if world > 1 else None,
                   "n": n, "index": index, "covered": cov_count, "algorithmic_bytes": algo,
                   "parallelism": f"shard{world}", "exchange": args.exchange if world > 1 else None,
                   "shard_plan": (("coverage-balanced two-range" if args.plan == "balanced" else "uniform one-range")
                                  if world > 1 else None),
                   "exchange_note": exchange_note, "inputs": "seeded synthetic D0 unit grid (gen/), generated in HBM",
                   "l2": f"no flush: {4 * nloc / 2**30:.1f} GiB input per GPU >> 126 MB L2"},
        "frac_of_hbm_peak": value / (world * peak),
        "frac_of_datasheet": value / (world * DATASHEET_GBS),
        "calibration": calib,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak,
                     "traffic": load_traffic("vector", index) if (world == 1 and n == 2**32) else None,
                     "kernel": ("fused_kernel (reduce + grid barrier + exchange + scale: the whole step)"
                                if fused_step else
                                ("reduce_dyn_kernel (TMA-bulk reduce, dynamic deterministic tail)"
                                 if nloc >= (1 << 22) else "reduce_kernel")
                                + " (the hoisted sum: 94% of the literal step's bytes)"),
                     "algorithmic_bytes_per_launch": red_bytes, "avg_launch_ms": red_ms_avg,
                     "share_of_step": red_ms_avg / ms_instr, "instrumented_ms_per_step": ms_instr,
                     "frac_of_same_run_read_stream": (achieved / calib["torch_sum_gbs"]) if calib else None,
                     "peak_source": peak_src},
        "gpu_launches": launches_per_step * args.steps,
        "clocks": clk.summary(),
    }
    line.update(extra)
    if e2e:
        line["e2e"] = e2e
    if cpu:
        line["cpu_baseline"] = cpu
    print(json.dumps(line), flush=True)
    if comm:
        comm.destroy()


def local_covered_prefix(ranges, prefix):
    """Locally covered elements as a prefix [0, Lloc) of the local buffer, else -1
    (mirrors comm.cpp local_covered_prefix; prefix = global L, -1 if not a prefix)."""
    if prefix < 0:
        return -1
    off = lloc = 0
    ended = False
    for b, ln in ranges:
        clen = max(0, min(b + ln, prefix) - b)
        if clen > 0:
            if ended or off != lloc:
                return -1
            lloc += clen
        if clen < ln:
            ended = True
        off += ln
    return lloc


def run_e2e(args, world, rank, local, mine, n, index):
    """Host buffers in pinned memory; every step copies its input H2D and its
    covered output D2H inside the timed region."""
    import torch
    import gen
    import paper_2207_00257_b200 as L
    nloc = sum(ln for _, ln in mine)
    host_in = torch.empty(nloc, dtype=torch.float32, pin_memory=True)
    # fill from a device-generated copy (fast), then free it
    off = 0
    for b, ln in mine:
        t = torch.empty(ln, dtype=torch.float32, device="cuda")
        gen.fill_cuda(t, seed=2207, dist="unit", offset=b)
        host_in[off:off + ln].copy_(t)
        del t
        off += ln
    cov_local = 0
    count, prefix = L.coverage(n, index)
    for b, ln in mine:
        cov_local += max(0, min(b + ln, prefix) - b) if prefix >= 0 else 0
    host_out = torch.empty(nloc, dtype=torch.float32, pin_memory=True)
    steps = max(1, min(args.steps, args.e2e_steps))
    stream = torch.cuda.current_stream()
    comm = None
    if world > 1:
        comm = {"nccl": L.Comm, "p2p": L.PeerComm,
                "nccl-allreduce": lambda: L.Comm(allreduce=True)}.get(args.exchange, lambda: None)()
        ag = host_all_gather(world)
        din = torch.empty(nloc, dtype=torch.float32, device="cuda")
        dout = torch.empty_like(din)

    def step():
        if world == 1:
            L.normalize_host(host_out, host_in, index=index)
        else:
            din.copy_(host_in, non_blocking=True)
            if comm is not None:
                comm.normalize_sharded(dout, din, mine, n, index=index)
            else:
                L.normalize_sharded_via(dout, din, mine, n, ag, index=index)
            o = 0
            for b, ln in mine:
                c = max(0, min(b + ln, prefix) - b)
                if c:
                    host_out[o:o + c].copy_(dout[o:o + c], non_blocking=True)
                o += ln

    step()
    torch.cuda.synchronize()
    barrier(world)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(steps):
        step()
    b.record(stream)
    torch.cuda.synchronize()
    ms = max_over_ranks(a.elapsed_time(b) / steps, world)
    if comm:
        comm.destroy()
    # the link this number is bound by: a plain pinned H2D copy of 1 GiB pieces of
    # the same host buffer (the e2e step moves 4n bytes host -> device)
    piece = min(nloc, 1 << 28)
    dbuf = torch.empty(piece, dtype=torch.float32, device="cuda")
    dbuf.copy_(host_in[:piece], non_blocking=True)
    k = max(1, min(4, nloc // piece))
    a.record(stream)
    for j in range(k):
        dbuf.copy_(host_in[j * piece:(j + 1) * piece], non_blocking=True)
    b.record(stream)
    torch.cuda.synchronize()
    h2d_gbs = 4 * piece * k / (a.elapsed_time(b) / 1e3) / 1e9
    del dbuf
    algo = L.algorithmic_bytes(n, index)
    h2d = 4 * n
    d2h = 4 * count
    step_h2d_gbs = h2d / world / (ms / 1e3) / 1e9
    return {"value": algo / (ms / 1e3) / 1e9, "unit": "GB/s", "ms_per_step": ms, "steps": steps,
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "pcie_h2d_gbs": h2d_gbs, "step_h2d_gbs": step_h2d_gbs,
            "frac_of_pcie_h2d": step_h2d_gbs / h2d_gbs,
            "api": "norm_launch_host (pinned host buffers, chunked H2D overlapped with the reduce)"
            if world == 1 else ("H2D + norm_launch_sharded + D2H of covered elements" if comm else
                                "H2D + norm_shard_partial/all-gather/norm_shard_finish + D2H of covered elements")}


def run_rows(args, world, rank, local):
    import torch
    import gen
    import paper_2207_00257_b200 as L
    R, C = 65536, 4096
    r0, r1 = R * rank // world, R * (rank + 1) // world
    rl = r1 - r0
    inp = torch.empty(rl * C, dtype=torch.float32, device="cuda")
    gen.fill_cuda(inp, seed=2207, dist="unit", offset=r0 * C)
    inp = inp.view(rl, C)
    out = torch.empty_like(inp)
    flush = L2Flush()
    stream = torch.cuda.current_stream()
    for _ in range(args.warmup):
        L.normalize_rows(out, inp, index=args.index)
    times = []
    barrier(world)
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            L.normalize_rows(out, inp, index=args.index)
            b.record(stream)
            torch.cuda.synchronize()
            times.append(a.elapsed_time(b))
    barrier(world)
    ms = max_over_ranks(sum(times) / len(times), world)
    cov, _ = L.coverage(C, args.index)
    algo = R * (4 * C + 4 * cov)  # single pass: read each row once, write its covered part
    value = algo / (ms / 1e3) / 1e9
    peak, src = load_peak()
    if rank != 0:
        return
    line = {
        "metric": "normalize GB/s and % of HBM peak (batched rows 65536x4096 fp32)",
        "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"norm_rows 65536x4096 fp32, {args.index} index, rows sharded",
                   "rows": R, "cols": C, "index": args.index, "algorithmic_bytes": algo,
                   "l2": "flushed before every step (256 MiB write, then a 256 MiB read so the write-back happens outside the timed region)"},
        "frac_of_hbm_peak": value / (world * peak),
        "roofline": {"bound": "hbm", "achieved": value / world, "peak": peak, "unit": "GB/s",
                     "frac": value / world / peak, "traffic": load_traffic("rows", args.index),
                     "kernel": "rows_kernel (single kernel per step)", "peak_source": src},
        "gpu_launches": args.steps,
        "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)


def run_paths28(args, world, rank, local):
    """BASELINE configs[2]: n = 2^28 on one GPU, HBM-bound two-pass vs L2-fused single pass."""
    import torch
    import gen
    import paper_2207_00257_b200 as L
    n = 2**28
    inp = torch.empty(n, dtype=torch.float32, device="cuda")
    gen.fill_cuda(inp, seed=2207, dist="unit")
    out = torch.empty_like(inp)
    flush = L2Flush()
    stream = torch.cuda.current_stream()
    res = {}
    peak, src = load_peak()
    for path in ("two_pass", "fused"):
        for _ in range(args.warmup):
            L.normalize(out, inp, index=args.index, path=path)
        times = []
        for _ in range(args.steps):
            flush()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            L.normalize(out, inp, index=args.index, path=path)
            b.record(stream)
            torch.cuda.synchronize()
            times.append(a.elapsed_time(b))
        ms = sum(times) / len(times)
        algo = L.algorithmic_bytes(n, args.index)
        res[path] = {"ms_per_step": ms, "value": algo / (ms / 1e3) / 1e9, "frac": algo / (ms / 1e3) / 1e9 / peak}
    best = max(res, key=lambda k: res[k]["value"])
    line = {"metric": "normalize GB/s and % of HBM peak (n=2^28, two-pass vs fused)",
            "value": res[best]["value"], "unit": "GB/s", "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": res[best]["ms_per_step"], "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": f"normalize n=2^28 fp32, {args.index}, best path = {best}",
                       "l2": "flushed before every step (256 MiB write, then a 256 MiB read so the write-back happens outside the timed region)"},
            "paths": res, "peak": peak, "gpu_launches": args.steps}
    if rank == 0:
        print(json.dumps(line), flush=True)


def run_softmax(args, world, rank, local):
    """row softmax over the rows config (65536 x 4096 fp32)."""
    import torch
    import gen
    import paper_2207_00257_b200 as L
    R, C = 65536, 4096
    inp = torch.empty(R * C, dtype=torch.float32, device="cuda")
    gen.fill_cuda(inp, seed=2207, dist="signed")
    inp = inp.view(R, C)
    out = torch.empty_like(inp)
    flush = L2Flush()
    stream = torch.cuda.current_stream()
    res = {}
    peak, src = load_peak()
    for log in (False, True):
        for _ in range(args.warmup):
            L.softmax_rows(out, inp, log=log)
        times = []
        for _ in range(args.steps):
            flush()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            L.softmax_rows(out, inp, log=log)
            b.record(stream)
            torch.cuda.synchronize()
            times.append(a.elapsed_time(b))
        ms = sum(times) / len(times)
        v = 8 * R * C / (ms / 1e3) / 1e9
        res["log_softmax" if log else "softmax"] = {"ms_per_step": ms, "value": v, "frac": v / peak}
        # torch's own kernel on the same data, for context
        times = []
        for _ in range(args.steps):
            flush()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            y = (torch.log_softmax if log else torch.softmax)(inp, dim=1)
            b.record(stream)
            torch.cuda.synchronize()
            times.append(a.elapsed_time(b))
        tms = sum(times) / len(times)
        res[("log_softmax" if log else "softmax") + "_torch"] = {"ms_per_step": tms,
                                                                 "value": 8 * R * C / (tms / 1e3) / 1e9}
    # ClassNLLCriterion on the same shape (log-probs = log_softmax output)
    L.softmax_rows(out, inp, log=True)
    tgt = torch.empty(R, dtype=torch.float32, device="cuda")
    gen.fill_cuda(tgt, seed=5, dist="unit")
    tgt = (tgt * C).long()
    grad = torch.empty_like(out)
    g1 = torch.ones(1, device="cuda")
    for _ in range(args.warmup):
        loss, tw = L.nll_forward(out, tgt)
        L.nll_backward(g1, (R, C), tgt, tw, grad=grad)
    for name in ("nll_forward", "nll_backward"):
        times = []
        for _ in range(args.steps):
            flush()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            if name == "nll_forward":
                loss, tw = L.nll_forward(out, tgt)
            else:
                L.nll_backward(g1, (R, C), tgt, tw, grad=grad)
            b.record(stream)
            torch.cuda.synchronize()
            times.append(a.elapsed_time(b))
        ms = sum(times) / len(times)
        nbytes = R * (8 + 4) if name == "nll_forward" else 4 * R * C  # gathered reads / dense write
        res[name] = {"ms_per_step": ms, "value": nbytes / (ms / 1e3) / 1e9, "bytes": nbytes}
    line = {"metric": "row softmax GB/s and % of HBM peak (65536x4096 fp32)",
            "value": res["softmax"]["value"], "unit": "GB/s", "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": res["softmax"]["ms_per_step"], "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": "norm_softmax_rows 65536x4096 fp32 (D3 signed logits)",
                       "l2": "flushed before every step (256 MiB write, then a 256 MiB read so the write-back happens outside the timed region)"},
            "frac_of_hbm_peak": res["softmax"]["frac"], "peak": peak, "results": res,
            "gpu_launches": args.steps}
    if rank == 0:
        print(json.dumps(line), flush=True)


def run_backprop(args, world, rank, local):
    """Rodinia bpnn_layerforward (Fig. backprop) as printed vs
    with the paper's barrier elimination + mem2reg vs the register (0-barrier) form."""
    import torch
    import gen
    import paper_2207_00257_b200 as L
    n_in = 2**22
    x = torch.empty(n_in + 1, device="cuda")
    gen.fill_cuda(x, seed=1, dist="unit")
    w0 = torch.empty((n_in + 1) * 17, device="cuda")
    gen.fill_cuda(w0, seed=2, dist="unit")
    w0 = w0.view(n_in + 1, 17)
    h = w0.clone()
    o = torch.empty(n_in, device="cuda")
    flush = L2Flush()
    stream = torch.cuda.current_stream()
    nbytes = (16 * n_in * 4) * 2 + n_in * 4 * 2  # hidden read + write, input read, output write
    res = {}
    for v in ("printed", "eliminated", "register", "tma"):
        for _ in range(args.warmup):
            L.bpnn_layerforward(x, h, o, variant=v)
        times = []
        for _ in range(args.steps):
            flush()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            L.bpnn_layerforward(x, h, o, variant=v)
            b.record(stream)
            torch.cuda.synchronize()
            times.append(a.elapsed_time(b))
        ms = sum(times) / len(times)
        res[v] = {"ms_per_step": ms, "value": nbytes / (ms / 1e3) / 1e9}
    peak, _ = load_peak()
    line = {"metric": "bpnn_layerforward GB/s (Rodinia backprop, Fig. backprop), in=2^22, hid=16",
            "value": res["tma"]["value"], "unit": "GB/s", "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": res["tma"]["ms_per_step"],
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic", "config": {"workload": "norm_bpnn_layerforward in=2^22 hid=16",
                                            "l2": "flushed before every step (256 MiB write, then a 256 MiB read so the write-back happens outside the timed region)"},
            "variants": res, "frac_of_hbm_peak": res["tma"]["value"] / peak,
            "speedup_eliminated_over_printed": res["printed"]["ms_per_step"] / res["eliminated"]["ms_per_step"],
            "speedup_register_over_printed": res["printed"]["ms_per_step"] / res["register"]["ms_per_step"],
            "speedup_tma_over_printed": res["printed"]["ms_per_step"] / res["tma"]["ms_per_step"],
            "gpu_launches": args.steps * len(res)}
    if rank == 0:
        print(json.dumps(line), flush=True)


def run_licm(args, world, rank, local):
    """Fig. 1 before/after parallel LICM on the GPU — the
    printed per-thread O(N^2) kernel, the per-block O(N^2/B) variant and the
    hoisted O(N) path, timed at small n."""
    import torch
    import gen
    import paper_2207_00257_b200 as L
    stream = torch.cuda.current_stream()
    res = []
    launches = 0
    for e in (10, 12, 14, 16, 18):
        n = 2**e
        inp = torch.empty(n, dtype=torch.float32, device="cuda")
        gen.fill_cuda(inp, seed=2207, dist="unit")
        out = torch.empty_like(inp)
        row = {"n": n}
        for form in ("per_thread", "per_block", "hoisted"):
            if form == "per_thread" and e > 16:
                continue
            for _ in range(2):
                L.normalize_form(out, inp, form=form, index=args.index)
            reps = 5 if form != "hoisted" else 50
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            for _ in range(reps):
                L.normalize_form(out, inp, form=form, index=args.index)
            b.record(stream)
            torch.cuda.synchronize()
            row[form + "_ms"] = a.elapsed_time(b) / reps
            # the un-hoisted forms are one kernel; hoisted: one (small path) or reduce + scale
            launches += reps * (2 if form == "hoisted" and n > 2**17 else 1)
        if "per_thread_ms" in row:
            row["per_thread_over_hoisted"] = row["per_thread_ms"] / row["hoisted_ms"]
        row["per_block_over_hoisted"] = row["per_block_ms"] / row["hoisted_ms"]
        res.append(row)
    last = res[-1]
    # cpu_baseline leg of this workload: the oracle's three forms of Fig. 1 at
    # BASELINE configs[0] (n = 1024, grid 32 x 32), with their exact add counts
    cpu = None
    if rank == 0 and not args.no_cpu:
        import oracle
        x = gen.make_host(1024, seed=2207, dist="unit")
        forms = {}
        for name, fn in (("per_thread", oracle.form_thread), ("per_block", oracle.form_block),
                         ("hoisted", oracle.form_hoisted)):
            reps = 3
            t0 = time.perf_counter()
            for _ in range(reps):
                _, adds = fn(x, args.index)
            forms[name] = {"ms": (time.perf_counter() - t0) / reps * 1e3, "adds": adds}
        cpu = {"value": forms["per_thread"]["ms"] / forms["hoisted"]["ms"], "unit": "x (per-thread / hoisted, oracle, n=1024)",
               "cores": 1, "kind": "oracle",
               "sample": f"oracle forms of Fig. 1 at n=1024 ({args.index} index), 3 reps each, 1 thread of "
                         f"{os.cpu_count()} ({cpu_model()}); adds = 32*G*n, G*n, n",
               "forms": forms}
    line = {"metric": "Fig. 1 before/after parallel LICM on B200 (ms per call)",
            "value": last["per_block_over_hoisted"], "unit": "x (per-block / hoisted, n=2^18)",
            "n_gpus": 1, "steps": 5, "warmup": 2, "higher_is_better": True, "vs_baseline": None,
            "dtype": "f32", "data": "synthetic", "config": {"workload": f"normalize_form, {args.index} index"},
            "forms": res, "gpu_launches": launches}
    if cpu:
        line["cpu_baseline"] = cpu
    if rank == 0:
        print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="libnorm", choices=["libnorm", "reference"])
    ap.add_argument("--workload", default="vector", choices=["vector", "rows", "paths28", "licm", "softmax", "backprop"])
    ap.add_argument("--index", default="literal", choices=["literal", "dense"])
    ap.add_argument("--path", default="auto", choices=["auto", "two_pass", "fused", "small"])
    ap.add_argument("--numel", dest="n", type=int, default=2**32)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--plan", default="balanced", choices=["balanced", "uniform"],
                    help="N > 1 literal shard plan (SURVEY §8(e)): coverage-balanced two-range "
                         "(default) or uniform one-range (rank 0 holds the whole covered prefix)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--also-dense", action="store_true", default=True)
    ap.add_argument("--exchange", default="p2p", choices=["nccl", "nccl-allreduce", "p2p", "host"],
                    help="N > 1: norm_launch_sharded (ncclAllGather), the fused peer-memory "
                         "exchange (norm_launch_sharded_peer), or the two-phase API over the "
                         "torch.distributed process group")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3  # timing rule: >= 3 untimed warm-up steps
    if args.impl == "reference":
        run_reference(args)
        return
    _wait_for_cuda()
    world, rank, local = dist_setup(args)
    try:
        if args.workload == "vector":
            run_vector(args, world, rank, local)
        elif args.workload == "rows":
            run_rows(args, world, rank, local)
        elif args.workload == "softmax":
            run_softmax(args, world, rank, local)
        elif args.workload == "backprop":
            run_backprop(args, world, rank, local)
        elif args.workload == "licm":
            run_licm(args, world, rank, local)
        else:
            run_paths28(args, world, rank, local)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
