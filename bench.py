#!/usr/bin/env python
"""bench.py — libnorm throughput on B200 (BASELINE.json metric:
"normalize GB/s and % of HBM peak, n=2^32 fp32, at 1/2/4/8 B200").

One step = one normalize of the whole workload (hoisted global sum over all n
elements, then the scale of the covered elements): two kernels (reduce, scale)
per rank, plus one 8-byte ncclAllGather when N > 1.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload vector|rows|fused28]
                  [--index literal|dense] [--impl libnorm|reference]

For N > 1 the driver launches it under torchrun (one process per GPU); a plain
`python bench.py --gpus N` re-executes itself under torch.distributed.run with N
ranks.  Rank 0 prints ONE JSON line.
value = algorithmic bytes of the whole job (4n + 8|C(n)|) per second
of the max-over-ranks device time.  Inputs (16 GiB at n = 2^32) are far larger than
the 126 MB L2, so no flush is needed between steps; the rows and softmax workloads
follow the same rule per GPU (timed_calls), the 2^28 path comparison and backprop flush.
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


# Source files that define each workload's dominant kernel: a committed ncu
# traffic figure counts only while their SHA-256 equals the one recorded at capture.
_CS = "paper_2207_00257_b200/csrc/"
_COMMON = [_CS + "device_common.cuh", _CS + "stream_common.cuh", _CS + "norm_internal.h"]
TRAFFIC_SOURCES = {
    "vector": [_CS + "reduce.cu"] + _COMMON,
    "scale": [_CS + "scale.cu"] + _COMMON,
    "paths28": [_CS + "fused.cu"] + _COMMON,
    "rows": [_CS + "rows.cu"] + _COMMON,
    "softmax": [_CS + "rowops.cu", _CS + "device_common.cuh", _CS + "norm_internal.h"],
    "backprop": [_CS + "backprop.cu"] + _COMMON,
    "small": [_CS + "fused.cu", _CS + "scale.cu"] + _COMMON,
}


def sources_sha256(files):
    import hashlib
    h = hashlib.sha256()
    for f in files:
        with open(os.path.join(ROOT, f), "rb") as fh:
            h.update(f.encode() + b"\0" + fh.read())
    return h.hexdigest()


def load_traffic(workload, index):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the workload's
    dominant kernel, from the committed ncu --set full capture
    (profiles/ncu_traffic.json, written by scripts/ncu_traffic_update.py), or None
    when there is no capture or the kernel's sources changed since it was taken."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            e = json.load(f).get(f"{workload}:{index}")
        if not isinstance(e, dict) or e.get("sources_sha256") != sources_sha256(e["sources"]):
            return None
        return e["bytes"]
    except Exception:
        return None


def single_kernel_roofline(algo_bytes, ms, peak, peak_src, kernel, traffic):
    """roofline object for a workload whose step is ONE kernel launch (the
    dominant kernel is the whole step): achieved = algorithmic bytes / launch time."""
    a = algo_bytes / (ms / 1e3) / 1e9
    return {"bound": "hbm", "achieved": a, "peak": peak, "unit": "GB/s", "frac": a / peak,
            "traffic": traffic, "kernel": kernel, "algorithmic_bytes_per_launch": algo_bytes,
            "avg_launch_ms": ms, "share_of_step": 1.0, "peak_source": peak_src}


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


def timed_calls(call, steps, in_bytes, flush, stream):
    """Device ms per call under the vector workload's timing rule: an input of at
    least 4 x L2 per GPU is timed as K back-to-back calls in one event pair (the
    previous call's dirty lines are written back inside the next one, as in a
    steady stream of calls); a smaller input gets the L2 flush before every call,
    outside per-call event pairs.  Also returns the per-call time with the flush
    ("isolated": cold L2, launch latency exposed) so both are on record."""
    import torch
    l2 = torch.cuda.get_device_properties(torch.cuda.current_device()).L2_cache_size
    per = []
    for _ in range(steps):
        flush()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        call()
        b.record(stream)
        torch.cuda.synchronize()
        per.append(a.elapsed_time(b))
    isolated = sum(per) / len(per)
    if in_bytes < 4 * l2:
        return isolated, isolated, "flushed before every step (256 MiB write, then a 256 MiB read so the " \
                                   "write-back happens outside the timed region)"
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(steps):
        call()
    b.record(stream)
    torch.cuda.synchronize()
    return (a.elapsed_time(b) / steps, isolated,
            f"no flush: {in_bytes / 2**30:.2f} GiB input per GPU >= 4 x L2 ({l2 >> 20} MiB), K calls back "
            f"to back in one event pair; isolated_ms = the same call with the L2 flushed before it")


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def oracle_bytes(n, index):
    """Algorithmic bytes 4n + 8|C(n)| from the ORACLE's closed-form coverage (the
    reference arm never loads the product library)."""
    import oracle
    count, _ = oracle.coverage_closed(n, index)
    return 4 * n + 8 * count


def oracle_sample(index, n_sample=2**28, reps=5):
    """Time the CPU oracle (form 3, hoisted O(N): exact sum, then the scale of
    C(n)) as it stands on a bounded sample of the same workload, on all of the
    host's cores (oracle_form_hoisted_mt: contiguous chunks accumulated exactly,
    merged in chunk order -- bit-identical to the single-thread form 3) and on one
    thread (the form as written); returns GB/s of algorithmic bytes."""
    import gen
    import oracle
    x = gen.make_host(n_sample, seed=2207, dist="unit")
    out = x.copy()
    T = os.cpu_count() or 1
    b = oracle_bytes(n_sample, index)

    def med(fn, k):
        ts = []
        for _ in range(k):
            t0 = time.perf_counter()
            fn()
            ts.append(time.perf_counter() - t0)
        return statistics.median(ts)
    tT = med(lambda: oracle.form_hoisted_mt(x, index, threads=T, out=out), reps)
    t1 = med(lambda: oracle.form_hoisted(x, index, out=out), 3)
    return {"value": b / tT / 1e9, "unit": "GB/s", "cores": T, "kind": "oracle",
            "sample": f"oracle form 3 (exact sum of all n, then in[i]/val over C(n)), n={n_sample} "
                      f"{index} index, {T} threads (contiguous chunks, exact chunk-order merge), "
                      f"median of {reps}: {tT:.3f} s; {cpu_model()}",
            "single_thread": {"value": b / t1 / 1e9, "unit": "GB/s", "cores": 1,
                              "sample": f"same sample, oracle_form_hoisted (1 thread), median of 3: {t1:.3f} s"}}


def run_meta(world=1):
    """Versions of everything the number depends on (SURVEY §5 run metadata;
    PAPER.md:770-774 records its own machine and versions)."""
    import ctypes
    import platform
    m = {"torch": None, "cuda_runtime": None, "gpu": None, "driver": None, "nccl_libnorm": None,
         "nccl_torch": None, "host_cpu": cpu_model(), "host_cores": os.cpu_count(),
         "python": platform.python_version(), "world_size": world}
    try:
        import torch
        m["torch"] = torch.__version__
        m["cuda_runtime"] = torch.version.cuda
        if torch.cuda.is_available():
            m["gpu"] = torch.cuda.get_device_name()
            cc = torch.cuda.get_device_capability()
            m["sm"] = f"sm_{cc[0]}{cc[1]}"
        try:
            v = torch.cuda.nccl.version()
            m["nccl_torch"] = ".".join(map(str, v)) if isinstance(v, tuple) else str(v)
        except Exception:  # noqa: BLE001
            pass
    except Exception:  # noqa: BLE001
        pass
    try:
        v = ctypes.c_int()
        ctypes.CDLL("libnccl.so.2").ncclGetVersion(ctypes.byref(v))  # the one libnorm.so links (rpath)
        m["nccl_libnorm"] = f"{v.value // 10000}.{(v.value % 10000) // 100}.{v.value % 100}"
    except Exception:  # noqa: BLE001
        pass
    try:
        r = subprocess.run(["nvidia-smi", "--query-gpu=driver_version", "--format=csv,noheader"],
                           capture_output=True, text=True, timeout=20)
        m["driver"] = r.stdout.strip().splitlines()[0] if r.returncode == 0 and r.stdout.strip() else None
    except Exception:  # noqa: BLE001
        pass
    return m


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
    """The reference arm for this tier: the CPU oracle (form 3) as it stands, on
    all host cores, over a bounded sample of the workload per step.  Loads only
    oracle/ and gen/ -- never the product library."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    n_sample = 2**26
    steps = []
    import gen
    import oracle
    T = os.cpu_count() or 1
    x = gen.make_host(n_sample, seed=2207, dist="unit")
    out = x.copy()
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        oracle.form_hoisted_mt(x, args.index, threads=T, out=out)
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            steps.append(dt)
    ms = 1e3 * sum(steps) / len(steps)
    b = oracle_bytes(n_sample, args.index)
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
        "cpu_baseline": {"value": v, "unit": "GB/s", "cores": T, "kind": "oracle",
                         "sample": f"n={n_sample} per step, oracle_form_hoisted_mt on {T} threads "
                                   f"(exact chunk accumulators; bit-identical to form 3) ({cpu_model()})"},
        "e2e": {"value": v, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "meta": {"host_cpu": cpu_model(), "host_cores": T, "world_size": world,
                 "note": "oracle only: loads oracle/liboracle.so and gen/libnormgen.so, not libnorm.so"},
    }
    emit(line)


def min_over_ranks(v, world):
    return -max_over_ranks(-v, world)


def _emulated():
    """N > 1 ranks time-slicing one GPU over gloo (harness tests only): NCCL
    refuses two ranks on one device, so the NCCL exchanges are not run."""
    return os.environ.get("NORM_BENCH_BACKEND", "nccl") != "nccl"


def make_exchange(L, name, world):
    """A libnorm communicator for one of the N > 1 exchanges, or None for the
    caller-collective path ("host")."""
    if name == "p2p":
        return L.PeerComm()
    if name in ("nccl", "nccl-allreduce"):
        return L.Comm(allreduce=name == "nccl-allreduce")
    return None


def sharded_step_fn(L, comm, out, inp, mine, n, index, world, path="auto"):
    if comm is None:
        ag = host_all_gather(world)
        return lambda ev=None: L.normalize_sharded_via(out, inp, mine, n, ag, index=index, events=ev)
    if isinstance(comm, L.PeerComm):
        return lambda ev=None: comm.normalize_sharded(out, inp, mine, n, index=index, events=ev, path=path)
    return lambda ev=None: comm.normalize_sharded(out, inp, mine, n, index=index, events=ev)


def time_steps(step, steps, world, flush=None):
    """Device time per step (ms, this rank): K steps bracketed by barrier + sync.
    Without flush: one event pair around the K back-to-back steps.  With flush:
    the L2 flush runs between steps, outside per-step event pairs."""
    import torch
    stream = torch.cuda.current_stream()
    barrier(world)
    if flush is None:
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(steps):
            step()
        b.record(stream)
        torch.cuda.synchronize()
        barrier(world)
        return a.elapsed_time(b) / steps
    per = []
    for _ in range(steps):
        flush()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        step()
        b.record(stream)
        torch.cuda.synchronize()
        per.append(a.elapsed_time(b))
    barrier(world)
    return sum(per) / len(per)


def reduce_times(step, steps, world, flush=None):
    """Average duration of the step's dominant kernel (norm_debug_set_events on the
    launch stream) and of the instrumented step, in a separate pass: an event
    between the reduce and the scale would defeat their programmatic dependent
    launch, so the headline steps carry none.  With flush: L2 flushed before
    every step, outside the step's events."""
    import torch
    stream = torch.cuda.current_stream()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    barrier(world)
    if flush is None:
        i0, i1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        i0.record(stream)
        for k in range(steps):
            step(evs[k])
        i1.record(stream)
        torch.cuda.synchronize()
        instr = i0.elapsed_time(i1) / steps
    else:
        per = []
        for k in range(steps):
            flush()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            step(evs[k])
            b.record(stream)
            torch.cuda.synchronize()
            per.append(a.elapsed_time(b))
        instr = sum(per) / len(per)
    barrier(world)
    red = [b.elapsed_time(e) for b, e in evs]
    return sum(red) / len(red), instr


def exchange_record(L, name, out, inp, mine, n, index, world, args, flush):
    """The same sharded step through another exchange (N > 1): step time (max
    and min over ranks), the dominant kernel's time, and the rest (exchange +
    scale, or the fused kernel's own exchange inside it)."""
    comm = make_exchange(L, name, world)
    try:
        step = sharded_step_fn(L, comm, out, inp, mine, n, index, world)
        for _ in range(args.warmup):
            step()
        ms_local = time_steps(step, args.steps, world, flush)
        red, instr = reduce_times(step, args.steps, world, flush)
        algo = L.algorithmic_bytes(n, index)
        ms = max_over_ranks(ms_local, world)
        return {"exchange": name, "value": algo / (ms / 1e3) / 1e9, "unit": "GB/s", "ms_per_step": ms,
                "rank_ms_min": min_over_ranks(ms_local, world), "rank_ms_max": ms,
                "dominant_kernel_ms_max": max_over_ranks(red, world),
                "rest_of_step_ms_max": max_over_ranks(instr - red, world)}
    finally:
        if comm is not None:
            comm.destroy()


def plan_record(L, comm, plan_name, n, index, world, rank, args, flush):
    """The same sharded step under the OTHER literal shard plan (SURVEY §8(e):
    report both): the coverage-balanced two-range plan, or the uniform one-range
    plan in which rank 0 scales the whole covered prefix after the exchange.
    Fresh buffers for this plan's ranges, same exchange, max over ranks."""
    import torch
    import gen
    plan = L.plan_shards(n, world, index, plan_name == "balanced")
    mine = plan[rank]
    nloc = sum(ln for _, ln in mine)
    inp = torch.empty(max(nloc, 1), dtype=torch.float32, device="cuda")[:nloc]
    off = 0
    for b, ln in mine:
        gen.fill_cuda(inp[off:off + ln], seed=2207, dist="unit", offset=b)
        off += ln
    out = torch.empty_like(inp)
    try:
        step = sharded_step_fn(L, comm, out, inp, mine, n, index, world)
        for _ in range(args.warmup):
            step()
        ms_local = time_steps(step, args.steps, world, flush)
        ms = max_over_ranks(ms_local, world)
        algo = L.algorithmic_bytes(n, index)
        return {"plan": "coverage-balanced two-range" if plan_name == "balanced" else "uniform one-range",
                "value": algo / (ms / 1e3) / 1e9, "unit": "GB/s", "ms_per_step": ms,
                "rank_ms_min": min_over_ranks(ms_local, world), "rank_ms_max": ms}
    finally:
        del inp, out
        torch.cuda.empty_cache()


def exchange_latency(L, names, world, index, reps=200):
    """Latency of one sharded normalize over a tiny vector (8192 elements per
    rank: the kernels are launch-bound, so the step is launch + exchange +
    launch), per exchange, max over ranks -- the cost the exchange adds to a
    step, measured on the device."""
    import torch
    n = 8192 * world
    mine = L.plan_shards(n, world, index, True)[torch.distributed.get_rank()]
    nl = sum(ln for _, ln in mine)
    inp = torch.ones(nl, device="cuda")
    out = torch.empty_like(inp)
    res = {}
    for name in names:
        comm = make_exchange(L, name, world)
        try:
            step = sharded_step_fn(L, comm, out, inp, mine, n, index, world)
            for _ in range(10):
                step()
            ms = time_steps(step, reps, world)
            res[name] = {"us_per_step_max": 1e3 * max_over_ranks(ms, world),
                         "us_per_step_min": 1e3 * min_over_ranks(ms, world)}
        except Exception as e:  # noqa: BLE001
            res[name] = {"unavailable": str(e)[:200]}
        finally:
            if comm is not None:
                comm.destroy()
    res["n_per_rank"] = nl
    return res


def parity_record(L, out, inp, n, index, sentinel_bits):
    """Parity of the benched launch (N = 1) against the oracle, on the bench's own
    buffers (SURVEY §5 'parity status in the JSON line'): one extra call with
    sum_out; s vs the oracle's exact sum of all n inputs (oracle_sum_exact_mt
    over a host copy); 2^20 sampled covered outputs
    replayed bitwise (in[i] / s in binary32) and within 1e-5 of in[i] / S; 2^16
    sampled uncovered outputs still hold the sentinel."""
    import numpy as np
    import torch
    import oracle
    nl = inp.numel()
    need = 4 * nl
    try:
        avail = 0
        for line in open("/proc/meminfo"):
            if line.startswith("MemAvailable:"):
                avail = int(line.split()[1]) * 1024
        if avail and avail < 3 * need:
            return {"ok": None, "skipped": f"host MemAvailable {avail >> 30} GiB < 3 x {need >> 30} GiB shard"}
    except OSError:
        pass
    s = torch.zeros(1, device="cuda")
    L.normalize(out, inp, index=index, sum_out=s)
    torch.cuda.synchronize()
    x = np.empty(nl, dtype=np.float32)
    step = 1 << 28
    for a in range(0, nl, step):
        x[a:a + step] = inp[a:a + step].cpu().numpy()
    S = oracle.sum_exact_mt(x)
    sv = np.float32(s.item())
    rel_s = abs(float(sv) - S) / abs(S)
    count, prefix = oracle.coverage_closed(n, index)
    rng = np.random.default_rng(2207)
    if prefix >= 0:
        ci = rng.integers(0, prefix, 1 << 20) if prefix > 0 else np.zeros(0, np.int64)
        ui = rng.integers(prefix, n, 1 << 16) if prefix < n else np.zeros(0, np.int64)
    else:
        mask = oracle.covered_mask(n, index)
        ci = rng.choice(np.nonzero(mask)[0], 1 << 20)
        ui = rng.choice(np.nonzero(~mask)[0], 1 << 16) if (~mask).any() else np.zeros(0, np.int64)
    idx = torch.from_numpy(np.concatenate([ci, ui])).cuda()
    o = out[idx].cpu().numpy()
    oc, ou = o[:ci.size], o[ci.size:]
    replay = bool(np.array_equal(oc.view(np.uint32), (x[ci] / sv).view(np.uint32)))
    ref = x[ci].astype(np.float64) / S
    max_rel = float(np.max(np.abs(oc - ref) / ref)) if ci.size else 0.0
    untouched = bool(np.all(ou.view(np.uint32) == sentinel_bits))
    ok = rel_s <= 1e-6 and replay and max_rel <= 1e-5 and untouched
    del x
    return {"ok": ok, "s": float(sv), "S_exact": S, "rel_err_s": rel_s, "tol_s": 1e-6,
            "covered_sampled": int(ci.size), "replay_bitwise": replay, "max_rel_err": max_rel, "tol": 1e-5,
            "uncovered_sampled": int(ui.size), "uncovered_untouched": untouched,
            "oracle": "oracle_sum_exact_mt (exact superaccumulator) over all n inputs on the host"}


SENTINEL_BITS = 0x7FC0FFEE


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
    # uncovered outputs are never written: prefill a sentinel so parity can see that
    out = torch.empty_like(inp)
    out.view(torch.int32).fill_(SENTINEL_BITS)
    torch.cuda.synchronize()
    l2 = torch.cuda.get_device_properties(torch.cuda.current_device()).L2_cache_size
    # Timing rule: inputs larger than L2 or an L2 flush between timed steps.
    flush = None if 4 * nloc >= 4 * l2 else L2Flush()
    l2_note = (f"no flush: {4 * nloc / 2**30:.2f} GiB input per GPU >= 4 x L2 ({l2 >> 20} MiB)" if flush is None
               else f"L2 flushed before every step (256 MiB write + 256 MiB read, outside the per-step "
                    f"events): {4 * nloc / 2**20:.1f} MiB input per GPU < 4 x L2")
    comm = None
    exchange_note = None
    if world > 1 and args.exchange == "p2p":
        # the fused peer-memory exchange, cross-checked once against the gathered
        # partials (same kernels, exchange over the process group); any failure or
        # mismatch falls back to NCCL and is recorded in the JSON line
        # Every rank runs the same sequence of collectives whatever fails locally
        # (PeerComm agrees on set-up failures itself; the check below is one
        # all-gather of the ranks' errors), so a failure on one rank cannot leave the others waiting
        # in a collective the failed rank never enters.
        import torch.distributed as dist
        err = None
        try:
            comm = L.PeerComm()
        except Exception as e:  # noqa: BLE001  (raised on every rank together)
            err = str(e)
        if comm is not None:
            s_p = torch.zeros(1, device="cuda")
            s_g = torch.zeros(1, device="cuda")
            try:
                comm.normalize_sharded(out, inp, mine, n, index=index, sum_out=s_p)
            except Exception as e:  # noqa: BLE001
                err = f"norm_launch_sharded_peer: {e}"
            try:
                L.normalize_sharded_via(out, inp, mine, n, host_all_gather(world), index=index, sum_out=s_g)
                torch.cuda.synchronize()
            except Exception as e:  # noqa: BLE001
                err = err or f"gathered cross-check: {e}"
            if err is None and not torch.equal(s_p, s_g):
                err = "p2p divisor != gathered divisor"
            if err is None and os.environ.get("NORM_BENCH_FAULT_P2P_RANK") == str(rank):
                err = "injected fault (NORM_BENCH_FAULT_P2P_RANK, tests only)"
            errs = [None] * world
            dist.all_gather_object(errs, err)
            bad = [f"rank {r}: {e}" for r, e in enumerate(errs) if e]
            err = "; ".join(bad) if bad else None
        if err is not None:
            # NCCL on a real node; the caller-collective path when the ranks
            # time-slice one GPU (NCCL refuses two ranks on one device)
            fallback = "host" if _emulated() else "nccl"
            exchange_note = f"p2p unavailable ({err}); fell back to {fallback}"
            print(f"[bench] {exchange_note}", file=sys.stderr)
            if comm is not None:
                try:
                    comm.destroy()
                except Exception:  # noqa: BLE001
                    pass
            comm = None
            args.exchange = fallback
    if world > 1 and args.exchange in ("nccl", "nccl-allreduce") and comm is None:
        comm = L.Comm(allreduce=args.exchange == "nccl-allreduce")
    stream = torch.cuda.current_stream()

    if world == 1:
        def step(ev=None):
            L.normalize(out, inp, index=index, path=args.path, events=ev)
    else:
        step = sharded_step_fn(L, comm, out, inp, mine, n, index, world)

    for _ in range(args.warmup):
        step()
    # Timed region: K whole steps, bracketed by barrier + sync.
    barrier(world)
    with ClockSampler(local) as clk:
        ms_local = time_steps(step, args.steps, world, flush)
    # Timing rule: a region that saw hw_slowdown / hw_thermal_slowdown /
    # sw_thermal_slowdown on any rank is rejected and re-measured once (the
    # first attempt is recorded in the line); sw_power_cap is kept and noted.
    remeasured = None
    first_reasons = clk.summary().get("reasons", [])
    if os.environ.get("NORM_BENCH_FAKE_THROTTLE"):  # tests only: exercise the re-measure path
        first_reasons = sorted(set(first_reasons) | {"hw_slowdown"})
    bad = any(r in ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown") for r in first_reasons)
    if max_over_ranks(1.0 if bad else 0.0, world) > 0:
        remeasured = {"first_ms_per_step": max_over_ranks(ms_local, world), "first_reasons_rank0": first_reasons}
        barrier(world)
        with ClockSampler(local) as clk:
            ms_local = time_steps(step, args.steps, world, flush)
    ms = max_over_ranks(ms_local, world)
    ms_min = min_over_ranks(ms_local, world)
    red_ms_avg, ms_instr = reduce_times(step, args.steps, world, flush)
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
    fused_step = kpath in ("fused", "mid", "cluster")
    small_step = kpath == "small"
    # the kernel libnorm brackets with the bench events (norm_debug_set_events):
    # the one kernel of a fused / mid / cluster / small step; on a two-pass step the
    # reduce (4n), or at N = 1 the scale when it moves more (8|C| > 4n, dense)
    scale_dom = (world == 1 and not (fused_step or small_step) and lloc >= 0 and 2 * lloc > nloc)
    red_bytes = (8 * lloc if scale_dom else
                 4 * nloc + (8 * max(lloc, 0) if (fused_step or small_step) else 0))
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
        scratch = torch.empty_like(inp)
        cms = _t(lambda: scratch.copy_(inp))
        rms = _t(lambda: torch.sum(inp))
        del scratch
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
             "p90_ms": max_over_ranks(per[min(len(per) - 1, int(0.9 * len(per)))], world),
             "rank_ms_min": ms_min, "rank_ms_max": ms}
    if world == 1:
        g = L.NormGraph(out, inp, index=index, path=args.path)
        for _ in range(2):
            g.launch()
        gms = time_steps(g.launch, args.steps, world, flush)
        stats["graph_ms_per_step"] = gms
        stats["graph_value"] = L.algorithmic_bytes(n, index) / (gms / 1e3) / 1e9
        g.destroy()
    extra["step_stats"] = stats
    # N > 1: the same step through the other exchanges, so one driver run measures
    # the north_star's NCCL all-reduce of the scalar beside the fused peer exchange
    if world > 1:
        alt = {}
        for name in ("nccl-allreduce", "nccl", "p2p", "host"):
            if name == args.exchange or (name.startswith("nccl") and _emulated()):
                continue
            try:
                alt[name] = exchange_record(L, name, out, inp, mine, n, index, world, args, flush)
            except Exception as e:  # noqa: BLE001
                alt[name] = {"exchange": name, "unavailable": str(e)[:300]}
        if _emulated():
            alt["note"] = "ranks time-slice one GPU over gloo: NCCL exchanges not run (NCCL needs one GPU per rank)"
        extra["exchanges"] = alt
        if "nccl-allreduce" in alt:
            extra["nccl_allreduce"] = alt["nccl-allreduce"]
        names = ["p2p", "host"] + ([] if _emulated() else ["nccl-allreduce", "nccl"])
        extra["exchange_latency"] = exchange_latency(L, names, world, index)
        if index == "literal":  # both literal shard plans in one driver run
            other = "uniform" if args.plan == "balanced" else "balanced"
            try:
                extra["other_shard_plan"] = plan_record(L, comm, other, n, index, world, rank, args, flush)
            except Exception as e:  # noqa: BLE001
                extra["other_shard_plan"] = {"plan": other, "unavailable": str(e)[:300]}
    # dense-index figure on the same buffers (caption reading R1), reported beside the headline
    if args.also_dense and index == "literal" and (world == 1 or comm is not None):
        dense_mine = L.plan_shards(n, world, "dense", True)[rank]
        if dense_mine == mine or world == 1:
            if world == 1:
                def dstep():
                    L.normalize(out, inp, index="dense", path="auto")
            else:
                dstep = sharded_step_fn(L, comm, out, inp, mine, n, "dense", world)
            for _ in range(2):
                dstep()
            dms = max_over_ranks(time_steps(dstep, args.steps, world, flush), world)
            dbytes = L.algorithmic_bytes(n, "dense")
            extra["dense_index"] = {"value": dbytes / (dms / 1e3) / 1e9, "unit": "GB/s", "ms_per_step": dms,
                                    "frac_of_peak": dbytes / (dms / 1e3) / 1e9 / (world * peak)}
            out.view(torch.int32).fill_(SENTINEL_BITS)  # dense wrote every element: restore the sentinel
            for _ in range(1):
                step()
            torch.cuda.synchronize()
    # e2e: same metric through the public API with host buffers, copies inside the timed region
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, world, rank, local, mine, n, index)
    launches_per_step = 1 if (fused_step or small_step) else 2
    # The cpu_baseline leg (rank 0 at N = 1, after every GPU measurement) -- with
    # --impl reference the only place bench.py runs oracle/: the oracle timed on a
    # bounded sample, and the benched launch's parity against the oracle.
    cpu = None
    parity = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = oracle_sample(index)
        if not args.no_parity:
            parity = parity_record(L, out, inp, n, index, SENTINEL_BITS)
            parity["leg"] = "cpu_baseline (oracle on the host, after the GPU measurements)"
    meta = run_meta(world)
    if rank != 0:
        return
    cov_count, prefix = L.coverage(n, index)
    kname = ("cluster_kernel (one 16-CTA cluster: reduce, DSMEM combine, scale: the whole step)"
             if kpath == "cluster" else
             "mid_kernel (256-bit loads, grid barrier, exchange, scale: the whole step)" if kpath == "mid" else
             "fused_kernel (reduce + grid barrier + exchange + scale: the whole step)" if fused_step else
             "small_kernel (one CTA: sum, barrier, scale: the whole step)" if small_step else
             "scale_tile_kernel (one 8 KiB tile per CTA: 8|C| of the step's 4n + 8|C| bytes)" if scale_dom else
             ("reduce_dyn_kernel (TMA-bulk reduce, dynamic deterministic tail)" if nloc >= (1 << 22)
              else "reduce_kernel") + " (the hoisted sum: 4n of the step's 4n + 8|C| bytes)")
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
                   "l2": l2_note},
        "frac_of_hbm_peak": value / (world * peak),
        "frac_of_datasheet": value / (world * DATASHEET_GBS),
        "calibration": calib,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak,
                     "traffic": (load_traffic("scale" if scale_dom else "vector", index)
                                 if (world == 1 and n == 2**32) else None),
                     "kernel": kname,
                     "algorithmic_bytes_per_launch": red_bytes, "avg_launch_ms": red_ms_avg,
                     "share_of_step": red_ms_avg / ms_instr, "instrumented_ms_per_step": ms_instr,
                     ("frac_of_same_run_copy_stream" if scale_dom else "frac_of_same_run_read_stream"):
                         (achieved / calib["torch_copy_gbs" if scale_dom else "torch_sum_gbs"]) if calib else None,
                     "peak_source": peak_src},
        "gpu_launches": launches_per_step * args.steps,
        "clocks": clk.summary(),
        "meta": meta,
    }
    line.update(extra)
    if remeasured is not None:
        line["remeasured"] = remeasured
    if parity is not None:
        line["parity"] = parity
    if e2e:
        line["e2e"] = e2e
    if cpu:
        line["cpu_baseline"] = cpu
    emit(line)
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
    barrier(world)
    with ClockSampler(local) as clk:
        ms_local, iso_local, l2_note = timed_calls(lambda: L.normalize_rows(out, inp, index=args.index),
                                                   args.steps, 4 * rl * C, flush, stream)
    barrier(world)
    ms = max_over_ranks(ms_local, world)
    iso = max_over_ranks(iso_local, world)
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
                   "rows": R, "cols": C, "index": args.index, "algorithmic_bytes": algo, "l2": l2_note},
        "frac_of_hbm_peak": value / (world * peak),
        "isolated": {"ms_per_step": iso, "value": algo / (iso / 1e3) / 1e9},
        # one kernel per step; which one is libnorm's launch_rows rule for 4096-float
        # rows: the TMA warp-per-row kernel when at most half of a row is covered
        # (literal: 1120 of 4096), else the register kernel with the row queue
        "roofline": single_kernel_roofline(
            rl * (4 * C + 4 * cov), ms, peak, src,
            ("rows_bulk_kernel (TMA warp-per-row)" if 2 * cov <= C else "rows_vec_kernel (register rows, row queue)")
            + " -- the whole step", load_traffic("rows", args.index) if world == 1 else None),
        "gpu_launches": args.steps,
        "clocks": clk.summary(),
    }
    emit(line)


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
    # the gradient at the same n (norm_launch_backward): a dot over the covered set
    # (reads g, y there) and an elementwise pass (reads g, writes gx): 8|C| + 8n bytes
    y = inp.clone()
    s = torch.zeros(1, device="cuda")
    L.normalize(y, y, index=args.index, sum_out=s)
    g = torch.empty_like(inp)
    gen.fill_cuda(g, seed=2208, dist="signed")
    gx = torch.empty_like(inp)
    for _ in range(args.warmup):
        L.normalize_backward(gx, g, y, s, index=args.index)
    bms, biso, bnote = timed_calls(lambda: L.normalize_backward(gx, g, y, s, index=args.index), args.steps,
                                   8 * n, flush, stream)
    cov, _ = L.coverage(n, args.index)
    bbytes = 8 * cov + 8 * n
    backward = {"ms_per_step": bms, "isolated_ms": biso, "value": bbytes / (bms / 1e3) / 1e9,
                "frac": bbytes / (bms / 1e3) / 1e9 / peak, "bytes": bbytes, "l2": bnote,
                "kernels": "vec_bwd_dot_kernel + vec_bwd_apply_kernel"}
    del y, g, gx
    line = {"metric": "normalize GB/s and % of HBM peak (n=2^28, two-pass vs fused)",
            "value": res[best]["value"], "unit": "GB/s", "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": res[best]["ms_per_step"], "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": f"normalize n=2^28 fp32, {args.index}, best path = {best}",
                       "l2": "flushed before every step (256 MiB write, then a 256 MiB read so the write-back happens outside the timed region)"},
            "paths": res, "backward": backward, "peak": peak,
            "gpu_launches": args.steps * 3}  # two-pass (2 kernels) + fused (1) per step
    if best == "fused":
        line["roofline"] = single_kernel_roofline(
            L.algorithmic_bytes(n, args.index), res["fused"]["ms_per_step"], peak, src,
            "fused_kernel (single pass, grid barrier; scored on 4n + 8|C|)",
            load_traffic("paths28", args.index))
    if rank == 0:
        emit(line)


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
        ms, iso, l2_note = timed_calls(lambda: L.softmax_rows(out, inp, log=log), args.steps, 4 * R * C,
                                       flush, stream)
        v = 8 * R * C / (ms / 1e3) / 1e9
        res["log_softmax" if log else "softmax"] = {"ms_per_step": ms, "value": v, "frac": v / peak,
                                                    "isolated_ms": iso}
        # torch's own kernel on the same data and timing, for context
        fn = torch.log_softmax if log else torch.softmax
        for _ in range(args.warmup):
            fn(inp, dim=1)
        tms, tiso, _ = timed_calls(lambda: fn(inp, dim=1), args.steps, 4 * R * C, flush, stream)
        res[("log_softmax" if log else "softmax") + "_torch"] = {"ms_per_step": tms, "isolated_ms": tiso,
                                                                 "value": 8 * R * C / (tms / 1e3) / 1e9}
    # gradients (norm_softmax_rows_backward, norm_rows_backward): read g and y, write gx
    g = torch.empty_like(inp)
    gen.fill_cuda(g.view(-1), seed=2208, dist="signed")
    gx = torch.empty_like(inp)
    for log in (False, True):
        L.softmax_rows(out, inp, log=log)
        for _ in range(args.warmup):
            L.softmax_rows_backward(gx, g, out, log=log)
        ms, iso, _ = timed_calls(lambda: L.softmax_rows_backward(gx, g, out, log=log), args.steps, 8 * R * C,
                                 flush, stream)
        nm = "log_softmax_backward" if log else "softmax_backward"
        res[nm] = {"ms_per_step": ms, "isolated_ms": iso, "value": 12 * R * C / (ms / 1e3) / 1e9,
                   "frac": 12 * R * C / (ms / 1e3) / 1e9 / peak}
        for _ in range(args.warmup):
            torch._softmax_backward_data(g, out, 1, torch.float32) if not log else \
                torch._log_softmax_backward_data(g, out, 1, torch.float32)
        tms, tiso, _ = timed_calls(
            (lambda: torch._log_softmax_backward_data(g, out, 1, torch.float32)) if log else
            (lambda: torch._softmax_backward_data(g, out, 1, torch.float32)), args.steps, 8 * R * C, flush, stream)
        res[nm + "_torch"] = {"ms_per_step": tms, "isolated_ms": tiso, "value": 12 * R * C / (tms / 1e3) / 1e9}
    srow = torch.zeros(R, device="cuda")
    L.normalize_rows(out, inp.abs(), index="dense", sum_out=srow)
    for _ in range(args.warmup):
        L.normalize_rows_backward(gx, g, out, srow, index="dense")
    ms, iso, _ = timed_calls(lambda: L.normalize_rows_backward(gx, g, out, srow, index="dense"), args.steps,
                             8 * R * C, flush, stream)
    res["rows_normalize_backward_dense"] = {"ms_per_step": ms, "isolated_ms": iso,
                                            "value": 12 * R * C / (ms / 1e3) / 1e9,
                                            "frac": 12 * R * C / (ms / 1e3) / 1e9 / peak}
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
                       "l2": "softmax / log-softmax (libnorm and torch): " + l2_note + "; nll_forward / "
                             "nll_backward: flushed before every step (their reads are far below 4 x L2)"},
            "frac_of_hbm_peak": res["softmax"]["frac"], "peak": peak, "results": res,
            "roofline": single_kernel_roofline(8 * R * C, res["softmax"]["ms_per_step"], peak, src,
                                               "softmax_vec_kernel (one read + one write per element)",
                                               load_traffic("softmax", "dense")),
            "gpu_launches": args.steps}
    if rank == 0:
        emit(line)


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
    peak, peak_src = load_peak()
    line = {"metric": "bpnn_layerforward GB/s (Rodinia backprop, Fig. backprop), in=2^22, hid=16",
            "value": res["tma"]["value"], "unit": "GB/s", "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": res["tma"]["ms_per_step"],
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic", "config": {"workload": "norm_bpnn_layerforward in=2^22 hid=16",
                                            "l2": "flushed before every step (256 MiB write, then a 256 MiB read so the write-back happens outside the timed region)"},
            "variants": res, "frac_of_hbm_peak": res["tma"]["value"] / peak,
            "roofline": single_kernel_roofline(nbytes, res["tma"]["ms_per_step"], peak, peak_src,
                                               "bpnn_tma_kernel (hidden read + write, input read, output write)",
                                               load_traffic("backprop", "tma")),
            "speedup_eliminated_over_printed": res["printed"]["ms_per_step"] / res["eliminated"]["ms_per_step"],
            "speedup_register_over_printed": res["printed"]["ms_per_step"] / res["register"]["ms_per_step"],
            "speedup_tma_over_printed": res["printed"]["ms_per_step"] / res["tma"]["ms_per_step"],
            "gpu_launches": args.steps * len(res)}
    if rank == 0:
        emit(line)


def run_small(args, world, rank, local):
    """BASELINE configs[0] and configs[1] ("latency-bound (us)",
    "report us hot and with L2 flushed"): n = 1024 (Fig. 1's 32 x 32 literal
    grid) and n = 2^20 + 7 (ragged: literal coverage leaves
    outputs untouched), on every path.  Per path and size:
      device_hot_us    -- one CUDA graph of R back-to-back calls, replayed; device
                          time / R (no host in the loop);
      device_flushed_us-- graph of R x (L2 flush + call) minus graph of R x flush,
                          / R: the call with its input evicted from L2;
      python_us        -- back-to-back calls through the Python binding
                          (trusted pointers), wall time / call;
      python_bound_us  -- the same through L.BoundNormalize (arguments
                          marshalled once, one ctypes call per call);
      c_*              -- examples/latency_c: host enqueue and back-to-back wall
                          time per call from plain C, with and without libnorm's
                          pointer checks, and through a norm_graph_t replay;
      parity           -- each path's output vs the oracle (exact S within 1e-6,
                          bitwise replay, uncovered outputs untouched), taken in
                          the cpu_baseline leg after every GPU measurement."""
    import numpy as np
    import torch
    import gen
    import paper_2207_00257_b200 as L
    stream = torch.cuda.current_stream()
    ws = torch.zeros(L.workspace_bytes(), dtype=torch.uint8, device="cuda")
    R = 100
    flush_w = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    flush_r = torch.ones(64 << 20, dtype=torch.float32, device="cuda")

    def flush():
        flush_w.zero_()
        flush_r.sum()

    def graph_us(body, reps=10):
        side = torch.cuda.Stream()
        side.wait_stream(stream)
        with torch.cuda.stream(side):
            body()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=side):
                body()
        torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(reps):
            g.replay()
        b.record(stream)
        torch.cuda.synchronize()
        return a.elapsed_time(b) * 1e3 / reps

    res = []
    outputs = []
    for n in (1024, 2**20 + 7):
        xh = gen.make_host(n, seed=2207, dist="unit")
        x = torch.from_numpy(xh).cuda()
        out = torch.empty_like(x)
        count, prefix = L.coverage(n, args.index)
        t_flush = graph_us(lambda: [flush() for _ in range(20)]) / 20
        for path in ("auto", "small", "cluster", "mid", "two_pass", "fused"):
            chosen = L.choose_path(n, prefix, path)

            def call():
                L.normalize(out, x, index=args.index, path=path, workspace=ws, trusted=True)
            # this path's output for the parity check of the cpu_baseline leg
            # (sentinel-filled output, then one call)
            out.view(torch.int32).fill_(SENTINEL_BITS)
            s = torch.zeros(1, device="cuda")
            L.normalize(out, x, index=args.index, path=path, workspace=ws, sum_out=s)
            torch.cuda.synchronize()
            outputs.append((xh, out.cpu().numpy(), np.float32(s.item())))
            hot = graph_us(lambda: [call() for _ in range(R)]) / R
            fl = (graph_us(lambda: [(flush(), call()) for _ in range(20)]) / 20) - t_flush
            for _ in range(200):
                call()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(2000):
                call()
            torch.cuda.synchronize()
            py = (time.perf_counter() - t0) / 2000 * 1e6
            bound = L.BoundNormalize(out, x, index=args.index, path=path)
            for _ in range(200):
                bound()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(2000):
                bound()
            torch.cuda.synchronize()
            py_bound = (time.perf_counter() - t0) / 2000 * 1e6
            res.append({"n": n, "path": path, "runs": chosen, "device_hot_us": hot, "device_flushed_us": fl,
                        "python_us": py, "python_bound_us": py_bound})
    # plain C: host enqueue / back-to-back per call
    cres = []
    exe = os.path.join(ROOT, "examples", "latency_c")
    if os.path.exists(exe):
        r = subprocess.run([exe, "1024", str(2**20 + 7)], capture_output=True, text=True, timeout=600)
        cres = [json.loads(ln) for ln in r.stdout.splitlines() if ln.startswith("{")]
    for row in res:
        for c in cres:
            if c.get("n") == row["n"] and c.get("path") == row["path"]:
                row.update({("c_" + k): v for k, v in c.items() if k not in ("n", "path", "runs")})
    # cpu_baseline leg (after every GPU measurement; the only use of oracle/ here):
    # each path's output against the oracle, and the oracle's own time per call
    parity = cpu = None
    if not args.no_cpu:
        import oracle
        ok_all = True
        for row, (xh, o, sv) in zip(res, outputs):
            S = oracle.sum_exact(xh)
            sent = np.full(xh.size, SENTINEL_BITS, np.uint32).view(np.float32)
            rep = oracle.replay(xh, sv, args.index, out=sent.copy())
            ok = abs(float(sv) - S) <= 1e-6 * S and np.array_equal(o.view(np.uint32), rep.view(np.uint32))
            row["parity_ok"] = bool(ok)
            ok_all &= bool(ok)
        parity = {"ok": ok_all, "leg": "cpu_baseline (oracle on the host, after the GPU measurements)",
                  "what": "per path and size: |s - S| <= 1e-6 S and the whole output == oracle_replay(x, s) bitwise"}
        xh = gen.make_host(1024, seed=2207, dist="unit")
        ob = np.empty_like(xh)
        oracle.form_hoisted(xh, args.index, out=ob)
        t0 = time.perf_counter()
        for _ in range(2000):
            oracle.form_hoisted(xh, args.index, out=ob)
        cpu = {"value": (time.perf_counter() - t0) / 2000 * 1e6, "unit": "us per call", "cores": 1,
               "kind": "oracle", "sample": "oracle form 3 (hoisted) at n = 1024, 2000 calls from Python (ctypes), "
                                           "1 thread"}
    head = next(r for r in res if r["n"] == 1024 and r["path"] == "auto")
    value = head.get("c_trusted_back_to_back_us", head["python_us"])
    line = {"metric": "normalize latency per call, configs 1-2 (n=1024 32x32 literal grid; n=2^20+7)",
            "value": value, "unit": "us per call (n=1024, AUTO path, back to back from C, trusted pointers)",
            "n_gpus": 1, "steps": R, "warmup": args.warmup, "higher_is_better": False, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": f"normalize n=1024 and n=2^20+7 fp32 (Fig. 1), {args.index} index, every path",
                       "l2": "device_hot_us: input L2-resident; device_flushed_us: 256 MiB write + 256 MiB read "
                             "before every call inside the graph, flush time subtracted"},
            "results": res, "parity": parity, "cpu_baseline": cpu,
            "gpu_launches": len(res) * R}
    if rank == 0:
        emit(line)


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
        emit(line)


def emit(line):
    """Print the one JSON line (rank 0), with the run metadata (versions) added."""
    if "meta" not in line:
        line["meta"] = run_meta(line.get("n_gpus", 1))
    print(json.dumps(line), flush=True)


def _free_port():
    import socket
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    return port


def self_launch(nproc):
    """`python bench.py --gpus N` without torchrun: re-execute this command under
    torch.distributed.run with N ranks on this node (rendezvous on 127.0.0.1), the
    launch the driver uses for N > 1.  Rank 0's JSON line passes through stdout.
    NCCL's init log (communicator ranks, transports, NVLS) is kept on stderr."""
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(nproc),
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.run(cmd, env=env).returncode


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="libnorm", choices=["libnorm", "reference"])
    ap.add_argument("--workload", default="vector", choices=["vector", "rows", "paths28", "licm", "softmax", "backprop", "small"])
    ap.add_argument("--index", default="literal", choices=["literal", "dense"])
    ap.add_argument("--path", default="auto", choices=["auto", "two_pass", "fused", "small", "mid", "cluster"])
    ap.add_argument("--numel", dest="n", type=int, default=2**32)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--plan", default="balanced", choices=["balanced", "uniform"],
                    help="N > 1 literal shard plan (SURVEY §8(e)): coverage-balanced two-range "
                         "(default) or uniform one-range (rank 0 holds the whole covered prefix)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--also-dense", action="store_true", default=True)
    ap.add_argument("--exchange", default="p2p", choices=["nccl", "nccl-allreduce", "p2p", "host"],
                    help="N > 1: norm_launch_sharded (ncclAllGather), the fused peer-memory "
                         "exchange (norm_launch_sharded_peer), or the two-phase API over the "
                         "torch.distributed process group")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3  # timing rule: >= 3 untimed warm-up steps
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(self_launch(args.gpus))
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
        elif args.workload == "small":
            run_small(args, world, rank, local)
        else:
            run_paths28(args, world, rank, local)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
