"""bench.py's N > 1 path end to end: `torch.distributed.run --nproc-per-node 2
bench.py --gpus 2`, the launch the driver uses for the scaling run, with both
ranks on the one GPU of this box (gloo process group, NORM_BENCH_BACKEND=gloo:
NCCL refuses two ranks on one device).  Checks that rank 0 prints exactly one
JSON line with the contract's keys, that the fused peer-memory exchange was used
(no NCCL fallback note), and that the other rank prints nothing."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _torchrun(args, timeout=600):
    env = dict(os.environ, NORM_BENCH_BACKEND="gloo", NORM_BENCH_DEVICE="0")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "bench.py"),
           "--gpus", "2"] + args
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=timeout)
    assert r.returncode == 0, r.stderr[-4000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-4000:]
    return json.loads(lines[0]), r


@pytest.mark.parametrize("exchange,n,plan", [("p2p", 2**24 + 7, "balanced"), ("host", 2**24 + 7, "balanced"),
                                             ("p2p", 2**27 + 7, "balanced"), ("p2p", 2**27 + 7, "uniform")])
def test_bench_vector_two_ranks(exchange, n, plan):
    d, r = _torchrun(["--numel", str(n), "--steps", "3", "--warmup", "3", "--exchange", exchange,
                      "--e2e-steps", "1", "--plan", plan])
    assert d["config"]["shard_plan"].startswith("coverage-balanced" if plan == "balanced" else "uniform")
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches",
              "clocks"):
        assert k in d, k
    assert d["n_gpus"] == 2 and d["steps"] == 3 and d["value"] > 0
    assert d["config"]["exchange"] == exchange
    assert d["config"]["exchange_note"] is None, d["config"]["exchange_note"]
    assert d["e2e"]["h2d_bytes_per_step"] == 4 * n
    # each rank's local input exceeds L2 at 2^27: the peer path runs one fused kernel per rank
    assert ("fused_kernel" in d["roofline"]["kernel"]) == (exchange == "p2p" and n > 2**26)
    one = any(k in d["roofline"]["kernel"] for k in ("fused_kernel", "mid_kernel", "cluster_kernel"))
    assert d["gpu_launches"] == d["steps"] * (1 if one else 2)
    assert "cpu_baseline" not in d or d["cpu_baseline"] is None  # rank 0 at N = 1 only
    other = d["other_shard_plan"]  # both literal shard plans measured in one run
    assert other["plan"].startswith("uniform" if plan == "balanced" else "coverage-balanced"), other
    assert other["value"] > 0 and other["rank_ms_max"] >= other["rank_ms_min"] > 0


def test_bench_rows_two_ranks():
    d, _ = _torchrun(["--workload", "rows", "--steps", "3", "--warmup", "3"])
    assert d["n_gpus"] == 2 and d["value"] > 0


def test_bench_reference_two_ranks():
    """--impl reference under torchrun: rank 0 alone times the oracle and prints."""
    d, _ = _torchrun(["--impl", "reference", "--steps", "1", "--warmup", "3"])
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0


def test_bench_plain_python_launch_two_ranks():
    """`python bench.py --gpus 2` with no torchrun: bench.py re-executes itself under
    torch.distributed.run; one JSON line from rank 0, the peer exchange used, the
    other exchanges' records present (NCCL ones marked not run under the one-GPU
    gloo emulation), the exchange latency record, and the run metadata."""
    env = dict(os.environ, NORM_BENCH_BACKEND="gloo", NORM_BENCH_DEVICE="0")
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK"):
        env.pop(k, None)
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--numel", str(2**24 + 7),
           "--steps", "3", "--warmup", "3", "--e2e-steps", "1"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-4000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-4000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["exchange"] == "p2p" and d["config"]["exchange_note"] is None
    assert "host" in d["exchanges"] and d["exchanges"]["host"]["value"] > 0
    assert "NCCL" in d["exchanges"]["note"]
    lat = d["exchange_latency"]
    assert lat["p2p"]["us_per_step_max"] > 0 and lat["host"]["us_per_step_max"] > 0
    assert d["meta"]["world_size"] == 2 and d["meta"]["torch"]
    assert d["step_stats"]["rank_ms_max"] >= d["step_stats"]["rank_ms_min"] > 0
    # 2^24 + 7 elements split over 2 ranks: 32 MiB per rank < 4 x L2 -> flushed
    assert "flushed" in d["config"]["l2"]


def test_bench_p2p_failure_on_one_rank_falls_back_everywhere():
    """A peer-exchange failure seen by ONE rank (injected on rank 1 after the
    cross-check) must move every rank to the same fallback exchange through the
    same collectives (no rank left waiting in a collective the other skipped):
    one JSON line, the fallback named in exchange_note, and a valid step."""
    env_extra = {"NORM_BENCH_FAULT_P2P_RANK": "1"}
    old = {k: os.environ.get(k) for k in env_extra}
    os.environ.update(env_extra)
    try:
        d, _ = _torchrun(["--numel", str(2**24 + 7), "--steps", "3", "--warmup", "3", "--e2e-steps", "1"],
                         timeout=300)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    note = d["config"]["exchange_note"]
    assert note and "rank 1: injected fault" in note and "fell back to host" in note, note
    assert d["config"]["exchange"] == "host"
    assert d["n_gpus"] == 2 and d["value"] > 0


def test_sharded_example_two_ranks():
    """examples/sharded_normalize.py (the README's multi-GPU usage) under
    torch.distributed.run with 2 ranks on this GPU: the same divisor on both."""
    env = dict(os.environ, NORM_EXAMPLE_BACKEND="gloo", NORM_EXAMPLE_DEVICE="0")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()),
           os.path.join(ROOT, "examples", "sharded_normalize.py"), "--numel", str(2**24 + 7)]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-3000:]
    assert "identical on every rank: True" in r.stdout, r.stdout[-2000:]
