"""The N > 1 path as the driver's scaling run launches it: one process per GPU,
NCCL process group, each rank on its own device.

Every other multi-process test puts all ranks on cuda:0 over gloo (NCCL refuses
two ranks on one device), so cross-device CUDA IPC mapping, system-scope peer
stores over NVLink and the NCCL exchanges at W > 1 run only here.  Skipped on a
box with fewer than two GPUs (this project's GPU allocation is one B200); on a
multi-GPU node it checks, before the driver's scaling run depends on it, that:
  * the fused peer-memory exchange is used with no fallback note,
  * the NCCL all-gather and the north_star's NCCL all-reduce of the scalar both
    run and give a value,
  * the divisor is the same on every rank and within 1e-6 of the oracle's exact
    sum, through both the peer exchange and NCCL (examples/sharded_normalize.py)."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _gpus():
    try:
        import torch
        return torch.cuda.device_count()
    except Exception:  # noqa: BLE001
        return 0


needs_two = pytest.mark.skipif(_gpus() < 2, reason="needs >= 2 GPUs (one process per GPU over NCCL)")


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _torchrun(script_args, nproc, timeout=900):
    env = dict(os.environ)
    for k in ("NORM_BENCH_BACKEND", "NORM_BENCH_DEVICE", "WORLD_SIZE", "RANK", "LOCAL_RANK"):
        env.pop(k, None)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(nproc),
           "--master-addr", "127.0.0.1", "--master-port", str(_port())] + script_args
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=timeout)
    assert r.returncode == 0, r.stderr[-4000:]
    return r


@needs_two
@pytest.mark.parametrize("index", ["literal", "dense"])
def test_bench_one_process_per_gpu(index):
    n = 2**28 + 7
    r = _torchrun([os.path.join(ROOT, "bench.py"), "--gpus", "2", "--numel", str(n), "--index", index,
                   "--steps", "5", "--warmup", "3", "--e2e-steps", "1"], 2)
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-4000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0
    assert d["config"]["exchange"] == "p2p"
    assert d["config"]["exchange_note"] is None, d["config"]["exchange_note"]
    ex = d["exchanges"]
    for name in ("nccl-allreduce", "nccl", "host"):
        assert "unavailable" not in ex[name], ex[name]
        assert ex[name]["value"] > 0 and ex[name]["rank_ms_max"] >= ex[name]["rank_ms_min"] > 0
    assert d["nccl_allreduce"]["exchange"] == "nccl-allreduce"
    lat = d["exchange_latency"]
    for name in ("p2p", "nccl-allreduce", "nccl"):
        assert lat[name].get("us_per_step_max", 0) > 0, lat


@needs_two
@pytest.mark.parametrize("exchange", ["p2p", "nccl"])
def test_sharded_example_one_process_per_gpu(exchange):
    """examples/sharded_normalize.py on two devices, peer exchange and NCCL: the
    divisor is identical on both ranks and within 1e-6 of the oracle's exact sum
    of the same seeded input (regenerated on the host)."""
    import re

    import numpy as np

    import gen
    import oracle
    n = 2**24 + 7
    r = _torchrun([os.path.join(ROOT, "examples", "sharded_normalize.py"), "--numel", str(n),
                   "--exchange", exchange], 2)
    m = re.search(r"s=([0-9.e+-]+) identical on every rank: (True|False)", r.stdout)
    assert m, r.stdout[-2000:]
    assert m.group(2) == "True"
    x = np.empty(n, dtype=np.float32)
    gen.fill_host(x, seed=7, dist="unit")
    S = oracle.sum_exact(x)
    assert abs(float(m.group(1)) - S) <= 1e-6 * abs(S), (m.group(1), S)
