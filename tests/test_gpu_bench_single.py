"""bench.py at N = 1: the roofline object names the step's dominant kernel and
its bytes: on a two-pass step the reduce (4n) for
the literal index, the scale (8|C| = 8n) for the dense index, each measured with
libnorm's own events around that kernel (norm_debug_set_events)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench(args):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, cwd=ROOT, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


@pytest.mark.parametrize("index", ["literal", "dense"])
def test_roofline_names_dominant_kernel(index):
    n = 2**28  # large enough that launch gaps do not blur the shares (at 2^26 the dense scale measured 0.497-0.6)
    d = _bench(["--index", index, "--numel", str(n), "--path", "two_pass", "--steps", "5", "--warmup", "3",
                "--no-e2e"])  # the parity record is taken in the cpu_baseline leg
    r = d["roofline"]
    assert d["config"]["path"] == "two_pass"
    if index == "dense":
        assert r["kernel"].startswith("scale_tile_kernel"), r["kernel"]
        assert r["algorithmic_bytes_per_launch"] == 8 * n
        assert r["share_of_step"] > 0.5
    else:
        assert r["kernel"].startswith("reduce"), r["kernel"]
        assert r["algorithmic_bytes_per_launch"] == 4 * n
        assert r["share_of_step"] > 0.5  # dominant (0.69-0.8 at 2^26, where launch costs weigh; 0.93 at 2^32)
    assert 0 < r["avg_launch_ms"] < d["ms_per_step"] * 1.05
    assert d["parity"]["ok"]


def test_throttled_region_is_remeasured_once():
    """Timing rule: a timed region that saw hw_slowdown (injected here) is
    re-measured once; the line records the first attempt and reports the second."""
    os.environ["NORM_BENCH_FAKE_THROTTLE"] = "1"
    try:
        d = _bench(["--numel", str(2**26), "--path", "two_pass", "--steps", "3", "--warmup", "3",
                    "--no-e2e", "--no-cpu", "--no-parity"])
    finally:
        os.environ.pop("NORM_BENCH_FAKE_THROTTLE", None)
    r = d["remeasured"]
    assert "hw_slowdown" in r["first_reasons_rank0"] and r["first_ms_per_step"] > 0
    assert d["ms_per_step"] > 0


@pytest.mark.parametrize("workload", ["rows", "softmax"])
def test_large_row_workloads_follow_the_vector_timing_rule(workload):
    """65536 x 4096 fp32 = 1 GiB of input >= 4 x L2: timed back to back like the
    vector workload, with the flushed per-call ("isolated") time beside it."""
    d = _bench(["--workload", workload, "--steps", "5", "--warmup", "3"])
    assert "no flush" in d["config"]["l2"], d["config"]["l2"]
    iso = d["isolated"]["ms_per_step"] if workload == "rows" else d["results"]["softmax"]["isolated_ms"]
    # back to back hides the launch latency and ramp; it cannot be much slower than a cold call
    assert 0 < d["ms_per_step"] < iso * 1.05, (d["ms_per_step"], iso)
