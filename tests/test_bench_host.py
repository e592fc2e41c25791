"""Host-side logic of bench.py (CPU): the local covered-prefix rule that picks
the kernel the bench's roofline names must agree with the shard plans."""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import paper_2207_00257_b200 as L  # noqa: E402


@pytest.mark.parametrize("n", [2**32, 2**28 + 77, 5000, 2**20 + 7])
@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_local_covered_prefix_matches_plans(n, world):
    count, prefix = L.coverage(n, "literal")
    for balanced in (True, False):
        plan = L.plan_shards(n, world, "literal", balanced)
        total = 0
        for ranges in plan:
            lloc = bench.local_covered_prefix(ranges, prefix)
            covered = sum(max(0, min(b + ln, prefix) - b) for b, ln in ranges)
            # literal coverage is a global prefix: every plan keeps it a local prefix
            assert lloc == covered
            total += covered
        assert total == count
    # dense: everything covered, the whole local buffer
    _, dprefix = L.coverage(n, "dense")
    for ranges in L.plan_shards(n, world, "dense", True):
        assert bench.local_covered_prefix(ranges, dprefix) == sum(ln for _, ln in ranges)


def test_local_covered_prefix_rejects_gaps():
    # covered elements after uncovered ones (in local order) are not a local prefix
    assert bench.local_covered_prefix([(100, 10), (0, 5)], 50) == -1
    assert bench.local_covered_prefix([(0, 10), (20, 5)], 12) == 10  # 10, 11 live on another rank
    # two fully covered ranges concatenate into one local prefix
    assert bench.local_covered_prefix([(0, 10), (20, 5)], 50) == 15
    assert bench.local_covered_prefix([(0, 10), (10, 5)], 12) == 12
    assert bench.local_covered_prefix([(0, 4)], -1) == -1


def test_reference_arm_json_contract():
    """`bench.py --impl reference` (the oracle on the host cores) prints one JSON
    line with the libnorm arm's metric, unit, direction and workload name."""
    import json
    import subprocess
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "3"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference"
    assert d["metric"] == "normalize GB/s and % of HBM peak, n=2^32 fp32, at 1/2/4/8 B200"
    assert d["unit"] == "GB/s" and d["higher_is_better"] is True and d["value"] > 0
    assert d["config"]["workload"] == bench.workload_name(2**32, "literal")
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["value"] == d["value"]
    assert d["cpu_baseline"]["cores"] == os.cpu_count()
    assert d["e2e"] == {"value": d["value"], "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


def test_reference_arm_loads_no_product_library():
    """The reference arm (the oracle) never maps libnorm.so: run it in-process and
    read this process's own memory map afterwards."""
    import subprocess
    code = ("import runpy, sys; sys.argv = ['bench.py', '--impl', 'reference', '--steps', '1', '--warmup', '3'];"
            "runpy.run_path('bench.py', run_name='__main__');"
            "print('MAPS', sorted({l.split()[-1] for l in open('/proc/self/maps') if l.strip().endswith('.so')}))")
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    maps = [ln for ln in r.stdout.splitlines() if ln.startswith("MAPS")][0]
    assert "liboracle.so" in maps and "libnormgen.so" in maps
    assert "libnorm.so" not in maps.replace("libnormgen", "")


def test_plain_launch_self_execs_two_ranks():
    """`python bench.py --gpus 2` without torchrun re-executes itself under
    torch.distributed.run (the driver may call it either way); rank 0 alone prints
    one JSON line.  The reference arm runs on CPU, so this covers the launcher here."""
    import json
    import subprocess
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2",
                        "--steps", "1", "--warmup", "3"], capture_output=True, text=True, timeout=900, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["meta"]["world_size"] == 2


def test_traffic_bound_to_kernel_sources(tmp_path, monkeypatch):
    """roofline.traffic is reported only while the kernel sources hash to the value
    recorded at ncu capture time; any edit to them makes it null (stale)."""
    import json
    import shutil
    root = tmp_path / "r"
    for f in set(sum(bench.TRAFFIC_SOURCES.values(), [])):
        (root / os.path.dirname(f)).mkdir(parents=True, exist_ok=True)
        shutil.copy(os.path.join(ROOT, f), root / f)
    (root / "profiles").mkdir()
    src = bench.TRAFFIC_SOURCES["vector"]
    monkeypatch.setattr(bench, "ROOT", str(root))
    e = {"bytes": 123, "sources": src, "sources_sha256": bench.sources_sha256(src)}
    (root / "profiles" / "ncu_traffic.json").write_text(json.dumps({"vector:literal": e, "rows:dense": 7}))
    assert bench.load_traffic("vector", "literal") == 123
    assert bench.load_traffic("rows", "dense") is None       # no hash: not trusted
    assert bench.load_traffic("softmax", "dense") is None    # no capture
    with open(root / src[0], "a") as f:
        f.write("\n// edited\n")
    assert bench.load_traffic("vector", "literal") is None   # source changed since capture
