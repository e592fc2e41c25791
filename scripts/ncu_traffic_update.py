"""Record `dram__bytes_read.sum + dram__bytes_write.sum` per launch of a
workload's dominant kernel into profiles/ncu_traffic.json, bound to a SHA-256 of
the kernel's source files so that bench.py reports `roofline.traffic` only while
the captured kernel is still the one it times (else null + a "stale" note).

  python scripts/ncu_traffic_update.py KEY RAW_CSV KERNEL_REGEX [--capture DESC]

KEY is "<workload>:<index>" as bench.py asks for it (e.g. vector:literal);
RAW_CSV an `ncu -i rep --page raw --csv` export; KERNEL_REGEX selects the rows
(launches) to average."""
import argparse
import csv
import json
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import TRAFFIC_SOURCES, sources_sha256  # noqa: E402

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def per_launch_bytes(path, kregex):
    rows = list(csv.reader(open(path)))
    head, units, data = rows[0], rows[1], rows[2:]
    ik = head.index("Kernel Name")
    cols = [head.index("dram__bytes_read.sum"), head.index("dram__bytes_write.sum")]
    tot, k = 0.0, 0
    for r in data:
        if not re.search(kregex, r[ik]):
            continue
        tot += sum(float(r[c].replace(",", "")) * UNIT[units[c]] for c in cols)
        k += 1
    if not k:
        raise SystemExit(f"no launch of /{kregex}/ in {path}")
    return int(round(tot / k)), k


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("key")
    ap.add_argument("raw_csv")
    ap.add_argument("kernel_regex")
    ap.add_argument("--capture", default="")
    ap.add_argument("--json", default=os.path.join(ROOT, "profiles", "ncu_traffic.json"),
                    help="file to update (on the GPU box: one under gpurun_out/, copied back)")
    a = ap.parse_args()
    wl = a.key.split(":")[0]
    if wl not in TRAFFIC_SOURCES:
        raise SystemExit(f"unknown workload {wl}: add its source files to bench.TRAFFIC_SOURCES")
    b, k = per_launch_bytes(a.raw_csv, a.kernel_regex)
    p = a.json
    d = json.load(open(p)) if os.path.exists(p) else {}
    d[a.key] = {"bytes": b, "launches_averaged": k, "kernel_regex": a.kernel_regex,
                "csv": os.path.relpath(os.path.abspath(a.raw_csv), ROOT), "capture": a.capture,
                "sources": TRAFFIC_SOURCES[wl], "sources_sha256": sources_sha256(TRAFFIC_SOURCES[wl])}
    json.dump(d, open(p, "w"), indent=1, sort_keys=True)
    print(a.key, b, f"({k} launches)")


if __name__ == "__main__":
    main()
