"""Classify every compute-sanitizer racecheck report into the documented
patterns (profiles/r05/sanitize_r05.md), by the source text at
the reported lines.  Usage: python scripts/racecheck_classify.py sanitize_racecheck.log

Reads both report shapes racecheck prints:
  analysis: "Race reported between <T> access at <fn>+0x.. in file:line" followed by
            "and <T> access at ... in file:line [N hazards]" lines
  hazard:   "Potential <RAW|WAR|WAW> hazard detected at __shared__ ..." followed by
            "<T> Thread (..) at ... in file:line:fn" lines
Exit status 1 if any report falls outside the documented patterns."""
import collections
import glob
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC_DIRS = [os.path.join(ROOT, "paper_2207_00257_b200", "csrc"), os.path.join(ROOT, "gen")]

PATTERNS = [
    ("P1 TMA refill vs earlier ld.shared (mbarrier release/acquire + proxy fence)",
     lambda txt: any("cp.async.bulk" in t or "bulk_g2s" in t or "bulk_copy" in t or "bulk_s2g" in t
                     for t in txt)),
    ("P2 stage tag written before expect_tx, read after try_wait (mbarrier-ordered)",
     lambda txt: any("stage_chunk" in t for t in txt)),
    ("P3 warp-sum slot hand-off by fence + atomic counter",
     lambda txt: any("slot[" in t for t in txt)),
]

LOC = re.compile(r"in ([\w./-]+\.(?:cu|cuh|h|cpp)):(\d+)")
START = re.compile(r"(Race reported between|hazard detected)")


def source_line(fname, line):
    base = os.path.basename(fname)
    for d in SRC_DIRS:
        for p in glob.glob(os.path.join(d, base)):
            with open(p) as f:
                lines = f.readlines()
            if 0 < line <= len(lines):
                return lines[line - 1].strip()
    return "?"


def parse(path):
    recs, cur = [], None
    with open(path, errors="replace") as f:
        for ln in f:
            if START.search(ln):
                if cur:
                    recs.append(cur)
                cur = {"head": ln.strip(), "locs": [], "hazards": 0, "fns": set()}
            if cur is None:
                continue
            for m in re.finditer(r"(?:at|:)\s*(?:[\w:<>(), &*]*?)(lnorm::\w+|\w+_kernel\w*)", ln):
                cur["fns"].add(m.group(1))
            for m in LOC.finditer(ln):
                cur["locs"].append((os.path.basename(m.group(1)), int(m.group(2))))
            h = re.search(r"\[(\d+) hazards?\]", ln)
            if h:
                cur["hazards"] += int(h.group(1))
            if "RACECHECK SUMMARY" in ln:
                recs.append(cur)
                cur = None
    if cur:
        recs.append(cur)
    return recs


def main(path):
    recs = parse(path)
    groups = collections.OrderedDict()
    for r in recs:
        key = tuple(sorted(set(r["locs"])))
        g = groups.setdefault(key, {"reports": 0, "hazards": 0, "kind": r["head"][:60], "fns": set()})
        g["fns"] |= r["fns"]
        g["reports"] += 1
        g["hazards"] += max(r["hazards"], 1)
    by_pat = collections.Counter()
    unclassified = 0
    print(f"{len(recs)} reports in {len(groups)} distinct location sets ({path})\n")
    for key, g in groups.items():
        txt = [source_line(f, l) for f, l in key]
        pat = next((name for name, pred in PATTERNS if pred(txt + sorted(g["fns"]))), None)
        if pat is None:
            unclassified += g["reports"]
            pat = "UNCLASSIFIED"
        by_pat[pat] += g["reports"]
        print(f"[{pat}] reports={g['reports']} hazards={g['hazards']} in {', '.join(sorted(g['fns']))}")
        for (f, l), t in zip(key, txt):
            print(f"    {f}:{l}: {t}")
    print("\nper pattern:")
    for p, c in by_pat.items():
        print(f"  {c:6d}  {p}")
    summ = [ln.strip() for ln in open(path, errors="replace") if "SUMMARY" in ln]
    print("\n" + "\n".join(summ))
    return 1 if unclassified else 0


if __name__ == "__main__":
    sys.exit(main(sys.argv[1]))
