"""Top SASS lines of an `ncu -i rep --page source --csv` export by share of the
warp-stall samples, with each line's dominant stall reasons (the evidence
behind DESIGN.md's "what bounds this kernel" notes).

  python scripts/ncu_top_stalls.py SOURCE_CSV [TOP]"""
import csv
import sys


def main():
    path = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    head, data = rows[hi], rows[hi + 1:]
    isrc = head.index("Source")
    isamp = head.index("Warp Stall Sampling (All Samples)")
    stalls = [(i, h[len("stall_"):]) for i, h in enumerate(head) if h.startswith("stall_") and "Not Issued" not in h]

    def num(x):
        try:
            return float(x.replace(",", ""))
        except ValueError:
            return 0.0
    lines = []
    for r in data:
        if len(r) <= isamp:
            continue
        s = num(r[isamp])
        reasons = sorted(((num(r[i]), n) for i, n in stalls if num(r[i]) > 0), reverse=True)[:3]
        lines.append((s, r[isrc].strip(), reasons))
    tot = sum(s for s, _, _ in lines) or 1.0
    by_reason = {}
    for r in data:
        for i, n in stalls:
            if len(r) > i:
                by_reason[n] = by_reason.get(n, 0.0) + num(r[i])
    print(f"total samples {tot:.0f}")
    print("by reason: " + ", ".join(f"{n} {100 * v / tot:.1f}%" for v, n in
                                    sorted(((v, n) for n, v in by_reason.items()), reverse=True)[:8]))
    for s, src, reasons in sorted(lines, key=lambda t: -t[0])[:top]:
        rs = " ".join(f"{n}={v:.0f}" for v, n in reasons)
        print(f"{100 * s / tot:5.1f}%  {rs:<50} | {src}")


if __name__ == "__main__":
    main()
