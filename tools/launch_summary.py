"""Per-kernel totals from an ncu `--metrics gpu__time_duration.sum --csv` launch list:
launches, total and mean duration, share of all kernel time."""
import csv
import sys
from collections import defaultdict


def main(path, out=None):
    rows = [r for r in csv.reader(open(path)) if r]
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    ui = h.index("Metric Unit") if "Metric Unit" in h else None
    tot = defaultdict(lambda: [0, 0.0])
    for r in rows[hi + 1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        v = float(r[vi].replace(",", ""))
        unit = r[ui] if ui is not None else "nsecond"
        v *= {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "second": 1e6}.get(unit, 1e-3)
        name = r[ki].split("(")[0]
        tot[name][0] += 1
        tot[name][1] += v
    allus = sum(t for _, t in tot.values())
    lines = [f"{'kernel':60s} {'launches':>8s} {'total us':>12s} {'mean us':>10s} {'share':>7s}"]
    for name, (n, t) in sorted(tot.items(), key=lambda x: -x[1][1]):
        lines.append(f"{name[:60]:60s} {n:8d} {t:12.1f} {t / n:10.1f} {t / allus * 100:6.1f}%")
    lines.append(f"{'all kernels':60s} {sum(n for n, _ in tot.values()):8d} {allus:12.1f}")
    text = "\n".join(lines)
    print(text)
    if out:
        open(out, "w").write(text + "\n")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None)
