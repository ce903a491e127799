"""Per-region totals (warp instructions, thread instructions, stall samples) of an
.ncu-rep, regions = (file, first line, last line) ranges given on the command line
as name=file:a-b; everything else is 'other'."""
import csv
import subprocess
import sys


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                         capture_output=True, text=True).stdout
    fname, hdr = "?", None
    for r in csv.reader(out.splitlines()):
        if r and r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if not hdr or not r or not r[0]:
            continue
        try:
            yield (fname, int(r[0]), float(r[hdr.index("Instructions Executed")]),
                   float(r[hdr.index("Thread Instructions Executed")]),
                   float(r[hdr.index("Warp Stall Sampling (All Samples)")]))
        except (ValueError, IndexError):
            continue


def main(rep, specs):
    regs = []
    for s in specs:
        name, rest = s.split("=")
        f, ab = rest.split(":")
        a, b = ab.split("-")
        regs.append((name, f, int(a), int(b)))
    tot = {}
    for f, ln, ins, thr, st in rows(rep):
        key = "other"
        for name, rf, a, b in regs:
            if f == rf and a <= ln <= b:
                key = name
                break
        t = tot.setdefault(key, [0.0, 0.0, 0.0])
        t[0] += ins
        t[1] += thr
        t[2] += st
    ti = sum(v[0] for v in tot.values()) or 1
    ts = sum(v[2] for v in tot.values()) or 1
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1][2]):
        print(f"{k:14s} ins {v[0] / ti * 100:5.1f}%  {v[1] / max(v[0], 1):5.1f} thr/ins  stall {v[2] / ts * 100:5.1f}%  "
              f"({v[0]:.3e} warp ins)")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2:])
