"""Per-CUDA-source-line totals of an .ncu-rep: instructions executed (warp and thread
level) and warp stall samples, from the `--print-source=cuda,sass` source page."""
import csv
import subprocess
import sys


def main(rep, top=30):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                         capture_output=True, text=True).stdout
    res, fname, hdr = [], "?", None
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
            ins = float(r[hdr.index("Instructions Executed")])
            thr = float(r[hdr.index("Thread Instructions Executed")])
            st = float(r[hdr.index("Warp Stall Sampling (All Samples)")])
        except (ValueError, IndexError):
            continue
        res.append((ins, thr, st, f"{fname}:{r[0]}", r[1].strip()[:80]))
    ti = sum(x[0] for x in res) or 1
    tt = sum(x[1] for x in res) or 1
    ts = sum(x[2] for x in res) or 1
    print(f"warp instr {ti:.3e}  thread instr {tt:.3e}  stall samples {ts:.0f}")
    for title, key in (("instructions", 0), ("stall samples", 2)):
        print(f"--- top lines by {title}")
        for x in sorted(res, key=lambda x: -x[key])[:top]:
            print(f"{x[0] / ti * 100:5.1f}% ins {x[1] / max(x[0], 1):5.1f} thr/ins {x[2] / ts * 100:5.1f}% stall  "
                  f"{x[3]:18s} {x[4]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)


def by_ranges(rep, ranges):
    """Sum instructions / stall samples over named (file, first, last) line ranges."""
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                         capture_output=True, text=True).stdout
    tot = {name: [0.0, 0.0] for name in ranges}
    fname, hdr, ti, ts = "?", None, 0.0, 0.0
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
            ins = float(r[hdr.index("Instructions Executed")])
            st = float(r[hdr.index("Warp Stall Sampling (All Samples)")])
            line = int(r[0])
        except (ValueError, IndexError):
            continue
        ti += ins
        ts += st
        for name, (f, a, b) in ranges.items():
            if fname == f and a <= line <= b:
                tot[name][0] += ins
                tot[name][1] += st
    for name, (i, s) in tot.items():
        print(f"{name:24s} {i / ti * 100:5.1f}% instr  {s / ts * 100:5.1f}% stall")
