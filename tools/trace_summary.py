"""Summarise a frame trace written by bench.py (CINR_TRACE=...): per iteration the
barrier spread, scan time and phase completion spread over CTAs, and the time
split by iteration size."""
import json
import sys

import numpy as np


def main(path):
    d = json.load(open(path))
    bar, scan, ph = (np.array(d[k], dtype=np.int64) for k in ("bar", "scan", "phase"))
    n = np.array(d["samples"])
    K = d["iters"]
    # absolute iteration length is not recorded; phase max + next barrier ~ iteration
    print(f"iters {K}  rays {d['rays']}  samples {n.sum()}")
    for k in [0, 1, 5, 10, 20, 40, 60, 80, 100, 120, 150, 180, 200]:
        if k >= K:
            break
        print(f"k={k:3d} n={n[k]:7d}  scan med {np.median(scan[k]):6.0f}  phase min/med/max "
              f"{ph[k].min():7d}/{np.median(ph[k]):7.0f}/{ph[k].max():7d}")
    ph_max = ph.max(axis=1)
    sc_med = np.median(scan, axis=1)
    for lo, hi in [(0, 1000), (1000, 10000), (10000, 100000), (100000, 1e9)]:
        m = (n[:K] >= lo) & (n[:K] < hi)
        print(f"n in [{lo},{hi}): iters {m.sum():3d}  sum(phase max) {ph_max[m].sum() / 1e3:7.0f} us  "
              f"sum(scan) {sc_med[m].sum() / 1e3:6.0f} us  samples {n[:K][m].sum()}")


if __name__ == "__main__":
    for p in sys.argv[1:]:
        main(p)
