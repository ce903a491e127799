"""Summarise an .ncu-rep: key SOL/occupancy metrics, DRAM bytes, top stalled SASS lines."""
import csv
import subprocess
import sys


def run(args):
    return subprocess.run(["ncu", "-i", *args], capture_output=True, text=True).stdout


def main(rep, top=25):
    out = {}
    rows = list(csv.reader(run([rep, "--page", "details", "--csv"]).splitlines()))
    h = rows[0]
    keep = ["Duration", "SM Active Cycles", "Elapsed Cycles", "L2 Cache Throughput", "L1/TEX Cache Throughput",
            "DRAM Throughput", "Executed Ipc Active", "Achieved Occupancy", "Theoretical Occupancy", "L1/TEX Hit Rate",
            "L2 Hit Rate", "Warp Cycles Per Issued Instruction", "Avg. Active Threads Per Warp",
            "Executed Instructions", "Grid Size", "Registers Per Thread", "Block Size"]
    for r in rows[1:]:
        d = dict(zip(h, r))
        if d.get("Metric Name") in keep:
            print(f"{d['Metric Name']:40s} {d['Metric Value']} {d['Metric Unit']}")
            out[d["Metric Name"]] = (d["Metric Value"], d["Metric Unit"])
    raw = list(csv.reader(run([rep, "--page", "raw", "--csv"]).splitlines()))
    hh, uu, vv = raw[0], raw[1], raw[2]
    for n, u, v in zip(hh, uu, vv):
        if n in ("dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum", "smsp__inst_executed.sum"):
            print(f"{n:40s} {v} {u}")
            out[n] = (v, u)
    sass = list(csv.reader(run([rep, "--page", "source", "--csv", "--print-source=sass"]).splitlines()))
    hi = [i for i, r in enumerate(sass) if "Address" in r][0]
    h = sass[hi]
    data = sass[hi + 1:]
    ai, si, wi = h.index("Address"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
    tot = sum(float(r[wi] or 0) for r in data if len(r) > wi)
    print("stall samples", tot)
    order = sorted(range(len(data)), key=lambda k: -float(data[k][wi] or 0))[:top]
    for k in order:
        r = data[k]
        print(f"{float(r[wi]) / tot * 100:5.1f}% {r[ai][-5:]} {r[si][:64]:64s} | prev {data[k - 1][si][:36]}")
    return out


if __name__ == "__main__":
    import contextlib
    import io
    import json

    rep = sys.argv[1]
    buf = io.StringIO()
    with contextlib.redirect_stdout(buf):
        res = main(rep, int(sys.argv[2]) if len(sys.argv) > 2 else 25)
    text = buf.getvalue()
    print(text)
    if len(sys.argv) > 3:  # write profiles/<tag>.txt + .json
        tag = sys.argv[3]
        open(f"profiles/{tag}.txt", "w").write(text)
        def num(k):
            v = res.get(k)
            return float(v[0].replace(",", "")) if v else None
        rd, wr = num("dram__bytes_read.sum"), num("dram__bytes_write.sum")
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        rdu = scale.get(res.get("dram__bytes_read.sum", (0, "byte"))[1], 1)
        wru = scale.get(res.get("dram__bytes_write.sum", (0, "byte"))[1], 1)
        out = {"report": rep, "dram_bytes_per_launch": (rd * rdu + wr * wru) if rd is not None else None,
               "metrics": {k: v for k, v in res.items()}}
        json.dump(out, open(f"profiles/{tag}.json", "w"), indent=1)
