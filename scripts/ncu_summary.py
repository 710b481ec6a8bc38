"""Summarise an ncu --set full report: key metrics per profiled kernel, and optionally the
hottest SASS of one kernel (by stall samples) with its executed-instruction counts.
usage: python scripts/ncu_summary.py REPORT.ncu-rep [--sass KERNEL_ID] [--json OUT]"""
import csv
import io
import json
import subprocess
import sys

WANT = ["Duration", "DRAM Throughput", "Memory Throughput", "Registers Per Thread", "Achieved Occupancy",
        "Executed Instructions", "Issue Slots Busy", "L2 Hit Rate", "Elapsed Cycles", "SM Active Cycles",
        "Grid Size", "Dynamic Shared Memory Per Block", "Compute (SM) Throughput"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
       "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
       "sm__inst_executed_pipe_tensor.sum", "lts__t_bytes.sum"]


def _csv(args):
    out = subprocess.run(["ncu", "-i"] + args + ["--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def _f(v):
    try:
        return float(v.replace(",", ""))
    except ValueError:
        return 0.0


def main():
    rep = sys.argv[1]
    rows = _csv([rep, "--page", "details"])
    h = rows[0]
    ix = {n: i for i, n in enumerate(h)}
    kern = {}
    for r in rows[1:]:
        if len(r) <= ix["Metric Value"]:
            continue
        k = kern.setdefault(r[ix["ID"]], {"name": r[ix["Kernel Name"]]})
        if r[ix["Metric Name"]] in WANT:
            k[r[ix["Metric Name"]]] = r[ix["Metric Value"]] + " " + r[ix["Metric Unit"]]
    raw = _csv([rep, "--page", "raw"])
    if raw:
        hr = raw[0]
        rix = {n: i for i, n in enumerate(hr)}
        units = raw[1] if len(raw) > 1 else [""] * len(hr)
        scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        for r in raw[2:]:
            if len(r) != len(hr):
                continue
            k = kern.get(r[rix["ID"]])
            if k is None:
                continue
            for m in RAW:
                if m in rix:
                    # byte counters are stored in bytes (ncu picks a unit per value)
                    k[m] = _f(r[rix[m]]) * scale.get(units[rix[m]], 1.0) if "bytes" in m else _f(r[rix[m]])
    for kid, k in kern.items():
        print("[%s] %s" % (kid, k["name"][:110]))
        for m in WANT + RAW:
            if m in k:
                print("      %-62s %s" % (m, k[m]))
    if "--json" in sys.argv:
        json.dump(kern, open(sys.argv[sys.argv.index("--json") + 1], "w"), indent=1)
    if "--sass" in sys.argv:
        kid = sys.argv[sys.argv.index("--sass") + 1]
        src = _csv([rep, "--page", "source", "--print-source", "sass", "--kernel-id", "::" + kid]) if False else \
            _csv([rep, "--page", "source", "--print-source", "sass"])
        # sections: one per kernel, each starting with a "Kernel Name" row
        sec, cur = [], None
        for r in src:
            if r and r[0] == "Kernel Name":
                cur = []
                sec.append(cur)
            elif cur is not None:
                cur.append(r)
        s = sec[int(kid)]
        hh = s[0]
        jx = {n: i for i, n in enumerate(hh)}
        data = [r for r in s[1:] if len(r) == len(hh)]
        samp = "Warp Stall Sampling (All Samples)"
        tot = sum(_f(r[jx[samp]]) for r in data) or 1
        cols = [c for c in hh if c.startswith("stall_") and "Not Issued" not in c]
        agg = {c: sum(_f(r[jx[c]]) for r in data) for c in cols}
        print("stall breakdown:", ", ".join("%s %.0f%%" % (c[6:], 100 * v / tot)
                                            for c, v in sorted(agg.items(), key=lambda kv: -kv[1])[:8]))
        for r in sorted(data, key=lambda r: -_f(r[jx[samp]]))[:30]:
            top = sorted(((c, _f(r[jx[c]])) for c in cols), key=lambda kv: -kv[1])[:2]
            print("%5.1f%% exec=%-7d %-58s %s" % (100 * _f(r[jx[samp]]) / tot, _f(r[jx["Instructions Executed"]]),
                                                  r[jx["Source"]][:58], " ".join("%s=%d" % (c[6:], v) for c, v in top)))


if __name__ == "__main__":
    main()
