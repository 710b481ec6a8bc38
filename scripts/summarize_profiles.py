"""Turn the raw ncu outputs of scripts/profile_round.sh (gpurun_out/) into the tracked summaries
under profiles/.  usage: python scripts/summarize_profiles.py TAG"""
import collections
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TAG = sys.argv[1] if len(sys.argv) > 1 else "r1"
OUT = os.path.join(ROOT, "profiles")
os.makedirs(OUT, exist_ok=True)


def short(name):
    n = name.split("(")[0].replace("void ", "")
    return n.split("::")[-1] if "lora" in n else n[:70]


def launches():
    path = os.path.join(ROOT, "gpurun_out", "launches_%s.csv" % TAG)
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ix = {n: i for i, n in enumerate(h)}
    per = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) < len(h):
            continue
        key = (r[ix["ID"]], short(r[ix["Kernel Name"]]))
        d = per.setdefault(key, {})
        unit = r[ix["Metric Unit"]]
        v = float(r[ix["Metric Value"]].replace(",", ""))
        scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6,
                 "Gbyte": 1e9}.get(unit, 1.0)
        d[r[ix["Metric Name"]]] = v * scale
    with open(os.path.join(OUT, "%s_launches.csv" % TAG), "w") as fh:
        fh.write("id,kernel,duration_us,dram_read_bytes,dram_write_bytes\n")
        for (kid, name), d in per.items():
            fh.write("%s,%s,%.3f,%.0f,%.0f\n" % (kid, name, d.get("gpu__time_duration.sum", 0),
                                                  d.get("dram__bytes_read.sum", 0), d.get("dram__bytes_write.sum", 0)))
    agg = collections.OrderedDict()
    for (kid, name), d in per.items():
        a = agg.setdefault(name, [0, 0.0, 0.0, 0.0])
        a[0] += 1
        a[1] += d.get("gpu__time_duration.sum", 0)
        a[2] += d.get("dram__bytes_read.sum", 0)
        a[3] += d.get("dram__bytes_write.sum", 0)
    tot = sum(a[1] for a in agg.values())
    lines = ["ncu launch list (--clock-control none, serialised, cold caches: compare SHARES, not absolutes)",
             "command: bench.py --layers 4 --steps 10 --prefill-layers 1 --c4-steps 0 --c5-reps 0 (scripts/profile_round.sh)", "",
             "%-34s %6s %10s %8s %14s %14s" % ("kernel", "count", "mean_us", "share", "dram_rd/launch", "dram_wr/launch")]
    for name, (n, t, rd, wr) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append("%-34s %6d %10.2f %7.1f%% %14.0f %14.0f" % (name, n, t / n, 100 * t / tot, rd / n, wr / n))
    open(os.path.join(OUT, "%s_launch_summary.txt" % TAG), "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))
    return agg


def full(kind):
    rep = os.path.join(ROOT, "gpurun_out", "prof_%s_%s.ncu-rep" % (kind, TAG))
    out = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "ncu_summary.py"), rep, "--sass", "0",
                          "--json", os.path.join(OUT, "%s_ncu_%s.json" % (TAG, kind))],
                         capture_output=True, text=True).stdout
    open(os.path.join(OUT, "%s_ncu_%s.txt" % (TAG, kind)), "w").write(
        "ncu --set full --clock-control none (one capture; kernel in isolation)\n\n" + out)
    return json.load(open(os.path.join(OUT, "%s_ncu_%s.json" % (TAG, kind))))


if __name__ == "__main__":
    agg = launches()
    dec = full("decode")
    pf = full("prefill")
    if os.path.exists(os.path.join(ROOT, "gpurun_out", "prof_fused_%s.ncu-rep" % TAG)):
        full("fused")
    # decode capture = one c2 layer step (scripts/ncu_decode_step.py): the q/k/v lora_apply_multi pair and
    # the o pair, i.e. 4 projection applies -> DRAM bytes per projection apply for bench.py's roofline
    rd = lambda v: v.get("dram__bytes_read.sum", 0) + v.get("dram__bytes_write.sum", 0)  # noqa  (bytes)
    dec_k = [v for v in dec.values() if "shrink" in v["name"] or "expand" in v["name"]]
    summ = {"tag": TAG,
            "dram_bytes_per_launch": round(sum(map(rd, dec_k)) / 4) if len(dec_k) == 4 else None,
            "decode_kernels_captured": [v["name"] for v in dec_k],
            "note": "DRAM bytes per projection apply = (q/k/v lora_apply_multi pair + o pair) / 4, ncu --set full, "
                    "cold caches; writes to y can remain in L2 at kernel end",
            "prefill_dram_bytes_per_launch": round(sum(map(rd, pf.values())) / len(pf)) if pf else None}
    json.dump(summ, open(os.path.join(OUT, "ncu_decode_summary.json"), "w"), indent=1)
    print(summ)
