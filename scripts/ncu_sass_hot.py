"""Summarise an ncu --page source --print-source sass CSV: top instructions by stall samples
and the aggregate stall-reason breakdown.  usage: python scripts/ncu_sass_hot.py file.csv [N]"""
import csv
import sys

def _f(v):
    try:
        return float(v.replace(",", ""))
    except ValueError:
        return 0.0


rows = list(csv.reader(open(sys.argv[1])))
N = int(sys.argv[2]) if len(sys.argv) > 2 else 25
hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
h = rows[hdr_i]
ix = {n: i for i, n in enumerate(h)}
data = []
for r in rows[hdr_i + 1:]:
    if r and r[0] in ("Address", "Kernel Name"):
        break          # next kernel section: summarise the first one only
    if len(r) == len(h):
        data.append(r)
samp = "Warp Stall Sampling (All Samples)"
tot = sum(_f(r[ix[samp]]) for r in data)
stall_cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
agg = {c: sum(_f(r[ix[c]]) for r in data) for c in stall_cols}
print("total samples", tot)
for c, v in sorted(agg.items(), key=lambda kv: -kv[1])[:10]:
    print("  %-28s %6.1f%%" % (c, 100 * v / max(tot, 1)))
print()
for r in sorted(data, key=lambda r: -_f(r[ix[samp]]))[:N]:
    top = sorted(((c, _f(r[ix[c]])) for c in stall_cols), key=lambda kv: -kv[1])[:2]
    print("%6.1f%%  %-60s %s" % (100 * _f(r[ix[samp]]) / max(tot, 1), r[ix["Source"]][:60],
                                  " ".join("%s=%d" % (c[6:], v) for c, v in top)))
