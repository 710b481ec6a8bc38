"""Per-kernel SASS census of liblora.so: how many instructions of each kind that proves the hardware
path (tcgen05 UTCHMMA / LDTM / UTCBAR, TMA UTMALDG / UTMAPF, bulk copy UBLKCP, mma.sync HMMA, LDGSTS,
FFMA, griddepcontrol ACQBULK/PREEXIT...).  Static counts (instructions in the binary, not executed).
usage: python scripts/sass_census.py [liblora.so] > profiles/r2_sass_census.txt"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
so = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "paper_2401_11240_b200", "lib", "liblora.so")
KINDS = ["UTCHMMA", "UTCBAR", "LDTM", "STTM", "UTMALDG", "UTMAPF", "UBLKCP", "UBLKPF", "HMMA", "LDGSTS", "LDSM",
         "FFMA", "SYNCS", "ACQBULK", "PREEXIT", "REDG", "ATOMG", "MEMBAR"]
sass = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True).stdout
cur, counts = None, collections.OrderedDict()
for ln in sass.splitlines():
    m = re.match(r"\s*Function : (\S+)", ln)
    if m:
        cur = m.group(1)
        counts[cur] = collections.Counter()
        continue
    if cur is None:
        continue
    m = re.match(r"\s*/\*[0-9a-f]+\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", ln)
    if m:
        op = m.group(2)
        for k in KINDS:
            if op == k or op.startswith(k + "_") or op.startswith(k + "."):
                counts[cur][k] += 1
        counts[cur]["_total"] += 1


def demangle(n):
    try:
        return subprocess.run(["c++filt", n], capture_output=True, text=True).stdout.strip()
    except Exception:
        return n


print("# SASS census of %s (static instruction counts per kernel; cuobjdump -sass)" % os.path.relpath(so, ROOT))
print("# %-62s %s" % ("kernel", " ".join("%7s" % k for k in KINDS + ["_total"])))
for fn, c in counts.items():
    name = demangle(fn)
    name = re.sub(r"\(.*$", "", name).replace("lora::", "")
    print("%-64s %s" % (name[:64], " ".join("%7d" % c[k] for k in KINDS + ["_total"])))
