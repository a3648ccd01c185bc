"""Per-kernel share of an ncu launch list (--metrics gpu__time_duration.sum --csv).

  python tools/launch_summary.py gpurun_out/launches.csv
"""
import csv
import re
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(r for r in rows if "Kernel Name" in r)
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
tot = defaultdict(float)
cnt = defaultdict(int)
for r in rows[rows.index(hdr) + 1:]:
    if len(r) > vi and r[mi] == "gpu__time_duration.sum":
        name = re.sub(r"\(.*", "", r[ki]).replace("(anonymous namespace)::", "").replace("feb200::", "")
        v = float(r[vi].replace(",", ""))
        unit = r[hdr.index("Metric Unit")] if "Metric Unit" in hdr else "ns"
        scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "nsecond": 1e-6, "msecond": 1.0, "ms": 1.0}.get(unit, 1e-6)
        tot[name] += v * scale
        cnt[name] += 1
s = sum(tot.values()) or 1.0
for name, t in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{name[:60]:60s} launches={cnt[name]:4d} total_ms={t:10.3f} share={100 * t / s:5.1f}%")
