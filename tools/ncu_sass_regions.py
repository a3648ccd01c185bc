"""Split a kernel's SASS (ncu source page, sass view) into regions at
barrier / branch-target boundaries and print per-region stall samples,
DFMA count, shared wavefronts (ideal / excess), with the dominant stall
reasons. Usage: python tools/ncu_sass_regions.py report.ncu-rep [min_pct]"""
import csv
import io
import subprocess
import sys

path = sys.argv[1]
min_pct = float(sys.argv[2]) if len(sys.argv) > 2 else 0.5
raw = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = None
data = []
for r in rows:
    if "Source" in r and "Warp Stall Sampling (All Samples)" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(r)
H = {h: i for i, h in enumerate(hdr)}
f = lambda r, k: float(r[H[k]] or 0) if k in H else 0.0
tot = sum(f(r, "Warp Stall Sampling (All Samples)") for r in data) or 1
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
regions = []
cur = None
for r in data:
    src = r[H["Source"]].strip()
    if cur is None or src.startswith("BAR") or src.startswith("WARPSYNC") or "SYNCS" in src:
        cur = {"first": r[H["Address"]], "label": src[:60], "samples": 0, "dfma": 0, "inst": 0, "wf": 0, "wfi": 0,
               "st": {s: 0.0 for s in stalls}, "n": 0}
        regions.append(cur)
    s = f(r, "Warp Stall Sampling (All Samples)")
    cur["samples"] += s
    ie = f(r, "Instructions Executed")
    cur["inst"] += ie
    if src.split()[0:1] and ("DFMA" in src or "DMUL" in src or "DADD" in src):
        cur["dfma"] += ie
    cur["wf"] += f(r, "L1 Wavefronts Shared")
    cur["wfi"] += f(r, "L1 Wavefronts Shared Ideal")
    for st in stalls:
        cur["st"][st] += f(r, st)
    cur["n"] += 1
for g in regions:
    pct = 100 * g["samples"] / tot
    if pct < min_pct:
        continue
    top = sorted(g["st"].items(), key=lambda kv: -kv[1])[:3]
    ts = ", ".join(f"{k[6:]} {100 * v / max(g['samples'], 1):.0f}%" for k, v in top)
    print(f"{pct:5.1f}%  n={g['n']:4d} dfma={g['dfma']:.3g} inst={g['inst']:.3g} wf={g['wf']:.3g}/{g['wfi']:.3g}  [{g['label']}]  {ts}")
