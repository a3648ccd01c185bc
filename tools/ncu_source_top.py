"""Top SASS lines by stall samples from an ncu report (source page)."""
import csv
import io
import subprocess
import sys

path = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
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
i_src = hdr.index("Source")
i_s = hdr.index("Warp Stall Sampling (All Samples)")
stall_cols = [(i, h) for i, h in enumerate(hdr) if h.startswith("stall_") or "Stall" in h and h not in (hdr[i_s],)]
tot = sum(float(r[i_s] or 0) for r in data) or 1
for r in sorted(data, key=lambda r: -float(r[i_s] or 0))[:n]:
    print(f"{100 * float(r[i_s] or 0) / tot:5.1f}%  {r[i_src][:90]}")
