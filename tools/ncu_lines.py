"""Per-CUDA-source-line metrics from an ncu report (needs -lineinfo).

  python tools/ncu_lines.py REPORT [N] [COLUMN ...]

Default column: warp stall samples. Other useful columns:
"L1 Wavefronts Shared", "L1 Wavefronts Shared Excessive", "Instructions Executed".
"""
import csv
import io
import subprocess
import sys

path = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 20
cols = sys.argv[3:] or ["Warp Stall Sampling (All Samples)"]
raw = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = next(r for r in rows if r and r[0] == "Line No")
idx = [hdr.index(c) for c in cols]
out = []
for r in rows:
    if len(r) > max(idx) and r[0].isdigit():
        try:
            out.append(([float(r[i] or 0) for i in idx], int(r[0]), r[1]))
        except ValueError:
            pass
tot = [sum(x[k] for x, _, _ in out) or 1.0 for k in range(len(idx))]
print("columns:", " | ".join(cols), "| totals:", " ".join(f"{t:.4g}" for t in tot))
for x, line, src in sorted(out, key=lambda o: o[0][0], reverse=True)[:n]:
    vals = " ".join(f"{100 * v / t:5.1f}%" for v, t in zip(x, tot))
    print(f"{vals}  L{line:<4d} {src.strip()[:100]}")
