"""Per-CUDA-source-line stall samples from an ncu report (needs -lineinfo)."""
import csv
import io
import subprocess
import sys

path = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 20
raw = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
out = []
for r in rows:
    if len(r) > 6 and r[0] not in ("", "Line No") and r[0].isdigit():
        try:
            out.append((float(r[4] or 0), int(r[0]), r[1]))
        except ValueError:
            pass
tot = sum(x for x, _, _ in out) or 1.0
for x, line, src in sorted(out, reverse=True)[:n]:
    print(f"{100 * x / tot:5.1f}%  L{line:<4d} {src.strip()[:100]}")
