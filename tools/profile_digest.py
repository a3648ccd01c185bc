"""Digest the captures of profiles/collect.sh (run here, after gpurun):
writes profiles/<round>/launches_summary.txt, ncu_full_summary.txt and
traffic.json (per-config DRAM bytes of the dominant kernel, read by bench.py).

  python tools/profile_digest.py r01
"""
import json
import os
import re
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rnd = sys.argv[1] if len(sys.argv) > 1 else "r01"
out = os.path.join(ROOT, "profiles", rnd)
os.makedirs(out, exist_ok=True)
go = os.path.join(ROOT, "gpurun_out")

launches = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "launch_summary.py"), os.path.join(go, "launches.csv")],
                          capture_output=True, text=True).stdout
shutil.copy(os.path.join(go, "launches.csv"), os.path.join(out, "launches.csv"))  # the raw list the summary is from
with open(os.path.join(out, "launches_summary.txt"), "w") as f:
    f.write("ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised) over\n"
            "python bench.py --configs C1,C2,C3,C4-f64,C4-f32,C5 --steps 2 --warmup 1 (incl. data fill + L2 flush kernels)\n\n")
    f.write(launches)

reps = sorted(p for p in os.listdir(go) if p.startswith("prof_") and p.endswith(".ncu-rep") and p.count("_") >= 2)
summ = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py")] + [os.path.join(go, r) for r in reps],
                      capture_output=True, text=True).stdout
with open(os.path.join(out, "ncu_full_summary.txt"), "w") as f:
    f.write(summ)

traffic = {"source": "ncu --set full --clock-control none, one launch per config (profiles/collect.sh); "
                     "dram__bytes_read.sum + dram__bytes_write.sum", "per_config": {}}
cur = None
for line in summ.splitlines():
    m = re.match(r"== .*prof_(\w+?)_(C[\w-]+)\.ncu-rep", line)
    if m:
        cur = {"kernel": m.group(1), "config": m.group(2), "rd": 0.0, "wr": 0.0}
        continue
    if cur is None:
        continue
    parts = line.split()
    if len(parts) >= 3 and parts[0] in ("dram_read", "dram_write", "time"):
        val = float(parts[1])
        unit = parts[2]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
        if parts[0] == "time":
            cur["time"] = f"{parts[1]} {unit}"
        else:
            cur["rd" if parts[0] == "dram_read" else "wr"] = val * scale
        if parts[0] == "dram_write":
            traffic["per_config"][cur["config"]] = {"kernel": cur["kernel"], "dram_bytes": cur["rd"] + cur["wr"],
                                                   "ncu_time": cur.get("time")}
with open(os.path.join(out, "traffic.json"), "w") as f:
    json.dump(traffic, f, indent=1)
print(launches)
print(json.dumps(traffic, indent=1))
