"""Summarise ncu reports (run here, on the CPU box): key throughput metrics and
the top stall reasons per kernel. Usage: python tools/ncu_summary.py rep..."""
import csv
import io
import subprocess
import sys

WANT = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram_%"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64_pipe_%"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor_pipe_%"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "lsu_%"),
    ("sm__issue_active.avg.pct_of_peak_sustained_elapsed", "issue_%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps_active_%"),
    ("launch__registers_per_thread", "regs"),
    ("smsp__inst_executed.sum", "warp_insts"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem_wavefronts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem_conflicts"),
    ("lts__t_sector_hit_rate.pct", "l2_hit_%"),
]


def summarise(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    idx = {h: i for i, h in enumerate(hdr)}
    name = vals[idx["Kernel Name"]][:90] if "Kernel Name" in idx else path
    out = [f"== {path}", f"   kernel: {name}"]
    for key, label in WANT:
        if key in idx:
            out.append(f"   {label:16s} {vals[idx[key]]:>14s} {units[idx[key]]}")
    stalls = []
    for h, i in idx.items():
        if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
            try:
                stalls.append((float(vals[i]), h[len("smsp__pcsamp_warps_issue_stalled_"):]))
            except ValueError:
                pass
    tot = sum(x for x, _ in stalls) or 1.0
    out.append("   stalls: " + ", ".join(f"{h} {100 * x / tot:.0f}%" for x, h in sorted(stalls, reverse=True)[:5]))
    return "\n".join(out)


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print(summarise(p))
