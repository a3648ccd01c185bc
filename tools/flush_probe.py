"""How the L2 flush before a timed launch affects a small config: times one
execute after (a) no flush, (b) the write flush, (c) the write flush followed
by a read of another buffer larger than L2 (L2 left clean), and a trivial
kernel under the same conditions.

  python tools/flush_probe.py C1 [reps]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2601_12220_b200 import feinsum as fe  # noqa: E402


def main():
    name = sys.argv[1]
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    torch.cuda.set_device(0)
    w = bench.Workload(name, 0, 1, torch, fe, 100)
    s = torch.cuda.current_stream()
    flush = torch.empty(bench.L2_FLUSH_BYTES // 4, dtype=torch.float32, device="cuda")
    rbuf = torch.ones(bench.L2_FLUSH_BYTES // 4, dtype=torch.float32, device="cuda")
    sink = torch.empty((), dtype=torch.float32, device="cuda")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    pi = [t.data_ptr() for t in w.ins]
    po = [t.data_ptr() for t in w.outs]
    tiny = torch.empty(1, dtype=torch.float64, device="cuda")

    def timed(fn, mode):
        for _ in range(3):
            fn()
        tot = []
        for _ in range(reps):
            if mode >= 1:
                fe.flush_l2(flush)
            if mode == 2:
                torch.sum(rbuf, dim=(0,), out=sink)
            e0.record(s)
            fn()
            e1.record(s)
            torch.cuda.synchronize()
            tot.append(e0.elapsed_time(e1) * 1e3)
        tot.sort()
        return tot[len(tot) // 2], tot[0]

    for mode, label in ((0, "no flush"), (1, "write flush"), (2, "write flush + read 256MiB")):
        a = timed(lambda: w.plan.execute(pi, po, s.cuda_stream), mode)
        b = timed(lambda: fe.fill_dyadic(tiny, 1), mode)
        print(f"{name} {label:28s}: median {a[0]:8.2f} us  min {a[1]:8.2f} | trivial kernel median {b[0]:6.2f} min {b[1]:6.2f}")


if __name__ == "__main__":
    main()
