"""Launch-overhead probe for one config: compares the bench-style single
timed execute (L2 flushed before it) with back-to-back executes and with the
execute captured in a CUDA graph.

  python tools/time_config.py C1 [reps]
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2601_12220_b200 import feinsum as fe  # noqa: E402


def main():
    name = sys.argv[1]
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 50
    torch.cuda.set_device(0)
    w = bench.Workload(name, 0, 1, torch, fe, 100)
    s = torch.cuda.current_stream()
    flush = torch.empty(bench.L2_FLUSH_BYTES // 4, dtype=torch.float32, device="cuda")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ptr_in = [t.data_ptr() for t in w.ins]
    ptr_out = [t.data_ptr() for t in w.outs]
    for _ in range(5):
        w.run(s.cuda_stream)
    torch.cuda.synchronize()

    def timed(fn, flush_first):
        tot = 0.0
        for _ in range(reps):
            if flush_first:
                fe.flush_l2(flush)
            e0.record(s)
            fn()
            e1.record(s)
            torch.cuda.synchronize()
            tot += e0.elapsed_time(e1) * 1e3
        return tot / reps

    t_single = timed(lambda: w.plan.execute(ptr_in, ptr_out, s.cuda_stream), True)
    t_warm = timed(lambda: w.plan.execute(ptr_in, ptr_out, s.cuda_stream), False)
    # host cost of one execute call
    torch.cuda.synchronize()
    h0 = time.perf_counter()
    for _ in range(reps):
        w.plan.execute(ptr_in, ptr_out, s.cuda_stream)
    h1 = time.perf_counter()
    torch.cuda.synchronize()
    n = 20
    e0.record(s)
    for _ in range(n):
        w.plan.execute(ptr_in, ptr_out, s.cuda_stream)
    e1.record(s)
    torch.cuda.synchronize()
    t_b2b = e0.elapsed_time(e1) * 1e3 / n
    g = torch.cuda.CUDAGraph()
    cs = torch.cuda.Stream()
    with torch.cuda.stream(cs):
        g.capture_begin()
        w.plan.execute(ptr_in, ptr_out, cs.cuda_stream)
        g.capture_end()
    torch.cuda.synchronize()
    t_graph = timed(g.replay, True)
    print(f"{name}: single(flushed) {t_single:.2f} us | single(warm L2) {t_warm:.2f} us | back-to-back {t_b2b:.2f} us"
          f" | graph(flushed) {t_graph:.2f} us | host per execute {(h1 - h0) / reps * 1e6:.2f} us")


if __name__ == "__main__":
    main()
