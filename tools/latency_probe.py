"""Fixed-cost probe: time one config at several sizes (bench-style: L2
flushed, CUDA events around a single execute) next to a trivial kernel, to
separate launch/latency overhead from size-proportional time.

  python tools/latency_probe.py C1 0.0032,0.1,1,10
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
    scales = [float(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "0.0032,0.1,1,10").split(",")]
    reps = 30
    torch.cuda.set_device(0)
    s = torch.cuda.current_stream()
    flush = torch.empty(bench.L2_FLUSH_BYTES // 4, dtype=torch.float32, device="cuda")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def timed(fn):
        for _ in range(3):
            fn()
        tot = 0.0
        for _ in range(reps):
            fe.flush_l2(flush)
            e0.record(s)
            fn()
            e1.record(s)
            torch.cuda.synchronize()
            tot += e0.elapsed_time(e1) * 1e3
        return tot / reps

    tiny = torch.empty(1, dtype=torch.float64, device="cuda")
    print(f"trivial fill kernel: {timed(lambda: fe.fill_dyadic(tiny, 1)):.2f} us")
    for sc in scales:
        kind, payload = bench.spec(name, sc)
        plan = fe.Plan(einsum=payload) if kind == "einsum" else fe.Plan(kernel=payload)
        ins = []
        for k, m in enumerate(plan.inputs):
            t = torch.empty(m["shape"], dtype=fe._torch_dtype(m["storage"]), device="cuda")
            fe.fill_dyadic(t, 100 + k)
            ins.append(t)
        outs = plan.alloc_outputs()
        pi, po = [t.data_ptr() for t in ins], [t.data_ptr() for t in outs]
        t = timed(lambda: plan.execute(pi, po, s.cuda_stream))
        mb = plan.info.get("bytes", 0) / 1e6
        print(f"{name} scale {sc:g}: {t:8.2f} us  ({mb:.2f} MB, {plan.info['transform']} {plan.info.get('meta', '')})")


if __name__ == "__main__":
    main()
