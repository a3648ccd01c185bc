"""Run one config with forced kernel parameters (for ncu captures / A-B runs).

  python tools/run_variant.py C5 "mma=1;stages=4" [reps]
  python tools/run_variant.py C5-nonlinear generic     # force the generic kernel
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2601_12220_b200 import feinsum as fe  # noqa: E402


def main():
    name, meta = sys.argv[1], sys.argv[2]
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
    if name == "C5-nonlinear":
        from paper_2601_12220_b200 import configs as C
        kind, payload = "kernel", C.wave_kernel_nonlinear()
    else:
        kind, payload = bench.spec(name)
    base = fe.Plan(einsum=payload) if kind == "einsum" else fe.Plan(kernel=payload)
    if meta == "generic":
        opts = {"transform": "generic/v1"}
    else:
        opts = {"meta": meta, "transform": base.info["transform"]} if meta else {}
    plan = fe.Plan(einsum=payload, options=opts) if kind == "einsum" else fe.Plan(kernel=payload, options=opts)
    ins = []
    for k, m in enumerate(plan.inputs):
        t = torch.empty(m["shape"], dtype=fe._torch_dtype(m["storage"]), device="cuda")
        fe.fill_dyadic(t, 100 + k)
        ins.append(t)
    outs = plan.alloc_outputs()
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(reps):
        e0.record(s)
        plan.execute([t.data_ptr() for t in ins], [t.data_ptr() for t in outs], s.cuda_stream)
        e1.record(s)
        torch.cuda.synchronize()
        print(f"{name} {plan.info['transform']} {plan.info['meta']}: {e0.elapsed_time(e1) * 1e3:.1f} us")


if __name__ == "__main__":
    main()
