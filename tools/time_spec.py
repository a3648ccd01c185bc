"""Time one einsum / kernel spec from paper_2601_12220_b200.configs with CUDA
events (no flush; for quick A/B checks, not bench numbers).

  python tools/time_spec.py "tccg(dtype='float32')" [reps]
  python tools/time_spec.py "wave_kernel_nonlinear()" 3
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2601_12220_b200 import configs as C  # noqa: E402
from paper_2601_12220_b200 import feinsum as fe  # noqa: E402


def main():
    spec = eval("C." + sys.argv[1], {"C": C})  # noqa: S307 (tool input)
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    plan = fe.Plan(kernel=spec) if isinstance(spec, str) else fe.Plan(einsum=spec)
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
        ms = e0.elapsed_time(e1)
        print(f"{sys.argv[1]} {plan.info['transform']} {plan.info['meta']}: {ms * 1e3:.1f} us "
              f"({plan.info["algorithmic_flops"] / ms / 1e9:.2f} TFLOP/s)")


if __name__ == "__main__":
    main()
