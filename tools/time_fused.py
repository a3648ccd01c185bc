"""C5 nonlinear step (s = u*u - sin(k)/(2+exp(u))) at E=2e6: generated
fem_grad instance (programs in the prologue, optional epilogues) against the
table path (codegen off: device-VM tables + prebuilt kernel). CUDA events,
L2 flushed before every rep, median of reps.

  python tools/time_fused.py [reps] [variants]   variants: fused,tables,epi,meta=...
"""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2601_12220_b200 import configs as C  # noqa: E402
from paper_2601_12220_b200 import feinsum as fe  # noqa: E402

EPI = ("epi y1[r,e,i] := u1[e,i] + 0.25*y1[r,e,i]\n"
       "epi y2[r,e,i] := u2[e,i] + 0.25*y2[r,e,i]\n"
       "epi y3[r,e,i] := u3[e,i] + 0.25*y3[r,e,i]\n")


def time_plan(plan, reps):
    ins = []
    for k, m in enumerate(plan.inputs):
        t = torch.empty(m["shape"], dtype=fe._torch_dtype(m["storage"]), device="cuda")
        fe.fill_dyadic(t, 100 + k)
        ins.append(t)
    outs = plan.alloc_outputs()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for r in range(reps + 2):
        fe.flush_l2(flush)
        e0.record(s)
        plan.execute([t.data_ptr() for t in ins], [t.data_ptr() for t in outs], s.cuda_stream)
        e1.record(s)
        torch.cuda.synchronize()
        if r >= 2:
            ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
    variants = sys.argv[2].split(",") if len(sys.argv) > 2 else ["fused", "tables", "epi"]
    fk = C.wave_kernel_nonlinear()
    for v in variants:
        opts, text = {}, fk
        if v == "tables":
            opts = {"codegen": False}
        elif v == "epi":
            text = fk + EPI
        elif v.startswith("meta="):
            opts = {"meta": v[5:]}
        plan = fe.Plan(kernel=text, options=opts)
        ms = time_plan(plan, reps)
        roof = plan.info["bytes"] / 6457.7e9 * 1e3
        print(f"{v:24s} {plan.info.get('fem_codegen', '-'):8s} {plan.info['meta']:24s} {ms * 1e3:8.1f} us  "
              f"bytes {plan.info['bytes'] / 1e9:.3f} GB -> {plan.info['bytes'] / ms / 1e6:.0f} GB/s "
              f"(HBM roof {roof * 1e3:.1f} us, frac {roof / ms:.2f})", flush=True)


if __name__ == "__main__":
    main()
