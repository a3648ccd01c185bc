"""Bitwise A/B of two kernel variants of one config (same inputs):
  python tools/ab_compare.py C2 "" "v=4"
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2601_12220_b200 import feinsum as fe  # noqa: E402


def main():
    name, ma, mb = sys.argv[1], sys.argv[2], sys.argv[3]
    kind, payload = bench.spec(name)
    base = fe.Plan(einsum=payload) if kind == "einsum" else fe.Plan(kernel=payload)
    outs = []
    ins = None
    for meta in (ma, mb):
        opts = {"meta": meta, "transform": base.info["transform"]} if meta else {}
        plan = fe.Plan(einsum=payload, options=opts) if kind == "einsum" else fe.Plan(kernel=payload, options=opts)
        if ins is None:
            ins = []
            for k, m in enumerate(plan.inputs):
                t = torch.empty(m["shape"], dtype=fe._torch_dtype(m["storage"]), device="cuda")
                fe.fill_dyadic(t, 100 + k)
                ins.append(t)
        outs.append(plan(*ins))
        torch.cuda.synchronize()
    for k, (a, b) in enumerate(zip(*outs)):
        d = (a - b).abs()
        print(f"output {k}: equal={torch.equal(a, b)} max|diff|={d.max().item():.3e} ndiff={int((d > 0).sum())}")


if __name__ == "__main__":
    main()
