"""Run one small plan of a given family with synchronous error checking
(for compute-sanitizer / CUDA_LAUNCH_BLOCKING debugging on the GPU box)."""
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2601_12220_b200 import feinsum as fe, configs as C

which = sys.argv[1] if len(sys.argv) > 1 else "gett"
am = lambda n, s, d="float64": {"name": n, "shape": s, "dtype": d}  # noqa: E731
if which == "gett":
    lens = {"a": 2, "b": 72, "c": 2, "d": 72, "e": 8, "f": 8}
    e = {"i_out": list("abcd"), "i_in": [list("aebf"), list("dfce")],
         "args": [[am("A", [lens[s] for s in "aebf"]), am("B", [lens[s] for s in "dfce"])]]}
elif which == "gett72":
    e = C.tccg(ext=72)
elif which == "tt":
    e = C.tensor_train(n=8)
else:
    e = C.tensor_train(n=8, dtype="float32")
plan = fe.Plan(einsum=e)
print(plan.info["transform"], plan.info.get("roles"))
ins = []
for k, m in enumerate(plan.inputs):
    t = torch.empty(m["shape"], dtype=fe._torch_dtype(m["storage"]), device="cuda")
    fe.fill_dyadic(t, k + 1)
    ins.append(t)
outs = plan(*ins)
torch.cuda.synchronize()
print("ok", [o.float().abs().sum().item() for o in outs])
