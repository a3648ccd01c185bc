"""Per-warp phase timeline of the merged hex kernel (meta v=7 = the traced
instance): CTA 0, clock64 stamps per warp.
  python tools/hex_trace.py [C2] [nshow]
Events: 0 loop top, 1 G landed, 2 B done, 3 after barrier 1, 4 C sweeps done,
5 U landed (A starts), 6 A done, 7 chain done (before barrier 2)."""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2601_12220_b200 import feinsum as fe  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
nshow = int(sys.argv[2]) if len(sys.argv) > 2 else 3
kind, payload = bench.spec(name)
base = fe.Plan(einsum=payload)
plan = fe.Plan(einsum=payload, options={"meta": "v=7", "transform": base.info["transform"]})
ins = []
for k, m in enumerate(plan.inputs):
    t = torch.empty(m["shape"], dtype=fe._torch_dtype(m["storage"]), device="cuda")
    fe.fill_dyadic(t, 100 + k)
    ins.append(t)
outs = plan.alloc_outputs()
s = torch.cuda.current_stream()
for _ in range(2):
    plan.execute([t.data_ptr() for t in ins], [t.data_ptr() for t in outs], s.cuda_stream)
torch.cuda.synchronize()
lib = ctypes.CDLL(fe.LIB_PATH)
NIT, NW, NEV = 48, 16, 8
buf = np.zeros(NIT * NW * NEV, dtype=np.uint64)
rc = lib.fe_debug_hex_trace(buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(buf.nbytes))
assert rc == 0, rc
tr = buf.reshape(NIT, NW, NEV).astype(np.int64)
names = ["top", "Gok", "Bdone", "bar1", "Cdone", "Uok", "Adone", "chain"]
rows = []
for it in range(8, 40):
    t0 = tr[it, :15, 3].min()
    rows.append(dict(
        stage_clk=int(tr[it + 1, :15, 3].min() - t0),
        B_first=int(tr[it, :13, 2].min() - tr[it, :15, 1].min()),
        B_last=int(tr[it, :13, 2].max() - tr[it, :15, 1].min()),
        Gwait=int(tr[it, :15, 1].max() - tr[it, :15, 0].max()),
        bar1=int(tr[it, :15, 3].min() - tr[it, :16, 2].max()),
        C=float(np.mean(tr[it, :15, 4] - tr[it, :15, 3])),
        Uwait=float(np.mean(tr[it, :15, 5] - tr[it, :15, 4])),
        A=float(np.mean(tr[it, :15, 6] - tr[it, :15, 5])),
        chain=float(np.mean(tr[it, :15, 7] - tr[it, :15, 6])),
        CA_first=int(tr[it, :15, 7].min() - t0),
        CA_last=int(tr[it, :15, 7].max() - t0),
        bar2=int(tr[it + 1, :15, 0].min() - tr[it, :16, 7].max()),
    ))
print("mean over stages 8-39 (clk):")
for k in rows[0]:
    print(f"  {k:10s} {np.mean([r[k] for r in rows]):9.0f}")
for it in range(10, 10 + nshow):
    t0 = tr[it, :, 0].min()
    print(f"stage {it}:")
    for w in range(16):
        print(f"  w{w:2d} " + " ".join(f"{n}={int(tr[it, w, e] - t0):6d}" for e, n in enumerate(names)))
