"""Host enqueue time vs device time of fe_plan_execute_host for one config
(host pipeline overrides via FE_PIPE_MIN_MB / FE_PIPE_CHUNKS).
  python tools/e2e_probe.py C1 [reps]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2601_12220_b200 import feinsum as fe  # noqa: E402

name = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
kind, payload = bench.spec(name)
plan = fe.Plan(einsum=payload) if kind == "einsum" else fe.Plan(kernel=payload)
hin = []
for k, m in enumerate(plan.inputs):
    t = torch.empty(m["shape"], dtype=fe._torch_dtype(m["storage"]), device="cuda")
    fe.fill_dyadic(t, 100 + k)
    hin.append(t.cpu().pin_memory())
hout = [torch.empty(o.shape, dtype=o.dtype).pin_memory() for o in plan.alloc_outputs()]
s = torch.cuda.current_stream()
pi, po = [h.data_ptr() for h in hin], [h.data_ptr() for h in hout]
plan.execute_host(pi, po, s.cuda_stream)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for _ in range(reps):
    torch.cuda.synchronize()
    e0.record(s)
    t0 = time.perf_counter()
    plan.execute_host(pi, po, s.cuda_stream)
    t1 = time.perf_counter()
    e1.record(s)
    torch.cuda.synchronize()
    print(f"{name} env={os.environ.get('FE_PIPE_CHUNKS', '-')}: host enqueue {1e6 * (t1 - t0):8.1f} us, device {1e3 * e0.elapsed_time(e1):8.1f} us")
