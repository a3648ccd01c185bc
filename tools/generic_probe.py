"""Time the generic-path einsums (matmul, batched matmul, 3-operand chain) on the GPU."""
import sys, os
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import torch
from paper_2601_12220_b200 import feinsum as fe
def m(n, s): return {"name": n, "shape": s, "dtype": "float64"}
cases = {
 "matmul512": {"i_out": ["a","c"], "i_in": [["a","b"],["b","c"]], "args": [[m("A",[512,512]), m("B",[512,512])]]},
 "matmul4096": {"i_out": ["a","c"], "i_in": [["a","b"],["b","c"]], "args": [[m("A",[4096,4096]), m("B",[4096,4096])]]},
 "bmm64x128": {"i_out": ["z","a","c"], "i_in": [["z","a","b"],["z","b","c"]], "args": [[m("A",[64,128,128]), m("B",[64,128,128])]]},
 "contract3": {"i_out": ["a","d"], "i_in": [["a","b"],["b","c"],["c","d"]], "args": [[m("A",[128,128]), m("B",[128,128]), m("C",[128,128])]]},
}
s = torch.cuda.current_stream()
for name, e in cases.items():
    plan = fe.Plan(einsum=e)
    ins = []
    for k, mm in enumerate(plan.inputs):
        t = torch.empty(mm["shape"], dtype=torch.float64, device="cuda"); fe.fill_dyadic(t, k); ins.append(t)
    outs = plan.alloc_outputs()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(2):
        e0.record(s); plan.execute([t.data_ptr() for t in ins], [t.data_ptr() for t in outs], s.cuda_stream); e1.record(s)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(name, plan.info["transform"], f"{ms:.3f} ms", f"{plan.info['algorithmic_flops']/ms/1e9:.3f} TFLOP/s")
