"""Coverage beyond the suite configs, timed on the GPU (CUDA events, no L2
flush, second of two runs): which transform the planner picks for common
einsum shapes and how fast it runs. Output kept in profiles/r01/coverage_probe.txt.

  python tools/coverage_probe.py
"""
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
 "matmul2048-f32": {"i_out": ["a","c"], "i_in": [["a","b"],["b","c"]], "args": [[{"name": "A", "shape": [2048, 2048], "dtype": "float32"}, {"name": "B", "shape": [2048, 2048], "dtype": "float32"}]]},
 "tccg6-abcdef-dega-gfbc": {"i_out": list("abcdef"), "i_in": [list("dega"), list("gfbc")], "args": [[m("A",[24,16,64,24]), m("B",[64,24,16,16])]]},
 "chain4-256": {"i_out": ["a","e"], "i_in": [["a","b"],["b","c"],["c","d"],["d","e"]], "args": [[m("A",[256,256]), m("B",[256,256]), m("C",[256,256]), m("D",[256,256])]]},
}
s = torch.cuda.current_stream()
for name, e in cases.items():
    plan = fe.Plan(einsum=e)
    ins = []
    for k, mm in enumerate(plan.inputs):
        t = torch.empty(mm["shape"], dtype=fe._torch_dtype(mm["storage"]), device="cuda"); fe.fill_dyadic(t, k); ins.append(t)
    outs = plan.alloc_outputs()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(2):
        e0.record(s); plan.execute([t.data_ptr() for t in ins], [t.data_ptr() for t in outs], s.cuda_stream); e1.record(s)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(name, plan.info["transform"], f"{ms:.3f} ms", f"{plan.info['algorithmic_flops']/ms/1e9:.3f} TFLOP/s")
