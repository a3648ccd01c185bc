"""One small execute of every kernel family, for compute-sanitizer
(memcheck / racecheck / synccheck). Extents are small so the
instrumented runs finish in minutes; every case is checked against the
reference evaluator (oracle/_ref) or exactness so a sanitizer-clean run is
also a correct one.

  compute-sanitizer --tool memcheck python tools/sanitize_cases.py [case,...]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import refpy  # noqa: E402
from paper_2601_12220_b200 import configs as C  # noqa: E402
from paper_2601_12220_b200 import feinsum as fe  # noqa: E402


def run(plan, b):
    ins = [torch.from_numpy(np.ascontiguousarray(np.real(np.asarray(b[m["name"]])).astype(
        {"f64": np.float64, "f32": np.float32}[m["storage"]]).reshape(m["shape"]))).cuda() for m in plan.inputs]
    outs = plan(*ins)
    torch.cuda.synchronize()
    return [o.double().cpu().numpy() for o in outs]


def check(got, want, tol):
    for g, w in zip(got, want):
        w = np.real(w).reshape(g.shape)
        err = float(np.max(np.abs(g - w) / np.maximum(1.0, np.abs(w)))) if w.size else 0.0
        assert err <= tol, err


def einsum_case(e, opts=None, tol=1e-12, seed=3):
    plan = fe.Plan(einsum=e, options=opts or {})
    b = refpy.random_bindings(e, seed)
    check(run(plan, b), refpy.evaluate(e, b), tol)
    return plan.info["transform"] + " " + plan.info.get("meta", "")


def hex_merged_case():
    """The merged-stage hex kernel (eight fields) with two stages on the first
    CTAs (E = 600: 150 four-element stages over the 148-CTA grid), so C(s) and
    A(s+1) share a segment; bitwise against the three-barrier kernel (v=3),
    which the parity suite pins to the reference."""
    e = C.hex_poisson(E=600, b=8)
    b = refpy.random_bindings(e, 7)
    got = run(fe.Plan(einsum=e), b)
    want = run(fe.Plan(einsum=e, options={"meta": "v=3", "transform": "hex_sumfact/v1"}), b)
    for g, w in zip(got, want):
        assert np.array_equal(g, w)
    return "hex_sumfact/v1 (merged, vs v=3)"


def kernel_case(fk, rows, shape, opts=None, seed=5, post=None):
    import re
    arrays = []
    for line in fk.splitlines():
        m = re.match(r"array: (\w+) (\w+) (\S+)", line)
        if m:
            arrays.append({"name": m.group(1), "dtype": m.group(2),
                           "shape": [] if m.group(3) == "scalar" else [int(x) for x in m.group(3).split("x")]})
    b = refpy.random_bindings({"i_out": [], "i_in": [[] for _ in arrays], "args": [arrays]}, seed)
    plan = fe.Plan(kernel=fk, options=opts or {})
    stripped = "\n".join(x for x in fk.splitlines() if not x.startswith("epi ")) + "\n"
    want = refpy.eval_kernel(stripped, arrays, b, rows, shape)
    got = run(plan, b)
    want = [np.real(w) for w in want]
    if post is not None:
        want = post(want, b)
    check(got, want, 1e-12)
    return plan.info["transform"] + " " + plan.info.get("fem_codegen", "")


CASES = {
    "fem_grad": lambda: einsum_case(C.fem_grad(E=2048)),
    "fem_grad_ept1": lambda: einsum_case(C.fem_grad(E=2048), {"meta": "stages=4;te=32;ept=1"}),
    "fem_grad_f32": lambda: einsum_case(C.fem_grad(E=2048, dtype="float32"), tol=1e-5),
    "fem_rtc": lambda: kernel_case(C.wave_kernel_nonlinear(E=1026)
                                   + "epi y1[r,e,i] := u1[e,i] + 0.25*y1[r,e,i]\n", 3, [3, 1026, 10],
                                   post=lambda w, b: [np.real(np.asarray(b["u1"]))[None] + 0.25 * w[0]] + w[1:]),
    "fem_mma": lambda: einsum_case(C.fem_grad(E=2048), {"meta": "mma=1"}),
    "generic": lambda: einsum_case({"i_out": ["i", "j"], "i_in": [["i", "k"], ["k", "j"]],
                                    "args": [[{"name": "A", "shape": [10, 4], "dtype": "float64"},
                                              {"name": "B", "shape": [4, 10], "dtype": "float64"}]]},
                                   {"transform": "generic/v1"}, tol=0.0),
    "gett": lambda: einsum_case({"i_out": list("abcd"), "i_in": [list("aebf"), list("dfce")],
                                 "args": [[{"name": "A", "shape": [2, 8, 72, 8], "dtype": "float64"},
                                           {"name": "B", "shape": [72, 8, 2, 8], "dtype": "float64"}]]}),
    "gett_splitk": lambda: einsum_case({"i_out": ["i", "j"], "i_in": [["i", "k"], ["k", "j"]],
                                        "args": [[{"name": "A", "shape": [144, 512], "dtype": "float64"},
                                                  {"name": "B", "shape": [512, 144], "dtype": "float64"}]]}),
    "gett_affine": lambda: kernel_case(C.tccg_kernel(ext=24, a_ext=2), 1, [2, 24, 24, 24]),
    "tt": lambda: einsum_case(C.tensor_train(n=4, r=64)),
    "tt_tc": lambda: einsum_case(C.tensor_train(n=4, r=64, dtype="float32"), {"meta": "tc=1"}, tol=1e-4),
    "hex2": lambda: einsum_case(C.hex_poisson(E=8, b=2)),
    "hex1": lambda: einsum_case(C.hex_poisson(E=8, b=2), {"meta": "v=1"}),
    "hex5": lambda: hex_merged_case(),
    "path": lambda: einsum_case({"i_out": ["a", "d"], "i_in": [["a", "b"], ["b", "c"], ["c", "d"]],
                                 "args": [[{"name": n, "shape": [48, 48], "dtype": "float64"} for n in "ABC"]]}),
    "tab_vm": lambda: kernel_case(C.wave_kernel_nonlinear(E=512), 3, [3, 512, 10], {"codegen": False}),
    "epi_pass": lambda: kernel_case("domain: n<4 i<64 j<64 k<64 l<64\n"
                                    "array: G float64 64x64\narray: H float64 64x64\narray: X float64 4x64x64\n"
                                    "stmt y[n,i,k] = sum([j,l], G[i,j]*H[k,l]*X[n,j,l])\n"
                                    "epi y[n,i,k] := 0.5*y[n,i,k]\n", 1, [4, 64, 64],
                                    post=lambda w, b: [0.5 * w[0]]),
}


def main():
    names = sys.argv[1].split(",") if len(sys.argv) > 1 else list(CASES)
    torch.cuda.set_device(0)
    for n in names:
        print(f"case {n}: {CASES[n]()}", flush=True)
    print("all cases ok", flush=True)


if __name__ == "__main__":
    main()
