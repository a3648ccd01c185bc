"""TEST ORACLE — regenerate tests/golden/ from the reference (run HERE, where
/root/reference exists; the GPU box only reads the committed JSON).

  python oracle/gen_golden.py

Writes
  tests/golden/fixtures.json   the reference's own fixture documents
                               (proj/tests/fixtures/*.es, *.fk), verbatim;
  tests/golden/reference.json  outputs of the unmodified reference library
                               (oracle/_ref) on those fixtures and on the
                               BASELINE config spellings at small extents:
                               canonical forms, keys, sigma maps, cost model,
                               raise/identify results, and evaluate() results
                               on random_bindings inputs.
"""
import glob
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)

from oracle import refpy as R  # noqa: E402
from paper_2601_12220_b200 import configs as C  # noqa: E402

FIXTURES = "/root/reference/proj/tests/fixtures"


def cplx_list(a):
    a = np.asarray(a).reshape(-1)
    return [[float(x.real), float(x.imag)] for x in a]


def main():
    fx = {}
    for p in sorted(glob.glob(os.path.join(FIXTURES, "*"))):
        with open(p) as f:
            fx[os.path.basename(p)] = f.read()
    out_dir = os.path.join(ROOT, "tests", "golden")
    os.makedirs(out_dir, exist_ok=True)
    with open(os.path.join(out_dir, "fixtures.json"), "w") as f:
        json.dump(fx, f, indent=1, sort_keys=True)

    ref = {"canon": {}, "cost": {}, "evaluate": {}, "raise": {}, "identify": {}, "configs": {}}
    for name, text in fx.items():
        if name.endswith(".es"):
            e = R.parse_classic(text)
            ref["canon"][name] = R.canonicalize(e)
            ref["cost"][name] = R.cost(e)
    # evaluate goldens: small fixtures with the reference's seeds
    for name, seed in [("matmul.es", 42), ("iso_plain_first.es", 404), ("iso_batched_first.es", 405),
                       ("squared_ref.es", 7), ("canon_first.es", 11)]:
        e = R.parse_classic(fx[name])
        b = R.random_bindings(e, seed)
        outs = R.evaluate(e, b)
        ref["evaluate"][name] = {"seed": seed, "outputs": [cplx_list(o) for o in outs]}
    # functional kernel
    fk = fx["squared_kernel.fk"]
    ref["raise"]["squared_kernel.fk"] = R.raise_kernel(fk)
    ref["identify"]["squared_kernel.fk"] = R.identify(fk, R.parse_classic(fx["squared_ref.es"]))
    # BASELINE configs (small extents): keys and sigma maps
    small = {
        "C1": C.fem_grad(E=64),
        "C1-permuted": C.fem_grad_permuted(E=64),
        "C2": C.hex_poisson(E=6, b=2),
        "C3": C.tccg(ext=6),
        "C4": C.tensor_train(n=8, r=4),
    }
    for name, e in small.items():
        ref["configs"][name] = {"einsum": e, "canon": R.canonicalize(e)}
    for sib in C.TCCG_SIBLINGS:
        e = C.tccg(sib, ext=5)
        ref["configs"]["tccg:" + sib] = {"einsum": e, "canon": R.canonicalize(e)}
    ref["configs"]["C5"] = {"raise": R.raise_kernel(C.wave_kernel(E=64))}
    ref["configs"]["C5-renamed"] = {"raise": R.raise_kernel(C.wave_kernel(E=64, renamed=True))}
    with open(os.path.join(out_dir, "reference.json"), "w") as f:
        json.dump(ref, f, indent=1, sort_keys=True)
    print("wrote", out_dir)


if __name__ == "__main__":
    main()
