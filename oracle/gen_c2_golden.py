"""TEST ORACLE — golden outputs of the unmodified reference evaluator
(oracle/_ref, proj/src/core.cpp:269-358) for the C2 spelling at E = 64
elements, b = 8 fields (the benched row structure, 16 stages of the hex
kernel's four-element pipeline). Run HERE (8 host cores, ~2 min):

  python oracle/gen_c2_golden.py

Inputs are the reference's own random_bindings (proj/tests/test_util.hpp:19-29,
mt19937_64 seed 64) of the full E = 64 einsum; the GPU test regenerates them
with the same call. The reference evaluates each output point (e, i, m, n)
from element e's data alone, so evaluating element slices in parallel
processes gives bit-identical outputs to one full call (the slices are
checked against one full call at E = 2 below).

Writes tests/golden/c2_e64_b8.npz: y[8, 64, 5, 5, 5] (real parts; the
imaginary parts are exactly zero for real data).
"""
import multiprocessing as mp
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)

E, B, SEED = 64, 8, 64
OUT = os.path.join(ROOT, "tests", "golden", "c2_e64_b8.npz")


def _slice(binds, lo, hi):
    out = {}
    for k, v in binds.items():
        if k == "G":
            out[k] = v[:, :, lo:hi]
        elif k.startswith("u"):
            out[k] = v[lo:hi]
        else:
            out[k] = v
    return out


def _work(rng):
    from oracle import refpy as R
    from paper_2601_12220_b200 import configs as C
    lo, hi = rng
    e_full = C.hex_poisson(E=E, b=B)
    binds = R.random_bindings(e_full, SEED)
    e = C.hex_poisson(E=hi - lo, b=B)
    ys = R.evaluate(e, _slice(binds, lo, hi))
    return lo, np.stack([y.real for y in ys])


def main():
    from oracle import refpy as R
    from paper_2601_12220_b200 import configs as C
    # slicing check at E = 2: two one-element calls == one two-element call
    e2 = C.hex_poisson(E=2, b=2)
    b2 = R.random_bindings(e2, 5)
    whole = np.stack([y.real for y in R.evaluate(e2, b2)])
    e1 = C.hex_poisson(E=1, b=2)
    parts = [np.stack([y.real for y in R.evaluate(e1, _slice(b2, k, k + 1))]) for k in (0, 1)]
    assert np.array_equal(whole, np.concatenate(parts, axis=1)), "element slices differ from one call"

    chunks = [(lo, lo + 1) for lo in range(E)]
    y = np.zeros((B, E, 5, 5, 5))
    with mp.get_context("spawn").Pool(os.cpu_count()) as pool:
        for lo, part in pool.imap_unordered(_work, chunks):
            y[:, lo:lo + 1] = part
    np.savez_compressed(OUT, y=y, E=E, b=B, seed=SEED)
    print("wrote", OUT, y.shape, float(np.abs(y).max()))


if __name__ == "__main__":
    main()
