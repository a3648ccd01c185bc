"""Pin the oracle before trusting it (CPU).

oracle/_ref is the unmodified reference library; these tests check it (and the
plain-C restatement oracle/evaluate_port.c) against the reference's own
known-answer tests and the committed golden vectors."""
import numpy as np
import pytest


def am(name, shape, dtype="float64"):
    return {"name": name, "shape": list(shape), "dtype": dtype}


def test_worked_golden_key(ref):
    # proj/tests/test_notation.cpp:126-130
    e = {"i_out": ["i"], "i_in": [["i", "j"], ["i", "k"]], "args": [[am("A", [72, 18]), am("B", [72, 18])]]}
    c = ref.canonicalize(e)
    assert c["key"] == "FE1|b=1|n=2|out=a|in=ab;ac|rows=A0,A1|A0=float64:72x18|A1=float64:72x18"
    # proj/tests/test_canonicalize.cpp:23-33
    assert c["sigma_idx"] == {"a": "i", "b": "j", "c": "k"}
    assert c["sigma_arg"] == {"A0": "A", "A1": "B"}
    assert c["sigma_row"] == [0] and c["sigma_slot"] == [0, 1]


def test_batched_golden_key(ref, fixtures):
    # proj/tests/test_notation.cpp:131-135
    c = ref.canonicalize(ref.parse_classic(fixtures["squared_ref.es"]))
    assert c["key"] == "FE1|b=2|n=2|out=b|in=ba;a|rows=A0,A1;A0,A2|A0=float64:96x4|A1=float64:4|A2=float64:4"


def test_goldens_reproduce(ref, fixtures, golden):
    for name, want in golden["canon"].items():
        assert ref.canonicalize(ref.parse_classic(fixtures[name])) == want, name
    for name, want in golden["evaluate"].items():
        e = ref.parse_classic(fixtures[name])
        outs = ref.evaluate(e, ref.random_bindings(e, want["seed"]))
        for o, w in zip(outs, want["outputs"]):
            w = np.array([complex(a, b) for a, b in w])
            assert np.array_equal(o.reshape(-1), w), name


def test_complex_no_conjugation(ref):
    # proj/tests/test_core.cpp:219-229: (i)(i) + (1)(2) = 1 exactly
    e = {"i_out": [], "i_in": [["i"], ["i"]], "args": [[am("x", [2], "complex128"), am("y", [2], "complex128")]]}
    out = ref.evaluate(e, {"x": np.array([1j, 1]), "y": np.array([1j, 2])})
    assert out[0].reshape(-1)[0] == 1 + 0j


def test_matmul_vs_loop(ref):
    # proj/tests/test_core.cpp:154-174
    e = {"i_out": ["i", "j"], "i_in": [["i", "k"], ["k", "j"]], "args": [[am("A", [10, 4]), am("B", [4, 10])]]}
    b = ref.random_bindings(e, 42)
    got = ref.evaluate(e, b)[0].real
    assert np.max(np.abs(got - b["A"] @ b["B"])) < 1e-13


@pytest.mark.parametrize("seed", range(40))
def test_port_matches_reference_bitwise(ref, seed):
    """The C restatement of evaluate() is bit-identical to the reference."""
    e = ref.generate_random(seed, b_max=3, n_max=3, max_indices=5, shape_pool=[2, 3, 4])
    b = ref.random_bindings(e, seed + 1000)
    for x, y in zip(ref.evaluate(e, b), ref.port_evaluate(e, b)):
        assert np.array_equal(x, y)


def test_port_complex_and_diagonal(ref):
    e = {"i_out": ["i"], "i_in": [["i", "i"], ["i"]], "args": [[am("A", [5, 5], "complex128"), am("v", [5], "complex128")]]}
    rng = np.random.default_rng(3)
    b = {"A": rng.standard_normal((5, 5)) + 1j * rng.standard_normal((5, 5)),
         "v": rng.standard_normal(5) + 1j * rng.standard_normal(5)}
    for x, y in zip(ref.evaluate(e, b), ref.port_evaluate(e, b)):
        assert np.array_equal(x, y)
