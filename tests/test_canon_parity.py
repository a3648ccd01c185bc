"""Host side of the hot path: the B200 build's canonicalizer, keys, notation
and raising must be byte-identical to the reference (CPU, differential against
oracle/_ref). Sweeps mirror proj/tests/test_canonicalize.cpp and
proj/tests/acceptance.cpp (criteria 1-3)."""
import pytest

GEN_DEFAULT = {}
GEN_WIDE = {"b_max": 5, "n_max": 5, "max_indices": 8, "max_dim": 4, "shape_pool": [2, 3, 4, 5, 7]}
GEN_DTYPES = {"dtype_pool": ["float32", "float64", "complex128", "int8"]}


def test_fixtures_canonicalize_identically(fe, ref, fixtures, golden):
    for name, text in fixtures.items():
        if not name.endswith(".es"):
            continue
        e = fe.parse_classic(text)
        assert e == ref.parse_classic(text), name
        assert fe.canonicalize(e) == golden["canon"][name], name
        assert fe.print_classic(e) == ref.print_classic(e), name


@pytest.mark.parametrize("block", range(10))
def test_generated_and_scrambled(fe, ref, block):
    """1000 seeds: canonical form, key and all four sigma maps bytewise equal,
    for the instance and a scrambled copy (acceptance crit. 1)."""
    for seed in range(1 + 100 * block, 1 + 100 * (block + 1)):
        e = ref.generate_random(seed)
        assert fe.generate_random(seed) == e
        sc = ref.scramble(e, seed * 7919 + 13)
        assert fe.scramble(e, seed * 7919 + 13) == sc
        for x in (e, sc["e"]):
            assert fe.canonicalize(x) == ref.canonicalize(x), seed
        assert fe.canonicalize(e)["canonical"] == fe.canonicalize(sc["e"])["canonical"]


@pytest.mark.parametrize("params", [GEN_WIDE, GEN_DTYPES, {"allow_repeated_index": False, "allow_empty_out": False}])
def test_generated_param_families(fe, ref, params):
    for seed in range(300):
        e = ref.generate_random(seed, **params)
        assert fe.generate_random(seed, **params) == e
        assert fe.canonicalize(e) == ref.canonicalize(e), seed


def test_symmetric_rows(fe, ref):
    """Many interchangeable rows (the reference's blow-up case)."""
    for b in (2, 4, 8):
        rows = [[{"name": "A", "shape": [3, 4], "dtype": "float64"},
                 {"name": f"B{q}", "shape": [5, 4], "dtype": "float64"},
                 {"name": "C", "shape": [5, 2], "dtype": "float64"}] for q in range(b)]
        e = {"i_out": ["i", "k"], "i_in": [["i", "j"], ["k", "j"], ["k", "l"]], "args": rows}
        assert fe.canonicalize(e) == ref.canonicalize(e)


def _sym_cases():
    """Row-symmetric einsums for the seeded-automorphism fast path: fully
    interchangeable rows, rows in two classes, argument involutions between
    rows (A,B / B,A), swapped arguments that are also read by a third row (the
    candidate is not an automorphism), and equal-shape rows with different
    structure."""
    m = lambda n, s, d="float64": {"name": n, "shape": list(s), "dtype": d}
    cases = []
    for b in (3, 5, 9):
        cases.append({"i_out": ["i", "k"], "i_in": [["i", "j"], ["k", "j"], ["j", "l"]],
                      "args": [[m("G1", (4, 3)), m("G2", (4, 3)), m(f"X{q}", (3, 2))] for q in range(b)]})
        # two classes: even rows read P, odd rows read Q in slot 0
        cases.append({"i_out": ["i"], "i_in": [["i", "j"], ["j"]],
                      "args": [[m("P" if q % 2 else "Q", (3, 3)), m(f"v{q}", (3,))] for q in range(b)]})
    # involution between two rows: (A, B) and (B, A)
    cases.append({"i_out": ["i", "j"], "i_in": [["i", "k"], ["k", "j"]],
                  "args": [[m("A", (3, 3)), m("B", (3, 3))], [m("B", (3, 3)), m("A", (3, 3))], [m("C", (3, 3)), m("D", (3, 3))]]})
    # rows 0/1 swap X0 <-> X1 but row 2 also reads X1
    cases.append({"i_out": ["i"], "i_in": [["i", "j"], ["j"]],
                  "args": [[m("M", (2, 2)), m("X0", (2,))], [m("M", (2, 2)), m("X1", (2,))],
                           [m("N", (2, 2)), m("X1", (2,))],
                           [m("M", (2, 2)), m("X3", (2,))]]})
    # equal shapes, different dtypes in one row
    cases.append({"i_out": ["i"], "i_in": [["i", "j"], ["j"]],
                  "args": [[m("M", (2, 2)), m(f"y{q}", (2,), "float32" if q == 2 else "float64")] for q in range(5)]})
    return cases


def test_seeded_automorphisms_keep_the_labeling(fe, ref):
    """The B200 canonicalizer seeds its search with verified row-swap
    automorphisms (orders of magnitude faster for many interchangeable rows);
    outputs must stay byte-identical to the reference, for the instances and
    scrambled copies."""
    for t, e in enumerate(_sym_cases()):
        assert fe.canonicalize(e) == ref.canonicalize(e), t
        for seed in (3, 17):
            sc = ref.scramble(e, seed)["e"]
            assert fe.canonicalize(sc) == ref.canonicalize(sc), (t, seed)


def test_many_symmetric_rows_are_fast(fe):
    """b = 64 interchangeable rows: seconds-to-minutes for the plain search
    (it grows like b^5), milliseconds with the seeded automorphisms; spellings
    with permuted rows land on the same key."""
    import time
    m = lambda n, s: {"name": n, "shape": list(s), "dtype": "float64"}
    e = {"i_out": ["i", "k"], "i_in": [["i", "j"], ["k", "l"], ["j", "l"]],
         "args": [[m("G1", (8, 8)), m("G2", (8, 8)), m(f"X{q}", (8, 8))] for q in range(64)]}
    t0 = time.time()
    c = fe.canonicalize(e)
    assert time.time() - t0 < 5.0
    e2 = dict(e, args=list(reversed(e["args"])))
    assert fe.canonicalize(e2)["canonical"] == c["canonical"]


def test_baseline_configs(fe, golden):
    for name, item in golden["configs"].items():
        if "einsum" in item:
            assert fe.canonicalize(item["einsum"]) == item["canon"], name
        else:
            # functional configs: the raised skeleton
            assert item["raise"]["skeleton"]["i_out"]
    c1 = golden["configs"]["C1"]["canon"]
    assert golden["configs"]["C1-permuted"]["canon"]["key"] == c1["key"]
    assert c1["key"].startswith("FE1|b=3|n=3|out=dae|in=bda;bec;ac|")


def test_is_isomorphic_and_brute_force(fe, ref, fixtures):
    pairs = [("iso_plain_first.es", "iso_plain_second.es"), ("iso_batched_first.es", "iso_batched_second.es"),
             ("canon_first.es", "canon_second.es"), ("matmul.es", "squared_ref.es")]
    for a, b in pairs:
        ea, eb = fe.parse_classic(fixtures[a]), fe.parse_classic(fixtures[b])
        assert fe.is_isomorphic(ea, eb) == ref.is_isomorphic(ea, eb)
        assert fe.brute_force_isomorphic(ea, eb) == ref.brute_force_isomorphic(ea, eb)
    fa, fb = fe.parse_classic(fixtures["fig_pair_first.es"]), fe.parse_classic(fixtures["fig_pair_second.es"])
    with pytest.raises(fe.FeinsumError) as ex:
        fe.brute_force_isomorphic(fa, fb)
    assert ex.value.kind == "domain"
    with pytest.raises(ref.RefError) as rx:
        ref.brute_force_isomorphic(fa, fb)
    assert str(ex.value) == str(rx.value)


def test_verify_witness_messages(fe, ref):
    for seed in range(60):
        e = ref.generate_random(seed)
        sc = ref.scramble(e, seed + 5)
        w = dict(sc["w"])
        assert fe.verify_witness(sc["e"], e, w) == ref.verify_witness(sc["e"], e, w)
        if len(w["sigma_slot"]) > 1:
            w["sigma_slot"] = list(reversed(w["sigma_slot"]))
        if w["sigma_idx"]:
            k = sorted(w["sigma_idx"])[0]
            w["sigma_idx"] = dict(w["sigma_idx"], **{k: "zz"})
        assert fe.verify_witness(sc["e"], e, w) == ref.verify_witness(sc["e"], e, w)


def test_induced_graph_and_labeling(fe, ref):
    for seed in range(80):
        e = ref.generate_random(seed)
        for shuffle in (-1, seed):
            g = fe.induced_graph(e, shuffle)
            assert g == ref.induced_graph(e, shuffle)
            assert fe.canonical_labeling(g) == ref.canonical_labeling(g)
            assert fe.check_compliance(g) == ref.check_compliance(g) == []


def test_compliance_damage_messages(fe, ref):
    """Hand-made damage (proj/tests/test_induced_graph.cpp:219-302 style)."""
    e = {"i_out": ["i", "j"], "i_in": [["i", "k"], ["k", "j"]],
         "args": [[{"name": "A", "shape": [10, 4], "dtype": "float64"},
                   {"name": "B", "shape": [4, 10], "dtype": "float64"}]]}
    g = ref.induced_graph(e)
    variants = []
    g1 = dict(g, edges=[x for x in g["edges"] if x != [5, 0]])
    variants.append(g1)
    g2 = dict(g, edges=g["edges"] + [[0, 1]])
    variants.append(g2)
    g3 = dict(g, colors=[c if i != 3 else 4 for i, c in enumerate(g["colors"])])
    variants.append(g3)
    g4 = dict(g, edges=[x for x in g["edges"] if x != [17, 18]])
    variants.append(g4)
    g5 = dict(g, colors=[10] + g["colors"][1:])
    variants.append(g5)
    damaged = 0
    for v in variants:
        assert fe.check_compliance(v) == ref.check_compliance(v)
        damaged += bool(fe.check_compliance(v))
    assert damaged >= 3


def test_validate_messages(fe, ref):
    bad = [
        {"i_out": ["i", "i"], "i_in": [["i"]], "args": [[{"name": "A", "shape": [3], "dtype": "float64"}]]},
        {"i_out": ["z"], "i_in": [["i", "j"]], "args": [[{"name": "A", "shape": [3], "dtype": "float64"}]]},
        {"i_out": [], "i_in": [["i"], ["i"]], "args": [[{"name": "A", "shape": [3], "dtype": "float64"},
                                                         {"name": "A", "shape": [4], "dtype": "float64"}]]},
        {"i_out": [], "i_in": [["i"]], "args": []},
        {"i_out": [], "i_in": [], "args": [[]]},
        {"i_out": ["i"], "i_in": [["i"]], "args": [[{"name": "", "shape": [0], "dtype": "float64"}],
                                                   [{"name": "B", "shape": [-1], "dtype": "float64"}]]},
        {"i_out": [""], "i_in": [["i", ""]], "args": [[{"name": "A", "shape": [2, 2], "dtype": "float64"}]]},
        {"i_out": ["i"], "i_in": [["i"]], "args": [[{"name": "A", "shape": [3], "dtype": "float64"}],
                                                   [{"name": "B", "shape": [4], "dtype": "float64"}],
                                                   [{"name": "C", "shape": [3], "dtype": "float64"},
                                                    {"name": "D", "shape": [3], "dtype": "float64"}]]},
    ]
    for e in bad:
        assert fe.validate(e) == ref.validate(e)
        assert fe.validate(e)


CLASSIC_ERRORS = [
    "einsum: i->i\nrow: A\narray: A float64 3\narray: A float64 3\n",
    "einsum: i->i\nrow: A\narray: A floatt64 3\n",
    "einsum: i->i\nrow: A\narray: A float64 3x\n",
    "einsum: i->i\nrow: A\narray: A float64 0\n",
    "",
    "einsum: i->i\n",
    "einsum: i,j->ij\nrow: A\narray: A float64 3\n",
    "einsum: i->i\nrow: X\narray: A float64 3\n",
    "einsum: i->i\nrow: A\narray: A float64 3\narray: Z float64 9\n",
    "einsum: i->i\nfoo: bar\n",
    "einsum: i->i\njust words\n",
    "einsum: ii->ii\nrow: A\narray: A float64 3x3\n",
    "einsum: iJ->i\nrow: A\narray: A float64 3x3\n",
    "einsum: i-i\nrow: A\n",
    "row: A\n",
    "einsum: i->i\narray: A float64 3\nrow: A\n",
    "einsum: i->i\nrow: 9A\n",
    "einsum: i->i\neinsum: i->i\n",
    "einsum: i->i\nrow: A\narray: A float64 3 extra\n",
]


def test_classic_parse_errors(fe, ref):
    for text in CLASSIC_ERRORS:
        with pytest.raises(fe.FeinsumError) as ex:
            fe.parse_classic(text)
        with pytest.raises(ref.RefError) as rx:
            ref.parse_classic(text)
        assert str(ex.value) == str(rx.value)
        assert ex.value.code == rx.value.code


def test_canonical_key_requires_canonical(fe, ref):
    e = {"i_out": ["i"], "i_in": [["i", "j"], ["i", "k"]],
         "args": [[{"name": "A", "shape": [72, 18], "dtype": "float64"},
                   {"name": "B", "shape": [72, 18], "dtype": "float64"}]]}
    with pytest.raises(fe.FeinsumError) as ex:
        fe.canonical_key(e)
    assert str(ex.value) == "canonical_key wants a canonical form; canonicalize first"
    c = fe.canonicalize(e)
    assert fe.canonical_key(c["canonical"]) == ref.canonical_key(c["canonical"]) == c["key"]


def test_zero_dim_operand_rejected_by_encoder(fe, ref):
    e = {"i_out": ["i"], "i_in": [["i"], []],
         "args": [[{"name": "x", "shape": [5], "dtype": "float64"}, {"name": "c", "shape": [], "dtype": "float64"}]]}
    with pytest.raises(fe.FeinsumError) as ex:
        fe.canonicalize(e)
    with pytest.raises(ref.RefError) as rx:
        ref.canonicalize(e)
    assert str(ex.value) == str(rx.value)
