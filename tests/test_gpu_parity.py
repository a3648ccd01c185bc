"""GPU parity: the sm_100a kernels, called through the C-ABI, against the
reference evaluator (oracle/_ref) on the same inputs.

Bars:
  * generic kernel: bit-identical to feinsum::evaluate (same product order and
    pairwise summation tree), every dtype, complex included;
  * tuned fp64 kernels (different contraction order, FMA): max rel_err <= 1e-12
    with rel_err = |got - want| / max(1, |want|) (proj/tests/test_util.hpp:31-42);
  * fp32 kernels: <= 1e-5 against the double-computed reference.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

FP64_TOL = 1e-12


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return torch


def rel_err(got, want):
    got = np.asarray(got).reshape(-1)
    want = np.asarray(want).reshape(-1)
    return float(np.max(np.abs(got - want) / np.maximum(1.0, np.abs(want)))) if want.size else 0.0


def run_plan(torch, plan, bindings):
    ins = []
    for m in plan.inputs:
        a = np.asarray(bindings[m["name"]]).reshape(m["shape"])
        np_dt = {"f64": np.float64, "c128": np.complex128, "f32": np.float32}[m["storage"]]
        a = a.astype(np_dt) if np_dt != np.float64 else np.real(a).astype(np.float64)
        ins.append(torch.from_numpy(np.ascontiguousarray(a)).cuda())
    outs = plan(*ins)
    torch.cuda.synchronize()
    return [o.cpu().numpy() for o in outs]


def test_device_visible(fe, torch_cuda):
    assert fe.lib().fe_device_check() == 0
    assert fe.lib().fe_sm_count() >= 1


@pytest.mark.parametrize("params", [
    {},
    {"b_max": 3, "n_max": 4, "max_indices": 6, "shape_pool": [2, 3, 5]},
    {"dtype_pool": ["float32", "float64", "int8", "int32"]},
])
def test_generic_bit_exact_random(fe, ref, torch_cuda, params):
    """The generic kernel reproduces feinsum::evaluate bit for bit."""
    gen = {"transform": "generic/v1"}
    for seed in range(40):
        e = ref.generate_random(seed, **params)
        b = ref.random_bindings(e, seed + 17)
        want = ref.evaluate(e, b)
        got = fe.evaluate(e, b, gen)
        for g, w in zip(got, want):
            assert np.array_equal(g.reshape(-1), w.reshape(-1)), (seed, e)


def test_default_plans_random(fe, ref, torch_cuda):
    """Whatever the planner picks for random einsums (generic, a tuned family,
    or a contraction path for three or more operands) stays within the fp64
    bar of the reference."""
    picked = set()
    for seed in range(60):
        e = ref.generate_random(seed, b_max=1 + seed % 2, n_max=4, max_indices=6, shape_pool=[2, 3, 5, 8])
        b = ref.random_bindings(e, seed + 23)
        want = ref.evaluate(e, b)
        got = fe.evaluate(e, b)
        picked.add(fe.Plan(einsum=e, options={"dry_run": True}).info["transform"])
        for g, w in zip(got, want):
            assert rel_err(g, w) <= FP64_TOL, (seed, e)
    assert "generic/v1" in picked


def _random_gett_einsum(rng):
    """A random 2-operand contraction: M / N / K groups of 1-2 indices, an
    optional batch index, random index orders in A, B and C."""
    letters = iter("abcdefghij")
    def group(n, big):
        g = [(next(letters), big if k == 0 else int(rng.choice([2, 3]))) for k in range(n)]
        return g
    M = group(int(rng.integers(1, 3)), int(rng.choice([24, 32])))
    N = group(int(rng.integers(1, 3)), int(rng.choice([24, 32])))
    K = group(int(rng.integers(1, 3)), 64)
    Z = group(int(rng.integers(0, 2)), 3)
    ext = dict(M + N + K + Z)
    def order(*gs):
        xs = [x for g in gs for x, _ in g]
        rng.shuffle(xs)
        return xs
    a, b, c = order(M, K, Z), order(K, N, Z), order(Z, M, N)
    m = lambda n, ix: {"name": n, "shape": [ext[x] for x in ix], "dtype": "float64"}  # noqa: E731
    return {"i_out": c, "i_in": [a, b], "args": [[m("A", a), m("B", b)]]}


def test_gett_random_two_operand(fe, ref, torch_cuda):
    """Random two-operand contractions (groups of one or two indices, random
    orders, optional batch index): whatever the planner picks matches the
    reference exactly on dyadic data, and most of them take the GETT kernel
    (split / folded / repacked / batched forms)."""
    rng = np.random.default_rng(5)
    taken = 0
    for k in range(24):
        e = _random_gett_einsum(rng)
        b = ref.random_bindings(e, 100 + k)
        plan = fe.Plan(einsum=e)
        taken += plan.info["transform"] == "gett_dmma/v1"
        got = run_plan(torch_cuda, plan, b)[0]
        assert np.array_equal(got, ref.evaluate(e, b)[0].real), (k, e, plan.info["transform"])
    assert taken >= 12, taken


def test_contraction_path(fe, ref, torch_cuda):
    """Three- and four-operand chains run as pairwise GETT / generic steps in
    the optimal order (operands with private indices reduced first); within
    the fp64 bar of the naive reference sum."""
    m = lambda n, s: {"name": n, "shape": s, "dtype": "float64"}  # noqa: E731
    cases = [
        {"i_out": ["a", "d"], "i_in": [["a", "b"], ["b", "c"], ["c", "d"]],
         "args": [[m("A", [48, 64]), m("B", [64, 72]), m("C", [72, 40])]]},
        {"i_out": ["a", "e"], "i_in": [["a", "b"], ["b", "c"], ["c", "d"], ["d", "e"]],
         "args": [[m("A", [30, 64]), m("B", [64, 24]), m("C", [24, 48]), m("D", [48, 36])]]},
        {"i_out": ["z", "a", "c"], "i_in": [["z", "a", "b"], ["b", "k"], ["z", "k", "c"]],
         "args": [[m("A", [3, 40, 64]), m("B", [64, 64]), m("C", [3, 64, 30])]]},
        # two operands, one with a private index: reduced first, then GETT
        {"i_out": ["a", "d"], "i_in": [["a", "x", "c"], ["c", "d"]], "args": [[m("A", [48, 6, 64]), m("B", [64, 40])]]},
        # two rows: each row planned on its own (here: a path each)
        {"i_out": ["a", "d"], "i_in": [["a", "b"], ["b", "c"], ["c", "d"]],
         "args": [[m("A", [48, 64]), m("B", [64, 72]), m("C", [72, 40])], [m("A", [48, 64]), m("D", [64, 72]), m("C", [72, 40])]]},
    ]
    for k, e in enumerate(cases):
        plan = fe.Plan(einsum=e)
        assert plan.info["transform"] == "path/v1", (k, plan.info)
        b = ref.random_bindings(e, 80 + k)
        got = run_plan(torch_cuda, plan, b)
        want = [w.real for w in ref.evaluate(e, b)]
        for g, w in zip(got, want):
            assert rel_err(g, w) <= FP64_TOL, k
        # float32 arrays: fp32 intermediates, the fp32 bar
        e32 = {**e, "args": [[{**a, "dtype": "float32"} for a in row] for row in e["args"]]}
        plan = fe.Plan(einsum=e32)
        assert plan.info["transform"] == "path/v1", (k, plan.info)
        for g, w in zip(run_plan(torch_cuda, plan, b), want):
            assert g.dtype == np.float32 and rel_err(g, w) <= 1e-5, k


def test_path_plans_execute_many(fe, ref, torch_cuda):
    """A path plan executes its step plans while holding its scratch lock;
    with the lock a plain mutex hashed by plan address, a step plan that
    hashed to the same bucket deadlocked (1 in 16 per step). 48 fresh
    three-step plans make a collision near certain if the lock regressed."""
    m = lambda n, s: {"name": n, "shape": s, "dtype": "float64"}  # noqa: E731
    e = {"i_out": ["a", "d"], "i_in": [["a", "b"], ["b", "c"], ["c", "d"]],
         "args": [[m("A", [48, 64]), m("B", [64, 72]), m("C", [72, 40])]]}
    b = ref.random_bindings(e, 5)
    want = [w.real for w in ref.evaluate(e, b)]
    for _ in range(48):
        plan = fe.Plan(einsum=e)
        assert plan.info["transform"] == "path/v1"
        for g, w in zip(run_plan(torch_cuda, plan, b), want):
            assert rel_err(g, w) <= FP64_TOL


def test_generic_complex_bit_exact(fe, ref, torch_cuda):
    rng = np.random.default_rng(0)
    for seed in range(20):
        e = ref.generate_random(seed, dtype_pool=["complex128", "float64"])
        b = {}
        for m in ref.universe(e):
            shp = m["shape"]
            b[m["name"]] = rng.standard_normal(shp) + (1j * rng.standard_normal(shp) if m["dtype"] == "complex128" else 0)
        want = ref.evaluate(e, b)
        got = fe.evaluate(e, b)
        for g, w in zip(got, want):
            assert np.array_equal(g.reshape(-1), w.reshape(-1)), seed


def test_reference_known_answers(fe, torch_cuda, fixtures, golden):
    # complex without conjugation (proj/tests/test_core.cpp:219-229)
    am = lambda n, s, d="float64": {"name": n, "shape": s, "dtype": d}  # noqa: E731
    e = {"i_out": [], "i_in": [["i"], ["i"]], "args": [[am("x", [2], "complex128"), am("y", [2], "complex128")]]}
    out = fe.evaluate(e, {"x": np.array([1j, 1]), "y": np.array([1j, 2])})
    assert out[0].reshape(-1)[0] == 1 + 0j
    # diagonal, 0-dim operand, dot product (test_core.cpp:195-217)
    e = {"i_out": ["i"], "i_in": [["i", "i"]], "args": [[am("A", [4, 4])]]}
    A = np.arange(16.0).reshape(4, 4)
    assert np.array_equal(fe.evaluate(e, {"A": A})[0].real, np.diag(A))
    e = {"i_out": ["i"], "i_in": [["i"], []], "args": [[am("x", [5]), am("c", [])]]}
    x = np.arange(5.0) - 2.5
    assert np.array_equal(fe.evaluate(e, {"x": x, "c": np.array(0.75)})[0].real, x * 0.75)
    # golden evaluate vectors of the reference fixtures
    from oracle import refpy
    for name, want in golden["evaluate"].items():
        e = fe.parse_classic(fixtures[name])
        b = refpy.random_bindings(e, want["seed"])
        for g, w in zip(fe.evaluate(e, b), want["outputs"]):
            w = np.array([complex(a, c) for a, c in w])
            assert np.array_equal(g.reshape(-1), w), name


def test_binding_errors(fe, torch_cuda):
    e = {"i_out": ["i"], "i_in": [["i"]], "args": [[{"name": "x", "shape": [5], "dtype": "float64"}]]}
    with pytest.raises(fe.FeinsumError, match="no binding for array x"):
        fe.evaluate(e, {})
    with pytest.raises(fe.FeinsumError, match="wrong element count"):
        fe.evaluate(e, {"x": np.zeros(6)})


def test_fem_grad_c1_full(fe, ref, torch_cuda):
    """C1 at full size (E = 1e4) through the tuned K1 kernel."""
    from paper_2601_12220_b200 import configs as C
    e = C.fem_grad(E=10_000)
    plan = fe.Plan(einsum=e)
    assert plan.info["transform"] == "fem_grad/v1"
    b = ref.random_bindings(e, 7)
    got = run_plan(torch_cuda, plan, b)
    want = ref.evaluate(e, b)
    for g, w in zip(got, want):
        assert rel_err(g, w) <= FP64_TOL


def test_fem_grad_permuted_spelling_same_kernel(fe, ref, torch_cuda):
    from paper_2601_12220_b200 import configs as C
    e1, e2 = C.fem_grad(E=2_000), C.fem_grad_permuted(E=2_000)
    p1, p2 = fe.Plan(einsum=e1), fe.Plan(einsum=e2)
    assert p1.info["key"] == p2.info["key"]
    assert p2.info["transform"] == "fem_grad/v1"
    b = ref.random_bindings(e2, 3)
    got = run_plan(torch_cuda, p2, b)
    for g, w in zip(got, ref.evaluate(e2, b)):
        assert rel_err(g, w) <= FP64_TOL


def test_fem_grad_odd_sizes(fe, ref, torch_cuda):
    from paper_2601_12220_b200 import configs as C
    for E, b in [(2, 1), (34, 2), (1002, 5), (66, 3)]:
        e = C.fem_grad(E=E, b=b)
        plan = fe.Plan(einsum=e)
        assert plan.info["transform"] == "fem_grad/v1"
        bind = ref.random_bindings(e, E)
        for g, w in zip(run_plan(torch_cuda, plan, bind), ref.evaluate(e, bind)):
            assert rel_err(g, w) <= FP64_TOL, E
    # odd element count: bulk copies need 16-byte runs -> generic path, still exact
    e = C.fem_grad(E=33)
    plan = fe.Plan(einsum=e)
    assert plan.info["transform"] == "generic/v1"
    bind = ref.random_bindings(e, 1)
    for g, w in zip(run_plan(torch_cuda, plan, bind), ref.evaluate(e, bind)):
        assert np.array_equal(g, w.real)


FEM_VARIANTS = ["stages=2", "stages=4;te=16", "stages=3;dsmem=1", "stages=4;ept=2", "stages=2;ept=2;te=64", "stages=4;ept=2;te=34", "stages=3;ept=2;te=68", "mma=1;stages=4", "mma=1;stages=2;te=16",
                "mma=1;stages=3;te=64"]


@pytest.mark.parametrize("meta", FEM_VARIANTS)
def test_fem_grad_variants(fe, ref, torch_cuda, meta):
    """Every tuned K1 variant (DFMA, D in smem, half tiles, DMMA) on ragged
    tails, several rows, and the C5 functional operands."""
    from paper_2601_12220_b200 import configs as C
    opts = {"meta": meta, "transform": "fem_grad/v1"}
    for E, nb in [(2, 1), (34, 2), (1002, 5), (66, 3), (10_000, 3)]:
        e = C.fem_grad(E=E, b=nb)
        plan = fe.Plan(einsum=e, options=opts)
        assert plan.info["transform"] == "fem_grad/v1" and plan.info["meta"] == meta
        bind = ref.random_bindings(e, E + 1)
        for g, w in zip(run_plan(torch_cuda, plan, bind), ref.evaluate(e, bind)):
            assert rel_err(g, w) <= FP64_TOL, (meta, E)
    fk = C.wave_kernel(E=4_002)
    info, arrays, b = _kernel_bindings(ref, fk, 13)
    plan = fe.Plan(kernel=fk, options=opts)
    got = run_plan(torch_cuda, plan, b)
    want = ref.eval_kernel(fk, arrays, b, 3, [3, 4_002, 10])
    for g, w in zip(got, want):
        assert rel_err(g, w) <= FP64_TOL, meta


@pytest.mark.parametrize("meta", ["", "stages=4", "stages=3;dsmem=1", "stages=2;ept=2;te=64", "stages=4;te=16"])
def test_fem_grad_fp32(fe, ref, torch_cuda, meta):
    """float32 arrays take the fp32 instance of K1 (same kernel, half the
    bytes): within the fp32 bar of the reference (which computes in double),
    plain and functional (u + 0.5 k) operands, ragged tails."""
    from paper_2601_12220_b200 import configs as C
    opts = {"meta": meta, "transform": "fem_grad/v1"} if meta else None
    for E, nb in [(4, 1), (1_004, 3), (10_000, 3)]:
        e = C.fem_grad(E=E, b=nb, dtype="float32")
        plan = fe.Plan(einsum=e, options=opts) if opts else fe.Plan(einsum=e)
        assert plan.info["transform"] == "fem_grad/v1", plan.info
        assert plan.outputs[0]["storage"] == "f32"
        bind = ref.random_bindings(e, E + 3)
        for g, w in zip(run_plan(torch_cuda, plan, bind), ref.evaluate(e, bind)):
            assert g.dtype == np.float32 and rel_err(g, w.real) <= 1e-5, (meta, E)
    fk = C.wave_kernel(E=4_000).replace("float64", "float32")
    info, arrays, b = _kernel_bindings(ref, fk, 19)
    plan = fe.Plan(kernel=fk, options=opts) if opts else fe.Plan(kernel=fk)
    assert plan.info["transform"] == "fem_grad/v1"
    want = ref.eval_kernel(fk, arrays, b, 3, [3, 4_000, 10])
    for g, w in zip(run_plan(torch_cuda, plan, b), want):
        assert rel_err(g, w) <= 1e-5, meta


def _kernel_bindings(ref, fk, seed):
    info = ref.raise_kernel(fk)
    import re
    arrays = []
    for line in fk.splitlines():
        m = re.match(r"array: (\w+) (\w+) (\S+)", line)
        if m:
            shape = [] if m.group(3) == "scalar" else [int(x) for x in m.group(3).split("x")]
            arrays.append({"name": m.group(1), "shape": shape, "dtype": m.group(2)})
    fake = {"i_out": [], "i_in": [[] for _ in arrays], "args": [arrays]}
    b = ref.random_bindings(fake, seed)
    return info, arrays, b


def test_wave_step_c5_functional(fe, ref, torch_cuda):
    """C5: s_q = u_q + 0.5 k_q fused into the K1 prologue."""
    from paper_2601_12220_b200 import configs as C
    for renamed in (False, True):
        fk = C.wave_kernel(E=4_000, renamed=renamed)
        info, arrays, b = _kernel_bindings(ref, fk, 11)
        plan = fe.Plan(kernel=fk)
        assert plan.info["transform"] == "fem_grad/v1"
        got = run_plan(torch_cuda, plan, b)
        want = ref.eval_kernel(fk, arrays, b, 3, [3, 4_000, 10])
        for g, w in zip(got, want):
            assert rel_err(g, w) <= FP64_TOL
    k1 = fe.Plan(kernel=C.wave_kernel(E=4_000)).info["key"]
    k2 = fe.Plan(kernel=C.wave_kernel(E=4_000, renamed=True)).info["key"]
    assert k1 == k2 == fe.Plan(einsum=C.fem_grad(E=4_000)).info["key"]


def test_tabulated_vm_operands_take_tuned_kernels(fe, ref, torch_cuda):
    """Non-affine functional operands (here u*u - sin(k)/(2+exp(u))) are
    tabulated on the device at the start of the execute (the reference's
    materialize, same programs) and read as plain leaves, so the tuned family
    runs instead of the generic kernel; results agree with the reference and
    with the generic kernel evaluating the programs in place."""
    from paper_2601_12220_b200 import configs as C
    fk = C.wave_kernel_nonlinear(E=2_000)
    info, arrays, b = _kernel_bindings(ref, fk, 13)
    plan = fe.Plan(kernel=fk)
    assert plan.info["transform"] == "fem_grad/v1", plan.info
    # fem_grad computes the programs in its generated prologue (no tables,
    # tests/test_epilogue.py); with codegen off the device VM tabulates them
    assert plan.info["tabulated"] == [] and plan.info["fem_codegen"] == "nvrtc"
    got = run_plan(torch_cuda, plan, b)
    want = ref.eval_kernel(fk, arrays, b, 3, [3, 2_000, 10])
    vm = fe.Plan(kernel=fk, options={"codegen": False})
    assert vm.info["tab_codegen"] == ["vm: codegen disabled"] * 3
    for g, v in zip(got, run_plan(torch_cuda, vm, b)):
        assert np.array_equal(g, v)
    gen = fe.Plan(kernel=fk, options={"transform": "generic/v1"})
    assert gen.info["tabulated"] == []
    got_g = run_plan(torch_cuda, gen, b)
    for g, w, gg in zip(got, want, got_g):
        assert rel_err(g, w) <= FP64_TOL
        assert rel_err(gg, w) <= FP64_TOL
    # tensor train with a transcendental core: tt kernel over the table
    fk = ("domain: n<64 i<64 j<64 k<64 l<64\n"
          "def g(a,c) := exp(H[a,c] / 4)\n"
          "def h(a,c) := K[a,c]\n"
          "def x(m,a,c) := X[m,a,c]\n"
          "array: H float64 64x64\narray: K float64 64x64\narray: X float64 64x64x64\n"
          "stmt y[n,i,k] = sum([j,l], g(i,j)*h(k,l)*x(n,j,l))\n")
    info, arrays, b = _kernel_bindings(ref, fk, 17)
    plan = fe.Plan(kernel=fk)
    assert plan.info["transform"] == "tt/v1" and len(plan.info["tabulated"]) == 1, plan.info
    assert plan.info["tab_codegen"] == ["nvrtc"]
    got = run_plan(torch_cuda, plan, b)
    want = ref.eval_kernel(fk, arrays, b, 1, [64, 64, 64])
    assert rel_err(got[0], want[0]) <= FP64_TOL
    # the generated tabulation kernel reproduces the device VM bit for bit
    vm = fe.Plan(kernel=fk, options={"codegen": False})
    assert vm.info["tab_codegen"] == ["vm: codegen disabled"]
    assert np.array_equal(got[0], run_plan(torch_cuda, vm, b)[0])


def test_squared_kernel_vm(fe, ref, torch_cuda, fixtures):
    """Transcendental functional operands run in the device VM."""
    fk = fixtures["squared_kernel.fk"]
    info, arrays, b = _kernel_bindings(ref, fk, 5)
    plan = fe.Plan(kernel=fk)
    got = run_plan(torch_cuda, plan, b)
    want = ref.eval_kernel(fk, arrays, b, 2, [96])
    for g, w in zip(got, want):
        assert rel_err(g, w) <= FP64_TOL


def test_vm_complex_sqrt(fe, ref, torch_cuda):
    fk = ("domain: i<6 j<3\n"
          "def f(p) := sqrt(X[p]) * reciprocal(Y[p]) - exp(X[p]) / 3\n"
          "array: X float64 6\narray: Y float64 6\narray: W float64 6x3\n"
          "stmt y[j] = sum([i], f(i)*W[i,j])\n")
    info, arrays, b = _kernel_bindings(ref, fk, 9)
    plan = fe.Plan(kernel=fk, options={"storage": "wide"})
    assert plan.info["complex"] and plan.outputs[0]["storage"] == "c128"
    got = run_plan(torch_cuda, plan, b)
    want = ref.eval_kernel(fk, arrays, b, 1, [3])
    assert rel_err(got[0], want[0]) <= FP64_TOL


def _tccg_small(ref, fe, a_ext=2, c_ext=2, e_ext=8, f_ext=8):
    am = lambda n, s: {"name": n, "shape": s, "dtype": "float64"}  # noqa: E731
    lens = {"a": a_ext, "b": 72, "c": c_ext, "d": 72, "e": e_ext, "f": f_ext}
    return {"i_out": list("abcd"), "i_in": [list("aebf"), list("dfce")],
            "args": [[am("A", [lens[s] for s in "aebf"]), am("B", [lens[s] for s in "dfce"])]]}


def test_gett_split_groups_matmul_shapes(fe, ref, torch_cuda):
    """Contractions whose M / N / K groups have one index (matmul shapes) run
    on the GETT kernel by reshaping the index into (outer, inner) dims; exact
    on dyadic data like the TCCG form (float32: the reference's double value
    rounded once)."""
    m = lambda n, s, dt="float64": {"name": n, "shape": s, "dtype": dt}  # noqa: E731
    cases = [
        {"i_out": ["a", "c"], "i_in": [["a", "b"], ["b", "c"]], "args": [[m("A", [128, 256]), m("B", [256, 96])]]},
        {"i_out": ["a", "c"], "i_in": [["b", "a"], ["c", "b"]], "args": [[m("A", [256, 120]), m("B", [72, 256])]]},
        {"i_out": ["a", "b", "d"], "i_in": [["a", "b", "c"], ["c", "d"]], "args": [[m("A", [30, 40, 64]), m("B", [64, 48])]]},
        {"i_out": ["d", "a"], "i_in": [["a", "c"], ["c", "d"]], "args": [[m("A", [50, 72]), m("B", [72, 144])]]},
        {"i_out": ["a", "b"], "i_in": [["a", "c"], ["b", "c"]],
         "args": [[m("A", [100, 128], "float32"), m("B", [96, 128], "float32")]]},
    ]
    for k, e in enumerate(cases):
        plan = fe.Plan(einsum=e)
        assert plan.info["transform"] == "gett_dmma/v1", (k, plan.info)
        b = ref.random_bindings(e, 40 + k)
        got = run_plan(torch_cuda, plan, b)[0]
        want = ref.evaluate(e, b)[0].real
        if got.dtype == np.float32:
            assert np.array_equal(got, want.astype(np.float32)), k
        else:
            assert np.array_equal(got, want), k


def test_gett_folded_groups_tccg6(fe, ref, torch_cuda):
    """6-index TCCG contractions whose groups have three indices fold the
    ones that stay adjacent in every array (abcdef-dega-gfbc: de and bc)
    into one dim; exact on dyadic data."""
    m = lambda n, s: {"name": n, "shape": s, "dtype": "float64"}  # noqa: E731

    def tc(out, a, b, L):
        return {"i_out": list(out), "i_in": [list(a), list(b)], "args": [[m("A", [L[x] for x in a]), m("B", [L[x] for x in b])]]}
    cases = [
        tc("abcdef", "dega", "gfbc", {"a": 24, "b": 2, "c": 3, "d": 2, "e": 3, "f": 24, "g": 64}),
        tc("abcdef", "gdab", "efgc", {"a": 4, "b": 6, "c": 3, "d": 2, "e": 2, "f": 12, "g": 64}),
    ]
    for k, e in enumerate(cases):
        plan = fe.Plan(einsum=e)
        assert plan.info["transform"] == "gett_dmma/v1", (k, plan.info)
        b = ref.random_bindings(e, 90 + k)
        got = run_plan(torch_cuda, plan, b)[0]
        assert np.array_equal(got, ref.evaluate(e, b)[0].real), k


@pytest.mark.parametrize("ks", ["ks=1", "ks=3", "ks=8"])
def test_gett_split_k(fe, ref, torch_cuda, ks):
    """Split K (slices of the k steps into a workspace, ordered reduce):
    forced slice counts on a matmul and a batched matmul, exact on dyadic
    data like the unsplit kernel."""
    m = lambda n, s: {"name": n, "shape": s, "dtype": "float64"}  # noqa: E731
    for k, e in enumerate([
        {"i_out": ["a", "c"], "i_in": [["a", "b"], ["b", "c"]], "args": [[m("A", [96, 512]), m("B", [512, 72])]]},
        {"i_out": ["z", "a", "c"], "i_in": [["z", "a", "b"], ["z", "b", "c"]], "args": [[m("A", [2, 48, 256]), m("B", [2, 256, 64])]]},
    ]):
        plan = fe.Plan(einsum=e, options={"transform": "gett_dmma/v1", "meta": ks})
        b = ref.random_bindings(e, 120 + k)
        got = run_plan(torch_cuda, plan, b)[0]
        assert np.array_equal(got, ref.evaluate(e, b)[0].real), (ks, k)


def test_gett_batched(fe, ref, torch_cuda):
    """A batch index (in A, B and C: batched matmul) rides on a fifth TMA
    dimension and the tile scheduler; repacks run per batch value in one
    launch. Exact on dyadic data."""
    m = lambda n, s, dt="float64": {"name": n, "shape": s, "dtype": dt}  # noqa: E731
    cases = [
        {"i_out": ["z", "a", "c"], "i_in": [["z", "a", "b"], ["z", "b", "c"]], "args": [[m("A", [4, 64, 96]), m("B", [4, 96, 48])]]},
        {"i_out": ["a", "z", "c"], "i_in": [["a", "z", "b"], ["b", "z", "c"]], "args": [[m("A", [72, 3, 64]), m("B", [64, 3, 48])]]},
        {"i_out": ["z", "a", "b", "c"], "i_in": [["z", "a", "b", "k"], ["z", "k", "c"]],
         "args": [[m("A", [3, 30, 40, 64]), m("B", [3, 64, 48])]]},
        {"i_out": ["z", "a", "c"], "i_in": [["z", "a", "b"], ["z", "b", "c"]],
         "args": [[m("A", [5, 50, 64], "float32"), m("B", [5, 64, 72], "float32")]]},
    ]
    for k, e in enumerate(cases):
        plan = fe.Plan(einsum=e)
        assert plan.info["transform"] == "gett_dmma/v1", (k, plan.info)
        b = ref.random_bindings(e, 60 + k)
        got = run_plan(torch_cuda, plan, b)[0]
        want = ref.evaluate(e, b)[0].real
        if got.dtype == np.float32:
            assert np.array_equal(got, want.astype(np.float32)), k
        else:
            assert np.array_equal(got, want), k


def test_gett_fp32_operands_widened(fe, ref, torch_cuda):
    """float32 TCCG operands run on the f64 DMMA GETT (widened in the pack pass,
    as the reference computes float32 in double); an fp32 output is narrowed
    once at the end. Dyadic inputs: exact sums, so the result equals the
    reference's double value rounded to float32 — bitwise. Mixed f32 / f64
    operands (f64 output) are exact too."""
    for dts, dims in [(("float32", "float32"), (2, 2, 8, 8)), (("float32", "float32"), (3, 1, 8, 16)),
                      (("float32", "float64"), (2, 2, 8, 8)), (("float64", "float32"), (1, 2, 16, 8))]:
        e = _tccg_small(ref, fe, *dims)
        for k, dt in enumerate(dts):
            e["args"][0][k]["dtype"] = dt
        plan = fe.Plan(einsum=e)
        assert plan.info["transform"] == "gett_dmma/v1", plan.info
        b = ref.random_bindings(e, sum(dims) + 5)
        got = run_plan(torch_cuda, plan, b)
        want = ref.evaluate(e, b)[0].real
        if dts == ("float32", "float32"):
            assert got[0].dtype == np.float32
            assert np.array_equal(got[0], want.astype(np.float32)), dims
        else:
            assert np.array_equal(got[0], want), dims


def test_gett_dmma_bit_exact_small(fe, ref, torch_cuda):
    """TCCG abcd-aebf-dfce through the TMA+DMMA kernel: dyadic inputs make
    every partial sum exact, so the result must equal the reference bitwise."""
    for dims in [(2, 2, 8, 8), (3, 1, 8, 16), (1, 2, 16, 8)]:
        e = _tccg_small(ref, fe, *dims)
        plan = fe.Plan(einsum=e)
        assert plan.info["transform"] == "gett_dmma/v1", plan.info
        b = ref.random_bindings(e, sum(dims))
        got = run_plan(torch_cuda, plan, b)
        want = ref.evaluate(e, b)
        assert np.array_equal(got[0], want[0].real), dims


def test_gett_functional_operands(fe, ref, torch_cuda):
    """(alpha1*A+beta1)(alpha2*B+beta2) operands (TCCG protocol, four separate
    scalars) fused into the GETT kernel."""
    fk = ("domain: a<2 b<72 c<2 d<72 e<8 f<8\n"
          "def opA(p,q,r,s) := alpha1[]*A[p,q,r,s] + beta1[]\n"
          "def opB(p,q,r,s) := alpha2[]*B[p,q,r,s] + beta2[]\n"
          "array: A float64 2x8x72x8\narray: B float64 72x8x2x8\n"
          "array: alpha1 float64 scalar\narray: beta1 float64 scalar\n"
          "array: alpha2 float64 scalar\narray: beta2 float64 scalar\n"
          "stmt C[a,b,c,d] = sum([e,f], opA(a,e,b,f)*opB(d,f,c,e))\n")
    info, arrays, b = _kernel_bindings(ref, fk, 4)
    plan = fe.Plan(kernel=fk)
    assert plan.info["transform"] == "gett_dmma/v1"
    got = run_plan(torch_cuda, plan, b)
    want = ref.eval_kernel(fk, arrays, b, 1, [2, 72, 2, 72])
    assert rel_err(got[0], want[0]) <= FP64_TOL


def test_gett_full_c3_exact_vs_torch(fe, torch_cuda):
    """C3 at full extent 72: dyadic data -> exact sums -> bitwise equal to an
    fp64 torch.einsum (cuBLAS) of the same inputs, whatever its order."""
    from paper_2601_12220_b200 import configs as C
    torch = torch_cuda
    e = C.tccg(ext=72)
    plan = fe.Plan(einsum=e)
    assert plan.info["transform"] == "gett_dmma/v1"
    A = torch.empty([72] * 4, dtype=torch.float64, device="cuda")
    B = torch.empty([72] * 4, dtype=torch.float64, device="cuda")
    fe.fill_dyadic(A, 1)
    fe.fill_dyadic(B, 2)
    (out,) = plan(A, B)
    want = torch.einsum("aebf,dfce->abcd", A, B)
    torch.cuda.synchronize()
    assert torch.equal(out, want)


@pytest.mark.parametrize("name", ["abcd-aebf-dfce", "abcd-aebf-fdec", "abcd-eafb-fdec", "abcd-eafd-fbec"])
def test_gett_tccg_siblings_exact(fe, torch_cuda, name):
    """Every TCCG sibling reading of the C3 contraction runs on the DMMA GETT
    kernel (operands whose unit-stride index is an output index are repacked
    per execute) and is exact on dyadic data against an fp64 torch.einsum."""
    from paper_2601_12220_b200 import configs as C
    torch = torch_cuda
    e = C.tccg(name, ext=72)
    plan = fe.Plan(einsum=e)
    assert plan.info["transform"] == "gett_dmma/v1", plan.info
    A = torch.empty([72] * 4, dtype=torch.float64, device="cuda")
    B = torch.empty([72] * 4, dtype=torch.float64, device="cuda")
    fe.fill_dyadic(A, 3)
    fe.fill_dyadic(B, 4)
    (out,) = plan(A, B)
    a, b = C.TCCG_SIBLINGS[name]
    want = torch.einsum(f"{a},{b}->abcd", A, B)
    torch.cuda.synchronize()
    assert torch.equal(out, want), name


@pytest.mark.parametrize("dtype,tol", [("float64", FP64_TOL), ("float32", 1e-5)])
def test_tensor_train_small(fe, ref, torch_cuda, dtype, tol):
    from paper_2601_12220_b200 import configs as C
    e = C.tensor_train(n=6, dtype=dtype)
    plan = fe.Plan(einsum=e)
    assert plan.info["transform"] == "tt/v1"
    b = ref.random_bindings(e, 12)
    got = run_plan(torch_cuda, plan, b)
    want = ref.evaluate(e, b)
    # fp32: the flat 1e-5 bar against the double-computed reference
    # on the reference's own random_bindings data
    assert rel_err(got[0], want[0]) <= tol


@pytest.mark.parametrize("dtype,tol", [("float64", FP64_TOL), ("float32", 1e-5)])
def test_tensor_train_full_vs_torch(fe, torch_cuda, dtype, tol):
    """C4 at full size (n = 4096) against an fp64 torch.einsum of the same data."""
    from paper_2601_12220_b200 import configs as C
    torch = torch_cuda
    plan = fe.Plan(einsum=C.tensor_train(n=4096, dtype=dtype))
    tdt = torch.float64 if dtype == "float64" else torch.float32
    G1 = torch.empty(64, 64, dtype=tdt, device="cuda")
    G2 = torch.empty(64, 64, dtype=tdt, device="cuda")
    X = torch.empty(4096, 64, 64, dtype=tdt, device="cuda")
    for k, t in enumerate((G1, G2, X)):
        fe.fill_dyadic(t, 30 + k)
    (Y,) = plan(G1, G2, X)
    want = torch.einsum("ij,kl,njl->nik", G1.double(), G2.double(), X.double())
    rel = lambda a: ((a.double() - want).abs() / want.abs().clamp(min=1.0)).max().item()  # noqa: E731
    assert rel(Y) <= tol  # fp32: flat 1e-5 on the config's dyadic data


@pytest.mark.parametrize("n", [1, 2, 7, 300, 4096])
@pytest.mark.parametrize("meta", ["tc=1", "tc=0"])
def test_tensor_train_f32_tensor_cores(fe, torch_cuda, n, meta):
    """fp32 C4 on tcgen05 (3xTF32 split, tc=1) and on the DMMA path (tc=0):
    full-mantissa random data (not tf32-representable), odd sample counts
    (the last pair half out of bounds), held to the fp32 bar against fp64."""
    from paper_2601_12220_b200 import configs as C
    torch = torch_cuda
    plan = fe.Plan(einsum=C.tensor_train(n=n, dtype="float32"), options={"meta": meta, "transform": "tt/v1"})
    g = torch.Generator(device="cuda").manual_seed(n)
    G1 = torch.randn(64, 64, device="cuda", generator=g)
    G2 = torch.randn(64, 64, device="cuda", generator=g)
    X = torch.randn(n, 64, 64, device="cuda", generator=g) * 3.0
    (Y,) = plan(G1, G2, X)
    torch.cuda.synchronize()
    want = torch.einsum("ij,kl,njl->nik", G1.double(), G2.double(), X.double())
    err = ((Y.double() - want).abs() / want.abs().clamp(min=1.0)).max().item()
    # plain fp32 (torch, CUDA cores) as the yardstick for "fp32 accuracy"
    f32 = torch.einsum("ij,kl,njl->nik", G1, G2, X)
    err_f32 = ((f32.double() - want).abs() / want.abs().clamp(min=1.0)).max().item()
    assert err <= max(1e-5, 4 * err_f32), (err, err_f32)


_HEX_WANT = {}


@pytest.mark.parametrize("meta", ["", "ne=2", "v=1", "v=3", "v=5", "v=6", "v=7", "v=9"])
def test_hex_sumfact_small(fe, ref, torch_cuda, meta):
    """C2's sum-factorised operator at oracle-sized extents, every kernel
    variant (default: merged C/A stages with eight fields; v=3 the
    three-barrier kernel; v=5 merged without the pass-B split; v=1 register
    planes), with shared (A_d) and six distinct forward/backward operators."""
    from paper_2601_12220_b200 import configs as C
    # E % 4 == 0 cases run the four-element stage, the others the two-element
    # one; b = 8 with E % 4 == 0 takes the merged-stage kernel
    for E, b, distinct in [(2, 1, False), (4, 3, False), (2, 8, True), (6, 5, True), (4, 2, True), (8, 1, False),
                           (8, 8, True), (12, 8, False)]:
        e = C.hex_poisson(E=E, b=b, distinct=distinct)
        opts = {"meta": meta, "transform": "hex_sumfact/v1"} if meta else None
        plan = fe.Plan(einsum=e, options=opts) if opts else fe.Plan(einsum=e)
        assert plan.info["transform"] == "hex_sumfact/v1"
        bind = ref.random_bindings(e, E + b)
        got = run_plan(torch_cuda, plan, bind)
        key = (E, b, distinct)
        if key not in _HEX_WANT:  # the oracle is slow here: evaluate once for all variants
            _HEX_WANT[key] = ref.evaluate(e, bind)
        want = _HEX_WANT[key]
        for g, w in zip(got, want):
            assert rel_err(g, w) <= FP64_TOL, (E, b)


def test_hex_sumfact_fp32(fe, ref, torch_cuda):
    """float32 arrays take the fp32 instance of the v2 hex kernel (FFMA,
    half the bytes), within the fp32 bar of the reference."""
    from paper_2601_12220_b200 import configs as C
    for E, b, distinct, P in [(4, 1, False, 5), (8, 8, True, 5), (4, 3, True, 4), (6, 2, False, 6)]:
        e = C.hex_poisson(E=E, b=b, distinct=distinct, P=P, dtype="float32")
        plan = fe.Plan(einsum=e)
        assert plan.info["transform"] == "hex_sumfact/v1", plan.info
        bind = ref.random_bindings(e, E + b + P)
        want = ref.evaluate(e, bind)
        for g, w in zip(run_plan(torch_cuda, plan, bind), want):
            assert g.dtype == np.float32 and rel_err(g, w.real) <= 1e-5, (E, b, P)


def test_hex_sumfact_large_sampled(fe, torch_cuda):
    """E = 200k elements, 8 fields (the C2 grid shape), checked on sampled
    elements against an independent fp64 torch evaluation of the same einsum."""
    from paper_2601_12220_b200 import configs as C
    torch = torch_cuda
    E = 200_000
    plan = fe.Plan(einsum=C.hex_poisson(E=E, b=8))
    assert plan.info["transform"] == "hex_sumfact/v1"
    ins = []
    for k, m in enumerate(plan.inputs):
        t = torch.empty(m["shape"], dtype=torch.float64, device="cuda")
        fe.fill_dyadic(t, 50 + k)
        ins.append(t)
    outs = plan(*ins)
    names = [m["name"] for m in plan.inputs]
    A1, A2, A3, G = (ins[names.index(n)] for n in ("A1", "A2", "A3", "G"))
    idx = torch.randint(0, E, (64,), device="cuda")
    Gs = G[:, :, idx]
    for q in range(8):
        u = ins[names.index(f"u{q + 1}")][idx]
        want = torch.einsum("xai,xbm,xcn,xyeabc,yaj,ybk,ycl,ejkl->eimn", A1, A2, A3, Gs, A1, A2, A3, u)
        got = outs[q][idx]
        err = ((got - want).abs() / want.abs().clamp(min=1.0)).max().item()
        assert err <= FP64_TOL, q


@pytest.mark.parametrize("name", ["C4-f64", "C2-small", "C3", "C1-f32-large", "hex-f32", "matmul-split", "path3",
                                  "C1-rows", "hex-rows"])
def test_execute_host_pipelined(fe, torch_cuda, name):
    """fe_plan_execute_host on plans above the pipelining threshold runs the
    chunked H2D / kernels / D2H pipeline (sub-plans along the shard axis on
    three streams); smaller plans with several rows (C1-rows: the C1 config;
    hex-rows: a small three-field hex) run the row pipeline (one single-row
    plan per row, row r's D2H under row r+1's kernels). Either way the results
    must equal the device-resident execute bitwise (the same per-element
    arithmetic on independent slices / rows)."""
    from paper_2601_12220_b200 import configs as C
    torch = torch_cuda
    if name == "C1-rows":
        plan = fe.Plan(einsum=C.fem_grad())
    elif name == "hex-rows":
        plan = fe.Plan(einsum=C.hex_poisson(E=4_000, b=3))
    elif name == "C4-f64":
        plan = fe.Plan(einsum=C.tensor_train(n=4096))
    elif name == "C2-small":
        plan = fe.Plan(einsum=C.hex_poisson(E=40_000, b=3))
    elif name == "C1-f32-large":
        plan = fe.Plan(einsum=C.fem_grad(E=2_000_000, dtype="float32"))
    elif name == "hex-f32":
        plan = fe.Plan(einsum=C.hex_poisson(E=40_000, b=3, dtype="float32"))
    elif name == "matmul-split":
        mm = lambda n, s: {"name": n, "shape": s, "dtype": "float64"}  # noqa: E731
        plan = fe.Plan(einsum={"i_out": ["a", "c"], "i_in": [["a", "b"], ["b", "c"]],
                               "args": [[mm("A", [4096, 2048]), mm("B", [2048, 1024])]]})
    elif name == "path3":
        mm = lambda n, s: {"name": n, "shape": s, "dtype": "float64"}  # noqa: E731
        plan = fe.Plan(einsum={"i_out": ["a", "d"], "i_in": [["a", "b"], ["b", "c"], ["c", "d"]],
                               "args": [[mm("A", [4096, 512]), mm("B", [512, 512]), mm("C", [512, 1024])]]})
    else:
        plan = fe.Plan(kernel=C.tccg_kernel(ext=72))
    ins = []
    for k, m in enumerate(plan.inputs):
        t = torch.empty(m["shape"], dtype=fe._torch_dtype(m["storage"]), device="cuda")
        fe.fill_dyadic(t, 70 + k)
        ins.append(t)
    want = plan(*ins)
    hin = [t.cpu().pin_memory() for t in ins]
    hout = [torch.empty(o.shape, dtype=o.dtype).pin_memory() for o in want]
    s = torch.cuda.current_stream()
    for _ in range(2):  # second call reuses the pipeline's buffers
        for h in hout:
            h.zero_()
        plan.execute_host([h.data_ptr() for h in hin], [h.data_ptr() for h in hout], s.cuda_stream)
        torch.cuda.synchronize()
        for g, w in zip(hout, want):
            if name == "path3":  # chunked sub-plans may split K differently: rounding of the 2nd step
                assert rel_err(g.numpy(), w.cpu().numpy()) <= FP64_TOL, name
            else:
                assert torch.equal(g, w.cpu()), name


@pytest.mark.parametrize("spec", [
    # (A subscripts, B subscripts, extents a b c d e f, expect the DMMA kernel)
    ("aebf", "dfce", (5, 40, 7, 50, 14, 18), True),   # short boxes, K tails (18 % 8, 14 % 4)
    ("aebf", "fdec", (3, 72, 4, 33, 10, 22), True),   # repacked B, odd ni
    ("eafd", "fbec", (30, 6, 5, 26, 8, 6), False),    # no M index fits a box: generic kernel
    ("aebf", "dfce", (2, 90, 3, 60, 8, 8), False),    # b = 90 > 72 and a = 2: generic kernel
])
def test_gett_general_extents_exact(fe, torch_cuda, spec):
    """GETT beyond extent 72: mi / ni boxes shorter than 72 (TMA zero fill,
    masked epilogue), K extents that are not box multiples, repacked operands;
    exact on dyadic data against fp64 torch.einsum. Shapes the kernel cannot
    take (an M/N extent above 72 with no alternative) stay on the generic
    kernel and are still correct."""
    torch = torch_cuda
    sa, sb, ext, dmma = spec
    lens = dict(zip("abcdef", ext))
    m = lambda n, s: {"name": n, "shape": [lens[x] for x in s], "dtype": "float64"}
    e = {"i_out": list("abcd"), "i_in": [list(sa), list(sb)], "args": [[m("A", sa), m("B", sb)]]}
    plan = fe.Plan(einsum=e)
    A = torch.empty([lens[x] for x in sa], dtype=torch.float64, device="cuda")
    B = torch.empty([lens[x] for x in sb], dtype=torch.float64, device="cuda")
    fe.fill_dyadic(A, 5)
    fe.fill_dyadic(B, 6)
    (out,) = plan(A, B)
    want = torch.einsum(f"{sa},{sb}->abcd", A, B)
    torch.cuda.synchronize()
    assert torch.equal(out, want), (spec, plan.info["transform"])
    assert (plan.info["transform"] == "gett_dmma/v1") == dmma, plan.info


@pytest.mark.parametrize("dims", [(16, 16, 16, 16), (32, 48, 24, 40), (64, 40, 64, 56), (50, 8, 20, 12)])
@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_tensor_train_padded_cores(fe, torch_cuda, dims, dtype):
    """TT cores smaller than 64 x 64 (and non-square) run the DMMA kernel on
    zero-padded tiles; against an fp64 torch.einsum (fp32: the fp32 bar)."""
    torch = torch_cuda
    NI, NJ, NK, NL = dims
    n = 37  # odd: a half-filled last pair
    m = lambda name, s: {"name": name, "shape": list(s), "dtype": dtype}
    e = {"i_out": ["n", "i", "k"], "i_in": [["i", "j"], ["k", "l"], ["n", "j", "l"]],
         "args": [[m("G1", (NI, NJ)), m("G2", (NK, NL)), m("X", (n, NJ, NL))]]}
    plan = fe.Plan(einsum=e)
    assert plan.info["transform"] == "tt/v1", plan.info
    tdt = torch.float64 if dtype == "float64" else torch.float32
    G1 = torch.randn(NI, NJ, dtype=tdt, device="cuda")
    G2 = torch.randn(NK, NL, dtype=tdt, device="cuda")
    X = torch.randn(n, NJ, NL, dtype=tdt, device="cuda")
    names = [mm["name"] for mm in plan.inputs]
    ins = {"G1": G1, "G2": G2, "X": X}
    (Y,) = plan(*[ins[k] for k in names])
    want = torch.einsum("ij,kl,njl->nik", G1.double(), G2.double(), X.double())
    err = ((Y.double() - want).abs() / want.abs().clamp(min=1.0)).max().item()
    if dtype == "float64":
        assert err <= FP64_TOL, err
    else:
        f32 = torch.einsum("ij,kl,njl->nik", G1, G2, X)
        err_f32 = ((f32.double() - want).abs() / want.abs().clamp(min=1.0)).max().item()
        assert err <= max(1e-5, 4 * err_f32), (err, err_f32)


@pytest.mark.parametrize("Q", [3, 4, 6])
def test_hex_other_orders(fe, torch_cuda, Q):
    """The v2 hex kernel templated on the points per direction (P2, P3, P5
    hexes besides C2's P4), shared and distinct operators, ragged element
    counts (the two-element stage), against an fp64 torch.einsum."""
    from paper_2601_12220_b200 import configs as C
    torch = torch_cuda
    for E, b, distinct in [(8, 3, True), (6, 8, False), (40, 5, True), (8, 8, True)]:
        e = C.hex_poisson(E=E, b=b, P=Q, distinct=distinct)
        plan = fe.Plan(einsum=e)
        assert plan.info["transform"] == "hex_sumfact/v1", plan.info
        ins = {}
        for k, m in enumerate(plan.inputs):
            t = torch.empty(m["shape"], dtype=torch.float64, device="cuda")
            fe.fill_dyadic(t, 90 + k + Q)
            ins[m["name"]] = t
        outs = plan(*[ins[m["name"]] for m in plan.inputs])
        A = [ins[f"A{d}"] for d in (1, 2, 3)]
        F = [ins[f"F{d}"] for d in (1, 2, 3)] if distinct else A
        for q in range(b):
            want = torch.einsum("xai,xbm,xcn,xyeabc,yaj,ybk,ycl,ejkl->eimn", A[0], A[1], A[2], ins["G"], F[0], F[1], F[2],
                                ins[f"u{q + 1}"])
            err = ((outs[q] - want).abs() / want.abs().clamp(min=1.0)).max().item()
            assert err <= FP64_TOL, (Q, E, b, q, err)
