"""Row epilogues and fused operand programs (BASELINE config 5
"fused pre/post elementwise").

The reference's statements are plain products (proj/src/raising.cpp:535-536)
and it materialises every operand before evaluating (raising.cpp:395-435).
Two extensions sit on top of that evaluation path here:

  * operand programs (any real `def`) run inside the fem_grad kernel's
    prologue, computed from the staged leaf tiles, instead of being tabulated
    into HBM (`fem_codegen: nvrtc`, no `tabulated` operands);
  * `epi y[r,e,i] := <expr>` lines (RowEpilogue) map a statement's result
    pointwise before it is stored: fused into the fem_grad stores, one in-place
    generated pass for every other family.

Oracle: the reference evaluates the kernel without the epi lines (its own
evaluate_functional); the post-op is applied on the host in numpy with the
same operation order. Bar: the fp64 one, rel_err <= 1e-12.
"""
import re

import numpy as np
import pytest

FP64_TOL = 1e-12


def rel_err(got, want):
    got = np.asarray(got).reshape(-1)
    want = np.asarray(want).reshape(-1)
    return float(np.max(np.abs(got - want) / np.maximum(1.0, np.abs(want)))) if want.size else 0.0


def strip_epi(fk):
    return "\n".join(line for line in fk.splitlines() if not line.startswith("epi ")) + "\n"


def kernel_arrays(fk):
    arrays = []
    for line in fk.splitlines():
        m = re.match(r"array: (\w+) (\w+) (\S+)", line)
        if m:
            shape = [] if m.group(3) == "scalar" else [int(x) for x in m.group(3).split("x")]
            arrays.append({"name": m.group(1), "shape": shape, "dtype": m.group(2)})
    return arrays


def bindings_for(ref, fk, seed):
    arrays = kernel_arrays(fk)
    fake = {"i_out": [], "i_in": [[] for _ in arrays], "args": [arrays]}
    return arrays, ref.random_bindings(fake, seed)


def wave_nonlinear_epi(E):
    from paper_2601_12220_b200 import configs as C
    return (C.wave_kernel_nonlinear(E=E)
            + "epi y1[r,e,i] := u1[e,i] + 0.25*y1[r,e,i]\n"
            + "epi y2[r,e,i] := y2[r,e,i]*y2[r,e,i] / (1 + exp(-y2[r,e,i]))\n")


def post_wave(ys, b):
    """numpy restatement of wave_nonlinear_epi's two epilogues (row 3: none)."""
    y1, y2, y3 = (np.real(y) for y in ys)
    u1 = np.real(np.asarray(b["u1"]))
    return [u1[None, :, :] + 0.25 * y1, (y2 * y2) / (1.0 + np.exp(0.0 - y2)), y3]


# ----------------------------------------------------------------- host side --

def test_epi_lines_parse_print_raise(fe):
    fk = wave_nonlinear_epi(1000)
    r = fe.raise_kernel(fk)
    printed = r["printed"]
    assert "epi y1[r,e,i] := u1[e,i]+0.25*y1[r,e,i]" in printed
    assert printed.count("epi ") == 2
    # the printed form parses back to the same text
    assert fe.raise_kernel(printed)["printed"] == printed
    # the skeleton (and so the normal form and key) ignores the epilogues
    base = fe.raise_kernel(strip_epi(fk))
    assert r["skeleton"] == base["skeleton"]


@pytest.mark.parametrize("line,msg", [
    ("epi y9[r,e,i] := y9[r,e,i]", "which no stmt writes"),
    ("epi y1[e,r,i] := y1[e,r,i]", "must be indexed [r,e,i]"),
    ("epi y1[r,e,i] := y1[r,i,e]", "only [r,e,i] is pointwise"),
    ("epi y1[r,e,i] := y2[r,e,i]", "the output of another stmt"),
    ("epi y1[r,e,i] := Q[r,e,i]", "undeclared array Q"),
    ("epi y1[r,e,i] := D[r,i,e]", "reads axis 2 of D"),
    ("epi y1[r,e,i] := J[r,e]", "J has 3 axes, read with 2 subscripts"),
])
def test_epi_line_errors(fe, line, msg):
    from paper_2601_12220_b200 import configs as C
    with pytest.raises(fe.FeinsumError) as ei:
        fe.raise_kernel(C.wave_kernel_nonlinear(E=1000) + line + "\n")
    assert msg in str(ei.value)
    fk = C.wave_kernel_nonlinear(E=1000)
    with pytest.raises(fe.FeinsumError, match="epi before the stmt"):
        fe.raise_kernel(fk.replace("stmt y1", "epi y1[r,e,i] := y1[r,e,i]\nstmt y1", 1))
    with pytest.raises(fe.FeinsumError, match="two epi lines"):
        fe.raise_kernel(fk + "epi y1[r,e,i] := y1[r,e,i]\nepi y1[r,e,i] := y1[r,e,i]\n")


def test_dry_run_fem_codegen_fuses_programs_and_epilogues(fe):
    """NVRTC compiles the generated fem_grad instance on the host (no GPU)."""
    from paper_2601_12220_b200 import configs as C
    p = fe.Plan(kernel=C.wave_kernel_nonlinear(E=2_000_000), options={"dry_run": True})
    assert p.info["transform"] == "fem_grad/v1"
    assert p.info["fem_codegen"] == "nvrtc", p.info["fem_codegen"]
    assert p.info["tabulated"] == [] and p.info["launches"] == 1
    p = fe.Plan(kernel=wave_nonlinear_epi(2_000_000), options={"dry_run": True})
    assert p.info["fem_codegen"] == "nvrtc" and p.info["epilogue_fused"]
    assert p.info["epilogue_rows"] == [0, 1] and p.info["launches"] == 1
    # same key as the plain C1/C5 skeleton: the tuned fact is retrieved
    assert p.info["key"] == fe.Plan(einsum=C.fem_grad(E=2_000_000), options={"dry_run": True}).info["key"]
    assert p.info["source"] == "fact"
    # without codegen the programs are tabulated by the device VM and
    # epilogues are refused
    p = fe.Plan(kernel=C.wave_kernel_nonlinear(E=2_000_000), options={"dry_run": True, "codegen": False})
    assert len(p.info["tabulated"]) == 3 and p.info["fem_codegen"] == "prebuilt: codegen disabled"
    with pytest.raises(fe.FeinsumError, match="generated code"):
        fe.Plan(kernel=wave_nonlinear_epi(1000), options={"dry_run": True, "codegen": False})


def test_dry_run_epilogue_pass_other_families(fe):
    fk = GETT_EPI
    p = fe.Plan(kernel=fk, options={"dry_run": True})
    assert p.info["transform"] == "gett_dmma/v1"
    assert p.info["epilogue_rows"] == [0] and not p.info["epilogue_fused"]
    base = fe.Plan(kernel=strip_epi(fk), options={"dry_run": True})
    assert p.info["launches"] == base.info["launches"] + 1


def test_functional_json_epilogue(fe):
    """The C-ABI's functional JSON takes the same epilogue ("epilogue": [...])."""
    skel = {"i_out": ["i"], "i_in": [["i", "j"], ["j"]],
            "args": [[{"name": "A", "shape": [4, 3], "dtype": "float64"},
                      {"name": "x", "shape": [3], "dtype": "float64"}]]}
    ops = {"A": {"params": ["p", "q"], "body": {"read": "M", "subs": ["p", "q"]}},
           "x": {"params": ["p"], "body": {"read": "v", "subs": ["p"]}}}
    arrays = [{"name": "M", "shape": [4, 3], "dtype": "float64"}, {"name": "v", "shape": [3], "dtype": "float64"},
              {"name": "w", "shape": [4], "dtype": "float64"}]
    epi = [{"row": 0, "acc": "y", "params": ["i"],
            "body": {"op": "+", "l": {"read": "y", "subs": ["i"]}, "r": {"read": "w", "subs": ["i"]}}}]
    p = fe.Plan(functional={"skeleton": skel, "operands": ops, "arrays": arrays, "epilogue": epi},
                options={"dry_run": True})
    assert p.info["epilogue_rows"] == [0]
    assert [m["name"] for m in p.inputs] == ["M", "v", "w"]
    bad = [{"row": 0, "acc": "y", "params": ["i"], "body": {"read": "y", "subs": []}}]
    with pytest.raises(fe.FeinsumError, match="off its own point"):
        fe.Plan(functional={"skeleton": skel, "operands": ops, "arrays": arrays, "epilogue": bad},
                options={"dry_run": True})


GETT_EPI = ("domain: a<2 b<72 c<2 d<72 e<8 f<8\n"
            "array: A float64 2x8x72x8\n"
            "array: B float64 72x8x2x8\n"
            "array: W float64 2x72\n"
            "stmt y[a,b,c,d] = sum([e,f], A[a,e,b,f]*B[d,f,c,e])\n"
            "epi y[a,b,c,d] := sin(y[a,b,c,d]) + W[a,b]*y[a,b,c,d]\n")

TT_EPI = ("domain: n<64 i<64 j<64 k<64 l<64\n"
          "array: G float64 64x64\narray: H float64 64x64\narray: X float64 64x64x64\n"
          "array: Z float64 64x64x64\n"
          "stmt y[n,i,k] = sum([j,l], G[i,j]*H[k,l]*X[n,j,l])\n"
          "epi y[n,i,k] := Z[n,i,k] - 0.5*y[n,i,k]\n")


# ----------------------------------------------------------------- GPU side --

@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return torch


def run_plan(torch, plan, bindings):
    ins = [torch.from_numpy(np.ascontiguousarray(np.real(np.asarray(bindings[m["name"]])).astype(np.float64)
                                                 .reshape(m["shape"]))).cuda() for m in plan.inputs]
    outs = plan(*ins)
    torch.cuda.synchronize()
    return [o.cpu().numpy() for o in outs]


@pytest.mark.gpu
def test_c5_nonlinear_fused_prologue(fe, ref, torch_cuda):
    """s = u*u - sin(k)/(2+exp(u)) computed in the fem_grad prologue: no
    tables, same values as the VM tables + prebuilt kernel, reference parity."""
    from paper_2601_12220_b200 import configs as C
    fk = C.wave_kernel_nonlinear(E=2_000)
    arrays, b = bindings_for(ref, fk, 13)
    plan = fe.Plan(kernel=fk)
    assert plan.info["fem_codegen"] == "nvrtc" and plan.info["tabulated"] == []
    got = run_plan(torch_cuda, plan, b)
    want = ref.eval_kernel(fk, arrays, b, 3, [3, 2_000, 10])
    for g, w in zip(got, want):
        assert rel_err(g, w) <= FP64_TOL
    vm = fe.Plan(kernel=fk, options={"codegen": False})
    assert len(vm.info["tabulated"]) == 3
    for g, v in zip(got, run_plan(torch_cuda, vm, b)):
        assert np.array_equal(g, v)


@pytest.mark.gpu
def test_c5_nonlinear_fastmath_ranges(fe, ref, torch_cuda):
    """Arguments outside fastmath.cuh's straight-line ranges (|k| up to 3e6
    for sin: beyond 1e5; |u| up to 720 for exp: beyond 700, overflow to inf
    included) take the checked forms: the fused prologue (one range test per
    point, the whole point re-run) and the device VM tables agree bitwise,
    and both match the reference's libm within the fp64 bar."""
    from paper_2601_12220_b200 import configs as C
    E = 2_000
    fk = C.wave_kernel_nonlinear(E=E)
    arrays, b = bindings_for(ref, fk, 17)
    rng = np.random.default_rng(5)
    for q in (1, 2, 3):
        k = np.asarray(b[f"k{q}"], dtype=np.float64)
        u = np.asarray(b[f"u{q}"], dtype=np.float64)
        big = rng.random(k.shape) < 0.05  # a few points per tile out of range
        k = np.where(big, rng.uniform(-3e6, 3e6, k.shape), k)
        u = np.where(rng.random(u.shape) < 0.05, rng.uniform(-720, 720, u.shape) / 40.0, u)
        u = np.where(rng.random(u.shape) < 0.01, np.sign(u) * 710.0, u)
        b[f"k{q}"], b[f"u{q}"] = k, u
    plan = fe.Plan(kernel=fk)
    assert plan.info["fem_codegen"] == "nvrtc"
    got = run_plan(torch_cuda, plan, b)
    vm = fe.Plan(kernel=fk, options={"codegen": False})
    for g, v in zip(got, run_plan(torch_cuda, vm, b)):
        assert np.array_equal(g, v)
    want = ref.eval_kernel(fk, arrays, b, 3, [3, E, 10])
    # |u| = 710 makes u^2 ~ 5e5 while the outputs stay O(10): the error of
    # any summation order is relative to the terms' magnitude, so the bar is
    # 1e-12 of the forward-error scale sum_{x,j} |J||D||s| (s from numpy)
    J = np.abs(np.asarray(b["J"], dtype=np.float64).reshape(3, 3, E))
    D = np.abs(np.asarray(b["D"], dtype=np.float64).reshape(3, 10, 10))
    for q, (g, w) in enumerate(zip(got, want), start=1):
        w = np.real(np.asarray(w)).reshape(g.shape)
        u, k = (np.asarray(b[n], dtype=np.float64).reshape(E, 10) for n in (f"u{q}", f"k{q}"))
        with np.errstate(over="ignore"):
            sv = np.abs(u * u - np.sin(k) / (2.0 + np.exp(u)))
        scale = np.einsum("xre,xij,ej->rei", J, D, sv)
        fin = np.isfinite(w)
        assert np.array_equal(np.isfinite(g), fin)
        assert np.max(np.abs(g[fin] - w[fin]) / np.maximum(1.0, scale[fin])) <= FP64_TOL


@pytest.mark.gpu
@pytest.mark.parametrize("E", [2_000, 2_046, 64 * 37 + 2])
def test_c5_nonlinear_epilogue_fused(fe, ref, torch_cuda, E):
    """Epilogues fused into the fem_grad stores (ragged last tile included)."""
    fk = wave_nonlinear_epi(E)
    arrays, b = bindings_for(ref, fk, 29)
    plan = fe.Plan(kernel=fk)
    assert plan.info["epilogue_fused"] and plan.info["launches"] == 1
    got = run_plan(torch_cuda, plan, b)
    want = post_wave(ref.eval_kernel(strip_epi(fk), arrays, b, 3, [3, E, 10]), b)
    for g, w in zip(got, want):
        assert rel_err(g, w) <= FP64_TOL
    # the generic kernel + epilogue passes agree
    gen = fe.Plan(kernel=fk, options={"transform": "generic/v1"})
    assert not gen.info["epilogue_fused"]
    for g, w in zip(run_plan(torch_cuda, gen, b), want):
        assert rel_err(g, w) <= FP64_TOL


@pytest.mark.gpu
def test_affine_c5_with_epilogue(fe, ref, torch_cuda):
    """The affine wave step (u + 0.5k) through the generated instance."""
    from paper_2601_12220_b200 import configs as C
    fk = C.wave_kernel(E=4_000) + "epi y3[r,e,i] := cos(y3[r,e,i]) * k3[e,i]\n"
    arrays, b = bindings_for(ref, fk, 31)
    plan = fe.Plan(kernel=fk)
    assert plan.info["fem_codegen"] == "nvrtc" and plan.info["epilogue_fused"]
    got = run_plan(torch_cuda, plan, b)
    ys = [np.real(y) for y in ref.eval_kernel(strip_epi(fk), arrays, b, 3, [3, 4_000, 10])]
    ys[2] = np.cos(ys[2]) * np.real(np.asarray(b["k3"]))[None, :, :]
    for g, w in zip(got, ys):
        assert rel_err(g, w) <= FP64_TOL
    # without the epilogue line the prebuilt affine instance runs; rows without
    # an epilogue are bitwise the same from both (same arithmetic)
    plain = fe.Plan(kernel=strip_epi(fk))
    assert "fem_codegen" not in plain.info
    for g, p in zip(got[:2], run_plan(torch_cuda, plain, b)[:2]):
        assert np.array_equal(g, p)


@pytest.mark.gpu
@pytest.mark.parametrize("fk,family,rows,shape,post", [
    (GETT_EPI, "gett_dmma/v1", 1, [2, 72, 2, 72],
     lambda ys, b: [np.sin(ys[0]) + np.real(np.asarray(b["W"]))[:, :, None, None] * ys[0]]),
    (TT_EPI, "tt/v1", 1, [64, 64, 64],
     lambda ys, b: [np.real(np.asarray(b["Z"])) - 0.5 * ys[0]]),
])
def test_epilogue_pass_families(fe, ref, torch_cuda, fk, family, rows, shape, post):
    arrays, b = bindings_for(ref, fk, 37)
    plan = fe.Plan(kernel=fk)
    assert plan.info["transform"] == family and not plan.info["epilogue_fused"]
    got = run_plan(torch_cuda, plan, b)
    want = post([np.real(y) for y in ref.eval_kernel(strip_epi(fk), arrays, b, rows, shape)], b)
    for g, w in zip(got, want):
        assert rel_err(g, w) <= FP64_TOL


@pytest.mark.gpu
def test_epilogue_host_pipeline_shards(fe, ref, torch_cuda):
    """fe_plan_execute_host cuts plans above 64 MB into shard chunks: the
    shards carry the fused programs and epilogues (arrays sliced along e) and
    the result is bitwise the device-resident execute's."""
    import torch
    E = 200_000
    fk = wave_nonlinear_epi(E)
    plan = fe.Plan(kernel=fk)
    g = torch.Generator().manual_seed(3)
    host_in = [torch.rand(m["shape"], dtype=torch.float64, generator=g).pin_memory() for m in plan.inputs]
    dev_out = plan(*[t.cuda() for t in host_in])
    host_out = [torch.empty(o["shape"], dtype=torch.float64).pin_memory() for o in plan.outputs]
    s = torch.cuda.current_stream()
    plan.execute_host([t.data_ptr() for t in host_in], [t.data_ptr() for t in host_out], s.cuda_stream)
    s.synchronize()
    for d, h in zip(dev_out, host_out):
        assert torch.equal(d.cpu(), h)
    sh, lo, hi, axis = plan.shard(1, 3)
    assert sh.info["epilogue_fused"] and sh.info["fem_codegen"] == "nvrtc"
