"""The C-ABI library loads and exports every entry point include/feinsum_b200.h
declares (no compute calls), and the C++ drop-in compiles against
include/feinsum unchanged (host checks on CPU, device checks on the GPU)."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "feinsum_b200.h")
LIB = os.path.join(ROOT, "paper_2601_12220_b200", "lib", "libfeinsum_b200.so")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\s*\*?\s*(fe_\w+)\s*\(", text, re.M)))


def test_header_declares_the_plan_api():
    syms = declared_symbols()
    for s in ("fe_plan_create", "fe_plan_execute", "fe_plan_destroy", "fe_last_error", "fe_canonicalize",
              "fe_plan_execute_host", "fe_plan_shard", "fe_retrieve"):
        assert s in syms


def test_library_exports_every_declared_symbol(fe):
    out = subprocess.run(["nm", "-D", "--defined-only", LIB], capture_output=True, text=True, check=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    missing = [s for s in declared_symbols() if s not in exported]
    assert not missing, missing
    lib = fe.lib()
    for s in declared_symbols():
        assert hasattr(lib, s)


def test_no_device_is_reported_not_faked(fe):
    """On a CPU-only host the library says so instead of computing on the CPU."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    assert fe.lib().fe_device_check() == 3
    with pytest.raises(fe.FeinsumError) as ex:
        fe.evaluate({"i_out": ["i"], "i_in": [["i"]], "args": [[{"name": "x", "shape": [3], "dtype": "float64"}]]},
                    {"x": [1.0, 2.0, 3.0]})
    assert ex.value.kind == "io"


def _build_dropin():
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tests", "cpp")], check=True)
    return os.path.join(ROOT, "tests", "cpp", "dropin_test")


def test_cpp_dropin_host(fe):
    exe = _build_dropin()
    r = subprocess.run([exe, "host"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.gpu
def test_cpp_dropin_gpu(fe):
    exe = _build_dropin()
    r = subprocess.run([exe, "gpu"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr


def test_vm_operands_planned_as_tables(fe):
    """Planning only (no device): a real-valued non-affine operand is planned
    as a tabulated leaf feeding the tuned family; a complex one (sqrt) and a
    plan with no tuned family keep the in-place VM on the generic kernel."""
    from paper_2601_12220_b200 import configs as C
    # fem_grad: the programs move into its generated prologue (no tables)
    p = fe.Plan(kernel=C.wave_kernel_nonlinear(E=2_000), options={"dry_run": True})
    assert p.info["transform"] == "fem_grad/v1" and p.info["tabulated"] == []
    assert p.info["fem_codegen"] == "nvrtc"
    assert len(p.info["inputs"]) == 2 + 2 * 3  # caller inputs only
    # tensor train: a transcendental core is tabulated by a generated kernel
    fk = ("domain: n<64 i<64 j<64 k<64 l<64\n"
          "def g(a,c) := exp(H[a,c] / 4)\n"
          "array: H float64 64x64\narray: K float64 64x64\narray: X float64 64x64x64\n"
          "stmt y[n,i,k] = sum([j,l], g(i,j)*K[k,l]*X[n,j,l])\n")
    p = fe.Plan(kernel=fk, options={"dry_run": True})
    assert p.info["transform"] == "tt/v1" and len(p.info["tabulated"]) == 1
    assert p.info["tab_codegen"] == ["nvrtc"]  # the generated kernel compiles for sm_100a
    fk = ("domain: i<6 j<3\n"
          "def f(p) := sqrt(X[p]) * reciprocal(Y[p])\n"
          "array: X float64 6\narray: Y float64 6\narray: W float64 6x3\n"
          "stmt y[j] = sum([i], f(i)*W[i,j])\n")
    p = fe.Plan(kernel=fk, options={"dry_run": True, "storage": "wide"})
    assert p.info["transform"] == "generic/v1" and p.info["tabulated"] == []
    p = fe.Plan(kernel=fk.replace("sqrt(X[p])", "exp(X[p])"), options={"dry_run": True})
    assert p.info["transform"] == "generic/v1" and p.info["tabulated"] == []
