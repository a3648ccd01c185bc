"""Python mirror of the feinsum API over the B200 C-ABI (include/feinsum_b200.h).

Same names, argument meaning and error behaviour as the reference C++ API
(proj/include/feinsum/*.hpp): einsums are plain dicts
``{"i_out": [...], "i_in": [[...], ...], "args": [[{"name", "shape", "dtype"}, ...], ...]}``
(the JSON transport of the C-ABI); failures raise :class:`FeinsumError`
carrying the reference's ``errc`` kind and message.

Numerics run only on the GPU through ``lib/libfeinsum_b200.so``; importing
this module without the built library raises, and evaluation without a CUDA
device raises ``FeinsumError(kind="io")`` — there is no CPU fallback.
"""
import ctypes
import json
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# FE_LIB_PATH: an alternative in-tree build of the same library (A/B kernel experiments)
LIB_PATH = os.environ.get("FE_LIB_PATH") or os.path.join(_HERE, "lib", "libfeinsum_b200.so")
HEADER_PATH = os.path.join(os.path.dirname(_HERE), "include", "feinsum_b200.h")

KINDS = {1: "domain", 2: "usage", 3: "io", 4: "cuda", 5: "internal"}
STORAGE = {"f64": 0, "f32": 1, "c128": 2, "c64": 3, "i8": 4, "i32": 5, "i64": 6, "f16": 7}
STORAGE_NP = {"f64": np.float64, "f32": np.float32, "c128": np.complex128, "c64": np.complex64,
              "i8": np.int8, "i32": np.int32, "i64": np.int64, "f16": np.float16}


class FeinsumError(RuntimeError):
    """feinsum::error: ``kind`` is "domain" | "usage" | "io" (+ "cuda", "internal")."""

    def __init__(self, code, message):
        super().__init__(message)
        self.code = code
        self.kind = KINDS.get(code, "internal")


_lib = None


def lib():
    """The loaded C-ABI library; raises ImportError if it was not built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() (make -C paper_2601_12220_b200)")
        L = ctypes.CDLL(LIB_PATH)
        L.fe_last_error.restype = ctypes.c_char_p
        L.fe_free.argtypes = [ctypes.c_void_p]
        L.fe_plan_create.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.POINTER(ctypes.c_void_p)]
        L.fe_plan_create_kernel.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.POINTER(ctypes.c_void_p)]
        L.fe_plan_create_functional.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.POINTER(ctypes.c_void_p)]
        L.fe_plan_describe.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_void_p)]
        L.fe_plan_execute.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        L.fe_plan_execute_host.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        L.fe_plan_tabulate.argtypes = [ctypes.c_void_p, ctypes.c_char_p, ctypes.c_void_p, ctypes.c_void_p,
                                       ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p]
        L.fe_plan_shard.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_char_p,
                                    ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(ctypes.c_int64),
                                    ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_void_p)]
        L.fe_plan_destroy.argtypes = [ctypes.c_void_p]
        L.fe_plan_num_inputs.argtypes = [ctypes.c_void_p]
        L.fe_plan_num_outputs.argtypes = [ctypes.c_void_p]
        L.fe_fill_dyadic.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_uint64, ctypes.c_void_p]
        L.fe_flush_l2.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p]
        L.fe_launch_probe.argtypes = [ctypes.c_void_p]
        L.fe_brute_force_isomorphic.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_uint64,
                                                ctypes.POINTER(ctypes.c_void_p)]
        L.fe_generate_random.argtypes = [ctypes.c_char_p, ctypes.c_uint64, ctypes.POINTER(ctypes.c_void_p)]
        L.fe_scramble.argtypes = [ctypes.c_char_p, ctypes.c_uint64, ctypes.POINTER(ctypes.c_void_p)]
        L.fe_induced_graph.argtypes = [ctypes.c_char_p, ctypes.c_int64, ctypes.POINTER(ctypes.c_void_p)]
        _lib = L
    return _lib


def _b(s):
    return s.encode() if isinstance(s, str) else s


def _js(obj):
    return json.dumps(obj).encode()


def _check(rc):
    if rc != 0:
        raise FeinsumError(rc, lib().fe_last_error().decode())


def _string_call(fn, *args):
    out = ctypes.c_void_p()
    _check(fn(*args, ctypes.byref(out)))
    s = ctypes.cast(out, ctypes.c_char_p).value.decode()
    lib().fe_free(out)
    return s


def _json_call(fn, *args):
    return json.loads(_string_call(fn, *args))


# ----------------------------------------------------------- host mirror --

def parse_classic(text):
    """notation.hpp parse_classic: ``.es`` document -> einsum dict."""
    return _json_call(lib().fe_parse_classic, _b(text))


def print_classic(e):
    return _string_call(lib().fe_print_classic, _js(e))


def validate(e):
    return _json_call(lib().fe_validate, _js(e))


def canonicalize(e):
    """Normal form + sigma maps (canonical -> original) + key."""
    return _json_call(lib().fe_canonicalize, _js(e))


def canonical_key(e):
    return _string_call(lib().fe_canonical_key, _js(e))


def is_isomorphic(a, b):
    return _json_call(lib().fe_is_isomorphic, _js(a), _js(b))


def brute_force_isomorphic(a, b, budget=10_000_000):
    return _json_call(lib().fe_brute_force_isomorphic, _js(a), _js(b), ctypes.c_uint64(budget))


def verify_witness(a, b, w):
    return _json_call(lib().fe_verify_witness, _js(a), _js(b), _js(w))


def generate_random(seed, **params):
    return _json_call(lib().fe_generate_random, _js(params), ctypes.c_uint64(seed))


def scramble(e, seed):
    return _json_call(lib().fe_scramble, _js(e), ctypes.c_uint64(seed))


def induced_graph(e, shuffle_seed=-1):
    return _json_call(lib().fe_induced_graph, _js(e), ctypes.c_int64(shuffle_seed))


def canonical_labeling(g):
    return _json_call(lib().fe_canonical_labeling, _js(g))


def check_compliance(g):
    return _json_call(lib().fe_check_compliance, _js(g))


def raise_kernel(fk_text):
    return _json_call(lib().fe_raise, _b(fk_text))


def identify_as_einsum(fk_text, ref):
    return _json_call(lib().fe_identify, _b(fk_text), _js(ref))


def cost(e):
    return _json_call(lib().fe_cost, _js(e))


def record_facts(path, facts):
    _check(lib().fe_record_facts(_b(path), _js(facts)))


def retrieve(path, key, device):
    return _json_call(lib().fe_retrieve, _b(path), _b(key), _b(device))


def universe(e):
    seen = {}
    for row in e["args"]:
        for m in row:
            seen.setdefault(m["name"], m)
    return [seen[k] for k in sorted(seen, key=lambda s: s.encode())]


def index_lengths(e):
    lens = {}
    for k, lst in enumerate(e["i_in"]):
        for d, s in enumerate(lst):
            lens.setdefault(s, e["args"][0][k]["shape"][d])
    return lens


# ---------------------------------------------------------------- plans --

def _ptr_array(ptrs):
    arr = (ctypes.c_void_p * max(1, len(ptrs)))(*[ctypes.c_void_p(int(p)) for p in ptrs])
    return arr


class Plan:
    """A planned batched einsum (evaluate's device path).

    ``Plan(einsum=e)`` for a plain batched einsum, ``Plan(kernel=fk_text)`` for
    a ``.fk`` loop-nest kernel with functional operands, or
    ``Plan(functional={"skeleton", "operands", "arrays"})``. ``options`` is the
    C-ABI options dict (storage, facts, device, transform).
    """

    def __init__(self, einsum=None, kernel=None, functional=None, options=None):
        L = lib()
        h = ctypes.c_void_p()
        opt = _js(options or {})
        if einsum is not None:
            _check(L.fe_plan_create(_js(einsum), opt, ctypes.byref(h)))
        elif kernel is not None:
            _check(L.fe_plan_create_kernel(_b(kernel), opt, ctypes.byref(h)))
        else:
            _check(L.fe_plan_create_functional(_js(functional), opt, ctypes.byref(h)))
        self._h = h
        self.info = _json_call(L.fe_plan_describe, h)

    @classmethod
    def _adopt(cls, handle):
        self = cls.__new__(cls)
        self._h = handle
        self.info = _json_call(lib().fe_plan_describe, handle)
        return self

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None:
            _lib.fe_plan_destroy(h)
            self._h = None

    @property
    def inputs(self):
        return self.info["inputs"]

    @property
    def outputs(self):
        return self.info["outputs"]

    def execute(self, d_in, d_out, stream=0):
        """Raw device pointers (ints), stream handle (int)."""
        _check(lib().fe_plan_execute(self._h, _ptr_array(d_in), _ptr_array(d_out), ctypes.c_void_p(int(stream))))

    def execute_host(self, h_in, h_out, stream=0):
        _check(lib().fe_plan_execute_host(self._h, _ptr_array(h_in), _ptr_array(h_out),
                                          ctypes.c_void_p(int(stream))))

    def tabulate(self, operand, d_in, d_out, first, count, stream=0):
        _check(lib().fe_plan_tabulate(self._h, _b(operand), _ptr_array(d_in), ctypes.c_void_p(int(d_out)),
                                      ctypes.c_int64(first), ctypes.c_int64(count), ctypes.c_void_p(int(stream))))

    def shard(self, rank, world, options=None):
        h = ctypes.c_void_p()
        lo, hi = ctypes.c_int64(), ctypes.c_int64()
        ax = ctypes.c_void_p()
        _check(lib().fe_plan_shard(self._h, rank, world, _js(options or {}), ctypes.byref(h), ctypes.byref(lo),
                                   ctypes.byref(hi), ctypes.byref(ax)))
        axis = ctypes.cast(ax, ctypes.c_char_p).value.decode()
        lib().fe_free(ax)
        return Plan._adopt(h), lo.value, hi.value, axis

    # -- torch convenience (device memory and streams are torch's) --
    def alloc_outputs(self, device="cuda"):
        import torch
        return [torch.empty(o["shape"], dtype=_torch_dtype(o["storage"]), device=device) for o in self.outputs]

    def __call__(self, *inputs, out=None, stream=None):
        import torch
        if len(inputs) != len(self.inputs):
            raise FeinsumError(2, f"plan takes {len(self.inputs)} inputs, got {len(inputs)}")
        for t, m in zip(inputs, self.inputs):
            if not t.is_cuda or not t.is_contiguous() or t.dtype != _torch_dtype(m["storage"]):
                raise FeinsumError(2, f"input {m['name']} must be a contiguous CUDA {_torch_dtype(m['storage'])} tensor")
        out = out if out is not None else self.alloc_outputs(inputs[0].device if inputs else "cuda")
        s = stream if stream is not None else torch.cuda.current_stream().cuda_stream
        self.execute([t.data_ptr() for t in inputs], [t.data_ptr() for t in out], s)
        return out


def _torch_dtype(storage):
    import torch
    return {"f64": torch.float64, "f32": torch.float32, "c128": torch.complex128, "c64": torch.complex64,
            "i8": torch.int8, "i32": torch.int32, "i64": torch.int64, "f16": torch.float16}[storage]


def fill_dyadic(tensor, seed, stream=None):
    import torch
    st = {torch.float64: 0, torch.float32: 1, torch.complex128: 2, torch.complex64: 3}[tensor.dtype]
    s = stream if stream is not None else torch.cuda.current_stream().cuda_stream
    _check(lib().fe_fill_dyadic(ctypes.c_void_p(tensor.data_ptr()), st, tensor.numel(), ctypes.c_uint64(seed),
                                ctypes.c_void_p(int(s))))


def flush_l2(scratch, stream=None):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream().cuda_stream
    _check(lib().fe_flush_l2(ctypes.c_void_p(scratch.data_ptr()), scratch.numel() * scratch.element_size(),
                             ctypes.c_void_p(int(s))))


# ------------------------------------------------ drop-in numeric entries --

def _run_wide(plan, bindings, device="cuda"):
    import torch
    ins = []
    for m in plan.inputs:
        a = np.asarray(bindings[m["name"]]).reshape(m["shape"])
        dt = np.complex128 if m["storage"] == "c128" else np.float64
        a = a.astype(np.complex128) if dt == np.complex128 else np.real(a).astype(np.float64)
        ins.append(torch.from_numpy(np.ascontiguousarray(a)).to(device))
    outs = plan(*ins)
    torch.cuda.synchronize()
    return [o.cpu().numpy().astype(np.complex128) for o in outs]


def evaluate(e, bindings, options=None):
    """core.hpp evaluate: one complex128 array per row, computed on the GPU.

    ``bindings`` maps every array name of ``universe(e)`` to array data; values
    are uploaded unrounded (f64, or c128 if complex), like the reference's
    complex<double> DenseArrays. ``options``: extra plan options (e.g.
    ``{"transform": "generic/v1"}`` for the bit-exact generic kernel).
    """
    errs = validate(e)
    if errs:
        raise FeinsumError(1, "invalid batched einsum:" + "".join("\n  " + s for s in errs))
    names = []
    for m in universe(e):
        if m["name"] not in bindings:
            raise FeinsumError(1, "no binding for array " + m["name"])
        a = np.asarray(bindings[m["name"]])
        if a.size != int(np.prod(m["shape"])):
            raise FeinsumError(1, "binding for array " + m["name"] + " has wrong element count")
        names.append(m["name"])
    _check(lib().fe_device_check())
    opts = {**(options or {}), "storage": "wide",
            "leaf_storage": {n: ("c128" if np.iscomplexobj(np.asarray(bindings[n])) else "f64") for n in names}}
    return _run_wide(Plan(einsum=e, options=opts), bindings)


def evaluate_kernel(fk_text, bindings, options=None):
    """parse_kernel + raise + evaluate_functional on the GPU (operands fused)."""
    _check(lib().fe_device_check())
    storage = {n: ("c128" if np.iscomplexobj(np.asarray(v)) else "f64") for n, v in bindings.items()}
    plan = Plan(kernel=fk_text, options={**(options or {}), "storage": "wide", "leaf_storage": storage})
    return _run_wide(plan, bindings)
