"""TEST ORACLE — ctypes view of the reference library (oracle/_ref) and the
C restatement (oracle/_build). Checker / CPU-baseline only; never imported by
the product package paper_2601_12220_b200.

The reference holds every array as complex<double> (proj/include/feinsum/
core.hpp:125-134), so buffers cross as numpy complex128.
"""
import ctypes
import json
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libfeinsum_ref.so")
PORT_SO = os.path.join(HERE, "_build", "libfeinsum_port.so")


class RefError(Exception):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code  # 1 + feinsum::errc (domain=1, usage=2, io=3); 9 other


_ref = None
_port = None


def available():
    return os.path.exists(REF_SO)


def ref():
    global _ref
    if _ref is None:
        lib = ctypes.CDLL(REF_SO)
        lib.ref_last_error.restype = ctypes.c_char_p
        lib.ref_free.argtypes = [ctypes.c_void_p]
        _ref = lib
    return _ref


def port():
    global _port
    if _port is None:
        lib = ctypes.CDLL(PORT_SO)
        lib.port_evaluate_row.restype = ctypes.c_int
        _port = lib
    return _port


def _call_str(fn, *args):
    lib = ref()
    out = ctypes.c_void_p()
    rc = fn(*args, ctypes.byref(out))
    if rc != 0:
        raise RefError(rc, lib.ref_last_error().decode())
    s = ctypes.cast(out, ctypes.c_char_p).value.decode()
    lib.ref_free(out)
    return s


def _b(s):
    return s.encode() if isinstance(s, str) else s


def _js(obj):
    return _b(json.dumps(obj))


def parse_classic(text):
    return json.loads(_call_str(ref().ref_parse_classic, _b(text)))


def print_classic(e):
    return _call_str(ref().ref_print_classic, _js(e))


def validate(e):
    return json.loads(_call_str(ref().ref_validate, _js(e)))


def canonicalize(e):
    return json.loads(_call_str(ref().ref_canonicalize, _js(e)))


def canonical_key(e):
    return _call_str(ref().ref_canonical_key, _js(e))


def generate_random(seed, **params):
    return json.loads(_call_str(ref().ref_generate_random, _js(params), ctypes.c_uint64(seed)))


def scramble(e, seed):
    return json.loads(_call_str(ref().ref_scramble, _js(e), ctypes.c_uint64(seed)))


def is_isomorphic(a, b):
    return json.loads(_call_str(ref().ref_is_isomorphic, _js(a), _js(b)))


def brute_force_isomorphic(a, b, budget=10_000_000):
    return json.loads(_call_str(ref().ref_brute_force_isomorphic, _js(a), _js(b),
                                ctypes.c_uint64(budget)))


def verify_witness(a, b, w):
    return json.loads(_call_str(ref().ref_verify_witness, _js(a), _js(b), _js(w)))


def induced_graph(e, shuffle_seed=-1):
    return json.loads(_call_str(ref().ref_induced_graph, _js(e), ctypes.c_int64(shuffle_seed)))


def canonical_labeling(g):
    return json.loads(_call_str(ref().ref_canonical_labeling, _js(g)))


def check_compliance(g):
    return json.loads(_call_str(ref().ref_check_compliance, _js(g)))


def raise_kernel(fk):
    return json.loads(_call_str(ref().ref_raise, _b(fk)))


def identify(fk, e):
    return json.loads(_call_str(ref().ref_identify, _b(fk), _js(e)))


def cost(e):
    return json.loads(_call_str(ref().ref_cost, _js(e)))


def record_facts(path, facts):
    lib = ref()
    rc = lib.ref_record_facts(_b(path), _js(facts))
    if rc != 0:
        raise RefError(rc, lib.ref_last_error().decode())


def retrieve(path, key, device):
    return json.loads(_call_str(ref().ref_retrieve, _b(path), _b(key), _b(device)))


# ---- numerics -------------------------------------------------------------

def universe(e):
    seen = {}
    for row in e["args"]:
        for m in row:
            seen.setdefault(m["name"], m)
    return [seen[k] for k in sorted(seen, key=lambda s: s.encode())]


def _ptrs(arrs):
    return (ctypes.c_void_p * len(arrs))(*[a.ctypes.data for a in arrs])


def index_lengths(e):
    lens = {}
    for k, l in enumerate(e["i_in"]):
        for d, s in enumerate(l):
            lens.setdefault(s, e["args"][0][k]["shape"][d])
    return lens


def out_shape(e):
    lens = index_lengths(e)
    return [lens[s] for s in e["i_out"]]


def evaluate(e, bindings):
    """Reference feinsum::evaluate. bindings: name -> ndarray (any numeric
    dtype; converted to complex128). Returns one complex128 array per row."""
    lib = ref()
    ins = [np.ascontiguousarray(np.asarray(bindings[m["name"]]).astype(np.complex128).reshape(m["shape"]))
           for m in universe(e)]
    shape = out_shape(e)
    outs = [np.zeros(shape, dtype=np.complex128) for _ in e["args"]]
    rc = lib.ref_evaluate(_js(e), _ptrs(ins), _ptrs(outs))
    if rc != 0:
        raise RefError(rc, lib.ref_last_error().decode())
    return outs


def eval_kernel(fk, arrays, bindings, n_rows, out_shape_):
    """raise_to_batched_einsum + evaluate_functional. arrays: declared kernel
    array metas in name order; returns n_rows complex128 outputs."""
    lib = ref()
    ins = [np.ascontiguousarray(np.asarray(bindings[m["name"]]).astype(np.complex128).reshape(m["shape"]))
           for m in sorted(arrays, key=lambda m: m["name"].encode())]
    outs = [np.zeros(out_shape_, dtype=np.complex128) for _ in range(n_rows)]
    rc = lib.ref_eval_kernel(_b(fk), _ptrs(ins), _ptrs(outs))
    if rc != 0:
        raise RefError(rc, lib.ref_last_error().decode())
    return outs


def port_evaluate(e, bindings):
    """The C restatement (evaluate_port.c); the per-row plan (loop symbols,
    positions, strides) is restated from proj/src/core.cpp:281-324."""
    lib = port()
    lens = index_lengths(e)
    out_syms = list(e["i_out"])
    red = []
    for l in e["i_in"]:
        for s in l:
            if s not in out_syms and s not in red:
                red.append(s)
    syms = out_syms + red
    pos_of = {s: i for i, s in enumerate(syms)}
    extent = (ctypes.c_int64 * max(1, len(syms)))(*[lens[s] for s in syms])
    shape = out_shape(e)
    outs = []
    for row in e["args"]:
        ndim, pos, stride, data = [], [], [], []
        keep = []
        for k, m in enumerate(row):
            a = np.ascontiguousarray(np.asarray(bindings[m["name"]]).astype(np.complex128).reshape(m["shape"]))
            keep.append(a)
            ndim.append(len(m["shape"]))
            st = 1
            ps, ss = [], []
            for d in range(len(m["shape"]) - 1, -1, -1):
                ps.append(pos_of[e["i_in"][k][d]])
                ss.append(st)
                st *= m["shape"][d]
            pos += ps[::-1]
            stride += ss[::-1]
            data.append(a)
        out = np.zeros(shape, dtype=np.complex128)
        rc = lib.port_evaluate_row(
            ctypes.c_int(len(syms)), extent, ctypes.c_int(len(out_syms)), ctypes.c_int(len(row)),
            (ctypes.c_int * max(1, len(ndim)))(*ndim), (ctypes.c_int * max(1, len(pos)))(*pos),
            (ctypes.c_int64 * max(1, len(stride)))(*stride), _ptrs(data), ctypes.c_void_p(out.ctypes.data))
        if rc != 0:
            raise MemoryError("port_evaluate_row")
        outs.append(out)
    return outs


def random_bindings(e, seed):
    """test::random_bindings (proj/tests/test_util.hpp:19-29) through the
    reference's own draw_below: mt19937_64(seed), arrays in universe (name)
    order, values m/2^19 - 1 in [-1, 1). Returns name -> float64 ndarray."""
    metas = universe(e)
    outs = [np.zeros(m["shape"], dtype=np.float64) for m in metas]
    sizes = (ctypes.c_int64 * max(1, len(outs)))(*[a.size for a in outs])
    ref().ref_random_fill(ctypes.c_uint64(seed), ctypes.c_int(len(outs)), sizes, _ptrs(outs))
    return {m["name"]: a for m, a in zip(metas, outs)}
