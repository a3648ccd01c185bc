"""The BASELINE.json workloads, spelled as batched einsums / .fk kernels.

Pinned spellings (the builder's choice, recorded in DESIGN.md):

C1  FEM P2-tet gradient   xre,xij,ej->rei, b=3 fields, E=1e4, fp64
C2  FEM P4-hex Poisson    xai,xbm,xcn,xyeabc,yaj,ybk,ycl,ejkl->eimn, b=8, E=2e6
C3  TCCG abcd-aebf-dfce   aebf,dfce->abcd at extent 72, operands (a1*A+b1)(a2*B+b2)
C4  tensor-train layer    ij,kl,njl->nik, n=4096, 64^4 per sample, fp64 / fp32
C5  FEM wave step         C1 skeleton at E=2e6 with s_q = u_q + 0.5 k_q fused

Each builder takes the extents as arguments so the parity tests can run the
same notation at oracle-sized extents.
"""


def _m(name, shape, dtype="float64"):
    return {"name": name, "shape": list(shape), "dtype": dtype}


def fem_grad(E=10_000, b=3, NX=3, NI=10, dtype="float64"):
    """C1: y_q[r,e,i] = sum_{x,j} J[x,r,e] D[x,i,j] u_q[e,j]."""
    J = _m("J", (NX, NX, E), dtype)
    D = _m("D", (NX, NI, NI), dtype)
    rows = [[J, D, _m(f"u{q + 1}", (E, NI), dtype)] for q in range(b)]
    return {"i_out": ["r", "e", "i"], "i_in": [["x", "r", "e"], ["x", "i", "j"], ["e", "j"]], "args": rows}


def fem_grad_permuted(E=10_000, b=3, NX=3, NI=10):
    """C1 spelled differently: slots reordered, indices renamed, rows reversed.
    Isomorphic to fem_grad(), so it must retrieve the same key and kernel."""
    J = _m("Jac", (NX, NX, E))
    D = _m("Dref", (NX, NI, NI))
    rows = [[_m(f"w{q}", (E, NI)), J, D] for q in reversed(range(b))]
    return {"i_out": ["p", "k", "m"], "i_in": [["k", "n"], ["a", "p", "k"], ["a", "m", "n"]], "args": rows}


def hex_poisson(E=2_000_000, b=8, P=5, ND=3, distinct=False, dtype="float64"):
    """C2: sum-factorised P4 hex operator, 8 fields sharing G and A1..A3.
    distinct=True uses six different 1-D operators (F1..F3 forward, B1..B3
    backward) instead of A_d on both sides."""
    A1, A2, A3 = (_m(f"A{d}", (ND, P, P), dtype) for d in (1, 2, 3))
    F1, F2, F3 = (_m(f"F{d}", (ND, P, P), dtype) for d in (1, 2, 3)) if distinct else (A1, A2, A3)
    G = _m("G", (ND, ND, E, P, P, P), dtype)
    rows = [[A1, A2, A3, G, F1, F2, F3, _m(f"u{q + 1}", (E, P, P, P), dtype)] for q in range(b)]
    return {"i_out": ["e", "i", "m", "n"],
            "i_in": [["x", "a", "i"], ["x", "b", "m"], ["x", "c", "n"], ["x", "y", "e", "a", "b", "c"],
                     ["y", "a", "j"], ["y", "b", "k"], ["y", "c", "l"], ["e", "j", "k", "l"]],
            "args": rows}


TCCG_SIBLINGS = {
    # TCCG C-A-B readings -> abcd
    "abcd-aebf-dfce": ("aebf", "dfce"),
    "abcd-aebf-fdec": ("aebf", "fdec"),
    "abcd-eafb-fdec": ("eafb", "fdec"),
    "abcd-eafd-fbec": ("eafd", "fbec"),
}


def tccg(name="abcd-aebf-dfce", ext=72, dtype="float64"):
    """C3 (plain operands): C[abcd] = sum_{ef} A[..] B[..]."""
    a, b = TCCG_SIBLINGS[name]
    lens = {s: ext for s in "abcdef"}
    A = _m("A", [lens[s] for s in a], dtype)
    B = _m("B", [lens[s] for s in b], dtype)
    return {"i_out": list("abcd"), "i_in": [list(a), list(b)], "args": [[A, B]]}


def tccg_kernel(name="abcd-aebf-dfce", ext=72, a_ext=None):
    """C3 with the TCCG protocol's functional operands (alpha1*A+beta1) and
    (alpha2*B+beta2), four separate runtime scalars, as a
    .fk kernel. ``a_ext`` overrides the extent of output index a (the
    multi-GPU shard axis)."""
    a, b = TCCG_SIBLINGS[name]
    lens = {s: ext for s in "abcdef"}
    lens["a"] = a_ext or ext
    da = "x".join(str(lens[s]) for s in a)
    db = "x".join(str(lens[s]) for s in b)
    return (f"domain: a<{lens['a']} b<{ext} c<{ext} d<{ext} e<{ext} f<{ext}\n"
            "def opA(p,q,r,s) := alpha1[]*A[p,q,r,s] + beta1[]\n"
            "def opB(p,q,r,s) := alpha2[]*B[p,q,r,s] + beta2[]\n"
            f"array: A float64 {da}\n"
            f"array: B float64 {db}\n"
            "array: alpha1 float64 scalar\n"
            "array: alpha2 float64 scalar\n"
            "array: beta1 float64 scalar\n"
            "array: beta2 float64 scalar\n"
            f"stmt C[a,b,c,d] = sum([e,f], opA({','.join(a)})*opB({','.join(b)}))\n")


def tensor_train(n=4096, r=64, dtype="float64"):
    """C4: Y[n,i,k] = sum_{j,l} G1[i,j] G2[k,l] X[n,j,l] (batch spelled as an index)."""
    return {"i_out": ["n", "i", "k"], "i_in": [["i", "j"], ["k", "l"], ["n", "j", "l"]],
            "args": [[_m("G1", (r, r), dtype), _m("G2", (r, r), dtype), _m("X", (n, r, r), dtype)]]}


def wave_kernel(E=2_000_000, b=3, NX=3, NI=10, renamed=False):
    """C5: the C1 skeleton with functional operands s_q = u_q + 0.5 k_q.
    ``renamed=True`` spells the same computation with renamed loop indices,
    reversed statements and reordered factors (must retrieve the same fact)."""
    if not renamed:
        lines = [f"domain: x<{NX} r<{NX} e<{E} i<{NI} j<{NI}"]
        for q in range(1, b + 1):
            lines.append(f"def s{q}(p,t) := u{q}[p,t] + 0.5*k{q}[p,t]")
        lines.append(f"array: J float64 {NX}x{NX}x{E}")
        lines.append(f"array: D float64 {NX}x{NI}x{NI}")
        for q in range(1, b + 1):
            lines.append(f"array: u{q} float64 {E}x{NI}")
            lines.append(f"array: k{q} float64 {E}x{NI}")
        for q in range(1, b + 1):
            lines.append(f"stmt y{q}[r,e,i] = sum([x,j], J[x,r,e]*D[x,i,j]*s{q}(e,j))")
        return "\n".join(lines) + "\n"
    lines = [f"domain: el<{E} dof<{NI} dir<{NX} comp<{NX} q<{NI}"]
    for q in range(1, b + 1):
        lines.append(f"def stage{q}(a,c) := 0.5*kk{q}[a,c] + uu{q}[a,c]")
    lines.append(f"array: geo float64 {NX}x{NX}x{E}")
    lines.append(f"array: dmat float64 {NX}x{NI}x{NI}")
    for q in range(1, b + 1):
        lines.append(f"array: uu{q} float64 {E}x{NI}")
        lines.append(f"array: kk{q} float64 {E}x{NI}")
    for q in reversed(range(1, b + 1)):
        lines.append(f"stmt out{q}[comp,el,dof] = sum([dir,q], stage{q}(el,q)*dmat[dir,dof,q]*geo[dir,comp,el])")
    return "\n".join(lines) + "\n"


def wave_kernel_nonlinear(E=2_000_000, b=3, NX=3, NI=10):
    """The C5 skeleton with a non-affine stage operand
    s_q = u_q^2 - sin(k_q) / (2 + exp(u_q)): evaluated by the device VM into a
    table at the start of the execute, then read by the fem_grad kernel."""
    lines = [f"domain: x<{NX} r<{NX} e<{E} i<{NI} j<{NI}"]
    for q in range(1, b + 1):
        lines.append(f"def s{q}(p,t) := u{q}[p,t]*u{q}[p,t] - sin(k{q}[p,t]) / (2 + exp(u{q}[p,t]))")
    lines += [f"array: J float64 {NX}x{NX}x{E}", f"array: D float64 {NX}x{NI}x{NI}"]
    for q in range(1, b + 1):
        lines += [f"array: u{q} float64 {E}x{NI}", f"array: k{q} float64 {E}x{NI}"]
    for q in range(1, b + 1):
        lines.append(f"stmt y{q}[r,e,i] = sum([x,j], J[x,r,e]*D[x,i,j]*s{q}(e,j))")
    return "\n".join(lines) + "\n"


SUITE = ["C1", "C2", "C3", "C4-f64", "C4-f32", "C5"]
