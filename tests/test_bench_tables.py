"""bench.py's committed tables (CPU): the reference arm's sample FLOPs must
equal the product's own cost model on the same sample einsums, so the
reference arm can run without loading the product library."""
import bench


def test_sample_flops_match_cost_model(fe):
    for name in bench.CPU_SAMPLES:
        kind, payload = bench.cpu_sample(name)
        if kind == "tccg_slice":
            want = 2 * 72 ** 4  # C[1,1,72,72] = sum_{e,f} A B: one multiply-add per point
        elif kind == "einsum":
            want = fe.cost(payload)["algorithmic_flops"]
        else:
            want = fe.Plan(kernel=payload, options={"dry_run": True}).info["algorithmic_flops"]
        assert bench.SAMPLE_FLOPS[name] == want, name


def test_reference_arm_imports_no_product_library():
    """The reference arm's code path (cpu_sample / _cpu_worker) only reaches
    configs.py and the oracle; the product .so is never loaded by it."""
    import subprocess
    import sys
    code = ("import sys, bench; bench._cpu_worker(('C4-f64', 1)); "
            "maps = open('/proc/self/maps').read(); "
            "sys.exit(1 if 'libfeinsum_b200' in maps else (0 if 'libfeinsum_ref' in maps else 2))")
    r = subprocess.run([sys.executable, "-c", code], cwd=bench.ROOT, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, (r.returncode, r.stderr[-2000:])
