"""The `feinsum` command line (paper_2601_12220_b200/bin/feinsum) against the
reference CLI's goldens, byte for byte: every expected string below is the
command's entire stdout+stderr as pinned by /root/reference/proj/tests/
test_cli.cpp (cited per test). Runs on CPU (no subcommand here touches the
GPU); the fixtures are the reference's, from tests/golden/fixtures.json.
"""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_2601_12220_b200", "bin", "feinsum")


@pytest.fixture(scope="module")
def fx(tmp_path_factory):
    if not os.path.exists(CLI):
        subprocess.run(["make", "-C", os.path.join(ROOT, "paper_2601_12220_b200"), "-j8"], check=True,
                       capture_output=True)
    d = tmp_path_factory.mktemp("fixtures")
    with open(os.path.join(ROOT, "tests", "golden", "fixtures.json")) as f:
        for name, text in json.load(f).items():
            (d / name).write_text(text)
    return lambda name: str(d / name)


def run(args, stdin=None):
    """stdout+stderr merged, like the reference harness's `2>&1` (test_cli.cpp:20-31)"""
    p = subprocess.run(CLI + " " + args + " 2>&1", shell=True, capture_output=True, text=True, stdin=stdin)
    return p.returncode, p.stdout


def test_canonicalize_document_key_and_witness(fx):
    # test_cli.cpp:49-62
    code, out = run("canonicalize " + fx("canon_first.es"))
    assert code == 0
    assert out == ("einsum: ab,ac->a\n"
                   "row: A0,A1\n"
                   "array: A0 float64 72x18\n"
                   "array: A1 float64 72x18\n"
                   "key: FE1|b=1|n=2|out=a|in=ab;ac|rows=A0,A1|A0=float64:72x18|A1=float64:72x18\n"
                   "rows (canonical -> input): 1 -> 1\n"
                   "slots (canonical -> input): 1 -> 1, 2 -> 2\n"
                   "indices (canonical -> input): a -> i, b -> j, c -> k\n"
                   "arrays (canonical -> input): A0 -> A, A1 -> B\n")


def test_key_only_stable_across_renamings(fx):
    # test_cli.cpp:64-70
    c1, o1 = run("canonicalize --format key-only " + fx("canon_first.es"))
    c2, o2 = run("canonicalize --format key-only " + fx("canon_second.es"))
    assert c1 == 0 and c2 == 0
    assert o1 == "FE1|b=1|n=2|out=a|in=ab;ac|rows=A0,A1|A0=float64:72x18|A1=float64:72x18\n"
    assert o2 == o1


def test_dash_reads_stdin(fx):
    # test_cli.cpp:72-76
    with open(fx("matmul.es")) as f:
        code, out = run("canonicalize --format key-only -", stdin=f)
    assert code == 0
    assert out == "FE1|b=1|n=2|out=bc|in=ac;ba|rows=A0,A1|A0=float64:4x10|A1=float64:10x4\n"


def test_isomorphic_transposed_matmul(fx):
    # test_cli.cpp:78-87
    code, out = run("isomorphic " + fx("iso_plain_first.es") + " " + fx("iso_plain_second.es"))
    assert code == 0
    assert out == ("isomorphic\n"
                   "rows (first -> second): 1 -> 1\n"
                   "slots (first -> second): 1 -> 2, 2 -> 1\n"
                   "indices (second -> first): p -> i, q -> j, r -> k\n"
                   "arrays (second -> first): X -> B, Y -> A\n")


def test_isomorphic_batched_swapped_rows_and_slots(fx):
    # test_cli.cpp:89-98
    code, out = run("isomorphic " + fx("iso_batched_first.es") + " " + fx("iso_batched_second.es"))
    assert code == 0
    assert out == ("isomorphic\n"
                   "rows (first -> second): 1 -> 2, 2 -> 1\n"
                   "slots (first -> second): 1 -> 1, 2 -> 4, 3 -> 3, 4 -> 2\n"
                   "indices (second -> first): i -> i, j -> k, k -> j\n"
                   "arrays (second -> first): P -> A, Q -> D, R -> C, S -> B\n")


def test_not_isomorphic(fx):
    # test_cli.cpp:100-104
    assert run("isomorphic " + fx("matmul.es") + " " + fx("canon_first.es")) == (0, "not isomorphic\n")


def test_match_kernel_to_reference(fx):
    # test_cli.cpp:106-114
    code, out = run("match " + fx("squared_kernel.fk") + " " + fx("squared_ref.es"))
    assert code == 0
    assert out == ("match\n"
                   "rows (reference -> statement): 1 -> 1, 2 -> 2\n"
                   "indices (reference -> kernel): i -> i0, j -> i1\n"
                   "arrays (reference -> kernel): A -> u, B -> v, C -> w\n")


def test_match_rejects_other_computation(fx):
    # test_cli.cpp:116-123
    code, out = run("match " + fx("squared_kernel.fk") + " " + fx("canon_first.es"))
    assert code == 1
    assert "kernel does not compute the reference einsum" in out
    assert "reference key: FE1|b=1" in out
    assert "kernel key:    FE1|b=2" in out


def test_stats_every_preset(fx):
    # test_cli.cpp:125-135
    code, out = run("stats " + fx("gemm1024.es"))
    assert code == 0
    assert out == ("flops: 2147483648\n"
                   "bytes: 25165824\n"
                   "intensity: 85.333333333333329\n"
                   "device mi250x: roofline 14.9, compute bound\n"
                   "device h100: roofline 12.550000000000001, compute bound\n"
                   "device titanv: roofline 9.4100000000000001, compute bound\n"
                   "device p100: roofline 7.2400000000000002, compute bound\n")


def test_stats_one_preset_memory_bound(fx):
    # test_cli.cpp:137-145
    code, out = run("stats --device h100 " + fx("squared_ref.es"))
    assert code == 0
    assert out == ("flops: 1536\n"
                   "bytes: 4672\n"
                   "intensity: 0.32876712328767121\n"
                   "device h100: roofline 0.32876712328767121, memory bound\n")


def test_record_then_retrieve_through_scrambled_spelling(fx, tmp_path):
    # test_cli.cpp:147-171
    db = " --db " + str(tmp_path / "facts.db")
    code, out = run("record " + fx("canon_first.es") + db + " --device h100 --wall 0.5 --meta tile=8")
    assert code == 0
    assert out == "recorded FE1|b=1|n=2|out=a|in=ab;ac|rows=A0,A1|A0=float64:72x18|A1=float64:72x18\n"
    code, _ = run("record " + fx("canon_first.es") + db + " --device h100 --transform split-k --wall 0.25")
    assert code == 0
    code, out = run("retrieve " + fx("canon_second.es") + db + " --device h100")
    assert code == 0
    assert out.startswith("key: FE1|b=1|n=2|out=a|in=ab;ac|rows=A0,A1|A0=float64:72x18|A1=float64:72x18\n")
    assert "transform: split-k\n" in out
    assert "wall_time_s: 0.25\n" in out
    assert "flop_rate: 186624\n" in out  # 46656 flops / 0.25 s
    assert "recorded_at: 20" in out
    assert run("retrieve " + fx("canon_first.es") + db + " --device p100") == (0, "no facts for this einsum on p100\n")


def test_exit_codes(fx, tmp_path):
    # test_cli.cpp:173-197: usage 2, io 3, malformed input 1
    assert run("frobnicate")[0] == 2
    assert run("")[0] == 2
    assert run("canonicalize " + fx("matmul.es") + " extra")[0] == 2
    code, out = run("stats --device tpu " + fx("gemm1024.es"))
    assert code == 2
    assert "error: unknown device tpu (have: mi250x h100 titanv p100)" in out
    assert run("canonicalize /nonexistent_einsum_file.es") == (3, "error: cannot read /nonexistent_einsum_file.es\n")
    bad = tmp_path / "bad.es"
    bad.write_text("einsum: ij->\nrow: A\n")
    assert run("canonicalize " + str(bad)) == (1, "error: line 2: array A has no array line\n")


def test_fuzz_self_check(fx):
    # test_cli.cpp:199-203
    assert run("fuzz --count 5") == (0, "ok: 5 cases\n")


def test_options_and_help(fx):
    """B200 CLI specifics: --opt=value form, --format values checked, help exits 0,
    missing required options are usage errors, tune without a GPU is an io error."""
    assert run("canonicalize --format=key-only " + fx("matmul.es"))[1].startswith("FE1|b=1|n=2|out=bc")
    assert run("canonicalize --format json " + fx("matmul.es"))[0] == 2
    assert run("--help")[0] == 0
    assert run("record " + fx("matmul.es") + " --device h100")[0] == 2  # --wall is required
    assert run("retrieve " + fx("matmul.es"))[0] == 2  # --device is required


@pytest.mark.gpu
def test_tune_records_facts_that_retrieve_finds(fx, tmp_path):
    """`tune` times the planned transform under candidate parameter sets on the
    GPU and records one fact per candidate; `retrieve` (any spelling) returns
    the fastest one with device b200."""
    db = str(tmp_path / "tuned.db")
    code, out = run("tune " + fx("gemm1024.es") + " --db " + db + " --candidates ,, --reps 2 --warmup 1")
    assert code == 0, out
    assert "recorded 3 facts" in out
    code, out = run("retrieve " + fx("gemm1024.es") + " --db " + db + " --device b200")
    assert code == 0
    assert "transform: " in out and "wall_time_s: " in out
