"""The host-side differential suites (normal
forms, keys, sigma maps, facts DB, raising, validation messages, cost model,
CLI bytes, gloo shards) re-run on the GPU box under `-m gpu`, so the driver's
GPU test record carries them too. Each runs in its own pytest process (they
are CPU tests, selected there with `-m "not gpu"`), against the compiled
reference (oracle/_ref) shipped with the snapshot.
"""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.mark.parametrize("module", ["test_canon_parity.py", "test_cli.py", "test_oracle.py", "test_multiproc.py",
                                    "test_abi.py"])
def test_host_suite(module):
    r = subprocess.run([sys.executable, "-m", "pytest", os.path.join(HERE, module), "-q", "-m", "not gpu",
                        "-p", "no:cacheprovider"], capture_output=True, text=True, timeout=900,
                       cwd=os.path.dirname(HERE))
    tail = "\n".join(r.stdout.strip().splitlines()[-5:])
    assert r.returncode == 0, tail + "\n" + r.stderr[-2000:]
    assert " passed" in tail and "failed" not in tail, tail
