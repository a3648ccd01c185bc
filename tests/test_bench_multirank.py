"""bench.py's N>1 path end to end on one GPU: two ranks (gloo for the
collectives, both on cuda:0) shard the global problem, time it, max-reduce,
and verify every shard bitwise against an unsharded one-GPU evaluation, for
weak and strong scaling, the whole suite at reduced sizes (FE_BENCH_SCALE)."""
import json
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.gpu
@pytest.mark.parametrize("scaling", ["weak", "strong"])
def test_bench_two_ranks_verified(scaling):
    env = dict(os.environ, FE_DIST_BACKEND="gloo", FE_BENCH_SCALE="0.01")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={_port()}", os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--steps", "2", "--warmup", "1", "--configs", "C1,C2,C3,C4-f64,C4-f32,C5",
           "--no-e2e", "--no-cpu-baseline", "--scaling", scaling]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["scaling"] == scaling
    assert line["verify"]["ok"], line["verify"]
    assert "bitwise" in line["verify"]["method"]
    assert set(line["config"]["per_config"]) == {"C1", "C2", "C3", "C4-f64", "C4-f32", "C5"}
    for v in line["config"]["per_config"].values():
        assert v["transform"] != "generic/v1"
