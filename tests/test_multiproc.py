"""N>1 host path on CPU: world_size-2 gloo processes plan the global problem,
take their shards (no collective on the data path) and all-gather only the
shard descriptors to check that the shards tile the axis, run the same tuned
transform, and that the per-rank FLOPs add up to the global count."""
import os
import socket
import sys

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, results):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2601_12220_b200 import configs as C
    from paper_2601_12220_b200 import feinsum as fe
    cases = {
        "C1": dict(einsum=C.fem_grad(E=20_000)),
        "C2": dict(einsum=C.hex_poisson(E=4_000)),
        "C3": dict(kernel=C.tccg_kernel(a_ext=144)),
        "C4": dict(einsum=C.tensor_train(n=8192)),
        "C5": dict(kernel=C.wave_kernel(E=40_000)),
        "C1-f32": dict(einsum=C.fem_grad(E=20_004, dtype="float32")),  # fp32: shards in fours
        "matmul": dict(einsum={"i_out": ["a", "c"], "i_in": [["a", "b"], ["b", "c"]],  # split-form GETT
                               "args": [[{"name": "A", "shape": [1024, 256], "dtype": "float64"},
                                         {"name": "B", "shape": [256, 96], "dtype": "float64"}]]}),
        "generic": dict(einsum={"i_out": ["i", "j"], "i_in": [["i", "k"], ["k", "j"]],
                                "args": [[{"name": "A", "shape": [6, 3], "dtype": "float64"},
                                          {"name": "B", "shape": [3, 5], "dtype": "float64"}]]}),
    }
    mine = {}
    for name, kw in cases.items():
        full = fe.Plan(options={"dry_run": True}, **kw)
        shard, lo, hi, axis = full.shard(rank, world, {"dry_run": True})
        mine[name] = (lo, hi, axis, shard.info["transform"], full.info["transform"],
                      shard.info["algorithmic_flops"], full.info["algorithmic_flops"])
    gathered = [None] * world
    dist.all_gather_object(gathered, mine)
    if rank == 0:
        results.update({"gathered": gathered})
    dist.destroy_process_group()


def test_shards_tile_the_axis_gloo():
    world = 2
    port = _free_port()
    with mp.Manager() as m:
        results = m.dict()
        mp.spawn(_worker, args=(world, port, results), nprocs=world, join=True)
        gathered = results["gathered"]
    for name in gathered[0]:
        parts = sorted((g[name] for g in gathered), key=lambda t: t[0])
        assert parts[0][0] == 0
        for a, b in zip(parts, parts[1:]):
            assert a[1] == b[0], name  # contiguous, disjoint
        assert len({p[2] for p in parts}) == 1, name  # one axis
        for p in parts:
            assert p[3] == p[4], name  # the shard runs the global plan's transform
        if name in ("C2", "C1-f32"):  # hex stages of four; fp32 FEM 16-byte rows
            assert all(p[0] % 4 == 0 for p in parts), parts
        if name != "generic":
            # replicated operand prologues (C3's shared opB) may add a little
            total = sum(p[5] for p in parts)
            assert parts[0][6] <= total <= parts[0][6] * (1 + 1e-3), name
