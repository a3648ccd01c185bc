"""Autotuner: measure candidate parameters of each config's kernel family on
this GPU and append the results as tuning facts (the reference's
`feinsum-facts v1` format, device id "b200") keyed by the canonical key, so
every spelling of the einsum retrieves the winner.

  python tools/tune.py [--configs C1,C3,...] [--facts paper_2601_12220_b200/facts/b200.facts]

Each candidate is timed like bench.py: L2 flushed before every launch, CUDA
events on the launching stream, mean of --reps runs after --warmup runs.
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

CANDIDATES = {
    "fem_grad/v1": ["stages=4", "stages=2;te=16", "stages=4;te=16", "stages=8;te=16", "stages=3;dsmem=1",
                    "stages=2;ept=2", "stages=3;ept=2", "stages=4;ept=2", "stages=2;ept=2;te=64",
                    "stages=3;ept=2;te=64", "mma=1;stages=4"],
    "gett_dmma/v1": ["stages=2;group=12", "stages=3;group=6", "stages=3;group=12", "stages=3;group=24"],
    "tt/v1": ["stages=2"],
    "hex_sumfact/v1": [""],
    "generic/v1": [""],
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="C1,C2,C3,C4-f64,C4-f32,C5")
    ap.add_argument("--facts", default=os.path.join(ROOT, "paper_2601_12220_b200", "facts", "b200.facts"))
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=2)
    args = ap.parse_args()

    import torch

    import bench
    from paper_2601_12220_b200 import feinsum as fe

    torch.cuda.set_device(0)
    stream = torch.cuda.current_stream()
    flush = torch.empty(bench.L2_FLUSH_BYTES // 4, dtype=torch.float32, device="cuda")
    facts = []
    for name in args.configs.split(","):
        kind, payload = bench.spec(name)
        mk = (lambda opts: fe.Plan(einsum=payload, options=opts)) if kind == "einsum" else \
            (lambda opts: fe.Plan(kernel=payload, options=opts))
        base = mk({})
        transform = base.info["transform"]
        ins = []
        for k, m in enumerate(base.inputs):
            t = torch.empty(m["shape"], dtype=fe._torch_dtype(m["storage"]), device="cuda")
            fe.fill_dyadic(t, 100 + k)
            ins.append(t)
        outs = base.alloc_outputs()
        best = None
        for meta in CANDIDATES.get(transform, [""]):
            plan = mk({"meta": meta, "transform": transform}) if meta else base
            ptr_in = [t.data_ptr() for t in ins]
            ptr_out = [t.data_ptr() for t in outs]
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            tot = 0.0
            for r in range(args.warmup + args.reps):
                fe.flush_l2(flush)
                e0.record(stream)
                plan.execute(ptr_in, ptr_out, stream.cuda_stream)
                e1.record(stream)
                torch.cuda.synchronize()
                if r >= args.warmup:
                    tot += e0.elapsed_time(e1) * 1e-3
            t = tot / args.reps
            rate = base.info["algorithmic_flops"] / t
            print(f"{name:7s} {transform:15s} {meta or '(defaults)':22s} {t * 1e3:9.3f} ms {rate / 1e12:7.2f} TF/s")
            facts.append({"canonical_key": base.info["key"], "device_id": "b200", "transform_id": transform,
                          "wall_time_s": t, "flop_rate": rate, "meta": meta})
            if best is None or t < best[0]:
                best = (t, meta)
        print(f"  -> {name}: best {best[1] or '(defaults)'} {best[0] * 1e3:.3f} ms")
    os.makedirs(os.path.dirname(args.facts), exist_ok=True)
    fe.record_facts(args.facts, facts)
    print("recorded", len(facts), "facts into", args.facts)


if __name__ == "__main__":
    main()
