"""Benchmark: geomean GFLOP/s (and roofline fraction) over the TCCG+FEM
batched-einsum suite of BASELINE.json, on 1-8 B200s.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--configs C1,C5,...]
  python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N
  python bench.py --impl reference      # the reference CPU evaluator arm

A step evaluates every config of the suite once (one plan execution each).
Inputs are synthetic dyadic values generated on the device; every config is
preceded by an L2 flush (256 MiB written, then read back so the L2 is
also clean) and timed alone with CUDA events on
the launching stream; per-config times are max-reduced over ranks. FLOPs are
the algorithmic (optimal pairwise contraction path) counts, operand FLOPs of
functional operands included.

Multi-GPU: each config is sharded along its element/batch axis, no collective
on the hot path. --scaling weak (default): the global problem is world x the
config, every rank holds one config-sized shard; --scaling strong: the config
itself is split N ways (BASELINE config 2: one 2M-element mesh over 1-8 GPUs).
Shard outputs are verified bitwise against an unsharded one-GPU evaluation.

Extra lines (not in the geomean, one GPU): the launch floor, C1 in a CUDA
graph, C1 at E=2e6, the TCCG siblings of C3, the 3xTF32 C4-f32.
"""
import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

L2_FLUSH_BYTES = 256 << 20

# per-config workload: builder, plan kind, bound, element-axis sample for the CPU baseline
CONFIG_DOC = {
    "C1": "FEM P2-tet gradient xre,xij,ej->rei b=3 E=1e4 fp64",
    "C2": "FEM P4-hex sum-factorised Poisson b=8 E=2e6 fp64",
    "C3": "TCCG abcd-aebf-dfce extent 72 fp64, operands alpha*A+beta",
    "C4-f64": "tensor-train ij,kl,njl->nik n=4096 r=64 fp64",
    "C4-f32": "tensor-train ij,kl,njl->nik n=4096 r=64 fp32",
    "C5": "FEM wave step: C1 skeleton E=2e6 with s=u+0.5k fused",
}


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--configs", default="C1,C2,C3,C4-f64,C4-f32,C5")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=2.0, help="target seconds per CPU sample")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="weak: world x the config, one config-sized shard per rank; strong: the config split N ways")
    ap.add_argument("--no-extras", action="store_true", help="skip the extra (non-geomean) lines")
    return ap.parse_args()


# ------------------------------------------------------------------ specs --

def spec(name, scale=1.0):
    """(kind, payload) for a config; scale multiplies the sharded axis (world
    copies for weak scaling, a fraction for the CPU samples). FE_BENCH_SCALE
    shrinks the base extent first (reduced sizes for the multi-rank tests on
    one GPU), so world x the base is exactly world one-GPU shards."""
    from paper_2601_12220_b200 import configs as C
    env = float(os.environ.get("FE_BENCH_SCALE", "1"))

    def ext(full, even=False):
        base = max(2 if even else 1, int(full * env))
        if even:
            base = base // 2 * 2
        v = max(2 if even else 1, int(round(base * scale)))
        return v // 2 * 2 if even else v

    if name == "C1":
        return "einsum", C.fem_grad(E=ext(10_000, even=True))
    if name == "C2":
        return "einsum", C.hex_poisson(E=ext(2_000_000))
    if name == "C3":
        return "kernel", C.tccg_kernel(ext=72, a_ext=max(1, int(round(72 * scale))))
    if name == "C4-f64":
        return "einsum", C.tensor_train(n=ext(4096))
    if name == "C4-f32":
        return "einsum", C.tensor_train(n=ext(4096), dtype="float32")
    if name == "C5":
        return "kernel", C.wave_kernel(E=ext(2_000_000, even=True))
    raise ValueError(name)


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback"


# -------------------------------------------------------------- clocks ----

class ClockSampler:
    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def wait_first(self, timeout=5.0):
        """Block until nvidia-smi delivered its first sample (it needs ~0.3 s
        to start), so the samples cover the timed region."""
        t0 = time.time()
        while self.proc and not self.rows and time.time() - t0 < timeout:
            time.sleep(0.02)

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 9:
                self.rows.append(parts)

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = sorted(float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit())
        mx = max((float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()), default=None)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[5 + i].lower() == "active"})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(self.rows)}


# ------------------------------------------------------------ GPU arm -----

def bithash(torch, t):
    """Exact checksum of a tensor's bit patterns (int64 sums wrap mod 2^64,
    so the reduction order does not matter): equal hashes <=> bitwise equal
    up to astronomically unlikely collisions."""
    x = t.contiguous().view(-1)
    x = x.view(torch.int64) if x.element_size() == 8 else x.view(torch.int32).to(torch.int64)
    w = torch.arange(x.numel(), device=x.device, dtype=torch.int64) % 8191 + 1
    return [int(x.sum().item()), int((x * w).sum().item())]


def shard_dim(full_shape, part_shape):
    """The dimension a shard plan cut (None: replicated array)."""
    for d, (a, b) in enumerate(zip(full_shape, part_shape)):
        if a != b:
            return d
    return None


class Workload:
    def __init__(self, name, rank, world, torch, fe, seed, scaling="weak", extra=None):
        # weak scaling: the global problem is `world` copies of the config along
        # its shard axis; each rank plans the global einsum (same canonical
        # form family, same tuned transform) and runs its 1/world shard, which
        # is exactly the single-GPU config. strong scaling: the global problem
        # is the config itself (C2: one 2M-element mesh split N ways); every
        # rank fills the same global inputs from one seed and keeps its slice.
        self.name = name
        self.scaling = scaling
        self.options = (extra or {}).get("options")
        if extra is not None:
            kind, payload = extra["kind"], extra["payload"]
        else:
            kind, payload = spec(name, scale=world) if (world > 1 and scaling == "weak") else spec(name)
        self.kind, self.payload = kind, payload
        opts = self.options or {}
        full = fe.Plan(einsum=payload, options=opts) if kind == "einsum" else fe.Plan(kernel=payload, options=opts)
        self.full = full
        if world > 1:
            self.plan, self.lo, self.hi, self.axis = full.shard(rank, world)
        else:
            self.plan, self.lo, self.hi, self.axis = full, 0, 0, ""
        info = self.plan.info
        self.transform = info["transform"]
        self.pipe = info.get("pipe", "dfma")
        self.source = info["source"]
        self.key = full.info["key"]
        self.flops = info["algorithmic_flops"]  # this rank's shard
        self.global_flops = full.info["algorithmic_flops"]
        self.bytes = info["bytes"]
        self.ref_flops = info["reference_flops"]
        dev = torch.device("cuda", torch.cuda.current_device())
        self.seed = seed
        if world > 1 and scaling == "strong":
            self.ins = [t for t in self.slice_inputs(torch, fe, self.global_inputs(torch, fe, dev))]
        else:
            self.ins = []
            for k, m in enumerate(self.plan.inputs):
                t = torch.empty(m["shape"], dtype=fe._torch_dtype(m["storage"]), device=dev)
                fe.fill_dyadic(t, seed * 1000 + k)
                self.ins.append(t)
        self.outs = self.plan.alloc_outputs(dev)
        self.launches = int(info.get("launches", 1))  # kernels per execute (plan describe)

    def global_inputs(self, torch, fe, dev):
        ins = []
        for k, m in enumerate(self.full.inputs):
            t = torch.empty(m["shape"], dtype=fe._torch_dtype(m["storage"]), device=dev)
            fe.fill_dyadic(t, self.seed * 1000 + k)
            ins.append(t)
        return ins

    def slice_inputs(self, torch, fe, gins):
        out = []
        for g, mf, mp in zip(gins, self.full.inputs, self.plan.inputs):
            d = shard_dim(mf["shape"], mp["shape"])
            out.append(g if d is None else g.narrow(d, self.lo, self.hi - self.lo).contiguous())
        return out

    def run(self, stream):
        self.plan.execute([t.data_ptr() for t in self.ins], [t.data_ptr() for t in self.outs], stream)


def gpu_arm(args):
    import torch
    import torch.distributed as dist

    from paper_2601_12220_b200 import feinsum as fe

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # NCCL over NVLink for the timing barrier / max-reduce / verification
    # gather; FE_DIST_BACKEND=gloo exercises the multi-rank path on one GPU.
    backend = os.environ.get("FE_DIST_BACKEND", "nccl")
    if world > 1:
        dist.init_process_group(backend, init_method="env://")
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    cdev = dev if backend == "nccl" else torch.device("cpu")
    stream = torch.cuda.current_stream()
    sh = stream.cuda_stream

    names = [c for c in args.configs.split(",") if c]
    loads, skipped = [], {}
    for i, n in enumerate(names):
        try:
            w = Workload(n, rank, world, torch, fe, seed=(i + 1) * 100 + (rank if args.scaling == "weak" else 0),
                         scaling=args.scaling)
        except fe.FeinsumError as ex:
            skipped[n] = str(ex)
            continue
        if w.transform == "generic/v1" and w.ref_flops > 1e11:
            skipped[n] = "no tuned kernel yet (generic path too slow at full size)"
            continue
        loads.append(w)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=dev)
    torch.cuda.synchronize()

    def one_step(events):
        for k, w in enumerate(loads):
            fe.flush_l2(flush)
            events[k][0].record(stream)
            w.run(sh)
            events[k][1].record(stream)

    ev = [[torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)] for _ in loads]
    for _ in range(args.warmup):
        one_step(ev)
    torch.cuda.synchronize()

    times = [[] for _ in loads]
    with ClockSampler(local) as clocks:
        clocks.wait_first()
        n0 = len(clocks.rows)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t_wall = time.perf_counter()
        for _ in range(args.steps):
            one_step(ev)
            torch.cuda.synchronize()
            for k in range(len(loads)):
                times[k].append(ev[k][0].elapsed_time(ev[k][1]) * 1e-3)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t_wall
        # keep only samples taken while the timed loop ran (plus the last one before it)
        clocks.rows = clocks.rows[max(0, n0 - 1):]
    if world > 1:
        dist.barrier()

    # per config: the median of the K timed steps (each its own CUDA-event
    # pair on the launch stream, L2 flushed before it). The mean is reported
    # beside it: a multi-launch config occasionally waits for its host thread
    # between launches while nvidia-smi samples the clocks (the sampler must
    # run during the timed region), and one such step moved C5's mean by 40%.
    def median(v):
        v = sorted(v)
        n = len(v)
        return v[n // 2] if n % 2 else 0.5 * (v[n // 2 - 1] + v[n // 2])
    mean_t = torch.tensor([median(t) for t in times], dtype=torch.float64, device=cdev)
    avg_t = torch.tensor([sum(t) / len(t) for t in times], dtype=torch.float64, device=cdev)
    if world > 1:
        dist.all_reduce(mean_t, op=dist.ReduceOp.MAX)
        dist.all_reduce(avg_t, op=dist.ReduceOp.MAX)
    mean_t = mean_t.cpu().tolist()
    avg_t = avg_t.cpu().tolist()

    peaks, peak_src = measured_peaks()
    fp64 = {}
    for which, label in ((0, "dfma"), (1, "dmma")):
        import ctypes
        v = ctypes.c_double()
        if fe.lib().fe_fp64_peak(which, ctypes.byref(v)) == 0:
            fp64[label] = v.value

    def pipe_peak(pipe):
        """(TFLOP/s, source) of the arithmetic pipe a kernel issues to. FP64
        kernels (DFMA or DMMA) are held to the faster of the two measured FP64
        rates: the two share one datapath (tools/fp64_mixed_probe.py), and
        DMMA reaches the full rate where DFMA tops out ~10% lower."""
        if pipe in ("dfma", "dmma"):
            best = max(fp64.values()) if fp64 else 0.0
            return best, "max(DFMA, DMMA) measured on this GPU by fe_fp64_peak"
        if pipe == "tcgen05_tf32x3":
            # dense TF32 = half the measured bf16 rate; 3xTF32 spends three MMAs per product
            return peaks["bf16_tflops"] / 2 / 3, "MEASURED_PEAKS.json bf16_tflops / 2 (TF32) / 3 (3xTF32 passes)"
        return 0.0, "none"

    per = {}
    rates = []
    for w, t, ta in zip(loads, mean_t, avg_t):
        agg_flops = w.global_flops  # the global (world x config) problem, one shard per rank
        gflops = agg_flops / t / 1e9
        rates.append(gflops)
        # per-config roofline: slower of HBM (footprint bytes) and FP64 (DMMA
        # peak for the DMMA kernels, DFMA peak for the DFMA kernels)
        fp_peak = pipe_peak(w.pipe)[0] * 1e12
        roof_t = max(w.bytes / (peaks["hbm_gbs"] * 1e9), w.flops / fp_peak if fp_peak else 0.0)
        per[w.name] = {"ms": t * 1e3, "ms_mean": ta * 1e3, "gflops": gflops, "gbs": w.full.info["bytes"] / t / 1e9,
                       "transform": w.transform, "source": w.source, "flops": w.flops, "bytes": w.bytes,
                       "roof_ms": roof_t * 1e3, "roof_frac": roof_t / t,
                       "pipe": w.pipe,
                       "bound": "hbm" if w.bytes / (peaks["hbm_gbs"] * 1e9) >= roof_t else w.pipe}
    value = math.exp(sum(math.log(r) for r in rates) / len(rates)) if rates else 0.0
    ms_step = sum(mean_t) * 1e3

    # dominant kernel roofline (largest share of the step)
    dom = max(range(len(loads)), key=lambda k: mean_t[k]) if loads else None
    roof = None
    if dom is not None:
        w, t = loads[dom], mean_t[dom]
        fp64_peak, fp_src = pipe_peak(w.pipe)
        hbm_time = w.bytes / (peaks["hbm_gbs"] * 1e9)
        fp_time = w.flops / (fp64_peak * 1e12) if fp64_peak else 0
        if hbm_time >= fp_time:
            roof = {"bound": "hbm", "achieved": w.bytes / t / 1e9, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                    "peak_source": peak_src + " (MEASURED_PEAKS.json hbm_gbs)"}
        else:
            # FP64 work: tcgen05 has no f64 kind, so the denominator is the FP64
            # pipe this kernel issues to (DMMA tensor cores or DFMA), measured
            # on this GPU; MEASURED_PEAKS.json only carries HBM and bf16
            roof = {"bound": "tensor" if w.pipe in ("dmma", "tcgen05_tf32x3") else "fp64",
                    "achieved": w.flops / t / 1e12, "peak": fp64_peak, "unit": "TFLOP/s", "peak_source": fp_src}
        roof["frac"] = roof["achieved"] / roof["peak"]
        roof["kernel"] = w.name + ":" + w.transform
        roof["traffic"] = None
        for rnd in ("r02", "r01"):  # dram bytes per launch of this config's kernel, newest committed ncu capture
            try:
                with open(os.path.join(ROOT, "profiles", rnd, "traffic.json")) as f:
                    tr = json.load(f)["per_config"].get(w.name.split("@")[0])
            except (OSError, ValueError, KeyError):
                continue
            if tr:
                roof["traffic"] = tr["dram_bytes"]
                roof["traffic_source"] = "profiles/%s/traffic.json (ncu --set full, %s)" % (rnd, tr["kernel"])
                break

    extras = None
    if world == 1 and not args.no_extras:
        extras = extras_pass(args, torch, fe, stream, flush, peaks, pipe_peak)

    verify = verify_shards(loads, torch, fe, rank, world, dist, cdev, args.scaling) if world > 1 else None

    e2e = None
    if not args.no_e2e and loads:
        e2e = e2e_pass(args, loads, torch, fe, world, dist if world > 1 else None, cdev)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline([w.name for w in loads], args.cpu_seconds)

    if rank == 0:
        line = {
            "metric": "geomean GFLOP/s (and fraction of roofline) over TCCG+FEM batched einsums, 1-8 B200",
            "value": value, "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_step, "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
            "dtype": "f64 (C4-f32: f32)", "data": "synthetic dyadic values m/2^19-1 generated on device",
            "config": {"workload": "TCCG+FEM suite " + ",".join(w.name for w in loads),
                       "suite": {n: CONFIG_DOC[n] for n in names}, "per_config": per, "skipped": skipped,
                       "l2": "flushed before every config launch: 256 MiB write, then the same 256 MiB read back (L2 cold for the inputs and clean)",
                       "parallelism": f"dp{world} (element/batch-axis shards, no collective; {args.scaling} scaling)",
                       "statistic": "per config: median of the K timed steps (CUDA events; ms_mean beside it); "
                                    "ms_per_step = sum of the per-config medians",
                       "wall_s_timed_region": wall},
            "roofline": roof, "fp64_peak_tflops": fp64, "clocks": clocks.summary(),
            "gpu_launches": args.steps * sum(w.launches for w in loads),
            "e2e": e2e, "cpu_baseline": cpu,
        }
        if extras is not None:
            line["extras"] = extras
        if verify is not None:
            line["verify"] = verify
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


def verify_shards(loads, torch, fe, rank, world, dist, cdev, scaling):
    """Verification (outside the timed region): every rank hashes the bit
    patterns of its shard outputs (bithash) and all-gathers the hashes; rank 0
    recomputes every shard on ONE GPU WITHOUT sharding and compares bitwise:
      strong scaling: rank 0 runs the unsharded global plan on the same global
        inputs once and hashes each rank's slice of its outputs;
      weak scaling (the global problem is world x the one-GPU config and does
        not fit one GPU): rank 0 rebuilds rank r's inputs from its seeds and
        runs the standalone one-GPU config plan (its own plan and fact, not the
        shard plan) on them.
    Sharding never changes per-element arithmetic, so any difference fails."""
    report = {}
    for w in loads:
        mine = torch.tensor(sum((bithash(torch, o) for o in w.outs), []), dtype=torch.int64, device=cdev)
        got = [torch.zeros_like(mine) for _ in range(world)]
        dist.all_gather(got, mine)
        ok = True
        if rank == 0:
            dev = torch.device("cuda", torch.cuda.current_device())
            if scaling == "strong":
                full_outs = w.full(*w.global_inputs(torch, fe, dev))
                for r in range(world):
                    sh, lo, hi, _ = w.full.shard(r, world)
                    want = []
                    for o, mf, mp in zip(full_outs, w.full.outputs, sh.outputs):
                        d = shard_dim(mf["shape"], mp["shape"])
                        want += bithash(torch, o if d is None else o.narrow(d, lo, hi - lo))
                    ok = ok and want == got[r].cpu().tolist()
                del full_outs
            else:
                kind, payload = spec(w.name)
                solo = fe.Plan(einsum=payload) if kind == "einsum" else fe.Plan(kernel=payload)
                seed0 = w.seed - rank
                for r in range(world):
                    ins = []
                    for j, m in enumerate(solo.inputs):
                        t = torch.empty(m["shape"], dtype=fe._torch_dtype(m["storage"]), device=dev)
                        fe.fill_dyadic(t, (seed0 + r) * 1000 + j)
                        ins.append(t)
                    want = sum((bithash(torch, o) for o in solo(*ins)), [])
                    ok = ok and want == got[r].cpu().tolist()
                    del ins
            torch.cuda.synchronize()
            report[w.name] = bool(ok)
    return {"ok": all(report.values()), "per_config": report,
            "method": ("bitwise (exact bit-pattern hashes) against the unsharded one-GPU result: "
                       + ("the global plan on the global inputs" if scaling == "strong"
                          else "the standalone one-GPU config plan on each rank's inputs"))}


EXTRA_DOC = {
    "C1-graph": "C1 executed 20 times back to back inside one CUDA graph, per-execute time (launch cost "
                "amortised; the 10 MB working set is L2-resident after the first execute, so no HBM roofline)",
    "C1-L": "the C1 skeleton at E=2e6 (SURVEY.md 8d: C1 is below launch latency; its large case is HBM-bound)",
    "C3-aebf-fdec": "TCCG sibling abcd-aebf-fdec at extent 72, (a1*A+b1)(a2*B+b2) operands",
    "C3-eafb-fdec": "TCCG sibling abcd-eafb-fdec at extent 72, (a1*A+b1)(a2*B+b2) operands",
    "C3-eafd-fbec": "TCCG sibling abcd-eafd-fbec at extent 72, (a1*A+b1)(a2*B+b2) operands",
    "C4-f32-tf32": "C4-f32 on the tcgen05 3xTF32 kernel (precision class b200-tf32: ~1e-5 against double, above "
                   "the flat fp32 bar on some data, so not the suite's C4-f32)",
    "C5-nonlinear": "C5 skeleton with s = u*u - sin(k)/(2+exp(u)): the programs run in the prologue of a "
                    "generated fem_grad instance (no operand tables in HBM); FP64-heavy (sin/exp/div per point)",
    "C5-nonlinear-tables": "the same step with codegen off: device-VM tables in HBM + the prebuilt kernel",
    "C5-post": "C5 (u + 0.5k) with a fused post epilogue per field, y <- u + 0.25 y (pre and post elementwise "
               "fused: BASELINE config 5)",
}


def extra_specs():
    from paper_2601_12220_b200 import configs as C
    return {
        "C1-L": {"kind": "einsum", "payload": C.fem_grad(E=2_000_000)},
        "C3-aebf-fdec": {"kind": "kernel", "payload": C.tccg_kernel("abcd-aebf-fdec")},
        "C3-eafb-fdec": {"kind": "kernel", "payload": C.tccg_kernel("abcd-eafb-fdec")},
        "C3-eafd-fbec": {"kind": "kernel", "payload": C.tccg_kernel("abcd-eafd-fbec")},
        "C4-f32-tf32": {"kind": "einsum", "payload": C.tensor_train(n=4096, dtype="float32"),
                        "options": {"device": "b200-tf32"}},
        "C5-nonlinear": {"kind": "kernel", "payload": C.wave_kernel_nonlinear()},
        "C5-nonlinear-tables": {"kind": "kernel", "payload": C.wave_kernel_nonlinear(), "options": {"codegen": False}},
        "C5-post": {"kind": "kernel", "payload": C.wave_kernel() + "".join(
            f"epi y{q}[r,e,i] := u{q}[e,i] + 0.25*y{q}[r,e,i]\n" for q in (1, 2, 3))},
    }


def extras_pass(args, torch, fe, stream, flush, peaks, pipe_peak):
    """Lines reported beside the suite and NOT in its geomean (one GPU, same
    methodology: L2 flushed before every timed launch, CUDA events on the
    launching stream): the launch floor (an empty kernel), C1 inside a CUDA
    graph, C1's large case, the TCCG siblings of C3 and the 3xTF32 C4-f32."""
    sh = stream.cuda_stream
    steps = max(3, args.steps)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def timed(fn, warm=2):
        for _ in range(warm):
            fn()
        tot = 0.0
        for _ in range(steps):
            fe.flush_l2(flush)
            e0.record(stream)
            fn()
            e1.record(stream)
            torch.cuda.synchronize()
            tot += e0.elapsed_time(e1) * 1e-3
        return tot / steps

    out = {"doc": EXTRA_DOC}
    out["launch_floor_us"] = timed(lambda: fe.lib().fe_launch_probe(sh)) * 1e6

    def roofline(w, t):
        fp_peak = pipe_peak(w.pipe)[0] * 1e12
        hbm_t = w.bytes / (peaks["hbm_gbs"] * 1e9)
        roof_t = max(hbm_t, w.flops / fp_peak if fp_peak else 0.0)
        return {"ms": t * 1e3, "gflops": w.flops / t / 1e9, "gbs": w.bytes / t / 1e9, "transform": w.transform,
                "source": w.source, "pipe": w.pipe, "roof_ms": roof_t * 1e3, "roof_frac": roof_t / t,
                "bound": "hbm" if hbm_t >= roof_t else w.pipe}

    # C1 in a CUDA graph: 20 executes per replay
    try:
        w = Workload("C1", 0, 1, torch, fe, seed=11)
        reps = 20
        g = torch.cuda.CUDAGraph()
        cs = torch.cuda.Stream()
        cs.wait_stream(stream)
        with torch.cuda.stream(cs):
            w.run(cs.cuda_stream)  # warm (lazy module load, attributes) outside the capture
            torch.cuda.synchronize()
            with torch.cuda.graph(g, stream=cs):
                for _ in range(reps):
                    w.run(torch.cuda.current_stream().cuda_stream)
        stream.wait_stream(cs)
        t = timed(g.replay) / reps
        r = roofline(w, t)
        r.update({"executes_per_graph": reps, "roof_ms": None, "roof_frac": None,
                  "note": "L2-resident after the first execute: no HBM roofline"})
        out["C1-graph"] = r
        del g, w
    except Exception as ex:  # noqa: BLE001 — reported, never fatal
        out["C1-graph"] = {"error": str(ex)}
    for name, sp in extra_specs().items():
        try:
            w = Workload(name, 0, 1, torch, fe, seed=31, extra=sp)
            out[name] = roofline(w, timed(lambda: w.run(sh)))
            del w
        except Exception as ex:  # noqa: BLE001
            out[name] = {"error": str(ex)}
        torch.cuda.empty_cache()
    return out


def e2e_pass(args, loads, torch, fe, world, dist, cdev=None):
    """Same metric through the C-ABI with pinned HOST buffers: H2D of the
    inputs, kernels, D2H of the outputs, all inside the timed region."""
    stream = torch.cuda.current_stream()
    rates, h2d, d2h, ms = [], 0, 0, 0.0
    steps = max(1, min(args.steps, 5))
    bw = pcie_bandwidth(torch, stream)
    per = {}
    for w in loads:
        hin = [torch.empty(t.shape, dtype=t.dtype, pin_memory=True) for t in w.ins]
        for h, t in zip(hin, w.ins):
            h.copy_(t)
        hout = [torch.empty(t.shape, dtype=t.dtype, pin_memory=True) for t in w.outs]
        ptr_in = [h.data_ptr() for h in hin]
        ptr_out = [h.data_ptr() for h in hout]
        w.plan.execute_host(ptr_in, ptr_out, stream.cuda_stream)
        torch.cuda.synchronize()
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ts = []
        for _ in range(steps):
            t0.record(stream)
            w.plan.execute_host(ptr_in, ptr_out, stream.cuda_stream)
            t1.record(stream)
            torch.cuda.synchronize()
            ts.append(t0.elapsed_time(t1) * 1e-3)
        # median step: every step carries its copies; the median keeps one
        # host hiccup (page-cache / NUMA noise on the pinned buffers) out
        t = sorted(ts)[len(ts) // 2]
        if dist is not None:
            tt = torch.tensor([t], dtype=torch.float64, device=cdev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            t = tt.item()
        rates.append(w.global_flops / t / 1e9)
        bi = sum(x.numel() * x.element_size() for x in hin)
        bo = sum(x.numel() * x.element_size() for x in hout)
        h2d += bi
        d2h += bo
        ms += t * 1e3
        # PCIe floor: both directions overlapped (the host pipeline runs H2D,
        # kernels and D2H of different chunks on three streams)
        floor = max(bi / bw["h2d_gbs"], bo / bw["d2h_gbs"]) / 1e9
        per[w.name] = {"ms": t * 1e3, "gflops": w.global_flops / t / 1e9, "h2d_bytes": bi, "d2h_bytes": bo,
                       "pcie_floor_ms": floor * 1e3, "pcie_frac": floor / t}
        del hin, hout
    return {"value": math.exp(sum(math.log(r) for r in rates) / len(rates)), "unit": "GFLOP/s",
            "h2d_bytes_per_step": h2d * world, "d2h_bytes_per_step": d2h * world, "ms_per_step": ms,
            "steps": steps, "statistic": "median step per config",
            "path": "fe_plan_execute_host (C-ABI), pinned host buffers",
            "pcie": bw, "per_config": per}


def pcie_bandwidth(torch, stream, nbytes=1 << 30):
    """Pinned host <-> device copy bandwidth (GB/s), 1 GiB each way, events."""
    h = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    out = {}
    for key, fn in (("h2d_gbs", lambda: d.copy_(h, non_blocking=True)), ("d2h_gbs", lambda: h.copy_(d, non_blocking=True))):
        fn()
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(3):
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
        out[key] = 3 * nbytes / (e0.elapsed_time(e1) * 1e-3) / 1e9
    del h, d
    return out


# ------------------------------------------------------ CPU reference ----

# bounded samples: the work of every config is linear in its sharded axis
CPU_SAMPLES = {
    "C1": ("C1 at full size (E=1e4)", 1.0),
    "C2": ("C2 with E=1 element, b=1 field (x 2e6 elements x 8 fields)", None),
    "C3": ("C3 with output indices a,b fixed (1/72^2 of the work)", None),
    "C4-f64": ("C4 with n=1 sample (x 4096)", 1 / 4096),
    "C4-f32": ("C4-f32 with n=1 sample (x 4096)", 1 / 4096),
    "C5": ("C5 with E=2e3 elements (x 1000)", 1e-3),
}


def cpu_sample(name):
    """(einsum or kernel, kind) of the bounded CPU sample and its alg FLOPs."""
    from paper_2601_12220_b200 import configs as C
    if name == "C2":
        return "einsum", C.hex_poisson(E=1, b=1)
    if name == "C3":
        # a and b fixed: a one-element slice of both output axes
        return "tccg_slice", None
    return spec(name, CPU_SAMPLES[name][1])


# Algorithmic FLOPs of each bounded sample (optimal pairwise path per row x
# rows, operand FLOPs included), committed so the reference arm never loads
# the product library; tests/test_bench_tables.py checks them against the
# product's cost model (fe.cost / dry-run plans).
SAMPLE_FLOPS = {"C1": 23_400_000, "C2": 24_750, "C3": 53_747_712, "C4-f64": 1_048_576, "C4-f32": 1_048_576,
                "C5": 4_800_000}


def _cpu_worker(args):
    """One host process: evaluate the bounded sample `reps` times with the
    unmodified reference (oracle/_ref: feinsum::evaluate / evaluate_functional)
    and return the seconds spent evaluating (input generation excluded)."""
    name, reps = args
    sys.path.insert(0, ROOT)
    from oracle import refpy as R
    from paper_2601_12220_b200 import configs as C
    kind, payload = cpu_sample(name)
    if kind == "tccg_slice":
        e = C.tccg(ext=72)
        e["args"][0][0]["shape"] = [1, 72, 1, 72]   # A[a,e,b,f] with a=b=1
        e = {"i_out": ["a", "b", "c", "d"], "i_in": e["i_in"], "args": e["args"]}
        lens = {"a": 1, "b": 1, "c": 72, "d": 72, "e": 72, "f": 72}
        e["args"][0][1]["shape"] = [lens[s] for s in e["i_in"][1]]
        binds = R.random_bindings(e, 1)
        t0 = time.perf_counter()
        for _ in range(reps):
            R.evaluate(e, binds)
        return time.perf_counter() - t0
    if kind == "einsum":
        binds = R.random_bindings(payload, 1)
        t0 = time.perf_counter()
        for _ in range(reps):
            R.evaluate(payload, binds)
        return time.perf_counter() - t0
    import re
    arrays = []
    for line in payload.splitlines():
        m = re.match(r"array: (\w+) (\w+) (\S+)", line)
        if m:
            shape = [] if m.group(3) == "scalar" else [int(x) for x in m.group(3).split("x")]
            arrays.append({"name": m.group(1), "shape": shape, "dtype": m.group(2)})
    fake = {"i_out": [], "i_in": [[] for _ in arrays], "args": [arrays]}
    binds = R.random_bindings(fake, 1)
    raised = R.raise_kernel(payload)
    shape = [dict(zip(sum(raised["skeleton"]["i_in"], []),
                      sum([m["shape"] for m in raised["skeleton"]["args"][0]], [])))[s]
             for s in raised["skeleton"]["i_out"]]
    t0 = time.perf_counter()
    for _ in range(reps):
        R.eval_kernel(payload, arrays, binds, len(raised["skeleton"]["args"]), shape)
    return time.perf_counter() - t0


def cpu_baseline(names, seconds, cores=None):
    """Reference evaluator (oracle/_ref, the unmodified feinsum::evaluate /
    evaluate_functional) on the host cores. The parent process calibrates
    each sample with one single-core run (so the reference library is loaded
    here too), then `cores` spawned processes evaluate the same bounded
    sample `reps` times each (the shardable axes make per-core work
    independent); throughput = cores x reps x sample FLOPs / the slowest
    process's evaluation time. The reference has no threads, so the
    all-core figure is our harness's."""
    import multiprocessing as mp
    cores = cores or os.cpu_count() or 1
    out = {}
    rates = []
    ctx = mp.get_context("spawn")
    todo = [n for n in names if n in CPU_SAMPLES]
    calib = {n: _cpu_worker((n, 1)) for n in todo}
    with ctx.Pool(cores) as pool:
        for n in todo:
            t1 = calib[n]
            reps = max(1, int(seconds / max(t1, 1e-6)))
            ts = pool.map(_cpu_worker, [(n, reps)] * cores)
            rate = cores * reps * SAMPLE_FLOPS[n] / max(ts) / 1e9
            rates.append(rate)
            out[n] = {"gflops": rate, "sample": CPU_SAMPLES[n][0], "reps_per_core": reps, "single_core_s": t1,
                      "sample_flops": SAMPLE_FLOPS[n]}
    value = math.exp(sum(math.log(r) for r in rates) / len(rates)) if rates else None
    return {"value": value, "unit": "GFLOP/s", "cores": cores, "kind": "reference",
            "sample": "per config: " + "; ".join(f"{k}: {v['sample']}" for k, v in out.items()),
            "per_config": out,
            "same_config_note": ("bounded samples of each config, timed and scaled by their algorithmic FLOPs: the "
                                 "reference's cost is linear in the sharded axis (BASELINE.md §3); full size would "
                                 "take ~100 core-days for C2 alone")}


def reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    names = [c for c in args.configs.split(",") if c in CPU_SAMPLES]
    vals = []
    last = None
    for i in range(args.warmup + args.steps):
        r = cpu_baseline(names, args.cpu_seconds / 2)
        if i >= args.warmup:
            vals.append(r["value"])
            last = r
    value = sum(vals) / len(vals)
    line = {"metric": "geomean GFLOP/s (and fraction of roofline) over TCCG+FEM batched einsums, 1-8 B200",
            "value": value, "unit": "GFLOP/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "complex128 (reference)",
            "data": "synthetic dyadic (random_bindings)", "impl": "reference",
            "config": {"workload": "TCCG+FEM suite " + ",".join(names), "per_config": last["per_config"]},
            "cpu_baseline": {k: last[k] for k in ("kind", "cores", "sample")} | {"value": value, "unit": "GFLOP/s"},
            "e2e": {"value": value, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


if __name__ == "__main__":
    a = parse_args()
    if a.impl == "reference":
        reference_arm(a)
    else:
        gpu_arm(a)
