"""Benchmark: gradient evaluations/s of the BASELINE.json configs on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload C5/heat_3d]
    python bench.py --impl reference ...        (CPU reference arm)

One step = one gradient evaluation (forward + backward) of the
workload on synthetic inputs (reference sample_inputs rule). Default workload:
C5 heat_3d N=512^3, TSTEPS=100 fp64 — the config the metric is quoted on at
1/2/4/8 GPUs and the largest single-GPU config (configs[1], the literal 25 %
budget, is Infeasible in the reference itself). Under torchrun
(N>1) the 512^3 domain is slab-decomposed over the ranks (strong scaling) with
a halo exchange per timestep.

Timing: W untimed warm-up steps, then K steps between barrier+synchronize
fences, CUDA events on the launching stream, max over ranks. Inputs are 1 GiB
per array (> 126 MB L2), so no extra L2 flush is needed between steps.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

DEFAULT_WORKLOAD = "C5/heat_3d"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=("b200", "reference"))
    ap.add_argument("--workload", default=DEFAULT_WORKLOAD)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=8)
    ap.add_argument("--force-slab", action="store_true",
                    help="use the slab-decomposed engine even on one rank (exercises the multi-GPU path)")
    return ap.parse_args()


def measured_peaks():
    path = os.path.join(REPO, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.idx = device_index
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        time.sleep(0.25)
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        rows = []
        try:
            with open(self.path) as f:
                for line in f:
                    parts = [p.strip() for p in line.split(",")]
                    if len(parts) >= 9:
                        rows.append(parts)
        except OSError:
            pass
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        smax = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in rows for n, v in zip(names, r[5:9]) if v.lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": reasons, "samples": len(rows)}


def kernels_per_op(op) -> int:
    from paper_2509_02197_b200.lowering import CopyOp, GatherOp, MatmulOp, MatvecPairOp, ReduceOp

    if isinstance(op, CopyOp):
        return 0  # device-to-device memcpy or elided alias, not a kernel
    if isinstance(getattr(op, "edges", None), list):
        return len(op.edges)  # a slab's edge ranges (decomp.EdgeOp)
    if op.family in ("halo", "halo_wait", "allreduce"):
        return 0  # NCCL communication, not one of the engine's kernels
    if isinstance(op, ReduceOp):
        return 2
    if isinstance(op, GatherOp):
        return 2 if op.nsplit > 1 else 1
    if isinstance(op, MatvecPairOp):
        return 2  # streaming pass + column-partial finish
    if isinstance(op, MatmulOp):
        return 2 if op.workspace_bytes() > 0 else 1
    return 1


def roofline(exe, inputs, peak, peak_kind):
    """Per-launch CUDA-event times of one eager step; the dominant kernel
    family's algorithmic bytes / measured duration against the HBM peak."""
    rows = exe.timed_eager(inputs)
    fam_t, fam_b, fam_n = {}, {}, {}
    for fam, op, ms in rows:
        fam_t[fam] = fam_t.get(fam, 0.0) + ms
        fam_b[fam] = fam_b.get(fam, 0) + op.algorithmic_bytes()
        fam_n[fam] = fam_n.get(fam, 0) + 1
    total = sum(fam_t.values())
    dom = max(fam_t, key=fam_t.get)
    avg_ms = fam_t[dom] / fam_n[dom]
    avg_bytes = fam_b[dom] / fam_n[dom]
    achieved = avg_bytes / (avg_ms * 1e-3) / 1e9
    shares = {k: round(v / total, 4) for k, v in sorted(fam_t.items(), key=lambda kv: -kv[1])}
    traffic, dram_frac = None, None
    ncu = ncu_traffic().get(dom)
    if ncu is not None:
        # DRAM bytes per launch from the committed ncu --set full capture
        traffic = ncu["dram_bytes_per_launch"]
        dram_frac = round(traffic / (avg_ms * 1e-3) / 1e9 / peak, 4)
    return {"bound": "hbm", "kernel": dom, "achieved": round(achieved, 1), "peak": peak, "peak_kind": peak_kind,
            "unit": "GB/s", "frac": round(achieved / peak, 4), "traffic": traffic, "dram_frac": dram_frac,
            "bytes_per_launch": int(avg_bytes), "avg_launch_ms": round(avg_ms, 5), "launches_per_step": fam_n[dom],
            "step_share": shares,
            "note": "bytes_per_launch = SURVEY 8(d) algorithmic bytes of the sweeps one launch performs "
                    "(a fused star_pair launch performs two sweeps); traffic = measured DRAM bytes per launch"}


def ncu_traffic():
    path = os.path.join(REPO, "profiles", "ncu_traffic.json")
    if os.path.exists(path):
        with open(path) as f:
            return json.load(f)
    return {}


def cpu_baseline_stencil(name, params):
    """C restatement of the reference program (oracle/stencil_ref.c) on all
    host cores, on a bounded sample: the full spatial size with TSTEPS=2 and
    TSTEPS=hi (one and hi-1 timesteps, hi <= 8), extrapolated linearly to the
    config's TSTEPS from the per-timestep slope between the two runs."""
    from oracle import stencil_ref as S
    from paper_2509_02197_b200 import workloads as W

    prog, _ = W.load(name)
    T = params["TSTEPS"]
    times = {}
    hi = max(3, min(T, 8))
    for ts in (2, hi):
        p = dict(params, TSTEPS=ts)
        inputs = W.make_inputs(name, prog, p, 0)
        t0 = time.perf_counter()
        S.gradient(name, p, inputs)
        times[ts] = time.perf_counter() - t0
    per_step = max((times[hi] - times[2]) / (hi - 2), 1e-9)
    full = times[2] + (T - 2) * per_step
    cores = S.max_threads()
    return {"value": 1.0 / full, "unit": "evals/s", "cores": cores, "kind": "port",
            "sample": f"oracle/stencil_ref.c ({cores} threads) gradient of {name} at N={params['N']} with TSTEPS=2 "
                      f"and {hi} ({times[2]:.2f}s, {times[hi]:.2f}s), extrapolated to TSTEPS={T}: {full:.1f}s/eval"}


def reference_interpreter_sample(name, params):
    """The UNMODIFIED reference interpreter (gradflow ``gradient()``, installed
    offline into baseline/_ref), timed on this host at a reduced size and
    extrapolated (BASELINE.md CPU plan step 1): per-timestep slope between
    two trip counts at edge length n, scaled by the interior volume
    ((N - 2) / (n - 2))^d to the config, times the config's timesteps. It is
    one Python thread (the interpreter visits map points one at a time)."""
    ref = os.path.join(REPO, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "gradflow")):
        return {"unavailable": "baseline/_ref has no gradflow install"}
    if ref not in sys.path:
        sys.path.insert(0, ref)
    from gradflow.autodiff import gradient as ref_gradient  # the reference itself
    from gradflow.frontend import load_program as ref_load

    from paper_2509_02197_b200 import workloads as W

    prog = ref_load(os.path.join(W.PROG_DIR, name + ".fwd.json"))
    d = 3 if name == "heat_3d" else 2
    n, (t_lo, t_hi) = (12, (3, 5)) if d == 3 else (40, (3, 7))
    times = {}
    for ts in (t_lo, t_hi):
        p = {"N": n, "TSTEPS": ts}
        inputs = W.make_inputs(name, W.load(name)[0], p, 0)
        t0 = time.perf_counter()
        ref_gradient(prog, inputs, p)
        times[ts] = time.perf_counter() - t0
    per_step = max((times[t_hi] - times[t_lo]) / (t_hi - t_lo), 1e-9)
    scale = ((params["N"] - 2) / (n - 2)) ** d
    full = per_step * scale * (params["TSTEPS"] - 1)
    return {"value": 1.0 / full, "unit": "evals/s", "cores": 1, "kind": "reference", "extrapolated": True,
            "sample": f"gradflow.gradient (reference interpreter, baseline/_ref) of {name} at N={n}, "
                      f"TSTEPS={t_lo} and {t_hi} ({times[t_lo]:.2f}s, {times[t_hi]:.2f}s): {per_step:.3f}s per "
                      f"timestep, x{scale:.0f} volume to N={params['N']}, x{params['TSTEPS'] - 1} timesteps = "
                      f"{full:.0f}s/eval ({full / 86400:.1f} days)"}


def cpu_baseline_generic(name, params, budget_s=20.0):
    from oracle import interp as O
    from paper_2509_02197_b200 import workloads as W

    prog, b = W.load(name)
    inputs = W.make_inputs(name, prog, params, 0)
    t0 = time.perf_counter()
    n = 0
    while True:
        O.gradient(prog, b.backward, b.forwarding, b.required, inputs, params)
        n += 1
        if time.perf_counter() - t0 > budget_s or n >= 3:
            break
    dt = (time.perf_counter() - t0) / n
    return {"value": 1.0 / dt, "unit": "evals/s", "cores": 1, "kind": "port",
            "sample": f"oracle/interp.py (numpy) full gradient of {name} {params}, {n} run(s), {dt:.2f}s/eval"}


def cpu_baseline(name, params):
    if name in ("heat_3d", "jacobi_2d"):
        base = cpu_baseline_stencil(name, params)
        try:
            base["reference_interpreter"] = reference_interpreter_sample(name, params)
        except Exception as exc:  # reported, never fatal for the bench
            base["reference_interpreter"] = {"unavailable": f"{type(exc).__name__}: {exc}"}
        return base
    return cpu_baseline_generic(name, params)


def run_reference(args):
    """--impl reference: the CPU implementation of the path (the oracle port;
    the reference itself is a Python interpreter that needs days for C5)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_2509_02197_b200 import workloads as W

    name, params = W.CONFIGS[args.workload]
    prog, _ = W.load(name)
    f32 = any(d.element_kind == "real32" for d in prog.descriptors.values())
    # a CPU step has no warm-up state to build (no caches, no graphs); the
    # timed steps are bounded samples of the workload (cpu_baseline)
    samples = []
    base = None
    for _ in range(max(1, args.steps)):
        base = cpu_baseline(name, params)
        samples.append(base["value"])
    value = float(np.median(samples))
    line = {"impl": "reference", "metric": "gradient evals/sec (fwd+bwd)", "value": value, "unit": "evals/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32" if f32 else "f64",
            "data": "synthetic", "config": {"workload": args.workload, **params},
            "cpu_baseline": {**base, "value": value},
            "e2e": {"value": value, "unit": "evals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_b200(args):
    import torch
    import torch.distributed as dist

    from paper_2509_02197_b200 import Engine, workloads as W

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    slab = world > 1 or args.force_slab
    if slab:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29511")
        dist.init_process_group("nccl", device_id=dev, rank=rank, world_size=world)
    name, params = W.CONFIGS[args.workload]
    if slab:
        from paper_2509_02197_b200.decomp import SlabEngine

        eng = SlabEngine.from_workload(name, params, rank, world, dev)
        dev_inputs = eng.local_inputs(seed=0)
        host_inputs = {k: v.cpu().pin_memory() for k, v in dev_inputs.items()}
    else:
        prog, bundle = W.load(name)
        eng = Engine(prog, bundle, params)
        host_np = W.make_inputs(name, prog, params, 0)
        dev_inputs = {k: torch.from_numpy(v).to(dev) for k, v in host_np.items()}
        host_inputs = {k: torch.from_numpy(v).pin_memory() for k, v in host_np.items()}

    def barrier():
        if slab:
            dist.barrier()

    for _ in range(max(args.warmup, 3)):
        eng.step(dev_inputs)
    torch.cuda.synchronize(dev)
    stream = torch.cuda.current_stream(dev)
    with ClockSampler(local) as clocks:
        barrier()
        torch.cuda.synchronize(dev)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            eng.step(dev_inputs)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        barrier()
    ms = e0.elapsed_time(e1) / args.steps
    if slab:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    eng.check()
    value = 1000.0 / ms  # gradient evaluations per second, whole job

    e2e = None
    if not args.no_e2e and host_inputs is not None:
        # warm the host path the way the timed loop uses it: the previous
        # result stays referenced while the next call runs, so the pinned
        # result staging holds two generations (caching host allocator)
        res = None
        for res in eng.gradients([host_inputs] * max(4, args.warmup)):
            pass
        torch.cuda.synchronize(dev)
        barrier()
        # pipelined calls through the public API: step k+1's H2D and step
        # k-1's D2H overlap step k's launches; the timed region includes the
        # pipeline's fill (first H2D) and drain (last D2H)
        t0 = time.perf_counter()
        for res in eng.gradients([host_inputs] * args.e2e_steps):
            pass
        dt = (time.perf_counter() - t0) / args.e2e_steps
        h2d = sum(v.numel() * v.element_size() for v in host_inputs.values())
        d2h = int(np.asarray(res.value).nbytes + sum(np.asarray(g).nbytes for g in res.grads.values()))
        if slab:
            sizes = torch.tensor([h2d, d2h], device=dev, dtype=torch.int64)
            dist.all_reduce(sizes)
            h2d, d2h = int(sizes[0]), int(sizes[1])
        e2e = {"value": 1.0 / dt, "unit": "evals/s", "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": d2h,
               "api": ("SlabEngine.gradients(pinned local slabs) -> numpy owned-plane grads (all ranks), pipelined"
                       if slab else "Engine.gradients(host pinned inputs) -> numpy grads, pipelined H2D/compute/D2H"),
               "steps": args.e2e_steps}
    peak, peak_kind = measured_peaks()
    # the per-launch timing pass runs the launch list, halo exchanges and the
    # all-reduce included, so every rank takes part; rank 0 reports it
    roof = roofline(eng.exe, dev_inputs, peak, peak_kind) if (rank == 0 or slab) else None
    launches = args.steps * sum(kernels_per_op(op) for op in eng.exe.ops)
    base = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and not slab:
        base = cpu_baseline(name, params)
    if rank != 0:
        if slab:
            dist.destroy_process_group()
        return
    line = {
        "metric": "gradient evals/sec (fwd+bwd)",
        "value": round(value, 4),
        "unit": "evals/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": max(args.warmup, 3),
        "ms_per_step": round(ms, 4),
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64" if name not in ("softmax", "mlp", "conv2d_bias") else "f32",
        "data": "synthetic (reference sample_inputs rule: uniform(0.4,1.6), seed 0)",
        "config": {"workload": args.workload, **params,
                   "l2": "inputs 1 GiB/array > 126 MB L2; no extra flush",
                   "parallelism": f"slab{world}" if slab else "single"},
        "roofline": roof,
        "cpu_baseline": base,
        "e2e": e2e,
        "gpu_launches": launches,
        "clocks": clocks.summary(),
        "engine": {"ops_per_step": len(eng.exe.ops), "device_bytes": eng.exe.device_bytes,
                   "graph": eng.exe.graph is not None},
    }
    print(json.dumps(line), flush=True)
    if slab:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
