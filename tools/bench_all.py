"""Per-config benchmark table (1 GPU): every BASELINE.json config through the
engine, with the dominant kernel's roofline and a bounded CPU-oracle sample.

    python tools/bench_all.py [--steps 10] [--only C3/gemm,...] > profiles/rNN_configs.jsonl

One JSON line per config (same timing rules as bench.py: warm-up, CUDA
events on the launching stream, inputs resident in HBM).
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2509_02197_b200 import Engine, workloads as W  # noqa: E402

# bounded CPU samples: (sample params, scale = full work / sample work)
CPU_SAMPLES = {
    "C3/gemm": ({"NI": 1000, "NJ": 1000, "NK": 1000}, 64.0),
    "C4/softmax": ({"R": 64 * 16 * 8, "SM": 128}, 16.0),
    "C4/mlp": (None, 1.0),
    "C4/conv2d_bias": ({"NB": 2, "H": 64, "W": 64, "CI": 16, "CO": 32, "K": 3}, 32.0),
}


def fp64_tensor_peak():
    """cuBLAS DGEMM 8192^3 measured here (no fp64 figure in MEASURED_PEAKS)."""
    a = torch.randn(8192, 8192, dtype=torch.float64, device="cuda")
    b = torch.randn(8192, 8192, dtype=torch.float64, device="cuda")
    for _ in range(2):
        a @ b
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(5):
        a @ b
    e.record()
    torch.cuda.synchronize()
    return 2 * 8192**3 * 5 / (s.elapsed_time(e) * 1e-3) / 1e12


FP32_FFMA_NOMINAL = 148 * 128 * 2 * 1.965e9 / 1e12  # TFLOP/s, no measured fp32 SIMT figure


def tf32_peak():
    """Dense TF32 tensor peak: half the measured bf16 figure (MEASURED_PEAKS),
    else half the 2.25 PFLOP/s nominal bf16."""
    path = os.path.join(REPO, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            return float(json.load(f).get("bf16_tflops", 2250.0)) / 2.0
    return 1125.0


def family(op):
    """matmul launches with a unit dimension are HBM-bound matrix-vector /
    rank-1 passes; the rest are contractions."""
    if op.family == "matmul" and min(op.M, op.N, op.K) == 1:
        return "matvec"
    return op.family


def roofline(exe, inputs, peak_hbm, fp64_peak):
    rows = [(family(op), op, ms) for _, op, ms in exe.timed_eager(inputs)]
    fam_t, fam_b, fam_n, fam_f = {}, {}, {}, {}
    for fam, op, ms in rows:
        fam_t[fam] = fam_t.get(fam, 0.0) + ms
        fam_b[fam] = fam_b.get(fam, 0) + op.algorithmic_bytes()
        fam_n[fam] = fam_n.get(fam, 0) + 1
        if hasattr(op, "flops"):
            fam_f[fam] = fam_f.get(fam, 0) + op.flops()
    total = sum(fam_t.values())
    dom = max(fam_t, key=fam_t.get)
    shares = {k: round(v / total, 4) for k, v in sorted(fam_t.items(), key=lambda kv: -kv[1])}
    if dom in ("matmul", "contract") and fam_f.get(dom):
        ach = fam_f[dom] / (fam_t[dom] * 1e-3) / 1e12
        f64 = any(op.dst.dtype == 1 if hasattr(op, "dst") else op.out.dtype == 1 for f, op, _ in rows if f == dom)
        if f64 and dom == "matmul":
            return {"bound": "tensor(fp64 DMMA)", "kernel": dom, "achieved": round(ach, 2), "unit": "TFLOP/s",
                    "peak": round(fp64_peak, 2), "peak_kind": "cuBLAS DGEMM 8192^3 measured in this run",
                    "frac": round(ach / fp64_peak, 4), "step_share": shares}
        if dom == "matmul":
            # fp32 matmuls run 3xTF32 on tcgen05: each launch is bound by the
            # larger of its HBM time (A + B + C bytes) and its tensor time
            # (3 TF32 products); frac = roofline time / measured time
            tf = tf32_peak()
            t_roof = 0.0
            for fam, op, ms in rows:
                if fam != dom:
                    continue
                t_roof += max(op.algorithmic_bytes() / (peak_hbm * 1e9), 3 * op.flops() / (tf * 1e12))
            t_meas = fam_t[dom] * 1e-3
            return {"bound": "hbm|tensor (per launch)", "kernel": dom, "achieved": round(ach, 2),
                    "unit": "TFLOP/s (fp32-equivalent)", "peak": None,
                    "peak_kind": f"per launch max(bytes / {peak_hbm} GB/s, 3 x flops / {tf:.0f} TF/s TF32)",
                    "frac": round(t_roof / t_meas, 4), "roofline_ms": round(t_roof * 1e3, 4),
                    "measured_ms": round(t_meas * 1e3, 4), "step_share": shares}
        return {"bound": "fp32 FFMA", "kernel": dom, "achieved": round(ach, 2), "unit": "TFLOP/s",
                "peak": round(FP32_FFMA_NOMINAL, 1), "peak_kind": "nominal 148 SMs x 128 FMA/clk x 1965 MHz",
                "frac": round(ach / FP32_FFMA_NOMINAL, 4), "step_share": shares}
    ach = fam_b[dom] / (fam_t[dom] * 1e-3) / 1e9
    return {"bound": "hbm", "kernel": dom, "achieved": round(ach, 1), "unit": "GB/s", "peak": peak_hbm,
            "peak_kind": "measured", "frac": round(ach / peak_hbm, 4), "step_share": shares,
            "avg_launch_ms": round(fam_t[dom] / fam_n[dom], 5), "launches_per_step": fam_n[dom]}


def cpu_sample(cfg, name, params):
    if name in ("heat_3d", "jacobi_2d"):
        return bench.cpu_baseline_stencil(name, params)
    from oracle import interp as O

    sp, scale = CPU_SAMPLES.get(cfg, (None, 1.0))
    sp = sp or params
    prog, b = W.load(name)
    inputs = W.make_inputs(name, prog, sp, 0)
    t0 = time.perf_counter()
    O.gradient(prog, b.backward, b.forwarding, b.required, inputs, sp)
    dt = (time.perf_counter() - t0) * scale
    return {"value": 1.0 / dt, "unit": "evals/s", "cores": 1, "kind": "port",
            "sample": f"oracle/interp.py (numpy) at {sp}, x{scale:g} to the full config: {dt:.2f}s/eval"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--only", default="")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--plans", action="store_true", help="also the config-scale checkpoint plans")
    args = ap.parse_args()
    peak, _ = bench.measured_peaks()
    fp64_peak = fp64_tensor_peak()
    only = [c for c in args.only.split(",") if c]
    for cfg, (name, params) in W.CONFIGS.items():
        if only and cfg not in only:
            continue
        if cfg.startswith("C2"):
            params = dict(params)  # literal 25 % budget is Infeasible; gradient at plan(None)
        prog, bundle = W.load(name)
        try:
            eng = Engine(prog, bundle, params)
        except Exception as exc:  # report, keep going
            print(json.dumps({"config": cfg, "error": f"{type(exc).__name__}: {exc}"}), flush=True)
            continue
        host = W.make_inputs(name, prog, params, 0)
        dev = {k: torch.from_numpy(v).cuda() for k, v in host.items()}
        for _ in range(args.warmup):
            eng.step(dev)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(args.steps):
            eng.step(dev)
        e.record()
        torch.cuda.synchronize()
        eng.check()
        ms = s.elapsed_time(e) / args.steps
        line = {"config": cfg, "workload": name, "params": params, "ms_per_step": round(ms, 5),
                "value": round(1000.0 / ms, 3), "unit": "evals/s", "ops_per_step": len(eng.exe.ops),
                "roofline": roofline(eng.exe, dev, peak, fp64_peak)}
        if not args.no_cpu:
            line["cpu_baseline"] = cpu_sample(cfg, name, params)
        print(json.dumps(line), flush=True)
        del eng, dev
        torch.cuda.empty_cache()
    if args.plans or "plans" in only:
        planned(args, peak, fp64_peak)


def planned(args, peak, fp64_peak):
    """The config-scale checkpoint plans (paper_2509_02197_b200/programs/plans,
    reference plan() decisions) through the engine, recompute fused and not."""
    from paper_2509_02197_b200.api import load_plan

    pdir = os.path.join(W.PROG_DIR, "plans")
    index = json.load(open(os.path.join(pdir, "index.json")))
    for cid, meta in index.items():
        for fuse in ("1", "0"):
            os.environ["GFB_FUSE_RECOMPUTE"] = fuse
            pb = load_plan(os.path.join(pdir, cid))
            params = meta["params"]
            eng = Engine(None, params=params, plan=pb)
            host = W.make_inputs(meta["workload"], pb.forward, params, 0)
            dev = {k: torch.from_numpy(v).cuda() for k, v in host.items()}
            for _ in range(args.warmup):
                eng.step(dev)
            torch.cuda.synchronize()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            for _ in range(args.steps):
                eng.step(dev)
            e.record()
            torch.cuda.synchronize()
            eng.check()
            ms = s.elapsed_time(e) / args.steps
            print(json.dumps({"config": "plan:" + cid, "fused_recompute": fuse == "1", "ms_per_step": round(ms, 5),
                              "value": round(1000.0 / ms, 3), "unit": "evals/s", "ops_per_step": len(eng.exe.ops),
                              "payload_peak": eng.exe.payload_peak, "t_star": meta["t_star"],
                              "limit_bytes": meta["limit_bytes"], "decisions": meta["decisions"],
                              "roofline": roofline(eng.exe, dev, peak, fp64_peak)}), flush=True)
            del eng, dev
            torch.cuda.empty_cache()
    os.environ.pop("GFB_FUSE_RECOMPUTE", None)


if __name__ == "__main__":
    main()
