"""Per-launch timing table (1 GPU): every op of every config's gradient step
with its algorithmic bytes and achieved GB/s (or TFLOP/s for contractions).

    python tools/op_table.py [--only C4/softmax,...] > gpurun_out/ops.txt
"""
from __future__ import annotations

import argparse
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import torch  # noqa: E402

from paper_2509_02197_b200 import Engine, workloads as W  # noqa: E402


def describe(op):
    bufs = []
    for b in list(op.reads) + list(op.writes):
        s = f"{b.name}{list(b.shape)}"
        if s not in bufs:
            bufs.append(s)
    extra = ""
    for k in ("M", "N", "K"):
        if hasattr(op, k):
            extra += f" {k}={getattr(op, k)}"
    return type(op).__name__ + extra + " " + " ".join(bufs)[:150]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="")
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    only = [c for c in args.only.split(",") if c]
    for cfg, (name, params) in W.CONFIGS.items():
        if only and cfg not in only:
            continue
        if not only and cfg == "C5/heat_3d":
            continue
        prog, bundle = W.load(name)
        eng = Engine(prog, bundle, params)
        host = W.make_inputs(name, prog, params, 0)
        dev = {k: torch.from_numpy(v).cuda() for k, v in host.items()}
        for _ in range(3):
            eng.step(dev)
        torch.cuda.synchronize()
        best = None
        for _ in range(args.reps):
            rows = eng.exe.timed_eager(dev)
            best = rows if best is None else [(f, o, min(m, bm)) for (f, o, m), (_, _, bm) in zip(rows, best)]
        tot = sum(m for _, _, m in best)
        print(f"== {cfg} {params}: {len(best)} launches, {tot:.4f} ms eager sum", flush=True)
        for k, (fam, op, ms) in enumerate(best):
            nb = op.algorithmic_bytes()
            line = f"  {k:3d} {fam:14s} {ms * 1e3:9.1f} us {nb / 1e6:9.2f} MB {nb / (ms * 1e-3) / 1e9:7.0f} GB/s"
            if hasattr(op, "flops"):
                line += f" {op.flops() / (ms * 1e-3) / 1e12:6.2f} TF/s"
            print(line + "  " + describe(op), flush=True)
        del eng, dev
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
