"""Turn one tools/capture_profiles.sh run (gpurun_out/) into the committed
profiles/ summaries for a round:

    python tools/summarize_profiles.py r01

writes profiles/<tag>_bench.jsonl, _configs.jsonl, _ops.txt, _pytest_gpu.log,
_launches_summary.txt, _ncu_star_pair.txt and profiles/ncu_traffic.json (the
DRAM bytes per launch bench.py reports as roofline.traffic).
"""
from __future__ import annotations

import csv
import io
import json
import os
import shutil
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(REPO, "gpurun_out")
PROF = os.path.join(REPO, "profiles")
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import ncu_rep  # noqa: E402


def launches(tag):
    path = os.path.join(OUT, "launches.csv")
    if not os.path.exists(path):
        return
    lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    rows = list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))
    agg = {}
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"]
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        us = v / 1000.0 if unit == "ns" else (v * 1000.0 if unit == "ms" else v)
        n, t = agg.get(name, (0, 0.0))
        agg[name] = (n + 1, t + us)
    tot = sum(t for _, t in agg.values()) or 1.0
    with open(os.path.join(PROF, f"{tag}_launches_summary.txt"), "w") as f:
        f.write("ncu --metrics gpu__time_duration.sum --clock-control none, "
                "python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e (every launch of the run;\n"
                "cold-cache serialised times: compare shares, not absolutes)\n")
        f.write(f"{'kernel':90s} {'launches':>8s} {'total_us':>12s} {'avg_us':>10s} {'share':>6s}\n")
        for name, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
            f.write(f"{name[:90]:90s} {n:8d} {t:12.1f} {t / n:10.2f} {t / tot:6.3f}\n")


def ncu_full(tag):
    rep = os.path.join(OUT, "prof_top.ncu-rep")
    if not os.path.exists(rep):
        return
    lines, traffic = ncu_rep.summarize(rep)
    out = ["ncu --set full --clock-control none --import-source on -k regex:star_pair --launch-skip 1 -c 4 "
           "python tools/prof_stencil.py heat_3d 512 4", ""] + lines
    with open(os.path.join(PROF, f"{tag}_ncu_star_pair.txt"), "w") as f:
        f.write("\n".join(out))
    with open(os.path.join(PROF, "ncu_traffic.json"), "w") as f:
        json.dump({"star_pair": {"dram_bytes_per_launch": sum(traffic) / len(traffic),
                                 "launches": len(traffic),
                                 "source": f"profiles/{tag}_ncu_star_pair.txt (dram__bytes_read.sum + "
                                           "dram__bytes_write.sum, heat_3d 512^3, launches 1-4: steady forward and adjoint timesteps)"}},
                  f, indent=1)


def ncu_lines(tag):
    """Per-source-line instruction / stall attribution of the captured
    star-pair launches (tools/ncu_lines.py over nvdisasm's line table)."""
    rep = os.path.join(OUT, "prof_top.ncu-rep")
    obj = os.path.join(REPO, "build", "obj", "star_tma.o")
    if not (os.path.exists(rep) and os.path.exists(obj)):
        return
    import tempfile

    tmp = tempfile.mkdtemp()
    src_csv = os.path.join(tmp, "src.csv")
    with open(src_csv, "w") as f:
        subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], stdout=f,
                       stderr=subprocess.DEVNULL)
    subprocess.run(["cuobjdump", "-xelf", "all", obj], cwd=tmp, capture_output=True)
    cubins = [c for c in os.listdir(tmp) if c.endswith(".cubin")]
    sass = os.path.join(tmp, "all.sass")
    with open(sass, "w") as f:
        subprocess.run(["nvdisasm", "-g", "-c"] + [os.path.join(tmp, c) for c in cubins], stdout=f)
    kernels = [r.split('"')[3] for r in open(src_csv) if r.startswith('"Kernel Name"')]
    out = []
    src = os.path.join(REPO, "paper_2509_02197_b200", "csrc", "star_tma.cu")
    seen = set()
    for k, name in enumerate(kernels):
        modes = name.split("(int)")[-1].split(">")[0]
        if modes in seen:
            continue
        seen.add(modes)
        mangled = f"_ZN3gfb6tile3220star_pair_tma_kernelIdLb1ELi{modes}EEEv14CUtensorMap_stNS_11StarPairDevE"
        r = subprocess.run([sys.executable, os.path.join(REPO, "tools", "ncu_lines.py"), mangled, sass, src_csv,
                            str(k), src, "140", "900"], capture_output=True, text=True)
        lines = r.stdout.splitlines()
        body = [l for l in lines[2:] if l.strip() and float(l.split()[0]) >= 2.0]
        out += [f"== {name} (MODES {modes}): M warp instructions, stall samples, source line", *lines[:2], *body, ""]
    with open(os.path.join(PROF, f"{tag}_ncu_star_lines.txt"), "w") as f:
        f.write("\n".join(out))


def ncu_gemm(tag):
    """The mlp GEMM captures (tools/lab/mm_one.py) and the nine-shape timing
    table (tools/lab/mm_time.py)."""
    reps = sorted(f for f in os.listdir(OUT) if f.startswith("gemm_") and f.endswith(".ncu-rep"))
    if not reps:
        return
    out = []
    t = os.path.join(OUT, "mm_time.log")
    if os.path.exists(t):
        out += ["tools/lab/mm_time.py (graph replay, median of 30):", open(t).read(), ""]
    for r in reps:
        shape = r[len("gemm_"):-len(".ncu-rep")].replace("_", " ")
        out.append(f"ncu --set full -k regex:sgemm_tma python tools/lab/mm_one.py {shape}")
        out += ncu_rep.summarize(os.path.join(OUT, r))[0]
    with open(os.path.join(PROF, f"{tag}_ncu_gemm.txt"), "w") as f:
        f.write("\n".join(out))


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
    os.makedirs(PROF, exist_ok=True)
    lines = []
    for name in ("bench.jsonl", "bench_ref.jsonl"):
        p = os.path.join(OUT, name)
        if os.path.exists(p):
            lines += [l for l in open(p).read().splitlines() if l.startswith("{")]
    if lines:
        open(os.path.join(PROF, f"{tag}_bench.jsonl"), "w").write("\n".join(lines) + "\n")
    p = os.path.join(OUT, "bench_slab1.jsonl")
    if os.path.exists(p):
        keep = [l for l in open(p).read().splitlines() if l.startswith("{")]
        open(os.path.join(PROF, f"{tag}_bench_slab1.jsonl"), "w").write("\n".join(keep) + "\n")
    for src, dst in (("configs.jsonl", f"{tag}_configs.jsonl"), ("ops.txt", f"{tag}_ops.txt"),
                     ("pytest_gpu.log", f"{tag}_pytest_gpu.log")):
        if os.path.exists(os.path.join(OUT, src)):
            shutil.copy(os.path.join(OUT, src), os.path.join(PROF, dst))
    launches(tag)
    ncu_full(tag)
    ncu_lines(tag)
    ncu_gemm(tag)
    print("\n".join(sorted(os.listdir(PROF))))


if __name__ == "__main__":
    main()
