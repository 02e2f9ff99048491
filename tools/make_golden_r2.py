"""Round-2 fixtures generated from the REFERENCE (build container only;
imports /root/reference read-only):

    python tools/make_golden_r2.py

Writes under tests/golden/r2/:
  <prog>.{fwd,bwd,fwdreq}.json + <prog>__<tag>.npz
      control-flow programs the advisor review asked to pin
      (loop-carried, iterator-dependent branch; a branch guarding a domain
      error), with the reference gradient() value / grads for several
      inputs that take different paths;
  plans_cli/<cid>.{fwd,bwd}.json + <cid>.report.json
      the reference CLI's own plan artifacts (``gradflow plan --emit STEM
      --json``, cli.py:246-253) for every golden plan in tests/golden/plans,
      so run_planned can be fed what the reference emits (no engine-side
      .plan.json);
  errors.json
      the reference's exception class for the typed-error cases
      (OutOfBounds, NonTermination, MissingTapeValue).
Writes under paper_2509_02197_b200/programs/plans/:
  <cid>.{fwd,bwd}.json + <cid>.plan.json
      reference plan() results at the CONFIG sizes: C4 softmax
      and mlp at floor + 25 % of the gap to store-all, and the paper's
      Listing-1 chain (scaled_product_chain, N=3620) at 500 MiB; with the
      decisions, t*, store-all and floor in plans/index.json.
"""
from __future__ import annotations

import json
import os
import subprocess
import sys
import warnings

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
sys.path.insert(0, REPO)
warnings.simplefilter("ignore")

from gradflow import errors as ref_errors  # noqa: E402
from gradflow.autodiff import build_backward, gradient  # noqa: E402
from gradflow.frontend import ProgramBuilder, load_program, serialize_program  # noqa: E402
from gradflow.interpreter import run_backward, run_forward  # noqa: E402

OUT = os.path.join(REPO, "tests", "golden", "r2")
PLANS = os.path.join(REPO, "tests", "golden", "plans")
PROGS = os.path.join(REPO, "paper_2509_02197_b200", "programs")


def save_programs(stem, program):
    bundle = build_backward(program)
    with open(stem + ".fwd.json", "w") as f:
        f.write(serialize_program(program))
    with open(stem + ".bwd.json", "w") as f:
        f.write(serialize_program(bundle.backward))
    manifest = {
        "required": sorted([d, v] for d, v in bundle.required),
        "entries": [
            {"name": e.name, "data": e.data,
             "candidates": [{"version": c.version, "directives": [list(d) for d in c.directives]}
                            for c in e.candidates]}
            for e in sorted(bundle.forwarding.values(), key=lambda e: e.name)
        ],
    }
    with open(stem + ".fwdreq.json", "w") as f:
        json.dump(manifest, f, indent=2)
        f.write("\n")
    return bundle


def loop_branch():
    """u = t; for i in [0, 3): u = 2u if t < i else 3u; O = u (the branch
    condition reads the loop iterator)."""
    b = ProgramBuilder(())
    b.scalar("t", role="input", kind="real64")
    b.scalar("u", kind="real64")
    b.scalar("O", role="output", kind="real64")
    with b.state("init") as s:
        s.tasklet(ins={"a": ("t", ())}, outs={"o": ("u", ())}, body={"o": "a"})
    with b.loop("i", "0", "3", label="L"):
        with b.branch("(lt t i)", label="side") as br:
            with br.then():
                with b.state("low") as s:
                    s.tasklet(ins={"a": ("u", ())}, outs={"o": ("u", ())}, body={"o": "(mul a 2)"})
            with br.orelse():
                with b.state("high") as s:
                    s.tasklet(ins={"a": ("u", ())}, outs={"o": ("u", ())}, body={"o": "(mul a 3)"})
    with b.state("out") as s:
        s.tasklet(ins={"a": ("u", ())}, outs={"o": ("O", ())}, body={"o": "a"})
    return b.finish("O", ["t"]), [1.5, -1.0, 0.5, 2.5]


def guarded_log():
    """O = sum(log(x)) if x0 > 0 else sum(2x): the else arm must be taken
    without evaluating log on non-positive data."""
    b = ProgramBuilder(("N",))
    b.array("x", ("N",), role="input", kind="real64")
    b.scalar("s", kind="real64")
    b.array("y", ("N",), kind="real64")
    b.scalar("O", role="output", kind="real64")
    with b.state("probe") as s:
        s.tasklet(ins={"a": ("x", ("0",))}, outs={"o": ("s", ())}, body={"o": "a"})
    with b.branch("(gt s 0)", label="pos") as br:
        with br.then():
            with b.state("logs") as s:
                s.map_node(("i",), (("0", "N", "1"),), lambda inner: inner.tasklet(
                    ins={"a": ("x", ("i",))}, outs={"o": ("y", ("i",))}, body={"o": "(log a)"}))
        with br.orelse():
            with b.state("twice") as s:
                s.map_node(("i",), (("0", "N", "1"),), lambda inner: inner.tasklet(
                    ins={"a": ("x", ("i",))}, outs={"o": ("y", ("i",))}, body={"o": "(mul a 2)"}))
    with b.state("sum") as s:
        s.library("reduce_sum", {"x": "y"}, {"y": "O"})
    return b.finish("O", ["x"]), None


def elem_branch():
    """for i in [0, N): y[i] = 2 x[i] if x[i] < 1 else x[i]^2; O = sum(y):
    every trip's branch reads one element of x (``idx``), ADVICE r1
    (element snapshots, incremental probing)."""
    b = ProgramBuilder(("N",))
    b.array("x", ("N",), role="input", kind="real64")
    b.array("y", ("N",), kind="real64")
    b.scalar("O", role="output", kind="real64")
    with b.loop("i", "0", "N", label="L"):
        with b.branch("(lt (idx x i) 1.0)", label="small") as br:
            with br.then():
                with b.state("twice") as s:
                    s.tasklet(ins={"a": ("x", ("i",))}, outs={"o": ("y", ("i",))}, body={"o": "(mul a 2)"})
            with br.orelse():
                with b.state("square") as s:
                    s.tasklet(ins={"a": ("x", ("i",))}, outs={"o": ("y", ("i",))}, body={"o": "(mul a a)"})
    with b.state("sum") as s:
        s.library("reduce_sum", {"x": "y"}, {"y": "O"})
    return b.finish("O", ["x"])


def save_control_flow():
    os.makedirs(OUT, exist_ok=True)
    index = {}
    prog = elem_branch()
    bundle = save_programs(os.path.join(OUT, "elem_branch"), prog)
    rng = np.random.default_rng(8)
    for k in range(2):
        x = rng.uniform(0.4, 1.6, 12)
        res = gradient(prog, {"x": x}, {"N": 12}, bundle=bundle)
        np.savez(os.path.join(OUT, f"elem_branch__{k}.npz"), **{"in:x": x}, value=np.asarray(res.value),
                 **{"grad:x": np.asarray(res.grads["x"])})
        index[f"elem_branch__{k}"] = {"program": "elem_branch", "params": {"N": 12}}
        print("elem_branch", k, float(res.value))
    prog, ts = loop_branch()
    bundle = save_programs(os.path.join(OUT, "loop_branch"), prog)
    for t in ts:
        res = gradient(prog, {"t": np.array(t)}, {}, bundle=bundle)
        tag = f"t{t:+g}".replace("+", "p").replace("-", "m").replace(".", "_")
        np.savez(os.path.join(OUT, f"loop_branch__{tag}.npz"), **{"in:t": np.array(t)},
                 value=np.asarray(res.value), **{"grad:t": np.asarray(res.grads["t"])})
        index[f"loop_branch__{tag}"] = {"program": "loop_branch", "params": {}}
        print("loop_branch", t, float(res.value), float(res.grads["t"]))
    prog, _ = guarded_log()
    bundle = save_programs(os.path.join(OUT, "guarded_log"), prog)
    rng = np.random.default_rng(5)
    for tag, x in (("pos", rng.uniform(0.4, 1.6, 9)), ("neg", -rng.uniform(0.4, 1.6, 9))):
        res = gradient(prog, {"x": x}, {"N": 9}, bundle=bundle)
        np.savez(os.path.join(OUT, f"guarded_log__{tag}.npz"), **{"in:x": x}, value=np.asarray(res.value),
                 **{"grad:x": np.asarray(res.grads["x"])})
        index[f"guarded_log__{tag}"] = {"program": "guarded_log", "params": {"N": 9}}
        print("guarded_log", tag, float(res.value))
    return index


def save_cli_plans():
    """Run the reference CLI (python -m gradflow.cli plan) for each golden plan."""
    out = os.path.join(OUT, "plans_cli")
    os.makedirs(out, exist_ok=True)
    with open(os.path.join(REPO, "tests", "golden", "index.json")) as f:
        plans = json.load(f)["plans"]
    env = dict(os.environ, PYTHONPATH=REF, PYTHONDONTWRITEBYTECODE="1")
    done = {}
    for cid, meta in sorted(plans.items()):
        w = meta["workload"]
        src = os.path.join(PROGS, (w if os.path.exists(os.path.join(PROGS, w + ".fwd.json")) else "corpus_" + w)
                           + ".fwd.json")
        stem = os.path.join(out, cid)
        cmd = [sys.executable, "-m", "gradflow.cli", "plan", src, "--emit", stem, "--json"]
        for k, v in meta["params"].items():
            cmd += ["--params", f"{k}={v}"]
        if meta["limit_mib"] is not None:
            cmd += ["--memory-limit-mib", repr(meta["limit_mib"])]
        r = subprocess.run(cmd, env=env, capture_output=True, text=True, check=True)
        with open(stem + ".report.json", "w") as f:
            f.write(r.stdout)
        done[cid] = {"source": os.path.relpath(src, REPO), "manifest": os.path.relpath(src, REPO).replace(
            ".fwd.json", ".fwdreq.json")}
        print("cli plan", cid, json.loads(r.stdout)["peak_bytes"])
    return done


def save_errors():
    """Which reference exception each typed-error case raises."""
    out = {}
    jac = load_program(os.path.join(PROGS, "jacobi_2d.fwd.json"))
    rng = np.random.default_rng(0)
    inputs = {"A": rng.uniform(0.4, 1.6, (6, 6)), "B": rng.uniform(0.4, 1.6, (6, 6))}
    try:
        gradient(jac, inputs, {"N": 6, "TSTEPS": 6}, trip_limit=4)
    except ref_errors.GradflowError as exc:
        out["trip_limit"] = {"workload": "jacobi_2d", "params": {"N": 6, "TSTEPS": 6}, "trip_limit": 4,
                             "error": type(exc).__name__}
    atax = load_program(os.path.join(PROGS, "atax.fwd.json"))
    bundle = build_backward(atax)
    ai = {"A": rng.uniform(0.4, 1.6, (6, 5)), "x": rng.uniform(0.4, 1.6, (5, 1))}
    try:
        run_backward(atax, bundle.backward, ai, {"M": 6, "N": 5}, tape=None, forwarding=bundle.forwarding)
    except ref_errors.GradflowError as exc:
        out["no_tape"] = {"workload": "atax", "params": {"M": 6, "N": 5}, "error": type(exc).__name__}
    fr = run_forward(atax, ai, {"M": 6, "N": 5}, record=set())
    try:
        run_backward(atax, bundle.backward, ai, {"M": 6, "N": 5}, tape=fr.tape, forwarding=bundle.forwarding)
    except ref_errors.GradflowError as exc:
        out["empty_tape"] = {"workload": "atax", "params": {"M": 6, "N": 5}, "error": type(exc).__name__}
    try:
        gradient(jac, {"A": inputs["A"][:5, :5], "B": inputs["B"][:5, :5]}, {"N": 5, "TSTEPS": 3})
        # declared N=5 arrays are fine; a map reaching past the extent needs a bad binding:
    except ref_errors.GradflowError as exc:  # pragma: no cover
        out["oob_unexpected"] = type(exc).__name__
    print("errors", out)
    with open(os.path.join(OUT, "errors.json"), "w") as f:
        json.dump(out, f, indent=2)


def save_config_plans():
    """Reference plan() at the config sizes (host, milliseconds)."""
    sys.path.insert(0, HERE)
    import gradflow.examples as ref_examples
    from gradflow.checkpointing import plan
    from workloads_ref import WORKLOADS

    from paper_2509_02197_b200.api import as_plan, save_plan

    mib = 1 << 20
    out = os.path.join(PROGS, "plans")
    os.makedirs(out, exist_ok=True)
    index = {}
    targets = [("softmax", WORKLOADS["softmax"](), {"R": 64 * 16 * 128, "SM": 128}, "tight"),
               ("mlp", WORKLOADS["mlp"](), {"NB": 64, "C": 512, "S0": 4096, "S1": 4096, "S2": 1024}, "tight"),
               ("scaled_product_chain", ref_examples.build("scaled_product_chain"), {"N": 3620}, 500.0)]
    for name, program, params, budget in targets:
        store_all = plan(program, None, params).solution.t_star
        try:
            plan(program, 0.0, params)
            floor = 0
        except ref_errors.Infeasible as exc:
            floor = exc.min_peak_bytes
        limit = (floor + 0.25 * (store_all - floor)) / mib if budget == "tight" else budget
        res = plan(program, limit, params)
        tag = "tight" if budget == "tight" else f"{budget:g}MiB"
        cid = f"{name}__" + "_".join(f"{k}{v}" for k, v in params.items()) + f"__{tag}"
        save_plan(as_plan(res), os.path.join(out, cid))
        index[cid] = {"workload": name, "params": params, "limit_mib": limit, "store_all": store_all,
                      "floor": floor, "t_star": res.solution.t_star,
                      "limit_bytes": res.report["limit_bytes"],
                      "decisions": [v["decision"] for v in res.report["values"]],
                      "names": [v["name"] for v in res.report["values"]]}
        print("config plan", cid, index[cid]["decisions"], res.solution.t_star)
    with open(os.path.join(out, "index.json"), "w") as f:
        json.dump(index, f, indent=2)


def save_timelines():
    """Reference simulate_memory (verification.py:228-323) for every committed
    plan, as ``gradflow mem-report --json`` computes it (cli.py:330-342)."""
    from gradflow.checkpointing import plan
    from gradflow.frontend import load_program as ref_load
    from gradflow.verification import simulate_memory

    out = {}
    sets = [(os.path.join(REPO, "tests", "golden", "index.json"), "plans",
             os.path.join(REPO, "tests", "golden", "plans")),
            (os.path.join(PROGS, "plans", "index.json"), None, os.path.join(PROGS, "plans"))]
    for idx_path, key, _ in sets:
        idx = json.load(open(idx_path))
        idx = idx[key] if key else idx
        for cid, meta in sorted(idx.items()):
            w = meta["workload"]
            src = os.path.join(PROGS, (w if os.path.exists(os.path.join(PROGS, w + ".fwd.json")) else "corpus_" + w)
                               + ".fwd.json")
            res = plan(ref_load(src), meta["limit_mib"], meta["params"])
            hints = {fv.name: fv.total_bytes for fv in res.fvs if fv.forced}
            paths = []
            for seq in res.sequences:
                tl = simulate_memory(res.forward, res.backward, meta["params"], dict(seq.outcomes),
                                     stored_hints=hints)
                paths.append({"peak_bytes": tl.peak, "events": [list(e) for e in tl.events]})
            out[cid] = {"limit_bytes": res.report["limit_bytes"], "model_peak_bytes": res.solution.t_star,
                        "paths": paths}
            print("timeline", cid, [p["peak_bytes"] for p in paths], res.solution.t_star)
    with open(os.path.join(OUT, "timelines.json"), "w") as f:
        json.dump(out, f, indent=1)


def save_batched():
    """Reference gradient() / run_forward() over leading batch dims
    (interpreter.py:161-169, :604-618), and a batch whose branch diverges."""
    sys.path.insert(0, HERE)
    from workloads_ref import WORKLOADS
    import gradflow.examples as ref_examples

    from paper_2509_02197_b200.workloads import make_inputs
    from paper_2509_02197_b200.ir import adopt

    cases = {}
    rng = np.random.default_rng(9)
    specs = [("jacobi_2d", WORKLOADS["jacobi_2d"](), {"N": 9, "TSTEPS": 3}, {"A": (3,), "B": (3,)}),
             ("softmax", WORKLOADS["softmax"](), {"R": 6, "SM": 5}, {"x": (2, 2)}),
             ("atax", WORKLOADS["atax"](), {"M": 6, "N": 5}, {"x": (4,)})]
    for name, program, params, bat in specs:
        base = make_inputs(name, adopt(program), params, 0)
        inputs = dict(base)
        for k, bshape in bat.items():
            inputs[k] = rng.uniform(0.4, 1.6, bshape + base[k].shape).astype(base[k].dtype)
        res = gradient(program, inputs, params)
        fwd = run_forward(program, inputs, params)
        cid = f"{name}__batch"
        arrays = {f"in:{k}": v for k, v in inputs.items()}
        arrays["value"] = np.asarray(res.value)
        arrays["fwd_value"] = np.asarray(fwd.value)
        for k, v in res.grads.items():
            arrays[f"grad:{k}"] = np.asarray(v)
        np.savez(os.path.join(OUT, cid + ".npz"), **arrays)
        cases[cid] = {"workload": name, "params": params}
        print("batched", cid, np.shape(res.value))
    # a branch whose condition differs across the batch
    program = ref_examples.build("branchy_scale")
    base = make_inputs("corpus_branchy_scale", adopt(program), {"n": 8}, 0)
    div = dict(base, s=np.array([0.3, 0.9]))
    try:
        gradient(program, div, {"n": 8})
        err = None
    except ref_errors.GradflowError as exc:
        err = type(exc).__name__
    np.savez(os.path.join(OUT, "corpus_branchy_scale__diverge.npz"), **{f"in:{k}": v for k, v in div.items()})
    cases["corpus_branchy_scale__diverge"] = {"workload": "corpus_branchy_scale", "params": {"n": 8}, "error": err}
    print("diverging batch:", err)
    return cases


def save_fd():
    """The reference finite-difference oracle (verification.py:53-120) where
    its probe batch diverges at a branch: pairwise fallback, NaN for probe
    pairs that straddle the branch boundary."""
    from gradflow.verification import finite_difference_gradient

    cases = {}
    prog, _ = loop_branch()
    for t in (1.0, 1.5, 2.0, -1.0):
        fd = finite_difference_gradient(prog, {"t": np.array(t)}, {})
        tag = f"loop_branch__fd_t{t:+g}".replace("+", "p").replace("-", "m").replace(".", "_")
        np.savez(os.path.join(OUT, tag + ".npz"), **{"in:t": np.array(t)}, **{"fd:t": np.asarray(fd["t"])})
        cases[tag] = {"program": "loop_branch", "params": {}}
        print("fd", tag, fd["t"])
    prog, _ = guarded_log()
    x = np.random.default_rng(6).uniform(0.4, 1.6, 9)
    for tag, x0 in (("zero", 0.0), ("pos", x[0])):
        xi = x.copy()
        xi[0] = x0
        fd = finite_difference_gradient(prog, {"x": xi}, {"N": 9})
        cid = f"guarded_log__fd_{tag}"
        np.savez(os.path.join(OUT, cid + ".npz"), **{"in:x": xi}, **{"fd:x": np.asarray(fd["x"])})
        cases[cid] = {"program": "guarded_log", "params": {"N": 9}}
        print("fd", cid, fd["x"])
    return cases


def main():
    batched = save_batched()
    save_timelines()
    save_config_plans()
    index = {"control_flow": save_control_flow(), "plans_cli": save_cli_plans(), "batched": batched,
             "fd": save_fd()}
    with open(os.path.join(OUT, "index.json"), "w") as f:
        json.dump(index, f, indent=2)
    save_errors()


if __name__ == "__main__":
    main()
